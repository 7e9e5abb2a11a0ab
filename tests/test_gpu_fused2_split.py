"""Work-split paths of the two-level fused kernel that only large launches take
(f2_work_space, csrc/fused2_kernel.cuh): static super-strip slices over a
whole multiple of the super-strip count (and the CTAs beyond it starting on
the dynamic queue), fewer CTAs than super-strips, the dynamic edge units, the
per-super-strip dynamic row space with guided or fixed claims.

At test sizes every fused launch is small (all static), so each case runs in a
subprocess with the env overrides that force the large-launch path
(B2DWT_F2_DYN_MIN, B2DWT_F2_MIN_ROWS: they are read once per process) and
checks the pair bit-identical to two single-level launches, strict and fast.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (H, W): level-(l+1) rows x super-strips (224 level-l quads) vs the CTA count
# min(resident, ceil(total / B2DWT_F2_MIN_ROWS)) the overrides below give
SHAPES = [
    (2048, 8192),  # 19 super-strips x 512 rows; 98 CTAs at 100 rows: 95 static (5 per super-strip) + 3 dynamic-only
    (512, 32768),  # 74 super-strips x 128 rows; fewer CTAs than super-strips at 200 rows (range split)
    (1024, 1792),  # 4 super-strips x 256 rows; a whole multiple at 32 rows (8 per super-strip)
    (520, 900),    # ragged: 3 super-strips (the last partial), 130 rows
]

CASE = r"""
import json, sys, torch
from paper_1705_08266_b200 import CDF97, CDF53, Transform, build_scheme
shapes = json.loads(sys.argv[1])
bad = []
for plan, scheme in ((CDF97, "non-separable-split"), (CDF53, "separable-lifting")):
    for fast in (False, True):
        tr = Transform(build_scheme(scheme, plan), "single", fast=fast)
        for h, w in shapes:
            x = torch.rand((h, w), device="cuda", generator=torch.Generator(device="cuda").manual_seed(h + 3 * w))
            got = tr.forward2(x)
            if got is None:
                bad.append([scheme, fast, h, w, "refused"])
                continue
            ll0, hl0, lh0, hh0 = tr.forward(x)
            want = (hl0, lh0, hh0) + tuple(tr.forward(ll0.contiguous()))
            for i, (g, wv) in enumerate(zip(got[0] + got[1], want)):
                if not torch.equal(g, wv):
                    bad.append([scheme, fast, h, w, i, int((g != wv).sum())])
            for _ in range(3):  # the tail counter slot is reset by the last CTA: repeat launches
                again = tr.forward2(x)
                if not all(torch.equal(a, b) for a, b in zip(again[0] + again[1], got[0] + got[1])):
                    bad.append([scheme, fast, h, w, "repeat"])
                    break
print(json.dumps(bad))
"""

ENVS = {
    "slices-guided": {"B2DWT_F2_DYN_MIN": "1", "B2DWT_F2_MIN_ROWS": "100"},
    "all-dynamic": {"B2DWT_F2_DYN_MIN": "1", "B2DWT_F2_MIN_ROWS": "200", "B2DWT_F2_STATIC_FRAC": "0"},
    "fixed-chunks": {"B2DWT_F2_DYN_MIN": "1", "B2DWT_F2_MIN_ROWS": "32", "B2DWT_F2_STATIC_FRAC": "1000",
                     "B2DWT_F2_GUIDED": "0", "B2DWT_F2_TAIL_ROWS": "8"},
    "half-share": {"B2DWT_F2_DYN_MIN": "1", "B2DWT_F2_MIN_ROWS": "48", "B2DWT_F2_GUIDED": "2",
                   "B2DWT_F2_EDGE_ROWS": "3"},
}


@pytest.mark.parametrize("name", list(ENVS))
def test_large_launch_work_split_bit_identical(name):
    env = dict(os.environ, **ENVS[name])
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    p = subprocess.run([sys.executable, "-c", CASE, json.dumps(SHAPES)], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    bad = json.loads(p.stdout.strip().splitlines()[-1])
    assert bad == [], (name, bad)
