"""Experiment build: relink libb2dwt with some units recompiled with extra flags.

    python tools/build_variant.py NAME --units fused2_cdf97_nssplit_fwd --flags=-DB2DWT_F2_NOSYNC

writes paper_1705_08266_b200/libb2dwt_NAME.so (load it with B2DWT_LIB=...).
Units are object names from build/link_manifest.txt (without .o).
"""
import argparse, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_08266_b200 import build as B

ap = argparse.ArgumentParser()
ap.add_argument("name")
ap.add_argument("--units", required=True)
ap.add_argument("--flags", default="")
ap.add_argument("--link-only", action="store_true", help="reuse build_exp/NAME objects")
a = ap.parse_args()
objs = open(os.path.join(B.BUILD, "link_manifest.txt")).read().split()
out_dir = os.path.join(B.ROOT, "build_exp", a.name)
os.makedirs(out_dir, exist_ok=True)
new = []
for o in objs:
    unit = os.path.basename(o)[:-2]
    if unit not in a.units.split(","):
        new.append(o)
        continue
    tag = unit[2:] if unit.startswith("v_") else unit  # build.py names v_<prog>_<vid> logs ptxas_<prog>_<vid>
    log = open(os.path.join(B.BUILD, f"ptxas_{tag}.log")).readline().split()
    cmd = log[:log.index("-c")] + a.flags.split() + log[log.index("-c"):]
    dst = os.path.join(out_dir, unit + ".o")
    cmd[cmd.index("-o") + 1] = dst
    if a.link_only and os.path.exists(dst):
        new.append(dst)
        continue
    print(" ".join(cmd[-6:]), flush=True)
    subprocess.run(cmd, check=True, capture_output=True)
    new.append(dst)
lib = os.path.join(B.HERE, f"libb2dwt_{a.name}.so")
subprocess.run([B.nvcc(), "-shared", *B.ARCH, "-o", lib, *new], check=True)
print(lib)
