#!/usr/bin/env python
"""Benchmark: Gpixel/s of the 2-D CDF 9/7 forward DWT on B200 vs the HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3|c4|c5|c2|c1] [--arith strict|fast] [--bands K]

Default workload (BASELINE.json configs[2], the north-star target, "C3"):
one 16384x16384 float32 image, operation-reduced non-separable CDF 9/7
("non-separable-split") forward transform, 5-level pyramid, per GPU.  A step is
one replay of a CUDA graph holding the whole pyramid (6 launches: level 0 as
two footprint-bounded row bands, levels 1-3 streamed, level 4 tiled).  `e2e`
runs the same pyramid from pinned host memory to pinned host memory through
Transform.dwt_host.  Under torchrun (N > 1) every rank
transforms its own image: batch sharding, no data-path collective ("weak").

--config c4 : BASELINE configs[3], 1024 x 2048^2 images, non-separable CDF 9/7,
              1 level, batch-sharded over N GPUs ("strong", total work fixed).
--config c5 : BASELINE configs[4], one 65536^2 image, non-separable CDF 9/7,
              1 level, row strips over N GPUs with an NCCL halo exchange.
--config c2 : 4096^2, one line per scheme x wavelet x direction (parity sizes).
--config c1 : BASELINE configs[0], 1024^2 9/7 separable lifting, 1 level: device
              kernel, host-array call end to end, and the CPU oracle on the same image.

--impl reference times the reference algorithm's CPU implementation on this
box's host cores (the oracle port, oracle/dwt_oracle.c -- the reference itself
is Python and is not installable on the GPU box) on a bounded sample of the
same workload, and prints the same JSON line with "impl": "reference".

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpixel/s (and ns/pixel) for 2-D CDF 9/7 fwd DWT vs HBM roofline, 1/2/4/8 B200"
UNIT = "Gpixel/s"
SPEC_HBM_GBS = 8000.0


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic(key):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and "Active" in s[3 + i]
                          and "Not" not in s[3 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# -- CPU reference arm ----------------------------------------------------------------


def _cpu_model():
    """The host CPU model (lscpu's "Model name"), from /proc/cpuinfo."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _stock_reference_sample(config):
    """The UNMODIFIED reference (liftfuse, pip-installed into the git-ignored
    baseline/_ref) through its own timed region, liftfuse/bench.py:71-79:
    run_tiled on pre-deinterleaved components, TileConfig((256, 256),
    os.cpu_count()), median of 3 after one warm-up, iterated on LL for the
    pyramid.  Bounded sample: a quarter-side crop of the workload image (C3:
    4096^2, 5 levels).  Returns None when baseline/_ref is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "liftfuse")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        from liftfuse.engine import Image2D, TileConfig, compile_scheme, deinterleave, run_tiled
        from liftfuse.schemes import build_scheme
        from liftfuse.wavelets import CDF97
    except Exception as exc:  # pragma: no cover - broken install
        return {"unavailable": f"baseline/_ref import failed: {exc}"}
    n, levels, scheme = {"c1": (1024, 1, "separable-lifting"), "c4": (2048, 1, "non-separable-split"),
                         "c5": (4096, 1, "non-separable-split"), "c2": (4096, 1, "non-separable-split")}.get(
        config, (4096, 5, "non-separable-split"))
    threads = os.cpu_count() or 1
    prog = compile_scheme(build_scheme(scheme, CDF97))
    cfg = TileConfig((256, 256), threads)
    comps0 = deinterleave(Image2D.random(n, n, seed=0, precision="single"))

    def pyramid():  # seconds inside run_tiled
        comps, spent = comps0, 0.0
        for lvl in range(levels):
            t0 = time.perf_counter()
            out = run_tiled(prog, comps, cfg)
            spent += time.perf_counter() - t0
            if lvl + 1 < levels:
                comps = deinterleave(Image2D(out[0]))
        return spent

    pyramid()  # warm-up, excluded
    med = statistics.median(pyramid() for _ in range(3))
    return {"value": n * n / med / 1e9, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{n}x{n} f32, CDF 9/7 {scheme}, {levels} level(s): stock liftfuse run_tiled "
                      f"(TileConfig((256,256), {threads})), deinterleave between levels excluded",
            "ms_per_sample": med * 1e3}


def _cpu_sample(config, steps=1, warmup=0):
    """Time the oracle port on a bounded sample; returns (gpx_per_s, sample_desc, threads, per_step_s)."""
    import numpy as np

    from oracle import oracle
    from paper_1705_08266_b200 import CDF97, build_scheme, compile_scheme

    threads = os.cpu_count() or 1
    if config == "c3":
        n, levels, scheme = 16384, 5, "non-separable-split"
        desc = "the whole C3 workload: 16384x16384 f32, CDF 9/7 non-separable-split, 5-level pyramid"
        px = n * n
    elif config == "c4":
        n, levels, scheme = 2048, 1, "non-separable-split"
        desc = "2 of the 1024 C4 images (2048x2048 f32), CDF 9/7 non-separable-split, 1 level"
        px = 2 * n * n
    elif config == "c1":
        n, levels, scheme = 1024, 1, "separable-lifting"
        desc = "the whole C1 image (1024x1024 f32), CDF 9/7 separable-lifting, 1 level"
        px = n * n
    elif config == "c5":
        n, levels, scheme = 8192, 1, "non-separable-split"
        desc = "one 8192x8192 f32 block (1/64 of the C5 area), CDF 9/7 non-separable-split, 1 level"
        px = n * n
    else:
        n, levels, scheme = 4096, 1, "non-separable-split"
        desc = "4096x4096 f32, CDF 9/7 non-separable-split, 1 level"
        px = n * n
    prog = compile_scheme(build_scheme(scheme, CDF97))
    img = np.random.default_rng(0).random((n, n), dtype=np.float64).astype(np.float32)
    reps = 2 if config == "c4" else 1

    def one():
        for _ in range(reps):
            oracle.dwt(img, prog, levels, threads=threads)

    for _ in range(warmup):
        one()
    times = []
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        one()
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    return px / med / 1e9, desc, threads, med, times


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    steps = max(1, args.steps)
    gpx, desc, threads, med, times = _cpu_sample(args.config, steps=steps, warmup=min(args.warmup, 1))
    stock = _stock_reference_sample(args.config)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": gpx,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": med * 1e3,
        "higher_is_better": True,
        "scaling": "weak" if args.config == "c3" else "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (uniform [0,1), numpy PCG64 seed 0)",
        "config": {"workload": _workload_name(args.config), "sample": desc,
                   "same_config": args.config != "c4"},
        "cpu_baseline": {"value": gpx, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc,
                         "cpu_model": _cpu_model(), "stock_reference": stock},
        "e2e": {"value": gpx, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "value: oracle/dwt_oracle.c, the C restatement of liftfuse run_reference (bit-identical to the "
                "reference, pinned by tests/test_oracle.py), on all host threads; cpu_baseline.stock_reference: "
                "the unmodified liftfuse package (baseline/_ref) on a bounded sample",
    }
    print(json.dumps(line), flush=True)
    return 0


def _workload_name(config):
    return {
        "c3": "C3: 16384x16384 f32, CDF 9/7 non-separable-split (operation-reduced) forward, 5-level pyramid, per GPU",
        "c4": "C4: 1024 x 2048x2048 f32, CDF 9/7 non-separable-split forward, 1 level, batch-sharded",
        "c5": "C5: 65536x65536 f32, CDF 9/7 non-separable-split forward, 1 level, row strips + NCCL halo exchange",
        "c2": "C2: 4096x4096 f32, all schemes x CDF 5/3, 9/7 x fwd/inv, 1 level",
        "c1": "C1: 1024x1024 f32, CDF 9/7 separable-lifting forward, 1 level (the reference's CPU-runnable case)",
    }[config]


# -- GPU arm ------------------------------------------------------------------------------


def _dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if world > 1:
        # NCCL communicator setup in the log (which transport / NVLS the box uses)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        import datetime

        # a stuck collective raises instead of hanging the run
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), timeout=datetime.timedelta(seconds=300))
    return torch, dist, world, rank, local


def _barrier(torch, dist):
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()


def _max_over_ranks(torch, dist, x):
    if dist is None:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _launches(rows, cols, batch=1, levels=1):
    """Kernel launches of one request (mirrors b2dwt_host.cu: stream-kernel
    requests above B2DWT_MAX_LAUNCH_BYTES (512 MiB of f32 input) are split
    into batch chunks / row bands; levels of <= 512^2 quads run one tile launch)."""
    cap = int(os.environ.get("B2DWT_MAX_LAUNCH_BYTES", 512 << 20))
    total = 0
    for l in range(levels):
        r, c = rows >> l, cols >> l
        quads = batch * r * c
        if quads <= (1 << 18):
            total += 1
            continue
        parts = -(-quads * 16 // cap) if cap > 0 else 1
        parts = min(parts, batch) if batch > 1 else min(parts, max(1, r // 256))
        total += max(1, parts)
    return total


def _c3_launches(groups, n):
    """Kernel launches of one C3 pyramid: a fused level pair runs as row bands of
    <= 1 GiB of level-l input (b2dwt_host.cu run_fused2_pair), a single level
    as _launches counts it."""
    cap = int(os.environ.get("B2DWT_F2_MAX_LAUNCH_BYTES", 1 << 30))
    total = 0
    for a, b in groups:
        r = n >> (a + 1)
        if a == b:
            total += _launches(r, r, 1, 1)
        else:
            parts = -(-r * r * 16 // cap) if cap > 0 else 1
            total += max(1, min(parts, (r // 2) // 128))
    return total


def _time_graph(torch, dist, graph, steps, warmup):
    """K replays between barrier + synchronize; returns ms per step (max over ranks)."""
    for _ in range(max(3, warmup)):
        graph.replay()
    _barrier(torch, dist)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        graph.replay()
    t1.record()
    t1.synchronize()
    _barrier(torch, dist)
    return _max_over_ranks(torch, dist, t0.elapsed_time(t1)) / steps


def run_c3(args):
    torch, dist, world, rank, local = _dist_setup(args)
    from paper_1705_08266_b200 import CDF97, Transform, build_scheme

    n, levels = 16384, 5
    scheme = build_scheme("non-separable-split", CDF97)
    fast = args.arith == "fast"
    tr = Transform(scheme, "single", fast=fast)
    assert tr.fwd_plan.fused, "fused kernel not selected"
    gen = torch.Generator(device="cuda")
    gen.manual_seed(rank)
    x = torch.rand((n, n), device="cuda", generator=gen)
    # The product pyramid path: the whole 5-level pyramid is ONE CUDA graph of
    # one b2dwt_dwt call (levels 0+1 and 2+3 as two-level fused kernels, whose
    # LL bands never reach HBM, level 4 tiled; launches chained by
    # programmatic dependent launch).
    graph = tr.capture_dwt(x, levels)

    with ClockSampler(local) as clk:
        ms_step = _time_graph(torch, dist, graph, args.steps, args.warmup)
    del graph
    # launch-group breakdown: the same pyramid captured with external event
    # nodes bracketing every launch group (a fused level pair or a single
    # level; the events serialise the groups, so this graph is a little slower
    # than the timed one), K replays, events read after each
    ev_graph = tr.capture_dwt(x, levels, level_events=True)
    groups = ev_graph.groups
    per_level_runs = []
    for _ in range(args.warmup + args.steps):
        ev_graph.replay()
        torch.cuda.synchronize()
        per_level_runs.append(ev_graph.level_ms())
    per_level_runs = per_level_runs[args.warmup:]
    del ev_graph
    per_group = [statistics.median(r[g] for r in per_level_runs) for g in range(len(groups))]
    l0_ms = statistics.mean(r[0] for r in per_level_runs)
    # the other arithmetic mode, same protocol (reported beside the headline)
    other = Transform(scheme, "single", fast=not fast)
    other_graph = other.capture_dwt(x, levels)
    other_ms = _time_graph(torch, dist, other_graph, args.steps, args.warmup)
    del other_graph

    px = n * n * world
    value = px / (ms_step * 1e-3) / 1e9
    alg_bytes_step = 8 * n * n * sum(4.0 ** -l for l in range(levels))
    # dominant launch = the first group (levels 0+1 fused, or level 0 alone):
    # SURVEY 8(d) algorithmic bytes = 1 read + 1 write of every level's input
    # area it processes; the fused kernel's compulsory HBM bytes are smaller
    # (level 0's LL band never leaves the SM): read the image, write level 0's
    # HL/LH/HH and level 1's four planes
    g0a, g0b = groups[0]
    l0_bytes = 8 * n * n * sum(4.0 ** -l for l in range(g0a, g0b + 1))
    l0_compulsory = 4 * n * n * (1 + 0.75 + (0.25 if g0b > g0a else 0.25))
    peak, peak_src = _peaks()
    achieved = l0_bytes / (l0_ms * 1e-3) / 1e9

    # end to end through the public API with host (pinned) buffers
    e2e = _e2e_c3(torch, tr, n, levels, rank, dist, args)

    # the BASELINE scaling configs ride along at every N, so the driver's
    # N = 1, 2, 4, 8 runs give their strong-scaling curves beside the C3 line:
    # C4 (batch shards) and C5 (row strips + NCCL halo exchange), same ranks
    scale_keys = {}
    if not args.no_scale_configs:
        for key, fn in (("c4", _measure_c4), ("c5", _measure_c5)):
            torch.cuda.empty_cache()
            try:
                scale_keys[key] = fn(args, torch, dist, world, rank, local, e2e_sample=False)
            except Exception as exc:  # the C3 line must still be printed
                scale_keys[key] = {"error": repr(exc)[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        gpx, desc, threads, med, _ = _cpu_sample("c3")
        cpu = {"value": gpx, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc,
               "cpu_model": _cpu_model(), "stock_reference": _stock_reference_sample("c3")}

    strict_desc = "strict: bit-identical to the reference (separate IEEE mul/add, compiled term order)"
    fast_desc = "fast: FMA in the compiled term order, max err <= 1e-4 x input range (tests/test_gpu_parity.py)"
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(3, args.warmup),
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (torch.rand on device, seed = rank)",
            "config": {
                "workload": _workload_name("c3"),
                "image": [n, n],
                "levels": levels,
                "scheme": "non-separable-split",
                "wavelet": "cdf97",
                "arith": fast_desc if fast else strict_desc,
                "other_arith": {"mode": "strict" if fast else "fast", "value": px / (other_ms * 1e-3) / 1e9,
                                "ms_per_step": other_ms},
                "step": "one CUDA-graph replay of the 5-level pyramid (Transform.capture_dwt)",
                "l2": "input 1 GiB > 126 MB L2 per step; no flush",
                "parallelism": f"batch-shard x{world} (one image per GPU, no collective)",
                "ns_per_px": 1.0 / value,
                "launch_groups": [f"L{a}" if a == b else f"L{a}+L{b} fused" for a, b in groups],
                "ms_per_group": per_group,
                "alg_bytes_per_step": alg_bytes_step,
                "frac_of_8TBps": (alg_bytes_step / (ms_step * 1e-3) / 1e9) / SPEC_HBM_GBS,
            },
            "roofline": {
                "bound": "hbm",
                "kernel": ("fused2_kernel<cdf97_nssplit_fwd, f32>: levels 0+1 in one launch (16384^2 -> "
                           "HL/LH/HH 8192^2 + 4 x 4096^2; level 0's LL stays in shared memory)"
                           if g0b > g0a else
                           "stream_kernel<cdf97_nssplit_fwd, f32> level 0 (16384^2 -> 4 x 8192^2; two "
                           "footprint-bounded launches of 4096 quad rows)"),
                "achieved": achieved,
                "peak": peak,
                "peak_source": peak_src,
                "unit": "GB/s",
                "frac": achieved / peak,
                "traffic": _traffic(f"c3_group0_{args.arith}" if g0b > g0a else f"c3_level0_{args.arith}"),
                "alg_bytes_per_launch": l0_bytes,
                "alg_bytes_rule": "SURVEY 8(d): 8 B/px of every level the launch processes",
                "compulsory_bytes": l0_compulsory,
                "frac_compulsory": l0_compulsory / (l0_ms * 1e-3) / 1e9 / peak,
                "note": ("a fused pair's frac can exceed 1: the 8 B/px rule counts level l's LL write and level "
                         "l+1's re-read, which the fused kernel keeps in shared memory; frac_compulsory counts "
                         "only the bytes it must move") if g0b > g0a else None,
                "launch_ms": l0_ms,
                "timing": "event nodes around the first launch group inside the captured graph, mean over K replays",
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            "gpu_launches": args.steps * _c3_launches(groups, n),
        }
        line.update(scale_keys)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def _e2e_c3(torch, tr, n, levels, rank, dist, args):
    """Public-API pyramid with host buffers (Transform.dwt_host ->
    b2dwt_dwt_host): pinned H2D of the image, the pyramid, pinned D2H of every
    subband and the final LL, all inside the timed region.  The library cuts
    the image into row bands so the upload, the kernels and the download run
    concurrently (host_pipeline.cu)."""
    host_in = torch.empty((n, n), dtype=torch.float32).pin_memory()
    host_in.uniform_()
    details = [tuple(torch.empty((n >> (l + 1), n >> (l + 1)), dtype=torch.float32).pin_memory()
                     for _ in range(3)) for l in range(levels)]
    host_ll = torch.empty((n >> levels, n >> levels), dtype=torch.float32).pin_memory()

    def step():
        tr.dwt_host(host_in, levels, details=details, ll=host_ll, bands=args.bands, sync=False)

    steps = max(2, min(args.steps, 5))
    for _ in range(2):
        step()
    _barrier(torch, dist)
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        step()
    e.record()
    e.synchronize()
    ms = _max_over_ranks(torch, dist, s.elapsed_time(e) / steps)
    world = dist.get_world_size() if dist is not None else 1
    h2d = n * n * 4
    d2h = sum(t.numel() * 4 for d in details for t in d) + host_ll.numel() * 4
    return {"value": n * n * world / (ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "bands": args.bands,
            "api": "Transform.dwt_host (b2dwt_dwt_host) with pinned host buffers: H2D, pyramid and D2H inside "
                   "the timed region, overlapped in row bands"}


def run_c4(args):
    torch, dist, world, rank, local = _dist_setup(args)
    line = _measure_c4(args, torch, dist, world, rank, local, e2e_sample=True)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def _measure_c4(args, torch, dist, world, rank, local, e2e_sample=True):
    """C4: 1024 x 2048^2 images batch-sharded over the ranks (no collective)."""
    from paper_1705_08266_b200 import CDF97, Transform, build_scheme
    from paper_1705_08266_b200.distributed import shard_range

    n_img, n = 1024, 2048
    lo, hi = shard_range(n_img, rank, world)
    mine = hi - lo
    chunk = 64
    tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=(args.arith == "fast"))
    x = torch.empty((mine, n, n), device="cuda")
    for i in range(0, mine, chunk):
        x[i:i + chunk].uniform_()
    outs = tuple(torch.empty((mine, n // 2, n // 2), device="cuda") for _ in range(4))

    def step():  # one API call; the library splits it into footprint-bounded launches
        tr.forward(x, out=outs)

    for _ in range(max(3, args.warmup)):
        step()
    with ClockSampler(local) as clk:
        _barrier(torch, dist)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            step()
        e.record()
        e.synchronize()
        _barrier(torch, dist)
    ms = _max_over_ranks(torch, dist, s.elapsed_time(e)) / args.steps
    value = n_img * n * n / (ms * 1e-3) / 1e9
    peak, src = _peaks()
    # end to end on a 128-image sample per rank: pinned host batch in, pinned
    # subbands out, chunked upload / kernel / download overlap
    # (Transform.forward_host_batch); 2 GiB each way per rank
    del x, outs
    torch.cuda.empty_cache()
    if not e2e_sample:
        return {"value": value, "unit": UNIT, "ms_per_step": ms, "scaling": "strong", "images_per_gpu": mine,
                "roofline_frac": 8.0 * mine * n * n / (ms * 1e-3) / 1e9 / peak, "clocks": clk.summary()}
    sample = min(mine, 128)
    host_in = torch.empty((sample, n, n), dtype=torch.float32).pin_memory()
    host_in.uniform_()
    host_out = tuple(torch.empty((sample, n // 2, n // 2), dtype=torch.float32).pin_memory() for _ in range(4))
    for _ in range(2):
        tr.forward_host_batch(host_in, out=host_out, sync=False)
    _barrier(torch, dist)
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es.record()
    for _ in range(3):
        tr.forward_host_batch(host_in, out=host_out, sync=False)
    ee.record()
    ee.synchronize()
    e2e_ms = _max_over_ranks(torch, dist, es.elapsed_time(ee)) / 3
    e2e = {"value": sample * world * n * n / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": sample * n * n * 4, "d2h_bytes_per_step": sample * n * n * 4, "ms_per_step": e2e_ms,
           "sample": f"{sample} images per rank", "api": "Transform.forward_host_batch (pinned host batch in and out)"}
    achieved = 8.0 * mine * n * n / (ms * 1e-3) / 1e9
    return {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (uniform on device)",
            "config": {"workload": _workload_name("c4"), "parallelism": f"batch-shard x{world}",
                       "images_per_gpu": mine, "arith": args.arith,
                       "launches": "one forward() per step, split by the library into <= 512 MiB-input launches"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "peak_source": src, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None},
            "cpu_baseline": None, "e2e": e2e, "clocks": clk.summary(),
            "gpu_launches": args.steps * _launches(n // 2, n // 2, mine),
        }


def run_c5(args):
    torch, dist, world, rank, local = _dist_setup(args)
    line = _measure_c5(args, torch, dist, world, rank, local, e2e_sample=True)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def _measure_c5(args, torch, dist, world, rank, local, e2e_sample=True):
    """C5: one 65536^2 image in row strips over the ranks, NCCL halo exchange."""
    from paper_1705_08266_b200 import CDF97, Transform, build_scheme
    from paper_1705_08266_b200.distributed import RowStrips

    n = 65536
    tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=(args.arith == "fast"))
    strips = RowStrips(n, n, rank, world, tr.cone[:2], levels=1)
    buf = strips.allocate(lambda shape: torch.empty(shape, device="cuda"))
    own = strips.owned(buf)
    for i in range(0, own.shape[0], 4096):
        own[i:i + 4096].uniform_()
    L = strips.layout(0)
    outs = tuple(torch.empty((L.rows // 2, n // 2), device="cuda") for _ in range(4))

    def band_forward(band, band_row0, height, r0, r1, out):
        tr.forward_rows(band, band_row0, height, r0, r1, out=out)

    def step():
        strips.forward(band_forward, buf, outs, 0, None, overlap=True)

    for _ in range(max(3, args.warmup)):
        step()
    with ClockSampler(local) as clk:
        _barrier(torch, dist)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            step()
        e.record()
        e.synchronize()
        _barrier(torch, dist)
    ms = _max_over_ranks(torch, dist, s.elapsed_time(e)) / args.steps
    value = n * n / (ms * 1e-3) / 1e9
    interior, edges = strips._bands(0)
    # end to end on a 16384 x 65536 sample per rank (4 GiB each way): pinned
    # host rows in, pinned subbands out, through the banded host pipeline
    del buf, own, outs
    torch.cuda.empty_cache()
    peak, src = _peaks()
    if not e2e_sample:
        return {"value": value, "unit": UNIT, "ms_per_step": ms, "scaling": "strong",
                "rows_per_gpu": L.rows, "halo_rows_per_side_px": [L.halo_top, L.halo_bot],
                "roofline_frac": 8.0 * L.rows * n / (ms * 1e-3) / 1e9 / peak, "clocks": clk.summary()}
    sh = 16384
    host_in = torch.empty((sh, n), dtype=torch.float32).pin_memory()
    host_in.uniform_()
    det = [tuple(torch.empty((sh // 2, n // 2), dtype=torch.float32).pin_memory() for _ in range(3))]
    host_ll = torch.empty((sh // 2, n // 2), dtype=torch.float32).pin_memory()
    tr.dwt_host(host_in, 1, details=det, ll=host_ll, bands=args.bands, sync=True)
    _barrier(torch, dist)
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es.record()
    for _ in range(2):
        tr.dwt_host(host_in, 1, details=det, ll=host_ll, bands=args.bands, sync=False)
    ee.record()
    ee.synchronize()
    e2e_ms = _max_over_ranks(torch, dist, es.elapsed_time(ee)) / 2
    e2e = {"value": sh * n * world / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": sh * n * 4,
           "d2h_bytes_per_step": sh * n * 4, "ms_per_step": e2e_ms, "sample": f"{sh} x {n} rows per rank",
           "api": "Transform.dwt_host(levels=1) (b2dwt_dwt_host) with pinned host buffers"}
    achieved = 8.0 * L.rows * n / (ms * 1e-3) / 1e9
    return {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (uniform on device)",
            "config": {"workload": _workload_name("c5"), "parallelism": f"row-strips x{world}",
                       "halo_rows_per_side_px": [L.halo_top, L.halo_bot],
                       "exchange": "torch.distributed batch_isend_irecv (NCCL) overlapped with interior rows",
                       "arith": args.arith},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "peak_source": src, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None},
            "cpu_baseline": None, "e2e": e2e, "clocks": clk.summary(),
            "gpu_launches": args.steps * (_launches(interior[1] - interior[0], n // 2) + len(edges)),
        }


def run_c1(args):
    """C1 on one GPU: the device kernel (CUDA graph of K forwards, L2-warm: the
    1024^2 image is 4 MiB), the reference-shaped host call end to end, and the
    CPU oracle on the same image."""
    import numpy as np
    import torch

    from paper_1705_08266_b200 import CDF97, Image2D, Transform, build_scheme, forward

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    n = 1024
    scheme = build_scheme("separable-lifting", CDF97)
    tr = Transform(scheme, "single", fast=(args.arith == "fast"))
    img = Image2D.random(n, n, seed=0, precision="single")
    x = torch.from_numpy(img.data).cuda()
    out = tr.forward(x)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        tr.forward(x, out=out)
    with ClockSampler(0) as clk:
        ms = _time_graph(torch, None, graph, args.steps, args.warmup)
    value = n * n / (ms * 1e-3) / 1e9
    for _ in range(2):
        forward(img, scheme)
    t0 = time.perf_counter()
    reps = max(3, args.steps)
    for _ in range(reps):
        forward(img, scheme)
    e2e_ms = (time.perf_counter() - t0) / reps * 1e3
    peak, src = _peaks()
    cpu = None
    if not args.no_cpu:
        gpx, desc, threads, _, _ = _cpu_sample("c1", steps=3, warmup=1)
        cpu = {"value": gpx, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc}
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (Image2D.random, PCG64 seed 0)",
        "config": {"workload": _workload_name("c1"), "arith": args.arith,
                   "l2": "4 MiB image: L2-resident (warm), a latency-bound launch"},
        "roofline": {"bound": "hbm", "achieved": 8.0 * n * n / (ms * 1e-3) / 1e9, "peak": peak, "peak_source": src,
                     "unit": "GB/s", "frac": 8.0 * n * n / (ms * 1e-3) / 1e9 / peak, "traffic": None},
        "cpu_baseline": cpu,
        "e2e": {"value": n * n / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": n * n * 4,
                "d2h_bytes_per_step": n * n * 4, "ms_per_step": e2e_ms,
                "api": "paper_1705_08266_b200.forward(Image2D, scheme) (NumPy in, NumPy out), wall clock"},
        "clocks": clk.summary(), "gpu_launches": args.steps,
    }), flush=True)
    return 0


def run_c2(args):
    import torch

    from paper_1705_08266_b200 import CDF53, CDF97, SCHEME_NAMES, Transform, build_scheme

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    n = 4096
    x = torch.rand((n, n), device="cuda")
    peak, _ = _peaks()
    for plan in (CDF53, CDF97):
        for name in SCHEME_NAMES:
            tr = Transform(build_scheme(name, plan), "single", fast=(args.arith == "fast"))
            outs = tr.forward(x)
            rec = torch.empty_like(x)
            for direction in ("fwd", "inv"):
                fn = (lambda: tr.forward(x, out=outs)) if direction == "fwd" else (lambda: tr.inverse(*outs, out=rec))
                for _ in range(max(3, args.warmup)):
                    fn()
                torch.cuda.synchronize()
                s = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(args.steps):
                    fn()
                e.record()
                e.synchronize()
                ms = s.elapsed_time(e) / args.steps
                gbs = 8.0 * n * n / (ms * 1e-3) / 1e9
                print(json.dumps({"config": f"C2 {plan.name} {name} {direction}", "ms": ms,
                                  "Gpixel/s": n * n / (ms * 1e-3) / 1e9, "GB/s": gbs, "frac": gbs / peak,
                                  "note": "4096^2 (64 MiB) is partly L2-resident"}), flush=True)
    return 0


def _spawn(args):
    """`bench.py --gpus N` (N > 1) run directly: re-launch as N ranks, one per
    GPU, exactly as the driver does (torch.distributed.run, 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=("c3", "c4", "c5", "c2", "c1"), default="c3")
    ap.add_argument("--arith", choices=("strict", "fast"), default="fast",
                    help="fast: FMA within the north-star tolerance (default); strict: bit-exact")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--bands", type=int, default=16, help="row bands of the host-buffer (e2e) pipeline")
    ap.add_argument("--no-scale-configs", action="store_true",
                    help="skip the C4 / C5 strong-scaling keys of the default (C3) line")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _spawn(args)
    if args.impl == "reference":
        return run_reference(args)
    return {"c3": run_c3, "c4": run_c4, "c5": run_c5, "c2": run_c2, "c1": run_c1}[args.config](args)


if __name__ == "__main__":
    sys.exit(main())
