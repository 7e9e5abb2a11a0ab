"""Build libb2dwt.so in-tree with nvcc for sm_100a (no GPU needed).

Translation units:
  csrc/b2dwt_host.cu        C ABI, plan matching, generic interpreter kernel
  csrc/host_pipeline.cu     b2dwt_dwt_host: host-buffer pyramid, copies overlapped in row bands
  csrc/lift1d.cu            batched 1-D lifting (b2dwt_lift1d / b2dwt_unlift1d)
  csrc/prog_dispatch.cu     per built-in program: variant selection, cone
  csrc/prog_variant.cu      ONE fused kernel per unit (program x element type x
                            layout x arithmetic x fill), compiled in parallel
  csrc/prog_tile.cu         per built-in program: the small-level tile kernels
  csrc/prog_fused2.cu       per forward lifting program: two pyramid levels in one
                            kernel (fused2_kernel.cuh), strict + fast

Flags: -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 (ptxas -v output is
kept in build/ptxas_<unit>.log for register / spill review).

    python -m paper_1705_08266_b200.build [--force] [--jobs N]
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(HERE, "libb2dwt.so")
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
N_VARIANTS = 8  # see csrc/prog_variant.cu
NVCC_FLAGS = ["-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v", *ARCH]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libb2dwt.so")


def _program_units():
    """(ident, is_inverse) for every built-in program, from programs.inc."""
    units = []
    with open(os.path.join(CSRC, "programs.inc")) as fh:
        for line in fh:
            line = line.strip()
            if line.startswith("struct ") and line.endswith("{"):
                ident = line.split()[1]
                units.append((ident, ident.endswith("_inv")))
    return units


def _deps(src: str, seen=None):
    """The source and every file it includes with #include "..." (recursively)."""
    seen = set() if seen is None else seen
    src = os.path.normpath(src)
    if src in seen or not os.path.exists(src):
        return seen
    seen.add(src)
    with open(src) as fh:
        for line in fh:
            line = line.strip()
            if line.startswith("#include") and '"' in line:
                name = line.split('"')[1]
                for base in (os.path.dirname(src), CSRC, INCLUDE):
                    cand = os.path.join(base, name)
                    if os.path.exists(cand):
                        _deps(cand, seen)
                        break
    return seen


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(args):
    src, obj, defines, log = args
    extra = os.environ.get("B2DWT_NVCC_EXTRA", "").split()  # experiments, e.g. -DB2DWT_F32_RPS=8
    cmd = [nvcc(), *NVCC_FLAGS, *extra, *defines, "-I", CSRC, "-I", INCLUDE, "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(obj)}:\n{res.stderr[-4000:]}")
    return obj


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    jobs = jobs or max(1, os.cpu_count() or 1)
    # host TU in C++17 (nvcc 12.9's C++20 front end trips over libstdc++ 13
    # containers); kernel TUs need C++20 for the phase-unrolled tick loop
    tasks = [(os.path.join(CSRC, f"{u}.cu"), os.path.join(BUILD, f"{u}.o"), ["-std=c++17"],
              os.path.join(BUILD, f"ptxas_{u}.log")) for u in ("b2dwt_host", "host_pipeline", "lift1d")]
    # dev builds: B2DWT_PROGRAMS=ident,... and/or B2DWT_VARIANTS=0,1 compile
    # only that subset; the rest are stubs (the host falls back to the generic
    # interpreter for them).  Release builds compile everything.
    only = os.environ.get("B2DWT_PROGRAMS")
    only = set(only.split(",")) if only else None
    vonly = os.environ.get("B2DWT_VARIANTS")
    vonly = {int(v) for v in vonly.split(",")} if vonly else None
    for ident, inv in _program_units():
        defs = [f"-DB2DWT_PROG={ident}", f"-DB2DWT_PROG_INV={int(inv)}"]
        tasks.append((os.path.join(CSRC, "prog_dispatch.cu"), os.path.join(BUILD, f"dispatch_{ident}.o"),
                      ["-std=c++20", *defs], os.path.join(BUILD, f"ptxas_dispatch_{ident}.log")))
        # two-level fused kernel: forward lifting programs (per-sub-step
        # horizontal reach <= 1); a stub elsewhere
        f2 = not inv and ident != "cdf97_conv_fwd" and (only is None or ident in only)
        tasks.append((os.path.join(CSRC, "prog_fused2.cu"), os.path.join(BUILD, f"fused2_{ident}{'' if f2 else '_stub'}.o"),
                      ["-std=c++20", *defs] + ([] if f2 else ["-DB2DWT_STUB"]),
                      os.path.join(BUILD, f"ptxas_fused2_{ident}{'' if f2 else '_stub'}.log")))
        tag = "" if (only is None or ident in only) else "_stub"
        tasks.append((os.path.join(CSRC, "prog_tile.cu"), os.path.join(BUILD, f"tile_{ident}{tag}.o"),
                      ["-std=c++20", *defs] + (["-DB2DWT_STUB"] if tag else []),
                      os.path.join(BUILD, f"ptxas_tile_{ident}{tag}.log")))
        for vid in range(N_VARIANTS):
            real = (only is None or ident in only) and (vonly is None or vid in vonly)
            tag = "" if real else "_stub"
            tasks.append((
                os.path.join(CSRC, "prog_variant.cu"),
                os.path.join(BUILD, f"v_{ident}_{vid}{tag}.o"),
                ["-std=c++20", *defs, f"-DB2DWT_VID={vid}"] + ([] if real else ["-DB2DWT_STUB"]),
                os.path.join(BUILD, f"ptxas_{ident}_{vid}{tag}.log"),
            ))
    # objects built with other experiment flags are stale too
    flags_file = os.path.join(BUILD, "nvcc_extra.txt")
    extra = os.environ.get("B2DWT_NVCC_EXTRA", "")
    if os.path.exists(flags_file) and open(flags_file).read() != extra:
        force = True
    with open(flags_file, "w") as fh:
        fh.write(extra)
    dep_cache = {}

    def unit_deps(src):
        if src not in dep_cache:
            dep_cache[src] = sorted(_deps(src))
        return dep_cache[src]

    todo = [t for t in tasks if force or _stale(t[1], unit_deps(t[0]))]
    if verbose:
        print(f"[b2dwt] compiling {len(todo)} units with {jobs} jobs", file=sys.stderr)
    todo.sort(key=lambda t: ("_stub" in t[1] or "dispatch_" in t[1], t[1]))
    with ThreadPoolExecutor(max_workers=jobs) as pool:
        list(pool.map(_compile, todo))
    objs = [t[1] for t in tasks]
    manifest = os.path.join(BUILD, "link_manifest.txt")
    want = "\n".join(objs)
    have = open(manifest).read() if os.path.exists(manifest) else ""
    if not force and not todo and have == want and not _stale(LIB, objs):
        return LIB
    tmp = LIB + ".tmp"
    cmd = [nvcc(), "-shared", *ARCH, "-o", tmp, *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
    os.replace(tmp, LIB)
    with open(manifest, "w") as fh:
        fh.write(want)
    return LIB


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=None)
    a = ap.parse_args()
    print(build(force=a.force, jobs=a.jobs, verbose=True))


if __name__ == "__main__":
    main()
