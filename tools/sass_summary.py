"""Per-kernel SASS evidence for the hot kernels of libb2dwt.so (cuobjdump -sass):
instruction counts that prove TMA loads (UTMALDG), mbarrier use (SYNCS),
warp shuffles (SHFL), vector global stores (STG.E.64 / STG.E.128), shared
ring traffic (LDS/STS), FP work (FFMA/FMUL/FADD), spills (LDL/STL), plus the
innermost FP loop of each kernel (the steady tick loop) and its mix.

    python tools/sass_summary.py [lib.so] > profiles/r02_sass_summary.txt
"""
import collections, os, re, subprocess, sys

LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                         "paper_1705_08266_b200", "libb2dwt.so")
WANT = ("cdf97_nssplit_fwd",)  # the C3 program
KEYS = ("UTMALDG", "UTMASTG", "SYNCS", "SHFL", "STG.E.64", "STG.E.128", "STG.E", "LDS", "STS", "FFMA", "FMUL", "FADD",
        "LDL", "STL", "BAR")


def demangle(n):
    try:
        return subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    except OSError:
        return n


txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
print(f"# SASS summary of {os.path.basename(LIB)} (cuobjdump -sass), sm_100a")
for fn in re.split(r"\n\s+Function : ", txt)[1:]:
    name = fn.split("\n")[0].strip()
    dn = demangle(name)
    if not any(w in dn for w in WANT) and "fused2" not in dn:
        continue
    if "fused2" in dn and "cdf97_nssplit_fwd" not in dn:
        continue
    ins = []
    for l in fn.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for _, t in ins)
    cnt = {k: sum(v for o, v in ops.items() if o == k or o.startswith(k + ".")) for k in KEYS}
    cnt["STG.E.64"] = ops.get("STG.E.64", 0)
    cnt["STG.E.128"] = ops.get("STG.E.128", 0)
    addr = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, t) in enumerate(ins):
        if "BRA" in t:
            m = re.search(r"0x([0-9a-f]+)", t)
            if m and int(m.group(1), 16) < a and int(m.group(1), 16) in addr:
                s = addr[int(m.group(1), 16)]
                c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x).split()[0].split(".")[0] for _, x in ins[s:i + 1])
                if c["FFMA"] > 50:
                    loops.append((i - s + 1, c))
    print(f"\n## {dn[:200]}")
    print(f"total {len(ins)} instructions; " + ", ".join(f"{k} {v}" for k, v in cnt.items()))
    if loops:
        n, c = min(loops, key=lambda x: x[0])
        print(f"innermost FP loop: {n} instructions: " + ", ".join(
            f"{k} {c[k]}" for k in ("FFMA", "FMUL", "FADD", "SHFL", "LDS", "STS", "STG", "SYNCS", "LDL", "STL", "BRA")))
