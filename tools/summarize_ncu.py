"""Summarise ncu outputs into profiles/: launch-list shares and the top kernel's counters."""
import collections, csv, json, subprocess, sys

def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ik, iv, iu, ig = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "Grid Size"))
    agg = collections.defaultdict(list)
    for r in data:
        v = float(r[iv].replace(",", ""))
        v = v / 1000 if r[iu] == "ns" else (v * 1000 if r[iu] == "ms" else v)
        name = r[ik].split("<")[0].replace("void ", "")
        if "stream_kernel" in r[ik]:
            prog = r[ik].split("<")[1].split(",")[0].split("::")[-1]
            name = f"stream_kernel<{prog}> grid {r[ig]}"
        agg[name].append(v)
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append({"kernel": k, "launches": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / tot})
    return out

def counters(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_l1tex2xbar_write_bytes.sum",
            "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum",
            "launch__grid_size", "launch__block_size", "sm__cycles_active.avg", "sm__cycles_active.max"]
    return {n: (u[i], v[i]) for i, n in enumerate(h) if n in want}

if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    if kind == "launches":
        for r in launches(path):
            print(f"{r['share']*100:5.1f}%  {r['mean_us']:9.1f} us x{r['launches']:3d}  {r['kernel']}")
    else:
        for k, (unit, val) in counters(path).items():
            print(f"{k:60s} {val:>16s} {unit}")
