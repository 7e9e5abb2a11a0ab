"""Per-launch counters and stall-sample breakdown of every kernel in an ncu
report (`ncu --set full` capture), one column per launch:

    python tools/ncu_counters.py gpurun_out/r02_fused_c3.ncu-rep > profiles/r02_ncu_fused_c3_counters.txt
"""
import csv, subprocess, sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "smsp__inst_executed.sum",
        "sm__cycles_active.avg", "sm__cycles_active.max", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "lts__t_sector_op_read_hit_rate.pct", "lts__t_sector_op_write_hit_rate.pct",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def main(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units, data = rows[0], rows[1], rows[2:]
    col = {n: i for i, n in enumerate(h)}
    print("Kernel Name ", [r[col["Kernel Name"]][:60] for r in data])
    for n in WANT:
        if n in col:
            print(n, units[col[n]], [r[col[n]] for r in data])
    stalls = sorted((n for n in h if n.startswith(STALL) and not n.endswith("_not_issued")),
                    key=lambda n: -float(data[0][col[n]].replace(",", "") or 0))
    print("# stall samples (smsp__pcsamp_warps_issue_stalled_*), per launch")
    for n in stalls:
        vals = [r[col[n]] for r in data]
        if any(float(v.replace(",", "") or 0) > 0 for v in vals):
            print(n[len(STALL):], vals)


if __name__ == "__main__":
    main(sys.argv[1])
