"""Summarise ncu outputs brought back in gpurun_out/ into small committed text files.

    python tools/ncu_summary.py launches <launches.csv> > profiles/<round>_launches.txt
    python tools/ncu_summary.py full <report.ncu-rep> > profiles/<round>_<kernel>_full.txt
"""
import collections
import csv
import io
import subprocess
import sys

FULL_KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    iN, iV, iU, iM = (hdr.index(x) for x in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
    for r in data:
        if r[iM] != "gpu__time_duration.sum":
            continue
        v = float(r[iV].replace(",", "")) * scale.get(r[iU], 1e-6)
        nm = r[iN].split("(")[0].replace("s2l::<unnamed>::", "")
        agg[nm][0] += 1
        agg[nm][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list ({path}); gpu__time_duration.sum, --clock-control none (cold, serialised)")
    print(f"# {'kernel':40s} {'launches':>8s} {'total ms':>10s} {'avg us':>10s} {'share':>7s}")
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {k:40s} {n:8d} {ms:10.3f} {1000 * ms / n:10.1f} {100 * ms / tot:6.1f}%")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {path}")
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"## kernel: {name[:100]}")
        for k in FULL_KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:80s} {vals[i]:>16s} {units[i]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
