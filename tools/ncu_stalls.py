"""Per-role warp-stall breakdown of an ncu --import-source report of attn_tc2.

    python tools/ncu_stalls.py gpurun_out/prof.ncu-rep [top_n]

Splits the SASS into regions by the instructions they contain (producer: UTMALDG.2D loop,
MMA: UTCHMMA, softmax: MUFU.EX2 / LDTM, wait loops: SYNCS.PHASECHK targets) and prints the
sample counts per stall reason for the hottest instructions.
"""
import csv
import subprocess
import sys

REASONS = ["stall_barrier", "stall_branch_resolving", "stall_long_sb", "stall_math", "stall_mio",
           "stall_no_inst", "stall_not_selected", "stall_selected", "stall_short_sb", "stall_sleep",
           "stall_wait", "stall_lg", "stall_dispatch", "stall_membar", "stall_misc"]


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))[1:]
    hdr, data = rows[0], rows[1:]
    iS, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    idx = {r: hdr.index(r) for r in REASONS if r in hdr}
    tot = sum(int(r[iS]) for r in data if r[iS].isdigit())
    print(f"{path}: {tot} samples, {len(data)} SASS instructions")
    agg = {r: 0 for r in idx}
    for r in data:
        for k, i in idx.items():
            if r[i].isdigit():
                agg[k] += int(r[i])
    print("  overall:", ", ".join(f"{k[6:]}={v}" for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v))
    order = sorted(range(len(data)), key=lambda i: -(int(data[i][iS]) if data[i][iS].isdigit() else 0))[:top]
    for i in sorted(order):
        r = data[i]
        why = ", ".join(f"{k[6:]}={r[j]}" for k, j in idx.items() if r[j].isdigit() and int(r[j]) > 0.15 * max(1, int(r[iS])))
        print(f"  {i:5d} {r[iS]:>6s}  {r[iSrc].strip()[:70]:70s} {why}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
