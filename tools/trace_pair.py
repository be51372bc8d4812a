"""Timeline experiment for the CTA-pair attention kernel: run the C2 stream once with an
S2L_TRACE build and decode the leader CTA of cluster 0 of attention launch S2L_TRACE_LAUNCH
(default 31 = the last chunk).  Writers: 0 MMA warp, 1 / 2 softmax warps 4 / 8 (lane 0),
3 producer."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("S2L_TRACE", "1")
os.environ.setdefault("S2L_TRACE_LAUNCH", "31")
os.environ.setdefault("S2L_TRACE_FILE", os.path.join(ROOT, "gpurun_out", "trace_pair.bin"))
import bench  # noqa: E402

NAMES = {10: "mma:wait_P", 11: "mma:got_PL", 12: "mma:got_PH(PV issued)", 13: "mma:S_issue(buf)",
         20: "sm:wait_S", 21: "sm:got_S", 22: "sm:max_done", 25: "sm:got_m_prev", 23: "sm:P_lo",
         24: "sm:P_hi", 30: "tma:wait_slot(idx)", 31: "tma:issue(idx)"}


def main():
    torch.cuda.set_device(0)
    rids, toks, data = bench.make_stream_data(0)
    S = bench.Stream(rids, toks, data, "cuda:0")
    ctx, pool = bench.make_ctx(0)
    bench.run_step(ctx, S)
    torch.cuda.synchronize()
    ctx.close()
    raw = np.fromfile(os.environ["S2L_TRACE_FILE"], dtype=np.uint32)
    rows = []
    for w in range(4):
        n = int(raw[w])
        seg = raw[16 + w * 4096 * 2: 16 + w * 4096 * 2 + 2 * n].reshape(n, 2).astype(np.int64)
        for code, c in seg:
            rows.append((w, code >> 24, code & 0xffff, c))
    ev = np.array(rows, dtype=np.int64)
    ev = ev[np.argsort(ev[:, 3], kind="stable")]
    t0 = ev[0, 3]
    print(f"{len(ev)} events")
    lo = int(os.environ.get("TRACE_LO", "40"))
    for w, e, j, c in ev:
        jj = j // 2 if e in (30, 31) else j
        if lo <= jj < lo + 4 or (e == 13 and lo <= 0):
            print(f"{c - t0:9d}  w{w} {NAMES.get(int(e), e):24s} {j}")

    def series(w, code):
        return {int(r[2]): int(r[3]) for r in ev if r[0] == w and r[1] == code}
    for w in (1, 2):
        ws, gs, mx, mp, pl, ph = (series(w, c) for c in (20, 21, 22, 25, 23, 24))
        ks = [k for k in gs if k in ph and k in ws and k in mp and k in mx]
        if not ks:
            continue
        f = lambda a, b: np.mean([b[k] - a[k] for k in ks])
        print(f"softmax w{w}: wait S {f(ws, gs):.0f}, got S -> max {f(gs, mx):.0f}, max -> m_prev {f(mx, mp):.0f}, "
              f"m_prev -> P_lo {f(mp, pl):.0f}, P_lo -> P_hi {f(pl, ph):.0f}  ({len(ks)} steps)")
    si, gl, gh = series(0, 13), series(0, 11), series(0, 12)
    ks = [k for k in gl if k in gh and k in si]
    print("mma: S(j) issue -> PV(j) first half %.0f, PV halves apart %.0f" % (
        np.mean([gl[k] - si[k] for k in ks]), np.mean([gh[k] - gl[k] for k in ks])))
    ph = series(0, 12)
    st = sorted(ph)
    d = np.diff([ph[k] for k in st])
    print("period between PV issues: mean %.0f median %.0f cycles" % (d.mean(), np.median(d)))


if __name__ == "__main__":
    main()
