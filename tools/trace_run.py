"""Timeline experiment: run the C2 stream once with an S2L_TRACE build and decode the trace of
CTA 0 of attention launch S2L_TRACE_LAUNCH (default 31 = the last chunk)."""
import json
import os
import struct
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("S2L_TRACE", "1")
os.environ.setdefault("S2L_TRACE_LAUNCH", "31")
os.environ.setdefault("S2L_TRACE_FILE", os.path.join(ROOT, "gpurun_out", "trace.bin"))
import bench  # noqa: E402

NAMES = {10: "mma:wait_P_lo", 11: "mma:got_P_lo", 12: "mma:got_P_hi", 13: "mma:S_issue_begin",
         14: "mma:S_issue_end", 20: "sm:wait_S", 21: "sm:got_S", 22: "sm:max_done", 23: "sm:P_lo_arrived",
         24: "sm:P_hi_arrived"}


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
            rows.append((code >> 24, (code >> 16) & 0xff, code & 0xffff, c))
    ev = np.array(rows, dtype=np.int64)
    ev = ev[np.argsort(ev[:, 3], kind="stable")]
    n = len(ev)
    t0 = ev[0, 3]
    print(f"{n} events")
    # per-step intervals for steps 40..44
    for row in ev:
        e, tile, j, c = row
        if 40 <= j <= 43 or e in (13, 14) and 40 <= 0:
            print(f"{c - t0:9d}  {NAMES.get(int(e), e):20s} tile {tile} step {j}")
    # averages: S-wait time, softmax time (got_S -> P_hi), MMA wait for P
    def series(code):
        return {(int(r[1]), int(r[2])): int(r[3]) for r in ev if r[0] == code}
    got_s, p_hi, p_lo, mx = series(21), series(24), series(23), series(22)
    w_s, m_lo, m_hi = series(20), series(11), series(12)
    sm = [p_hi[k] - got_s[k] for k in got_s if k in p_hi]
    mx_t = [mx[k] - got_s[k] for k in got_s if k in mx]
    wait_s = [got_s[k] - w_s[k] for k in got_s if k in w_s]
    print("softmax got_S -> P_hi: mean %.0f cycles, got_S -> max %.0f, waiting for S %.0f" %
          (np.mean(sm), np.mean(mx_t), np.mean(wait_s)))
    wp = series(10)
    mw = [m_lo[k] - wp[k] for k in m_lo if k in wp]
    print("mma wait for P_lo: mean %.0f cycles" % np.mean(mw))
    steps = sorted({k[1] for k in got_s})
    per = [got_s[(0, j + 1)] - got_s[(0, j)] for j in steps if (0, j + 1) in got_s]
    print("period (tile 0 got_S to got_S): mean %.0f cycles over %d steps" % (np.mean(per), len(per)))
    # steady state (steps 10 .. last-10): per tile, the chain S ready -> P halves -> MMA -> next S
    lo_j, hi_j = 10, max(steps) - 10
    out = {}
    for i in (0, 1):
        ks = [(i, j) for j in range(lo_j, hi_j) if (i, j) in got_s and (i, j) in p_lo and (i, j) in p_hi]
        f = lambda a, b: float(np.mean([a[k] - b[k] for k in ks if k in a and k in b]))
        nxt = [got_s[(i, j + 1)] - m_hi[(i, j)] for (_, j) in ks if (i, j + 1) in got_s and (i, j) in m_hi]
        out[f"tile{i}"] = {"gotS_to_Plo": f(p_lo, got_s), "gotS_to_Phi": f(p_hi, got_s),
                           "Plo_to_mma_got": f(m_lo, p_lo), "Phi_to_mma_got": f(m_hi, p_hi),
                           "mma_waiting_for_Plo": f(m_lo, wp), "softmax_waiting_for_S": f(got_s, w_s),
                           "mma_gotPhi_to_next_gotS": float(np.mean(nxt)) if nxt else None}
    print(json.dumps({"period": float(np.mean(per)), "steady": out}))


if __name__ == "__main__":
    main()
