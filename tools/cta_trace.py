"""CTA-phase timeline of one attention launch of the C2 stream (timing experiment).

Needs a libs2l build with -DS2L_CTATRACE (S2L_NVCC_FLAGS="-DS2L_CTATRACE" python -m
paper_2604_16395_b200.build --force).  Every CTA of attention launch L (the C2 chunk index)
stamps its phases (see attn_tc.cu, cta_stamp); this prints the launch span, the per-CTA phase
durations and the gaps between consecutive CTAs on an SM.

    python tools/cta_trace.py L [L ...]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def run(launch):
    path = os.path.join(ROOT, "gpurun_out", f"ctatrace_{launch}.bin")
    os.environ["S2L_TRACE"] = "1"
    os.environ["S2L_TRACE_LAUNCH"] = str(launch)
    os.environ["S2L_TRACE_FILE"] = path
    rids, toks, data = bench.make_stream_data(0)
    S = bench.Stream(rids, toks, data, "cuda:0")
    for _ in range(2):                     # warm-up stream, then the traced one
        ctx, pool = bench.make_ctx(0)
        bench.run_step(ctx, S)
        torch.cuda.synchronize()
        ctx.close()
    raw = np.fromfile(path, dtype=np.uint64)
    n = len(raw) // 32
    t = raw[: n * 32].reshape(n, 32).astype(np.int64)
    t = t[t[:, 0] > 0]
    g0 = t[:, 0].min()
    ent, ext = (t[:, 0] - g0) / 1e3, (t[:, 1] - g0) / 1e3         # us
    clk = t[:, 2:9].astype(np.float64)
    clk_exit = t[:, 11].astype(np.float64)
    sm = t[:, 9] >> 32
    nT = t[:, 9] & 0xffffffff
    dur_us = ext - ent
    cyc = clk_exit - clk[:, 0]
    mhz = cyc / np.maximum(dur_us, 1e-3)
    ph = {"decode": t[:, 14].astype(np.float64) - clk[:, 0], "mbar_init": t[:, 15].astype(np.float64) - clk[:, 0],
          "init": t[:, 12].astype(np.float64) - clk[:, 0], "alloc": t[:, 13].astype(np.float64) - clk[:, 0],
          "setup": clk[:, 1] - clk[:, 0], "to_Q": clk[:, 2] - clk[:, 1], "to_K0": clk[:, 3] - clk[:, 2],
          "to_S0": clk[:, 4] - clk[:, 3], "loop": clk[:, 5] - clk[:, 4], "epilogue": clk[:, 6] - clk[:, 5],
          "epi_wait_O": t[:, 16].astype(np.float64) - clk[:, 5], "epi_work": clk[:, 6] - t[:, 16].astype(np.float64),
          "exit": clk_exit - clk[:, 6]}
    gaps = []
    for s in np.unique(sm):
        idx = np.where(sm == s)[0]
        idx = idx[np.argsort(ent[idx])]
        for a, b in zip(idx[:-1], idx[1:]):
            gaps.append(ent[b] - ext[a])
    loop_per_tile = ph["loop"] / np.maximum(nT, 1)
    res = {"launch": launch, "ctas": int(len(t)), "span_us": float(ext.max()), "sm_count": int(len(np.unique(sm))),
           "cta_us_mean": float(dur_us.mean()), "clock_mhz_median": float(np.median(mhz)),
           "nT_mean": float(nT.mean()), "nT_max": int(nT.max()),
           "phase_cycles_mean": {k: float(v.mean()) for k, v in ph.items()},
           "split_ctas": int(((t[:, 10] & 0xff) > 1).sum()),
           "epilogue_cycles_median": {"plain": float(np.median(ph["epilogue"][(t[:, 10] & 0xff) == 1])),
                                      "split": float(np.median(ph["epilogue"][(t[:, 10] & 0xff) > 1]))
                                      if ((t[:, 10] & 0xff) > 1).any() else None},
           "loop_cycles_per_kv_step_median": float(np.median(loop_per_tile[nT > 2])) if (nT > 2).any() else None,
           "gap_us_between_ctas_on_sm": {"mean": float(np.mean(gaps)) if gaps else None,
                                         "max": float(np.max(gaps)) if gaps else None},
           "last_entry_us": float(ent.max()), "first_exit_us": float(ext.min()),
           "ctas_per_sm_max": int(np.bincount(sm).max())}
    print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    torch.cuda.set_device(0)
    out = [run(int(a)) for a in (sys.argv[1:] or ["31"])]
    with open(os.path.join(ROOT, "gpurun_out", "cta_trace.json"), "w") as f:
        json.dump(out, f, indent=1)
