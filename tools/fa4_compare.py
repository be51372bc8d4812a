"""Same-window comparison of libs2l's attention with the FlashAttention-4 Blackwell forward
kernel (CuTe-DSL, shipped inside vllm as `vllm.vllm_flash_attn.cute`) on the C2 stream.

    python tools/fa4_compare.py [--reps 5] [--c5] [--out gpurun_out/fa4_compare.json]

A LIBRARY comparator (like timing cuBLAS beside a GEMM): it is not on libs2l's path and nothing
in the product imports it.  Workload = bench.py's C2 (BJ:L8): 8 requests, 32 q / 8 kv heads,
d 128, 512-token chunks from 0 to 16K; per step the chunk's queries attend causally
(bottom-right, Z3) over p0 + 512 keys.  Both sides get the same device N(0,1) bf16 Q/K/V.

  * s2l      : s2l_prefill_batch over the paged pool (block 16), per-launch device time from the
               library's own timing events (the bench's roofline source).
  * fa4_paged: FA4 with page_table over a [pages][16][h_kv][d] K and V cache (same page ids).
  * fa4_dense: FA4 over batch-padded contiguous K/V ([8][16384][h_kv][d]) with seqused_k -- FA4's
               best case (no paging).
--c5: the long-chunk config instead (BJ:L11: one request, 128K context, 2K chunks, 64q/8kv).
Timing: CUDA events around each launch on the current stream, median of --reps replays per step.
The outputs of step 31 are compared (per-row normwise difference, the parity metric of the tests).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402

NREQ, CHUNK, TOTAL, H_Q, H_KV, D, KB = bench.NREQ, bench.CHUNK, bench.TOTAL, bench.H_Q, bench.H_KV, bench.D, bench.KB
if "--c5" in sys.argv:
    NREQ, CHUNK, TOTAL, H_Q = 1, 2048, 131072, 64
STEPS = TOTAL // CHUNK


def ev_time(fn, reps):
    out = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "fa4_compare.json"))
    ap.add_argument("--c5", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    q = [torch.randn(NREQ * CHUNK, H_Q, D, device=dev, generator=g).to(torch.bfloat16) for _ in range(STEPS)]
    k = [torch.randn(1, NREQ * CHUNK, H_KV, D, device=dev, generator=g).to(torch.bfloat16) for _ in range(STEPS)]
    v = [torch.randn(1, NREQ * CHUNK, H_KV, D, device=dev, generator=g).to(torch.bfloat16) for _ in range(STEPS)]
    ap_c5 = "--c5" in sys.argv
    fl = [NREQ * bench.attn_flops(CHUNK, j * CHUNK, h_q=H_Q) for j in range(STEPS)]
    res = {"workload": ("C5 (BJ:L11) stream, 1 x 2048-token chunks to 128K, 64q/8kv, d 128" if ap_c5 else
                        "C2 (BJ:L8) stream, 8 x 512-token chunks to 16K, 32q/8kv, d 128"), "reps": a.reps}

    # ---- libs2l
    from paper_2604_16395_b200 import s2l
    nblk_all = NREQ * TOTAL // KB
    cfg = s2l.make_config(1, H_Q, H_KV, D, KB, nblk_all, 0, max_requests=NREQ, max_blocks_per_request=TOTAL // KB)
    pool = torch.empty(nblk_all * s2l.block_bytes(cfg) // 2, dtype=torch.bfloat16, device=dev)
    ctx = s2l.Context(cfg, pool, None, torch.cuda.current_stream(), None)
    rids = list(range(NREQ))
    toks = [list(range(TOTAL)) for _ in rids]
    items_a = [[(r, None, CHUNK, i * CHUNK) for i, r in enumerate(rids)] for _ in range(STEPS)]
    items_p = [[(r, j * CHUNK, CHUNK, i * CHUNK) for i, r in enumerate(rids)] for j in range(STEPS)]
    o_s2l = torch.empty_like(q[0])
    for r, t in zip(rids, toks):
        ctx.new_request(r, t)
    s2l_ms = []
    for j in range(STEPS):
        ctx.append_chunk(items_a[j], k[j], v[j])
        torch.cuda.synchronize()
        for _ in range(2):
            ctx.prefill_batch(0, items_p[j], q[j], o_s2l)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            ctx.set_timing(True)
            ctx.prefill_batch(0, items_p[j], q[j], o_s2l)
            torch.cuda.synchronize()
            ts.append(ctx.timing_read()["attn_ms"])
            ctx.set_timing(False)
        s2l_ms.append(statistics.median(ts))
    o_s2l_last = o_s2l.clone()
    bt = [ctx.block_table(r) for r in rids]

    # ---- FA4 (CuTe-DSL), paged over the same page ids
    from vllm.vllm_flash_attn.cute.interface import _flash_attn_fwd
    nblk = NREQ * TOTAL // KB
    kc = torch.zeros(nblk, KB, H_KV, D, dtype=torch.bfloat16, device=dev)
    vc = torch.zeros_like(kc)
    pt = torch.tensor(bt, dtype=torch.int32, device=dev)
    for j in range(STEPS):
        for i, r in enumerate(rids):
            rows = slice(i * CHUNK, (i + 1) * CHUNK)
            ids = pt[i, j * CHUNK // KB:(j + 1) * CHUNK // KB].long()
            kc[ids] = k[j][0, rows].reshape(CHUNK // KB, KB, H_KV, D)
            vc[ids] = v[j][0, rows].reshape(CHUNK // KB, KB, H_KV, D)
    cu_q = torch.arange(0, NREQ + 1, device=dev, dtype=torch.int32) * CHUNK
    scale = 1.0 / math.sqrt(D)

    def fa_paged(j, out):
        used = torch.full((NREQ,), (j + 1) * CHUNK, dtype=torch.int32, device=dev)
        return lambda: _flash_attn_fwd(q[j], kc, vc, cu_seqlens_q=cu_q, seqused_k=used, max_seqlen_q=CHUNK,
                                       page_table=pt, softmax_scale=scale, causal=True, out=out)

    kd = torch.zeros(NREQ, TOTAL, H_KV, D, dtype=torch.bfloat16, device=dev)
    vd = torch.zeros_like(kd)
    for j in range(STEPS):
        for i in range(NREQ):
            kd[i, j * CHUNK:(j + 1) * CHUNK] = k[j][0, i * CHUNK:(i + 1) * CHUNK]
            vd[i, j * CHUNK:(j + 1) * CHUNK] = v[j][0, i * CHUNK:(i + 1) * CHUNK]

    def fa_dense(j, out):
        used = torch.full((NREQ,), (j + 1) * CHUNK, dtype=torch.int32, device=dev)
        return lambda: _flash_attn_fwd(q[j], kd, vd, cu_seqlens_q=cu_q, seqused_k=used, max_seqlen_q=CHUNK,
                                       softmax_scale=scale, causal=True, out=out)

    for name, mk in (("fa4_paged", fa_paged), ("fa4_dense", fa_dense)):
        out = torch.empty_like(q[0])
        try:
            mk(STEPS - 1, out)()           # JIT compile
            torch.cuda.synchronize()
        except Exception as ex:  # noqa: BLE001
            res[name] = {"error": f"{type(ex).__name__}: {ex}"[:400]}
            continue
        ms = []
        for j in range(STEPS):
            f = mk(j, out)
            f(); f()
            torch.cuda.synchronize()
            ms.append(ev_time(f, a.reps))
        o_last = torch.empty_like(q[0])
        mk(STEPS - 1, o_last)()
        torch.cuda.synchronize()
        diff = ((o_last.float() - o_s2l_last.float()).abs().amax(-1)
                / o_last.float().abs().amax(-1).clamp_min(1e-6)).max().item()
        res[name] = {"ms_per_step": [round(x, 4) for x in ms], "stream_ms": sum(ms),
                     "tflops": sum(fl) / (sum(ms) * 1e-3) / 1e12,
                     "last_step_tflops": fl[-1] / (ms[-1] * 1e-3) / 1e12,
                     "max_normwise_diff_vs_s2l_step31": diff}
    res["s2l"] = {"ms_per_step": [round(x, 4) for x in s2l_ms], "stream_ms": sum(s2l_ms),
                  "tflops": sum(fl) / (sum(s2l_ms) * 1e-3) / 1e12,
                  "last_step_tflops": fl[-1] / (s2l_ms[-1] * 1e-3) / 1e12}
    pk = bench.peaks()
    res["peak_bf16_tflops"] = pk["bf16"]
    for n in ("s2l", "fa4_paged", "fa4_dense"):
        if "tflops" in res.get(n, {}):
            res[n]["frac"] = res[n]["tflops"] / pk["bf16"]
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({n: {kk: vv for kk, vv in res[n].items() if kk != "ms_per_step"}
                      for n in ("s2l", "fa4_paged", "fa4_dense") if n in res}))


if __name__ == "__main__":
    main()
