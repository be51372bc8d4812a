"""B200 TTFT of the paper's streaming scheduler (§6.2) on
synthetic crawler (append) / ANNS (update) traces (synth/traces.py), every step executed on the
GPU through libs2l: one append of the step's K/V (all layers) + one chunked-prefill attention
launch per layer; with --gemm, the Llama-3-8B dense layers of the same tokens run as cuBLAS
bf16 GEMMs with random weights (QKV, O, gate/up, down per layer: the model work the paper's
C_prefill includes; library GEMMs, not this repo's kernels).

The clock is virtual: chunks arrive at their trace times, each step takes its measured GPU
time (CUDA events, synchronised), and arrivals are admitted between steps.  TTFT = finish of
the prefill of the complete input - arrival of its last chunk (reading Z17).  The streaming
policies (DEFAULT / FCFS / MCPS / LCAS, §4.4) run with cost-based preemption (§4.3) using the
B200 cost model if profiles/r01/costmodel_b200.json exists; "NS" is the non-streaming
baseline (DEFAULT policy, requests visible only when complete).

    python tools/ttft_sim.py crawler --qps 4 --n 64 [--layers 32] [--gemm] [--gpu-blocks N]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_16395_b200 import costmodel, model as M, s2l, scheduler as S  # noqa: E402
from synth import traces  # noqa: E402

H_Q, H_KV, D, K = 32, 8, 128, 16
HIDDEN, INTER = 4096, 14336


class Model:
    """Per-step device work for the scheduled items."""

    def __init__(self, ctx, layers, budget, gemm, seed=7):
        g = torch.Generator(device="cuda").manual_seed(seed)
        self.ctx, self.L = ctx, layers
        self.k = torch.randn(layers, budget, H_KV, D, generator=g, device="cuda").to(torch.bfloat16)
        self.v = torch.randn(layers, budget, H_KV, D, generator=g, device="cuda").to(torch.bfloat16)
        self.q = torch.randn(budget, H_Q, D, generator=g, device="cuda").to(torch.bfloat16)
        self.o = torch.empty_like(self.q)
        self.gemm = gemm
        if gemm:
            s = 0.02
            self.w = [(torch.randn(HIDDEN, (H_Q + 2 * H_KV) * D, generator=g, device="cuda") * s).to(torch.bfloat16),
                      (torch.randn(H_Q * D, HIDDEN, generator=g, device="cuda") * s).to(torch.bfloat16),
                      (torch.randn(HIDDEN, 2 * INTER, generator=g, device="cuda") * s).to(torch.bfloat16),
                      (torch.randn(INTER, HIDDEN, generator=g, device="cuda") * s).to(torch.bfloat16)]
            self.x = torch.randn(budget, HIDDEN, generator=g, device="cuda").to(torch.bfloat16)
            self.h = torch.randn(budget, INTER, generator=g, device="cuda").to(torch.bfloat16)

    def step(self, items):
        rows, app, pre = 0, [], []
        for r, q_pos, n in items:
            app.append((r, None, n, rows))
            pre.append((r, q_pos, n, rows))
            rows += n
        self.ctx.append_chunk(app, self.k, self.v, kv_rows=self.k.shape[1])
        x = self.x[:rows] if self.gemm else None
        for layer in range(self.L):
            if self.gemm:
                torch.matmul(x, self.w[0])
            self.ctx.prefill_batch(layer, pre, self.q, self.o)
            if self.gemm:
                torch.matmul(x, self.w[1])
                torch.matmul(x, self.w[2])
                torch.matmul(self.h[:rows], self.w[3])


class DecoderModel:
    """--model: the step is a real forward pass of a random-weight Llama-3-8B-shaped decoder
    (paper_2604_16395_b200.model, NEXT-4): per layer the projections produce the chunk's Q/K/V
    and one s2l_prefill_append stores K/V and computes the attention (token ids are synthetic:
    the weights are random)."""

    def __init__(self, ctx, layers):
        shape = M.Shape(layers=layers, hidden=HIDDEN, h_q=H_Q, h_kv=H_KV, d=D, inter=INTER)
        self.dec = M.StreamingDecoder(shape, ctx, seed=7)

    def step(self, items):
        its, toks, rows = [], [], 0
        for r, q_pos, n in items:
            its.append((r, q_pos, n, rows))
            toks.append((torch.arange(q_pos, q_pos + n) * 7919 + r * 104729) % 32768)
            rows += n
        self.dec.chunk(its, torch.cat(toks).cuda())


def run(trace, policy, streaming, args, cm, pools):
    gpool, cpool = pools
    cfg = s2l.make_config(args.layers, H_Q, H_KV, D, K, args.gpu_blocks, args.cpu_blocks,
                          max_requests=len({e[1] for e in trace}) + 1, max_blocks_per_request=32768 // K)
    ctx = s2l.Context(cfg, gpool, cpool, torch.cuda.current_stream(), None)
    sch = S.StreamingScheduler(ctx, policy, K, args.budget, args.gpu_blocks, cost_model=cm,
                               preemption=args.preemption if cm is not None or args.preemption != "cost" else "recompute",
                               streaming=streaming, feasibility=args.feasibility, default_lifo=args.default_lifo)
    model = DecoderModel(ctx, args.layers) if args.model else Model(ctx, args.layers, args.budget, args.gemm)
    t, i, steps, gpu_ms, host_s = 0.0, 0, 0, 0.0, 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    while True:
        while i < len(trace) and trace[i][0] <= t:
            tc, rid, n, tok, new, mode = trace[i]
            sch.on_chunk(tc, rid, n, tokens=tok, new_input=new, mode=mode)
            i += 1
        h0 = time.perf_counter()
        items = sch.step(t)
        host_s += time.perf_counter() - h0
        if not items:
            if i >= len(trace):
                break
            t = trace[i][0]
            continue
        e0.record()
        model.step(items)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        gpu_ms += ms
        t += ms * 1e-3
        steps += 1
        sch.finish_step(t, items)
    ctx.close()
    tt = list(sch.ttfts().values())
    ev = [e[1] for e in sch.events]
    return {"policy": policy if streaming else "NS", "requests": len(tt),
            "ttft_p50_s": S.percentile(tt, 50), "ttft_p95_s": S.percentile(tt, 95),
            "ttft_p99_s": S.percentile(tt, 99), "ttft_mean_s": float(np.mean(tt)) if tt else None,
            "trace_completion_s": t, "steps": steps, "gpu_busy_s": gpu_ms / 1e3, "sched_host_s": host_s,
            "preempt_swap": ev.count("PREEMPTED_SWAP"), "preempt_recompute": ev.count("PREEMPTED_RECOMPUTE"),
            "tokens_invalidated": int(sum(r.tokens_invalidated for r in sch.reqs.values()))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", choices=["crawler", "anns"])
    ap.add_argument("--qps", type=float, default=4.0)
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--budget", type=int, default=8192)
    ap.add_argument("--gpu-blocks", type=int, default=8192)
    ap.add_argument("--cpu-blocks", type=int, default=8192)
    ap.add_argument("--delay-scale", type=float, default=1.0)
    ap.add_argument("--gemm", action="store_true")
    ap.add_argument("--feasibility", choices=["pool", "free"], default="pool",
                    help="Phase-1 rule: pool (reading Z18, the round-1 tables) or free (SPEC S:L325)")
    ap.add_argument("--default-lifo", action="store_true", help="DEFAULT evicts LIFO over its running order (S:L335)")
    ap.add_argument("--model", action="store_true",
                    help="real decoder forward (random weights) through the per-layer fused API")
    ap.add_argument("--preemption", default="cost", choices=["cost", "recompute", "swap"])
    ap.add_argument("--policies", default="NS,DEFAULT,FCFS,MCPS,LCAS")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    seed = 2026
    tr = (traces.crawler_trace if args.workload == "crawler" else traces.anns_trace)(
        seed, args.n, args.qps, delay_scale=args.delay_scale)
    # cost model matching the simulated prefill: with --gemm the full-prefill profile (attention +
    # append + dense layers), else attention + append only
    cmp = os.path.join(ROOT, "profiles", "r01",
                       "costmodel_b200_full.json" if (args.gemm or args.model) else "costmodel_b200.json")
    cm = costmodel.CostModel.load(cmp) if os.path.exists(cmp) else None
    mb = 2 * args.layers * K * H_KV * D * 2
    gpool = torch.empty(args.gpu_blocks * mb // 2, dtype=torch.bfloat16, device="cuda")
    cpool = torch.empty(args.cpu_blocks * mb // 2, dtype=torch.bfloat16, pin_memory=True)
    out = {"workload": f"TTFT {args.workload} trace (synthetic, synth/traces.py)", "qps": args.qps,
           "queries": args.n, "layers": args.layers, "gemm": args.gemm, "model": args.model, "budget": args.budget,
           "gpu_blocks": args.gpu_blocks, "cpu_blocks": args.cpu_blocks, "delay_scale": args.delay_scale,
           "cost_model": os.path.relpath(cmp, ROOT) if cm else None, "runs": []}
    for p in args.policies.split(","):
        res = run(tr, "DEFAULT" if p == "NS" else p, p != "NS", args, cm, (gpool, cpool))
        out["runs"].append(res)
        print(json.dumps(res), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
