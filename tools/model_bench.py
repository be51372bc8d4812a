"""NEXT-4 measurement: a Llama-3-8B-shaped random-weight decoder (paper_2604_16395_b200.model,
32 layers) prefilled as a C2-like stream (8 requests x 512-token chunks) with the per-layer
fused append + attention (s2l_prefill_append); dense layers are cuBLAS bf16 GEMMs via torch.
Prints one JSON line: prefill tokens/s, model TFLOP/s, and the attention launches' share of the
device time (CUDA events around each libs2l launch).

    python tools/model_bench.py [--chunks 8] [--requests 8]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_16395_b200 import model as M  # noqa: E402
from paper_2604_16395_b200 import s2l  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", type=int, default=8)
    ap.add_argument("--requests", type=int, default=8)
    ap.add_argument("--chunk", type=int, default=512)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    shape = M.LLAMA3_8B
    total = args.chunks * args.chunk
    nblk = args.requests * total // 16 + 8
    cfg = s2l.make_config(shape.layers, shape.h_q, shape.h_kv, shape.d, 16, nblk, 0,
                          max_requests=args.requests, max_blocks_per_request=total // 16)
    pool = torch.empty(nblk * s2l.block_bytes(cfg) // 2, dtype=torch.bfloat16, device="cuda")
    ctx = s2l.Context(cfg, pool, None, torch.cuda.current_stream(), None)
    dec = M.StreamingDecoder(shape, ctx, seed=1)
    g = torch.Generator(device="cuda").manual_seed(2)
    toks = [torch.randint(0, 32768, (total,), generator=g, device="cuda") for _ in range(args.requests)]

    def stream(timing=False):
        for r in range(args.requests):
            ctx.new_request(r, toks[r].tolist())
        fl = 0.0
        for j in range(args.chunks):
            a = j * args.chunk
            items = [(r, a, args.chunk, r * args.chunk) for r in range(args.requests)]
            fl += dec.flops_per_chunk(items)
            dec.chunk(items, torch.cat([t[a:a + args.chunk] for t in toks]))
        for r in range(args.requests):
            ctx.release(r)
        return fl

    stream()                                  # warm-up (cuBLAS heuristics, clocks)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.set_timing(True)
    e0.record()
    fl = stream()
    e1.record()
    tinfo = ctx.timing_read()
    ctx.set_timing(False)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    tokens = args.requests * total
    print(json.dumps({
        "workload": f"NEXT-4: Llama-3-8B-shaped decoder (32 layers, random weights), {args.requests} requests x "
                    f"{args.chunk}-token chunks to {total}, per-layer s2l_prefill_append",
        "ms": ms, "prefill_tokens_per_s": tokens / (ms * 1e-3), "model_tflops": fl / (ms * 1e-3) / 1e12,
        "attention_ms": tinfo["attn_ms"], "attention_launches": tinfo["attn_launches"],
        "attention_share": tinfo["attn_ms"] / ms, "append_launches": tinfo["append_launches"]}))
    ctx.close()


if __name__ == "__main__":
    main()
