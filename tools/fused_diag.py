"""NEXT-2 diagnosis: per-kernel CUDA-event times of the C2 stream step, unfused (append kernel +
attention kernel per chunk) vs fused (one append + attention kernel per chunk), for one or
more builds side by side (alternating rounds).

    python tools/fused_diag.py ab_libs/new.so ab_libs/new.so:FUSED=1 [rounds]
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2604_16395_b200 import s2l  # noqa: E402


def main():
    specs = [a for a in sys.argv[1:] if ".so" in a]
    rounds = int(([a for a in sys.argv[1:] if ".so" not in a] or ["6"])[0])
    torch.cuda.set_device(0)
    rids, toks, data = bench.make_stream_data(0)
    S = bench.Stream(rids, toks, data, "cuda:0")
    nblk = bench.NREQ * bench.TOTAL // bench.KB
    runs = []
    for spec in specs:
        path = spec.partition(":")[0]
        cfg = s2l.make_config(1, bench.H_Q, bench.H_KV, bench.D, bench.KB, nblk, 0, max_requests=bench.NREQ,
                              max_blocks_per_request=bench.TOTAL // bench.KB)
        pool = torch.empty(nblk * s2l.block_bytes(cfg) // 2, dtype=torch.bfloat16, device="cuda")
        ctx = s2l.Context(cfg, pool, None, torch.cuda.current_stream(), None, lib_path=path)
        fn = bench.run_step_fused if "FUSED=1" in spec else bench.run_step
        runs.append((spec, ctx, pool, fn, {"step": [], "attn": [], "append": []}))
    for _, ctx, _, fn, _ in runs:
        for _ in range(3):
            fn(ctx, S)
    torch.cuda.synchronize()
    flops = bench.step_flops()
    for _ in range(rounds):
        for spec, ctx, _, fn, res in runs:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ctx.set_timing(True)
            e0.record()
            fn(ctx, S)
            e1.record()
            t = ctx.timing_read()
            ctx.set_timing(False)
            torch.cuda.synchronize()
            res["step"].append(e0.elapsed_time(e1))
            res["attn"].append(t["attn_ms"])
            res["append"].append(t["append_ms"])
    for spec, _, _, _, res in runs:
        st, at, ap = (statistics.median(res[k]) for k in ("step", "attn", "append"))
        print(f"{spec:32s} step {st:7.3f} ms ({flops / (st * 1e-3) / 1e12:7.1f} TFLOP/s)  "
              f"attention {at:7.3f} ms  append {ap:6.3f} ms")


if __name__ == "__main__":
    main()
