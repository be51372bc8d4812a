"""A/B timing of several builds of libs2l on the same device-resident C2 stream.

    S2L_NVCC_FLAGS=... python -m paper_2604_16395_b200.build --force; cp .../libs2l.so /tmp/A.so
    python tools/ab.py /tmp/A.so /tmp/B.so [rounds]

Each library gets its own context (same pool size, same inputs); the C2 stream step is
timed alternately A, B, A, B, ... and the median per library is printed (TFLOP/s).
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2604_16395_b200 import s2l  # noqa: E402


def c5_main(specs, rounds):
    """A/B on the C5 stream (BJ:L11: one 128K request, 2K chunks, 64q/8kv) -- attention
    kernel TFLOP/s per build, alternating builds per round (median)."""
    T, chunk, HQ, HKV, D, KB = 131072, 2048, 64, 8, 128, 16
    g = torch.Generator(device="cuda").manual_seed(1005)
    K = torch.randn(T, HKV, D, generator=g, device="cuda").to(torch.bfloat16)
    V = torch.randn(T, HKV, D, generator=g, device="cuda").to(torch.bfloat16)
    Q = torch.randn(T, HQ, D, generator=g, device="cuda").to(torch.bfloat16)
    nch = T // chunk
    Ks = [K[j * chunk:(j + 1) * chunk].unsqueeze(0).contiguous() for j in range(nch)]
    Vs = [V[j * chunk:(j + 1) * chunk].unsqueeze(0).contiguous() for j in range(nch)]
    Qs = [Q[j * chunk:(j + 1) * chunk].contiguous() for j in range(nch)]
    Os = [torch.empty_like(x) for x in Qs]
    flops = sum(bench.attn_flops(chunk, j * chunk, h_q=HQ) for j in range(nch))
    toks = list(range(T))
    ctxs = []
    for spec in specs:
        path, _, envs = spec.partition(":")
        for kv in filter(None, envs.split(",")):
            k_, v_ = kv.split("=")
            os.environ[k_] = v_
        cfg = s2l.make_config(1, HQ, HKV, D, KB, T // KB + 64, 0, max_requests=1, max_blocks_per_request=T // KB)
        pool = torch.empty(cfg.num_gpu_blocks * s2l.block_bytes(cfg) // 2, dtype=torch.bfloat16, device="cuda")
        ctxs.append((s2l.Context(cfg, pool, None, torch.cuda.current_stream(), None, lib_path=path), pool))
    res = {s: [] for s in specs}

    def stream(ctx):
        ctx.new_request(0, toks)
        for j in range(nch):
            ctx.append_chunk([(0, None, chunk, 0)], Ks[j], Vs[j])
            ctx.prefill_batch(0, [(0, j * chunk, chunk, 0)], Qs[j], Os[j])
        ctx.release(0)
    for ctx, _ in ctxs:
        stream(ctx)
    for _ in range(rounds):
        for spec, (ctx, _) in zip(specs, ctxs):
            ctx.set_timing(True)
            stream(ctx)
            ti = ctx.timing_read()
            ctx.set_timing(False)
            res[spec].append(flops / (ti["attn_ms"] * 1e-3) / 1e12)
    for spec in specs:
        v = res[spec]
        print(f"C5 {spec.split('/')[-1]:40s} attn kernel median {statistics.median(v):8.1f}  min {min(v):8.1f}  max {max(v):8.1f}")


def main():
    # specs: path.so[:ENV=VAL[,ENV=VAL]] (env applied while that context is created)
    specs = [a for a in sys.argv[1:] if ".so" in a]
    if "--c5" in sys.argv:
        torch.cuda.set_device(0)
        return c5_main(specs, int(([a for a in sys.argv[1:] if a.isdigit()] or ["5"])[0]))
    rounds = int(([a for a in sys.argv[1:] if a.isdigit()] or ["8"])[0])
    libs = specs
    torch.cuda.set_device(0)
    rids, toks, data = bench.make_stream_data(0)
    S = bench.Stream(rids, toks, data, "cuda:0")
    ctxs = []
    for spec in libs:
        path, _, envs = spec.partition(":")
        saved = {}
        for kv in filter(None, envs.split(",")):
            k, v = kv.split("=")
            saved[k] = os.environ.get(k)
            os.environ[k] = v
        nblk = bench.NREQ * bench.TOTAL // bench.KB
        # "KV=1" in a spec's env list: that context's pool is FP8 E4M3 (kv_dtype 1)
        cfg = s2l.make_config(1, bench.H_Q, bench.H_KV, bench.D, bench.KB, nblk, 0, max_requests=bench.NREQ,
                              max_blocks_per_request=bench.TOTAL // bench.KB,
                              kv_dtype=int(os.environ.get("KV", "0")))
        pool = torch.empty(nblk * s2l.block_bytes(cfg) // 2, dtype=torch.bfloat16, device="cuda")
        ctxs.append((s2l.Context(cfg, pool, None, torch.cuda.current_stream(), None, lib_path=path), pool))
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    # "FUSED=1" in a spec's env list: time bench.run_step_fused (NEXT-2) for that context
    step_fn = [bench.run_step_fused if "FUSED=1" in spec else bench.run_step for spec in libs]
    flops = bench.step_flops()
    res = {p: [] for p in libs}
    assert len(set(libs)) == len(libs), "specs must differ"
    for fn, (ctx, _) in zip(step_fn, ctxs):      # warm every context (clocks, caches)
        bench.timed(lambda: fn(ctx, S), 1, 4)
    for r in range(rounds):
        for path, fn, (ctx, _) in zip(libs, step_fn, ctxs):
            ms = bench.timed(lambda: fn(ctx, S), 3, 1)
            res[path].append(flops * 3 / (ms * 1e-3) / 1e12)
    kern = {}
    for path, fn, (ctx, _) in zip(libs, step_fn, ctxs):   # attention-kernel-only (per-launch events)
        ctx.set_timing(True)
        bench.timed(lambda: fn(ctx, S), 3, 0)
        ti = ctx.timing_read()
        ctx.set_timing(False)
        kern[path] = flops * 3 / (ti["attn_ms"] * 1e-3) / 1e12
    for path in libs:
        v = res[path]
        print(f"{path.split('/')[-1]:40s} median {statistics.median(v):8.1f}  min {min(v):8.1f}  max {max(v):8.1f} "
              f"TFLOP/s (step)  attn kernel {kern[path]:8.1f}")


if __name__ == "__main__":
    main()
