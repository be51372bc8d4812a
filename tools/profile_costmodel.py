"""Profiles the B200 recompute and swap latency curves with libs2l and fits the cost model
(NEXT-1; the paper's Fig. 5 / P:L188 for this hardware):

  recompute_latency(T): append + chunked-prefill attention of T tokens from an empty cache,
      Llama-3.1-8B KV geometry (32 q / 8 kv heads, d 128, k 16), 8192-token chunks (the paper's
      largest token budget), one layer measured and scaled by L = 32 layers
      (attention + KV write only: the model GEMMs of the paper's C_prefill are out of scope);
  swap_latency(C): s2l_swap_out then s2l_swap_in of C blocks of M_block = 2 MiB (L = 32,
      P:L188 "2 MB"), per direction, on the copy stream.

  --gemm: the recompute curve also runs the Llama-3-8B dense layers of the same tokens as
      cuBLAS bf16 GEMMs with random weights (QKV, O, gate/up, down per layer), i.e. the whole
      C_prefill of the paper -- library GEMMs, not this repo's kernels.

    python tools/profile_costmodel.py [out.json] [--gemm]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_16395_b200 import s2l  # noqa: E402
from paper_2604_16395_b200.costmodel import CostModel, PiecewiseLinear  # noqa: E402
from synth import workloads as W  # noqa: E402

L_MODEL, H_Q, H_KV, D, K = 32, 32, 8, 128, 16
CHUNK = 8192


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).view(torch.bfloat16).cuda()


HIDDEN, INTER = 4096, 14336


class Dense:
    """Per-layer dense work of Llama-3-8B for n tokens (cuBLAS bf16, random weights)."""

    def __init__(self, nmax):
        g = torch.Generator(device="cuda").manual_seed(1)
        mk = lambda a, b: (torch.randn(a, b, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
        self.w = [mk(HIDDEN, (H_Q + 2 * H_KV) * D), mk(H_Q * D, HIDDEN), mk(HIDDEN, 2 * INTER), mk(INTER, HIDDEN)]
        self.x = mk(nmax, HIDDEN)
        self.h = mk(nmax, INTER)

    def layer(self, n):
        torch.matmul(self.x[:n], self.w[0])
        torch.matmul(self.x[:n], self.w[1])
        torch.matmul(self.x[:n], self.w[2])
        torch.matmul(self.h[:n], self.w[3])


def recompute_point(T, q, k, v, dense=None):
    cfg = s2l.make_config(1, H_Q, H_KV, D, K, T // K + 8, 0, max_requests=1, max_blocks_per_request=T // K + 8)
    pool = torch.empty(cfg.num_gpu_blocks * s2l.block_bytes(cfg) // 2, dtype=torch.bfloat16, device="cuda")
    ctx = s2l.Context(cfg, pool, None, torch.cuda.current_stream(), None)
    chunks = [(a, min(CHUNK, T - a)) for a in range(0, T, CHUNK)]
    Q = [dev(q[a:a + n]) for a, n in chunks]
    Kd = [dev(k[:, a:a + n]) for a, n in chunks]
    Vd = [dev(v[:, a:a + n]) for a, n in chunks]
    O = [torch.empty_like(x) for x in Q]

    def once():
        ctx.new_request(0, np.zeros(T, np.int32))
        for (a, n), qq, kk, vv, oo in zip(chunks, Q, Kd, Vd, O):
            ctx.append_chunk([(0, None, n, 0)], kk, vv)
            ctx.prefill_batch(0, [(0, a, n, 0)], qq, oo)
            if dense is not None:
                dense.layer(n)
        ctx.release(0)

    for _ in range(2):
        once()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        once()
    e1.record()
    torch.cuda.synchronize()
    ctx.close()
    return e0.elapsed_time(e1) / reps * 1e-3          # seconds per layer


def swap_points(counts):
    nmax = max(counts)
    cfg = s2l.make_config(L_MODEL, H_Q, H_KV, D, K, nmax + 8, nmax + 8, max_requests=2, max_blocks_per_request=nmax + 8)
    mb = s2l.block_bytes(cfg)
    gp = torch.empty((nmax + 8) * mb // 2, dtype=torch.bfloat16, device="cuda")
    cp = torch.empty((nmax + 8) * mb // 2, dtype=torch.bfloat16).pin_memory()
    cs, cs_in = torch.cuda.Stream(), torch.cuda.Stream()      # swap-out / swap-in streams
    ctx = s2l.Context(cfg, gp, cp, torch.cuda.current_stream(), cs, swap_in_stream=cs_in)
    kv = torch.zeros(L_MODEL, 1024, H_KV, D, dtype=torch.bfloat16, device="cuda")
    out = {}
    for c in counts:
        ctx.new_request(1, np.zeros(c * K, np.int32))
        done = 0
        while done < c * K:
            n = min(1024, c * K - done)
            ctx.append_chunk([(1, None, n, 0)], kv, kv)
            done += n
        ctx.sync()
        best_o = best_i = 1e9
        for _ in range(3):
            e0, e1, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
            e0.record(cs)
            ctx.swap_out([1])
            e1.record(cs)
            ctx.sync()
            e2.record(cs_in)
            ctx.swap_in([1])
            e3.record(cs_in)
            ctx.sync()
            best_o = min(best_o, e0.elapsed_time(e1) * 1e-3)
            best_i = min(best_i, e2.elapsed_time(e3) * 1e-3)
        out[c] = (best_o, best_i)
        ctx.release(1)
    ctx.close()
    return out, mb


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    gemm = "--gemm" in sys.argv
    path = args[0] if args else os.path.join(ROOT, "gpurun_out", "costmodel_b200%s.json" % ("_full" if gemm else ""))
    torch.cuda.set_device(0)
    Ts = [1024 * 2 ** i for i in range(8)]                # 1K .. 128K
    toks = W.request_tokens(W.seed_of(4), 0, Ts[-1])
    q, k, v = W.request_qkv(W.seed_of(4), toks, W.LLAMA3_8B)
    dense = Dense(CHUNK) if gemm else None
    rec = [recompute_point(T, q[:T], k[:, :T], v[:, :T], dense) * L_MODEL for T in Ts]
    counts = [1, 8, 64, 256, 512, 1024]
    sw, mb = swap_points(counts)
    swap_s = [0.5 * (sw[c][0] + sw[c][1]) for c in counts]
    cm = CostModel(K, PiecewiseLinear(Ts, rec), PiecewiseLinear(counts, swap_s),
                   {"gpu": torch.cuda.get_device_name(0), "m_block_bytes": mb, "layers": L_MODEL,
                    "recompute": ("append + chunked-prefill attention + cuBLAS dense layers (random weights)"
                                  if gemm else "append + chunked-prefill attention only (no model GEMMs)")
                                 + ", 8192-token chunks",
                    "swap_out_s": {c: sw[c][0] for c in counts}, "swap_in_s": {c: sw[c][1] for c in counts}})
    cm.save(path)
    print(json.dumps({"recompute_s": dict(zip(Ts, rec)), "swap_s_per_direction": dict(zip(counts, swap_s)),
                      "crossover_tokens": cm.crossover_tokens(),
                      "decisions": {T: cm.choose_eviction(T) for T in Ts}}, indent=1))


if __name__ == "__main__":
    main()
