"""Times the append kernel alone (C2 pattern: 32 launches of 8 items x 512 tokens, Llama-3-8B
KV geometry) for one or more builds of libs2l:  python tools/append_bench.py A.so [B.so ...]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_16395_b200 import s2l  # noqa: E402


def run(path, reps=5):
    nreq, chunk, total = 8, 512, 16384
    cfg = s2l.make_config(1, 32, 8, 128, 16, nreq * total // 16, 0, max_requests=nreq,
                          max_blocks_per_request=total // 16)
    pool = torch.empty(cfg.num_gpu_blocks * s2l.block_bytes(cfg) // 2, dtype=torch.bfloat16, device="cuda")
    k = torch.randn(1, nreq * chunk, 8, 128, device="cuda").to(torch.bfloat16)
    v = torch.randn_like(k)
    best = None
    for _ in range(reps):
        ctx = s2l.Context(cfg, pool, None, torch.cuda.current_stream(), None, lib_path=path)
        for r in range(nreq):
            ctx.new_request(r, list(range(total)))
        ctx.set_timing(True)
        for j in range(total // chunk):
            ctx.append_chunk([(r, None, chunk, r * chunk) for r in range(nreq)], k, v)
        torch.cuda.synchronize()
        ti = ctx.timing_read()
        us = ti["append_ms"] * 1e3 / ti["append_launches"]
        best = us if best is None else min(best, us)
        ctx.close()
    gb = 2 * 2 * nreq * chunk * 8 * 128 * 2 / (best * 1e-6) / 1e9
    print(f"{os.path.basename(path):30s} {best:7.2f} us/launch  {gb:7.1f} GB/s (read + write)")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        run(p)
