"""Times the append kernel alone (C2 pattern: 32 launches of 8 items x 512 tokens, Llama-3-8B
KV geometry, a distinct 16 MiB K/V input per launch so reads come from HBM, not L2) for one or
more builds / settings of libs2l:

    python tools/append_bench.py A.so[:ENV=VAL,...] [B.so[:ENV=VAL] ...]

Per-launch time from the library's CUDA events around each append launch (best of 5 streams)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_16395_b200 import s2l  # noqa: E402


def run(spec, reps=5):
    path, _, envs = spec.partition(":")
    saved = {}
    for kv in filter(None, envs.split(",")):
        k_, v_ = kv.split("=")
        saved[k_] = os.environ.get(k_)
        os.environ[k_] = v_
    nreq, chunk, total = 8, 512, 16384
    cfg = s2l.make_config(1, 32, 8, 128, 16, nreq * total // 16, 0, max_requests=nreq,
                          max_blocks_per_request=total // 16)
    pool = torch.empty(cfg.num_gpu_blocks * s2l.block_bytes(cfg) // 2, dtype=torch.bfloat16, device="cuda")
    ks = [torch.randn(1, nreq * chunk, 8, 128, device="cuda").to(torch.bfloat16) for _ in range(total // chunk)]
    vs = [torch.randn_like(k) for k in ks]
    best = None
    for _ in range(reps):
        ctx = s2l.Context(cfg, pool, None, torch.cuda.current_stream(), None, lib_path=path)
        for r in range(nreq):
            ctx.new_request(r, list(range(total)))
        ctx.set_timing(True)
        for j in range(total // chunk):
            ctx.append_chunk([(r, None, chunk, r * chunk) for r in range(nreq)], ks[j], vs[j])
        torch.cuda.synchronize()
        ti = ctx.timing_read()
        us = ti["append_ms"] * 1e3 / ti["append_launches"]
        best = us if best is None else min(best, us)
        ctx.close()
    for k_, v_ in saved.items():
        if v_ is None:
            os.environ.pop(k_, None)
        else:
            os.environ[k_] = v_
    gb = 2 * 2 * nreq * chunk * 8 * 128 * 2 / (best * 1e-6) / 1e9
    print(f"{spec:50s} {best:7.2f} us/launch  {gb:7.1f} GB/s (read + write)", flush=True)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        run(p)
