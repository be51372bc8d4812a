"""Run the C5 stream (BJ:L11: one 128K request, 2K-token chunks, 64q/8kv, block 16) once through
the library: 64 append + attention launches.  For ncu captures of one chunk's attention launch
(e.g. ncu -k regex:attn_tc2 -s 63 -c 1 python tools/c5_stream_once.py for the last chunk)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16395_b200 import s2l  # noqa: E402

T, chunk, HQ, HKV, D, KB = 131072, 2048, 64, 8, 128, 16
g = torch.Generator(device="cuda").manual_seed(1005)
K = torch.randn(T, HKV, D, generator=g, device="cuda").to(torch.bfloat16)
V = torch.randn(T, HKV, D, generator=g, device="cuda").to(torch.bfloat16)
Q = torch.randn(T, HQ, D, generator=g, device="cuda").to(torch.bfloat16)
O = torch.empty_like(Q)
cfg = s2l.make_config(1, HQ, HKV, D, KB, T // KB + 64, 0, max_requests=1, max_blocks_per_request=T // KB)
pool = torch.empty(cfg.num_gpu_blocks * s2l.block_bytes(cfg) // 2, dtype=torch.bfloat16, device="cuda")
ctx = s2l.Context(cfg, pool, None, torch.cuda.current_stream(), None)
ctx.new_request(0, list(range(T)))
for j in range(T // chunk):
    a = j * chunk
    ctx.append_chunk([(0, None, chunk, 0)], K[a:a + chunk].unsqueeze(0).contiguous(), V[a:a + chunk].unsqueeze(0).contiguous())
    ctx.prefill_batch(0, [(0, a, chunk, 0)], Q[a:a + chunk], O[a:a + chunk])
torch.cuda.synchronize()
print("c5 stream ok")
