"""Per-step A/B of library builds on the C2 stream: python tools/step_ab.py A.so[:ENV=v,...] B.so ... [rounds]
Each build gets its own context; bench.c2_breakdown (median per step over 10 replays) is run
alternately per round; prints per-step TFLOP/s per build (median over rounds)."""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2604_16395_b200 import s2l  # noqa: E402

specs = [a for a in sys.argv[1:] if ".so" in a]
rounds = int(([a for a in sys.argv[1:] if a.isdigit()] or ["3"])[0])
torch.cuda.set_device(0)
rids, toks, data = bench.make_stream_data(0)
S = bench.Stream(rids, toks, data, "cuda:0")
ctxs = []
for spec in specs:
    path, _, envs = spec.partition(":")
    for kv in filter(None, envs.split(",")):
        k_, v_ = kv.split("=")
        os.environ[k_] = v_
    nblk = bench.NREQ * bench.TOTAL // bench.KB
    cfg = s2l.make_config(1, bench.H_Q, bench.H_KV, bench.D, bench.KB, nblk, 0, max_requests=bench.NREQ,
                          max_blocks_per_request=bench.TOTAL // bench.KB)
    pool = torch.empty(nblk * s2l.block_bytes(cfg) // 2, dtype=torch.bfloat16, device="cuda:0")
    ctxs.append((s2l.Context(cfg, pool, None, torch.cuda.current_stream(), None, lib_path=path), pool))
res = {s: [] for s in specs}
for _ in range(rounds):
    for spec, (ctx, _) in zip(specs, ctxs):
        res[spec].append(bench.c2_breakdown(ctx, S, reps=10)["step_tflops"])
for spec in specs:
    med = [statistics.median(x[j] for x in res[spec]) for j in range(S.steps)]
    print(f"{spec:45s}", " ".join(f"{m:6.0f}" for m in med))
