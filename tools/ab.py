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


def main():
    libs = [a for a in sys.argv[1:] if a.endswith(".so")]
    rounds = int(([a for a in sys.argv[1:] if not a.endswith(".so")] or ["6"])[0])
    torch.cuda.set_device(0)
    rids, toks, data = bench.make_stream_data(0)
    S = bench.Stream(rids, toks, data, "cuda:0")
    ctxs = []
    for path in libs:
        nblk = bench.NREQ * bench.TOTAL // bench.KB
        cfg = s2l.make_config(1, bench.H_Q, bench.H_KV, bench.D, bench.KB, nblk, 0, max_requests=bench.NREQ,
                              max_blocks_per_request=bench.TOTAL // bench.KB)
        pool = torch.empty(nblk * s2l.block_bytes(cfg) // 2, dtype=torch.bfloat16, device="cuda")
        ctxs.append((s2l.Context(cfg, pool, None, torch.cuda.current_stream(), None, lib_path=path), pool))
    flops = bench.step_flops()
    res = {p: [] for p in libs}
    for r in range(rounds):
        for path, (ctx, _) in zip(libs, ctxs):
            ms = bench.timed(lambda: bench.run_step(ctx, S), 3, 2 if r == 0 else 1)
            res[path].append(flops * 3 / (ms * 1e-3) / 1e12)
    for path in libs:
        v = res[path]
        print(f"{os.path.basename(path):24s} median {statistics.median(v):8.1f}  min {min(v):8.1f}  max {max(v):8.1f} TFLOP/s")


if __name__ == "__main__":
    main()
