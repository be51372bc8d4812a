"""Multi-GPU partitioning of the streaming-prefill path.

The path shards with no collective on the hot path:
  * by request (C2-C4): requests are independent units; `assign_requests` balances predicted
    attention FLOPs with longest-processing-time greedy (ties -> lower request id);
  * by KV head (C5, one long request): GQA groups are independent, so rank g owns kv heads
    [g*h_kv/N, (g+1)*h_kv/N) and their q heads; the output slices are disjoint.
NCCL (or gloo in CPU tests) is used only after timing: to reduce the max time and to gather
sampled output rows for the oracle check (`gather_rows`).  Host-side logic only.
"""
from __future__ import annotations

import heapq


def request_flops(n_tokens: int, chunk: int, h_q: int, d: int) -> float:
    """Causal attention FLOPs of prefilling n_tokens in `chunk`-token pieces (4·d·h_q per pair)."""
    total, p0 = 0.0, 0
    while p0 < n_tokens:
        n = min(chunk, n_tokens - p0)
        total += 4.0 * d * h_q * (n * p0 + n * (n + 1) / 2)
        p0 += n
    return total


def assign_requests(lengths: dict, world: int, chunk: int = 512, h_q: int = 32, d: int = 128) -> list:
    """LPT greedy: requests by descending predicted FLOPs, each to the least-loaded rank
    (ties -> lower rank); returns [sorted request ids of rank r for r in range(world)]."""
    order = sorted(lengths, key=lambda r: (-request_flops(lengths[r], chunk, h_q, d), r))
    heap = [(0.0, rank) for rank in range(world)]
    out = [[] for _ in range(world)]
    for rid in order:
        load, rank = heapq.heappop(heap)
        out[rank].append(rid)
        heapq.heappush(heap, (load + request_flops(lengths[rid], chunk, h_q, d), rank))
    return [sorted(x) for x in out]


def kv_head_shard(rank: int, world: int, h_q: int, h_kv: int):
    """(kv heads, q heads) owned by `rank` when one request is sharded by KV head."""
    if h_kv % world:
        raise ValueError(f"h_kv={h_kv} not divisible by world={world}")
    per = h_kv // world
    g = h_q // h_kv
    kv = list(range(rank * per, (rank + 1) * per))
    q = list(range(rank * per * g, (rank + 1) * per * g))
    return kv, q


def max_time(dist, ms: float, device=None) -> float:
    """Max over ranks of a per-rank time (the bench's whole-job clock)."""
    import torch
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(dist, rows, world: int):
    """All-gather equally shaped per-rank tensors of sampled output rows (checking only)."""
    import torch
    bufs = [torch.empty_like(rows) for _ in range(world)]
    dist.all_gather(bufs, rows)
    return bufs
