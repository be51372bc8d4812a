"""Synthetic workload recipes C1-C5 (BASELINE.json configs) — input shapes
and stream schedules only (token counts, chunk sizes, LCP draws).  No method arithmetic.

Each request's tokens come from `synth.tokens(seed, request_id, n)`; update-mode inputs keep
the first p tokens and redraw the rest from another token stream (so new[p] != old[p] is
forced and LCP == p exactly).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import VOCAB, prefix_hashes, qkv, tokens


@dataclass(frozen=True)
class Geometry:
    L: int
    h_q: int
    h_kv: int
    d: int
    k: int


C1 = Geometry(L=1, h_q=2, h_kv=1, d=16, k=4)          # BJ:L7
LLAMA3_8B = Geometry(L=1, h_q=32, h_kv=8, d=128, k=16)  # BJ:L8/L9 (attention shape, one layer)
LLAMA3_70B = Geometry(L=1, h_q=64, h_kv=8, d=128, k=16)  # BJ:L11


def seed_of(config_index: int) -> int:
    """seed = 1000 + config index."""
    return 1000 + config_index


def request_tokens(seed: int, rid: int, n: int) -> np.ndarray:
    return tokens(seed, rid, n)


def updated_tokens(seed: int, rid: int, old: np.ndarray, p: int, new_len: int, round_: int) -> np.ndarray:
    """Update-mode input: old[:p] + fresh tokens, with new[p] != old[p] (so LCP == p)."""
    tail = tokens(seed, 100000 * (round_ + 1) + rid, max(0, new_len - p))
    new = np.concatenate([old[:p], tail]).astype(np.int32)
    if p < min(len(old), new_len) and new[p] == old[p]:
        new[p] = (new[p] + 1) % VOCAB
    return new


def c3_lcp_draws(seed: int, n_requests: int, total: int = 8192, round_: int = 0) -> np.ndarray:
    """Reading Z14: p uniform in [ceil(0.2*total), floor(0.8*total)]."""
    rng = np.random.default_rng(seed * 7919 + round_)
    lo, hi = -(-2 * total // 10), (8 * total) // 10
    return rng.integers(lo, hi + 1, size=n_requests)


def request_qkv(seed: int, toks: np.ndarray, geo: Geometry, q_scale: float = 1.0):
    """Q [n][h_q][d], K/V [L][n][h_kv][d] bf16 bits for every position of `toks` (Z10)."""
    H = prefix_hashes(seed, toks)
    return qkv(seed, H, geo.L, geo.h_q, geo.h_kv, geo.d, q_scale=q_scale)
