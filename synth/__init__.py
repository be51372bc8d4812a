"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no LCP, no allocation, no attention,
no swap). It only draws inputs: token ids, a per-position prefix hash, and Q/K/V rows
as bf16 bit patterns.  Both sides receive the same arrays; neither side's arithmetic
lives here (task rule ③: "only the seeded input generators serve both").

Recipe (reading Z10):
  * counter-based RNG: splitmix64 (Steele/Lea/Flood 2014 finaliser), all in uint64;
  * token ids uniform in [0, 128256) (Llama-3 vocabulary size);
  * prefix hash H_i = splitmix64(H_{i-1} xor token_i), H_{-1} = splitmix64(seed);
    so K/V/Q of position i depend on tokens[0..i] only and an update that keeps the
    first p tokens reproduces the first p rows bit for bit;
  * each Q/K/V element = an N(0,1) draw by Box-Muller from the 64-bit
    word x = splitmix64(H_i xor key(kind, layer, head, c)): u1 = (x>>32 + 0.5)/2^32,
    u2 = (x & 0xffffffff)/2^32, z = sqrt(-2 ln u1) cos(2 pi u2) (|z| <= 6.8),
    then scaled by `scale` (1 normally, 4 for the "peaky" variant that exercises the
    running-max rescale), rounded float64 -> float32 (RNE) -> bf16 (RNE).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

MASK64 = (1 << 64) - 1
VOCAB = 128256
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

KIND_Q, KIND_K, KIND_V = 0, 1, 2


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 on a uint64 array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def splitmix64_int(x: int) -> int:
    """Scalar splitmix64 on a Python int (same function as `splitmix64`)."""
    z = (x + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def tokens(seed: int, stream: int, n: int, start: int = 0) -> np.ndarray:
    """n token ids of token stream `stream`, positions [start, start+n), int32."""
    ctr = np.arange(start, start + n, dtype=np.uint64)
    base = np.uint64(splitmix64_int((seed * 0x100000001B3 + stream * 0x2545F4914F6CDD1D) & MASK64))
    with np.errstate(over="ignore"):
        r = splitmix64(ctr ^ base)
    return (r % np.uint64(VOCAB)).astype(np.int32)


def prefix_hashes(seed: int, toks: np.ndarray) -> np.ndarray:
    """H_i for every position of `toks` (uint64). Sequential chain (Z10)."""
    h = splitmix64_int(seed & MASK64)
    out = np.empty(len(toks), dtype=np.uint64)
    for i, t in enumerate(np.asarray(toks, dtype=np.int64).tolist()):
        h = splitmix64_int(h ^ (t & MASK64))
        out[i] = h
    return out


def f64_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """float64 -> float32 (RNE) -> bf16 (RNE) bit patterns as uint16 (finite inputs only)."""
    b = np.asarray(x, dtype=np.float64).astype(np.float32).view(np.uint32)
    bias = np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))
    return ((b + bias) >> np.uint32(16)).astype(np.uint16)


def _keys(seed: int, kind: int, layer: int, heads: np.ndarray, d: int) -> np.ndarray:
    """Per-(head, c) salt, uint64 [len(heads)][d]."""
    c = np.arange(d, dtype=np.uint64)[None, :]
    hh = np.asarray(heads, dtype=np.uint64)[:, None]
    base = (seed * 0x9E3779B1 + kind * 0x85EBCA77 + layer * 0xC2B2AE3D) & MASK64
    with np.errstate(over="ignore"):
        return splitmix64(np.uint64(base) + hh * np.uint64(1 << 20) + c)


def _rows_chunk(h: np.ndarray, keys: np.ndarray, scale: float) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = splitmix64(h[:, None, None] ^ keys[None, :, :])
    u1 = ((x >> np.uint64(32)).astype(np.float64) + 0.5) * (1.0 / 4294967296.0)
    u2 = (x & np.uint64(0xFFFFFFFF)).astype(np.float64) * (1.0 / 4294967296.0)
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2) * scale
    return f64_to_bf16_bits(z)


def rows(seed: int, kind: int, layer: int, hashes: np.ndarray, heads, d: int,
         scale: float = 1.0, threads: int | None = None) -> np.ndarray:
    """bf16 bits [len(hashes)][len(heads)][d] for positions with prefix hashes `hashes`."""
    heads = np.asarray(heads, dtype=np.int64)
    keys = _keys(seed, kind, layer, heads, d)
    n = len(hashes)
    out = np.empty((n, len(heads), d), dtype=np.uint16)
    if n == 0:
        return out
    per = max(1, (1 << 20) // max(1, len(heads) * d))
    spans = [(a, min(n, a + per)) for a in range(0, n, per)]
    if len(spans) == 1:
        out[:] = _rows_chunk(hashes, keys, scale)
        return out
    threads = threads or min(16, os.cpu_count() or 1)

    def work(span):
        a, b = span
        out[a:b] = _rows_chunk(hashes[a:b], keys, scale)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, spans))
    return out


def qkv(seed: int, hashes: np.ndarray, num_layers: int, num_q_heads: int, num_kv_heads: int,
        d: int, q_layer: int = 0, q_scale: float = 1.0):
    """Q [n][h_q][d] for layer `q_layer`; K, V [L][n][h_kv][d]; all bf16 bits (uint16)."""
    q = rows(seed, KIND_Q, q_layer, hashes, range(num_q_heads), d, q_scale)
    k = np.stack([rows(seed, KIND_K, l, hashes, range(num_kv_heads), d) for l in range(num_layers)])
    v = np.stack([rows(seed, KIND_V, l, hashes, range(num_kv_heads), d) for l in range(num_layers)])
    return q, k, v
