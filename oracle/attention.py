"""Causal GQA attention in fp64 — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What it computes (the plain definition):
  P:L59 (§2.1)  prefill "computing attention scores" for token positions;
  P:L69 (§2.2)  "For computing attention at position t, the system retrieves all blocks
                {B_1..B_⌈t/k⌉} containing KV pairs for positions [1, t]" — i.e. query t
                attends causally to keys 1..t (reading Z3: a chunk's query row t sits at
                absolute position q_pos + t and sees keys 0..q_pos+t inclusive);
  P:L63 (§2.1)  GQA: h_kv < h key/value heads; reading Z2: q head h reads kv head
                g(h) = floor(h / (h/h_kv));
  reading Z1    softmax scale 1/sqrt(d_head).
For row t, head h:  s_j = q·K_j / sqrt(d) (j <= q_pos+t),  m = max s,
  O = Σ exp(s_j - m) V_j / Σ exp(s_j - m),  LSE = m + ln Σ exp(s_j - m).
K/V here are the request's CONTIGUOUS rows (not the paged pool): the oracle never reads
the block table for attention, so a paging bug cannot hide in both sides.
Library primitives used as steps: numpy matmul, exp, log (fp64).
Pinned by tests/test_oracle_attention.py (closed forms, pure-Python brute force,
torch fp64 SDPA with an explicit mask, chunked == one-shot).
"""
from __future__ import annotations

import numpy as np


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """Exact decoding of bf16 bit patterns (uint16) to float64."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32).astype(np.float64)


def attention(q_bits: np.ndarray, k_bits: np.ndarray, v_bits: np.ndarray, q_pos: int):
    """Causal GQA attention of one chunk.

    q_bits : [n][h_q][d] bf16 bits — query rows of positions q_pos .. q_pos+n-1
    k_bits, v_bits : [T][h_kv][d] bf16 bits — the request's keys/values, T >= q_pos+n
    returns (O [n][h_q][d] float64, LSE [n][h_q] float64 natural log)
    """
    n, h_q, d = q_bits.shape
    h_kv = k_bits.shape[1]
    assert h_q % h_kv == 0
    group = h_q // h_kv
    T = q_pos + n
    assert k_bits.shape[0] >= T and v_bits.shape[0] >= T
    q = bf16_to_f64(q_bits)
    k = bf16_to_f64(k_bits[:T])
    v = bf16_to_f64(v_bits[:T])
    out = np.zeros((n, h_q, d), dtype=np.float64)
    lse = np.zeros((n, h_q), dtype=np.float64)
    if n == 0:
        return out, lse
    key_pos = np.arange(T)[None, :]
    row_pos = (q_pos + np.arange(n))[:, None]
    visible = key_pos <= row_pos                      # keys 1..t (0-based: 0..q_pos+t)
    scale = 1.0 / np.sqrt(d)                          # Z1
    for h in range(h_q):
        g = h // group                                # Z2
        s = (q[:, h, :] @ k[:, g, :].T) * scale       # s_j = q·K_j / sqrt(d)
        s = np.where(visible, s, -np.inf)
        m = s.max(axis=1, keepdims=True)
        w = np.exp(s - m)                             # exp(-inf) = 0 for masked keys
        l = w.sum(axis=1, keepdims=True)
        out[:, h, :] = (w @ v[:, g, :]) / l
        lse[:, h] = (m + np.log(l))[:, 0]
    return out, lse


def attention_rows(q_bits: np.ndarray, k_bits: np.ndarray, v_bits: np.ndarray, q_pos: int,
                   rows) -> tuple[np.ndarray, np.ndarray]:
    """Same definition evaluated only at chunk rows `rows` (for sampled full-size parity).

    Returns (O [len(rows)][h_q][d], LSE [len(rows)][h_q]) in fp64.
    """
    rows = list(rows)
    n, h_q, d = q_bits.shape
    h_kv = k_bits.shape[1]
    group = h_q // h_kv
    out = np.zeros((len(rows), h_q, d), dtype=np.float64)
    lse = np.zeros((len(rows), h_q), dtype=np.float64)
    scale = 1.0 / np.sqrt(d)
    if not rows:
        return out, lse
    T = q_pos + max(rows) + 1
    k_all = bf16_to_f64(k_bits[:T])
    v_all = bf16_to_f64(v_bits[:T])
    for ri, t in enumerate(rows):
        i = q_pos + t
        k = k_all[: i + 1]
        v = v_all[: i + 1]
        q = bf16_to_f64(q_bits[t])
        for h in range(h_q):
            g = h // group
            s = (k[:, g, :] @ q[h]) * scale
            m = s.max()
            w = np.exp(s - m)
            l = w.sum()
            out[ri, h] = (w @ v[:, g, :]) / l
            lse[ri, h] = m + np.log(l)
    return out, lse
