"""KV byte formulas — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:L63 (§2.1): each token stores 2·L·d·(h_kv/h) values; M_KV = that × b bytes per token
  (reading Z8: the printed formula omits the factor ℓ; the "≈4.0 GB at 32K" example fixes it).
P:L67 (§2.2): a sequence of ℓ tokens occupies ⌈ℓ/k⌉ blocks.
P:L73 (§2.2): M_block = 2·L·k·d·(h_kv/h)·b.
With d = h·d_h this is 2·L·k·h_kv·d_h·b, the form used below.
"""
from __future__ import annotations


def blocks_needed(tokens: int, k: int) -> int:
    """⌈tokens/k⌉."""
    return -(-tokens // k)


def kv_bytes_per_token(L: int, h_kv: int, d_head: int, b: int = 2) -> int:
    """2·L·d·(h_kv/h)·b with d·(h_kv/h) = h_kv·d_head."""
    return 2 * L * h_kv * d_head * b


def kv_bytes(tokens: int, L: int, h_kv: int, d_head: int, b: int = 2) -> int:
    """M_KV(ℓ) = ℓ · 2·L·d·(h_kv/h)·b (reading Z8)."""
    return tokens * kv_bytes_per_token(L, h_kv, d_head, b)


def block_bytes(L: int, k: int, h_kv: int, d_head: int, b: int = 2) -> int:
    """M_block = 2·L·k·d·(h_kv/h)·b."""
    return 2 * L * k * h_kv * d_head * b
