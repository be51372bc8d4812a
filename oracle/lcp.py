"""Longest common prefix — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:L170 (§4.2): "computing the longest common prefix (LCP) between the old and new input
token sequences".  Reading Z6: 0-based positions; the LCP is the count of
equal leading tokens.  Pinned by tests/test_oracle_lcp.py (paper example P:L172-L178,
SPEC examples S:L71-L74, brute force, symmetry).
"""
from __future__ import annotations


def lcp(old, new) -> int:
    """p = max{i : old[0:i] == new[0:i]} by a plain element-by-element scan."""
    n = min(len(old), len(new))
    i = 0
    while i < n and int(old[i]) == int(new[i]):
        i += 1
    return i
