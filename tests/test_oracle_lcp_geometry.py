"""Pins of oracle.lcp and oracle.geometry against the paper, SPEC examples and brute force."""
import json
import os
import random

import pytest

from oracle.geometry import block_bytes, blocks_needed, kv_bytes
from oracle.lcp import lcp

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_paper_worked_example_units():
    g = _gold("paper_lcp_example.json")
    sym = {}
    old = [sym.setdefault(s, len(sym)) for s in g["old"]]
    new = [sym.setdefault(s, len(sym)) for s in g["new"]]
    assert lcp(old, new) == g["lcp"] == 1
    assert g["old"][: lcp(old, new)] == g["kept"]


def test_paper_worked_example_tokens():
    """Same example at token level: documents are token runs; d2' differs in its first token."""
    rng = random.Random(7)
    d1 = [rng.randrange(1000) for _ in range(37)]
    d2 = [rng.randrange(1000) for _ in range(50)]
    d2p = [d2[0] + 1] + d2[1:]
    q, o1, o2 = [5, 6, 7], [8], [9, 10]
    old = d1 + d2 + q + o1 + o2
    new = d1 + d2p + q + o1 + o2
    assert lcp(old, new) == len(d1)


@pytest.mark.parametrize("a,b,expect", [
    ([], [1, 2], 0),                 # S:L73 empty prefix
    ([1, 2, 3], [1, 2, 3], 3),       # S:L72 identity
    ([1, 2, 3], [1, 2, 3, 4], 3),    # append: LCP = old length
    ([1, 2, 3, 4], [1, 2], 2),
    ([9, 2, 3], [1, 2, 3], 0),       # S:L84 change at position 0
])
def test_spec_examples(a, b, expect):
    assert lcp(a, b) == expect


def _brute(a, b):
    best = 0
    for i in range(min(len(a), len(b)) + 1):
        if all(a[j] == b[j] for j in range(i)):
            best = i
    return best


def test_bruteforce_10000_pairs():
    """S:L613 acceptance #8: 10,000 random pairs equal a brute-force prefix check; symmetry."""
    rng = random.Random(1)
    for _ in range(10000):
        n = rng.randrange(0, 24)
        a = [rng.randrange(3) for _ in range(n)]
        if rng.random() < 0.5:
            b = a[: rng.randrange(0, n + 1)] + [rng.randrange(3) for _ in range(rng.randrange(0, 8))]
        else:
            b = [rng.randrange(3) for _ in range(rng.randrange(0, 24))]
        p = lcp(a, b)
        assert p == _brute(a, b)
        assert p == lcp(b, a)
    assert lcp(a, a) == len(a)


def test_geometry_paper_numbers():
    g = _gold("geometry.json")
    m = g["llama31_8b"]
    d_head = m["d_model"] // m["h"]
    assert d_head == m["d_head"]
    # M_KV(32K) ≈ 4.0 GB — exactly 4 GiB
    assert kv_bytes(32768, m["L"], m["h_kv"], d_head, m["b"]) == g["m_kv_32k"]["bytes"]
    assert abs(g["m_kv_32k"]["bytes"] / 2**30 - 4.0) < 1e-12
    # "typical block sizes 2 MB" for k = 16
    assert block_bytes(m["L"], 16, m["h_kv"], d_head, m["b"]) == g["m_block_k16"]["bytes"]
    c = g["c1_block"]
    assert block_bytes(c["L"], c["k"], c["h_kv"], c["d_head"]) == c["bytes"]
    for tok, k, nb in g["blocks_needed"]["cases"]:
        assert blocks_needed(tok, k) == nb


def test_geometry_linearity():
    # S:L140 k=1 vs k=16 -> exactly 1/16; kv_bytes(k tokens) = block_bytes
    assert block_bytes(32, 16, 8, 128) == 16 * block_bytes(32, 1, 8, 128)
    assert kv_bytes(16, 32, 8, 128) == block_bytes(32, 16, 8, 128)
    assert kv_bytes(0, 32, 8, 128) == 0
    assert block_bytes(1, 1, 1, 1, 1) == 2
