"""CPU tests of libs2l's host logic (no GPU): the ABI exports, and the bookkeeping of a
host-only context compared bit-exact with the oracle's state machine (block tables of both
tiers, nc, LCP, invalidated counts, total_tokens_invalidated, free counts, status codes,
swap bytes)."""
import json
import os
import random
import re

import numpy as np
import pytest

from oracle import kvcache as O
from oracle.kvcache import OracleKV
from paper_2604_16395_b200 import s2l

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2604_16395_b200 import build
    build.build()


def test_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "s2l.h")).read()
    declared = set(re.findall(r"\b(s2l_[a-z_]+)\s*\(", hdr))
    L = s2l.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert declared == set(s2l.EXPORTS)
    assert b"sm_100a" in L.s2l_version()


def test_block_bytes_matches_paper_formula():
    # P:L73 / P:L188: 2 MiB for Llama-3.1-8B, k = 16, all 32 layers
    cfg = s2l.make_config(32, 32, 8, 128, 16, 1, 0)
    assert s2l.block_bytes(cfg) == 2 * 1024 * 1024
    assert s2l.block_bytes(s2l.make_config(1, 2, 1, 16, 4, 1, 0)) == 256
    # FP8 KV cache (kv_dtype 1): b = 1 byte per value instead of P:L63's 2
    assert s2l.block_bytes(s2l.make_config(32, 32, 8, 128, 16, 1, 0, kv_dtype=1)) == 1024 * 1024


def test_config_validation():
    for bad in [s2l.make_config(1, 3, 2, 16, 4, 8, 8),        # h % h_kv
                s2l.make_config(1, 2, 1, 12, 4, 8, 8),        # head_dim % 8
                s2l.make_config(1, 2, 1, 16, 3, 8, 8),        # block not power of two
                s2l.make_config(1, 2, 1, 16, 4, 8, 8, lcp_block_aligned=2),
                s2l.make_config(1, 2, 1, 16, 4, 8, 8, alloc_cooling=2),
                s2l.make_config(1, 2, 1, 16, 4, 8, 8, kv_dtype=2),
                # token positions / table indices are 32-bit on the device
                s2l.make_config(1, 2, 1, 16, 256, 8, 8, max_blocks_per_request=1 << 23),
                s2l.make_config(1, 2, 1, 16, 4, 8, 8, max_requests=1 << 16, max_blocks_per_request=1 << 15)]:
        with pytest.raises(s2l.S2LError) as e:
            s2l.Context(bad, host_only=True)
        assert e.value.status == s2l.E_INVAL
    # the largest accepted geometry just below both limits
    s2l.Context(s2l.make_config(1, 2, 1, 16, 256, 8, 8, max_requests=1,
                                max_blocks_per_request=(1 << 23) - 1), host_only=True).close()


def _pair(L=1, h_q=2, h_kv=1, d=16, k=4, ng=8, nc=8, aligned=False, max_requests=64, max_blocks=None,
          cooling=False):
    cfg = s2l.make_config(L, h_q, h_kv, d, k, ng, nc, max_requests=max_requests,
                          max_blocks_per_request=max_blocks or (ng + nc), lcp_block_aligned=int(aligned),
                          alloc_cooling=int(cooling))
    lib = s2l.Context(cfg, host_only=True)
    ora = OracleKV(L, h_q, h_kv, d, k, ng, nc, max_requests=max_requests,
                   max_blocks_per_request=max_blocks or (ng + nc), lcp_block_aligned=aligned,
                   mirror_pools=False, alloc_cooling=cooling)
    return lib, ora


def _same_state(lib, ora):
    assert lib.free_blocks() == ora.free_counts()
    for rid in ora.reqs:
        assert lib.query(rid) == ora.info(rid), rid
        assert lib.block_table(rid) == ora.block_table(rid), rid


@pytest.mark.parametrize("aligned,cooling", [(False, False), (True, False), (False, True)])
def test_c1_walk_matches_oracle(aligned, cooling):
    lib, ora = _pair(aligned=aligned, cooling=cooling)
    toks = list(range(100, 124))
    for x in (lib, ora):
        x.new_request(1, [])
    z = np.zeros((1, 8, 1, 16), np.uint16)
    for i in range(3):
        lib.append_chunk([(1, toks[8 * i: 8 * i + 8], 8, 0)], kv_rows=8)
        assert ora.append([(1, toks[8 * i: 8 * i + 8], 8, 0)], z, z) == O.OK
        _same_state(lib, ora)
    new = toks[:10] + [999] + list(range(500, 513))
    st, p, inv = ora.invalidate_lcp(1, new)
    assert lib.invalidate_lcp(1, new) == (p, inv) == (10, 16 if aligned else 14)
    _same_state(lib, ora)
    n = 24 - lib.query(1)["num_computed"]
    lib.append_chunk([(1, None, n, 0)], kv_rows=n)
    ora.append([(1, None, n, 0)], np.zeros((1, n, 1, 16), np.uint16), np.zeros((1, n, 1, 16), np.uint16))
    _same_state(lib, ora)
    assert lib.swap_out([1]) == ora.swap_out([1])[1] == 6 * 256
    _same_state(lib, ora)
    assert lib.swap_in([1]) == ora.swap_in([1])[1]
    _same_state(lib, ora)
    # the hand-derived golden of each allocation order (tests/golden/c1_walk.json)
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "c1_walk.json")))
    if not aligned:
        assert lib.block_table(1) == gold["swap_in_alloc_cooling" if cooling else "swap_in"]["gpu_table"]


def test_spec_invalidate_numbers_via_library():
    # S:L194-L196 (aligned): computed 2048, k 16, lcp 100 -> 96 / 1952 / 122 freed
    for aligned, exp in ((True, (96, 1952, 122)), (False, (100, 1948, 121))):
        lib, _ = _pair(L=1, h_q=1, h_kv=1, d=8, k=16, ng=200, nc=0, aligned=aligned)
        toks = list(range(2048))
        lib.new_request(0, toks)
        lib.append_chunk([(0, None, 2048, 0)], kv_rows=2048)
        g0 = lib.free_blocks()[0]
        p, inv = lib.invalidate_lcp(0, toks[:100] + [-1] * 1948)
        assert (lib.query(0)["num_computed"], inv, lib.free_blocks()[0] - g0) == exp
        assert p == 100


def _apply(x, op, args):
    """Run op on library or oracle, return (status, result)."""
    is_lib = isinstance(x, s2l.Context)
    if op == "new":
        rid, toks = args
        return (s2l.status_of(x.new_request, rid, toks), None) if is_lib else (x.new_request(rid, toks), None)
    if op == "append":
        items = args
        if is_lib:
            return s2l.status_of(x.append_chunk, items, kv_rows=64), None
        z = np.zeros((1, 64, 1, 16), np.uint16)
        return x.append(items, z, z), None
    if op == "inval":
        rid, new = args
        if is_lib:
            try:
                return s2l.OK, x.invalidate_lcp(rid, new)
            except s2l.S2LError as e:
                return e.status, None
        st, p, inv = x.invalidate_lcp(rid, new)
        return st, ((p, inv) if st == O.OK else None)
    if op in ("swap_out", "swap_in"):
        rids = args
        if is_lib:
            try:
                return s2l.OK, getattr(x, op)(rids)
            except s2l.S2LError as e:
                return e.status, None
        st, b = getattr(x, op)(rids)
        return st, (b if st == O.OK else None)
    if op == "release":
        return (s2l.status_of(x.release, args), None) if is_lib else (x.release(args), None)
    if op == "preempt":
        return (s2l.status_of(x.preempt_recompute, args), None) if is_lib else (x.preempt_recompute(args), None)
    raise ValueError(op)


@pytest.mark.parametrize("aligned,cooling", [(False, False), (True, False), (False, True)])
def test_fuzz_10000_steps_bit_exact(aligned, cooling):
    """Random interleavings of every bookkeeping call: library == oracle after every step,
    under Z9's plain order and the opt-in alloc_cooling order."""
    rng = random.Random(11 + aligned + 2 * cooling)
    lib, ora = _pair(L=1, h_q=2, h_kv=1, d=16, k=4, ng=24, nc=16, aligned=aligned, max_requests=5,
                     max_blocks=12, cooling=cooling)
    for step in range(10000):
        op = rng.choice(["new", "append", "append", "append", "inval", "swap_out", "swap_in",
                         "release", "preempt"])
        rid = rng.randrange(7)
        if op == "new":
            args = (rid, [rng.randrange(3) for _ in range(rng.randrange(0, 6))])
        elif op == "append":
            items = []
            for r in rng.sample(range(7), rng.randrange(1, 3)):
                toks = [rng.randrange(3) for _ in range(rng.randrange(0, 6))] if rng.random() < 0.7 else None
                pend = (len(ora.reqs[r].input) - ora.reqs[r].nc) if r in ora.reqs else 0
                n_kv = rng.randrange(0, pend + (len(toks) if toks else 0) + 2)
                items.append((r, toks, n_kv, rng.randrange(0, 8)))
            if rng.random() < 0.05:
                items.append(items[0])                      # duplicate -> E_INVAL
            args = items
        elif op == "inval":
            base = ora.reqs[rid].input if rid in ora.reqs else []
            args = (rid, list(base[: rng.randrange(0, len(base) + 1)]) + [rng.randrange(3) for _ in range(rng.randrange(0, 8))])
        elif op in ("swap_out", "swap_in"):
            args = rng.sample(range(7), rng.randrange(0, 3))
        else:
            args = rid
        a = _apply(lib, op, args)
        b = _apply(ora, op, args)
        assert a == b, (step, op, args, a, b)
        _same_state(lib, ora)


def test_z9_plain_lowest_free_id_independent_of_free_order():
    """Reading Z9 (default): the lowest free ids, ascending, whatever order they were freed
    in -- ids released by a swap-out are reused at once.  Hand-derived tables."""
    lib, ora = _pair(ng=12, nc=12, max_blocks=12)
    z = np.zeros((1, 64, 1, 16), np.uint16)
    for x in (lib, ora):
        x.new_request(1, list(range(16)))
        x.new_request(2, list(range(32)))
        x.new_request(3, list(range(8)))
    lib.append_chunk([(3, None, 8, 0)], kv_rows=64)             # ids 0-1
    ora.append([(3, None, 8, 0)], z, z)
    lib.append_chunk([(1, None, 16, 0)], kv_rows=64)            # ids 2-5
    ora.append([(1, None, 16, 0)], z, z)
    assert lib.swap_out([1]) == ora.swap_out([1])[1]             # frees 2-5
    lib.release(3); ora.release(3)                               # frees 0-1 (later)
    lib.append_chunk([(2, None, 24, 0)], kv_rows=64)            # 6 blocks: 0-5, ascending
    ora.append([(2, None, 24, 0)], z, z)
    assert lib.block_table(2) == ora.block_table(2) == [0, 1, 2, 3, 4, 5]
    assert lib.swap_in([1]) == ora.swap_in([1])[1]               # 6-9
    assert lib.block_table(1) == ora.block_table(1) == [6, 7, 8, 9]
    assert lib.free_blocks() == ora.free_counts() == (2, 12)


def test_alloc_cooling_ids_released_by_the_last_swap_out_are_allocated_last():
    """Opt-in alloc_cooling (a performance variant of Z9, not the paper's): the GPU ids
    released by the most recent swap-out come after every other free id; they become
    ordinary free ids at the next swap-out.  Library and oracle agree on every table."""
    lib, ora = _pair(ng=12, nc=12, max_blocks=12, cooling=True)
    z = np.zeros((1, 64, 1, 16), np.uint16)
    for x in (lib, ora):
        x.new_request(1, list(range(16)))
        x.new_request(2, list(range(32)))
    lib.append_chunk([(1, None, 16, 0)], kv_rows=64)            # ids 0-3
    ora.append([(1, None, 16, 0)], z, z)
    assert lib.swap_out([1]) == ora.swap_out([1])[1]             # 0-3 cooling
    lib.append_chunk([(2, None, 32, 0)], kv_rows=64)            # 8 blocks: 4-11 first, then none cooling
    ora.append([(2, None, 32, 0)], z, z)
    assert lib.block_table(2) == ora.block_table(2) == list(range(4, 12))
    assert lib.swap_in([1]) == ora.swap_in([1])[1]               # only cooling ids left: 0-3
    assert lib.block_table(1) == ora.block_table(1) == [0, 1, 2, 3]
    # next swap-out thaws the previous cooling set: request 2's ids cool, request 1 comes back
    # into the lowest ordinary free ids
    assert lib.swap_out([2]) == ora.swap_out([2])[1]
    assert lib.swap_out([1]) == ora.swap_out([1])[1]             # 2's ids thaw, 1's ids cool
    assert lib.swap_in([2]) == ora.swap_in([2])[1]
    assert lib.block_table(2) == ora.block_table(2) == list(range(4, 12))
    assert lib.free_blocks() == ora.free_counts()


def test_z19_token_only_append_on_the_cpu_tier():
    """Reading Z19: input keeps arriving while a request is swapped out; a
    token-only append (n_kv = 0) is valid on either tier, K/V writes need the GPU tier."""
    lib, ora = _pair(ng=8, nc=8, max_blocks=8)
    z = np.zeros((1, 16, 1, 16), np.uint16)
    for x in (lib, ora):
        x.new_request(3, [1, 2, 3, 4, 5, 6, 7, 8])
    lib.append_chunk([(3, None, 8, 0)], kv_rows=16)
    ora.append([(3, None, 8, 0)], z, z)
    assert lib.swap_out([3]) == ora.swap_out([3])[1]
    assert s2l.status_of(lib.append_chunk, [(3, [9, 10, 11], 0, 0)], kv_rows=16) == s2l.OK
    assert ora.append([(3, [9, 10, 11], 0, 0)], z, z) == O.OK
    assert lib.query(3) == ora.info(3) and lib.query(3)["num_tokens"] == 11
    assert s2l.status_of(lib.append_chunk, [(3, None, 3, 0)], kv_rows=16) == s2l.E_STATE
    assert ora.append([(3, None, 3, 0)], z, z) == O.E_STATE
    assert lib.swap_in([3]) == ora.swap_in([3])[1]
    lib.append_chunk([(3, None, 3, 0)], kv_rows=16)
    ora.append([(3, None, 3, 0)], z, z)
    assert lib.query(3) == ora.info(3) and lib.query(3)["num_computed"] == 11
    assert lib.block_table(3) == ora.block_table(3)


def test_binding_refuses_strided_tensors():
    """The ABI takes dense row-major arrays: a strided view (e.g. the V columns of a fused QKV
    projection output) must be refused by the binding instead of being read as dense rows."""
    import torch
    qkv = torch.zeros(4, 3 * 8, dtype=torch.bfloat16)
    v = qkv[:, 16:].view(4, 1, 8)
    assert not v.is_contiguous()
    with pytest.raises(ValueError):
        s2l._ptr(v)
    assert s2l._ptr(v.contiguous()) is not None
    assert s2l._ptr(None) is None
