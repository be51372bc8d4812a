"""Pins of oracle.kvcache: hand-derived C1 walk, SPEC numbers, atomicity, conservation fuzz,
swap identity, invalidation while swapped, accounting."""
import json
import os
import random

import numpy as np
import pytest

from oracle import kvcache as O
from oracle.kvcache import OracleKV

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _rows(rng, L, n, h_kv, d):
    return rng.integers(0, 1 << 16, size=(L, n, h_kv, d), dtype=np.uint16)


def _c1(aligned=False, cooling=False):
    g = _gold("c1_walk.json")["geometry"]
    return OracleKV(g["L"], g["h_q"], g["h_kv"], g["d"], g["k"], g["num_gpu_blocks"],
                    g["num_cpu_blocks"], lcp_block_aligned=aligned, alloc_cooling=cooling)


@pytest.mark.parametrize("variant,cooling", [("token", False), ("aligned", False), ("token", True)])
def test_c1_walk(variant, cooling):
    """Hand-derived C1 walk; Z9's plain lowest-free-id order by default, and the opt-in
    alloc_cooling variant against its own golden swap-in table."""
    gold = _gold("c1_walk.json")
    kv = _c1(aligned=(variant == "aligned"), cooling=cooling)
    rng = np.random.default_rng(0)
    toks = list(range(100, 124))
    assert kv.new_request(1, []) == O.OK
    for i, exp in enumerate(gold["after_appends"]):
        k, v = _rows(rng, 1, 8, 1, 16), _rows(rng, 1, 8, 1, 16)
        assert kv.append([(1, toks[8 * i: 8 * i + 8], 8, 0)], k, v) == O.OK
        assert kv.info(1)["num_computed"] == exp["nc"]
        assert kv.block_table(1) == exp["table"]
    up = gold["update"]
    new = toks[:10] + [999] + list(range(500, 513))
    assert len(new) == up["new_len"]
    st, p, inval = kv.invalidate_lcp(1, new)
    e = up[variant]
    assert (st, p, inval) == (O.OK, up["lcp"], e["invalidated"])
    assert kv.block_table(1) == e["table"]
    assert kv.info(1)["num_computed"] == e["nc"]
    assert kv.free_counts()[0] == e["gpu_free"]
    assert kv.info(1)["total_tokens_invalidated"] == e["invalidated"]
    if variant == "token":
        ra = gold["reappend_token"]
        k, v = _rows(rng, 1, 14, 1, 16), _rows(rng, 1, 14, 1, 16)
        assert kv.append([(1, None, ra["n_kv"], 0)], k, v) == O.OK
        assert kv.info(1)["num_computed"] == ra["nc"]
        assert kv.block_table(1) == ra["table"]
        so = gold["swap_out"]
        assert kv.swap_out([1]) == (O.OK, so["bytes"])
        assert kv.block_table(1) == so["cpu_table"]
        assert kv.free_counts() == (so["gpu_free"], so["cpu_free"])
        si = gold["swap_in_alloc_cooling" if cooling else "swap_in"]
        assert kv.swap_in([1]) == (O.OK, si["bytes"])
        assert kv.block_table(1) == si["gpu_table"]
        assert kv.free_counts() == (si["gpu_free"], si["cpu_free"])


def test_c1_prime_interleaved():
    gold = _gold("c1_walk.json")["c1_prime"]
    kv = _c1()
    rng = np.random.default_rng(1)
    inputs = {1: list(range(1000, 1100)), 2: list(range(2000, 2100))}
    kv.new_request(1, inputs[1])
    kv.new_request(2, inputs[2])
    for step in gold["steps"]:
        if step[0] == "append":
            _, rid, n, table = step
            k, v = _rows(rng, 1, n, 1, 16), _rows(rng, 1, n, 1, 16)
            assert kv.append([(rid, None, n, 0)], k, v) == O.OK
            assert kv.block_table(rid) == table
        else:
            _, rid, p, e = step
            new = inputs[rid][:p] + [7] + inputs[rid][p + 1:]
            inputs[rid] = new
            assert kv.invalidate_lcp(rid, new) == (O.OK, p, e["invalidated"])
            assert kv.block_table(rid) == e["kept"]
            assert kv.info(rid)["num_computed"] == e["nc"]


@pytest.mark.parametrize("variant", ["token", "aligned"])
def test_spec_invalidate_numbers(variant):
    g = _gold("spec_invalidate.json")
    for case in g["cases"]:
        kv = OracleKV(1, 1, 1, 8, g["k"], 200, 200, lcp_block_aligned=(variant == "aligned"),
                      mirror_pools=False)
        toks = list(range(g["computed"]))
        kv.new_request(0, toks)
        kv.append([(0, None, g["computed"], 0)], np.zeros((1, g["computed"], 1, 8), np.uint16),
                  np.zeros((1, g["computed"], 1, 8), np.uint16))
        free0 = kv.free_counts()[0]
        new = toks[: case["lcp"]] + [-1] * (g["computed"] - case["lcp"])
        st, p, inval = kv.invalidate_lcp(0, new)
        e = case[variant]
        assert (st, p, inval) == (O.OK, case["lcp"], e["invalidated"])
        assert kv.info(0)["num_computed"] == e["nc"]
        assert kv.free_counts()[0] - free0 == e["freed"]
        assert kv.info(0)["num_blocks"] == e["kept"]


def test_append_all_or_nothing():
    kv = OracleKV(1, 1, 1, 8, 16, 9, 4, mirror_pools=False)
    kv.new_request(0, list(range(200)))
    kv.new_request(1, list(range(200)))
    z = np.zeros((1, 200, 1, 8), np.uint16)
    # need 10 > 9 free: nothing changes, including the other item
    st = kv.append([(1, [1, 2], 16, 0), (0, None, 144, 16)], z, z)
    assert st == O.E_NO_GPU_BLOCKS
    assert kv.free_counts() == (9, 4)
    assert kv.info(1)["num_tokens"] == 200 and kv.info(1)["num_computed"] == 0
    assert kv.append([(0, None, 144, 0)], z, z) == O.OK
    assert kv.free_counts() == (0, 4)
    # n_kv beyond pending tokens
    assert kv.append([(1, None, 201, 0)], z, z) == O.E_INVAL
    assert kv.append([(5, None, 1, 0)], z, z) == O.E_NO_REQUEST
    assert kv.append([(1, None, 1, 0), (1, None, 1, 0)], z, z) == O.E_INVAL


def test_swap_atomicity():
    kv = OracleKV(1, 1, 1, 8, 16, 20, 5, mirror_pools=False)
    kv.new_request(0, list(range(96)))
    z = np.zeros((1, 96, 1, 8), np.uint16)
    kv.append([(0, None, 96, 0)], z, z)                      # 6 blocks
    assert kv.swap_out([0]) == (O.E_NO_CPU_BLOCKS, 0)         # S:L179 cpu_free=5, blocks=6
    assert kv.free_counts() == (14, 5)
    assert kv.info(0)["tier"] == O.GPU
    assert kv.swap_in([0]) == (O.E_STATE, 0)


def _check_conservation(kv):
    held = {O.GPU: [], O.CPU: []}
    for r in kv.reqs.values():
        held[r.tier].extend(r.blocks)
        assert len(r.blocks) == -(-r.nc // kv.k)             # held blocks = ceil(nc/k)
    for tier, cap in ((O.GPU, kv.num_gpu_blocks), (O.CPU, kv.num_cpu_blocks)):
        assert len(held[tier]) == len(set(held[tier]))        # one owner per block
        assert not (set(held[tier]) & kv.free[tier])
        assert len(held[tier]) + len(kv.free[tier]) == cap    # S:L199 conservation


def test_conservation_fuzz_10000():
    """S:L614 acceptance #9: 10,000 random alloc/free/swap/invalidate steps."""
    rng = random.Random(3)
    kv = OracleKV(1, 2, 1, 4, 4, 24, 16, mirror_pools=False)
    z = np.zeros((1, 64, 1, 4), np.uint16)
    inputs = {}
    sum_inval = 0
    for step in range(10000):
        op = rng.randrange(6)
        rid = rng.randrange(6)
        if op == 0:
            if kv.new_request(rid, []) == O.OK:
                inputs[rid] = []
        elif op == 1 and rid in kv.reqs:
            n = rng.randrange(0, 12)
            toks = [rng.randrange(4) for _ in range(n)]
            r = kv.reqs[rid]
            n_kv = rng.randrange(0, len(r.input) + n - r.nc + 1)
            st = kv.append([(rid, toks, n_kv, 0)], z, z)
            assert st in (O.OK, O.E_NO_GPU_BLOCKS, O.E_STATE)
        elif op == 2 and rid in kv.reqs:
            r = kv.reqs[rid]
            new = list(r.input[: rng.randrange(0, len(r.input) + 1)]) + [rng.randrange(4) for _ in range(rng.randrange(0, 10))]
            st, p, inval = kv.invalidate_lcp(rid, new)
            sum_inval += inval
        elif op == 3:
            kv.swap_out([rid])
        elif op == 4:
            kv.swap_in([rid])
        elif op == 5 and rng.random() < 0.3:
            if rid in kv.reqs:
                sum_inval -= kv.reqs[rid].tti
            if rng.random() < 0.5:
                kv.release(rid)
            else:
                kv.preempt_recompute(rid)
            if rid in kv.reqs:
                sum_inval += kv.reqs[rid].tti
        _check_conservation(kv)
    # S:L617 acceptance #12: Σ total_tokens_invalidated = Σ per-update returns (live requests)
    assert sum(r.tti for r in kv.reqs.values()) == sum_inval


def test_swap_round_trip_identity_and_mirror():
    """P:L77 swap "preserve[s] computed KV values": pool bytes of every block identical."""
    rng = np.random.default_rng(5)
    kv = OracleKV(2, 4, 2, 8, 4, 16, 16)
    kv.new_request(0, list(range(30)))
    kv.new_request(1, list(range(30)))
    k, v = _rows(rng, 2, 40, 2, 8), _rows(rng, 2, 40, 2, 8)
    assert kv.append([(0, None, 13, 0), (1, None, 27, 13)], k, v) == O.OK
    before = {rid: kv.pool[O.GPU][kv.block_table(rid)].copy() for rid in (0, 1)}
    Kc = kv.reqs[0].Kc.copy()
    assert kv.swap_out([1, 0])[0] == O.OK
    for rid in (0, 1):
        assert np.array_equal(kv.pool[O.CPU][kv.block_table(rid)], before[rid])
    assert kv.swap_in([0, 1])[0] == O.OK
    for rid in (0, 1):
        assert np.array_equal(kv.pool[O.GPU][kv.block_table(rid)], before[rid])
        for pos, (blk, slot) in enumerate(kv.valid_slots(rid)):
            assert np.array_equal(kv.pool[O.GPU][blk, :, 0, :, slot], kv.reqs[rid].Kc[:, pos])
            assert np.array_equal(kv.pool[O.GPU][blk, :, 1, :, slot], kv.reqs[rid].Vc[:, pos])
    assert np.array_equal(kv.reqs[0].Kc, Kc)


@pytest.mark.parametrize("cooling", [False, True])
def test_invalidate_while_swapped_then_resume(cooling):
    """invalidate on CPU, free CPU blocks beyond the LCP, swap in the prefix,
    recompute from the LCP."""
    rng = np.random.default_rng(9)
    kv = OracleKV(1, 2, 1, 8, 4, 16, 16, alloc_cooling=cooling)
    toks = list(range(20))
    kv.new_request(0, toks)
    k, v = _rows(rng, 1, 20, 1, 8), _rows(rng, 1, 20, 1, 8)
    kv.append([(0, None, 20, 0)], k, v)                      # 5 blocks
    kv.swap_out([0])
    assert kv.block_table(0) == [0, 1, 2, 3, 4]
    st, p, inval = kv.invalidate_lcp(0, toks[:9] + [77, 78])
    assert (st, p, inval) == (O.OK, 9, 11)
    assert kv.block_table(0) == [0, 1, 2] and kv.info(0)["tier"] == O.CPU
    assert kv.free_counts() == (16, 13)
    assert kv.swap_in([0])[0] == O.OK
    # Z9: the lowest free ids 0-2; alloc_cooling: ids 0-4 were released by the swap-out, so
    # the free ids 5.. go first
    assert kv.info(0)["num_computed"] == 9
    assert kv.block_table(0) == ([5, 6, 7] if cooling else [0, 1, 2])
    # fully invalidated while swapped -> fresh GPU request with no blocks
    kv.swap_out([0])
    st, p, inval = kv.invalidate_lcp(0, [5])
    assert (p, inval) == (0, 9) and kv.info(0)["tier"] == O.GPU and kv.block_table(0) == []


def test_preempt_recompute_and_release():
    kv = OracleKV(1, 1, 1, 8, 4, 8, 8, mirror_pools=False)
    z = np.zeros((1, 16, 1, 8), np.uint16)
    kv.new_request(0, list(range(16)))
    kv.append([(0, None, 16, 0)], z, z)
    assert kv.preempt_recompute(0) == O.OK
    assert kv.info(0) == dict(num_tokens=16, num_computed=0, total_tokens_invalidated=0, tier=O.GPU, num_blocks=0)
    assert kv.free_counts() == (8, 8)
    assert kv.release(0) == O.OK and kv.release(0) == O.E_NO_REQUEST
    assert kv.new_request(0) == O.OK and kv.new_request(0) == O.E_STATE


# ---- FP8 KV cache (the paper's b = 2, becomes 1) ----------------------
def test_fp8_codec_pins():
    """E4M3 (OCP FP8, 'FN'): values from the format's definition, RNE ties, saturation,
    signed zero; the whole codec agrees with torch's float8_e4m3fn cast on in-range values."""
    import torch
    from oracle import fp8
    t = fp8.decode_table()
    assert t[0x38] == 1.0 and t[0x7E] == 448.0 and t[0xC0] == -2.0 and t[0x01] == 2.0 ** -9
    assert t[0x08] == 2.0 ** -6 and t[0x07] == 7 * 2.0 ** -9 and np.isnan(t[0x7F]) and np.isnan(t[0xFF])
    assert len(set(t[~np.isnan(t)].tolist())) == 253            # 254 finite codes, +0 == -0
    x = np.array([1.0, 1.0625, 1.1875, 500.0, -1e9, 2.0 ** -10, 3 * 2.0 ** -11, -0.0, 448.0])
    assert [int(c) for c in fp8.encode(x)] == [0x38, 0x38, 0x3A, 0x7E, 0xFE, 0x00, 0x01, 0x80, 0x7E]
    c = np.arange(256, dtype=np.uint8)
    fin = ~np.isnan(t)
    assert np.array_equal(fp8.encode(t[fin]), c[fin])           # every finite code round-trips
    rng = np.random.default_rng(0)
    r = np.clip(rng.standard_normal(100000) * np.exp(rng.uniform(-8, 6, 100000)), -448, 448)
    ref = torch.from_numpy(r.astype(np.float32)).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(fp8.encode(r), ref)
    # every E4M3 value is a bf16 value: the dequantized rows are exact bf16 bits
    assert np.array_equal(fp8.bf16_bits_to_f64(fp8.f64_to_bf16_bits(t[fin])), t[fin])


def test_fp8_kv_oracle_stores_codes_and_attends_on_their_values():
    from oracle import fp8
    rng = np.random.default_rng(3)
    kv = OracleKV(1, 2, 1, 8, 4, 8, 8, kv_dtype="fp8")
    assert kv.m_block == 2 * 1 * 4 * 1 * 8 * 1                   # b = 1 byte per value
    k, v = _rows(rng, 1, 10, 1, 8), _rows(rng, 1, 10, 1, 8)
    k = fp8.f64_to_bf16_bits(rng.standard_normal((1, 10, 1, 8)) * 3)   # finite, in range
    v = fp8.f64_to_bf16_bits(rng.standard_normal((1, 10, 1, 8)))
    kv.new_request(0, list(range(10)))
    assert kv.append([(0, None, 10, 0)], k, v) == O.OK
    kc, kd = fp8.quantize_bf16_bits(k)
    blk = kv.block_table(0)
    for pos in range(10):
        assert np.array_equal(kv.pool[O.GPU][blk[pos // 4], :, 0, :, pos % 4, :], kc[:, pos])
    assert np.array_equal(kv.reqs[0].Kc[:, :10], kd)
    q = fp8.f64_to_bf16_bits(rng.standard_normal((10, 2, 8)))
    st, o, _ = kv.prefill([(0, 0, 10, 0)], q)
    from oracle.attention import attention
    vq = fp8.quantize_bf16_bits(v)[1]
    o_ref, _ = attention(q, kd[0], vq[0], 0)
    assert st == O.OK and np.array_equal(o, o_ref)
    st, b = kv.swap_out([0])
    assert st == O.OK and b == 3 * kv.m_block
