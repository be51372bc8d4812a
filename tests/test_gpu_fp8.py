"""GPU parity of the optional FP8 KV cache (s2l_config.kv_dtype = 1; SURVEY §8.5 f4 -- not the
paper's b = 2 bytes).  The library stores each bf16 K/V value as the nearest E4M3 code
(RNE, saturating, reading Z20) and its attention dequantizes exactly; the oracle
(oracle/kvcache.py kv_dtype="fp8", oracle/fp8.py) stores the codes of the same rows and
attends in fp64 on their exact values.  So: pool bytes (the codes) bit-exact, attention within
2e-2 normwise / 1e-2 LSE -- the same bars as bf16, against the quantised K/V."""
import numpy as np
import pytest
import torch

from synth import workloads as W
from tests.harness import Pair
from paper_2604_16395_b200 import s2l

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _dev():
    from paper_2604_16395_b200 import build
    build.build()
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.init()


def _qkv(seed, toks, geo, q_scale=1.0):
    return W.request_qkv(seed, np.asarray(toks, np.int32), geo, q_scale)


def test_fp8_block_bytes_halve():
    a = s2l.block_bytes(s2l.make_config(32, 32, 8, 128, 16, 1, 0))
    b = s2l.block_bytes(s2l.make_config(32, 32, 8, 128, 16, 1, 0, kv_dtype=1))
    assert a == 2 * b == 2 * 1024 * 1024


def test_fp8_c1_walk_generic_kernel():
    """C1 geometry (CUDA-core kernel): three appends, update with LCP 10, re-append, swap round
    trip -- codes bit-exact in both pools, attention vs the oracle on every row."""
    geo = W.C1
    seed = W.seed_of(41)
    P = Pair(geo.L, geo.h_q, geo.h_kv, geo.d, geo.k, 8, 8, kv_dtype=1)
    toks = W.request_tokens(seed, 0, 24)
    q, k, v = _qkv(seed, toks, geo)
    P.new(1, [])
    for i in range(3):
        sl = slice(8 * i, 8 * i + 8)
        P.append([(1, toks[sl], 8, 0)], k[:, sl], v[:, sl])
        P.prefill([(1, 8 * i, 8, 0)], q[sl])
        P.check_state()
        P.check_pool_valid_slots()
    new = W.updated_tokens(seed, 0, toks, 10, 24, 0)
    P.invalidate(1, new)
    q2, k2, v2 = _qkv(seed, new, geo)
    b = P.lib.query(1)["num_computed"]
    P.append([(1, None, 24 - b, 0)], k2[:, b:], v2[:, b:])
    P.prefill([(1, b, 24 - b, 0)], q2[b:])
    P.check_pools_whole()
    assert P.swap_out([1]) == (s2l.OK, 6 * 128)
    P.check_pools_whole()
    assert P.swap_in([1])[0] == s2l.OK
    P.check_pools_whole()
    P.prefill([(1, b, 24 - b, 0)], q2[b:])


@pytest.mark.parametrize("h_q,h_kv,k", [(32, 8, 16), (8, 2, 64), (16, 16, 128)])
def test_fp8_tensor_core_ragged(h_q, h_kv, k):
    """tcgen05 kernel with the FP8 staging + bf16 conversion path: ragged chunks over several
    KV tiles, peaky scores (the exact / rescale path), every row vs the oracle."""
    geo = W.Geometry(L=2, h_q=h_q, h_kv=h_kv, d=128, k=k)
    P = Pair(2, h_q, h_kv, 128, k, 160, 16, max_blocks=80, kv_dtype=1)
    seed = W.seed_of(42)
    lens = [700, 333, 129]
    data = {}
    for r, n in enumerate(lens):
        toks = W.request_tokens(seed, r, n)
        data[r] = _qkv(seed, toks, geo, q_scale=3.0 if r == 1 else 1.0)
        P.new(r, toks)
    # two chunks per request, the second ragged
    for c in range(2):
        items, ks, vs, qs, row = [], [], [], [], 0
        for r, n in enumerate(lens):
            a, e = (0, n // 2) if c == 0 else (n // 2, n)
            items.append((r, None, e - a, row))
            ks.append(data[r][1][:, a:e]); vs.append(data[r][2][:, a:e]); qs.append(data[r][0][a:e])
            row += e - a
        P.append(items, np.concatenate(ks, axis=1), np.concatenate(vs, axis=1))
        pre = [(r, (0 if c == 0 else lens[r] // 2), it[2], it[3]) for r, it in zip(range(3), items)]
        for layer in range(2):
            P.prefill(pre, np.concatenate(qs), layer=layer)
    P.check_state()
    P.check_pool_valid_slots()
    P.check_pools_whole()


def test_fp8_prefill_append_falls_back_and_swaps():
    """s2l_prefill_append on an FP8 pool appends with a separate launch (no in-kernel append);
    the result equals the oracle; swap-out / swap-in move half the bytes of a bf16 pool."""
    geo = W.Geometry(L=1, h_q=8, h_kv=2, d=128, k=16)
    P = Pair(1, 8, 2, 128, 16, 64, 64, max_blocks=64, kv_dtype=1)
    seed = W.seed_of(43)
    toks = W.request_tokens(seed, 0, 512)
    q, k, v = _qkv(seed, toks, geo)
    P.new(0, toks)
    P.append_reserve([(0, None, 512, 0)], k, v)
    P.prefill_append([(0, 0, 512, 0)], q, k[0], v[0])
    P.check_pools_whole()
    assert P.swap_out([0]) == (s2l.OK, 32 * P.m_block)
    assert P.m_block == 2 * 1 * 16 * 2 * 128
    assert P.swap_in([0])[0] == s2l.OK
    P.check_pools_whole()
    P.prefill([(0, 256, 256, 0)], q[256:])
