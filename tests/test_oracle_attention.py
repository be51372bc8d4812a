"""Pins of oracle.attention: closed forms, pure-Python brute force, torch fp64 SDPA with an
explicit bottom-right mask, scipy logsumexp for LSE, and the paper's invariants
(chunked prefill == one-shot prefill; update after LCP invalidation == fresh prefill)."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import kvcache as O
from oracle.attention import attention, attention_rows, bf16_to_f64
from oracle.kvcache import OracleKV


def _bits(x):
    return synth.f64_to_bf16_bits(np.asarray(x, dtype=np.float64))


def _rand(rng, *shape, scale=1.0):
    return _bits(rng.standard_normal(shape) * scale)


def test_bf16_decode_exact():
    vals = np.array([0.0, 1.0, -2.5, 0.15625, 3.0e38, -1.0e-30, 65504.0])
    bits = _bits(vals)
    dec = bf16_to_f64(bits)
    # decoding is exact: re-encoding gives the same bits, and powers of two are exact
    assert np.array_equal(_bits(dec), bits)
    assert dec[1] == 1.0 and dec[2] == -2.5 and dec[3] == 0.15625


def test_q_zero_gives_prefix_mean():
    """q = 0 => all scores equal => O_t = mean(V[0..q_pos+t])."""
    rng = np.random.default_rng(0)
    n, q_pos, h_q, h_kv, d = 5, 3, 4, 2, 16
    q = np.zeros((n, h_q, d), np.uint16)
    k, v = _rand(rng, 8, h_kv, d), _rand(rng, 8, h_kv, d)
    o, lse = attention(q, k, v, q_pos)
    vf = bf16_to_f64(v)
    for t in range(n):
        for h in range(h_q):
            g = h // 2
            np.testing.assert_allclose(o[t, h], vf[: q_pos + t + 1, g].mean(axis=0), rtol=0, atol=1e-14)
            assert abs(lse[t, h] - math.log(q_pos + t + 1)) < 1e-14


def test_single_key_gives_v0():
    rng = np.random.default_rng(1)
    q, k, v = _rand(rng, 1, 2, 8), _rand(rng, 1, 1, 8), _rand(rng, 1, 1, 8)
    o, _ = attention(q, k, v, 0)
    assert np.array_equal(o[0, 0], bf16_to_f64(v[0, 0]))
    assert np.array_equal(o[0, 1], bf16_to_f64(v[0, 0]))


def test_dominant_key_selects_its_value():
    """K_j* = c·q with large c, other keys orthogonal => O -> V_j*."""
    d = 16
    q = np.zeros((1, 1, d)); q[0, 0, 0] = 1.0
    k = np.zeros((6, 1, d)); k[:, 0, 1] = 1.0
    k[3, 0, 0] = 256.0                                   # s_3 = 256/4 = 64, others 0
    rng = np.random.default_rng(2)
    v = _rand(rng, 6, 1, d)
    o, _ = attention(_bits(q), _bits(k), v, 5)
    np.testing.assert_allclose(o[0, 0], bf16_to_f64(v[3, 0]), rtol=0, atol=1e-25)


def test_mask_is_bottom_right():
    """Row t at q_pos+t must not see key q_pos+t+1: changing later keys leaves it unchanged."""
    rng = np.random.default_rng(3)
    q, k, v = _rand(rng, 4, 2, 8), _rand(rng, 10, 1, 8), _rand(rng, 10, 1, 8)
    o1, _ = attention(q, k, v, 6)
    k2, v2 = k.copy(), v.copy()
    k2[8:] = _rand(rng, 2, 1, 8); v2[8:] = _rand(rng, 2, 1, 8)
    o2, _ = attention(q, k2, v2, 6)
    assert np.array_equal(o1[:2], o2[:2])              # rows at positions 6, 7
    assert not np.array_equal(o1[2:], o2[2:])


def _brute(q, k, v, q_pos):
    """Pure-Python scalar loops with math.exp (independent of numpy)."""
    n, h_q, d = q.shape
    h_kv = k.shape[1]
    qf, kf, vf = bf16_to_f64(q).tolist(), bf16_to_f64(k).tolist(), bf16_to_f64(v).tolist()
    out = [[[0.0] * d for _ in range(h_q)] for _ in range(n)]
    for t in range(n):
        for h in range(h_q):
            g = h // (h_q // h_kv)
            s = []
            for j in range(q_pos + t + 1):
                acc = 0.0
                for c in range(d):
                    acc += qf[t][h][c] * kf[j][g][c]
                s.append(acc / math.sqrt(d))
            m = max(s)
            w = [math.exp(x - m) for x in s]
            z = sum(w)
            for c in range(d):
                out[t][h][c] = sum(w[j] * vf[j][g][c] for j in range(len(w))) / z
    return np.array(out)


@pytest.mark.parametrize("shape", [(8, 0, 2, 1, 16), (3, 5, 4, 2, 8), (6, 9, 4, 1, 4), (2, 0, 1, 1, 16)])
def test_bruteforce_tiny(shape):
    n, q_pos, h_q, h_kv, d = shape
    rng = np.random.default_rng(sum(shape))
    q = _rand(rng, n, h_q, d, scale=2.0)
    k, v = _rand(rng, q_pos + n, h_kv, d), _rand(rng, q_pos + n, h_kv, d)
    o, _ = attention(q, k, v, q_pos)
    np.testing.assert_allclose(o, _brute(q, k, v, q_pos), rtol=0, atol=1e-12)
    o2, _ = attention_rows(q, k, v, q_pos, range(n))
    np.testing.assert_allclose(o2, o, rtol=0, atol=1e-12)


def _sdpa_ref(q, k, v, q_pos):
    qf = torch.from_numpy(bf16_to_f64(q)).permute(1, 0, 2)          # [h_q][n][d]
    kf = torch.from_numpy(bf16_to_f64(k[: q_pos + q.shape[0]])).permute(1, 0, 2)
    vf = torch.from_numpy(bf16_to_f64(v[: q_pos + q.shape[0]])).permute(1, 0, 2)
    g = q.shape[1] // k.shape[1]
    kf, vf = kf.repeat_interleave(g, dim=0), vf.repeat_interleave(g, dim=0)
    n, T = q.shape[0], kf.shape[1]
    mask = torch.arange(T)[None, :] <= (q_pos + torch.arange(n))[:, None]   # explicit bottom-right
    o = torch.nn.functional.scaled_dot_product_attention(qf, kf, vf, attn_mask=mask)
    return o.permute(1, 0, 2).numpy()


@pytest.mark.parametrize("shape", [(8, 16, 2, 1, 16), (40, 100, 8, 2, 64), (17, 0, 4, 4, 32)])
def test_torch_sdpa_fp64(shape):
    n, q_pos, h_q, h_kv, d = shape
    rng = np.random.default_rng(n + q_pos)
    q = _rand(rng, n, h_q, d, scale=4.0)                 # "peaky" scores
    k, v = _rand(rng, q_pos + n, h_kv, d), _rand(rng, q_pos + n, h_kv, d)
    o, _ = attention(q, k, v, q_pos)
    np.testing.assert_allclose(o, _sdpa_ref(q, k, v, q_pos), rtol=0, atol=1e-12)


def test_lse_matches_scipy_logsumexp():
    from scipy.special import logsumexp
    rng = np.random.default_rng(11)
    q, k, v = _rand(rng, 5, 2, 16, scale=3.0), _rand(rng, 12, 1, 16), _rand(rng, 12, 1, 16)
    _, lse = attention(q, k, v, 7)
    qf, kf = bf16_to_f64(q), bf16_to_f64(k)
    for t in range(5):
        for h in range(2):
            s = kf[: 7 + t + 1, 0] @ qf[t, h] / 4.0
            assert abs(lse[t, h] - logsumexp(s)) < 1e-12


def test_gqa_group_sharing_and_mha():
    rng = np.random.default_rng(4)
    q = _rand(rng, 4, 4, 8)
    q[:, 1] = q[:, 0]                                    # heads 0,1 share kv head 0
    k, v = _rand(rng, 9, 2, 8), _rand(rng, 9, 2, 8)
    o, _ = attention(q, k, v, 5)
    assert np.array_equal(o[:, 0], o[:, 1])
    # h_q == h_kv: plain MHA == per-head single-head attention
    qm = _rand(rng, 3, 2, 8)
    om, _ = attention(qm, k, v, 6)
    for h in range(2):
        oh, _ = attention(qm[:, h:h + 1], k[:, h:h + 1], v[:, h:h + 1], 6)
        assert np.array_equal(om[:, h], oh[:, 0])


def _stream_inputs(seed, toks, L, h_q, h_kv, d):
    H = synth.prefix_hashes(seed, np.array(toks))
    return synth.qkv(seed, H, L, h_q, h_kv, d)


def test_invariant_chunked_equals_one_shot():
    """Chunked prefill of c1..cn equals one-shot prefill of the concatenation."""
    L, h_q, h_kv, d, k = 2, 4, 2, 16, 4
    toks = synth.tokens(1, 0, 29).tolist()
    q, kk, vv = _stream_inputs(1, toks, L, h_q, h_kv, d)
    kv = OracleKV(L, h_q, h_kv, d, k, 16, 0)
    kv.new_request(0, [])
    chunks = [7, 1, 13, 8]
    outs = []
    pos = 0
    for c in chunks:
        assert kv.append([(0, toks[pos:pos + c], c, 0)], kk[:, pos:pos + c], vv[:, pos:pos + c]) == O.OK
        st, o, _ = kv.prefill([(0, pos, c, 0)], q[pos:pos + c], layer=1)
        assert st == O.OK
        outs.append(o)
        pos += c
    one = OracleKV(L, h_q, h_kv, d, k, 16, 0)
    one.new_request(0, toks)
    one.append([(0, None, 29, 0)], kk, vv)
    _, o_all, _ = one.prefill([(0, 0, 29, 0)], q, layer=1)
    np.testing.assert_allclose(np.concatenate(outs), o_all, rtol=0, atol=1e-13)


def test_invariant_update_equals_fresh():
    """After LCP invalidation + recompute of the suffix, outputs equal a fresh prefill of the
    new input (recompute "only for tokens that changed")."""
    L, h_q, h_kv, d, k = 1, 2, 1, 16, 4
    old = synth.tokens(2, 0, 24).tolist()
    new = old[:10] + synth.tokens(2, 1, 14).tolist()
    new[10] = (old[10] + 1) % synth.VOCAB
    q_o, k_o, v_o = _stream_inputs(2, old, L, h_q, h_kv, d)
    q_n, k_n, v_n = _stream_inputs(2, new, L, h_q, h_kv, d)
    assert np.array_equal(k_o[:, :10], k_n[:, :10])      # Z10: prefix rows identical
    assert not np.array_equal(k_o[:, 10], k_n[:, 10])
    kv = OracleKV(L, h_q, h_kv, d, k, 8, 8)
    kv.new_request(0, old)
    kv.append([(0, None, 24, 0)], k_o, v_o)
    st, p, inval = kv.invalidate_lcp(0, new)
    assert (p, inval) == (10, 14)
    kv.append([(0, None, 14, 0)], k_n[:, 10:], v_n[:, 10:])
    _, o_upd, _ = kv.prefill([(0, 10, 14, 0)], q_n[10:])
    fresh = OracleKV(L, h_q, h_kv, d, k, 8, 8)
    fresh.new_request(0, new)
    fresh.append([(0, None, 24, 0)], k_n, v_n)
    _, o_fresh, _ = fresh.prefill([(0, 0, 24, 0)], q_n)
    np.testing.assert_allclose(o_upd, o_fresh[10:], rtol=0, atol=1e-13)


def test_prefill_validation():
    kv = OracleKV(1, 2, 1, 8, 4, 8, 8, mirror_pools=False)
    kv.new_request(0, list(range(8)))
    z = np.zeros((1, 8, 1, 8), np.uint16)
    kv.append([(0, None, 6, 0)], z, z)
    q = np.zeros((8, 2, 8), np.uint16)
    assert kv.prefill([(0, 0, 7, 0)], q)[0] == O.E_INVAL       # q_pos + n_q > nc
    assert kv.prefill([(0, 0, 0, 0)], q)[0] == O.E_INVAL
    assert kv.prefill([(3, 0, 1, 0)], q)[0] == O.E_NO_REQUEST
    kv.swap_out([0])
    assert kv.prefill([(0, 0, 1, 0)], q)[0] == O.E_STATE
