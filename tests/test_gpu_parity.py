"""GPU parity tests (B200): libs2l through its C ABI vs the fp64 oracle on the same seeded
inputs.  Bit-exact for block tables, counts, LCP and pool / swap bytes; normwise relative
error <= 2e-2 for attention (BJ:L5), |dLSE| <= 1e-2."""
import numpy as np
import pytest
import torch

import synth
from synth import workloads as W
from tests.harness import Pair, bf16_dev_to_f64, normwise_err, to_dev
from paper_2604_16395_b200 import s2l

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _dev():
    from paper_2604_16395_b200 import build
    build.build()
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.init()


def _stream_qkv(seed, toks, geo, q_scale=1.0):
    return W.request_qkv(seed, np.asarray(toks, np.int32), geo, q_scale)


# ----------------------------------------------------------------------------- C1 (BJ:L7)
@pytest.mark.parametrize("aligned", [False, True])
def test_c1_full_walk(aligned):
    geo = W.C1
    seed = W.seed_of(1)
    P = Pair(geo.L, geo.h_q, geo.h_kv, geo.d, geo.k, 8, 8, aligned=aligned)
    toks = W.request_tokens(seed, 0, 24)
    q, k, v = _stream_qkv(seed, toks, geo)
    P.new(1, [])
    for i in range(3):
        sl = slice(8 * i, 8 * i + 8)
        P.append([(1, toks[sl], 8, 0)], k[:, sl], v[:, sl])
        P.prefill([(1, 8 * i, 8, 0)], q[sl])
        P.check_state()
        P.check_pool_valid_slots()
    assert P.lib.block_table(1) == [0, 1, 2, 3, 4, 5]
    new = W.updated_tokens(seed, 0, toks, 10, 24, 0)
    p, inval = P.invalidate(1, new)
    assert p == 10 and inval == (16 if aligned else 14)
    q2, k2, v2 = _stream_qkv(seed, new, geo)
    b = P.lib.query(1)["num_computed"]
    P.append([(1, None, 24 - b, 0)], k2[:, b:], v2[:, b:])
    P.prefill([(1, b, 24 - b, 0)], q2[b:])
    P.check_state()
    P.check_pool_valid_slots()
    P.check_pools_whole()
    before = P.gpu_pool_bits()[P.lib.block_table(1)].copy()
    assert P.swap_out([1]) == (s2l.OK, 6 * 256)
    assert np.array_equal(P.cpu_pool_bits()[P.lib.block_table(1)], before)
    P.check_pools_whole()
    assert P.swap_in([1]) == (s2l.OK, 6 * 256)
    P.check_state()
    P.check_pools_whole()
    # after the round trip attention is unchanged
    P.prefill([(1, b, 24 - b, 0)], q2[b:])


def test_c1_prime_interleaved_two_requests():
    geo = W.C1
    seed = W.seed_of(1)
    P = Pair(geo.L, geo.h_q, geo.h_kv, geo.d, geo.k, 8, 8)
    toks = {r: W.request_tokens(seed, r, 24) for r in (1, 2)}
    qkv = {r: _stream_qkv(seed, toks[r], geo) for r in (1, 2)}
    P.new(1, toks[1]); P.new(2, toks[2])
    sched = [(1, 0, 8), (2, 0, 8), (1, 8, 8)]
    for rid, a, n in sched:
        P.append([(rid, None, n, 0)], qkv[rid][1][:, a:a + n], qkv[rid][2][:, a:a + n])
        P.prefill([(rid, a, n, 0)], qkv[rid][0][a:a + n])
    new2 = W.updated_tokens(seed, 2, toks[2], 3, 12, 0)
    assert P.invalidate(2, new2) == (3, 5)
    q2, k2, v2 = _stream_qkv(seed, new2, geo)
    # one append call carrying both requests (freed id 3 reused by request 1)
    kk = np.concatenate([qkv[1][1][:, 16:20], k2[:, 3:12]], axis=1)
    vv = np.concatenate([qkv[1][2][:, 16:20], v2[:, 3:12]], axis=1)
    P.append([(1, None, 4, 0), (2, None, 9, 4)], kk, vv)
    assert P.lib.block_table(1) == [0, 1, 4, 5, 3] and P.lib.block_table(2) == [2, 6, 7]
    qq = np.concatenate([qkv[1][0][16:20], q2[3:12]])
    P.prefill([(1, 16, 4, 0), (2, 3, 9, 4)], qq)
    P.check_pools_whole()


# ----------------------------------------------------------------------------- tensor-core path
def _multi_request_case(P, seed, geo, lengths, chunks, q_scale=1.0):
    """Prefills each request's [0, lengths[i]) in `chunks[i]` pieces, all requests batched
    per round; checks every round against the oracle."""
    toks = {r: W.request_tokens(seed, r, L) for r, L in enumerate(lengths)}
    data = {r: _stream_qkv(seed, toks[r], geo, q_scale) for r in toks}
    for r in toks:
        P.new(r, toks[r])
    pos = {r: 0 for r in toks}
    rounds = max(len(c) for c in chunks)
    for j in range(rounds):
        items_a, items_p, ks, vs, qs = [], [], [], [], []
        row = 0
        for r in toks:
            if j >= len(chunks[r]):
                continue
            n = chunks[r][j]
            a = pos[r]
            items_a.append((r, None, n, row))
            items_p.append((r, a, n, row))
            ks.append(data[r][1][:, a:a + n]); vs.append(data[r][2][:, a:a + n]); qs.append(data[r][0][a:a + n])
            row += n
            pos[r] += n
        P.append(items_a, np.concatenate(ks, axis=1), np.concatenate(vs, axis=1))
        P.prefill(items_p, np.concatenate(qs))
    P.check_state()
    P.check_pool_valid_slots()
    return toks, data


@pytest.mark.parametrize("h_q,h_kv", [(8, 2), (4, 4), (16, 2), (4, 2)])
def test_tc_gqa_ragged(h_q, h_kv):
    """d = 128, k = 16: several tiles, ragged tails, varied GQA group sizes."""
    geo = W.Geometry(L=1, h_q=h_q, h_kv=h_kv, d=128, k=16)
    P = Pair(1, h_q, h_kv, 128, 16, 256, 0)
    _multi_request_case(P, 77, geo, [517, 300, 129], [[200, 317], [1, 299], [128, 1]])


@pytest.mark.parametrize("h_kv,kv_dtype", [(32, 0), (128, 0), (32, 1)])
def test_append_wide_token_rows(h_kv, kv_dtype):
    """Token rows wider than 128 16-byte vectors (h_kv * d > 1024: MHA shapes, h_q = h_kv at
    d = 128) take the append kernel's one-row-per-warp, 16-vectors-per-chunk path
    (append_kernel<16, 16> for h_kv = 32, <64, 0> for h_kv = 128), bf16 and FP8 pools: ragged
    chunks of two requests, pool bytes whole and every attention row vs the oracle."""
    geo = W.Geometry(L=1, h_q=h_kv, h_kv=h_kv, d=128, k=16)
    P = Pair(1, h_kv, h_kv, 128, 16, 24, 0, max_blocks=12, kv_dtype=kv_dtype)
    _multi_request_case(P, 313, geo, [161, 45], [[100, 61], [1, 44]])
    P.check_pools_whole()


def test_c2t_crawler_shaped_ragged_chunks():
    """C2t, reduced: Llama-3-8B attention shape, 6 requests whose totals are
    LogNormal(ln 5800, 0.976) draws scaled down to [97, 1500] tokens, each split into U{6..10}
    near-equal chunks, one chunk per request per round -- every round is a ragged
    batch (lengths and positions off the block size); every row of every round vs the oracle."""
    geo = W.LLAMA3_8B
    rng = np.random.default_rng(1002)
    tot = np.clip(np.round(rng.lognormal(np.log(5800.0), 0.976, 6) / 10), 97, 1500).astype(int)
    nch = rng.integers(6, 11, 6)
    chunks = [[int(t) // c + (1 if i < int(t) % c else 0) for i in range(c)] for t, c in zip(tot, nch)]
    P = Pair(1, 32, 8, 128, 16, 700, 0)
    _multi_request_case(P, W.seed_of(2), geo, [int(t) for t in tot], chunks)


@pytest.mark.parametrize("k", [32, 64, 128])
def test_tc_block_sizes(k):
    geo = W.Geometry(L=2, h_q=8, h_kv=2, d=128, k=k)
    P = Pair(2, 8, 2, 128, k, 64, 0)
    _multi_request_case(P, 78, geo, [700, 333], [[256, 444], [333]])


def test_tc_peaky_scores_rescale():
    """Q scaled by 4 (score std ~4): exercises the running-max rescale of O in TMEM."""
    geo = W.Geometry(L=1, h_q=8, h_kv=2, d=128, k=16)
    P = Pair(1, 8, 2, 128, 16, 256, 0)
    _multi_request_case(P, 79, geo, [1200, 640], [[64, 900, 236], [640]], q_scale=4.0)


def test_tc_layer_selection():
    geo = W.Geometry(L=3, h_q=8, h_kv=2, d=128, k=16)
    P = Pair(3, 8, 2, 128, 16, 64, 0)
    toks, data = _multi_request_case(P, 80, geo, [300], [[300]])
    q = data[0][0]
    for layer in range(3):
        P.prefill([(0, 0, 300, 0)], q, layer=layer)


def test_reduced_c2_two_requests_4k():
    """Reduced C2 (SURVEY d.5): Llama-3-8B attention shape, 2 requests x 4096 tokens in
    512-token chunks, all checked in full."""
    geo = W.LLAMA3_8B
    P = Pair(1, 32, 8, 128, 16, 1024, 0, mirror=False)
    _multi_request_case(P, W.seed_of(2), geo, [4096, 4096], [[512] * 8, [512] * 8])


def test_c3_small_update_equals_fresh():
    """Update mode (C3 shape, 4 requests x 2048): LCP invalidation of 20-80%, re-append and
    re-prefill of the suffix == fresh prefill of the new input."""
    geo = W.LLAMA3_8B
    seed = W.seed_of(3)
    P = Pair(1, 32, 8, 128, 16, 1024, 0, mirror=False)
    toks, data = _multi_request_case(P, seed, geo, [2048] * 4, [[1024, 1024]] * 4)
    ps = W.c3_lcp_draws(seed, 4, 2048)
    items_a, items_p, ks, vs, qs, row = [], [], [], [], [], 0
    fresh = {}
    for r in range(4):
        new = W.updated_tokens(seed, r, toks[r], int(ps[r]), 2048, 0)
        assert P.invalidate(r, new) == (int(ps[r]), 2048 - int(ps[r]))
        qn, kn, vn = _stream_qkv(seed, new, geo)
        fresh[r] = (new, qn, kn, vn)
        b = int(ps[r])
        items_a.append((r, None, 2048 - b, row)); items_p.append((r, b, 2048 - b, row))
        ks.append(kn[:, b:]); vs.append(vn[:, b:]); qs.append(qn[b:])
        row += 2048 - b
    P.append(items_a, np.concatenate(ks, axis=1), np.concatenate(vs, axis=1))
    o_gpu, o_ref, _, _ = P.prefill(items_p, np.concatenate(qs))
    # the same suffix rows from a fresh context holding only the new inputs
    F = Pair(1, 32, 8, 128, 16, 1024, 0, mirror=False)
    row = 0
    for r in range(4):
        new, qn, kn, vn = fresh[r]
        F.new(r, new)
        F.append([(r, None, 2048, 0)], kn, vn)
        b = int(ps[r])
        o_f, _, _, _ = F.prefill([(r, 0, 2048, 0)], qn)
        err = normwise_err(o_gpu[row:row + 2048 - b], o_f[b:])
        assert err.max() <= 2e-2
        row += 2048 - b


def test_c3_small_budget_split_update_round():
    """The C3 update round in scheduling steps of <= 1536 tokens (the token budget of P:L308,
    scaled with the 4 x 2048 case; the bench's c3.budget_8192 field at full size): suffixes packed
    in request order, a suffix that does not fit continues as the next chunk of that request
    (partial suffix items at q_pos = p + done).  Bookkeeping, pool bytes and every row of every
    step's attention vs the oracle (harness), and the outputs equal a fresh prefill's rows."""
    geo = W.LLAMA3_8B
    seed = W.seed_of(3) + 7
    P = Pair(1, 32, 8, 128, 16, 1024, 0)
    toks, data = _multi_request_case(P, seed, geo, [2048] * 4, [[1024, 1024]] * 4)
    ps = W.c3_lcp_draws(seed, 4, 2048)
    budget, steps, cur, fill = 1536, [], [], 0
    fresh = {}
    for r in range(4):
        new = W.updated_tokens(seed, r, toks[r], int(ps[r]), 2048, 0)
        assert P.invalidate(r, new) == (int(ps[r]), 2048 - int(ps[r]))
        fresh[r] = (new,) + tuple(_stream_qkv(seed, new, geo))
        done, n = 0, 2048 - int(ps[r])
        while done < n:
            take = min(n - done, budget - fill)
            cur.append((r, int(ps[r]) + done, take))
            done += take
            fill += take
            if fill == budget:
                steps.append(cur)
                cur, fill = [], 0
    if cur:
        steps.append(cur)
    assert len(steps) >= 2 and any(len({it[0] for it in s}) > 1 for s in steps)
    outs = {r: [] for r in range(4)}
    for s in steps:
        items_a, items_p, ks, vs, qs, row = [], [], [], [], [], 0
        for r, a, n in s:
            _, qn, kn, vn = fresh[r]
            items_a.append((r, None, n, row)); items_p.append((r, a, n, row))
            ks.append(kn[:, a:a + n]); vs.append(vn[:, a:a + n]); qs.append(qn[a:a + n])
            row += n
        P.append(items_a, np.concatenate(ks, axis=1), np.concatenate(vs, axis=1))
        o_gpu, _, _, _ = P.prefill(items_p, np.concatenate(qs))      # every row vs the oracle
        row = 0
        for r, a, n in s:
            outs[r].append(o_gpu[row:row + n])
            row += n
    P.check_state()
    P.check_pools_whole()
    F = Pair(1, 32, 8, 128, 16, 1024, 0, mirror=False)
    for r in range(4):
        new, qn, kn, vn = fresh[r]
        F.new(r, new)
        F.append([(r, None, 2048, 0)], kn, vn)
        o_f, _, _, _ = F.prefill([(r, 0, 2048, 0)], qn)
        b = int(ps[r])
        assert normwise_err(np.concatenate(outs[r]), o_f[b:]).max() <= 2e-2


def test_chunked_equals_one_shot_and_batch_independence():
    geo = W.LLAMA3_8B
    seed = 91
    toks = W.request_tokens(seed, 0, 1500)
    q, k, v = _stream_qkv(seed, toks, geo)
    A = Pair(1, 32, 8, 128, 16, 256, 0, mirror=False)
    A.new(0, toks)
    outs = []
    for a, n in ((0, 100), (100, 700), (800, 700)):
        A.append([(0, None, n, 0)], k[:, a:a + n], v[:, a:a + n])
        outs.append(A.prefill([(0, a, n, 0)], q[a:a + n])[0])
    B = Pair(1, 32, 8, 128, 16, 256, 0, mirror=False)
    B.new(0, toks)
    B.new(1, W.request_tokens(seed, 1, 900))
    q1, k1, v1 = _stream_qkv(seed, W.request_tokens(seed, 1, 900), geo)
    B.append([(1, None, 900, 0), (0, None, 1500, 900)], np.concatenate([k1, k], 1), np.concatenate([v1, v], 1))
    o_b, _, _, _ = B.prefill([(1, 0, 900, 0), (0, 0, 1500, 900)], np.concatenate([q1, q]))
    one = o_b[900:]
    chunked = np.concatenate(outs)
    assert normwise_err(chunked, one).max() <= 2e-2
    # batch-composition independence: request 0's chunk [800, 1500) alone vs inside a batch
    C = Pair(1, 32, 8, 128, 16, 256, 0, mirror=False)
    C.new(0, toks)
    C.append([(0, None, 1500, 0)], k, v)
    o_c, _, _, _ = C.prefill([(0, 800, 700, 0)], q[800:])
    assert np.array_equal(o_c, outs[2]) or normwise_err(o_c, outs[2]).max() <= 2e-2
    assert np.array_equal(o_c, one[800:])          # same tiles, same kernel -> bitwise


def test_swap_round_trip_scattered_and_resume_after_update():
    """Swap with scattered ids (interleaved allocation), invalidation while swapped, swap-in
    of the prefix and recompute from the LCP."""
    geo = W.Geometry(L=2, h_q=8, h_kv=2, d=128, k=16)
    seed = 92
    P = Pair(2, 8, 2, 128, 16, 96, 96)
    toks = {r: W.request_tokens(seed, r, 400) for r in range(3)}
    data = {r: _stream_qkv(seed, toks[r], geo) for r in range(3)}
    for r in range(3):
        P.new(r, toks[r])
    for a in range(0, 400, 100):                      # interleave -> scattered block ids
        for r in range(3):
            P.append([(r, None, 100, 0)], data[r][1][:, a:a + 100], data[r][2][:, a:a + 100])
    P.check_pools_whole()
    assert P.swap_out([2, 0]) == (s2l.OK, 2 * 25 * P.m_block)
    P.check_pools_whole()
    assert P.prefill([(1, 300, 100, 0)], data[1][0][300:])[0] is not None
    # update request 0 while swapped: keep 150 tokens
    new0 = W.updated_tokens(seed, 0, toks[0], 150, 400, 0)
    assert P.invalidate(0, new0) == (150, 250)
    assert P.swap_in([0, 2])[0] == s2l.OK
    P.check_state()
    P.check_pool_valid_slots()
    P.check_pools_whole()
    q0, k0, v0 = _stream_qkv(seed, new0, geo)
    P.append([(0, None, 250, 0)], k0[:, 150:], v0[:, 150:])
    P.prefill([(0, 150, 250, 0), (2, 0, 400, 250)], np.concatenate([q0[150:], data[2][0]]))
    P.check_pool_valid_slots()


def test_errors_and_edges_on_device():
    geo = W.Geometry(L=1, h_q=8, h_kv=2, d=128, k=16)
    P = Pair(1, 8, 2, 128, 16, 8, 4, max_blocks=64)
    toks = W.request_tokens(5, 0, 200)
    q, k, v = _stream_qkv(5, toks, geo)
    P.new(0, toks)
    # more blocks than the pool: all-or-nothing
    assert P.append([(0, None, 200, 0)], k, v) == s2l.E_NO_GPU_BLOCKS
    P.check_state()
    P2 = Pair(1, 8, 2, 128, 16, 8, 4)                                   # max_blocks_per_request = 8
    P2.new(0, toks)
    assert P2.append([(0, None, 200, 0)], k, v) == s2l.E_INVAL
    assert P.append([(0, None, 1, 0)], k[:, :1], v[:, :1]) == s2l.OK   # single token
    P.prefill([(0, 0, 1, 0)], q[:1])                                    # single row, one key
    assert P.append([(0, None, 127, 0)], k[:, 1:128], v[:, 1:128]) == s2l.OK
    P.prefill([(0, 127, 1, 0)], q[127:128])                             # exactly 128 keys
    P.prefill([(0, 0, 128, 0)], q[:128])
    with pytest.raises(s2l.S2LError) as e:
        P.lib.prefill_batch(0, [(0, 100, 29, 0)], to_dev(q[:29]), to_dev(q[:29]))
    assert e.value.status == s2l.E_INVAL                                # beyond nc
    assert P.swap_out([0])[0] == s2l.E_NO_CPU_BLOCKS                    # 8 blocks, 4 CPU
    P.lib.prefill_batch(0, [], to_dev(q[:1]), to_dev(q[:1]))            # empty batch is a no-op
    P.lib.sync()


# ----------------------------------------------------------------------------- full size, sampled
def _sample_rows(rng, n, extra=28):
    rows = {0, 1, n - 2, n - 1} | set(rng.integers(0, n, size=extra).tolist())
    return sorted(r for r in rows if 0 <= r < n)


@pytest.mark.slow
def test_c2_full_size_sampled_rows():
    """C2 (BJ:L8) at full size in the bench's launch configuration (8 requests, 512-token
    chunks, 32 steps to 16K): sampled rows of every step vs the oracle's row-wise fp64
    attention; one full request-step (the last) checked in full."""
    from oracle.attention import attention, attention_rows
    geo = W.LLAMA3_8B
    seed = W.seed_of(2)
    nreq, chunk, total = 8, 512, 16384
    cfg = s2l.make_config(1, 32, 8, 128, 16, nreq * total // 16 + 64, 0, max_requests=nreq,
                          max_blocks_per_request=total // 16)
    mb = s2l.block_bytes(cfg)
    pool = torch.empty(cfg.num_gpu_blocks * mb // 2, dtype=torch.bfloat16, device="cuda")
    lib = s2l.Context(cfg, pool, None, torch.cuda.current_stream(), None)
    toks = [W.request_tokens(seed, r, total) for r in range(nreq)]
    data = [_stream_qkv(seed, toks[r], geo) for r in range(nreq)]
    for r in range(nreq):
        lib.new_request(r, toks[r])
    rng = np.random.default_rng(0)
    worst = 0.0
    for j in range(total // chunk):
        a = j * chunk
        kk = to_dev(np.concatenate([data[r][1][:, a:a + chunk] for r in range(nreq)], axis=1))
        vv = to_dev(np.concatenate([data[r][2][:, a:a + chunk] for r in range(nreq)], axis=1))
        qq = to_dev(np.concatenate([data[r][0][a:a + chunk] for r in range(nreq)]))
        oo = torch.empty_like(qq)
        lib.append_chunk([(r, None, chunk, r * chunk) for r in range(nreq)], kk, vv)
        lib.prefill_batch(0, [(r, a, chunk, r * chunk) for r in range(nreq)], qq, oo)
        o = bf16_dev_to_f64(oo)
        if j % 4 == 3 or j == 0:
            r = j % nreq
            rows = _sample_rows(rng, chunk)
            o_ref, _ = attention_rows(data[r][0][a:a + chunk], data[r][1][0], data[r][2][0], a, rows)
            err = normwise_err(o[r * chunk:(r + 1) * chunk][rows], o_ref)
            worst = max(worst, float(err.max()))
            assert err.max() <= 2e-2, (j, r, float(err.max()))
    # last step, request 7, in full
    r = nreq - 1
    o_ref, _ = attention(data[r][0][total - chunk:], data[r][1][0], data[r][2][0], total - chunk)
    err = normwise_err(o[r * chunk:(r + 1) * chunk], o_ref)
    assert err.max() <= 2e-2, float(err.max())


def test_tc_tail_wave_kv_split_matches_unsplit(monkeypatch):
    """Few work units (< #SMs) -> the kernel splits each unit's KV range into pieces and the
    last piece merges the partial (O, m, l); must match the oracle and the unsplit kernel."""
    geo = W.LLAMA3_8B
    seed = 93
    toks = W.request_tokens(seed, 0, 3256)
    q, k, v = _stream_qkv(seed, toks, geo, q_scale=2.0)
    outs = []
    # unsplit; split with the last piece merging from its own TMEM when the others are
    # published (default); split with every merge through the workspace
    for no_split, direct in (("1", "1"), ("0", "1"), ("0", "0")):
        monkeypatch.setenv("S2L_NO_SPLIT", no_split)
        monkeypatch.setenv("S2L_SPLIT_DIRECT", direct)
        P = Pair(1, 32, 8, 128, 16, 256, 0, mirror=False)
        P.new(0, toks)
        P.append([(0, None, 3256, 0)], k, v)
        # 256 rows at p0 = 3000: 8 tiles -> 4 pairs x 8 heads = 32 units, ~24 KV tiles each
        o, _, l, _ = P.prefill([(0, 3000, 256, 0)], q[3000:])
        outs.append((o, l))
        # a second launch reuses the (self-resetting) arrival counters
        P.prefill([(0, 3000, 256, 0)], q[3000:])
    for o_, l_ in outs[1:]:
        assert normwise_err(outs[0][0], o_).max() <= 1e-2
        assert np.abs(outs[0][1] - l_).max() <= 1e-3


def test_c5_shape_reduced_long_request():
    """C5 shape (BJ:L11): Llama-3-70B attention (64 q / 8 kv heads, GQA group 8), one long
    request streamed in 2K-token chunks (reduced to 8K context so every row is checked)."""
    geo = W.LLAMA3_70B
    seed = W.seed_of(5)
    P = Pair(1, 64, 8, 128, 16, 600, 0, mirror=False)
    _multi_request_case(P, seed, geo, [8192], [[2048] * 4])


def test_c5_kv_head_sharding_on_device():
    """KV-head sharding: a context holding only kv heads {2,3} (q heads 16..31)
    reproduces the matching slice of the full-head computation."""
    from paper_2604_16395_b200 import shard
    geo = W.Geometry(L=1, h_q=64, h_kv=8, d=128, k=16)
    seed = 95
    toks = W.request_tokens(seed, 0, 1024)
    q, k, v = _stream_qkv(seed, toks, geo)
    kv_h, q_h = shard.kv_head_shard(1, 4, 64, 8)
    S = Pair(1, 16, 2, 128, 16, 128, 0, mirror=False)
    S.new(0, toks)
    S.append([(0, None, 1024, 0)], np.ascontiguousarray(k[:, :, kv_h]), np.ascontiguousarray(v[:, :, kv_h]))
    o_s, o_ref_s, _, _ = S.prefill([(0, 512, 512, 0)], np.ascontiguousarray(q[512:, q_h]))
    F = Pair(1, 64, 8, 128, 16, 128, 0, mirror=False)
    F.new(0, toks)
    F.append([(0, None, 1024, 0)], k, v)
    o_f, _, _, _ = F.prefill([(0, 512, 512, 0)], q[512:])
    assert normwise_err(o_s, o_f[:, q_h]).max() <= 2e-2


@pytest.mark.parametrize("seed", [0, 1])
def test_c4_mixed_stream_under_memory_pressure(seed):
    """C4-like mix (BJ:L10) at small scale: append-mode and update-mode requests interleaved
    with swap-out / swap-in under a GPU pool smaller than the working set, recompute
    preemption and release; every prefill is checked against the oracle and every GPU block
    and CPU block is compared byte for byte at the end (hazards between the copy stream and
    the compute stream would show up as stale or torn blocks)."""
    import random
    geo = W.Geometry(L=2, h_q=8, h_kv=2, d=128, k=16)
    rng = random.Random(seed)
    sd = 2000 + seed
    P = Pair(2, 8, 2, 128, 16, 48, 96, max_blocks=64)
    reqs = {}
    for rid in range(10):
        n = rng.randrange(200, 700)
        toks = W.request_tokens(sd, rid, n)
        reqs[rid] = dict(toks=toks, data=_stream_qkv(sd, toks, geo), mode=("append" if rid % 2 == 0 else "update"),
                         updates=0)
        P.new(rid, toks)
    for step in range(60):
        rid = rng.randrange(10)
        if rid not in P.ora.reqs:
            continue
        r = reqs[rid]
        info = P.lib.query(rid)
        if info["tier"] == s2l.TIER_CPU:
            st, _ = P.swap_in([rid])
            if st != s2l.OK:
                # make room: swap out the GPU-resident request holding the most blocks
                victims = sorted((x for x in P.ora.reqs if P.ora.reqs[x].tier == 0 and x != rid),
                                 key=lambda x: -len(P.ora.reqs[x].blocks))
                if victims:
                    if P.swap_out([victims[0]])[0] != s2l.OK:
                        P.lib.preempt_recompute(victims[0]); P.ora.preempt_recompute(victims[0])
                continue
        nc = P.lib.query(rid)["num_computed"]
        total = len(r["toks"])
        if r["mode"] == "update" and nc == total and r["updates"] < 2:
            p = rng.randrange(0, total)
            new = W.updated_tokens(sd, rid, r["toks"], p, total, r["updates"])
            r["updates"] += 1
            r["toks"] = new
            r["data"] = _stream_qkv(sd, new, geo)
            P.invalidate(rid, new)
            continue
        if nc == total:
            if rng.random() < 0.3:
                assert P.lib.release(rid) == s2l.OK and P.ora.release(rid) == 0
            continue
        n = min(total - nc, rng.choice([64, 128, 200]))
        q, k, v = r["data"]
        st = P.append([(rid, None, n, 0)], k[:, nc:nc + n], v[:, nc:nc + n])
        if st == s2l.E_NO_GPU_BLOCKS:
            victims = [x for x in P.ora.reqs if P.ora.reqs[x].tier == 0 and x != rid and P.ora.reqs[x].blocks]
            if victims:
                vtm = rng.choice(victims)
                if P.swap_out([vtm])[0] != s2l.OK:
                    P.lib.preempt_recompute(vtm); P.ora.preempt_recompute(vtm)
            continue
        assert st == s2l.OK
        layer = rng.randrange(2)
        P.prefill([(rid, nc, n, 0)], q[nc:nc + n], layer=layer)
        P.check_state()
    P.check_state()
    P.check_pool_valid_slots()
    P.check_pools_whole()


def _sample_rows_small(rng, n, k=6):
    return sorted(set([0, n - 1] + rng.choice(n, size=k, replace=False).tolist()))


@pytest.mark.parametrize("cooling", [False, True])
def test_stream_hazards_without_host_syncs(cooling):
    """Swaps run on their own streams and overlap compute that does not touch their blocks; the
    library orders only real conflicts (DESIGN.md §5 stream hazards).  With no host
    synchronisation inside each race, three races are provoked (the pool is sized so that the
    contested ids must be reused; each race asserts it really reused them) and checked after:
      1. swap_out(A) then an append of B into A's released ids (the append waits for the D2H);
      2. attention of A in flight, swap_out(A), swap_in(C) into A's released ids (the H2D waits
         for A's attention, not only for A's appends);
      3. attention of A in flight, invalidate_lcp(A) frees A's tail, swap_in(D) lands in it."""
    from oracle.attention import attention_rows
    from oracle.kvcache import OracleKV
    geo = W.Geometry(L=2, h_q=64, h_kv=8, d=128, k=16)
    seed = 777
    rid = {"A": 0, "B": 1, "C": 2, "D": 3}
    n = {"A": 4096, "B": 2048, "C": 2048, "D": 1024}
    ng, nc = 300, 600
    cfg = s2l.make_config(2, 64, 8, 128, 16, ng, nc, max_requests=8, max_blocks_per_request=512,
                          alloc_cooling=int(cooling))
    mb = s2l.block_bytes(cfg)
    gpool = torch.empty(ng * mb // 2, dtype=torch.bfloat16, device="cuda")
    cpool = torch.empty(nc * mb // 2, dtype=torch.bfloat16).pin_memory()
    lib = s2l.Context(cfg, gpool, cpool, torch.cuda.current_stream(), None)
    ora = OracleKV(2, 64, 8, 128, 16, ng, nc, max_requests=8, max_blocks_per_request=512, mirror_pools=False,
                   alloc_cooling=cooling)
    toks = {r: W.request_tokens(seed, rid[r], n[r]) for r in rid}
    data = {r: _stream_qkv(seed, toks[r], geo) for r in rid}
    dev = {r: (to_dev(data[r][0]), to_dev(data[r][1]), to_dev(data[r][2])) for r in rid}
    rng = np.random.default_rng(5)
    outs = []

    def append(r):
        lib.append_chunk([(rid[r], None, n[r], 0)], dev[r][1], dev[r][2])
        assert ora.append([(rid[r], None, n[r], 0)], data[r][1], data[r][2]) == 0

    def swap(r, out):
        a = (lib.swap_out if out else lib.swap_in)([rid[r]])
        assert a == (ora.swap_out if out else ora.swap_in)([rid[r]])[1]

    def prefill(r, layer):
        o = torch.empty_like(dev[r][0])
        lib.prefill_batch(layer, [(rid[r], 0, n[r], 0)], dev[r][0], o)
        outs.append((o, layer, r))

    def same():
        for r in rid:
            if r in [x for x in rid if rid[x] in ora.reqs]:
                assert lib.query(rid[r]) == ora.info(rid[r])
                assert lib.block_table(rid[r]) == ora.block_table(rid[r])
        assert lib.free_blocks() == ora.free_counts()

    def check_bytes(r):
        lib.sync()
        g = gpool.view(torch.int16).cpu().numpy().view(np.uint16).reshape(ng, 2, 2, 8, 16, 128)
        ids = np.array(lib.block_table(rid[r]))
        pos = np.arange(n[r])
        for kv in (0, 1):
            got = g[ids[pos // 16], :, kv, :, pos % 16, :]
            assert np.array_equal(got, np.transpose(data[r][1 + kv], (1, 0, 2, 3))), (r, kv)

    def release(r):
        lib.release(rid[r])
        assert ora.release(rid[r]) == 0

    for r in rid:
        lib.new_request(rid[r], toks[r]); ora.new_request(rid[r], toks[r])
    for r in ("C", "D"):          # C and D start on the CPU tier
        append(r)
        swap(r, True)
    append("A")
    lib.sync()
    # race 1: swap_out(A) then an append of B that must reuse A's released ids
    a_ids = set(lib.block_table(rid["A"]))
    swap("A", True)
    append("B")
    assert set(lib.block_table(rid["B"])) & a_ids
    same()
    check_bytes("B")
    release("B")
    # race 2: attention of A in flight, swap A out, swap C in (C must reuse A's ids)
    swap("A", False)
    for layer in range(2):
        prefill("A", layer)
    a_ids = set(lib.block_table(rid["A"]))
    swap("A", True)
    swap("C", False)
    assert set(lib.block_table(rid["C"])) & a_ids
    prefill("C", 1)
    same()
    check_bytes("C")
    release("C")
    # race 3: attention of A in flight, invalidate frees A's tail, D is swapped into it
    swap("A", False)
    prefill("A", 0)
    tail = set(lib.block_table(rid["A"])[63:])
    newA = W.updated_tokens(seed, 9, toks["A"], 1000, n["A"], 0)
    assert lib.invalidate_lcp(rid["A"], newA) == ora.invalidate_lcp(rid["A"], newA)[1:]
    swap("D", False)
    assert set(lib.block_table(rid["D"])) & tail
    prefill("D", 0)
    same()
    check_bytes("D")
    torch.cuda.synchronize()
    for o, layer, r in outs:
        rows = _sample_rows_small(rng, n[r])
        o_ref, _ = attention_rows(data[r][0], data[r][1][layer], data[r][2][layer], 0, rows)
        err = normwise_err(bf16_dev_to_f64(o)[rows], o_ref)
        assert err.max() <= 2e-2, (r, layer, float(err.max()))


@pytest.mark.parametrize("serial,cost,prefetch,cooling", [(False, False, 0, False), (False, False, 0, True),
                                                          (True, False, 0, False), (False, True, 0, False),
                                                          (False, False, 2, True)])
def test_c4_pressure_driver_on_device(serial, cost, prefetch, cooling):
    """The C4 driver (paper_2604_16395_b200.pressure) at reduced size on the device: 16
    append / update requests, GPU pool 50% of the working set, swaps overlapping compute (or
    serialised), no host synchronisation inside the stream.  Bookkeeping is mirrored into the
    oracle call by call (Twin); every step's output is checked on sampled rows of its first
    item against the oracle over that request's K/V history (all layers' attention runs; the
    last layer's output is checked), and the pool bytes of the request are checked whole at
    every 8th step."""
    from oracle.attention import attention_rows
    from paper_2604_16395_b200 import pressure
    from tests.harness import Twin
    L, K, budget = 2, 16, 2048
    plans = pressure.c4_plans(31, 16, lo=256, hi=2048, budget=budget)
    ws = pressure.working_set_blocks(plans, K)
    ng, ncpu = ws // 2, ws
    cfg = s2l.make_config(L, 32, 8, 128, K, ng, ncpu, max_requests=16, max_blocks_per_request=2048 // K,
                          alloc_cooling=int(cooling))
    mb = s2l.block_bytes(cfg)
    gpool = torch.empty(ng * mb // 2, dtype=torch.bfloat16, device="cuda")
    cpool = torch.empty(ncpu * mb // 2, dtype=torch.bfloat16).pin_memory()
    cs = torch.cuda.Stream()
    lib = s2l.Context(cfg, gpool, cpool, torch.cuda.current_stream(), cs)
    tw = Twin(lib, K, ng, ncpu, 16, 2048 // K)
    g = torch.Generator(device="cuda").manual_seed(5)
    src_k = torch.randn(L, budget, 8, 128, generator=g, device="cuda").to(torch.bfloat16)
    src_v = torch.randn(L, budget, 8, 128, generator=g, device="cuda").to(torch.bfloat16)
    src_q = torch.randn(budget, 32, 128, generator=g, device="cuda").to(torch.bfloat16)
    kh = src_k.view(torch.int16).cpu().numpy().view(np.uint16)
    vh = src_v.view(torch.int16).cpu().numpy().view(np.uint16)
    qh = src_q.view(torch.int16).cpu().numpy().view(np.uint16)
    segs, checks, byte_checks = {}, [], []
    rng = np.random.default_rng(0)
    rule = (lambda nc, nb: "recompute" if nc < 700 else "swap") if cost else None
    drv = pressure.PressureDriver(pressure.SwapTimer(tw, serial=serial), plans, K, budget, cost=rule,
                                  prefetch_ahead=prefetch)
    out_holder = {}

    def on_step(sel, app, pre, rows):
        for (r, _, n, row), (_, q_pos, _, _) in zip(app, pre):
            kept, acc = [], 0
            for a, m in segs.get(r, []):
                if acc >= q_pos:
                    break
                kept.append((a, min(m, q_pos - acc)))
                acc += kept[-1][1]
            kept.append((row, n))
            segs[r] = kept
        r, q_pos, n, row = pre[0]
        rows_s = sorted(set([0, n - 1] + rng.integers(0, n, 4).tolist()))
        idx = torch.tensor([row + t for t in rows_s], device="cuda")
        checks.append((r, list(segs[r]), q_pos, row, rows_s, out_holder["o"].index_select(0, idx)))
        if drv.step % 8 == 0:
            ids = lib.block_table(r)
            nc_r = q_pos + n
            blk = torch.tensor([ids[p // K] for p in range(nc_r)], device="cuda")
            slot = torch.tensor([p % K for p in range(nc_r)], device="cuda")
            view = gpool.view(ng, L, 2, 8, K, 128)
            byte_checks.append((list(segs[r]), view[blk, :, :, :, slot, :].clone()))

    out = torch.empty_like(src_q)
    out_holder["o"] = out
    ex = pressure.device_executor(drv.ctx, src_q, src_k, src_v, out, L, on_step)
    drv.run(ex)
    lib.sync()
    torch.cuda.synchronize()
    assert drv.swap_out_calls > 0 and drv.swap_in_calls > 0
    if cost:
        assert drv.recompute_preemptions > 0
    assert lib.free_blocks() == (ng, ncpu)
    for r, seg, q_pos, row, rows_s, o in checks:
        kk = np.concatenate([kh[L - 1, a:a + m] for a, m in seg])
        vv = np.concatenate([vh[L - 1, a:a + m] for a, m in seg])
        n = seg[-1][1]
        o_ref, _ = attention_rows(qh[row:row + n], kk, vv, q_pos, rows_s)
        err = normwise_err(bf16_dev_to_f64(o), o_ref)
        assert err.max() <= 2e-2, (r, q_pos, float(err.max()))
    for seg, got in byte_checks:
        got = got.view(torch.int16).cpu().numpy().view(np.uint16)      # [nc][L][2][h_kv][d]
        want_k = np.concatenate([kh[:, a:a + m] for a, m in seg], axis=1)  # [L][nc][h_kv][d]
        want_v = np.concatenate([vh[:, a:a + m] for a, m in seg], axis=1)
        assert np.array_equal(got[:, :, 0], np.transpose(want_k, (1, 0, 2, 3)))
        assert np.array_equal(got[:, :, 1], np.transpose(want_v, (1, 0, 2, 3)))


@pytest.mark.parametrize("policy,preemption", [("FCFS", "cost"), ("LCAS", "swap"), ("MCPS", "recompute")])
def test_streaming_scheduler_on_device(policy, preemption):
    """NEXT-3 at the parity bar: the two-phase scheduler (paper_2604_16395_b200.scheduler)
    drives a device context through a short synthetic crawler / ANNS mix under a GPU pool small
    enough to force preemption; every library call is mirrored into the oracle (Twin), and each
    step's attention output is checked on sampled rows of its first item against the oracle over
    that request's K/V history (tracked through appends, LCP invalidations and recompute)."""
    from oracle.attention import attention_rows
    from paper_2604_16395_b200 import costmodel, scheduler as S
    from synth import traces
    from tests.harness import Twin
    L, K, budget = 2, 16, 1024
    tr = traces.crawler_trace(41, 6, qps=50.0, lo=256, hi=1536, delay_scale=0.01) + \
        [(e[0], e[1] + 100, *e[2:]) for e in traces.anns_trace(42, 6, qps=50.0, lo=256, hi=1536, delay_scale=0.1)]
    tr.sort(key=lambda e: (e[0], e[1]))
    ng, ncpu = 160, 640
    cfg = s2l.make_config(L, 32, 8, 128, K, ng, ncpu, max_requests=16, max_blocks_per_request=1536 // K)
    mb = s2l.block_bytes(cfg)
    gpool = torch.empty(ng * mb // 2, dtype=torch.bfloat16, device="cuda")
    cpool = torch.empty(ncpu * mb // 2, dtype=torch.bfloat16).pin_memory()
    lib = s2l.Context(cfg, gpool, cpool, torch.cuda.current_stream(), torch.cuda.Stream())
    tw = Twin(lib, K, ng, ncpu, 16, 1536 // K)
    cm = costmodel.analytic(K, mb, 50e9, 2e-6)
    sch = S.StreamingScheduler(tw, policy, K, budget, ng, cost_model=cm, preemption=preemption)
    g = torch.Generator(device="cuda").manual_seed(9)
    src_k = torch.randn(L, budget, 8, 128, generator=g, device="cuda").to(torch.bfloat16)
    src_v = torch.randn(L, budget, 8, 128, generator=g, device="cuda").to(torch.bfloat16)
    src_q = torch.randn(budget, 32, 128, generator=g, device="cuda").to(torch.bfloat16)
    kh = src_k.view(torch.int16).cpu().numpy().view(np.uint16)
    vh = src_v.view(torch.int16).cpu().numpy().view(np.uint16)
    qh = src_q.view(torch.int16).cpu().numpy().view(np.uint16)
    segs, checks = {}, []
    rng = np.random.default_rng(1)
    t, i = 0.0, 0
    while True:
        while i < len(tr) and tr[i][0] <= t:
            tc, rid, n, tok, new, mode = tr[i]
            sch.on_chunk(tc, rid, n, tokens=tok, new_input=new, mode=mode)
            i += 1
        items = sch.step(t)
        if not items:
            if i >= len(tr):
                break
            t = tr[i][0]
            continue
        rows, app, pre = 0, [], []
        for r, q_pos, n in items:
            app.append((r, None, n, rows))
            pre.append((r, q_pos, n, rows))
            kept, acc = [], 0
            for a, m in segs.get(r, []):          # K/V history: positions < q_pos survive
                if acc >= q_pos:
                    break
                kept.append((a, min(m, q_pos - acc)))
                acc += kept[-1][1]
            assert acc == q_pos
            segs[r] = kept + [(rows, n)]
            rows += n
        tw.append_chunk(app, src_k, src_v, kv_rows=budget)
        out = torch.empty_like(src_q)
        for layer in range(L):
            lib.prefill_batch(layer, pre, src_q, out)
        r, q_pos, n, row = pre[0]
        rs = sorted(set([0, n - 1] + rng.integers(0, n, 3).tolist()))
        checks.append((list(segs[r]), q_pos, row, rs, out.index_select(0, torch.tensor([row + x for x in rs], device="cuda"))))
        t += 1e-3
        sch.finish_step(t, items)
        for r in list(segs):
            if r not in lib_reqs(tw):
                segs.pop(r)                        # released (finished)
    lib.sync()
    torch.cuda.synchronize()
    assert len(sch.ttfts()) == 12
    ev = [e[1] for e in sch.events]
    assert ev.count("PREEMPTED_SWAP") + ev.count("PREEMPTED_RECOMPUTE") > 0
    for seg, q_pos, row, rs, o in checks:
        kk = np.concatenate([kh[L - 1, a:a + m] for a, m in seg])
        vv = np.concatenate([vh[L - 1, a:a + m] for a, m in seg])
        n = seg[-1][1]
        o_ref, _ = attention_rows(qh[row:row + n], kk, vv, q_pos, rs)
        err = normwise_err(bf16_dev_to_f64(o), o_ref)
        assert err.max() <= 2e-2, (q_pos, float(err.max()))


def lib_reqs(tw):
    return set(tw.ora.reqs)


def test_swap_round_trip_full_size_c4_blocks():
    """a5/a6 at the C4 / bench size: 512 blocks of M_block = 2 MiB (L = 32, Llama-3-8B KV)
    of four interleaved requests (scattered ids) swapped out and back in, twice (the second
    round reuses CPU ids freed by the first and GPU ids released by the swap-out);
    every request's blocks must come back bit-identical (whole blocks, Z12)."""
    L, nblk = 32, 512
    cfg = s2l.make_config(L, 32, 8, 128, 16, nblk + 64, nblk + 64, max_requests=8, max_blocks_per_request=nblk)
    mb = s2l.block_bytes(cfg)
    assert mb == 2 * 1024 * 1024
    gpool = torch.empty((nblk + 64) * mb // 2, dtype=torch.bfloat16, device="cuda")
    cpool = torch.empty((nblk + 64) * mb // 2, dtype=torch.bfloat16).pin_memory()
    lib = s2l.Context(cfg, gpool, cpool, torch.cuda.current_stream(), torch.cuda.Stream(),
                      swap_in_stream=torch.cuda.Stream())
    rids = [0, 1, 2, 3]
    g = torch.Generator(device="cuda").manual_seed(3)
    kv = torch.randn(L, 4 * 512, 8, 128, generator=g, device="cuda").to(torch.bfloat16)
    for r in rids:
        lib.new_request(r, np.zeros(2048, np.int32))
    for a in range(0, 2048, 512):
        lib.append_chunk([(r, None, 512, i * 512) for i, r in enumerate(rids)], kv, kv)
    lib.sync()
    view = gpool.view(nblk + 64, mb // 2)
    before = {r: view[torch.tensor(lib.block_table(r), device="cuda")].clone() for r in rids}
    for _ in range(2):
        assert lib.swap_out(rids) == nblk * mb
        cview = cpool.view(nblk + 64, mb // 2)
        lib.sync()
        for r in rids:                                     # host copy == device blocks before
            got = cview[torch.tensor(lib.block_table(r))].cuda()
            assert torch.equal(got.view(torch.int16), before[r].view(torch.int16)), r
        view.fill_(0)                                      # freed GPU blocks: clobber them
        torch.cuda.synchronize()                           # (caller-side write: finish it first)
        assert lib.swap_in(rids) == nblk * mb
        lib.sync()
        for r in rids:
            got = view[torch.tensor(lib.block_table(r), device="cuda")]
            assert torch.equal(got.view(torch.int16), before[r].view(torch.int16)), r


# ----------------------------------------------------------------------------- NEXT-2 fused append
def _fused_rounds(P, seed, geo, chunks, check_every=True, check_last=True):
    """Each round: append_chunk in reserve mode, then one fused append + attention call per
    layer (library) vs the oracle's append + per-layer attention (every round, or only the
    fused kernel's own output of the last round)."""
    lengths = [sum(c) for c in chunks]
    toks = {r: W.request_tokens(seed, r, n) for r, n in enumerate(lengths)}
    data = {r: _stream_qkv(seed, toks[r], geo) for r in toks}
    for r in toks:
        P.new(r, toks[r])
    pos = {r: 0 for r in toks}
    for j in range(max(len(c) for c in chunks)):
        items_a, items_p, ks, vs, qs, row = [], [], [], [], [], 0
        for r in toks:
            if j >= len(chunks[r]):
                continue
            n, a = chunks[r][j], pos[r]
            items_a.append((r, None, n, row))
            items_p.append((r, a, n, row))
            ks.append(data[r][1][:, a:a + n]); vs.append(data[r][2][:, a:a + n]); qs.append(data[r][0][a:a + n])
            row += n
            pos[r] += n
        kk, vv, qq = np.concatenate(ks, axis=1), np.concatenate(vs, axis=1), np.concatenate(qs)
        P.append_reserve(items_a, kk, vv)
        last = j == max(len(c) for c in chunks) - 1
        for layer in range(geo.L):
            P.prefill_append(items_p, qq, kk[layer], vv[layer], layer=layer,
                             check=check_every or (check_last and last))
        P.check_state()
        P.check_pool_valid_slots()
    P.check_pools_whole()


@pytest.mark.parametrize("h_q,h_kv,k,L", [(8, 2, 16, 2), (32, 8, 16, 1), (4, 4, 64, 2), (16, 2, 128, 1), (8, 8, 32, 1)])
def test_fused_append_prefill_aligned(h_q, h_kv, k, L):
    """Every q_pos block-aligned: the attention kernel reads the chunk's K/V from the caller's
    rows and writes the pool itself (full blocks by TMA store, the partial last block by plain
    stores); pool bytes bit-exact, attention within tolerance, every layer."""
    geo = W.Geometry(L=L, h_q=h_q, h_kv=h_kv, d=128, k=k)
    P = Pair(L, h_q, h_kv, 128, k, 256, 8, max_blocks=128)
    b = k
    _fused_rounds(P, W.seed_of(21), geo, [[4 * b, 8 * b, 37], [b, 300], [200], [2 * b, 2 * b, 2 * b, 5]])


def test_fused_append_prefill_unaligned_falls_back():
    """A q_pos inside a block (token-granular appends / invalidation): the same call runs a
    one-layer append launch before the attention; results and bytes identical to the oracle."""
    geo = W.Geometry(L=2, h_q=8, h_kv=2, d=128, k=16)
    P = Pair(2, 8, 2, 128, 16, 128, 8, max_blocks=64)
    _fused_rounds(P, W.seed_of(22), geo, [[10, 50, 130], [16, 7, 200]])


def test_fused_append_prefill_after_update_and_errors():
    """Update mode then the fused path from the LCP; error cases."""
    geo = W.Geometry(L=1, h_q=8, h_kv=2, d=128, k=16)
    P = Pair(1, 8, 2, 128, 16, 64, 8, max_blocks=64)
    seed = W.seed_of(23)
    toks = W.request_tokens(seed, 0, 256)
    q, k, v = _stream_qkv(seed, toks, geo)
    P.new(0, toks)
    P.append_reserve([(0, None, 256, 0)], k, v)
    P.prefill_append([(0, 0, 256, 0)], q, k[0], v[0])
    new = W.updated_tokens(seed, 0, toks, 100, 300, 0)
    p, inval = P.invalidate(0, new)
    q2, k2, v2 = _stream_qkv(seed, new, geo)
    c = P.lib.query(0)["num_computed"]
    P.append_reserve([(0, None, 300 - c, 0)], k2[:, c:], v2[:, c:])
    P.prefill_append([(0, c, 300 - c, 0)], q2[c:], k2[0, c:], v2[0, c:])
    P.check_pool_valid_slots()
    qd, kd = to_dev(q2[c:]), to_dev(k2[0, c:])
    od = torch.zeros_like(qd)
    with pytest.raises(s2l.S2LError) as e:
        P.lib.prefill_append(0, [(0, c, 300 - c, 0)], qd, kd, None, od)
    assert e.value.status == s2l.E_INVAL
    with pytest.raises(s2l.S2LError) as e:
        P.lib.prefill_append(0, [(0, c, 10, 0), (0, c + 10, 10, 10)], qd, kd, kd, od)
    assert e.value.status == s2l.E_INVAL


def test_fused_append_prefill_c2_shape():
    """C2 geometry and launch shape (Llama-3-8B attention: 32 q / 8 kv heads, k = 16, 8
    requests x 512-token chunks) to 4K through the fused path: pool bytes bit-exact after
    every round, and the FUSED kernel's own output (every row, every head, LSE) vs the oracle
    at the last round (the earlier rounds run unchecked for speed)."""
    geo = W.Geometry(L=1, h_q=32, h_kv=8, d=128, k=16)
    P = Pair(1, 32, 8, 128, 16, 8 * 256 + 8, 8, max_blocks=256)
    _fused_rounds(P, W.seed_of(24), geo, [[512] * 8] * 8, check_every=False, check_last=True)


def test_fused_append_then_swap_without_host_sync():
    """Stream hazard of the fused path: a swap-out issued right after s2l_prefill_append (no host
    synchronisation) must copy the blocks that kernel writes (the D2H waits for it, §5), and a
    later append reusing the freed ids must not overtake the D2H."""
    geo = W.Geometry(L=2, h_q=8, h_kv=2, d=128, k=16)
    P = Pair(2, 8, 2, 128, 16, 48, 64, max_blocks=64)   # request 1 must reuse 16 of request 0's ids
    seed = W.seed_of(25)
    toks = {r: W.request_tokens(seed, r, 512) for r in (0, 1)}
    data = {r: _stream_qkv(seed, toks[r], geo) for r in (0, 1)}
    P.new(0, toks[0]); P.new(1, toks[1])
    q, k, v = data[0]
    P.append_reserve([(0, None, 512, 0)], k, v)
    qd, od = to_dev(q), torch.zeros(512, 8, 128, dtype=torch.bfloat16, device="cuda")
    kd = [to_dev(k[l]) for l in range(2)]
    vd = [to_dev(v[l]) for l in range(2)]
    for l in range(2):
        P.lib.prefill_append(l, [(0, 0, 512, 0)], qd, kd[l], vd[l], od)
    P.swap_out([0])                      # no synchronisation since the fused launches
    q1, k1, v1 = data[1]
    P.append([(1, None, 512, 0)], k1, v1)   # reuses ids request 0 just released
    assert set(P.lib.block_table(1)) & set(range(32))
    P.check_state()
    P.check_pools_whole()                # request 0's CPU copy == the oracle's bytes
    P.prefill([(1, 384, 128, 0)], q1[384:])


# ----------------------------------------------------------------------------- NEXT-4 per-layer API in a forward pass
def test_streaming_decoder_chunked_equals_one_shot_and_oracle():
    """A 2-layer random-weight decoder (paper_2604_16395_b200.model) prefilled chunk by chunk
    through s2l_prefill_append (reserve once per chunk, one fused launch per layer) gives the
    same last-layer hidden states as one-shot prefill of the whole input (chunked prefill
    reuses the cache of earlier chunks); every layer's attention output of the chunked run equals
    the fp64 oracle on the layer's own Q/K/V at sampled rows."""
    from oracle.attention import attention_rows
    from paper_2604_16395_b200 import model as M
    shape = M.Shape(layers=2, hidden=1024, h_q=8, h_kv=2, d=128, inter=2048)
    lens = {0: 300, 1: 200}
    chunks = {0: [128, 128, 44], 1: [64, 64, 72]}
    gtok = torch.Generator().manual_seed(5)
    toks = {r: torch.randint(0, 32768, (n,), generator=gtok) for r, n in lens.items()}

    def make(ng):
        cfg = s2l.make_config(shape.layers, shape.h_q, shape.h_kv, shape.d, 16, ng, 0, max_requests=4,
                              max_blocks_per_request=64)
        pool = torch.empty(ng * s2l.block_bytes(cfg) // 2, dtype=torch.bfloat16, device="cuda")
        ctx = s2l.Context(cfg, pool, None, torch.cuda.current_stream(), None)
        for r in lens:
            ctx.new_request(r, toks[r].tolist())
        return ctx, pool

    ca, pa = make(64)
    A = M.StreamingDecoder(shape, ca, seed=3)
    pos = {r: 0 for r in lens}
    last = {}
    traces = []
    for j in range(3):
        items, tt, row = [], [], 0
        for r in lens:
            n = chunks[r][j]
            items.append((r, pos[r], n, row))
            tt.append(toks[r][pos[r]:pos[r] + n])
            row += n
        tr = []
        x = A.chunk(items, torch.cat(tt).cuda(), trace=tr)
        traces.append((items, tr))
        for r, p, n, rw in items:
            last[r] = (p, x[rw:rw + n].float().cpu())
            pos[r] += n
    cb, pb = make(64)
    B = M.StreamingDecoder(shape, cb, seed=3)
    items = [(0, 0, 300, 0), (1, 0, 200, 300)]
    xb = B.chunk(items, torch.cat([toks[0], toks[1]]).cuda()).float().cpu()
    for r, p, n, rw in items:
        pl, xl = last[r]
        ref = xb[rw + pl: rw + p + n]
        err = ((xl - ref).abs().amax(-1) / ref.abs().amax(-1).clamp_min(1e-6)).max().item()
        assert err <= 2e-2, (r, err)
    # every layer's attention of the last chunk vs the oracle on that layer's own Q/K/V history
    bits = lambda t: t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    for layer in range(shape.layers):
        for r in lens:
            ks, vs = [], []
            for items_j, tr in traces:
                _, q, k, v, o = tr[layer]
                for rr, p, n, rw in items_j:
                    if rr == r:
                        ks.append(bits(k[rw:rw + n])); vs.append(bits(v[rw:rw + n]))
                        qr, orow, qp, nn = bits(q[rw:rw + n]), o[rw:rw + n], p, n
            rows_s = [0, nn // 2, nn - 1]
            o_ref, _ = attention_rows(qr, np.concatenate(ks), np.concatenate(vs), qp, rows_s)
            og = orow[rows_s].float().cpu().numpy().astype(np.float64)
            err = normwise_err(og, o_ref).max()
            assert err <= 2e-2, (layer, r, err)
    ca.close(); cb.close()


def test_fused_append_then_invalidate_and_swap_in_without_host_sync():
    """Stream hazard of the fused path (WAW across streams): the fused kernel writes request A's
    blocks; without a host sync A is invalidated to 0 and request B is swapped in, receiving
    those ids.  The H2D must wait for the fused kernel, else the kernel's late writes would
    corrupt B's restored blocks."""
    geo = W.Geometry(L=1, h_q=8, h_kv=2, d=128, k=16)
    P = Pair(1, 8, 2, 128, 16, 48, 64, max_blocks=64)
    seed = W.seed_of(26)
    toks = {r: W.request_tokens(seed, r, 512) for r in (0, 1)}
    data = {r: _stream_qkv(seed, toks[r], geo) for r in (0, 1)}
    P.new(0, toks[0]); P.new(1, toks[1])
    qb, kb_, vb = data[1]
    P.append_reserve([(1, None, 256, 0)], kb_[:, :256], vb[:, :256])
    P.prefill_append([(1, 0, 256, 0)], qb[:256], kb_[0, :256], vb[0, :256])
    assert P.swap_out([1])[0] == s2l.OK                  # B on the CPU tier, ids 0..15 released
    qa, ka, va = data[0]
    P.append_reserve([(0, None, 512, 0)], ka, va)        # A takes 32 of the 48 ids
    a_ids = set(P.lib.block_table(0))
    qd, kd, vd = to_dev(qa), to_dev(ka[0]), to_dev(va[0])
    od = torch.zeros_like(qd)
    P.lib.prefill_append(0, [(0, 0, 512, 0)], qd, kd, vd, od)   # no synchronisation after this
    P.invalidate(0, [])                                   # frees all of A's blocks
    assert P.swap_in([1])[0] == s2l.OK                    # B lands in ids A's kernel writes
    assert set(P.lib.block_table(1)) & a_ids
    P.check_state()
    P.check_pools_whole()
    P.prefill([(1, 128, 128, 0)], qb[128:256])


@pytest.mark.parametrize("released,min_runs", [(list(range(0, 64, 2)), 16), ([3, 9, 10, 17, 30, 31], 4)])
def test_swap_scattered_ids_staged_path(released, min_runs):
    """a5 / a6 with scattered GPU ids (one-block requests released first, so the swapped
    request's 32 blocks start with one- and two-block runs: every other of 64 -> 32 runs, or six
    ids -> 5 runs, the smallest run count the staged path takes): the library stages the copies
    through device memory (gather kernel + one DMA per CPU-id run; H2D + scatter kernel).
    Whole blocks must round-trip bit-exactly and match the oracle's pool mirrors; attention
    after the round trip matches the oracle."""
    geo = W.Geometry(L=1, h_q=8, h_kv=2, d=128, k=16)
    P = Pair(1, 8, 2, 128, 16, 96, 64, max_requests=80, max_blocks=64)
    seed = W.seed_of(27)
    one = _stream_qkv(seed, W.request_tokens(seed, 99, 16), geo)
    for f in range(64):
        P.new(f, W.request_tokens(seed, 1000 + f, 16))
    P.append([(f, None, 16, 0) for f in range(64)], one[1], one[2])
    for f in released:
        P.lib.release(f)
        assert P.ora.release(f) == 0
    toks = W.request_tokens(seed, 7, 512)
    q, k, v = _stream_qkv(seed, toks, geo)
    P.new(500, toks)
    P.append([(500, None, 512, 0)], k, v)
    ids = P.lib.block_table(500)
    runs = 1 + sum(1 for a, b in zip(ids, ids[1:]) if b != a + 1)
    assert runs >= min_runs, runs
    before = P.gpu_pool_bits()[ids].copy()
    assert P.swap_out([500])[0] == s2l.OK
    assert np.array_equal(P.cpu_pool_bits()[P.lib.block_table(500)], before)
    P.check_pools_whole()
    assert P.swap_in([500])[0] == s2l.OK
    P.check_state()
    P.check_pools_whole()
    P.prefill([(500, 384, 128, 0)], q[384:])
