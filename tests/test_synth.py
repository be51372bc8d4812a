"""The shared seeded input generator: determinism, bf16 rounding, distribution, prefix property."""
import numpy as np
import torch

import synth


def test_splitmix64_known_values():
    # splitmix64 reference sequence for state 0 (Vigna's splitmix64.c: next() from x=0)
    assert synth.splitmix64_int(0) == 0xE220A8397B1DCDAF
    assert int(synth.splitmix64(np.array([0], np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100000) * 10.0 ** rng.integers(-8, 8, 100000),
                        [0.0, -0.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, 65280.5]])
    ours = synth.f64_to_bf16_bits(x)
    ref = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)


def test_rows_deterministic_and_prefix_stable():
    t = synth.tokens(3, 0, 50)
    assert t.dtype == np.int32 and t.min() >= 0 and t.max() < synth.VOCAB
    assert np.array_equal(t, synth.tokens(3, 0, 50))
    assert np.array_equal(t[10:], synth.tokens(3, 0, 40, start=10))
    H = synth.prefix_hashes(3, t)
    t2 = t.copy(); t2[20] += 1
    H2 = synth.prefix_hashes(3, t2)
    assert np.array_equal(H[:20], H2[:20]) and not np.any(H[20:] == H2[20:])
    a = synth.rows(3, synth.KIND_K, 0, H, range(4), 32)
    b = synth.rows(3, synth.KIND_K, 0, H2, range(4), 32)
    assert np.array_equal(a[:20], b[:20]) and not np.array_equal(a[20], b[20])


def test_rows_distribution():
    H = synth.prefix_hashes(9, synth.tokens(9, 0, 4096))
    r = synth.rows(9, synth.KIND_V, 0, H, range(8), 128)
    x = (r.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    # N(0,1): mean, variance, Gaussian kurtosis and tails
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1.0) < 0.01
    kurt = ((x - x.mean()) ** 4).mean() / x.var() ** 2
    assert abs(kurt - 3.0) < 0.05, kurt
    assert abs((np.abs(x) > 3.0).mean() - 0.0027) < 0.0006       # 2 * (1 - Phi(3)) = 0.0027
    assert 4.0 < np.abs(x).max() <= 6.8
    # multithreaded path == single chunk
    r1 = synth.rows(9, synth.KIND_V, 0, H[:7], range(8), 128)
    assert np.array_equal(r1, r[:7])
