"""CPU tests of the recompute-vs-swap cost model (NEXT-1), pinned to the paper's formulas
 and SPEC's tie rule."""
import math

import pytest

from oracle.geometry import block_bytes
from paper_2604_16395_b200.costmodel import CostModel, PiecewiseLinear, analytic


def test_piecewise_linear_interpolates_and_extrapolates():
    f = PiecewiseLinear([1000, 2000, 4000], [1.0, 3.0, 4.0])
    assert f(1000) == 1.0 and f(2000) == 3.0 and f(4000) == 4.0
    assert f(1500) == 2.0 and f(3000) == 3.5
    assert f(500) == 0.5           # below the first sample: through the origin
    assert f(0) == 0.0
    assert f(6000) == 5.0          # last segment's slope
    with pytest.raises(ValueError):
        PiecewiseLinear([1, 1], [0, 0])


def test_analytic_model_reproduces_paper_formulas():
    """C_recomp = ℓ·C_prefill; C_swap = ⌈ℓ/k⌉·M_block/BW; compare with 2·C_swap."""
    k = 16
    mb = block_bytes(32, 16, 8, 128)               # 2 MiB for Llama-3.1-8B
    bw = 55e9                                       # measured PCIe Gen5 x16 H2D on the B200 box
    c_pre = 50e-3 / 8192                            # the paper's illustrative "50 ms" scale
    cm = analytic(k, mb, bw, c_pre)
    for ell in (1, 15, 16, 17, 1000, 32768):
        nb = math.ceil(ell / k)
        assert math.isclose(cm.recompute_latency(ell), ell * c_pre, rel_tol=1e-12)
        assert math.isclose(cm.swap_latency(nb), nb * mb / bw, rel_tol=1e-12)
        want = "recompute" if ell * c_pre <= 2 * nb * mb / bw else "swap"
        assert cm.choose_eviction(ell) == want
    # per token: recompute 6.1 us vs swap 2 x (2 MiB / 16) / 55 GB/s = 4.8 us -> swap wins for
    # long requests; for 1 token the full-block swap (76 us) loses to recompute
    assert cm.choose_eviction(1) == "recompute"
    assert cm.choose_eviction(32768) == "swap"


def test_tie_goes_to_recompute():
    cm = CostModel(16, PiecewiseLinear([0, 16], [0.0, 2.0]), PiecewiseLinear([0, 1], [0.0, 1.0]))
    assert cm.recompute_latency(16) == 2 * cm.swap_latency(1)
    assert cm.choose_eviction(16) == "recompute"


def test_crossover_and_json_roundtrip(tmp_path):
    # recompute grows superlinearly (attention ~ ℓ²), swap linearly: one crossing
    xs = [1024 * 2 ** i for i in range(8)]
    rec = PiecewiseLinear(xs, [4e-8 * x * x / 1024 for x in xs])
    swp = PiecewiseLinear([1, 8192], [1e-5, 8192e-5])
    cm = CostModel(16, rec, swp, {"kind": "test"})
    t = cm.crossover_tokens()
    assert t is not None
    assert cm.choose_eviction(t) == "swap" and cm.choose_eviction(t - 1) == "recompute"
    p = tmp_path / "cm.json"
    cm.save(p)
    cm2 = CostModel.load(p)
    for ell in (100, 5000, 70000):
        assert cm2.choose_eviction(ell) == cm.choose_eviction(ell)
        assert cm2.recompute_latency(ell) == cm.recompute_latency(ell)
