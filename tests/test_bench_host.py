"""Host-side pieces of bench.py (no GPU): the side-field guard and the algorithmic FLOP count
(causally visible pairs only)."""
import pytest

import bench


def test_guarded_side_field_records_errors_at_one_rank():
    line = {}
    bench._guarded(line, "ok", lambda: {"value": 1}, 1)
    bench._guarded(line, "none", lambda: None, 1)          # writes its own fields
    bench._guarded(line, "bad", lambda: 1 / 0, 1)
    assert line["ok"] == {"value": 1} and "none" not in line
    assert "bad" not in line and line["bad_error"].startswith("ZeroDivisionError")


def test_guarded_side_field_propagates_with_several_ranks():
    with pytest.raises(ZeroDivisionError):
        bench._guarded({}, "bad", lambda: 1 / 0, 2)


def test_attn_flops_is_the_causal_pair_count():
    # 4 d h_q per visible (q, k) pair: n p0 prefix pairs + n (n + 1) / 2 causal pairs in the chunk
    d, h = 128, 32
    assert bench.attn_flops(1, 0, h_q=h, d=d) == 4 * d * h * 1
    assert bench.attn_flops(3, 5, h_q=h, d=d) == 4 * d * h * (3 * 5 + 6)
    # chunked == one shot: the pairs of consecutive chunks add up to those of the whole input
    whole = bench.attn_flops(1024, 0, h_q=h, d=d)
    parts = sum(bench.attn_flops(256, 256 * j, h_q=h, d=d) for j in range(4))
    assert parts == whole
