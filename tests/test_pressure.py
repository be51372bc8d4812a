"""C4 memory-pressure driver (paper_2604_16395_b200.pressure) on a host-only context: every
library call it makes is mirrored into the oracle's state machine and must agree bit for bit
(block tables on both tiers, counts, LCP, swap sizes), and the workload recipe is checked
against its definition (BJ:L10)."""
import numpy as np
import pytest

from paper_2604_16395_b200 import pressure, s2l
from synth import workloads as W
from tests.harness import Twin


def _run_host(seed, n_req, lo, hi, budget, frac=0.5, k=16, cost=None, prefetch=0, reserve=0):
    plans = pressure.c4_plans(seed, n_req, lo=lo, hi=hi, budget=budget)
    ws = pressure.working_set_blocks(plans, k)
    biggest = max(-(-p.total // k) for p in plans)
    ng = max(int(ws * frac), 3 * biggest + budget // k + 2)
    nc = ws + 8
    cfg = s2l.make_config(1, 1, 1, 8, k, ng, nc, max_requests=n_req, max_blocks_per_request=biggest + 1)
    lib = s2l.Context(cfg, host_only=True)
    tw = Twin(lib, k, ng, nc, n_req, biggest + 1)
    drv = pressure.PressureDriver(tw, plans, k, budget, cost=cost, prefetch_ahead=prefetch,
                                  reserve=int(reserve * ng))

    def execute(sel, app, pre, rows):
        tw.append_chunk(app, None, None, kv_rows=rows)

    steps = drv.run(execute)
    return plans, drv, steps, ng, ws


@pytest.mark.parametrize("seed,prefetch", [(11, 0), (12, 0), (11, 2), (12, 1)])
def test_driver_bookkeeping_matches_oracle_under_pressure(seed, prefetch):
    plans, drv, steps, ng, ws = _run_host(seed, 24, 64, 1024, 512, prefetch=prefetch)
    if prefetch:
        assert drv.prefetched > 0
    assert ng < ws                                   # the pool really is under pressure
    assert drv.swap_out_calls > 0 and drv.swap_in_calls > 0
    assert not drv.live() and not drv.plans          # every request finished and was released
    tw = drv.ctx
    assert tw.lib.free_blocks() == (ng, tw.ora.num_cpu_blocks)
    # every token of every work item went through one append
    want = sum(w.n_kv for p in plans for w in p.work)
    assert drv.tokens == want
    # the op log names every library call; swaps in both directions are whole requests
    kinds = {op for op, _, _ in drv.log}
    assert {"new", "append", "prefill", "swap_out", "swap_in", "release", "invalidate"} <= kinds


def test_driver_free_block_reserve():
    """reserve > 0 (C4_RESERVE): the driver keeps extra GPU blocks free beyond the look-ahead's
    needs (best effort).  Every library call still agrees with the oracle (Twin), all requests
    finish, and it swaps out at least as many bytes as without the reserve."""
    _, d0, _, ng, _ = _run_host(11, 24, 64, 1024, 512)
    _, d1, _, ng1, _ = _run_host(11, 24, 64, 1024, 512, reserve=0.1)
    assert ng1 == ng
    assert not d1.live() and not d1.plans
    assert d1.ctx.lib.free_blocks() == (ng, d1.ctx.ora.num_cpu_blocks)
    assert d1.swapped_out_bytes >= d0.swapped_out_bytes
    assert d1.tokens == d0.tokens


def test_driver_steps_respect_budget_and_round_robin():
    plans = pressure.c4_plans(3, 16, lo=64, hi=1024, budget=700)
    lens = {p.rid: [w.n_kv for w in p.work] for p in plans}
    cfg = s2l.make_config(1, 1, 1, 8, 16, 4096, 4096, max_requests=16, max_blocks_per_request=128)
    lib = s2l.Context(cfg, host_only=True)
    drv = pressure.PressureDriver(lib, plans, 16, 700)
    seen_per_step = []

    def execute(sel, app, pre, rows):
        assert rows == sum(n for _, _, n, _ in app)
        assert rows <= 700 or len(sel) == 1          # budget, unless one item alone exceeds it
        assert len(set(sel)) == len(sel)
        for (r, _, n, row), (r2, q_pos, n_q, q_row) in zip(app, pre):
            assert r == r2 and n == n_q and row == q_row
        lib.append_chunk(app, None, None, kv_rows=rows)
        seen_per_step.append(list(sel))

    drv.run(execute)
    # round robin: each step is an increasing run of ids with at most one wrap-around, and
    # the next step starts after the previous step's last id unless it wraps
    for sel in seen_per_step:
        assert sum(1 for x, y in zip(sel, sel[1:]) if y < x) <= 1
    for a, b in zip(seen_per_step, seen_per_step[1:]):
        assert b[0] > a[-1] or b[0] <= min(b)
    # work order per request is preserved
    got = {}
    for step in seen_per_step:
        for r in step:
            got[r] = got.get(r, 0) + 1
    assert got == {r: len(v) for r, v in lens.items()}


def test_c4_recipe():
    """BJ:L10 / SURVEY d.2 C4 recipe: even ids append-mode (6-10 chunks, tokens arrive with
    the chunks), odd ids update-mode (whole input, 2 chunks, 1-2 updates with LCP in
    [ceil(0.2T), floor(0.8T)], recompute T - p in budget-sized pieces); totals in [lo, hi]."""
    plans = pressure.c4_plans(1004, 128, budget=8192)
    assert len(plans) == 128
    for p in plans:
        assert 1024 <= p.total <= 16384
        if p.rid % 2 == 0:
            assert p.mode == "append" and 6 <= len(p.work) <= 10 and len(p.initial_tokens) == 0
            assert sum(w.n_kv for w in p.work) == p.total
            assert np.array_equal(np.concatenate([w.append_tokens for w in p.work]),
                                  W.request_tokens(1004, p.rid, p.total))
            assert max(w.n_kv for w in p.work) - min(w.n_kv for w in p.work) <= 1
        else:
            assert p.mode == "update" and len(p.initial_tokens) == p.total
            assert p.work[0].n_kv + p.work[1].n_kv == p.total
            ups = [w for w in p.work[2:] if w.new_input is not None]
            assert 1 <= len(ups) <= 2
            for w in ups:
                assert len(w.new_input) == p.total
            rec = sum(w.n_kv for w in p.work[2:])
            assert all(w.n_kv <= 8192 for w in p.work)
            # each update recomputes T - p with p in [ceil(0.2T), floor(0.8T)]
            assert len(ups) * (p.total - (8 * p.total) // 10) <= rec <= len(ups) * (p.total - (-(-2 * p.total // 10)))
    # lognormal medians: append ~5.8K, update ~10K, loosely
    a = np.median([p.total for p in plans if p.mode == "append"])
    u = np.median([p.total for p in plans if p.mode == "update"])
    assert 3500 < a < 9000 and 7000 < u < 13000


def test_cost_based_preemption_recomputes_small_victims():
    """With a cost rule (P:L79 / §4.3) small victims are dropped and re-prefilled instead of
    swapped; bookkeeping still mirrors the oracle call by call, every request finishes, and the
    recomputed tokens are exactly the dropped prefixes."""
    rule = lambda nc, nb: "recompute" if nc < 400 else "swap"
    plans, drv, steps, ng, ws = _run_host(13, 24, 64, 1024, 512, cost=rule)
    assert drv.recompute_preemptions > 0 and drv.swap_out_calls > 0
    assert not drv.live() and not drv.plans
    want = sum(w.n_kv for p in plans for w in p.work) + drv.recomputed_tokens
    assert drv.tokens == want
    assert drv.ctx.lib.free_blocks() == (ng, drv.ctx.ora.num_cpu_blocks)
