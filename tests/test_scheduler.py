"""Two-phase streaming scheduler (paper_2604_16395_b200.scheduler) on host-only
contexts: policy orderings as §4.4 defines them, Phase 1 budget / feasibility, Phase 2
preemption order and the cost-based recompute-vs-swap choice, LCP invalidation on
update chunks, and whole synthetic traces run to completion with every library
call mirrored into the oracle's state machine (Twin)."""
import numpy as np
import pytest

from paper_2604_16395_b200 import costmodel, s2l, scheduler as S
from synth import traces
from tests.harness import Twin


def _ctx(ng, nc, k=16, max_req=256, max_blocks=4096, twin=True):
    cfg = s2l.make_config(1, 1, 1, 8, k, ng, nc, max_requests=max_req, max_blocks_per_request=max_blocks)
    lib = s2l.Context(cfg, host_only=True)
    return Twin(lib, k, ng, nc, max_req, max_blocks) if twin else lib


def _cm(crossover_tokens=4096, k=16):
    """Analytic model whose recompute/2x-swap crossover is at `crossover_tokens`."""
    m_block, bw = 1 << 21, 50e9
    per_tok = 2 * (m_block / k) / bw * 1.0          # recompute = 2*swap exactly at slope level
    cm = costmodel.analytic(k, m_block, bw, per_tok * 1.0, max_tokens=1 << 17)
    # shift: recompute gets a fixed cost so that it loses above the crossover
    rec = costmodel.PiecewiseLinear([0, crossover_tokens, 1 << 17],
                                    [0.0, crossover_tokens * per_tok, (1 << 17) * per_tok * 3])
    return costmodel.CostModel(k, rec, cm.swap_s, {})


def _exec(ctx):
    def run(items):
        if items:
            ctx.append_chunk([(r, None, n, 0) for r, _, n in items], None, None,
                             kv_rows=max(n for _, _, n in items))
    return run


def test_policy_orderings():
    ctx = _ctx(1024, 0)
    sch = S.StreamingScheduler(ctx, "FCFS", 16, 1 << 20, 1024, preemption="recompute")
    # r0: arrived first, partial; r1: complete, arrived second; r2: complete, newest chunk
    sch.on_chunk(0.0, 0, 3, tokens=np.arange(10))
    sch.on_chunk(1.0, 1, 1, tokens=np.arange(20))
    sch.on_chunk(2.0, 2, 2, tokens=np.arange(5))
    sch.on_chunk(5.0, 2, 2, tokens=np.arange(5))
    sch.on_chunk(3.0, 0, 3, tokens=np.arange(10))
    info = {r: ctx.query(r) for r in (0, 1, 2)}
    assert sch.order([0, 1, 2], info) == [1, 2, 0]          # FCFS: complete tier by arrival
    sch.policy = "LCAS"
    assert sch.order([0, 1, 2], info) == [2, 1, 0]          # LCAS: complete tier, newest chunk first
    sch.policy = "MCPS"
    ctx.append_chunk([(1, None, 8, 0)], None, None, kv_rows=8)
    ctx.append_chunk([(0, None, 12, 0)], None, None, kv_rows=12)
    info = {r: ctx.query(r) for r in (0, 1, 2)}
    assert sch.order([0, 1, 2], info) == [0, 1, 2]          # MCPS: most computed first
    sch.policy = "DEFAULT"
    sch.running = [2]
    sch.reqs[1].preempted_front = True
    assert sch.order([0, 1, 2], info) == [2, 1, 0]          # running, then preempted at front, FIFO


def test_phase1_budget_clamps_and_phase2_preempts_lowest_priority():
    ng = 64
    ctx = _ctx(ng, 256)
    sch = S.StreamingScheduler(ctx, "FCFS", 16, 512, ng, preemption="swap")
    run = _exec(ctx)
    # three requests, 400 tokens each (25 blocks), arriving in order; budget 512 per step
    for r in range(3):
        sch.on_chunk(float(r), r, 1, tokens=np.arange(400))
    items = sch.step(3.0)
    assert items == [(0, 0, 400), (1, 0, 112)]               # budget-clamped partial chunk
    run(items)
    sch.finish_step(3.1, items)
    assert 0 not in ctx.ora.reqs                             # r0 finished and released
    items = sch.step(3.2)
    assert items == [(1, 112, 288), (2, 0, 224)]
    run(items)
    sch.finish_step(3.3, items)
    # a new high-priority request (older arrival cannot exist; FCFS complete tier) -> pressure:
    # fill the pool with r3 (complete) while r2 is partial-but-running and holds blocks
    sch.on_chunk(0.5, 3, 1, tokens=np.arange(16 * 60))      # arrival 0.5: ranks before r2
    sch.budget = 1024
    items = sch.step(3.4)
    # r3 needs 60 blocks; r2 (lower priority, holds 14 blocks) is the victim -> swapped
    assert items[0][0] == 3
    assert any(e[1] == "PREEMPTED_SWAP" and e[2] == 2 for e in sch.events)
    assert ctx.query(2)["tier"] == S.TIER_CPU


def test_cost_based_choice_follows_model():
    cm = _cm(crossover_tokens=4096)
    assert cm.choose_eviction(1000) == "recompute" and cm.choose_eviction(20000) == "swap"
    ng = 1100
    ctx = _ctx(ng, 4096)
    sch = S.StreamingScheduler(ctx, "LCAS", 16, 1 << 20, ng, cost_model=cm, preemption="cost")
    run = _exec(ctx)
    sch.on_chunk(0.0, 0, 2, tokens=np.arange(1000))          # small, partial
    sch.on_chunk(0.1, 1, 2, tokens=np.arange(12000))         # large, partial
    items = sch.step(0.2)
    run(items)
    sch.finish_step(0.3, items)
    # a complete request needing almost the whole pool arrives: both partials are victims
    sch.on_chunk(1.0, 2, 1, tokens=np.arange(16 * 1090))
    items = sch.step(1.1)
    assert items and items[0][0] == 2
    kinds = {e[2]: e[1] for e in sch.events if e[1].startswith("PREEMPTED")}
    assert kinds == {0: "PREEMPTED_RECOMPUTE", 1: "PREEMPTED_SWAP"}
    assert ctx.query(0)["num_computed"] == 0 and ctx.query(1)["tier"] == S.TIER_CPU


def test_update_chunk_invalidates_beyond_lcp():
    ctx = _ctx(256, 64)
    sch = S.StreamingScheduler(ctx, "LCAS", 16, 1 << 20, 256, preemption="recompute")
    run = _exec(ctx)
    old = np.arange(1000, dtype=np.int32)
    sch.on_chunk(0.0, 7, 2, new_input=old, mode="update")
    items = sch.step(0.1)
    assert items == [(7, 0, 1000)]
    run(items)
    sch.finish_step(0.2, items)
    new = old.copy()
    new[300:] += 5
    sch.on_chunk(0.3, 7, 2, new_input=new, mode="update")   # LCP 300
    assert sch.reqs[7].tokens_invalidated == 700
    items = sch.step(0.4)
    assert items == [(7, 300, 700)]                          # recompute from the LCP
    run(items)
    sch.finish_step(0.5, items)
    assert sch.reqs[7].finish == 0.5 and abs(sch.reqs[7].ttft - 0.2) < 1e-12


def _simulate(trace, policy, streaming, ng, nc, budget=2048, preemption="cost", tok_s=1e-5):
    ctx = _ctx(ng, nc, max_req=len({e[1] for e in trace}) + 1)
    sch = S.StreamingScheduler(ctx, policy, 16, budget, ng, cost_model=_cm(), preemption=preemption,
                               streaming=streaming)
    run = _exec(ctx)
    t, i = 0.0, 0
    while True:
        while i < len(trace) and trace[i][0] <= t:
            tc, rid, n, tok, new, mode = trace[i]
            sch.on_chunk(tc, rid, n, tokens=tok, new_input=new, mode=mode)
            i += 1
        items = sch.step(t)
        if not items:
            if i >= len(trace):
                break
            t = trace[i][0]
            continue
        run(items)
        t += 1e-3 + tok_s * sum(n for _, _, n in items)       # modelled step time
        sch.finish_step(t, items)
    return sch, ctx


@pytest.mark.parametrize("policy", S.POLICIES)
def test_crawler_trace_completes_under_pressure(policy):
    tr = traces.crawler_trace(5, 24, qps=4.0, hi=8192)
    sch, ctx = _simulate(tr, policy, True, ng=900, nc=4096)
    tt = sch.ttfts()
    assert len(tt) == 24 and all(v >= 0 for v in tt.values())
    assert ctx.lib.free_blocks() == (900, 4096)              # everything released


def test_anns_trace_updates_and_streaming_beats_non_streaming():
    tr = traces.anns_trace(9, 24, qps=2.0, hi=8192)
    assert any(e[3] is None and e[4] is not None for e in tr)
    s_str, _ = _simulate(tr, "FCFS", True, ng=4096, nc=1024)
    s_ns, _ = _simulate(tr, "DEFAULT", False, ng=4096, nc=1024)
    a = np.median(list(s_str.ttfts().values()))
    b = np.median(list(s_ns.ttfts().values()))
    assert len(s_str.ttfts()) == len(s_ns.ttfts()) == 24
    assert a <= b                                            # prefill overlaps retrieval
    assert sum(r.tokens_invalidated for r in s_str.reqs.values()) > 0


def test_trace_marginals():
    cr = traces.crawler_trace(1, 400, qps=1.0)
    per = {}
    for e in cr:
        per.setdefault(e[1], []).append(e)
    assert all(6 <= len(v) <= 10 for v in per.values())
    gaps = np.concatenate([np.diff([e[0] for e in v]) for v in per.values()])
    assert 0.4 < np.median(gaps) < 1.2                        # ~700.7 ms median (Fig. 6)
    an = traces.anns_trace(1, 400, qps=1.0)
    cnt = {}
    for e in an:
        cnt[e[1]] = cnt.get(e[1], 0) + 1
    assert np.mean([c <= 3 for c in cnt.values()]) > 0.5     # majority 1-3 chunks (Fig. 7)
    tot = [len(e[4]) for e in an if e[4] is not None]
    assert 7000 < np.median(tot) < 13000                      # median ~10K (Table 2)


def test_spec_free_block_feasibility_example():
    """S:L325 / S:L330 (feasibility="free"): projected free blocks start at the pool's free
    count; a request needing 10 blocks with 9 projected free goes to not_scheduled, a later
    one needing 9 is still a candidate.  Under the default Z18 reading ("pool") both are
    selected and Phase 2 preempts the idle holder to place the first."""
    for rule in ("free", "pool"):
        ng = 20
        ctx = _ctx(ng, 64)
        sch = S.StreamingScheduler(ctx, "FCFS", 16, 1 << 20, ng, preemption="swap", feasibility=rule)
        run = _exec(ctx)
        sch.on_chunk(0.0, 0, 2, tokens=np.arange(16 * 11))   # holder: 11 blocks, then waits for input
        items = sch.step(0.1)
        run(items)
        sch.finish_step(0.1, items)
        assert ctx.free_blocks()[0] == 9
        sch.on_chunk(0.2, 1, 1, tokens=np.arange(16 * 10))   # needs 10 (complete, earlier)
        sch.on_chunk(0.3, 2, 1, tokens=np.arange(16 * 9))    # needs 9
        items = sch.step(0.4)
        if rule == "free":
            assert [r for r, _, _ in items] == [2]
            assert not any(e[1].startswith("PREEMPTED") for e in sch.events)
        else:
            assert [r for r, _, _ in items][0] == 1
            assert any(e[1] == "PREEMPTED_SWAP" and e[2] == 0 for e in sch.events)


def test_default_lifo_eviction_over_running_order():
    """DEFAULT with default_lifo (§4.4.1): the victim is the LAST request of the running
    order holding GPU blocks, not the lowest-priority entry of not_scheduled."""
    ng = 40
    ctx = _ctx(ng, 256)
    sch = S.StreamingScheduler(ctx, "DEFAULT", 16, 1 << 20, ng, preemption="swap", default_lifo=True)
    run = _exec(ctx)
    sch.on_chunk(0.0, 0, 2, tokens=np.arange(16 * 12))
    sch.on_chunk(0.1, 1, 2, tokens=np.arange(16 * 12))
    items = sch.step(0.2)
    run(items)
    sch.finish_step(0.2, items)
    assert sch.running == [0, 1]
    sch.on_chunk(0.3, 0, 2, tokens=np.arange(16 * 14))      # r0 grows: needs 14 more, 16 free
    sch.on_chunk(0.4, 2, 1, tokens=np.arange(16 * 10))      # a new request behind it
    items = sch.step(0.5)
    pre = [e[2] for e in sch.events if e[1] == "PREEMPTED_SWAP"]
    assert pre and pre[0] == 1                                # last of the running order
    assert 0 in [r for r, _, _ in items]


@pytest.mark.parametrize("policy", ["DEFAULT", "FCFS"])
def test_trace_under_spec_rules_completes(policy):
    tr = traces.crawler_trace(6, 24, qps=4.0, hi=8192)
    ctx = _ctx(900, 4096, max_req=25)
    sch = S.StreamingScheduler(ctx, policy, 16, 2048, 900, cost_model=_cm(), preemption="cost",
                               feasibility="free", default_lifo=True)
    run = _exec(ctx)
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
        run(items)
        t += 1e-3 + 1e-5 * sum(n for _, _, n in items)
        sch.finish_step(t, items)
    assert len(sch.ttfts()) == 24
    assert ctx.lib.free_blocks() == (900, 4096)
