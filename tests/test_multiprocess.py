"""World-size-2 CPU tests (gloo) of the multi-GPU host logic: request / KV-head sharding,
max-over-ranks time, gather of sampled output rows; and that KV-head sharding reproduces the
unsharded oracle output exactly (GQA groups are independent)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_16395_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # max over ranks
        t = shard.max_time(dist, 10.0 + rank)
        # gather sampled rows
        rows = torch.full((3, 4), float(rank))
        got = shard.gather_rows(dist, rows, world)
        # request sharding is identical on every rank
        lengths = {r: 1024 * (r % 5 + 1) for r in range(16)}
        asg = shard.assign_requests(lengths, world)
        q.put((rank, t, [g[0, 0].item() for g in got], asg))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_plumbing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(t == 11.0 for _, t, _, _ in res)
    assert all(g == [0.0, 1.0] for _, _, g, _ in res)
    assert res[0][3] == res[1][3]
    ids = sorted(res[0][3][0] + res[0][3][1])
    assert ids == list(range(16))


def test_lpt_balance():
    lengths = {r: 512 * (r + 1) for r in range(8)}
    asg = shard.assign_requests(lengths, 4)
    f = {r: shard.request_flops(lengths[r], 512, 32, 128) for r in lengths}
    loads = [sum(f[r] for r in a) for a in asg]
    # Graham's LPT bound: makespan <= 4/3 OPT, and OPT >= max(total/4, largest job)
    opt_lb = max(sum(f.values()) / 4, max(f.values()))
    assert max(loads) <= 4 / 3 * opt_lb
    assert sorted(sum(asg, [])) == list(range(8))


def test_kv_head_shard_reproduces_unsharded_oracle():
    """C5-style sharding: per-rank attention on its kv heads == the matching slice of the
    unsharded attention (the oracle, fp64)."""
    import synth
    from oracle.attention import attention
    rng = np.random.default_rng(0)
    n, p0, h_q, h_kv, d = 6, 10, 8, 4, 16
    q = synth.f64_to_bf16_bits(rng.standard_normal((n, h_q, d)))
    k = synth.f64_to_bf16_bits(rng.standard_normal((p0 + n, h_kv, d)))
    v = synth.f64_to_bf16_bits(rng.standard_normal((p0 + n, h_kv, d)))
    full, _ = attention(q, k, v, p0)
    for world in (1, 2, 4):
        parts = []
        for rank in range(world):
            kv, qh = shard.kv_head_shard(rank, world, h_q, h_kv)
            o, _ = attention(q[:, qh], k[:, kv], v[:, kv], p0)
            parts.append(o)
        assert np.array_equal(np.concatenate(parts, axis=1), full)
    with pytest.raises(ValueError):
        shard.kv_head_shard(0, 3, h_q, h_kv)


def _c4_worker(rank, world, port, q):
    """One rank of the request-sharded C4 mix: its requests (rid % world == rank) through the
    pressure driver on a host-only libs2l context, every library call mirrored into the oracle
    (tests.harness.Twin asserts bit-exact agreement); results gathered over gloo."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_16395_b200 import pressure, s2l
        from tests.harness import Twin
        k, budget = 16, 512
        plans = [p for p in pressure.c4_plans(21, 24, lo=64, hi=1024, budget=budget) if p.rid % world == rank]
        ws = pressure.working_set_blocks(plans, k)
        biggest = max(-(-p.total // k) for p in plans)
        ng = max(ws // 2, 3 * biggest + budget // k + 2)
        nc = ws + 8
        cfg = s2l.make_config(1, 1, 1, 8, k, ng, nc, max_requests=len(plans), max_blocks_per_request=biggest + 1,
                              alloc_cooling=1)
        lib = s2l.Context(cfg, host_only=True)
        tw = Twin(lib, k, ng, nc, len(plans), biggest + 1)
        drv = pressure.PressureDriver(tw, plans, k, budget)

        def execute(sel, app, pre, rows):
            assert all(r % world == rank for r in sel)      # a rank only touches its own shard
            tw.append_chunk(app, None, None, kv_rows=rows)

        steps = drv.run(execute)
        stats = torch.tensor([float(drv.tokens), float(drv.swapped_out_bytes), float(steps)])
        parts = [torch.zeros(3) for _ in range(world)]
        dist.all_gather(parts, stats)
        done = torch.zeros(24)
        for p in plans:
            done[p.rid] = 1.0
        dist.all_reduce(done)
        q.put((rank, [x.tolist() for x in parts], done.tolist(), ng < ws, tw.ops))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_c4_request_sharding_on_the_library():
    """C4 sharded by request across 2 ranks (BJ:L10) with the library's host-only
    contexts: each rank's shard is under memory pressure, every call agrees with the oracle, the
    shards partition the 24 requests and the gathered token totals equal the workload's."""
    from paper_2604_16395_b200 import pressure
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c4_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    plans = pressure.c4_plans(21, 24, lo=64, hi=1024, budget=512)
    want_tokens = sum(w.n_kv for p in plans for w in p.work)
    for rank, parts, done, pressured, ops in res:
        assert pressured and ops > 0
        assert done == [1.0] * 24                         # every request on exactly one rank
        assert sum(x[0] for x in parts) == want_tokens
        assert sum(x[1] for x in parts) > 0               # swaps happened on the shards
    assert res[0][1] == res[1][1]                         # both ranks gathered the same stats
