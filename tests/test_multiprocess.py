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
