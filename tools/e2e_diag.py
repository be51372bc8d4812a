"""Diagnoses bench.py's e2e leg: per-chunk CUDA-event timeline of the H2D copies (Q/K/V),
the library's append + attention, and the D2H of O for one C2 step, plus copy-only
references (H2D alone, D2H alone, both directions concurrently) for the same byte counts."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    torch.cuda.set_device(0)
    rids, toks, data = bench.make_stream_data(0)
    S_host = bench.Stream(rids, toks, data, "cuda:0", pinned=True)
    S_dev = bench.Stream(rids, toks, data, "cuda:0")
    ctx, pool = bench.make_ctx(0)
    nb = bench.E2E_BUFS
    dev_bufs = tuple([torch.empty_like(S_dev.q[0] if i in (0, 3) else S_dev.k[0]) for _ in range(nb)] for i in range(4))
    streams = (torch.cuda.Stream(), torch.cuda.Stream())
    for _ in range(2):
        bench.e2e_run(ctx, S_host, dev_bufs, streams)
    torch.cuda.synchronize()
    s, e = ev(), ev()
    s.record()
    bench.e2e_run(ctx, S_host, dev_bufs, streams)
    e.record()
    torch.cuda.synchronize()
    print(f"e2e step: {s.elapsed_time(e):.2f} ms")
    # per-chunk timeline of one e2e step (events on each stream)
    import types
    comp = torch.cuda.current_stream()
    h2d, d2h = streams
    qd, kd, vd, od = dev_bufs
    T = {k: [] for k in ("h0", "h1", "c0", "ca", "c1", "d0", "d1")}
    for r, t in zip(S_host.rids, S_host.toks):
        ctx.new_request(r, t)
    ev_loaded = [torch.cuda.Event() for _ in range(nb)]
    ev_done = [torch.cuda.Event() for _ in range(nb)]
    ev_free = [None] * nb
    torch.cuda.synchronize()
    t0 = ev()
    t0.record()
    for j in range(S_host.steps):
        b = j % nb
        with torch.cuda.stream(h2d):
            if ev_free[b] is not None:
                h2d.wait_event(ev_free[b])
            x = ev(); x.record(h2d); T["h0"].append(x)
            qd[b].copy_(S_host.q[j], non_blocking=True)
            kd[b].copy_(S_host.k[j], non_blocking=True)
            vd[b].copy_(S_host.v[j], non_blocking=True)
            x = ev(); x.record(h2d); T["h1"].append(x)
            ev_loaded[b].record(h2d)
        comp.wait_event(ev_loaded[b])
        x = ev(); x.record(comp); T["c0"].append(x)
        ctx.append_chunk(S_host.items_a[j], kd[b], vd[b])
        x = ev(); x.record(comp); T["ca"].append(x)
        ctx.prefill_batch(0, S_host.items_p[j], qd[b], od[b])
        x = ev(); x.record(comp); T["c1"].append(x)
        ev_done[b].record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(ev_done[b])
            x = ev(); x.record(d2h); T["d0"].append(x)
            S_host.o[j].copy_(od[b], non_blocking=True)
            x = ev(); x.record(d2h); T["d1"].append(x)
            fe = torch.cuda.Event()
            fe.record(d2h)
            ev_free[b] = fe
    comp.wait_stream(d2h)
    torch.cuda.synchronize()
    for r in S_host.rids:
        ctx.release(r)
    print("chunk  h2d[start,end]   compute[start,append end,end]   d2h[start,end]  (ms)")
    for j in list(range(0, 8)) + list(range(28, 32)):
        f = lambda k: t0.elapsed_time(T[k][j])
        print(f"{j:3d}  {f('h0'):7.2f} {f('h1'):7.2f}   {f('c0'):7.2f} {f('ca'):7.2f} {f('c1'):7.2f}   {f('d0'):7.2f} {f('d1'):7.2f}")
    h2d, d2h = streams
    qd, kd, vd, od = dev_bufs
    for name, do_h2d, do_d2h in (("h2d only", True, False), ("d2h only", False, True), ("both", True, True)):
        torch.cuda.synchronize()
        s, e = ev(), ev()
        s.record()
        for j in range(S_host.steps):
            b = j % nb
            if do_h2d:
                with torch.cuda.stream(h2d):
                    qd[b].copy_(S_host.q[j], non_blocking=True)
                    kd[b].copy_(S_host.k[j], non_blocking=True)
                    vd[b].copy_(S_host.v[j], non_blocking=True)
            if do_d2h:
                with torch.cuda.stream(d2h):
                    S_host.o[j].copy_(od[b], non_blocking=True)
        for st in streams:
            x = torch.cuda.Event()
            x.record(st)
            torch.cuda.current_stream().wait_event(x)
        e.record()
        torch.cuda.synchronize()
        print(f"{name:10s}: {s.elapsed_time(e):.2f} ms")
    # compute only (device-resident inputs)
    torch.cuda.synchronize()
    s, e = ev(), ev()
    s.record()
    bench.run_step(ctx, S_dev)
    e.record()
    torch.cuda.synchronize()
    print(f"compute only: {s.elapsed_time(e):.2f} ms")


if __name__ == "__main__":
    main()
