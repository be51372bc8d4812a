"""C4 memory-pressure mix (BJ:L10): a deterministic round-robin driver
that streams append-mode and update-mode requests through one libs2l context whose GPU pool
is smaller than the working set, swapping requests out to pinned host memory and back in
("Transfer all blocks ... from GPU to CPU memory ... swap blocks back to GPU with
symmetric cost") to make room for each step.

This is a harness driver, not the paper's scheduler (two-phase scheduling and the
recompute-vs-swap policy are P:L134-L237): requests are stepped in
round-robin order under a token budget (2048-8192 tokens per batch), and the victims
of a swap-out are the GPU-resident requests whose next round-robin turn is furthest away.  All state it plans with
comes from the library's own queries (`query`, `free_blocks`), so the same driver runs on a
device context (bench) and on a host-only context (CPU tests, where `tests/` replays its op
log through the oracle).

Overlap (SURVEY NEXT-2, P:L184 resume): the swaps that prepare step s+1 are issued on the copy
stream right after step s's compute has been enqueued, so they run while step s computes;
the library orders them only against the kernels they actually conflict with.

Workload recipe: request r is append-mode if r is even, update-mode if odd.
  * append: total T ~ LogNormal(ln 5800, 0.976) (crawler trace, Tab. 2 median 5.8K)
    truncated to [lo, hi]; U{6..10} chunks of near-equal size, tokens arrive with
    each chunk;
  * update: T ~ LogNormal(ln 10000, 0.688) (ANNS trace) truncated to [lo, hi]; the
    input arrives whole and is prefilled as two chunks, then U{1, 2} update rounds, each an
    LCP p ~ U[ceil(0.2 T), floor(0.8 T)] (reading Z14) with new length T, recomputing T - p
    tokens (split into budget-sized pieces, budget-clamped partial chunks).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

TIER_GPU, TIER_CPU = 0, 1


@dataclass
class Work:
    """One step's work for one request: optional update (new input -> invalidate_lcp first),
    optional appended tokens, then K/V + attention for the next n_kv pending positions."""
    n_kv: int
    append_tokens: np.ndarray | None = None
    new_input: np.ndarray | None = None


@dataclass
class Plan:
    rid: int
    mode: str
    total: int
    initial_tokens: np.ndarray
    work: list = field(default_factory=list)


def _lognormal_len(rng, median, sigma, lo, hi):
    return int(min(hi, max(lo, round(math.exp(math.log(median) + sigma * rng.standard_normal())))))


def c4_plans(seed: int, n_requests: int, lo: int = 1024, hi: int = 16384, budget: int = 8192,
             rids=None) -> list:
    """Per-request work lists (token ids from synth; lengths / chunking / LCP draws here)."""
    from synth import workloads as W
    rng = np.random.default_rng(seed)
    plans = []
    for r in range(n_requests):
        mode = "append" if r % 2 == 0 else "update"
        if mode == "append":
            T = _lognormal_len(rng, 5800, 0.976, lo, hi)
            n_chunks = int(rng.integers(6, 11))
        else:
            T = _lognormal_len(rng, 10000, 0.688, lo, hi)
            rounds = int(rng.integers(1, 3))
            ps = [int(rng.integers(-(-2 * T // 10), (8 * T) // 10 + 1)) for _ in range(rounds)]
        if rids is not None and r not in rids:
            continue
        toks = W.request_tokens(seed, r, T)
        if mode == "append":
            bounds = [T * i // n_chunks for i in range(n_chunks + 1)]
            work = [Work(n_kv=b - a, append_tokens=toks[a:b]) for a, b in zip(bounds, bounds[1:])]
            plans.append(Plan(r, mode, T, toks[:0], work))
        else:
            work = [Work(n_kv=T // 2), Work(n_kv=T - T // 2)]
            cur = toks
            for i, p in enumerate(ps):
                new = W.updated_tokens(seed, r, cur, p, T, i)
                n = T - p
                first = True
                while n > 0:
                    m = min(n, budget)
                    work.append(Work(n_kv=m, new_input=new if first else None))
                    first = False
                    n -= m
                cur = new
            plans.append(Plan(r, mode, T, toks, work))
    return plans


def working_set_blocks(plans, k: int) -> int:
    return sum(-(-p.total // k) for p in plans)


class PressureDriver:
    """Round-robin stepping + furthest-next-use swap residency over one context.

    Loop (see `run`): sel = plan(); prepare(sel); while sel: items(sel) -> caller enqueues
    append + attention; finish(sel); nxt = plan(); prepare(nxt, protect=sel); sel = nxt.
    Every library call is appended to `log` as (op, args, result) for the oracle replay.
    """

    def __init__(self, ctx, plans, k: int, budget: int, evict_ahead: int = 2, cost=None,
                 prefetch_ahead: int = 0, reserve: int = 0):
        """cost: None -> every victim is swapped (the C4 definition, BJ:L10); else a callable
        cost(num_computed, num_blocks) -> "recompute" | "swap" (the paper's cost-based
        preemption, P:L79 / §4.3): a recompute victim drops its blocks (no D2H) and later
        re-prefills its computed prefix."""
        self.ctx, self.k, self.budget = ctx, k, budget
        self.evict_ahead = evict_ahead
        # prefetch_ahead: also swap in the CPU-tier requests of the next `prefetch_ahead` steps
        # after sel when the room is already there, so their H2D gets several steps of compute
        self.prefetch_ahead = prefetch_ahead
        # reserve: free GPU blocks kept beyond the look-ahead's needs (best effort), so that with
        # the cooling allocation order a step's swap-ins and appends take blocks freed earlier
        # rather than blocks the previous step's kernels or swap-outs may still be using
        self.reserve = reserve
        self.prefetched = 0
        self.cost = cost
        self.recompute_preemptions = 0
        self.recomputed_tokens = 0
        self.plans = {p.rid: p for p in plans}
        self.work = {p.rid: list(p.work) for p in plans}      # own copy: recompute inserts items
        self.next_work = {p.rid: 0 for p in plans}
        self.last_step = {p.rid: -1 for p in plans}
        self.order = sorted(self.plans)
        self.cursor = 0
        self.step = 0
        self.log = []
        self.swapped_out_bytes = 0
        self.swapped_in_bytes = 0
        self.swap_out_calls = 0
        self.swap_in_calls = 0
        self.tokens = 0
        self.deferred = []
        for p in plans:
            ctx.new_request(p.rid, p.initial_tokens)
            self.log.append(("new", (p.rid, p.initial_tokens), 0))

    # ---- planning ------------------------------------------------------------------------
    def live(self):
        return [r for r in self.order if r in self.plans and self.next_work[r] < len(self.work[r])]

    def plan(self, peek: bool = False):
        """Next step's requests: round-robin from the cursor, one work item each, until the
        token budget is reached (the first request is always taken).  peek: do not advance."""
        live = self.live()
        if not live:
            return []
        start = 0
        while start < len(live) and live[start] < self.cursor:
            start += 1
        rot = live[start:] + live[:start]
        sel, used = [], 0
        for r in rot:
            n = self.work[r][self.next_work[r]].n_kv
            if sel and used + n > self.budget:
                break
            sel.append(r)
            used += n
        if not peek:
            self.cursor = sel[-1] + 1
        return sel

    def _blocks(self, n):
        return -(-n // self.k)

    def _need(self, sel, info):
        """GPU blocks the step's requests still need: swap-ins + blocks their appends take."""
        need = 0
        for r in sel:
            q = info[r]
            w = self.work[r][self.next_work[r]]
            need += max(0, self._blocks(q["num_computed"] + w.n_kv) - q["num_blocks"])
            if q["tier"] == TIER_CPU:
                need += q["num_blocks"]
        return need

    def _pick(self, need, free_gpu, keep, avoid):
        """GPU requests outside `keep` (preferring those outside `avoid`) to swap out so that
        free_gpu >= need, those whose next round-robin turn is furthest away first (Belady's
        choice: the round-robin order is the future access order; LRU would evict exactly the
        requests due next).  Returns (victims, free_gpu after them); None if impossible."""
        if free_gpu >= need:
            return [], free_gpu
        live = self.live()
        pos = {r: i for i, r in enumerate(live)}
        start = 0
        while start < len(live) and live[start] < self.cursor:
            start += 1
        cands = []
        for r in self.order:
            if r in keep or r not in self.plans:
                continue
            q = self.ctx.query(r)
            if q["tier"] == TIER_GPU and q["num_blocks"] > 0:
                dist = (pos[r] - start) % len(live) if r in pos else len(live)
                cands.append((r in avoid, -dist, r, q["num_blocks"]))
        cands.sort()
        victims = []
        for _, _, r, nb in cands:
            if free_gpu >= need:
                break
            victims.append(r)
            free_gpu += nb
        return (victims, free_gpu) if free_gpu >= need else None

    def prepare(self, sel, protect=()):
        """Updates first (LCP invalidation on either tier), then make room: swap
        out GPU requests outside sel (and, if possible, outside `protect` = the step still
        computing) and swap in the members of sel on the CPU tier.  With evict_ahead the same
        swap-out call also makes room for the step after sel: its D2H then runs while this
        step and the next compute, and (with the opt-in s2l_config.alloc_cooling) the ids it
        releases are allocated only after every other free id, so the next step's appends and
        swap-ins avoid them."""
        for r in sel:
            w = self.work[r][self.next_work[r]]
            if w.new_input is not None:
                res = self.ctx.invalidate_lcp(r, w.new_input)
                self.log.append(("invalidate", (r, w.new_input), res))
        info = {r: self.ctx.query(r) for r in sel}
        need = self._need(sel, info)
        to_in = [r for r in sel if info[r]["tier"] == TIER_CPU]
        free_gpu, _ = self.ctx.free_blocks()
        got = self._pick(need, free_gpu, set(sel), set(protect))
        if got is None:
            raise RuntimeError(f"step {self.step}: cannot make room for {need} blocks")
        victims, free_after = got
        if self.evict_ahead:
            # room for the next `evict_ahead` steps too (best effort), so that a large D2H starts
            # while earlier steps compute instead of right before the step that needs the room
            keep, want = set(sel) | set(victims), need
            saved = self.cursor
            for _ in range(int(self.evict_ahead)):
                nxt = [r for r in self.plan(peek=True) if r not in keep]
                if not nxt:
                    break
                self.cursor = nxt[-1] + 1                  # peek one step further
                info2 = {r: self.ctx.query(r) for r in nxt}
                want += self._need(nxt, info2)
                keep |= set(nxt)
            self.cursor = saved
            more = self._pick(want + self.reserve, free_after, keep, set(protect))
            if more is None and self.reserve:
                more = self._pick(want, free_after, keep, set(protect))
            if more is not None:
                victims += more[0]
        if victims and self.cost is not None:
            swap_v = []
            for r in victims:
                q = self.ctx.query(r)
                if self.cost(q["num_computed"], q["num_blocks"]) == "recompute":
                    self._preempt_recompute(r, q["num_computed"])
                else:
                    swap_v.append(r)
            victims = swap_v
        if victims:
            b = self.ctx.swap_out(victims)
            self.log.append(("swap_out", tuple(victims), b))
            self.swapped_out_bytes += b
            self.swap_out_calls += 1
        if self.prefetch_ahead and victims is not None:
            free_now, _ = self.ctx.free_blocks()
            spare = free_now - need                      # sel's swap-ins and appends come first
            seen, saved = set(sel), self.cursor
            for _ in range(int(self.prefetch_ahead)):
                nxt = [r for r in self.plan(peek=True) if r not in seen]
                if not nxt:
                    break
                self.cursor = nxt[-1] + 1
                for r in nxt:
                    q = self.ctx.query(r)
                    upd = self.work[r][self.next_work[r]].new_input is not None   # would drop blocks
                    if q["tier"] == TIER_CPU and not upd and 0 < q["num_blocks"] <= spare:
                        to_in.append(r)
                        spare -= q["num_blocks"]
                        self.prefetched += 1
                seen |= set(nxt)
            self.cursor = saved
        if to_in:
            b = self.ctx.swap_in(to_in)
            self.log.append(("swap_in", tuple(to_in), b))
            self.swapped_in_bytes += b
            self.swap_in_calls += 1

    def _preempt_recompute(self, r, nc):
        """Recompute preemption: free the blocks now; the computed prefix [0, nc) of
        the current input is prefilled again, in budget-sized pieces, before its next work."""
        self.ctx.preempt_recompute(r)
        self.log.append(("preempt", (r,), 0))
        self.recompute_preemptions += 1
        self.recomputed_tokens += nc
        pieces, left = [], nc
        while left > 0:
            m = min(left, self.budget)
            pieces.append(Work(n_kv=m))
            left -= m
        i = self.next_work[r]
        self.work[r][i:i] = pieces

    def items(self, sel):
        """(append items, prefill items, n rows): rows of the step are packed in sel order."""
        app, pre, row = [], [], 0
        for r in sel:
            w = self.work[r][self.next_work[r]]
            nc = self.ctx.query(r)["num_computed"]
            app.append((r, w.append_tokens, w.n_kv, row))
            pre.append((r, nc, w.n_kv, row))
            row += w.n_kv
        self.log.append(("append", tuple((r, t, n) for r, t, n, _ in app), 0))
        self.log.append(("prefill", tuple((r, p, n) for r, p, n, _ in pre), 0))
        self.tokens += row
        return app, pre, row

    def finish(self, sel):
        """Advance each request; a request with no work left is finished.  Its release is
        deferred by one step: its blocks are still read by this step's attention, so a swap-in
        preparing the next step must not land in them (the library would order that H2D after
        this step's compute and the swap would no longer overlap it)."""
        self._release_deferred()
        for r in sel:
            self.next_work[r] += 1
            self.last_step[r] = self.step
            if self.next_work[r] == len(self.work[r]):
                self.deferred.append(r)
                del self.plans[r]
        self.step += 1

    def _release_deferred(self):
        for r in self.deferred:
            self.ctx.release(r)
            self.log.append(("release", (r,), 0))
        self.deferred = []

    def run(self, execute):
        """Drives the whole stream; execute(sel, app_items, prefill_items, rows) enqueues the
        step's append + attention.  Returns the number of steps."""
        sel = self.plan()
        self.prepare(sel)
        while sel:
            app, pre, rows = self.items(sel)
            execute(sel, app, pre, rows)
            self.finish(sel)
            nxt = self.plan()
            if nxt:
                self.prepare(nxt, protect=sel)
            sel = nxt
        self._release_deferred()
        return self.step


class SwapTimer:
    """Context wrapper around the swap calls.  `serial=True` drains all streams before and
    after every swap (the no-overlap baseline); `copy_stream` / `swap_in_stream` (the
    context's swap-out / swap-in streams) enable per-call CUDA events, read back with
    `copy_ms()` after synchronisation."""

    def __init__(self, ctx, serial: bool = False, copy_stream=None, swap_in_stream=None):
        self.ctx, self.serial = ctx, serial
        self.streams = {"out": copy_stream, "in": swap_in_stream}
        self.events = []

    def __getattr__(self, name):
        return getattr(self.ctx, name)

    def _swap(self, fn, rids, kind):
        if self.serial:
            self.ctx.sync()
        ev, cs = None, self.streams[kind]
        if cs is not None:
            import torch
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record(cs)
        b = fn(rids)
        if ev is not None:
            ev[1].record(cs)
            self.events.append((kind, b, ev))
        if self.serial:
            self.ctx.sync()
        return b

    def swap_out(self, rids):
        return self._swap(self.ctx.swap_out, rids, "out")

    def swap_in(self, rids):
        return self._swap(self.ctx.swap_in, rids, "in")

    def copy_ms(self):
        """{kind: (bytes, ms)} summed over calls (each interval spans the copy-stream time
        from the call's start to its end, including waits for the compute work it depends on)."""
        out = {}
        for kind, b, (e0, e1) in self.events:
            tb, tm = out.get(kind, (0, 0.0))
            out[kind] = (tb + b, tm + e0.elapsed_time(e1))
        return out


def device_executor(ctx, src_q, src_k, src_v, out, layers: int, on_step=None):
    """execute() for PressureDriver.run on a device context: one append_chunk of the step's
    K/V rows (taken from the source buffers at the step's packed rows) and one prefill_batch
    per layer.  `on_step(sel, app, pre, rows)` runs after the launches (e.g. snapshots)."""
    kv_rows = src_k.shape[1]

    def execute(sel, app, pre, rows):
        ctx.append_chunk(app, src_k, src_v, kv_rows=kv_rows)
        for layer in range(layers):
            ctx.prefill_batch(layer, pre, src_q, out)
        if on_step is not None:
            on_step(sel, app, pre, rows)

    return execute
