"""STREAM2LLM's two-phase streaming scheduler driving libs2l.

Host side, like the paper's (a vLLM scheduler extension).  One `step()`:

  Phase 1 — priority ordering and feasibility: the policy (§4.4) ranks every
  unfinished request that has pending tokens; walking that order, each request gets
  min(pending, budget left) tokens (budget-clamped partial chunks) if its block estimate fits.
  What "sufficient free GPU blocks remain" counts is a reading (`feasibility=`):
    "pool" (Z18, default): blocks that are free or held by requests Phase 2 may preempt, i.e.
           the selected requests' total demand must fit the pool;
    "free" (the SPEC's rule): projected free blocks start at the pool's free
           count and each candidate's NEW blocks (+ its CPU blocks if it needs a swap-in) are
           taken from them; preemption opportunities are left to Phase 2.  When nothing fits
           (every block held by requests that all need more -- a deadlock under this rule
           alone) the highest-priority request that fits the pool goes to Phase 2.
  Requests that do not fit, or that the token budget leaves out, go to `not_scheduled` in
  priority order.  No state changes.
  Phase 2 — resource acquisition with adaptive preemption: for each selected request
  in priority order, while the GPU pool is short, preempt the lowest-priority request of
  `not_scheduled` that still holds GPU blocks, choosing recomputation or swapping with the
  cost model (§4.3; `costmodel.CostModel.choose_eviction`) or a forced strategy
  (the paper's ablation, Table 3); then swap the request in if it is on the CPU tier.  A
  request that still cannot be placed is skipped this step.

Streaming inputs (§4.2): an append-mode chunk extends the request's input (s2l_append_chunk
with tokens and no K/V); an update-mode chunk replaces it (s2l_invalidate_lcp: LCP
invalidation, also on the CPU tier).  Non-streaming (vLLM-NS) requests become
visible only when their whole input has arrived.

Policies (§4.4; eviction is reverse priority among `not_scheduled` -- except DEFAULT with
`default_lifo=True` (§4.4.1 "LIFO eviction"): the last request of the running order
that holds GPU blocks and is not being placed this step):
  DEFAULT  vLLM: running requests in their execution order, then waiting requests FIFO by
           arrival with preempted ones re-queued at the front;
  FCFS     two tiers, complete inputs first, each by arrival time;
  MCPS     num_computed_tokens descending, ties by arrival;
  LCAS     two tiers, complete first, each by last chunk arrival, most recent first.

TTFT (reading Z17): the first token follows the prefill of the complete input, so a request
finishes when its input is complete and fully computed; TTFT = finish time - arrival of its
last chunk (the moment a non-streaming system receives the request; Table 3).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

TIER_GPU, TIER_CPU = 0, 1
POLICIES = ("DEFAULT", "FCFS", "MCPS", "LCAS")


@dataclass
class SReq:
    rid: int
    arrival: float                 # first chunk (query) arrival
    n_chunks: int                  # chunks expected
    mode: str = "append"           # "append" | "update"
    chunks_arrived: int = 0
    last_chunk_arrival: float = 0.0
    status: str = "waiting"        # waiting | running | finished
    preempted_front: bool = False  # DEFAULT: re-queued at the front of waiting
    finish: float | None = None
    preemptions_recompute: int = 0
    preemptions_swap: int = 0
    tokens_invalidated: int = 0

    @property
    def complete(self) -> bool:
        return self.chunks_arrived >= self.n_chunks

    @property
    def ttft(self):
        return None if self.finish is None else self.finish - self.last_chunk_arrival


class StreamingScheduler:
    def __init__(self, ctx, policy: str, block_size: int, budget: int, num_gpu_blocks: int,
                 cost_model=None, preemption: str = "cost", streaming: bool = True,
                 feasibility: str = "pool", default_lifo: bool = False):
        if policy not in POLICIES:
            raise ValueError(f"policy {policy} not in {POLICIES}")
        if preemption not in ("cost", "recompute", "swap"):
            raise ValueError("preemption must be cost | recompute | swap")
        if preemption == "cost" and cost_model is None:
            raise ValueError("cost-based preemption needs a cost model")
        if feasibility not in ("pool", "free"):
            raise ValueError("feasibility must be pool | free")
        self.feasibility, self.default_lifo = feasibility, default_lifo
        self.ctx, self.policy, self.k, self.budget = ctx, policy, block_size, budget
        self.num_gpu_blocks = num_gpu_blocks
        self.cm, self.preemption, self.streaming = cost_model, preemption, streaming
        self.reqs: dict[int, SReq] = {}
        self.running: list[int] = []        # DEFAULT's execution order
        self.staged: dict[int, list] = {}   # non-streaming: chunks held back until complete
        self.events = []                    # (time, kind, rid, detail): QUEUED, SCHEDULED, PREEMPTED_*, FINISHED

    # ---- arrivals ------------------------------------------------------------------------
    def on_chunk(self, t: float, rid: int, n_chunks: int, tokens=None, new_input=None, mode="append"):
        """A chunk of request rid arrives at time t: `tokens` are appended (append mode) or
        `new_input` replaces the input (update mode)."""
        r = self.reqs.get(rid)
        if r is None:
            r = SReq(rid, t, n_chunks, mode)
            self.reqs[rid] = r
        r.chunks_arrived += 1
        r.last_chunk_arrival = t
        if not self.streaming:
            self.staged.setdefault(rid, []).append((tokens, new_input))
            if not r.complete:
                return
            # vLLM-NS: the request is submitted once, with its final input
            final = None
            acc = []
            for tok, new in self.staged.pop(rid):
                if new is not None:
                    final, acc = list(new), []
                elif tok is not None:
                    acc.extend(int(x) for x in tok)
            inp = (final or []) + acc
            self.ctx.new_request(rid, inp)
            self.events.append((t, "QUEUED", rid, len(inp)))
            return
        if r.chunks_arrived == 1:
            first = new_input if new_input is not None else (tokens if tokens is not None else [])
            self.ctx.new_request(rid, first)
            self.events.append((t, "QUEUED", rid, len(first)))
        elif new_input is not None:
            _, inval = self.ctx.invalidate_lcp(rid, new_input)
            r.tokens_invalidated += inval
        elif tokens is not None and len(tokens):
            self.ctx.append_chunk([(rid, tokens, 0, 0)], None, None, kv_rows=0)

    # ---- policy ordering (§4.4) ----------------------------------------------------------
    def _pending(self, rid, info):
        return info["num_tokens"] - info["num_computed"]

    def order(self, rids, info):
        R = self.reqs
        if self.policy == "FCFS":
            return sorted(rids, key=lambda x: (not R[x].complete, R[x].arrival, x))
        if self.policy == "LCAS":
            return sorted(rids, key=lambda x: (not R[x].complete, -R[x].last_chunk_arrival, x))
        if self.policy == "MCPS":
            return sorted(rids, key=lambda x: (-info[x]["num_computed"], R[x].arrival, x))
        # DEFAULT vLLM: running in execution order, then waiting (preempted at the front, FIFO)
        run = [x for x in self.running if x in rids]
        wait = [x for x in rids if x not in run]
        wait.sort(key=lambda x: (not R[x].preempted_front, R[x].arrival, x))
        return run + wait

    # ---- one scheduling step --------------------------------------------------------------
    def _blocks(self, n):
        return -(-n // self.k)

    def step(self, t: float):
        """Returns [(rid, q_pos, n_tokens)] to compute this step (K/V append + attention at
        positions [q_pos, q_pos + n)); the caller executes it and calls finish_step()."""
        cands = [r for r in self.reqs if self.reqs[r].status != "finished"]
        if not self.streaming:
            cands = [r for r in cands if self.reqs[r].complete]
        info = {r: self.ctx.query(r) for r in cands}
        if not any(self._pending(r, info[r]) > 0 for r in cands):
            return []
        # all unfinished requests are ranked: those without pending tokens (waiting for their
        # next chunk) still hold blocks and land in not_scheduled, i.e. are preemptible
        order = self.order(cands, info)
        # ---- Phase 1: feasibility (no state change).  Every GPU block is free or held by a
        # request, and Phase 2 can preempt any request left out, so the selected requests fit
        # iff their total block demand (held + new, or swap-in + new) fits in the pool.
        selected, not_sched = [], []
        budget = self.budget
        reserved = 0
        free = self._free_now()                   # "free": projected free blocks
        for r in order:
            n = min(self._pending(r, info[r]), budget)
            if self.feasibility == "pool":
                total = self._blocks(info[r]["num_computed"] + n) if n > 0 else 0
                fits = reserved + total <= self.num_gpu_blocks
            else:
                q = info[r]
                total = (self._blocks(q["num_computed"] + n) - q["num_blocks"] +
                         (q["num_blocks"] if q["tier"] == TIER_CPU else 0)) if n > 0 else 0
                fits = total <= free
            if n > 0 and fits:
                selected.append((r, n))
                reserved += total
                free -= total if self.feasibility == "free" else 0
                budget -= n
            else:
                not_sched.append(r)
        if not selected and self.feasibility == "free":
            # the free-block rule alone can deadlock (every block held by requests that all
            # need more); Phase 2 is given the highest-priority request that fits the pool
            for i, r in enumerate(not_sched):
                n = min(self._pending(r, info[r]), self.budget)
                if n > 0 and self._blocks(info[r]["num_computed"] + n) <= self.num_gpu_blocks:
                    selected.append((r, n))
                    del not_sched[i]
                    break
        # ---- Phase 2: acquisition with preemption (victims: not_sched, lowest priority first)
        out = []
        victims = list(reversed(not_sched))
        if self.policy == "DEFAULT" and self.default_lifo:
            # LIFO over the running order, never a request placed in this step
            placing = {r for r, _ in selected}
            victims = [x for x in reversed(self.running) if x not in placing]
        claimed = 0                      # new blocks the appends of placed requests will take
        for r, n in selected:
            q = self.ctx.query(r)
            new = self._blocks(q["num_computed"] + n) - q["num_blocks"]
            need = new + (q["num_blocks"] if q["tier"] == TIER_CPU else 0)
            while self._free_now() - claimed < need:
                v = self._next_victim(victims)
                if v is None:
                    break
                self._preempt(v, t)
            if self._free_now() - claimed < need:
                not_sched.append(r)
                continue
            claimed += new
            if q["tier"] == TIER_CPU:
                self.ctx.swap_in([r])
            out.append((r, self.ctx.query(r)["num_computed"], n))
            rq = self.reqs[r]
            if rq.status != "running":
                rq.status = "running"
                rq.preempted_front = False
                self.events.append((t, "SCHEDULED", r, n))
            if r not in self.running:
                self.running.append(r)
        return out

    def _free_now(self):
        return self.ctx.free_blocks()[0]

    def _next_victim(self, victims):
        while victims:
            v = victims.pop(0)
            q = self.ctx.query(v)
            if q["tier"] == TIER_GPU and q["num_blocks"] > 0:
                return v
        return None

    def _preempt(self, v, t):
        q = self.ctx.query(v)
        how = self.preemption
        if how == "cost":
            how = self.cm.choose_eviction(q["num_computed"])
        if how == "swap" and self.ctx.free_blocks()[1] < q["num_blocks"]:
            how = "recompute"                          # CPU pool full
        if how == "swap":
            self.ctx.swap_out([v])
            self.reqs[v].preemptions_swap += 1
            self.events.append((t, "PREEMPTED_SWAP", v, q["num_blocks"]))
        else:
            self.ctx.preempt_recompute(v)
            self.reqs[v].preemptions_recompute += 1
            self.events.append((t, "PREEMPTED_RECOMPUTE", v, q["num_computed"]))
        r = self.reqs[v]
        r.status = "waiting"
        r.preempted_front = True
        if v in self.running:
            self.running.remove(v)

    def finish_step(self, t: float, scheduled):
        """After the step's compute: requests whose input is complete and fully computed
        have produced their first token (finish; blocks released)."""
        for r, _, _ in scheduled:
            rq = self.reqs[r]
            q = self.ctx.query(r)
            if rq.complete and q["num_computed"] == q["num_tokens"]:
                rq.finish = t
                rq.status = "finished"
                self.events.append((t, "FINISHED", r, q["num_tokens"]))
                self.ctx.release(r)
                if r in self.running:
                    self.running.remove(r)

    def ttfts(self):
        return {r: q.ttft for r, q in self.reqs.items() if q.finish is not None}


def percentile(xs, p):
    xs = sorted(xs)
    if not xs:
        return math.nan
    i = (len(xs) - 1) * p / 100.0
    lo, hi = int(math.floor(i)), int(math.ceil(i))
    return xs[lo] + (xs[hi] - xs[lo]) * (i - lo)
