"""Request / block state machine of the streaming KV cache — TEST INFRASTRUCTURE ONLY.

(see oracle/__init__.py).  Follows the paper step by step:

  new_request      P:L243-L266 new_stream: input := tokens, num_computed_tokens := 0
  append           P:L59 (K/V of each position "stored as the KV cache")
                   (block B_j holds positions [(j-1)k+1, jk]; blocks from "a free block
                   pool" on demand), P:L147-L149 (Phase 2 allocation; failure => nothing
                   allocated — reading Z15: all-or-nothing per call)
  invalidate_lcp   P:L170 (LCP of old/new input; invalidate blocks beyond it),
                   P:L180 (total_tokens_invalidated), P:L182 ("frees the corresponding
                   KV cache blocks ... For CPU-swapped requests ... also frees the
                   corresponding CPU blocks ... sets num_computed_tokens to the LCP
                   length"), P:L184 (swapped request: invalidate on CPU, resume = swap in
                   the prefix, recompute from the LCP)
  swap_out/in      P:L77 ("Transfer all blocks {B_1..B_⌈ℓ/k⌉} from GPU to CPU memory ...
                   swap blocks back to GPU with symmetric cost ... preserve computed KV")
  preempt_recompute P:L73-L75 ("Discard all KV cache blocks for r ... recompute the
                   prefill phase for all ℓ_r tokens")
  release          request finished: all blocks return to the pools

Readings: Z4 token-granular LCP by default (keep ⌈b/k⌉ blocks,
the boundary block's stale tail is never read), `lcp_block_aligned` reproduces SPEC's
block round-down; Z5 b = min(p, nc); Z9 lowest free id first on both tiers,
independent of free order (the paper only says "free block pool"),
items/requests served in call order; `alloc_cooling` is an OPT-IN performance variant of
Z9 (not the paper's) (GPU ids released by the most recent swap-out come after every other free id),
mirrored here as an explicit parameter with its own golden; Z12 swap copies whole blocks.

The oracle keeps its OWN model of everything:
  * per request: input tokens, nc, tier, ordered block ids, total_tokens_invalidated,
    and CONTIGUOUS K/V rows Kc/Vc [L][T][h_kv][d] (bf16 bits) used by attention;
  * a byte-exact mirror of the GPU pool and the CPU pool, layout
    [block][L][2 (K,V)][h_kv][k][d] bf16 (the layout fixed by include/s2l.h), both
    zero-initialised (s2l_create zero-fills the pools).
Status codes are the values documented in include/s2l.h (restated, not imported).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import fp8 as _fp8
from .attention import attention as _attention
from .geometry import block_bytes, blocks_needed
from .lcp import lcp

OK = 0
E_INVAL = -1
E_NO_GPU_BLOCKS = -2
E_NO_CPU_BLOCKS = -3
E_NO_REQUEST = -4
E_STATE = -5
E_CAPACITY = -7

GPU = 0
CPU = 1


@dataclass
class Req:
    input: list
    nc: int = 0
    tier: int = GPU
    blocks: list = field(default_factory=list)
    tti: int = 0
    Kc: np.ndarray | None = None   # [L][cap][h_kv][d] uint16
    Vc: np.ndarray | None = None


class OracleKV:
    def __init__(self, L, h_q, h_kv, d, k, num_gpu_blocks, num_cpu_blocks,
                 max_requests=1 << 30, max_blocks_per_request=1 << 30, lcp_block_aligned=False,
                 mirror_pools=True, alloc_cooling=False, kv_dtype="bf16"):
        """kv_dtype "fp8" (the optional FP8 KV cache; not the paper's b = 2): K/V
        are stored as E4M3 codes (oracle/fp8.py, b = 1); attention reads their exact values."""
        assert h_q % h_kv == 0
        self.L, self.h_q, self.h_kv, self.d, self.k = L, h_q, h_kv, d, k
        self.num_gpu_blocks, self.num_cpu_blocks = num_gpu_blocks, num_cpu_blocks
        self.max_requests, self.max_blocks = max_requests, max_blocks_per_request
        self.aligned = bool(lcp_block_aligned)
        if kv_dtype not in ("bf16", "fp8"):
            raise ValueError(kv_dtype)
        self.fp8 = kv_dtype == "fp8"
        self.free = {GPU: set(range(num_gpu_blocks)), CPU: set(range(num_cpu_blocks))}
        self.cooling = bool(alloc_cooling)
        self.cool = set()   # alloc_cooling: GPU ids released by the latest swap-out, subset of free
        self.reqs: dict[int, Req] = {}
        self.mirror = mirror_pools
        shape = (L, 2, h_kv, k, d)
        pdt = np.uint8 if self.fp8 else np.uint16
        self.pool = {GPU: np.zeros((num_gpu_blocks,) + shape, pdt) if mirror_pools else None,
                     CPU: np.zeros((num_cpu_blocks,) + shape, pdt) if mirror_pools else None}

    # ---- helpers -------------------------------------------------------------------
    @property
    def m_block(self) -> int:
        return block_bytes(self.L, self.k, self.h_kv, self.d, b=1 if self.fp8 else 2)

    def _take_lowest(self, tier, n):
        """Z9: the n lowest free ids, ascending.  alloc_cooling variant: GPU ids released by
        the most recent swap-out ("cooling") come after every other free id (lowest first)."""
        cool = self.cool if tier == GPU else set()
        ids = sorted(self.free[tier] - cool)[:n]
        if len(ids) < n:
            ids += sorted(cool)[: n - len(ids)]
        for i in ids:
            self.free[tier].remove(i)
            cool.discard(i)
        return ids

    def _give_back(self, tier, ids):
        for i in ids:
            assert i not in self.free[tier]
            self.free[tier].add(i)

    def _ensure_cap(self, r: Req, T: int):
        cap = 0 if r.Kc is None else r.Kc.shape[1]
        if cap >= T:
            return
        new = max(T, 2 * cap, 16)
        shape = (self.L, new, self.h_kv, self.d)
        Kc, Vc = np.zeros(shape, np.uint16), np.zeros(shape, np.uint16)
        if r.Kc is not None:
            Kc[:, :cap] = r.Kc
            Vc[:, :cap] = r.Vc
        r.Kc, r.Vc = Kc, Vc

    # ---- API -----------------------------------------------------------------------
    def new_request(self, rid, toks=()):
        """NewStream: input := tokens, nc := 0, GPU tier, no blocks."""
        if rid in self.reqs:
            return E_STATE
        if len(self.reqs) >= self.max_requests:
            return E_CAPACITY
        self.reqs[rid] = Req(input=[int(t) for t in toks])
        return OK

    def release(self, rid):
        """Request finished: its blocks on both tiers return to the free pools."""
        r = self.reqs.get(rid)
        if r is None:
            return E_NO_REQUEST
        self._give_back(r.tier, r.blocks)
        del self.reqs[rid]
        return OK

    def preempt_recompute(self, rid):
        """Recomputation preemption: discard all blocks, nc := 0, GPU tier."""
        r = self.reqs.get(rid)
        if r is None:
            return E_NO_REQUEST
        self._give_back(r.tier, r.blocks)
        r.blocks, r.nc, r.tier = [], 0, GPU
        return OK

    def append(self, items, k_rows=None, v_rows=None):
        """Append tokens and write K/V of the next n_kv pending positions, all-or-nothing.

        items: list of (rid, tokens_or_None, n_kv, kv_row); k_rows/v_rows [L][R][h_kv][d]
        (bf16 bits) hold the rows, item i's rows at [kv_row, kv_row+n_kv).
        Validation order (first failing item wins, capacity last) is the one documented
        for s2l_append_chunk in include/s2l.h.
        """
        seen = set()
        need_total = 0
        for rid, toks, n_kv, kv_row in items:
            r = self.reqs.get(rid)
            if r is None:
                return E_NO_REQUEST
            if rid in seen:
                return E_INVAL
            seen.add(rid)
            if r.tier != GPU and n_kv != 0:             # Z19: token-only append on either tier
                return E_STATE
            n_tok = 0 if toks is None else len(toks)
            if n_kv < 0 or kv_row < 0:
                return E_INVAL
            if n_kv > 0 and kv_row + n_kv > k_rows.shape[1]:
                return E_INVAL
            if n_kv > len(r.input) + n_tok - r.nc:
                return E_INVAL
            nb = blocks_needed(r.nc + n_kv, self.k)
            if nb > self.max_blocks:
                return E_INVAL
            need_total += nb - len(r.blocks)
        if need_total > len(self.free[GPU]):
            return E_NO_GPU_BLOCKS
        for rid, toks, n_kv, kv_row in items:
            r = self.reqs[rid]
            if toks is not None:
                r.input.extend(int(t) for t in toks)
            need = blocks_needed(r.nc + n_kv, self.k) - len(r.blocks)
            r.blocks.extend(self._take_lowest(GPU, need))
            if n_kv:
                self._ensure_cap(r, r.nc + n_kv)
                kr, vr = k_rows[:, kv_row:kv_row + n_kv], v_rows[:, kv_row:kv_row + n_kv]
                if self.fp8:                                # stored codes; attention reads their values
                    kc, kr = _fp8.quantize_bf16_bits(kr)
                    vc, vr = _fp8.quantize_bf16_bits(vr)
                else:
                    kc, vc = kr, vr
                r.Kc[:, r.nc:r.nc + n_kv] = kr
                r.Vc[:, r.nc:r.nc + n_kv] = vr
                if self.mirror:
                    for t in range(n_kv):
                        pos = r.nc + t
                        blk, slot = r.blocks[pos // self.k], pos % self.k
                        self.pool[GPU][blk, :, 0, :, slot, :] = kc[:, t]
                        self.pool[GPU][blk, :, 1, :, slot, :] = vc[:, t]
            r.nc += n_kv
        return OK

    def invalidate_lcp(self, rid, new_tokens):
        """Update event. Returns (status, p, invalidated)."""
        r = self.reqs.get(rid)
        if r is None:
            return E_NO_REQUEST, 0, 0
        new = [int(t) for t in new_tokens]
        p = lcp(r.input, new)
        b = min(p, r.nc)                                # Z5
        if self.aligned:
            b = (b // self.k) * self.k                  # S:L191 variant
        keep = blocks_needed(b, self.k)                 # Z4: keep the boundary block
        self._give_back(r.tier, r.blocks[keep:])        # free on the tier holding them
        r.blocks = r.blocks[:keep]
        inval = r.nc - b
        r.nc = b                                        # num_computed_tokens := LCP
        r.tti += inval
        r.input = new
        if r.tier == CPU and keep == 0:                 # nothing left to swap back
            r.tier = GPU
        return OK, p, inval

    def swap_out(self, rids):
        """All blocks of each listed request GPU -> CPU, in order. (status, bytes)."""
        return self._swap(rids, GPU, CPU, E_NO_CPU_BLOCKS)

    def swap_in(self, rids):
        """Mirror of swap_out ("symmetric"), prefix blocks only after an update."""
        return self._swap(rids, CPU, GPU, E_NO_GPU_BLOCKS)

    def _swap(self, rids, src, dst, e_full):
        seen = set()
        need = 0
        for rid in rids:
            r = self.reqs.get(rid)
            if r is None:
                return E_NO_REQUEST, 0
            if rid in seen:
                return E_INVAL, 0
            seen.add(rid)
            if r.tier != src:
                return E_STATE, 0
            need += len(r.blocks)
        if need > len(self.free[dst]):
            return e_full, 0
        if src == GPU and rids and self.cooling:
            self.cool = set()                           # the previous swap-out's ids thaw
        for rid in rids:
            r = self.reqs[rid]
            new_ids = self._take_lowest(dst, len(r.blocks))
            if self.mirror:
                for s, t in zip(r.blocks, new_ids):
                    self.pool[dst][t] = self.pool[src][s]   # whole block (Z12)
            self._give_back(src, r.blocks)
            if src == GPU and self.cooling:
                self.cool.update(r.blocks)
            r.blocks, r.tier = new_ids, dst
        return OK, need * self.m_block

    def prefill(self, items, q_rows, layer=0):
        """Attention for each item (rid, q_pos, n_q, q_row) of a batch; q_rows [R][h_q][d].

        Returns (status, O [R][h_q][d] fp64 with untouched rows = 0, LSE [R][h_q]).
        Reads each request's contiguous Kc/Vc, never the pool (see attention.py).
        """
        R = q_rows.shape[0]
        O = np.zeros((R, self.h_q, self.d))
        LSE = np.zeros((R, self.h_q))
        for rid, q_pos, n_q, q_row in items:
            r = self.reqs.get(rid)
            if r is None:
                return E_NO_REQUEST, None, None
            if r.tier != GPU:
                return E_STATE, None, None
            if n_q < 1 or q_pos < 0 or q_row < 0 or q_pos + n_q > r.nc or q_row + n_q > R:
                return E_INVAL, None, None
            if not (0 <= layer < self.L):
                return E_INVAL, None, None
        for rid, q_pos, n_q, q_row in items:
            r = self.reqs[rid]
            o, l = _attention(q_rows[q_row:q_row + n_q], r.Kc[layer], r.Vc[layer], q_pos)
            O[q_row:q_row + n_q] = o
            LSE[q_row:q_row + n_q] = l
        return OK, O, LSE

    # ---- queries -------------------------------------------------------------------
    def info(self, rid):
        r = self.reqs[rid]
        return dict(num_tokens=len(r.input), num_computed=r.nc, total_tokens_invalidated=r.tti,
                    tier=r.tier, num_blocks=len(r.blocks))

    def block_table(self, rid):
        return list(self.reqs[rid].blocks)

    def free_counts(self):
        return len(self.free[GPU]), len(self.free[CPU])

    def valid_slots(self, rid):
        """(block, slot) of positions [0, nc) of a request, in position order."""
        r = self.reqs[rid]
        return [(r.blocks[p // self.k], p % self.k) for p in range(r.nc)]
