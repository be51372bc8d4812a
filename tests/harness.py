"""Test harness: drives libs2l (through the C ABI binding) and the oracle side by side on the
same seeded inputs, and compares them (bit-exact for tables / bytes / counts, normwise
relative error for attention).  Only tests/ imports this module."""
from __future__ import annotations

import numpy as np
import torch

from oracle import kvcache as O
from oracle.kvcache import OracleKV
from paper_2604_16395_b200 import s2l

ATOL_NORMWISE = 2e-2   # BJ:L5: max relative error 2e-2 (bf16 in, fp32 accumulate)
LSE_ATOL = 1e-2


def to_dev(bits: np.ndarray, dev="cuda"):
    return torch.from_numpy(np.ascontiguousarray(bits)).view(torch.bfloat16).to(dev)


def bf16_dev_to_f64(t) -> np.ndarray:
    b = t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def normwise_err(o_gpu: np.ndarray, o_ref: np.ndarray) -> np.ndarray:
    """err(row, head) = ||O_gpu - O_ref||_inf / max(||O_ref||_inf, 1e-6) over d."""
    num = np.abs(o_gpu - o_ref).max(axis=-1)
    den = np.maximum(np.abs(o_ref).max(axis=-1), 1e-6)
    return num / den


class Pair:
    """A libs2l device context and an OracleKV with identical geometry."""

    def __init__(self, L, h_q, h_kv, d, k, ng, nc, aligned=False, max_requests=64, max_blocks=None,
                 mirror=True, stream=None, cooling=False, kv_dtype=0):
        self.geo = (L, h_q, h_kv, d, k)
        self.L, self.h_q, self.h_kv, self.d, self.k = L, h_q, h_kv, d, k
        cfg = s2l.make_config(L, h_q, h_kv, d, k, ng, nc, max_requests=max_requests,
                              max_blocks_per_request=max_blocks or max(ng, nc, 1),
                              lcp_block_aligned=int(aligned), alloc_cooling=int(cooling),
                              kv_dtype=int(kv_dtype))
        self.fp8 = kv_dtype == 1
        self.m_block = s2l.block_bytes(cfg)
        self.gpu_pool = torch.empty(max(1, ng) * self.m_block // 2, dtype=torch.bfloat16, device="cuda")
        self.cpu_pool = torch.empty(max(1, nc) * self.m_block // 2, dtype=torch.bfloat16).pin_memory()
        # non-zero garbage first: s2l_create must zero-fill both pools
        self.gpu_pool.view(torch.int16).fill_(0x7FC1)
        self.cpu_pool.view(torch.int16).fill_(0x7FC1)
        self.stream = stream or torch.cuda.current_stream()
        self.lib = s2l.Context(cfg, self.gpu_pool, self.cpu_pool if nc else None, self.stream, None)
        self.ora = OracleKV(L, h_q, h_kv, d, k, ng, nc, max_requests=max_requests,
                            max_blocks_per_request=max_blocks or max(ng, nc, 1), lcp_block_aligned=aligned,
                            mirror_pools=mirror, alloc_cooling=cooling,
                            kv_dtype="fp8" if kv_dtype == 1 else "bf16")
        self.ng, self.nc = ng, nc

    # ---- ops on both sides -----------------------------------------------------------
    def new(self, rid, toks=()):
        a = s2l.status_of(self.lib.new_request, rid, toks)
        b = self.ora.new_request(rid, toks)
        assert a == b
        return a

    def append(self, items, k_bits, v_bits):
        """items [(rid, toks|None, n_kv, kv_row)], k/v bits [L][R][h_kv][d]."""
        kd, vd = to_dev(k_bits), to_dev(v_bits)
        a = s2l.status_of(self.lib.append_chunk, items, kd, vd)
        b = self.ora.append(items, k_bits, v_bits)
        assert a == b, (a, b)
        self._keep = (kd, vd)
        return a

    def append_reserve(self, items, k_bits, v_bits):
        """Library: append_chunk in reserve mode (k = v = NULL, NEXT-2); oracle: the full append
        (its bytes are what the per-layer prefill_append calls must leave in the pool)."""
        a = s2l.status_of(self.lib.append_chunk, items, None, None, kv_rows=k_bits.shape[1])
        b = self.ora.append(items, k_bits, v_bits)
        assert a == b, (a, b)
        return a

    def prefill_append(self, items, q_bits, k_bits_l, v_bits_l, layer=0, check=True):
        """Fused append + attention of one layer (library) vs the oracle's attention over the
        pool its append wrote."""
        qd, kd, vd = to_dev(q_bits), to_dev(k_bits_l), to_dev(v_bits_l)
        od = torch.zeros_like(qd)
        ld = torch.zeros(q_bits.shape[0], self.h_q, dtype=torch.float32, device="cuda")
        self.lib.prefill_append(layer, items, qd, kd, vd, od, ld)
        torch.cuda.synchronize()
        st, o_ref, l_ref = self.ora.prefill(items, q_bits, layer)
        assert st == O.OK
        o_gpu = bf16_dev_to_f64(od)
        l_gpu = ld.cpu().numpy().astype(np.float64)
        if check:
            self.check_attention(items, o_gpu, o_ref, l_gpu, l_ref)
        return o_gpu, o_ref

    def invalidate(self, rid, new):
        a = self.lib.invalidate_lcp(rid, new)
        st, p, inv = self.ora.invalidate_lcp(rid, new)
        assert st == O.OK and a == (p, inv)
        return a

    def swap_out(self, rids):
        try:
            a = (s2l.OK, self.lib.swap_out(rids))
        except s2l.S2LError as e:
            a = (e.status, 0)
        b = self.ora.swap_out(rids)
        assert a == b, (a, b)
        return a

    def swap_in(self, rids):
        try:
            a = (s2l.OK, self.lib.swap_in(rids))
        except s2l.S2LError as e:
            a = (e.status, 0)
        b = self.ora.swap_in(rids)
        assert a == b, (a, b)
        return a

    def prefill(self, items, q_bits, layer=0, lse=True, check=True, rows=None):
        """Runs both sides; returns (O_gpu f64, O_ref f64, LSE_gpu, LSE_ref)."""
        qd = to_dev(q_bits)
        od = torch.zeros_like(qd)
        ld = torch.zeros(q_bits.shape[0], self.h_q, dtype=torch.float32, device="cuda") if lse else None
        self.lib.prefill_batch(layer, items, qd, od, ld)
        torch.cuda.synchronize()
        st, o_ref, l_ref = self.ora.prefill(items, q_bits, layer)
        assert st == O.OK
        o_gpu = bf16_dev_to_f64(od)
        l_gpu = ld.cpu().numpy().astype(np.float64) if lse else None
        if check:
            self.check_attention(items, o_gpu, o_ref, l_gpu, l_ref)
        return o_gpu, o_ref, l_gpu, l_ref

    def check_attention(self, items, o_gpu, o_ref, l_gpu=None, l_ref=None):
        for rid, q_pos, n_q, q_row in items:
            sl = slice(q_row, q_row + n_q)
            err = normwise_err(o_gpu[sl], o_ref[sl])
            assert np.isfinite(o_gpu[sl]).all()
            assert err.max() <= ATOL_NORMWISE, (rid, q_pos, n_q, float(err.max()), np.unravel_index(err.argmax(), err.shape))
            if l_gpu is not None:
                dl = np.abs(l_gpu[sl] - l_ref[sl])
                assert dl.max() <= LSE_ATOL, (rid, float(dl.max()))

    # ---- state / byte checks ---------------------------------------------------------
    def check_state(self):
        assert self.lib.free_blocks() == self.ora.free_counts()
        for rid in self.ora.reqs:
            assert self.lib.query(rid) == self.ora.info(rid)
            assert self.lib.block_table(rid) == self.ora.block_table(rid)

    def gpu_pool_bits(self):
        """The GPU pool as [block][L][2][h_kv][k][d] codes: bf16 bits (uint16) or E4M3 bytes."""
        torch.cuda.synchronize()
        self.lib.sync()
        dt = np.uint8 if self.fp8 else np.uint16
        b = self.gpu_pool.view(torch.int16).cpu().numpy().view(dt)
        return b[: self.ng * self.L * 2 * self.h_kv * self.k * self.d].reshape(self.ng, self.L, 2, self.h_kv, self.k, self.d)

    def cpu_pool_bits(self):
        self.lib.sync()
        dt = np.uint8 if self.fp8 else np.uint16
        b = self.cpu_pool.view(torch.int16).numpy().view(dt)
        return b[: self.nc * self.L * 2 * self.h_kv * self.k * self.d].reshape(self.nc, self.L, 2, self.h_kv, self.k, self.d)

    def check_pool_valid_slots(self):
        """GPU pool bytes at every valid slot of every GPU-tier request == oracle's rows (FP8:
        == the oracle's E4M3 codes of those rows, its pool mirror)."""
        g = self.gpu_pool_bits()
        if self.fp8:
            for rid, r in self.ora.reqs.items():
                if r.tier != O.GPU or r.nc == 0:
                    continue
                pos = np.arange(r.nc)
                blk = np.array(r.blocks)[pos // self.k]
                slot = pos % self.k
                m = self.ora.pool[O.GPU]
                assert np.array_equal(g[blk, :, :, :, slot, :], m[blk, :, :, :, slot, :]), rid
            return
        for rid, r in self.ora.reqs.items():
            if r.tier != O.GPU or r.nc == 0:
                continue
            pos = np.arange(r.nc)
            blk = np.array(r.blocks)[pos // self.k]
            slot = pos % self.k
            got_k = g[blk, :, 0, :, slot, :]            # [nc][L][h_kv][d]
            got_v = g[blk, :, 1, :, slot, :]
            assert np.array_equal(got_k, np.transpose(r.Kc[:, : r.nc], (1, 0, 2, 3))), rid
            assert np.array_equal(got_v, np.transpose(r.Vc[:, : r.nc], (1, 0, 2, 3))), rid

    def check_pools_whole(self):
        """Whole-block byte identity with the oracle's mirrors (stale tails included)."""
        g = self.gpu_pool_bits()
        for rid, r in self.ora.reqs.items():
            if r.tier == O.GPU and r.blocks:
                assert np.array_equal(g[r.blocks], self.ora.pool[O.GPU][r.blocks]), rid
        if self.nc:
            c = self.cpu_pool_bits()
            for rid, r in self.ora.reqs.items():
                if r.tier == O.CPU and r.blocks:
                    assert np.array_equal(c[r.blocks], self.ora.pool[O.CPU][r.blocks]), rid


class Twin:
    """Context interface for drivers (paper_2604_16395_b200.pressure) that applies every call
    to a libs2l context AND to a bookkeeping-only OracleKV (tiny geometry: block ids, counts,
    LCP and statuses do not depend on L / heads / d), asserting identical results; swap
    byte counts are compared in blocks (bytes / M_block of each side)."""

    def __init__(self, lib, k, ng, nc, max_requests, max_blocks):
        self.lib = lib
        self.ora = OracleKV(1, 1, 1, 8, k, ng, nc, max_requests=max_requests,
                            max_blocks_per_request=max_blocks, mirror_pools=False,
                            alloc_cooling=bool(lib.cfg.alloc_cooling))
        self.m_lib = s2l.block_bytes(lib.cfg)
        self.ops = 0

    def _same_state(self, rids):
        for r in rids:
            assert self.lib.query(r) == self.ora.info(r), r
            assert self.lib.block_table(r) == self.ora.block_table(r), r
        assert self.lib.free_blocks() == self.ora.free_counts()

    def new_request(self, rid, toks=()):
        self.lib.new_request(rid, toks)
        assert self.ora.new_request(rid, toks) == O.OK
        self.ops += 1

    def release(self, rid):
        self.lib.release(rid)
        assert self.ora.release(rid) == O.OK
        self._same_state([])

    def preempt_recompute(self, rid):
        self.lib.preempt_recompute(rid)
        assert self.ora.preempt_recompute(rid) == O.OK
        self._same_state([rid])

    def invalidate_lcp(self, rid, new):
        a = self.lib.invalidate_lcp(rid, new)
        st, p, inv = self.ora.invalidate_lcp(rid, new)
        assert st == O.OK and a == (p, inv), (a, p, inv)
        self._same_state([rid])
        return a

    def _swap(self, fn_lib, fn_ora, rids):
        b = fn_lib(rids)
        st, bo = fn_ora(rids)
        assert st == O.OK and b // self.m_lib == bo // self.ora.m_block and b % self.m_lib == 0
        self._same_state(rids)
        return b

    def swap_out(self, rids):
        return self._swap(self.lib.swap_out, self.ora.swap_out, rids)

    def swap_in(self, rids):
        return self._swap(self.lib.swap_in, self.ora.swap_in, rids)

    def append_chunk(self, items, k=None, v=None, kv_rows=None):
        rows = kv_rows if kv_rows is not None else (0 if k is None else k.shape[1])
        self.lib.append_chunk(items, k, v, kv_rows=rows)
        z = np.zeros((1, max(1, rows), 1, 8), np.uint16)
        assert self.ora.append(items, z, z) == O.OK
        self._same_state([it[0] for it in items])

    def query(self, rid):
        a = self.lib.query(rid)
        assert a == self.ora.info(rid)
        return a

    def free_blocks(self):
        a = self.lib.free_blocks()
        assert a == self.ora.free_counts()
        return a

    def prefill_batch(self, *a, **kw):
        return self.lib.prefill_batch(*a, **kw)

    def sync(self):
        return self.lib.sync()
