"""Thin ctypes binding of libs2l (include/s2l.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module converts
Python/torch arguments into the C ABI's plain pointers and sizes.  torch is used only for
device / pinned memory and stream handles.  If libs2l.so is missing the import of `lib()`
raises — there is no fallback path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# S2L_LIB selects another build of the same library (sanitizer builds, A/B experiments)
LIB_PATH = os.environ.get("S2L_LIB") or os.path.join(_PKG, "libs2l.so")

OK, E_INVAL, E_NO_GPU_BLOCKS, E_NO_CPU_BLOCKS, E_NO_REQUEST, E_STATE, E_CUDA, E_CAPACITY = 0, -1, -2, -3, -4, -5, -6, -7
TIER_GPU, TIER_CPU = 0, 1
KV_BF16, KV_FP8 = 0, 1
STATUS_NAMES = {0: "OK", -1: "E_INVAL", -2: "E_NO_GPU_BLOCKS", -3: "E_NO_CPU_BLOCKS",
                -4: "E_NO_REQUEST", -5: "E_STATE", -6: "E_CUDA", -7: "E_CAPACITY"}


class S2LError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_q_heads", C.c_int32), ("num_kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("block_size", C.c_int32), ("num_gpu_blocks", C.c_int32),
                ("num_cpu_blocks", C.c_int32), ("max_requests", C.c_int32),
                ("max_blocks_per_request", C.c_int32), ("lcp_block_aligned", C.c_int32),
                ("alloc_cooling", C.c_int32), ("kv_dtype", C.c_int32)]


class AppendItem(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("tokens", C.POINTER(C.c_int32)), ("n_tokens", C.c_int64),
                ("n_kv", C.c_int64), ("kv_row", C.c_int64)]


class PrefillItem(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("q_pos", C.c_int64), ("n_q", C.c_int64), ("q_row", C.c_int64)]


class ReqInfo(C.Structure):
    _fields_ = [("num_tokens", C.c_int64), ("num_computed", C.c_int64),
                ("total_tokens_invalidated", C.c_int64), ("tier", C.c_int32), ("num_blocks", C.c_int32)]


EXPORTS = ["s2l_block_bytes", "s2l_create", "s2l_create_host_only", "s2l_destroy", "s2l_new_request",
           "s2l_release_request", "s2l_preempt_recompute", "s2l_append_chunk", "s2l_invalidate_lcp",
           "s2l_prefill_batch", "s2l_prefill_append", "s2l_swap_out", "s2l_swap_in", "s2l_query", "s2l_block_table",
           "s2l_free_blocks", "s2l_sync", "s2l_set_swap_in_stream", "s2l_kernel_launches", "s2l_wait_counts", "s2l_set_timing", "s2l_timing_read",
           "s2l_last_error", "s2l_version"]

_libs: dict = {}


def lib(path: str | None = None) -> C.CDLL:
    """Loads libs2l.so (raises FileNotFoundError if it has not been built).  `path` selects
    another build of the same library (A/B timing experiments load several side by side)."""
    path = path or LIB_PATH
    if path in _libs:
        return _libs[path]
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built: run `python -m paper_2604_16395_b200.build`")
    L = C.CDLL(path)
    P, I32, I64, VP = C.POINTER, C.c_int32, C.c_int64, C.c_void_p
    sig = {
        "s2l_block_bytes": (I64, [P(Config)]),
        "s2l_create": (I32, [P(Config), VP, VP, VP, VP, P(VP)]),
        "s2l_create_host_only": (I32, [P(Config), P(VP)]),
        "s2l_destroy": (None, [VP]),
        "s2l_new_request": (I32, [VP, I64, P(I32), I64]),
        "s2l_release_request": (I32, [VP, I64]),
        "s2l_preempt_recompute": (I32, [VP, I64]),
        "s2l_append_chunk": (I32, [VP, I32, P(AppendItem), VP, VP, I64]),
        "s2l_invalidate_lcp": (I32, [VP, I64, P(I32), I64, P(I64), P(I64)]),
        "s2l_prefill_batch": (I32, [VP, I32, I32, P(PrefillItem), VP, VP, VP, I64]),
        "s2l_prefill_append": (I32, [VP, I32, I32, P(PrefillItem), VP, VP, VP, VP, VP, I64]),
        "s2l_swap_out": (I32, [VP, I32, P(I64), P(I64)]),
        "s2l_swap_in": (I32, [VP, I32, P(I64), P(I64)]),
        "s2l_query": (I32, [VP, I64, P(ReqInfo)]),
        "s2l_block_table": (I32, [VP, I64, P(I32), I64, P(I64)]),
        "s2l_free_blocks": (I32, [VP, P(I64), P(I64)]),
        "s2l_sync": (I32, [VP]),
        "s2l_set_swap_in_stream": (I32, [VP, VP]),
        "s2l_kernel_launches": (I64, [VP]),
        "s2l_wait_counts": (I32, [VP, P(I64)]),
        "s2l_set_timing": (I32, [VP, I32]),
        "s2l_timing_read": (I32, [VP, P(C.c_double), P(I64), P(C.c_double), P(I64)]),
        "s2l_last_error": (C.c_char_p, []),
        "s2l_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        if path != LIB_PATH and not hasattr(L, name):
            continue            # an older build loaded for an A/B comparison
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    _libs[path] = L
    return L


def _i32p(arr):
    return arr.ctypes.data_as(C.POINTER(C.c_int32))


def _ptr(t):
    """Device/host pointer of a torch tensor (or None -> NULL).  The ABI takes dense row-major
    arrays, so a strided view (e.g. a column slice of a fused QKV output) is refused."""
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("libs2l takes contiguous tensors (call .contiguous() on strided views)")
    return C.c_void_p(t.data_ptr())


def _stream(s):
    if s is None:
        return None
    return C.c_void_p(s.cuda_stream if hasattr(s, "cuda_stream") else int(s))


def make_config(num_layers, num_q_heads, num_kv_heads, head_dim, block_size, num_gpu_blocks,
                num_cpu_blocks, max_requests=256, max_blocks_per_request=None, lcp_block_aligned=0,
                alloc_cooling=0, kv_dtype=0):
    if max_blocks_per_request is None:
        max_blocks_per_request = max(1, num_gpu_blocks + num_cpu_blocks)
    return Config(num_layers, num_q_heads, num_kv_heads, head_dim, block_size, num_gpu_blocks,
                  num_cpu_blocks, max_requests, max_blocks_per_request, int(lcp_block_aligned),
                  int(alloc_cooling), int(kv_dtype))


def block_bytes(cfg: Config) -> int:
    return lib().s2l_block_bytes(C.byref(cfg))


class Context:
    """One libs2l context (one device).  Methods raise S2LError on a non-OK status."""

    def __init__(self, cfg: Config, gpu_pool=None, cpu_pool=None, compute_stream=None,
                 copy_stream=None, host_only=False, lib_path=None, swap_in_stream=None):
        self._L = lib(lib_path)
        self.cfg = cfg
        self.host_only = host_only
        h = C.c_void_p()
        if host_only:
            st = self._L.s2l_create_host_only(C.byref(cfg), C.byref(h))
        else:
            st = self._L.s2l_create(C.byref(cfg), _ptr(gpu_pool), _ptr(cpu_pool),
                                    _stream(compute_stream), _stream(copy_stream), C.byref(h))
        self._check(st)
        self._h = h
        self._keep = (gpu_pool, cpu_pool, compute_stream, copy_stream, swap_in_stream)
        if swap_in_stream is not None:
            self._check(self._L.s2l_set_swap_in_stream(h, _stream(swap_in_stream)))

    def _check(self, st):
        if st != OK:
            raise S2LError(st, self._L.s2l_last_error().decode())
        return st

    def close(self):
        if getattr(self, "_h", None):
            self._L.s2l_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- requests ----
    def new_request(self, rid: int, tokens=()):
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
        return self._check(self._L.s2l_new_request(self._h, rid, _i32p(t), len(t)))

    def release(self, rid: int):
        return self._check(self._L.s2l_release_request(self._h, rid))

    def preempt_recompute(self, rid: int):
        return self._check(self._L.s2l_preempt_recompute(self._h, rid))

    def append_chunk(self, items, k=None, v=None, kv_rows=None):
        """items: [(rid, tokens|None, n_kv, kv_row)]; k, v: [L][kv_rows][h_kv][d] bf16 (device)."""
        keep = []
        arr = (AppendItem * max(1, len(items)))()
        for i, (rid, toks, n_kv, kv_row) in enumerate(items):
            if toks is not None and len(toks):
                t = np.ascontiguousarray(np.asarray(toks, dtype=np.int32))
                keep.append(t)
                arr[i] = AppendItem(rid, _i32p(t), len(t), n_kv, kv_row)
            else:
                arr[i] = AppendItem(rid, None, 0, n_kv, kv_row)
        if kv_rows is None:
            kv_rows = 0 if k is None else k.shape[1]
        return self._check(self._L.s2l_append_chunk(self._h, len(items), arr, _ptr(k), _ptr(v), kv_rows))

    def invalidate_lcp(self, rid: int, new_tokens):
        t = np.ascontiguousarray(np.asarray(new_tokens, dtype=np.int32))
        p, inval = C.c_int64(), C.c_int64()
        self._check(self._L.s2l_invalidate_lcp(self._h, rid, _i32p(t), len(t), C.byref(p), C.byref(inval)))
        return p.value, inval.value

    def prefill_batch(self, layer: int, items, q, o, lse=None):
        """items: [(rid, q_pos, n_q, q_row)]; q, o: [rows][h_q][d] bf16; lse: [rows][h_q] f32."""
        arr = (PrefillItem * max(1, len(items)))(*[PrefillItem(*it) for it in items])
        return self._check(self._L.s2l_prefill_batch(self._h, layer, len(items), arr, _ptr(q), _ptr(o),
                                                     _ptr(lse), q.shape[0] if q is not None else 0))

    def prefill_append(self, layer: int, items, q, k, v, o, lse=None):
        """Fused append + attention of one layer (NEXT-2).  items: [(rid, q_pos, n_q, q_row)];
        q, o: [rows][h_q][d]; k, v: [rows][h_kv][d] bf16 of this layer; the blocks are held
        (append_chunk with k = v = None reserves them)."""
        arr = (PrefillItem * max(1, len(items)))(*[PrefillItem(*it) for it in items])
        return self._check(self._L.s2l_prefill_append(self._h, layer, len(items), arr, _ptr(q), _ptr(k),
                                                      _ptr(v), _ptr(o), _ptr(lse),
                                                      q.shape[0] if q is not None else 0))

    def swap_out(self, rids):
        ids = (C.c_int64 * max(1, len(rids)))(*rids)
        b = C.c_int64()
        self._check(self._L.s2l_swap_out(self._h, len(rids), ids, C.byref(b)))
        return b.value

    def swap_in(self, rids):
        ids = (C.c_int64 * max(1, len(rids)))(*rids)
        b = C.c_int64()
        self._check(self._L.s2l_swap_in(self._h, len(rids), ids, C.byref(b)))
        return b.value

    # ---- queries ----
    def query(self, rid: int) -> dict:
        info = ReqInfo()
        self._check(self._L.s2l_query(self._h, rid, C.byref(info)))
        return dict(num_tokens=info.num_tokens, num_computed=info.num_computed,
                    total_tokens_invalidated=info.total_tokens_invalidated, tier=info.tier,
                    num_blocks=info.num_blocks)

    def block_table(self, rid: int) -> list:
        n = C.c_int64()
        self._check(self._L.s2l_block_table(self._h, rid, None, 0, C.byref(n)))
        buf = np.zeros(max(1, n.value), dtype=np.int32)
        self._check(self._L.s2l_block_table(self._h, rid, _i32p(buf), n.value, C.byref(n)))
        return buf[: n.value].tolist()

    def free_blocks(self):
        g, c = C.c_int64(), C.c_int64()
        self._check(self._L.s2l_free_blocks(self._h, C.byref(g), C.byref(c)))
        return g.value, c.value

    def sync(self):
        return self._check(self._L.s2l_sync(self._h))

    def kernel_launches(self) -> int:
        return self._L.s2l_kernel_launches(self._h)

    def wait_counts(self) -> dict:
        """Cross-stream waits the runtime inserted (s2l_wait_counts), by kind."""
        w = (C.c_int64 * 4)()
        self._check(self._L.s2l_wait_counts(self._h, w))
        return dict(compute_on_d2h=w[0], compute_on_h2d=w[1], copy_on_compute=w[2], copy_on_copy=w[3])

    def set_timing(self, enable: bool):
        return self._check(self._L.s2l_set_timing(self._h, int(enable)))

    def timing_read(self):
        a, an, b, bn = C.c_double(), C.c_int64(), C.c_double(), C.c_int64()
        self._check(self._L.s2l_timing_read(self._h, C.byref(a), C.byref(an), C.byref(b), C.byref(bn)))
        return dict(attn_ms=a.value, attn_launches=an.value, append_ms=b.value, append_launches=bn.value)


def status_of(fn, *a, **kw) -> int:
    """Runs fn and returns its S2L status code (OK or the S2LError status)."""
    try:
        fn(*a, **kw)
        return OK
    except S2LError as e:
        return e.status
