"""Thin ctypes binding of libleanattn.so (include/la.h).  Argument marshalling only.

Every step of the decode path runs in the library's CUDA kernels; this module converts
torch tensors to raw pointers and the current CUDA stream to a ``cudaStream_t``.  There is
no fallback: if the shared library is missing or a call fails, it raises.

Names follow the C ABI: :func:`la_plan` -> :class:`Plan`, ``Plan.decode`` = ``la_decode``,
``Plan.decode_partial`` = ``la_decode_partial``, :func:`la_combine`, ``Plan.export`` =
``la_plan_export``, ``Plan.info`` = ``la_plan_info_get``, ``Plan.decode_host`` =
``la_decode_host``.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LEANATTN_LIB") or os.path.join(_HERE, "lib", "libleanattn.so")  # env: variant sweeps

LA_OK, LA_ERR_INVALID, LA_ERR_UNSUPPORTED, LA_ERR_CUDA, LA_ERR_NOMEM, LA_ERR_STATE, LA_ERR_TIMEOUT = range(7)
LA_XCHG_HANDLE_BYTES = 64
LA_BF16, LA_FP16, LA_FP32, LA_FP8_E4M3 = 0, 1, 2, 3
LA_KV_BHSD, LA_KV_PACKED, LA_KV_PAGED = 0, 1, 2
LA_SCHED_STREAMK, LA_SCHED_SEQUENTIAL, LA_SCHED_DYNAMIC, LA_SCHED_FIXED_SPLIT, LA_SCHED_AUTO = 0, 1, 2, 3, 4

_DTYPE_CODES = {"bf16": LA_BF16, "fp16": LA_FP16, "fp32": LA_FP32, "fp8": LA_FP8_E4M3}  # fp8: E4M3 K/V, bf16 q
_LAYOUT_CODES = {"bhsd": LA_KV_BHSD, "packed": LA_KV_PACKED, "paged": LA_KV_PAGED}
_SCHED_CODES = {"streamk": LA_SCHED_STREAMK, "sequential": LA_SCHED_SEQUENTIAL, "dynamic": LA_SCHED_DYNAMIC,
                "fixed_split": LA_SCHED_FIXED_SPLIT, "auto": LA_SCHED_AUTO}
SCHEDULE_NAMES = {v: k for k, v in _SCHED_CODES.items()}

# Every symbol include/la.h declares (tests check the library exports all of them).
EXPORTS = ("la_plan_opts_init", "la_plan", "la_plan_update", "la_plan_info_get", "la_plan_export",
           "la_plan_export_claims", "la_decode",
           "la_decode_partial", "la_combine", "la_combine_strided", "la_decode_host", "la_plan_status", "la_plan_destroy",
           "la_launch_count", "la_status_string", "la_last_error", "la_version", "la_plan_trace",
           "la_plan_xchg_handle", "la_plan_xchg_open", "la_plan_xchg_attach", "la_plan_xchg_status",
           "la_plan_set_weights", "la_plan_calibrate")


class LaError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: status {status}: {msg}")
        self.status = status


class la_plan_opts(ctypes.Structure):
    _fields_ = [("scale", ctypes.c_float), ("layout", ctypes.c_int), ("max_ctx", ctypes.c_int64),
                ("grid", ctypes.c_int), ("num_sms", ctypes.c_int), ("ctas_per_sm", ctypes.c_int),
                ("host_only", ctypes.c_int), ("schedule", ctypes.c_int), ("trace", ctypes.c_int),
                ("dyn_first_permille", ctypes.c_int), ("dyn_min_chunk", ctypes.c_int), ("split", ctypes.c_int),
                ("block_table", ctypes.POINTER(ctypes.c_int32)), ("pages_per_seq", ctypes.c_int),
                ("page_size", ctypes.c_int), ("num_pages", ctypes.c_int64), ("q_len", ctypes.c_int),
                ("causal", ctypes.c_int), ("xchg_world", ctypes.c_int), ("xchg_rank", ctypes.c_int),
                ("q_lens", ctypes.POINTER(ctypes.c_int32)), ("k_scale", ctypes.c_float),
                ("v_scale", ctypes.c_float), ("engine", ctypes.c_int), ("stream", ctypes.c_void_p)]


class la_plan_info(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("batch", "heads_q", "heads_kv", "head_dim", "group", "dtype",
                                            "layout", "schedule", "tile_n", "stage_tokens", "grid",
                                            "num_units")] + \
               [(n, ctypes.c_int64) for n in ("total_iters", "num_segments", "num_partials",
                                              "workspace_bytes", "kv_bytes")] + \
               [("scale", ctypes.c_float), ("num_vctas", ctypes.c_int64), ("split", ctypes.c_int),
                ("q_len", ctypes.c_int), ("tile_rows", ctypes.c_int), ("q_rows", ctypes.c_int64),
                ("engine", ctypes.c_int), ("quantization_efficiency", ctypes.c_double),
                ("slot_capacity", ctypes.c_int), ("updates", ctypes.c_int64), ("sm_weighted", ctypes.c_int)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libleanattn.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                           f"g.build()'` (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, f32p = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_float)
    L.la_plan_opts_init.argtypes = [ctypes.POINTER(la_plan_opts)]
    L.la_plan.argtypes = [i32, i32, i32, i32, ctypes.POINTER(ctypes.c_int32), i32, i32,
                          ctypes.POINTER(la_plan_opts), ctypes.POINTER(vp)]
    if hasattr(L, "la_plan_update"):  # (older builds, e.g. LEANATTN_LIB A/B variants, lack these)
        L.la_plan_update.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32), vp]
        L.la_plan_status.argtypes = [vp]
    L.la_plan_info_get.argtypes = [vp, ctypes.POINTER(la_plan_info)]
    L.la_plan_export.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), ctypes.c_size_t,
                                 ctypes.POINTER(ctypes.c_size_t)]
    if hasattr(L, "la_plan_export_claims"):
        L.la_plan_export_claims.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), ctypes.c_size_t,
                                            ctypes.POINTER(ctypes.c_size_t)]
    L.la_decode.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.la_decode_partial.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.la_combine.argtypes = [vp, vp, i32, i32, i32, vp, vp, vp]
    if hasattr(L, "la_combine_strided"):
        L.la_combine_strided.argtypes = [vp, i64, vp, i64, i32, i32, i32, vp, vp, vp]
    L.la_decode_host.argtypes = [vp, vp, vp, vp, i64, vp, vp, vp]
    L.la_plan_trace.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64), ctypes.c_size_t,
                                ctypes.POINTER(ctypes.c_size_t)]
    if hasattr(L, "la_plan_xchg_handle"):  # (older builds, e.g. LEANATTN_LIB bisects, lack it)
        L.la_plan_xchg_handle.argtypes = [vp, ctypes.c_char_p]
        L.la_plan_xchg_open.argtypes = [vp, i32, ctypes.c_char_p]
        L.la_plan_xchg_attach.argtypes = [vp, i32, vp]
        L.la_plan_xchg_status.argtypes = [vp]
    if hasattr(L, "la_plan_set_weights"):
        L.la_plan_set_weights.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), i32, vp]
        L.la_plan_calibrate.argtypes = [vp, vp, vp, vp, vp, vp, i32, i32, vp]
    L.la_plan_destroy.argtypes = [vp]
    L.la_plan_destroy.restype = None
    L.la_launch_count.restype = i64
    L.la_status_string.restype = ctypes.c_char_p
    L.la_last_error.restype = ctypes.c_char_p
    for name in ("la_plan_opts_init", "la_plan", "la_plan_update", "la_plan_status", "la_plan_info_get", "la_plan_export",
                 "la_plan_export_claims", "la_decode",
                 "la_decode_partial", "la_combine", "la_combine_strided", "la_decode_host", "la_plan_trace", "la_plan_xchg_handle",
                 "la_plan_xchg_open", "la_plan_xchg_attach", "la_plan_xchg_status", "la_plan_set_weights",
                 "la_plan_calibrate"):
        if hasattr(L, name):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _check(status: int, where: str):
    if status != LA_OK:
        raise LaError(status, where, lib().la_last_error().decode())


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def launch_count() -> int:
    return int(lib().la_launch_count())


_ENGINE_CODES = {"mma": 0, "tcgen05": 1, "auto": 2}


class Plan:
    """``la_plan``: the stream-K schedule (and, unless host_only, its device state)."""

    def __init__(self, batch: int, heads_q: int, heads_kv: int, head_dim: int, ctx_lens: Sequence[int],
                 tile_n: int = 0, dtype: str = "bf16", scale: float = 0.0, layout: str = "bhsd",
                 max_ctx: int = 0, grid: int = 0, host_only: bool = False, num_sms: int = 148,
                 ctas_per_sm: int = 1, schedule: str = "auto", trace: bool = False,
                 dyn_first_permille: int = 940, dyn_min_chunk: int = 2, split: int = 0,
                 block_table=None, page_size: int = 0, num_pages: int = 0, q_len: int = 1,
                 causal: bool = True, xchg_world: int = 0, xchg_rank: int = 0, q_lens=None,
                 k_scale: float = 0.0, v_scale: float = 0.0, engine: str = "auto", stream=None):
        L = lib()
        opts = la_plan_opts()
        _check(L.la_plan_opts_init(ctypes.byref(opts)), "la_plan_opts_init")
        opts.scale = float(scale)
        opts.layout = _LAYOUT_CODES[layout]
        opts.max_ctx = int(max_ctx)
        opts.grid = int(grid)
        opts.num_sms = int(num_sms)
        opts.ctas_per_sm = int(ctas_per_sm)
        opts.host_only = 1 if host_only else 0
        opts.schedule = _SCHED_CODES[schedule]
        opts.trace = 1 if trace else 0
        opts.dyn_first_permille = int(dyn_first_permille)
        opts.dyn_min_chunk = int(dyn_min_chunk)
        opts.split = int(split)
        if block_table is not None:  # paged layout: [batch][pages_per_seq] int32 (host)
            bt = np.ascontiguousarray(np.asarray(block_table, dtype=np.int32))
            self._bt = bt
            opts.block_table = bt.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            opts.pages_per_seq = int(bt.shape[1])
            opts.page_size = int(page_size)
            opts.num_pages = int(num_pages)
        opts.q_len = int(q_len)
        opts.causal = 1 if causal else 0
        opts.xchg_world = int(xchg_world)
        opts.xchg_rank = int(xchg_rank)
        opts.k_scale = float(k_scale)  # dtype "fp8": K = codes x k_scale, V = codes x v_scale
        opts.v_scale = float(v_scale)
        opts.engine = _ENGINE_CODES[engine]  # "auto", "mma" (mma.sync) or "tcgen05" (T_m > 1 tiles)
        if stream is not None:  # initial table upload left in flight on this stream
            opts.stream = _stream(stream)
        self.engine = engine
        if q_lens is not None:  # heterogeneous batch: N_b per request
            ql = np.ascontiguousarray(np.asarray(q_lens, dtype=np.int32))
            self._ql = ql
            opts.q_lens = ql.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        lens = (ctypes.c_int32 * len(ctx_lens))(*[int(x) for x in ctx_lens])
        h = ctypes.c_void_p()
        self._h = None
        _check(L.la_plan(int(batch), int(heads_q), int(heads_kv), int(head_dim), lens, int(tile_n),
                         _DTYPE_CODES[dtype], ctypes.byref(opts), ctypes.byref(h)), "la_plan")
        self._h = h
        self.dtype = dtype
        self.layout = layout
        self.ctx_lens = [int(x) for x in ctx_lens]
        self.q_lens = None if q_lens is None else [int(x) for x in q_lens]
        self.info = self._info()
        self._kv_rows = self._cache_rows(max_ctx, num_pages, page_size)

    def _cache_rows(self, max_ctx, num_pages, page_size):
        """Rows of one K (or V) cache in this plan's layout (binding-side size checks)."""
        inf = self.info
        if self.layout == "bhsd":
            return inf.batch * inf.heads_kv * (int(max_ctx) or max(self.ctx_lens))
        if self.layout == "packed":
            return inf.heads_kv * sum(self.ctx_lens)
        return int(num_pages) * inf.heads_kv * int(page_size)

    def update(self, ctx_lens: Sequence[int], block_table=None, stream=None):
        """``la_plan_update``: re-plan for new context lengths, one async table upload on
        ``stream`` (the current stream by default); no allocation, graph-replayable."""
        lens = (ctypes.c_int32 * len(ctx_lens))(*[int(x) for x in ctx_lens])
        bt_ptr = None
        if block_table is not None:
            bt = np.ascontiguousarray(np.asarray(block_table, dtype=np.int32))
            self._bt = bt
            bt_ptr = bt.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        strm = None if _is_host_only(self) else _stream(stream)
        _check(lib().la_plan_update(self._h, lens, bt_ptr, strm), "la_plan_update")
        self.ctx_lens = [int(x) for x in ctx_lens]
        if self.layout == "packed":
            self._kv_rows = self.info.heads_kv * sum(self.ctx_lens)
        self.info = self._info()

    def status(self):
        """``la_plan_status``: synchronises; raises LaError(LA_ERR_TIMEOUT) if an in-kernel wait gave up."""
        _check(lib().la_plan_status(self._h), "la_plan_status")

    def _info(self) -> la_plan_info:
        inf = la_plan_info()
        _check(lib().la_plan_info_get(self._h, ctypes.byref(inf)), "la_plan_info_get")
        return inf

    def export(self) -> np.ndarray:
        """``la_plan_export``: (n_segments, 7) int32 rows
        (cta, unit, local_begin, local_end, host, finishing, last_cta)."""
        n = ctypes.c_size_t()
        _check(lib().la_plan_export(self._h, None, 0, ctypes.byref(n)), "la_plan_export")
        buf = np.zeros((n.value, 7), dtype=np.int32)
        _check(lib().la_plan_export(self._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), n.value,
                                    ctypes.byref(n)), "la_plan_export")
        return buf

    def claims(self) -> np.ndarray:
        """``la_plan_export_claims``: claim c runs (virtual) CTA range claims[c]."""
        n = ctypes.c_size_t()
        _check(lib().la_plan_export_claims(self._h, None, 0, ctypes.byref(n)), "la_plan_export_claims")
        buf = np.zeros(n.value, dtype=np.int32)
        _check(lib().la_plan_export_claims(self._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), n.value,
                                           ctypes.byref(n)), "la_plan_export_claims")
        return buf

    def set_weights(self, weights=None, stream=None):
        """``la_plan_set_weights``: per-CTA stream-K weights (int32 in [1, 2^20], one per CTA of
        the launch grid), ranges floor(I * W_<g / W); None restores Eq. 2's equal ranges."""
        if weights is None:
            ptr, n = None, 0
        else:
            w = np.ascontiguousarray(np.asarray(weights, dtype=np.int32))
            self._w = w
            ptr, n = w.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), int(w.size)
        strm = None if _is_host_only(self) else _stream(stream)
        _check(lib().la_plan_set_weights(self._h, ptr, n, strm), "la_plan_set_weights")
        self.info = self._info()

    def calibrate(self, q, k, v, launches: int = 6, rounds: int = 2, stream=None):
        """``la_plan_calibrate``: measure each CTA's streaming rate on (q, k, v) and set
        rate-proportional stream-K weights (synchronises); returns the weights."""
        self._check_inputs(q, k, v)
        out, lse = self._outputs(q, None, None, True)
        _check(lib().la_plan_calibrate(self._h, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), int(launches),
                                       int(rounds), _stream(stream)), "la_plan_calibrate")
        self.info = self._info()
        return self.range_lengths()

    def range_lengths(self) -> np.ndarray:
        """LeanTiles per (virtual) CTA range of the current schedule (weighted or not)."""
        seg = self.export()
        return np.bincount(seg[:, 0], weights=seg[:, 3] - seg[:, 2], minlength=self.info.num_vctas).astype(np.int64)

    TRACE_FIELDS = 7

    def trace(self) -> np.ndarray:
        """``la_plan_trace``: (G, 7) uint64 per-CTA timeline of the last decode
        (smid, t_start, t_publish, t_wait_begin, t_wait_end, t_end, t_stream_end) in ns."""
        n = ctypes.c_size_t()
        _check(lib().la_plan_trace(self._h, None, 0, ctypes.byref(n)), "la_plan_trace")
        buf = np.zeros((n.value, self.TRACE_FIELDS), dtype=np.uint64)
        _check(lib().la_plan_trace(self._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n.value,
                                   ctypes.byref(n)), "la_plan_trace")
        return buf

    def _outputs(self, q, out, lse, need_lse):
        import torch
        B, H, D, nq = self.info.batch, self.info.heads_q, self.info.head_dim, self.info.q_len
        # uniform N_q: (B, H_q[, N_q]); per-request q_lens: (sum_b H_q N_b,) rows, request
        # blocks (H_q, N_b) in order
        rows = (B, H) if nq == 1 else ((B, H, nq) if nq > 1 else (int(self.info.q_rows),))
        if out is None:
            out = torch.empty(rows + (D,), dtype=torch.float32, device=q.device)
        if lse is None and need_lse:
            lse = torch.empty(rows, dtype=torch.float32, device=q.device)
        return out, lse

    _KV_DTYPE = {"bf16": ("bfloat16", 2), "fp16": ("float16", 2), "fp32": ("float32", 4), "fp8": (None, 1)}

    def _check_inputs(self, q, k, v, out=None, lse=None):
        """Marshalling checks only (the C ABI cannot see sizes): dtype, element count and
        device of every tensor against the plan, so no kernel or TMA descriptor can read or
        write outside an allocation."""
        import torch
        inf = self.info
        dev = q.device
        for name, t in (("q", q), ("k", k), ("v", v), ("out", out), ("lse", lse)):
            if t is None:
                continue
            if not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous CUDA tensor")
            if t.device != dev:
                raise ValueError(f"{name} is on {t.device}, q on {dev}")
        qdt = torch.bfloat16 if self.dtype == "fp8" else getattr(torch, self._KV_DTYPE[self.dtype][0])
        if q.dtype != qdt or q.numel() != inf.q_rows * inf.head_dim:
            raise ValueError(f"q must be {qdt} with {inf.q_rows * inf.head_dim} elements")
        kv_bytes = self._kv_rows * inf.head_dim * self._KV_DTYPE[self.dtype][1]
        for name, t in (("k", k), ("v", v)):
            if self.dtype != "fp8" and t.dtype != qdt:
                raise ValueError(f"{name} must be {qdt}")
            if t.element_size() * t.numel() < kv_bytes:
                raise ValueError(f"{name} holds {t.element_size() * t.numel()} bytes < the plan's {kv_bytes}")
        if out is not None and (out.dtype != torch.float32 or out.numel() < inf.q_rows * inf.head_dim):
            raise ValueError(f"out must be float32 with >= {inf.q_rows * inf.head_dim} elements")
        if lse is not None and (lse.dtype != torch.float32 or lse.numel() < inf.q_rows):
            raise ValueError(f"lse must be float32 with >= {inf.q_rows} elements")

    def decode(self, q, k, v, out=None, lse=None, stream=None, want_lse: bool = True):
        """``la_decode``; returns (out fp32 (B, H_q, d), lse fp32 (B, H_q) or None)."""
        out, lse = self._outputs(q, out, lse, want_lse)
        self._check_inputs(q, k, v, out, lse)
        _check(lib().la_decode(self._h, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), _stream(stream)),
               "la_decode")
        return out, lse

    def decode_partial(self, q, k_shard, v_shard, o_part=None, lse_part=None, stream=None):
        """``la_decode_partial`` on one sequence shard; lse is always produced."""
        o_part, lse_part = self._outputs(q, o_part, lse_part, True)
        self._check_inputs(q, k_shard, v_shard, o_part, lse_part)
        _check(lib().la_decode_partial(self._h, _ptr(q), _ptr(k_shard), _ptr(v_shard), _ptr(o_part),
                                       _ptr(lse_part), _stream(stream)), "la_decode_partial")
        return o_part, lse_part

    def decode_host(self, q, k, v, out, lse=None, stream=None):
        """``la_decode_host``: host (ideally pinned) tensors in, host tensors out."""
        rows = k.numel() // self.info.head_dim
        _check(lib().la_decode_host(self._h, _ptr(q), _ptr(k), _ptr(v), int(rows), _ptr(out), _ptr(lse),
                                    _stream(stream)), "la_decode_host")
        return out, lse

    # ---- NEXT-2 fused cross-GPU exchange (plans created with xchg_world = P > 1) ----------
    def xchg_handle(self) -> bytes:
        """``la_plan_xchg_handle``: this rank's exchange-buffer IPC handle (64 bytes)."""
        buf = ctypes.create_string_buffer(LA_XCHG_HANDLE_BYTES)
        _check(lib().la_plan_xchg_handle(self._h, buf), "la_plan_xchg_handle")
        return buf.raw

    def xchg_open(self, peer: int, handle: bytes):
        """``la_plan_xchg_open``: map rank ``peer``'s buffer (another process) from its handle."""
        _check(lib().la_plan_xchg_open(self._h, int(peer), bytes(handle)), "la_plan_xchg_open")

    def xchg_attach(self, peer: int, peer_plan: "Plan"):
        """``la_plan_xchg_attach``: rank ``peer`` is ``peer_plan`` in this process."""
        _check(lib().la_plan_xchg_attach(self._h, int(peer), peer_plan._h), "la_plan_xchg_attach")

    def xchg_status(self):
        """``la_plan_xchg_status``: synchronises; raises LaError(LA_ERR_TIMEOUT) if a wait gave up."""
        _check(lib().la_plan_xchg_status(self._h), "la_plan_xchg_status")

    def close(self):
        if self._h is not None:
            lib().la_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _is_host_only(plan: "Plan") -> bool:
    return plan.info.workspace_bytes == 0


def la_plan(*args, **kw) -> Plan:
    return Plan(*args, **kw)


def la_combine(o_parts, lse_parts, out=None, lse=None, stream=None):
    """``la_combine``: o_parts (P, rows..., d) fp32, lse_parts (P, rows...) fp32 (CUDA)."""
    import torch
    P = o_parts.shape[0]
    d = o_parts.shape[-1]
    rows = lse_parts[0].numel()
    if out is None:
        out = torch.empty(o_parts.shape[1:], dtype=torch.float32, device=o_parts.device)
    if lse is None:
        lse = torch.empty(lse_parts.shape[1:], dtype=torch.float32, device=o_parts.device)
    if not (o_parts.is_contiguous() and lse_parts.is_contiguous()):
        raise ValueError("o_parts / lse_parts must be contiguous")
    _check(lib().la_combine(_ptr(o_parts), _ptr(lse_parts), int(P), int(rows), int(d), _ptr(out), _ptr(lse),
                            _stream(stream)), "la_combine")
    return out, lse


def la_combine_packed(packed, parts: int, rows: int, head_dim: int, out=None, lse=None, stream=None):
    """``la_combine_strided`` over ``packed`` = (parts, rows * (head_dim + 1)) fp32: part p holds
    its O (rows, head_dim) then its L (rows) -- the layout one all-gather of a rank's packed
    (O_r, L_r) produces."""
    import torch
    if not packed.is_contiguous() or packed.numel() != parts * rows * (head_dim + 1):
        raise ValueError("packed must be contiguous (parts, rows * (head_dim + 1)) fp32")
    if out is None:
        out = torch.empty(rows, head_dim, dtype=torch.float32, device=packed.device)
    if lse is None:
        lse = torch.empty(rows, dtype=torch.float32, device=packed.device)
    stride = rows * (head_dim + 1)
    _check(lib().la_combine_strided(_ptr(packed), stride, packed.data_ptr() + rows * head_dim * 4, stride, int(parts),
                                    int(rows), int(head_dim), _ptr(out), _ptr(lse), _stream(stream)),
           "la_combine_strided")
    return out, lse
