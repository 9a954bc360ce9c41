"""ctypes binding of libmessi.so (include/messi.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``csrc/``; this module passes
pointers, sizes and the caller's CUDA stream through the C-ABI and raises on a non-zero
status.  There is no CPU fallback: importing it without the built library raises.

Function names follow the C-ABI (``messi_build``, ``messi_query_ed``, ``messi_query_dtw``,
``messi_free`` and the batch / inspection calls).  ``Index`` is a small convenience owner
around them for torch tensors.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# The in-tree build.  MESSI_LIB may select an alternative build of the same sources for A/B
# kernel experiments (tools/); bench.py refuses to run with it set.
LIB_PATH = os.environ.get("MESSI_LIB") or os.path.join(_HERE, "libmessi.so")

MESSI_OK, MESSI_EINVAL, MESSI_EEMPTY, MESSI_ENOMEM, MESSI_ECUDA = range(5)
_STATUS = {1: "EINVAL", 2: "EEMPTY", 3: "ENOMEM", 4: "ECUDA"}


class MessiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"MESSI_{_STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("length", ctypes.c_int32), ("segments", ctypes.c_int32), ("card_bits", ctypes.c_int32),
                ("window", ctypes.c_int32), ("device", ctypes.c_int32), ("keep_paa", ctypes.c_int32),
                ("row_begin", ctypes.c_int64), ("stream", ctypes.c_void_p)]


class Result(ctypes.Structure):
    _fields_ = [("dist", ctypes.c_double), ("id", ctypes.c_int64), ("d2", ctypes.c_double),
                ("reserved", ctypes.c_int64)]


class Stats(ctypes.Structure):
    _fields_ = [("lb_computed", ctypes.c_int64), ("tiles_scanned", ctypes.c_int64), ("candidates", ctypes.c_int64),
                ("lbk_pass", ctypes.c_int64),
                ("refined", ctypes.c_int64), ("abandoned", ctypes.c_int64), ("near_best", ctypes.c_int64),
                ("dtw_cells", ctypes.c_int64), ("exact", ctypes.c_int64), ("tiles_listed", ctypes.c_int64),
                ("coarse", ctypes.c_int64),
                ("seed_d2", ctypes.c_double), ("bsf_d2", ctypes.c_double), ("rev_paa_pass", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


STATS_FIELDS = [k for k, _ in Stats._fields_]

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.messi_build.argtypes = [vp, i64, ctypes.POINTER(Config), ctypes.POINTER(vp)]
        L.messi_query_ed.argtypes = [vp, vp, ctypes.POINTER(Result), vp]
        L.messi_query_dtw.argtypes = [vp, vp, i32, ctypes.POINTER(Result), vp]
        L.messi_query_ed_batch.argtypes = [vp, vp, i32, vp, vp]
        L.messi_query_dtw_batch.argtypes = [vp, vp, i32, i32, vp, vp]
        L.messi_query_ed_knn.argtypes = [vp, vp, i32, vp, vp]
        L.messi_query_ed_knn_batch.argtypes = [vp, vp, i32, i32, vp, vp]
        L.messi_query_dtw_knn.argtypes = [vp, vp, i32, i32, vp, vp]
        L.messi_query_ed_tc_batch.argtypes = [vp, vp, i32, vp, vp]
        L.messi_query_dtw_knn_batch.argtypes = [vp, vp, i32, i32, i32, vp, vp]
        L.messi_free.argtypes = [vp]
        L.messi_free.restype = None
        L.messi_last_error.restype = ctypes.c_char_p
        L.messi_launch_count.argtypes = [vp]
        L.messi_launch_count.restype = i64
        L.messi_profile_enable.argtypes = [vp, i32]
        L.messi_profile_read.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]
        L.messi_build_times.argtypes = [vp, ctypes.POINTER(ctypes.c_double)]
        L.messi_build_times.restype = ctypes.c_int
        L.messi_debug_scan_repeat.argtypes = [vp, vp, i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]
        L.messi_debug_breakpoints.argtypes = [i32, vp]
        L.messi_debug_summaries.argtypes = [vp, vp, vp]
        L.messi_debug_quantised.argtypes = [vp, vp, vp]
        L.messi_debug_coarse_bounds.argtypes = [vp, vp, i32, vp]
        if hasattr(L, "messi_batch_state_ipc"):  # (MESSI_LIB may name an older build in A/B runs)
            L.messi_batch_state_ipc.argtypes = [vp, i32, vp]
            L.messi_link_peers_ipc.argtypes = [vp, vp, i32]
            L.messi_link_peers_local.argtypes = [vp, ctypes.POINTER(vp), i32]
        L.messi_debug_order.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp)]
        L.messi_debug_lower_bounds.argtypes = [vp, vp, i32, vp]
        if hasattr(L, "messi_debug_rev_bounds"):  # (MESSI_LIB may name an older build in A/B runs)
            L.messi_debug_rev_bounds.argtypes = [vp, vp, i32, vp]
        L.messi_debug_tile_bounds.argtypes = [vp, vp, i32, vp]
        L.messi_debug_distances.argtypes = [vp, vp, i32, vp, i32, vp, vp, vp]
        L.messi_debug_super_bounds.argtypes = [vp, vp, vp]
        L.messi_debug_ed_refine.argtypes = [vp, vp, vp, i32, vp, vp, vp]
        L.messi_debug_dtw_stages.argtypes = [vp, vp, i32, vp, i32, vp, vp, ctypes.POINTER(i32), vp]
        for f in ("messi_build", "messi_query_ed", "messi_query_dtw", "messi_query_ed_batch",
                  "messi_query_dtw_batch", "messi_profile_enable", "messi_profile_read", "messi_debug_breakpoints", "messi_debug_summaries",
                  "messi_debug_order", "messi_debug_lower_bounds", "messi_debug_distances",
                  "messi_debug_scan_repeat", "messi_debug_tile_bounds", "messi_debug_super_bounds",
                  "messi_debug_ed_refine", "messi_debug_dtw_stages", "messi_debug_coarse_bounds",
                  "messi_debug_quantised"):
            getattr(L, f).restype = ctypes.c_int
        if hasattr(L, "messi_debug_rev_bounds"):
            L.messi_debug_rev_bounds.restype = ctypes.c_int
        _lib = L
    return _lib


EXPORTED = ["messi_build", "messi_query_ed", "messi_query_dtw", "messi_query_ed_batch", "messi_query_dtw_batch",
            "messi_free", "messi_last_error", "messi_launch_count", "messi_profile_enable", "messi_profile_read",
            "messi_debug_breakpoints",
            "messi_debug_summaries", "messi_debug_order", "messi_debug_lower_bounds", "messi_debug_rev_bounds", "messi_debug_distances",
            "messi_debug_scan_repeat", "messi_debug_tile_bounds", "messi_debug_quantised",
            "messi_debug_coarse_bounds", "messi_batch_state_ipc", "messi_link_peers_ipc",
            "messi_link_peers_local", "messi_query_ed_knn", "messi_query_ed_knn_batch", "messi_debug_super_bounds",
            "messi_debug_ed_refine", "messi_debug_dtw_stages", "messi_build_times", "messi_query_dtw_knn",
            "messi_query_dtw_knn_batch", "messi_query_ed_tc_batch"]


def _check(status: int):
    if status != MESSI_OK:
        raise MessiError(status, lib().messi_last_error().decode(errors="replace"))


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_handle(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


# ------------------------------------------------------------------ C-ABI, same names
def messi_build(rows_dev: torch.Tensor, *, window: int = 0, keep_paa: bool = False, row_begin: int = 0,
                stream=None, segments: int = 16, card_bits: int = 8, length: int | None = None):
    """Build over a [count, n] float32 CUDA tensor (borrowed: keep it alive); returns a handle."""
    if not (rows_dev.is_cuda and rows_dev.dtype == torch.float32 and rows_dev.is_contiguous()):
        raise MessiError(MESSI_EINVAL, "rows must be a contiguous float32 CUDA tensor")
    count = rows_dev.shape[0] if rows_dev.dim() == 2 else 0
    n = length if length is not None else (rows_dev.shape[1] if rows_dev.dim() == 2 else 0)
    cfg = Config(length=n, segments=segments, card_bits=card_bits, window=window,
                 device=rows_dev.device.index or 0, keep_paa=int(keep_paa), row_begin=row_begin,
                 stream=_stream_handle(stream))
    h = ctypes.c_void_p()
    _check(lib().messi_build(_ptr(rows_dev) if rows_dev.numel() else None, count, ctypes.byref(cfg), ctypes.byref(h)))
    return h


def messi_query_ed(handle, query, with_stats: bool = False):
    """query: host (numpy / CPU tensor) or CUDA tensor of n float32.  Returns (dist, id, d2[, stats])."""
    q, keep = _query_ptr(query)
    res, st = Result(), Stats()
    _check(lib().messi_query_ed(handle, q, ctypes.byref(res), ctypes.byref(st) if with_stats else None))
    return (res.dist, res.id, res.d2, st.as_dict()) if with_stats else (res.dist, res.id, res.d2)


def messi_query_dtw(handle, query, reach: int, with_stats: bool = False):
    q, keep = _query_ptr(query)
    res, st = Result(), Stats()
    _check(lib().messi_query_dtw(handle, q, int(reach), ctypes.byref(res), ctypes.byref(st) if with_stats else None))
    return (res.dist, res.id, res.d2, st.as_dict()) if with_stats else (res.dist, res.id, res.d2)


def _check_batch(queries_dev, results_dev, stats_dev, per_query_results=1, n=None):
    """Argument checks of the batch calls (the C-ABI takes raw pointers and counts): float32,
    contiguous, CUDA, [nq, n] queries; result / stats buffers on the same device, contiguous,
    large enough for nq * per_query_results records / nq stats."""
    def bad(msg):
        raise MessiError(MESSI_EINVAL, msg)
    if not isinstance(queries_dev, torch.Tensor) or not queries_dev.is_cuda:
        bad("queries must be a CUDA tensor")
    if queries_dev.dtype != torch.float32 or not queries_dev.is_contiguous() or queries_dev.dim() != 2:
        bad("queries must be a contiguous float32 [nq, n] tensor")
    if n is not None and queries_dev.shape[1] != n:
        bad(f"queries have length {queries_dev.shape[1]}, the index {n}")
    nq = queries_dev.shape[0]
    for name, buf, need in (("results", results_dev, nq * per_query_results * RESULT_BYTES),
                            ("stats", stats_dev, nq * STATS_BYTES)):
        if buf is None:
            if name == "results":
                bad("results buffer is required")
            continue
        if not buf.is_cuda or buf.device != queries_dev.device or not buf.is_contiguous():
            bad(f"{name} must be a contiguous tensor on {queries_dev.device}")
        if buf.numel() * buf.element_size() < need:
            bad(f"{name} buffer holds {buf.numel() * buf.element_size()} bytes, needs {need}")
    return nq


def messi_query_ed_batch(handle, queries_dev: torch.Tensor, results_dev: torch.Tensor, stats_dev=None, n=None):
    """Asynchronous on the build stream.  results_dev: uint8 CUDA tensor of nq*32 bytes (see
    ``result_buffer``); stats_dev: optional nq*112 bytes (``stats_buffer``)."""
    nq = _check_batch(queries_dev, results_dev, stats_dev, 1, n)
    _check(lib().messi_query_ed_batch(handle, _ptr(queries_dev), nq, _ptr(results_dev), _ptr(stats_dev)))


def messi_query_dtw_batch(handle, queries_dev: torch.Tensor, reach: int, results_dev: torch.Tensor, stats_dev=None,
                          n=None):
    nq = _check_batch(queries_dev, results_dev, stats_dev, 1, n)
    _check(lib().messi_query_dtw_batch(handle, _ptr(queries_dev), nq, int(reach), _ptr(results_dev), _ptr(stats_dev)))


def messi_batch_state_ipc(handle, set_index: int) -> bytes:
    """The 64-byte CUDA IPC handle of the index's state array `set_index` (0/1: the batched
    ED path's two query sets, 2: the DTW slots)."""
    buf = ctypes.create_string_buffer(64)
    _check(lib().messi_batch_state_ipc(handle, int(set_index), buf))
    return buf.raw


def messi_link_peers_ipc(handle, peer_handles):
    """peer_handles: list over peers of (set-0, set-1, set-2 handle) byte strings."""
    blob = b"".join(b"".join(h) for h in peer_handles)
    buf = ctypes.create_string_buffer(blob, len(blob)) if blob else None
    _check(lib().messi_link_peers_ipc(handle, buf, len(peer_handles)))


def messi_link_peers_local(handle, peer_handles_list):
    arr = (ctypes.c_void_p * max(1, len(peer_handles_list)))(*[h.value for h in peer_handles_list])
    _check(lib().messi_link_peers_local(handle, arr, len(peer_handles_list)))


def messi_query_ed_knn(handle, query, k: int, with_stats: bool = False):
    """Exact k-NN (ED) of one query: (dist float64[k], id int64[k], d2 float64[k][, stats])."""
    import numpy as np
    q, keep = _query_ptr(query)
    res = (Result * k)()
    st = Stats()
    _check(lib().messi_query_ed_knn(handle, q, int(k), res, ctypes.byref(st) if with_stats else None))
    dist = np.array([r.dist for r in res]); ids = np.array([r.id for r in res], dtype=np.int64)
    d2 = np.array([r.d2 for r in res])
    return (dist, ids, d2, st.as_dict()) if with_stats else (dist, ids, d2)


def messi_query_ed_tc_batch(handle, queries_dev: torch.Tensor, results_dev: torch.Tensor, stats_dev=None, n=None):
    """Exact 1-NN (ED) of nq queries by the tensor-core pass (n = 128 or 256); asynchronous like the batch call."""
    nq = _check_batch(queries_dev, results_dev, stats_dev, 1, n)
    _check(lib().messi_query_ed_tc_batch(handle, _ptr(queries_dev), nq, _ptr(results_dev), _ptr(stats_dev)))


def messi_query_dtw_knn(handle, query, reach: int, k: int, with_stats: bool = False):
    """Exact k-NN (DTW, reach points) of one query: (dist float64[k], id int64[k], d2 float64[k][, stats])."""
    import numpy as np
    q, keep = _query_ptr(query)
    res = (Result * k)()
    st = Stats()
    _check(lib().messi_query_dtw_knn(handle, q, int(reach), int(k), res, ctypes.byref(st) if with_stats else None))
    dist = np.array([r.dist for r in res]); ids = np.array([r.id for r in res], dtype=np.int64)
    d2 = np.array([r.d2 for r in res])
    return (dist, ids, d2, st.as_dict()) if with_stats else (dist, ids, d2)


def messi_query_dtw_knn_batch(handle, queries_dev: torch.Tensor, reach: int, k: int, results_dev: torch.Tensor,
                              stats_dev=None, n=None):
    """results_dev: uint8 CUDA tensor of nq*k*32 bytes (result_buffer(nq * k))."""
    nq = _check_batch(queries_dev, results_dev, stats_dev, max(1, int(k)), n)
    _check(lib().messi_query_dtw_knn_batch(handle, _ptr(queries_dev), nq, int(reach), int(k), _ptr(results_dev),
                                           _ptr(stats_dev)))


def messi_query_ed_knn_batch(handle, queries_dev: torch.Tensor, k: int, results_dev: torch.Tensor, stats_dev=None,
                             n=None):
    """results_dev: uint8 CUDA tensor of nq*k*32 bytes (result_buffer(nq * k))."""
    nq = _check_batch(queries_dev, results_dev, stats_dev, max(1, int(k)), n)
    _check(lib().messi_query_ed_knn_batch(handle, _ptr(queries_dev), nq, int(k), _ptr(results_dev), _ptr(stats_dev)))


def messi_free(handle):
    if handle:
        lib().messi_free(handle)


def messi_launch_count(handle) -> int:
    return int(lib().messi_launch_count(handle))


KERNEL_KINDS = {"seed": 0, "scan": 1, "refine": 2, "lbk": 3, "resolve": 4}


def messi_profile_enable(handle, enable: bool = True, serial: bool = False):
    """enable: per-kernel CUDA-event timing; serial: every per-query stage on the index stream."""
    _check(lib().messi_profile_enable(handle, int(bool(enable)) | (2 if serial else 0)))


def messi_build_times(handle):
    """Device ms of the build phases: summarise, key sort, layout, quantise; renv = the last
    DTW reverse-envelope symbol pass (per reach, built on the first strip-reach DTW query)."""
    out = (ctypes.c_double * 5)()
    _check(lib().messi_build_times(handle, out))
    return {"summarise": out[0], "sort": out[1], "layout": out[2], "quantise": out[3], "renv": out[4]}


def messi_profile_read(handle, kind):
    """(total milliseconds, launches) of one kernel kind since messi_profile_enable."""
    ms, cnt = ctypes.c_double(), ctypes.c_int64()
    k = KERNEL_KINDS[kind] if isinstance(kind, str) else int(kind)
    _check(lib().messi_profile_read(handle, k, ctypes.byref(ms), ctypes.byref(cnt)))
    return ms.value, cnt.value


def messi_debug_scan_repeat(handle, query_dev: torch.Tensor, reps: int):
    """(summed ms of `reps` isolated scans, candidates, tiles scanned)."""
    ms, c = ctypes.c_double(), ctypes.c_int64()
    _check(lib().messi_debug_scan_repeat(handle, _ptr(query_dev), int(reps), ctypes.byref(ms), ctypes.byref(c)))
    return ms.value, c.value & 0xFFFFFFFF, c.value >> 32


def messi_debug_breakpoints(device: int = 0):
    import numpy as np
    out = np.zeros(255, np.float32)
    _check(lib().messi_debug_breakpoints(device, out.ctypes.data_as(ctypes.c_void_p)))
    return out


def messi_debug_summaries(handle, count: int, device, with_paa: bool = False):
    sym = torch.empty((count, 16), dtype=torch.uint8, device=device)
    paa = torch.empty((count, 16), dtype=torch.float32, device=device) if with_paa else None
    _check(lib().messi_debug_summaries(handle, _ptr(sym), _ptr(paa)))
    return sym, paa


def messi_debug_quantised(handle, count: int, n: int, device):
    """(q8 [count, n] int8 c stored in a uint8 tensor (view as int8), meta float32 [count, 2] =
    {scale, error bound}), row order."""
    q8 = torch.empty((count, n), dtype=torch.uint8, device=device)
    meta = torch.empty((count, 2), dtype=torch.float32, device=device)
    _check(lib().messi_debug_quantised(handle, _ptr(q8), _ptr(meta)))
    return q8, meta


def messi_debug_order(handle, count: int, device):
    """(sorted keys as int64 view, permutation) copied into torch tensors."""
    k, p = ctypes.c_void_p(), ctypes.c_void_p()
    _check(lib().messi_debug_order(handle, ctypes.byref(k), ctypes.byref(p)))
    keys = torch.empty(count, dtype=torch.int64, device=device)
    perm = torch.empty(count, dtype=torch.int32, device=device)
    torch.cuda.synchronize(device)
    keys.copy_(_wrap_dev(k.value, count * 8, device).view(torch.int64))
    perm.copy_(_wrap_dev(p.value, count * 4, device).view(torch.int32))
    return keys, perm


def messi_debug_lower_bounds(handle, query_dev: torch.Tensor, reach: int, count: int):
    lb = torch.empty(count, dtype=torch.float32, device=query_dev.device)
    _check(lib().messi_debug_lower_bounds(handle, _ptr(query_dev), int(reach), _ptr(lb)))
    return lb


def messi_debug_rev_bounds(handle, query_dev: torch.Tensor, reach: int, count: int):
    """The DTW path's reverse envelope-PAA bound of every row (row order) for reach >= 1."""
    lb = torch.empty(count, dtype=torch.float32, device=query_dev.device)
    _check(lib().messi_debug_rev_bounds(handle, _ptr(query_dev), int(reach), _ptr(lb)))
    return lb


def messi_debug_coarse_bounds(handle, query_dev: torch.Tensor, reach: int, count: int):
    lb = torch.empty(count, dtype=torch.float32, device=query_dev.device)
    _check(lib().messi_debug_coarse_bounds(handle, _ptr(query_dev), int(reach), _ptr(lb)))
    return lb


def messi_debug_tile_bounds(handle, query_dev: torch.Tensor, reach: int, ntiles: int):
    lb = torch.empty(ntiles, dtype=torch.float32, device=query_dev.device)
    _check(lib().messi_debug_tile_bounds(handle, _ptr(query_dev), int(reach), _ptr(lb)))
    return lb


def messi_debug_super_bounds(handle, query_dev: torch.Tensor, nsuper: int):
    lb = torch.empty(nsuper, dtype=torch.float32, device=query_dev.device)
    _check(lib().messi_debug_super_bounds(handle, _ptr(query_dev), _ptr(lb)))
    return lb


def messi_debug_ed_refine(handle, query_dev: torch.Tensor, ids_dev: torch.Tensor):
    """(dh2 float64 [k], L float64 [k], d32 float32 [k], d64 float64 [k]) of the ED refine's device code."""
    ids = ids_dev.to(torch.int32).contiguous()
    k = ids.numel()
    dev = query_dev.device
    q8 = torch.empty((k, 2), dtype=torch.float64, device=dev)
    d32 = torch.empty(k, dtype=torch.float32, device=dev)
    d64 = torch.empty(k, dtype=torch.float64, device=dev)
    _check(lib().messi_debug_ed_refine(handle, _ptr(query_dev), _ptr(ids), k, _ptr(q8), _ptr(d32), _ptr(d64)))
    return q8[:, 0], q8[:, 1], d32, d64


def messi_debug_dtw_stages(handle, query_dev: torch.Tensor, reach: int, ids_dev: torch.Tensor, rev: bool = False):
    """(lbk float32 [k], d32 float32 [k], quantised: bool) of the DTW filter and refine kernels;
    with rev=True also the filter's reverse LB_Keogh bound (float32 [k], NaN where the filter
    computes none)."""
    ids = ids_dev.to(torch.int32).contiguous()
    k = ids.numel()
    lbk = torch.empty(k, dtype=torch.float32, device=query_dev.device)
    d32 = torch.empty(k, dtype=torch.float32, device=query_dev.device)
    lbr = torch.empty(k, dtype=torch.float32, device=query_dev.device) if rev else None
    qz = ctypes.c_int32()
    _check(lib().messi_debug_dtw_stages(handle, _ptr(query_dev), int(reach), _ptr(ids), k, _ptr(lbk), _ptr(d32),
                                        ctypes.byref(qz), _ptr(lbr) if rev else None))
    return (lbk, d32, bool(qz.value), lbr) if rev else (lbk, d32, bool(qz.value))


def messi_debug_distances(handle, query_dev: torch.Tensor, reach: int, ids_dev: torch.Tensor):
    k = ids_dev.numel()
    dev = query_dev.device
    d32 = torch.empty(k, dtype=torch.float32, device=dev)
    d64 = torch.empty(k, dtype=torch.float64, device=dev)
    lbk = torch.empty(k, dtype=torch.float32, device=dev) if reach >= 0 else None
    ids = ids_dev.to(torch.int32).contiguous()
    _check(lib().messi_debug_distances(handle, _ptr(query_dev), int(reach), _ptr(ids), k, _ptr(d32), _ptr(d64),
                                       _ptr(lbk)))
    return d32, d64, lbk


# ----------------------------------------------------------------------------- helpers
def _query_ptr(query):
    import numpy as np
    if isinstance(query, torch.Tensor):
        if query.is_cuda:
            q = query.contiguous().to(torch.float32)
            return ctypes.c_void_p(q.data_ptr()), q
        query = query.numpy()
    q = np.ascontiguousarray(query, dtype=np.float32)
    return q.ctypes.data_as(ctypes.c_void_p), q


def _wrap_dev(ptr: int, nbytes: int, device):
    """A uint8 CUDA tensor viewing library-owned device memory (no copy, not owned)."""
    class _Arr:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                    "strides": None}
    return torch.as_tensor(_Arr(), device=device)


RESULT_BYTES, STATS_BYTES = 32, 112


def result_buffer(nq: int, device) -> torch.Tensor:
    return torch.empty(nq * RESULT_BYTES, dtype=torch.uint8, device=device)


def stats_buffer(nq: int, device) -> torch.Tensor:
    return torch.empty(nq * STATS_BYTES, dtype=torch.uint8, device=device)


def decode_results(buf: torch.Tensor):
    """(dist float64[nq], id int64[nq], d2 float64[nq]) from a result buffer (copied to host)."""
    raw = buf.view(-1, RESULT_BYTES).cpu()
    return (raw[:, 0:8].contiguous().view(torch.float64).flatten(), raw[:, 8:16].contiguous().view(torch.int64).flatten(),
            raw[:, 16:24].contiguous().view(torch.float64).flatten())


def decode_results_device(buf: torch.Tensor):
    """(dist, id, d2) views of a result buffer, kept on the device (for the NCCL merge)."""
    raw = buf.view(-1, RESULT_BYTES)
    return (raw[:, 0:8].contiguous().view(torch.float64).flatten(), raw[:, 8:16].contiguous().view(torch.int64).flatten(),
            raw[:, 16:24].contiguous().view(torch.float64).flatten())


def decode_stats(buf: torch.Tensor):
    raw = buf.view(-1, STATS_BYTES).cpu()
    ints = raw[:, :88].contiguous().view(torch.int64)       # lb_computed .. coarse
    dbl = raw[:, 88:104].contiguous().view(torch.float64)   # seed_d2, bsf_d2
    tail = raw[:, 104:].contiguous().view(torch.int64)      # rev_paa_pass
    return [dict(zip(STATS_FIELDS, list(map(int, i.tolist())) + list(map(float, d.tolist())) + list(map(int, t.tolist()))))
            for i, d, t in zip(ints, dbl, tail)]


class Index:
    """Owner of one messi index over a [count, n] float32 CUDA tensor (kept alive here)."""

    def __init__(self, rows: torch.Tensor, *, window: int = 0, keep_paa: bool = False, row_begin: int = 0,
                 stream=None):
        self.rows = rows
        self.count, self.n = rows.shape
        self.device = rows.device
        self.row_begin = row_begin
        self.stream = stream if stream is not None else torch.cuda.current_stream(rows.device)
        self.handle = messi_build(rows, window=window, keep_paa=keep_paa, row_begin=row_begin, stream=self.stream)

    def query_ed(self, q, with_stats=False):
        return messi_query_ed(self.handle, q, with_stats)

    def query_dtw(self, q, reach, with_stats=False):
        return messi_query_dtw(self.handle, q, reach, with_stats)

    def query_batch(self, queries_dev: torch.Tensor, reach: int | None = None, results=None, stats=None):
        """Enqueue nq queries (ED if reach is None) on the index stream; returns the buffers."""
        nq = queries_dev.shape[0]
        results = results if results is not None else result_buffer(nq, self.device)
        if reach is None:
            messi_query_ed_batch(self.handle, queries_dev, results, stats, n=self.n)
        else:
            messi_query_dtw_batch(self.handle, queries_dev, reach, results, stats, n=self.n)
        return results, stats

    def query_knn(self, q, k: int, with_stats=False):
        return messi_query_ed_knn(self.handle, q, k, with_stats)

    def query_batch_knn(self, queries_dev: torch.Tensor, k: int, results=None, stats=None, reach: int | None = None):
        """Enqueue nq exact k-NN queries (ED, or DTW with `reach`); results: nq*k entries
        (decode_results -> [nq*k])."""
        nq = queries_dev.shape[0]
        results = results if results is not None else result_buffer(nq * k, self.device)
        if reach is None:
            messi_query_ed_knn_batch(self.handle, queries_dev, k, results, stats, n=self.n)
        else:
            messi_query_dtw_knn_batch(self.handle, queries_dev, reach, k, results, stats, n=self.n)
        return results, stats

    def query_batch_tc(self, queries_dev: torch.Tensor, results=None, stats=None):
        """Enqueue nq exact 1-NN (ED) queries on the tensor-core path."""
        nq = queries_dev.shape[0]
        results = results if results is not None else result_buffer(nq, self.device)
        messi_query_ed_tc_batch(self.handle, queries_dev, results, stats, n=self.n)
        return results, stats

    def query_dtw_knn(self, q, reach: int, k: int, with_stats=False):
        return messi_query_dtw_knn(self.handle, q, reach, k, with_stats)

    def launches(self) -> int:
        return messi_launch_count(self.handle)

    def close(self):
        if self.handle:
            messi_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
