"""CPU oracle for the MESSI exact 1-NN hot path (arXiv 2110.07519).

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product
path (``paper_2110_07519_b200``) never imports it and shares no code with it.

Thin ctypes marshalling over ``messi_oracle.c`` (plain serial fp64 C, compiled with
``-O2 -ffp-contract=off``, no fast-math).  Every arithmetic step lives in the C file,
which cites the PAPER.md passages it follows.  ``nn_*_parallel`` only splits rows into
chunks, runs one serial oracle call per chunk on a thread pool and merges the chunk
minima lexicographically on (d2, id) -- the result is independent of the thread count.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "messi_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_c_int, _c_i64, _c_d = ctypes.c_int, ctypes.c_int64, ctypes.c_double


def build(force: bool = False) -> str:
    """Compile liboracle.so with the flags the header requires (no FMA, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.oracle_inv_phi.argtypes = [_c_d]
        L.oracle_inv_phi.restype = _c_d
        L.oracle_breakpoints.argtypes = [_c_int, _f64p, _f32p]
        L.oracle_breakpoints.restype = _c_int
        L.oracle_paa32.argtypes = [_f32p, _c_int, _c_int, _f32p]
        L.oracle_paa32.restype = _c_int
        L.oracle_paa64.argtypes = [_f32p, _c_int, _c_int, _f64p]
        L.oracle_paa64.restype = _c_int
        L.oracle_symbol.argtypes = [ctypes.c_float, _f32p, _c_int]
        L.oracle_symbol.restype = _c_int
        L.oracle_isax.argtypes = [_f32p, _c_int, _c_int, _f32p, _c_int, _f32p, _u8p]
        L.oracle_isax.restype = _c_int
        L.oracle_isax_rows.argtypes = [_f32p, _c_i64, _c_int, _c_int, _f32p, _c_int, _f32p, _u8p]
        L.oracle_isax_rows.restype = _c_int
        L.oracle_mindist2.argtypes = [_f64p, _u8p, _c_int, _c_int, _f32p, _c_int]
        L.oracle_mindist2.restype = _c_d
        L.oracle_ed2.argtypes = [_f32p, _f32p, _c_int]
        L.oracle_ed2.restype = _c_d
        L.oracle_envelope.argtypes = [_f32p, _c_int, _c_int, _f32p, _f32p]
        L.oracle_envelope.restype = _c_int
        L.oracle_lb_keogh2.argtypes = [_f32p, _f32p, _f32p, _c_int]
        L.oracle_lb_keogh2.restype = _c_d
        L.oracle_lb_env_paa2.argtypes = [_f64p, _f64p, _u8p, _c_int, _c_int, _f32p, _c_int]
        L.oracle_lb_env_paa2.restype = _c_d
        L.oracle_renv_sym.argtypes = [_f32p, _c_int, _c_int, _c_int, _f32p, _c_int, _u8p, _u8p]
        L.oracle_renv_sym.restype = _c_int
        L.oracle_renv_sym_rows.argtypes = [_f32p, _c_i64, _c_int, _c_int, _c_int, _f32p, _c_int, _u8p, _u8p]
        L.oracle_renv_sym_rows.restype = _c_int
        L.oracle_lb_rev_paa2.argtypes = [_f64p, _u8p, _u8p, _c_int, _c_int, _f32p, _c_int]
        L.oracle_lb_rev_paa2.restype = _c_d
        L.oracle_lb_rev_paa2_rows.argtypes = [_f64p, _u8p, _u8p, _c_i64, _c_int, _c_int, _f32p, _c_int, _f64p]
        L.oracle_lb_rev_paa2_rows.restype = None
        L.oracle_dtw2.argtypes = [_f32p, _f32p, _c_int, _c_int]
        L.oracle_dtw2.restype = _c_d
        vp = ctypes.c_void_p
        L.oracle_nn_ed_multi.argtypes = [vp, _c_i64, _c_int, _f32p, _c_int, _c_i64, vp, vp]
        L.oracle_nn_ed_multi.restype = None
        L.oracle_nn_dtw_multi.argtypes = [vp, _c_i64, _c_int, _f32p, _c_int, _c_int, _c_i64, vp, vp]
        L.oracle_nn_dtw_multi.restype = None
        L.oracle_ed2_rows.argtypes = [_f32p, _c_i64, _c_int, _f32p, _f64p]
        L.oracle_ed2_rows.restype = None
        L.oracle_dtw2_rows.argtypes = [_f32p, _c_i64, _c_int, _f32p, _c_int, _f64p]
        L.oracle_dtw2_rows.restype = None
        _lib = L
    return _lib


def _f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


# ------------------------------------------------------------------ single steps
def inv_phi(p: float) -> float:
    return lib().oracle_inv_phi(float(p))


def breakpoints(card: int = 256):
    """(beta64, beta32): the card-1 N(0,1) breakpoints (O3)."""
    b64 = np.zeros(card - 1, np.float64)
    b32 = np.zeros(card - 1, np.float32)
    if lib().oracle_breakpoints(card, b64, b32):
        raise ValueError("cardinality must be a power of two in [2, 256]")
    return b64, b32


def paa32(x, w: int = 16):
    x = _f32(x)
    out = np.zeros(w, np.float32)
    if lib().oracle_paa32(x, x.size, w, out):
        raise ValueError("need 0 < w <= n and n % w == 0")
    return out


def paa64(x, w: int = 16):
    x = _f32(x)
    out = np.zeros(w, np.float64)
    if lib().oracle_paa64(x, x.size, w, out):
        raise ValueError("need 0 < w <= n and n % w == 0")
    return out


def symbol(v: float, beta32, card: int = 256) -> int:
    return lib().oracle_symbol(float(np.float32(v)), _f32(beta32), card)


def isax(x, w: int = 16, card: int = 256, beta32=None):
    """(paa32, sym) of one series (O2 + O4)."""
    x = _f32(x)
    if beta32 is None:
        beta32 = breakpoints(card)[1]
    p = np.zeros(w, np.float32)
    s = np.zeros(w, np.uint8)
    if lib().oracle_isax(x, x.size, w, _f32(beta32), card, p, s):
        raise ValueError("need 0 < w <= n and n % w == 0")
    return p, s


def isax_rows(data, w: int = 16, card: int = 256):
    """(paa32[rows, w], sym[rows, w]) of every row (O2 + O4)."""
    data = _f32(data)
    beta32 = breakpoints(card)[1]
    P = np.zeros((data.shape[0], w), np.float32)
    S = np.zeros((data.shape[0], w), np.uint8)
    if lib().oracle_isax_rows(data, data.shape[0], data.shape[1], w, _f32(beta32), card, P, S):
        raise ValueError("need 0 < w <= n and n % w == 0")
    return P, S


def mindist2(qpaa64, sym, n: int, card: int = 256, beta32=None) -> float:
    sym = np.ascontiguousarray(sym, np.uint8)
    if beta32 is None:
        beta32 = breakpoints(card)[1]
    q = np.ascontiguousarray(qpaa64, np.float64)
    return lib().oracle_mindist2(q, sym, sym.size, n, _f32(beta32), card)


def ed2(a, b) -> float:
    a, b = _f32(a), _f32(b)
    assert a.size == b.size
    return lib().oracle_ed2(a, b, a.size)


def envelope(q, r: int):
    q = _f32(q)
    U = np.zeros_like(q)
    L = np.zeros_like(q)
    if lib().oracle_envelope(q, q.size, r, U, L):
        raise ValueError("reach out of range")
    return U, L


def lb_keogh2(U, L, c) -> float:
    U, L, c = _f32(U), _f32(L), _f32(c)
    return lib().oracle_lb_keogh2(U, L, c, c.size)


def lb_env_paa2(Upaa64, Lpaa64, sym, n: int, card: int = 256, beta32=None) -> float:
    sym = np.ascontiguousarray(sym, np.uint8)
    if beta32 is None:
        beta32 = breakpoints(card)[1]
    return lib().oracle_lb_env_paa2(np.ascontiguousarray(Upaa64, np.float64),
                                    np.ascontiguousarray(Lpaa64, np.float64), sym, sym.size, n,
                                    _f32(beta32), card)


def renv_sym(x, r: int, w: int = 16, card: int = 256, beta32=None):
    """(usym, lsym): symbols of the per-segment means of x's envelope of reach r (O11b)."""
    x = _f32(x)
    if beta32 is None:
        beta32 = breakpoints(card)[1]
    u = np.zeros(w, np.uint8)
    l = np.zeros(w, np.uint8)
    if lib().oracle_renv_sym(x, x.size, int(r), w, _f32(beta32), card, u, l):
        raise ValueError("need 0 < w, n % w == 0, 0 <= r <= n")
    return u, l


def renv_sym_rows(data, r: int, w: int = 16, card: int = 256):
    data = _f32(data)
    beta32 = breakpoints(card)[1]
    U = np.zeros((data.shape[0], w), np.uint8)
    L = np.zeros((data.shape[0], w), np.uint8)
    if lib().oracle_renv_sym_rows(data, data.shape[0], data.shape[1], int(r), w, _f32(beta32), card, U, L):
        raise ValueError("need 0 < w, n % w == 0, 0 <= r <= n")
    return U, L


def lb_rev_paa2(qpaa64, usym, lsym, n: int, card: int = 256, beta32=None) -> float:
    """Reverse envelope-PAA bound (O11b) of one row from its envelope symbols."""
    usym = np.ascontiguousarray(usym, np.uint8)
    lsym = np.ascontiguousarray(lsym, np.uint8)
    if beta32 is None:
        beta32 = breakpoints(card)[1]
    return lib().oracle_lb_rev_paa2(np.ascontiguousarray(qpaa64, np.float64), usym, lsym, usym.size, n,
                                    _f32(beta32), card)


def lb_rev_paa2_rows(qpaa64, usym, lsym, n: int, card: int = 256):
    usym = np.ascontiguousarray(usym, np.uint8)
    lsym = np.ascontiguousarray(lsym, np.uint8)
    out = np.zeros(usym.shape[0], np.float64)
    lib().oracle_lb_rev_paa2_rows(np.ascontiguousarray(qpaa64, np.float64), usym, lsym, usym.shape[0],
                                  usym.shape[1], n, _f32(breakpoints(card)[1]), card, out)
    return out


def dtw2(q, c, r: int) -> float:
    q, c = _f32(q), _f32(c)
    assert q.size == c.size
    return lib().oracle_dtw2(q, c, q.size, int(r))


def ed2_rows(data, q):
    data, q = _f32(data), _f32(q)
    out = np.zeros(data.shape[0], np.float64)
    lib().oracle_ed2_rows(data, data.shape[0], data.shape[1], q, out)
    return out


def dtw2_rows(data, q, r: int):
    data, q = _f32(data), _f32(q)
    out = np.zeros(data.shape[0], np.float64)
    lib().oracle_dtw2_rows(data, data.shape[0], data.shape[1], q, int(r), out)
    return out


# ------------------------------------------------------------------------ 1-NN
def _nn_chunk(kind, data, queries, r, row_begin):
    nq, n = queries.shape
    d2 = np.full(nq, np.inf, np.float64)
    ids = np.full(nq, -1, np.int64)
    L = lib()
    dp = data.ctypes.data_as(ctypes.c_void_p)
    if kind == "ed":
        L.oracle_nn_ed_multi(dp, data.shape[0], n, queries, nq, row_begin,
                             d2.ctypes.data_as(ctypes.c_void_p), ids.ctypes.data_as(ctypes.c_void_p))
    else:
        L.oracle_nn_dtw_multi(dp, data.shape[0], n, queries, nq, int(r), row_begin,
                              d2.ctypes.data_as(ctypes.c_void_p), ids.ctypes.data_as(ctypes.c_void_p))
    return d2, ids


def merge(d2a, ida, d2b, idb):
    """Lexicographic (d2, id) min of two result sets (ties -> lowest id)."""
    take_b = (d2b < d2a) | ((d2b == d2a) & (idb < ida) & (idb >= 0)) | (ida < 0)
    return np.where(take_b, d2b, d2a), np.where(take_b, idb, ida)


def nn(kind: str, data, queries, r: int = 0, row_begin: int = 0, threads: int | None = None,
       chunk: int = 1 << 15):
    """Exact 1-NN of every query over every row (O8 / O13): returns (d2[nq], id[nq])."""
    data = _f32(data)
    queries = _f32(queries).reshape(-1, data.shape[1])
    rows = data.shape[0]
    threads = threads or len(os.sched_getaffinity(0))
    starts = list(range(0, rows, chunk)) or [0]
    d2 = np.full(queries.shape[0], np.inf)
    ids = np.full(queries.shape[0], -1, np.int64)
    if threads <= 1 or len(starts) == 1:
        parts = [_nn_chunk(kind, data[s:s + chunk], queries, r, row_begin + s) for s in starts]
    else:
        with ThreadPoolExecutor(threads) as ex:
            parts = list(ex.map(lambda s: _nn_chunk(kind, data[s:s + chunk], queries, r,
                                                    row_begin + s), starts))
    for pd, pi in parts:
        d2, ids = merge(d2, ids, pd, pi)
    return d2, ids


def knn(kind: str, data, queries, k: int, r: int = 0, row_begin: int = 0):
    """Exact k-NN by the plain definition: every row's distance by the C
    oracle (ed2_rows / dtw2_rows: fp64, sequential), then the k lexicographically smallest
    (d2, id) per query (ties -> lowest id).  Returns d2 [nq, k], ids [nq, k] (-1 past N)."""
    data = np.ascontiguousarray(data, dtype=np.float32)
    queries = np.atleast_2d(np.ascontiguousarray(queries, dtype=np.float32))
    nq, N = queries.shape[0], data.shape[0]
    out_d = np.full((nq, k), np.inf)
    out_i = np.full((nq, k), -1, np.int64)
    for qi in range(nq):
        d = ed2_rows(data, queries[qi]) if kind == "ed" else dtw2_rows(data, queries[qi], r)
        order = np.lexsort((np.arange(N), d))[:k]
        out_d[qi, :len(order)] = d[order]
        out_i[qi, :len(order)] = order + row_begin
    return out_d, out_i
