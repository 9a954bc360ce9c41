"""Seeded synthetic inputs shaped like the paper's workloads.

Random-walk series (x_0 ~ N(0,1), x_t = x_{t-1} + N(0,1)),
z-normalised with the population std (reading R10), rounded once to fp32;
query workloads "generated the same way" (seed 1) and the config-5 noise workload
(a uniformly chosen dataset row + N(0, sigma^2) per point, re-z-normalised).

This module holds none of the method's arithmetic; both the CUDA path (tests, bench) and
the oracle (tests) take their inputs from here.  Two implementations of the same
counter-based generator (Philox4x32-10 keyed by the seed, counter = (pair, row, stream),
Box-Muller in fp64):
  * ``*_cpu``  -- numpy, for CPU tests;
  * ``*_cuda`` -- datagen/libdatagen.so, writing straight into a torch CUDA tensor (the
    100M x 256 collection is generated on the device, shard by shard).
The two agree to within the last ulp of the fp64 transcendental functions (log, cos, sin),
which can flip the final fp32 rounding of a value; tests that compare the CUDA path with
the oracle always feed both the same (device-generated, copied back) rows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "datagen.cu")
_LIB = os.path.join(_HERE, "libdatagen.so")

STREAM_WALK, STREAM_ROWS, STREAM_NOISE = 0, 1, 2
DATA_SEED, QUERY_SEED = 0, 1  # BASELINE.json configs: dataset seed 0, queries seed 1

_M0, _M1, _W0, _W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85
_MASK = np.uint64(0xFFFFFFFF)


def _philox(c0, c1, c2, c3, k0, k1):
    c0, c1, c2, c3 = (np.asarray(c, np.uint64) & _MASK for c in (c0, c1, c2, c3))
    k0, k1 = np.uint64(k0) & _MASK, np.uint64(k1) & _MASK
    for _ in range(10):
        p0 = np.uint64(_M0) * c0
        p1 = np.uint64(_M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0 = (k0 + np.uint64(_W0)) & _MASK
        k1 = (k1 + np.uint64(_W1)) & _MASK
    return c0, c1, c2, c3


def _normals(seed, rows, stream, n):
    """[len(rows), n] standard normals: pair j of row r from one Philox block."""
    rows = np.asarray(rows, np.uint64)[:, None]
    j = np.arange(n // 2, dtype=np.uint64)[None, :]
    x0, x1, x2, x3 = _philox(j, rows & _MASK, rows >> np.uint64(32), np.uint64(stream),
                             seed & 0xFFFFFFFF, seed >> 32)
    a = (x1 << np.uint64(32)) | x0
    b = (x3 << np.uint64(32)) | x2
    u1 = ((a >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = (b >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    rad = np.sqrt(-2.0 * np.log(u1))
    ang = 6.283185307179586 * u2
    z = np.empty((rows.shape[0], n), np.float64)
    z[:, 0::2] = rad * np.cos(ang)
    z[:, 1::2] = rad * np.sin(ang)
    return z


def _znorm(x):
    mu = x.sum(1, keepdims=True) / x.shape[1]
    sd = np.sqrt(((x - mu) ** 2).sum(1, keepdims=True) / x.shape[1])
    with np.errstate(invalid="ignore", divide="ignore"):
        out = np.where(sd > 0, (x - mu) / np.where(sd > 0, sd, 1.0), 0.0)
    return out.astype(np.float32)


def walks_cpu(row_begin: int, rows: int, n: int, seed: int = DATA_SEED, chunk: int = 1 << 14):
    """Rows [row_begin, row_begin+rows) of the z-normalised random-walk collection (fp32)."""
    if n % 2:
        raise ValueError("n must be even")
    out = np.empty((rows, n), np.float32)
    for s in range(0, rows, chunk):
        e = min(rows, s + chunk)
        z = _normals(seed, np.arange(row_begin + s, row_begin + e), STREAM_WALK, n)
        out[s:e] = _znorm(np.cumsum(z, axis=1))
    return out


def noisy_rows(nq: int, N: int, query_seed: int = QUERY_SEED):
    """Source row of each config-5 query: uniform in [0, N) (mulhi of a 64-bit draw)."""
    x0, x1, _, _ = _philox(np.zeros(nq, np.uint64), np.arange(nq, dtype=np.uint64), np.zeros(nq, np.uint64),
                           np.uint64(STREAM_ROWS), query_seed & 0xFFFFFFFF, query_seed >> 32)
    u = [(int(h) << 32) | int(l) for h, l in zip(x1, x0)]
    return np.array([(v * N) >> 64 for v in u], np.int64)


def noisy_queries_cpu(nq: int, n: int, N: int, data_seed: int = DATA_SEED, query_seed: int = QUERY_SEED,
                      sigma: float = 0.1):
    rows = noisy_rows(nq, N, query_seed)
    src = np.concatenate([walks_cpu(int(r), 1, n, data_seed) for r in rows]).astype(np.float64)
    noise = _normals(query_seed, np.arange(nq), STREAM_NOISE, n)
    return _znorm(src + sigma * noise)


# ---------------------------------------------------------------------------- CUDA side
def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                               "-fmad=false", "-Xcompiler", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _cuda():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError(f"{_LIB} is not built (run __graft_entry__.build())")
        L = ctypes.CDLL(_LIB)
        L.dg_random_walks.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                      ctypes.c_uint64, ctypes.c_void_p]
        L.dg_noisy_queries.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                       ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p]
        _lib = L
    return _lib


def _stream_ptr(stream):
    import torch
    return (stream or torch.cuda.current_stream()).cuda_stream


def walks_cuda(out, row_begin: int, seed: int = DATA_SEED, stream=None):
    """Fill a [rows, n] float32 CUDA tensor with rows row_begin.. of collection `seed`."""
    assert out.is_cuda and out.dtype.is_floating_point and out.is_contiguous() and out.dim() == 2
    rc = _cuda().dg_random_walks(out.data_ptr(), int(row_begin), out.shape[0], out.shape[1], int(seed),
                                 _stream_ptr(stream))
    if rc:
        raise RuntimeError(f"dg_random_walks failed: cuda error {rc}")
    return out


def noisy_queries_cuda(out, N: int, data_seed: int = DATA_SEED, query_seed: int = QUERY_SEED,
                       sigma: float = 0.1, stream=None):
    assert out.is_cuda and out.is_contiguous() and out.dim() == 2
    rc = _cuda().dg_noisy_queries(out.data_ptr(), out.shape[0], out.shape[1], int(N), int(data_seed),
                                  int(query_seed), float(sigma), _stream_ptr(stream))
    if rc:
        raise RuntimeError(f"dg_noisy_queries failed: cuda error {rc}")
    return out
