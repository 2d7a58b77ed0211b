"""ORACLE — TEST INFRASTRUCTURE ONLY.  ctypes glue over contractions.c.

Every function converts its inputs to float64 exactly (fp32 and bf16 values are
exactly representable in fp64) and calls the direct loops of contractions.c,
which follow PAPER.md Def. 2.1 ("replaces each linear index ... with
a loop").  Layouts: dense/bmm X[b,m,k], W[b,n,k], Y[b,m,n]; conv2d X NHWC,
W KRSC, Y NPQK (DESIGN.md R-C1..R-C3); grouped conv W [K][R][S][C/G], depthwise
= groups C = K with W [C][R][S] (DESIGN.md R-C5).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build() -> str:
    """Compile liboracle.so in-tree (gcc + OpenMP)."""
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return os.path.join(_HERE, "liboracle.so")


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "contractions.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            build()
        lib = ctypes.CDLL(path)
        d = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        lib.oracle_bmm_f64.argtypes = [d, d, d, d, i64, i64, i64, i64]
        lib.oracle_conv2d_f64.argtypes = [d, d, d, d] + [i64] * 13
        lib.oracle_conv2d_at_f64.argtypes = [d, d, ctypes.POINTER(i64), i64, d, d] + [i64] * 13
        lib.oracle_bmm_at_f64.argtypes = [d, d, ctypes.POINTER(i64), i64, d, d, i64, i64, i64, i64]
        lib.oracle_gconv2d_f64.argtypes = [d, d, ctypes.POINTER(i64), i64, d, d] + [i64] * 14
        lib.oracle_num_threads.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def num_threads() -> int:
    return int(_lib().oracle_num_threads())


def conv_out_extent(h, pad, dil, r, stride):
    """P = floor((H + 2*pad - dil*(R-1) - 1)/stride) + 1  (standard conv2d extent)."""
    return (h + 2 * pad - dil * (r - 1) - 1) // stride + 1


def bmm(x, w):
    """Y[b,m,n] = sum_k X[b,m,k] W[b,n,k]; returns (Y, A) with A = sum |X||W|."""
    x = _f64(x)
    w = _f64(w)
    b, m, k = x.shape
    b2, n, k2 = w.shape
    assert b == b2 and k == k2
    y = np.empty((b, m, n), np.float64)
    a = np.empty((b, m, n), np.float64)
    _lib().oracle_bmm_f64(_dp(x), _dp(w), _dp(y), _dp(a), b, m, n, k)
    return y, a


def dense(x, w):
    """Y[m,n] = sum_k X[m,k] W[n,k] (weight [N,K]); returns (Y, A)."""
    y, a = bmm(np.asarray(x)[None], np.asarray(w)[None])
    return y[0], a[0]


def conv2d(x, w, stride=(1, 1), pad=(0, 0), dil=(1, 1)):
    """NHWC x KRSC -> NPQK, zero padding, groups = 1; returns (Y, A)."""
    x = _f64(x)
    w = _f64(w)
    n, h, wd, c = x.shape
    k, r, s, c2 = w.shape
    assert c == c2
    p = conv_out_extent(h, pad[0], dil[0], r, stride[0])
    q = conv_out_extent(wd, pad[1], dil[1], s, stride[1])
    y = np.empty((n, p, q, k), np.float64)
    a = np.empty((n, p, q, k), np.float64)
    _lib().oracle_conv2d_f64(_dp(x), _dp(w), _dp(y), _dp(a), n, h, wd, c, k, r, s,
                             stride[0], stride[1], pad[0], pad[1], dil[0], dil[1])
    return y, a


def conv2d_at(x, w, idx, stride=(1, 1), pad=(0, 0), dil=(1, 1)):
    """Only the outputs at linear NPQK indices ``idx``; returns (y, a) of len(idx)."""
    x = _f64(x)
    w = _f64(w)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    n, h, wd, c = x.shape
    k, r, s, _ = w.shape
    y = np.empty(idx.size, np.float64)
    a = np.empty(idx.size, np.float64)
    _lib().oracle_conv2d_at_f64(_dp(x), _dp(w), idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                idx.size, _dp(y), _dp(a), n, h, wd, c, k, r, s,
                                stride[0], stride[1], pad[0], pad[1], dil[0], dil[1])
    return y, a


def bmm_at(x, w, idx):
    """Only the outputs at linear (b,m,n) indices ``idx``; returns (y, a)."""
    x = _f64(x)
    w = _f64(w)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    b, m, k = x.shape
    _, n, _ = w.shape
    y = np.empty(idx.size, np.float64)
    a = np.empty(idx.size, np.float64)
    _lib().oracle_bmm_at_f64(_dp(x), _dp(w), idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                             idx.size, _dp(y), _dp(a), b, m, n, k)
    return y, a


def conv2d_grouped(x, w, groups, stride=(1, 1), pad=(0, 0), dil=(1, 1), idx=None):
    """Grouped conv2d: NHWC x [K][R][S][C/G] -> NPQK (every output, or only the linear
    NPQK indices ``idx``); returns (Y, A)."""
    x = _f64(x)
    w = _f64(w)
    n, h, wd, c = x.shape
    k, r, s, cg = w.shape
    assert c % groups == 0 and k % groups == 0 and cg == c // groups
    p = conv_out_extent(h, pad[0], dil[0], r, stride[0])
    q = conv_out_extent(wd, pad[1], dil[1], s, stride[1])
    if idx is None:
        shape, ip, cnt = (n, p, q, k), None, 0
    else:
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        shape, ip, cnt = (idx.size,), idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), idx.size
    y = np.empty(shape, np.float64)
    a = np.empty(shape, np.float64)
    _lib().oracle_gconv2d_f64(_dp(x), _dp(w), ip, cnt, _dp(y), _dp(a), n, h, wd, c, k, groups, r, s,
                              stride[0], stride[1], pad[0], pad[1], dil[0], dil[1])
    return y, a


def depthwise_conv2d(x, w, stride=(1, 1), pad=(0, 0), dil=(1, 1), idx=None):
    """Depthwise conv2d (groups = C = K): NHWC x W[C][R][S] -> NPQC; returns (Y, A)."""
    w = np.asarray(w)
    return conv2d_grouped(x, w[..., None], w.shape[0], stride, pad, dil, idx)
