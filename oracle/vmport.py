"""ctypes wrapper for oracle/libvmport.so -- TEST/BASELINE INFRASTRUCTURE ONLY.

The C restatement of the reference VM's f32 arithmetic (see vmport.c).  Used
as the CPU baseline in bench.py and cross-checked bit-for-bit against the
reference VM outputs stored in tests/golden/.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

OP = {"add": 0, "mul": 1, "max": 2, "min": 3}
EW = {"identity": 0, "relu": 1, "sigmoid": 2}


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "libvmport.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libvmport.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        i64, fp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        L.vmp_gemm.argtypes = [i64, i64, i64, fp, i64, i64, fp, i64, i64, fp, i64, i64,
                               ci, ci, fp, i64, ci, i64, i64, ci]
        L.vmp_gemm.restype = ci
        L.vmp_conv2d.argtypes = [i64] * 9 + [fp, fp, fp, i64, i64, ci]
        L.vmp_conv2d.restype = ci
        _LIB = L
    return _LIB


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def gemm(A, B, combine="mul", reduce="add", bias=None, post="identity",
         rows=None, out=None, threads=None):
    """C = post(reduce_k combine(A[m,k], B[k,n]) (+ bias[n])), VM f32 order.

    ``rows`` = (r0, r1) computes only those output rows (returned array has
    all M rows; rows outside stay as in ``out``)."""
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    C = out if out is not None else np.zeros((M, N), np.float32)
    r0, r1 = rows if rows is not None else (0, M)
    bptr = None
    if bias is not None:
        bias = np.ascontiguousarray(bias, np.float32)
        bptr = _ptr(bias)
    rc = lib().vmp_gemm(M, N, K, _ptr(A), K, 1, _ptr(B), N, 1, _ptr(C), N, 1,
                        OP[combine], OP[reduce], bptr, 1, EW[post], r0, r1,
                        threads or cores())
    assert rc == 0
    return C


def conv2d(x, w, stride=1, pad=0, images=None, out=None, threads=None):
    """NCHW conv, VM order (ci, r, s) per output point."""
    x = np.ascontiguousarray(x, np.float32)
    w = np.ascontiguousarray(w, np.float32)
    N, C, H, W = x.shape
    CO, C2, R, S = w.shape
    assert C == C2
    HO, WO = (H + 2 * pad - R) // stride + 1, (W + 2 * pad - S) // stride + 1
    o = out if out is not None else np.zeros((N, CO, HO, WO), np.float32)
    i0, i1 = images if images is not None else (0, N)
    rc = lib().vmp_conv2d(N, C, H, W, CO, R, S, stride, pad, _ptr(x), _ptr(w), _ptr(o),
                          i0, i1, threads or cores())
    assert rc == 0
    return o
