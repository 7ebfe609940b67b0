"""ORACLE (test infrastructure only -- never imported by the product path).

ctypes wrappers around oracle/_ref/libref_cpu*.so: the reference's OWN CPU
path for the benchmark programs, i.e. the C that the reference compiler
emits for oracle/ref_programs/*.dpia (`dpia compile --target c-openmp`,
/root/reference/pkg/src/dpia/cli.py:58-90), compiled by oracle/build_ref.py.
The GPU parity tests compare the CUDA kernels with these outputs on the
bench's exact inputs ("outputs of the reference itself run
here").  Sizes are the ones the programs were emitted for: dot / asum take
the chunk count n (1024 elements per chunk), gemv is 8192 x 8192, mm_bt is
4096^3 with B passed transposed (the reference language has no transpose).
"""
from __future__ import annotations

import ctypes

import numpy as np

_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        from . import build_ref
        path, _march = build_ref.native_lib()
        if path is None:
            raise FileNotFoundError("oracle/_ref/libref_cpu.so is not built (oracle/build_ref.py)")
        _LIB = ctypes.CDLL(path)
        vp, ci = ctypes.c_void_p, ctypes.c_int
        _LIB.dot.argtypes = [vp, vp, vp, ci]
        _LIB.asum_proxy.argtypes = [vp, vp, ci]
        _LIB.gemv.argtypes = [vp, vp, vp]
        _LIB.mm_bt.argtypes = [vp, vp, vp]
        _LIB.scal.argtypes = [vp, ctypes.c_float, vp, ci]
    return _LIB


def available() -> bool:
    try:
        lib()
        return True
    except (OSError, FileNotFoundError):
        return False


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def dot(xs, ys) -> float:
    """ref_programs/dot.dpia: mapGlobal over 1024-chunks + sequential reduces."""
    x, y = _f32(xs), _f32(ys)
    assert x.size == y.size and x.size % 1024 == 0
    out = np.zeros(1, np.float32)
    lib().dot(out.ctypes.data, x.ctypes.data, y.ctypes.data, x.size // 1024)
    return float(out[0])


def asum_proxy(xs) -> float:
    """ref_programs/asum_proxy.dpia: the sum of xs (the reference has no abs;
    pass |x| to get asum)."""
    x = _f32(xs)
    assert x.size % 1024 == 0
    out = np.zeros(1, np.float32)
    lib().asum_proxy(out.ctypes.data, x.ctypes.data, x.size // 1024)
    return float(out[0])


def gemv(A, x) -> np.ndarray:
    """ref_programs/gemv.dpia (8192 x 8192, toLocal x)."""
    A, x = _f32(A), _f32(x)
    assert A.shape == (8192, 8192) and x.shape == (8192,)
    out = np.zeros(8192, np.float32)
    lib().gemv(out.ctypes.data, A.ctypes.data, x.ctypes.data)
    return out


def mm(A, B) -> np.ndarray:
    """ref_programs/mm_bt.dpia (4096^3) on A and B.T."""
    A, Bt = _f32(A), _f32(np.asarray(B).T)
    assert A.shape == (4096, 4096) and Bt.shape == (4096, 4096)
    out = np.zeros((4096, 4096), np.float32)
    lib().mm_bt(out.ctypes.data, A.ctypes.data, Bt.ctypes.data)
    return out


def scal(alpha: float, xs) -> np.ndarray:
    x = _f32(xs)
    assert x.size % 1024 == 0
    y = np.zeros_like(x)
    lib().scal(y.ctypes.data, float(alpha), x.ctypes.data, x.size // 1024)
    return y

