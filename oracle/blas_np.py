"""ORACLE (test infrastructure only -- never imported by the product path).

NumPy float64 restatements of the benchmark programs at full size, where the
reference interpreter `eval_phrase` (/root/reference/pkg/src/dpia/eval_fn.py:
120-215) is too slow (~0.1 M elements/s).  Each returns the
float64 value of the program and the sum of |terms| that bounds any fp32
re-association error; tests accept

    |got - want| <= TOL * sum|terms|,   TOL = 1e-4

The restatements are cross-checked against `oracle.dpia_eval` (which is in
turn pinned to the reference's golden vectors) at small sizes in
tests/test_oracle.py, so they inherit its parity.

`hash_f32` reproduces libdpia_rt's device-side input generator bit-exactly,
so any shard of the N = 2^31 scale-out inputs can be regenerated on the host.
"""
from __future__ import annotations

import numpy as np

TOL = 1e-4


def seeded(shape, seed, lo, hi):
    """Synthetic inputs: numpy default_rng(seed) uniform in [lo, hi), float32."""
    return np.random.default_rng(seed).uniform(lo, hi, size=shape).astype(np.float32)


def dot(xs, ys):
    """(reduce (+) 0 (map (* fst snd) (zip xs ys))) in float64."""
    x = np.asarray(xs, np.float64)
    y = np.asarray(ys, np.float64)
    return float(np.dot(x, y)), float(np.dot(np.abs(x), np.abs(y)))


def asum(xs):
    x = np.abs(np.asarray(xs, np.float64))
    s = float(x.sum())
    return s, s


def gemv(A, x):
    A64 = np.asarray(A, np.float64)
    x64 = np.asarray(x, np.float64)
    return A64 @ x64, np.abs(A64) @ np.abs(x64)


def mm(A, B, rows=None):
    """C = A B (optionally only the given rows) and |A| |B|."""
    A64 = np.asarray(A if rows is None else np.asarray(A)[rows], np.float64)
    B64 = np.asarray(B, np.float64)
    return A64 @ B64, np.abs(A64) @ np.abs(B64)


def hash_f32(count: int, offset: int, seed: int, lo: float, hi: float) -> np.ndarray:
    """Bit-exact host copy of dpia_fill_hash_f32 (csrc/dpia_rt.cpp)."""
    k = np.arange(offset, offset + count, dtype=np.uint64)
    lo32 = (k & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    hi32 = (k >> np.uint64(32)).astype(np.uint32)
    with np.errstate(over="ignore"):
        h = (lo32 * np.uint32(0x9E3779B1)) ^ (hi32 * np.uint32(0x85EBCA77)) ^ np.uint32(seed)
        h ^= h >> np.uint32(16)
        h *= np.uint32(0x7FEB352D)
        h ^= h >> np.uint32(15)
        h *= np.uint32(0x846CA68B)
        h ^= h >> np.uint32(16)
    u = (h >> np.uint32(8)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    return np.float32(lo) + np.float32(hi - lo) * u


def hashed_dot(n: int, seed_x: int, seed_y: int, chunk: int = 1 << 24):
    """dot over hash-generated inputs, streamed in float64 chunks."""
    total = absum = 0.0
    for off in range(0, n, chunk):
        c = min(chunk, n - off)
        x = hash_f32(c, off, seed_x, -1.0, 1.0).astype(np.float64)
        y = hash_f32(c, off, seed_y, -1.0, 1.0).astype(np.float64)
        total += float(np.dot(x, y))
        absum += float(np.dot(np.abs(x), np.abs(y)))
    return total, absum


def hashed_asum(n: int, seed: int, chunk: int = 1 << 24):
    total = 0.0
    for off in range(0, n, chunk):
        c = min(chunk, n - off)
        total += float(np.abs(hash_f32(c, off, seed, -1.0, 1.0).astype(np.float64)).sum())
    return total, total


def within(got, want, absterms, tol=TOL) -> bool:
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return bool(np.all(np.abs(got - want) <= tol * np.asarray(absterms, np.float64) + 1e-30))
