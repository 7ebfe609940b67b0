"""Host <-> device marshalling of DPIA values.

Values use the reference's representation (`SRC/eval_fn.py:1-30`): numbers,
lists for arrays, 2-tuples for pairs and vector objects exposing `.items`
(the reference's VectorVal or this package's `VectorVal`).  On the device a
value of type d occupies `layout(d).size` bytes laid out like the C type the
emitter declares (structs for pairs, naturally aligned dpia::vec for
vectors), so the common cases -- arrays of num or of vectors -- are plain
contiguous scalar arrays and marshal without any scatter.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

from .dtypes import Array, DataType, Idx, Num, Pair, Vector


@dataclass(frozen=True)
class VectorVal:
    items: Tuple


@dataclass
class Layout:
    size: int
    align: int
    offsets: np.ndarray   # byte offset of every scalar leaf, leaf order
    kinds: np.ndarray     # 0 = num, 1 = idx (64-bit int)


def _vec_align(w: int, s: int) -> int:
    b = s * w
    if w & (w - 1) == 0:
        return b if b <= 16 else 16
    return s


def layout(d: DataType, sigma=None, scalar_bytes: int = 4) -> Layout:
    sigma = sigma or {}
    s = scalar_bytes
    if isinstance(d, Num):
        return Layout(s, s, np.zeros(1, np.int64), np.zeros(1, np.int8))
    if isinstance(d, Idx):
        return Layout(8, 8, np.zeros(1, np.int64), np.ones(1, np.int8))
    if isinstance(d, Vector):
        a = _vec_align(d.width, s)
        size = -(-s * d.width // a) * a
        return Layout(size, a, np.arange(d.width, dtype=np.int64) * s, np.zeros(d.width, np.int8))
    if isinstance(d, Array):
        n = d.size.evaluate(sigma)
        e = layout(d.elem, sigma, s)
        offs = (np.arange(n, dtype=np.int64)[:, None] * e.size + e.offsets[None, :]).ravel()
        return Layout(n * e.size, e.align, offs, np.tile(e.kinds, n))
    if isinstance(d, Pair):
        a, b = layout(d.fst, sigma, s), layout(d.snd, sigma, s)
        ob = -(-a.size // b.align) * b.align
        al = max(a.align, b.align)
        size = -(-(ob + b.size) // al) * al
        return Layout(size, al, np.concatenate([a.offsets, b.offsets + ob]),
                      np.concatenate([a.kinds, b.kinds]))
    raise TypeError(f"no layout for {d}")


def shape_of(d: DataType, sigma=None, scalar_bytes: int = 4) -> Tuple[int, int, bool]:
    """(size, align, dense) of type d without materialising per-leaf offsets:
    dense means the leaves are consecutive scalars of one kind (num), so the
    device image of a value is its flat scalar array (no scatter)."""
    sigma = sigma or {}
    s = scalar_bytes
    if isinstance(d, Num):
        return s, s, True
    if isinstance(d, Idx):
        return 8, 8, False
    if isinstance(d, Vector):
        a = _vec_align(d.width, s)
        size = -(-s * d.width // a) * a
        return size, a, size == s * d.width
    if isinstance(d, Array):
        n = d.size.evaluate(sigma)
        size, a, dense = shape_of(d.elem, sigma, s)
        return n * size, a, dense
    if isinstance(d, Pair):
        sa, aa, da = shape_of(d.fst, sigma, s)
        sb, ab, db = shape_of(d.snd, sigma, s)
        ob = -(-sa // ab) * ab
        al = max(aa, ab)
        size = -(-(ob + sb) // al) * al
        return size, al, da and db and ob == sa and size == sa + sb
    raise TypeError(f"no layout for {d}")


def flatten(v) -> List:
    """Scalar leaves of a value in layout order."""
    if hasattr(v, "items") and not isinstance(v, (list, tuple, dict)):
        return list(v.items)
    if isinstance(v, list):
        out = []
        for x in v:
            out.extend(flatten(x))
        return out
    if isinstance(v, tuple):
        return flatten(v[0]) + flatten(v[1])
    return [v]


def unflatten(d: DataType, leaves, sigma=None):
    it = iter(leaves)

    def build(t):
        if isinstance(t, (Num, Idx)):
            return _py(next(it))
        if isinstance(t, Vector):
            return VectorVal(tuple(_py(next(it)) for _ in range(t.width)))
        if isinstance(t, Array):
            return [build(t.elem) for _ in range(t.size.evaluate(sigma or {}))]
        a = build(t.fst)
        return (a, build(t.snd))

    return build(d)


def _py(x):
    return x.item() if hasattr(x, "item") else x


def to_bytes(v, d: DataType, sigma, float_mode: bool) -> np.ndarray:
    """Device image (uint8) of value v (nested value or numpy array of leaves)."""
    s = 4 if float_mode else 8
    sdt = np.float32 if float_mode else np.int64
    size, _, dense = shape_of(d, sigma, s)
    if dense and isinstance(v, np.ndarray):
        # fast path (no per-leaf offsets): a flat scalar array is the image
        if v.size * s != size:
            raise ValueError(f"value has {v.size} scalars, type {d} needs {size // s}")
        return np.ascontiguousarray(v.reshape(-1), dtype=sdt).view(np.uint8)
    lay = layout(d, sigma, s)
    leaves = np.asarray(v).ravel() if isinstance(v, np.ndarray) else np.asarray(flatten(v))
    n = lay.offsets.size
    if leaves.size != n:
        raise ValueError(f"value has {leaves.size} scalars, type {d} needs {n}")
    if not lay.kinds.any() and (n == 0 or (lay.offsets[-1] == (n - 1) * s and lay.size == n * s)):
        return np.ascontiguousarray(leaves, dtype=sdt).view(np.uint8)
    buf = np.zeros(lay.size, np.uint8)
    for kind, dt in ((0, sdt), (1, np.int64)):
        sel = lay.kinds == kind
        if sel.any():
            vals = np.asarray(leaves[sel], dtype=dt)
            w = np.dtype(dt).itemsize
            idx = lay.offsets[sel][:, None] + np.arange(w)[None, :]
            buf[idx.ravel()] = vals.view(np.uint8).reshape(-1, w).ravel()
    return buf


def from_bytes(raw: np.ndarray, d: DataType, sigma, float_mode: bool) -> np.ndarray:
    """Leaves (float64 / int64 numpy array) of a device image."""
    s = 4 if float_mode else 8
    sdt = np.float32 if float_mode else np.int64
    size, _, dense = shape_of(d, sigma, s)
    if dense:
        return raw[:size].view(sdt).copy()
    lay = layout(d, sigma, s)
    n = lay.offsets.size
    if not lay.kinds.any() and (n == 0 or (lay.offsets[-1] == (n - 1) * s and lay.size == n * s)):
        return raw[:n * s].view(sdt).copy()
    out = np.zeros(n, np.float64 if float_mode else np.int64)
    for kind, dt in ((0, sdt), (1, np.int64)):
        sel = lay.kinds == kind
        if sel.any():
            w = np.dtype(dt).itemsize
            idx = lay.offsets[sel][:, None] + np.arange(w)[None, :]
            out[sel] = raw[idx.ravel()].view(dt)
    return out


def nbytes(d: DataType, sigma, float_mode: bool) -> int:
    return shape_of(d, sigma, 4 if float_mode else 8)[0]
