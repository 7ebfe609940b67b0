"""ORACLE (test infrastructure only -- never imported by the product path).

CPU restatement of the reference's functional semantics `eval_phrase`
(/root/reference/pkg/src/dpia/eval_fn.py:120-215) over this repo's phrase AST,
plus the shim for primitives the reference lacks (SURVEY.md 8c "parity
unpinned" list): transpose, abs, reduceSeq, reduceLocal, mapWorkgroup1,
mapLocal1, let, lane indexing of vectors and array-splat literals.

Values follow the reference: numbers are Python int (exact "int mode") or
float (float64 "float mode"); index values are ints; arrays are lists; pairs
are 2-tuples; vectors are `Vec`.

Pinned against the reference itself: tests/golden/*.json are produced by
tests/golden/make_golden.py, which runs the reference's `eval_phrase` on the
same programs and inputs (see tests/test_oracle.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Tuple, Union

from paper_1710_08332_b200.dtypes import Array, DataType, Idx, Num, Pair, Vector
from paper_1710_08332_b200.terms import (App, Lam, Lit, PairP, Phrase, Proj,
                                         TApp, TLam, Var, unapply)

Number = Union[int, float]


@dataclass(frozen=True)
class Vec:
    """A vector value (reference VectorVal, eval_fn.py:23-28)."""
    items: Tuple[Number, ...]


class EvalError(Exception):
    pass


def c_divide(a: Number, b: Number) -> Number:
    """C semantics: truncating integer division (eval_fn.py:37-42)."""
    if isinstance(a, int) and isinstance(b, int):
        q = abs(a) // abs(b)
        return q if (a >= 0) == (b >= 0) else -q
    return a / b


_BIN = {"+": lambda a, b: a + b, "-": lambda a, b: a - b,
        "*": lambda a, b: a * b, "/": c_divide}


def binop(op: str, a, b):
    """Lane-wise on vectors, scalars splat (eval_fn.py:53-63)."""
    f = _BIN[op]
    if isinstance(a, Vec) or isinstance(b, Vec):
        w = len(a.items) if isinstance(a, Vec) else len(b.items)
        xa = a.items if isinstance(a, Vec) else (a,) * w
        xb = b.items if isinstance(b, Vec) else (b,) * w
        if len(xa) != len(xb):
            raise EvalError("vector width mismatch")
        return Vec(tuple(f(x, y) for x, y in zip(xa, xb)))
    return f(a, b)


def unop(op: str, v):
    g = (lambda x: -x) if op == "negate" else abs
    return Vec(tuple(g(x) for x in v.items)) if isinstance(v, Vec) else g(v)


def splat(value, d: DataType, sigma):
    if isinstance(d, Vector):
        return Vec((value,) * d.width)
    if isinstance(d, Array):
        n = d.size.evaluate(sigma)
        return [splat(value, d.elem, sigma) for _ in range(n)]
    return value


_MAPS = ("map", "mapGlobal", "mapWorkgroup", "mapWorkgroup1", "mapLocal", "mapLocal1", "mapSeq")


def eval_phrase(p: Phrase, env: Dict[str, object], sigma: Dict[str, int] = None):
    return _ev(p, env, sigma or {})


def _ev(p: Phrase, env, sigma):
    u = unapply(p)
    if u is not None:
        r = _prim(u[0], u[1], u[2], env, sigma)
        if r is not NotImplemented:
            return r
    if isinstance(p, Var):
        if p.name not in env:
            raise EvalError(f"unbound identifier: {p.name}")
        return env[p.name]
    if isinstance(p, Lit):
        return splat(p.value, p.dtype, sigma)
    if isinstance(p, Lam):
        return lambda v: _ev(p.body, {**env, p.binder: v}, sigma)
    if isinstance(p, App):
        return _ev(p.fn, env, sigma)(_ev(p.arg, env, sigma))
    if isinstance(p, TLam):
        return _ev(p.body, env, sigma)
    if isinstance(p, TApp):
        return _ev(p.fn, env, sigma)
    if isinstance(p, PairP):
        return (_ev(p.fst, env, sigma), _ev(p.snd, env, sigma))
    if isinstance(p, Proj):
        return _ev(p.target, env, sigma)[p.index - 1]
    raise EvalError(f"cannot evaluate {p!r}")


def _prim(name, targs, args, env, sigma):
    ev = lambda q: _ev(q, env, sigma)  # noqa: E731
    k = len(args)
    if name in _BIN and k == 1:
        a, b = ev(args[0])
        return binop(name, a, b)
    if name in ("negate", "abs") and k == 1:
        return unop(name, ev(args[0]))
    if name in _MAPS and k == 2:
        f = ev(args[0])
        return [f(x) for x in ev(args[1])]
    if name in _MAPS and k == 1:
        f = ev(args[0])
        return lambda xs: [f(x) for x in xs]
    if name in ("reduce", "reduceSeq", "reduceLocal") and k == 3:
        # left fold from the initial value (eval_fn.py:175-180); reduceLocal
        # shares the semantics (its operator is associative and commutative)
        f, acc = ev(args[0]), ev(args[1])
        for x in ev(args[2]):
            acc = f(x)(acc)
        return acc
    if name == "zip" and k == 2:
        xs, ys = ev(args[0]), ev(args[1])
        if len(xs) != len(ys):
            raise EvalError("zip of arrays of different lengths")
        return list(zip(xs, ys))
    if name == "split" and k == 1:
        n = targs[0].evaluate(sigma)
        flat = ev(args[0])
        return [flat[i * n:(i + 1) * n] for i in range(len(flat) // n)]
    if name == "join" and k == 1:
        return [x for row in ev(args[0]) for x in row]
    if name == "transpose" and k == 1:
        rows = ev(args[0])
        m = targs[1].evaluate(sigma)
        return [[row[j] for row in rows] for j in range(m)]
    if name == "pair" and k == 2:
        return (ev(args[0]), ev(args[1]))
    if name == "fst" and k == 1:
        return ev(args[0])[0]
    if name == "snd" and k == 1:
        return ev(args[0])[1]
    if name.startswith("idxVec") and k == 2:  # shim: lane of a vector
        v, i = ev(args[0]), ev(args[1])
        return v.items[i]
    if name == "let" and k == 2:  # shim: bind the value
        return ev(args[1])(ev(args[0]))
    if name in ("toGlobal", "toLocal", "toPrivate") and k == 2:
        return ev(args[0])(ev(args[1]))
    if name == "idx" and k == 2:
        xs, i = ev(args[0]), ev(args[1])
        if isinstance(xs, Vec):  # lane of a vector (shim)
            xs = list(xs.items)
        if not 0 <= i < len(xs):
            raise EvalError(f"index {i} out of bounds {len(xs)}")
        return xs[i]
    if name.startswith("asVector") and "Acc" not in name and k == 1:
        w = int(name[len("asVector"):])
        flat = ev(args[0])
        return [Vec(tuple(flat[i * w:(i + 1) * w])) for i in range(len(flat) // w)]
    if name.startswith("asScalar") and "Acc" not in name and k == 1:
        return [x for v in ev(args[0]) for x in v.items]
    return NotImplemented


# ------------------------------------------------- error bounds (float mode)

class Bounded:
    """A float-mode number carried with a first-order bound on its rounding
    sensitivity: t = sum of |terms| for + - *, propagated through / as
    t_a/|b| + |a| t_b/b^2.  Evaluating a program on Bounded inputs gives,
    per output, the normwise scale of the tolerance |got - want| <= tol * t
    that the fp32 parity tests state."""
    __slots__ = ("v", "t")

    def __init__(self, v, t=None):
        self.v = v
        self.t = abs(v) if t is None else t

    @staticmethod
    def _w(o):
        return o if isinstance(o, Bounded) else Bounded(o)

    def __add__(self, o):
        o = self._w(o)
        return Bounded(self.v + o.v, self.t + o.t)

    __radd__ = __add__

    def __sub__(self, o):
        o = self._w(o)
        return Bounded(self.v - o.v, self.t + o.t)

    def __rsub__(self, o):
        return self._w(o) - self

    def __mul__(self, o):
        o = self._w(o)
        return Bounded(self.v * o.v, self.t * o.t)

    __rmul__ = __mul__

    def __truediv__(self, o):
        o = self._w(o)
        return Bounded(self.v / o.v, self.t / abs(o.v) + abs(self.v) * o.t / (o.v * o.v))

    def __rtruediv__(self, o):
        return self._w(o) / self

    def __neg__(self):
        return Bounded(-self.v, self.t)

    def __abs__(self):
        return Bounded(abs(self.v), self.t)


def bounded(value):
    """Wrap every float leaf of an input value in Bounded."""
    if isinstance(value, float):
        return Bounded(value)
    if isinstance(value, Vec):
        return Vec(tuple(bounded(x) for x in value.items))
    if isinstance(value, tuple):
        return tuple(bounded(x) for x in value)
    if isinstance(value, list):
        return [bounded(x) for x in value]
    return value


def eval_with_bounds(p: Phrase, env: Dict[str, object], sigma: Dict[str, int] = None):
    """(values, bounds): the float64 result leaves and their sum|terms|."""
    out = flatten_value(eval_phrase(p, {k: bounded(v) for k, v in env.items()}, sigma))
    vals = [x.v if isinstance(x, Bounded) else x for x in out]
    bnds = [x.t if isinstance(x, Bounded) else abs(x) for x in out]
    return vals, bnds


# ------------------------------------------------------ value marshalling

def flatten_value(v) -> List[Number]:
    """Scalar leaves in row-major layout order (eval_fn.py:82-89)."""
    if isinstance(v, Vec):
        return list(v.items)
    if isinstance(v, list):
        return [x for item in v for x in flatten_value(item)]
    if isinstance(v, tuple):
        return flatten_value(v[0]) + flatten_value(v[1])
    return [v]


def unflatten_value(d: DataType, flat, sigma=None):
    it = iter(flat)

    def build(t):
        if isinstance(t, (Num, Idx)):
            return next(it)
        if isinstance(t, Vector):
            return Vec(tuple(next(it) for _ in range(t.width)))
        if isinstance(t, Array):
            return [build(t.elem) for _ in range(t.size.evaluate(sigma or {}))]
        if isinstance(t, Pair):
            a = build(t.fst)
            return (a, build(t.snd))
        raise EvalError(f"cannot build value of type {t}")

    out = build(d)
    if next(it, None) is not None:
        raise EvalError("too many scalars for type")
    return out


def to_json(v):
    if isinstance(v, Vec):
        return {"vec": list(v.items)}
    if isinstance(v, tuple):
        return {"pair": [to_json(v[0]), to_json(v[1])]}
    if isinstance(v, list):
        return [to_json(x) for x in v]
    return v


def from_json(j):
    if isinstance(j, dict) and "vec" in j:
        return Vec(tuple(j["vec"]))
    if isinstance(j, dict) and "pair" in j:
        return (from_json(j["pair"][0]), from_json(j["pair"][1]))
    if isinstance(j, list):
        return [from_json(x) for x in j]
    return j
