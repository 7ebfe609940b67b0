"""Translation Stage I: functional expressions -> higher-order imperative
phrases, by the mutually recursive acceptor-passing (A) and
continuation-passing (C) translations of the paper (section 5;
reference `SRC/translate.py:31-314`).

Strategy preservation: every map-family node yields exactly one mapI-family
node, every reduce one reduceI (or reduceIInit), every reduceLocal one
reduceILocal; nothing is fused, duplicated or re-scheduled.

Differences from the reference, all conservative extensions:
* ``transpose`` (acceptor dual ``transposeAcc``), ``abs``, ``reduceSeq`` and
  ``reduceLocal`` are translated;
* a ``toX`` space annotation reaches the map that is materialised *through*
  layout-only combinators (split/join/transpose/asVector/asScalar/idx), so
  ``toLocal (lam t (transpose (mapLocal F t))) E`` stages in local memory;
* a non-trivial reduce initial value is written straight into the
  accumulator by A (``reduceIInit``) instead of through a temporary;
* ``let``: A(let E f, a) = C(E, v. A(f v, a)) and C(let E f, c) =
  C(E, v. C(f v, c)) -- E is materialised once, where the let stands.
"""
from __future__ import annotations

from typing import Callable, Optional

from .dtypes import AccT, Array, DataType, ExpT, Idx, Num, Pair, Vector
from .signatures import (ARITH_OPS, MAP_FAMILY, MAP_TO_MAPI, REDUCE_FAMILY,
                         SPACE_NEW, TO_SPACE, UNARY_OPS, vector_prim)
from .terms import (App, Lam, PairP, Phrase, Prim, Proj, Var, apply_prim,
                    beta_normalize, seq, subtree_iter, unapply)

Cont = Callable[[Phrase], Phrase]

# heads that make an expression non-trivial (need a translation clause)
_NONTRIVIAL = set(MAP_FAMILY) | set(REDUCE_FAMILY) | {"reduceLocal", "let"} | set(TO_SPACE)
_LAYOUT = ("split", "join", "transpose")


def is_trivial(e: Phrase) -> bool:
    """No map/reduce/toX anywhere: passed through verbatim (`SRC/translate.py:292`)."""
    return not any(isinstance(s, Prim) and s.name in _NONTRIVIAL for s in subtree_iter(e))


class Translator:
    def __init__(self, default_space: Optional[str] = None):
        self.default_space = default_space
        self._k = 0

    def fresh(self, base: str) -> str:
        self._k += 1
        return f"{base}{self._k}"

    # ---------------------------------------------- generalised assignment
    def gen_assign(self, a: Phrase, d: DataType, e: Phrase) -> Phrase:
        if isinstance(d, (Num, Idx, Vector)):
            return apply_prim(":=", [d], [PairP(a, e)])
        if isinstance(d, Array):
            x, o = self.fresh("x"), self.fresh("a")
            f = Lam(x, Lam(o, self.gen_assign(Var(o), d.elem, Var(x)), AccT(d.elem)),
                    ExpT(d.elem))
            return apply_prim("mapI", [d.size, d.elem, d.elem], [f, e, a])
        if isinstance(d, Pair):
            parts = []
            for k, (proj, sub) in enumerate((("fst", d.fst), ("snd", d.snd)), start=1):
                parts.append(self.gen_assign(apply_prim(f"pairAcc{k}", [d.fst, d.snd], [a]), sub,
                                             apply_prim(proj, [d.fst, d.snd], [e])))
            return seq(parts[0], parts[1])
        raise ValueError(f"no assignment at type {d}")

    # ---------------------------------------------------------- helpers
    def _map_fn(self, f: Phrase, d1: DataType, d2: DataType) -> Phrase:
        x, o = self.fresh("x"), self.fresh("o")
        body = self.acceptor(beta_normalize(App(f, Var(x))), d2, Var(o))
        return Lam(x, Lam(o, body, AccT(d2)), ExpT(d1))

    def _reduce_fn(self, f: Phrase, d1: DataType, d2: DataType) -> Phrase:
        x, y, o = self.fresh("x"), self.fresh("y"), self.fresh("o")
        body = self.acceptor(beta_normalize(App(App(f, Var(x)), Var(y))), d2, Var(o))
        return Lam(x, Lam(y, Lam(o, body, AccT(d2)), ExpT(d2)), ExpT(d1))

    def _reify(self, d: DataType, c: Cont) -> Phrase:
        r = self.fresh("r")
        return Lam(r, c(Var(r)), ExpT(d))

    def _reduction(self, name, targs, args, k: Cont) -> Phrase:
        """Shared by A and C: k receives the reduced value."""
        if name == "reduceLocal":
            (n, d), (f, init, src) = targs, args
            fi = self._reduce_fn(f, d, d)
            return self.continuation(src, Array(n, d), lambda x: self.continuation(
                init, d, lambda y: apply_prim("reduceILocal", [n, d],
                                              [fi, y, x, self._reify(d, k)])))
        (n, d1, d2), (f, init, src) = targs, args
        fi = self._reduce_fn(f, d1, d2)
        if is_trivial(init):
            return self.continuation(src, Array(n, d1), lambda x: apply_prim(
                "reduceI", [n, d1, d2], [fi, init, x, self._reify(d2, k)]))
        o = self.fresh("o")
        init_cmd = Lam(o, self.acceptor(init, d2, Var(o)), AccT(d2))
        return self.continuation(src, Array(n, d1), lambda x: apply_prim(
            "reduceIInit", [n, d1, d2], [fi, init_cmd, x, self._reify(d2, k)]))

    # ------------------------------------------------ acceptor translation
    def acceptor(self, e: Phrase, d: DataType, a: Phrase) -> Phrase:
        u = unapply(e)
        name, targs, args = u if u else (None, [], [])

        if name in MAP_FAMILY and len(args) == 2:
            n, d1, d2 = targs
            fi = self._map_fn(args[0], d1, d2)
            return self.continuation(args[1], Array(n, d1),
                                     lambda x: apply_prim(MAP_TO_MAPI[name], [n, d1, d2], [fi, x, a]))
        if (name in REDUCE_FAMILY or name == "reduceLocal") and len(args) == 3:
            return self._reduction(name, targs, args, lambda r: self.gen_assign(a, d, r))
        if name in ARITH_OPS and len(args) == 1:
            (dd,), (ops,) = targs, args
            return self.continuation(ops.fst, dd, lambda x: self.continuation(
                ops.snd, dd, lambda y: apply_prim(":=", [dd], [PairP(a, apply_prim(
                    name, [dd], [PairP(x, y)]))])))
        if name in UNARY_OPS and len(args) == 1:
            dd = targs[0]
            return self.continuation(args[0], dd, lambda x: apply_prim(
                ":=", [dd], [PairP(a, apply_prim(name, [dd], [x]))]))
        if name == "zip" and len(args) == 2:
            n, d1, d2 = targs
            return seq(self.acceptor(args[0], Array(n, d1), apply_prim("zipAcc1", targs, [a])),
                       self.acceptor(args[1], Array(n, d2), apply_prim("zipAcc2", targs, [a])))
        if name == "pair" and len(args) == 2:
            d1, d2 = targs
            return seq(self.acceptor(args[0], d1, apply_prim("pairAcc1", targs, [a])),
                       self.acceptor(args[1], d2, apply_prim("pairAcc2", targs, [a])))
        if name == "split" and len(args) == 1:
            n, m, dd = targs
            return self.acceptor(args[0], Array(n * m, dd), apply_prim("splitAcc", targs, [a]))
        if name == "join" and len(args) == 1:
            n, m, dd = targs
            return self.acceptor(args[0], Array(n, Array(m, dd)), apply_prim("joinAcc", targs, [a]))
        if name == "transpose" and len(args) == 1:
            n, m, dd = targs
            return self.acceptor(args[0], Array(n, Array(m, dd)),
                                 apply_prim("transposeAcc", targs, [a]))
        if name in ("fst", "snd") and len(args) == 1:
            d1, d2 = targs
            return self.continuation(args[0], Pair(d1, d2), lambda x: self.gen_assign(
                a, d1 if name == "fst" else d2, apply_prim(name, targs, [x])))
        vp = vector_prim(name) if name else None
        if vp and vp[0] in ("asVector", "asScalar") and args:
            kind, w = vp
            (m,), (src,) = targs, args
            if kind == "asVector":
                return self.acceptor(src, Array(m * w, Num()), apply_prim(f"asVectorAcc{w}", [m], [a]))
            return self.acceptor(src, Array(m, Vector(w)), apply_prim(f"asScalarAcc{w}", [m], [a]))
        if name in TO_SPACE and len(args) == 2:
            return self.acceptor(beta_normalize(App(args[0], args[1])), d, a)
        if name == "let" and len(args) == 2:
            d1, _d2 = targs
            return self.continuation(args[0], d1, lambda v: self.acceptor(
                beta_normalize(App(args[1], v)), d, a))
        if name == "idx" and len(args) == 2 and not is_trivial(e):
            n, dd = targs
            return self.continuation(args[0], Array(n, dd), lambda x: self.gen_assign(
                a, dd, apply_prim("idx", targs, [x, args[1]])))
        if is_trivial(e):
            return self.gen_assign(a, d, e)
        raise ValueError(f"no acceptor-translation clause for {e!r}")

    # -------------------------------------------- continuation translation
    def continuation(self, e: Phrase, d: DataType, c: Cont, space: Optional[str] = None) -> Phrase:
        u = unapply(e)
        name, targs, args = u if u else (None, [], [])

        if name in MAP_FAMILY and len(args) == 2:
            n, _d1, d2 = targs
            out_t = Array(n, d2)
            tmp = self.fresh("tmp")
            body = seq(self.acceptor(e, out_t, Proj(Var(tmp), 1)), c(Proj(Var(tmp), 2)))
            return apply_prim(SPACE_NEW[space or self.default_space], [out_t], [Lam(tmp, body)])
        if (name in REDUCE_FAMILY or name == "reduceLocal") and len(args) == 3:
            return self._reduction(name, targs, args, c)
        if name in ARITH_OPS and len(args) == 1:
            (dd,), (ops,) = targs, args
            return self.continuation(ops.fst, dd, lambda x: self.continuation(
                ops.snd, dd, lambda y: c(apply_prim(name, [dd], [PairP(x, y)]))))
        if name in UNARY_OPS and len(args) == 1:
            return self.continuation(args[0], targs[0], lambda x: c(apply_prim(name, targs, [x])))
        if name in ("zip", "pair") and len(args) == 2:
            if name == "zip":
                n, d1, d2 = targs
                t1, t2 = Array(n, d1), Array(n, d2)
            else:
                t1, t2 = targs
            return self.continuation(args[0], t1, lambda x: self.continuation(
                args[1], t2, lambda y: c(apply_prim(name, targs, [x, y]))))
        if name in _LAYOUT and len(args) == 1:
            n, m, dd = targs
            src_t = Array(n * m, dd) if name == "split" else Array(n, Array(m, dd))
            return self.continuation(args[0], src_t, lambda x: c(apply_prim(name, targs, [x])),
                                     space=space)
        if name in ("fst", "snd") and len(args) == 1:
            return self.continuation(args[0], Pair(*targs), lambda x: c(apply_prim(name, targs, [x])))
        vp = vector_prim(name) if name else None
        if vp and vp[0] in ("asVector", "asScalar") and args:
            kind, w = vp
            (m,), (src,) = targs, args
            src_t = Array(m * w, Num()) if kind == "asVector" else Array(m, Vector(w))
            return self.continuation(src, src_t, lambda x: c(apply_prim(name, [m], [x])),
                                     space=space)
        if name in TO_SPACE and len(args) == 2:
            body = beta_normalize(App(args[0], args[1]))
            bu = unapply(body)
            if bu is not None and (bu[0] in _LAYOUT or (vector_prim(bu[0]) or ("",))[0] in
                                   ("asVector", "asScalar")) and not is_trivial(body):
                # a layout view of a computed value: store the value itself in
                # space X, written through the acceptor duals of the view
                tmp = self.fresh("tmp")
                stage = seq(self.acceptor(body, d, Proj(Var(tmp), 1)), c(Proj(Var(tmp), 2)))
                return apply_prim(SPACE_NEW[TO_SPACE[name]], [d], [Lam(tmp, stage)])
            return self.continuation(body, d, c, space=TO_SPACE[name])
        if name == "let" and len(args) == 2:
            d1, _d2 = targs
            return self.continuation(args[0], d1, lambda v: self.continuation(
                beta_normalize(App(args[1], v)), d, c))
        if name == "idx" and len(args) == 2 and not is_trivial(e):
            n, dd = targs
            return self.continuation(args[0], Array(n, dd),
                                     lambda x: c(apply_prim("idx", targs, [x, args[1]])), space=space)
        if is_trivial(e):
            return c(e)
        raise ValueError(f"no continuation-translation clause for {e!r}")


def acceptor_translate(e: Phrase, delta: DataType, a: Phrase,
                       default_space: Optional[str] = None) -> Phrase:
    return Translator(default_space).acceptor(e, delta, a)


def continuation_translate(e: Phrase, delta: DataType, c: Cont,
                           default_space: Optional[str] = None) -> Phrase:
    return Translator(default_space).continuation(e, delta, c)


def translate_program(body: Phrase, delta: DataType, out: str = "out",
                      default_space: Optional[str] = None) -> Phrase:
    """Stage I entry point (`SRC/translate.py:311`): the command `out :=_delta body`."""
    return Translator(default_space).acceptor(body, delta, Var(out))
