"""SCIR type checking: kinding, passivity and the
interference rule that makes `parfor` bodies race-free by construction.

Same judgement as the reference's checker (`SRC/checker.py:131-265`), stated
as a usage analysis: every phrase is assigned its type together with the
sets of identifiers it uses *actively* (may write) and *passively* (only
reads).  The rules:

  * a phrase of passive type (exp, passive functions, products of those)
    demotes all its active uses to passive;
  * in an application the active sets of function and argument must be
    disjoint (no two writers of the same resource) -- interference;
  * a lambda can be used where a *passive* function is expected (the body of
    every parfor / mapI) only if its body has no active free identifier:
    this is what rules out a work-item writing state shared with the others;
  * identifiers of the passive context zone may not be used actively.

The CUDA backend relies on this: emitted parallel loops need no atomics, and
the multi-GPU driver may split the outer parallel loop across devices.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, FrozenSet, Optional, Tuple

from .dtypes import (AccT, Array, CommT, DataType, DataVar, DepFnT, ExpT, FnT, Idx, Num,
                     Pair, PhraseType, ProdT, Vector, is_passive, phrase_type_equal,
                     subst_phrase_type)
from .signatures import PRIMITIVES
from .sizes import Nat
from .terms import App, Lam, Lit, PairP, Phrase, Prim, Proj, TApp, TLam, Var


class DpiaTypeError(Exception):
    def __init__(self, message: str, span=None):
        super().__init__(f"{span[0]}:{span[1]}: {message}" if span else message)
        self.span = span


@dataclass(frozen=True)
class Uses:
    active: FrozenSet[str] = frozenset()
    passive: FrozenSet[str] = frozenset()

    def __or__(self, o: "Uses") -> "Uses":
        return Uses(self.active | o.active, self.passive | o.passive)

    def without(self, name: str) -> "Uses":
        return Uses(self.active - {name}, self.passive - {name})

    def demoted(self) -> "Uses":
        return Uses(frozenset(), self.passive | self.active)

    def mode(self, name: str) -> str:
        return "active" if name in self.active else "passive" if name in self.passive else "unused"


NONE = Uses()

# -------------------------------------------------------------- kinding


def kind_of(delta: Dict[str, str], t) -> str:
    if isinstance(t, Nat):
        for v in t.free:
            if delta.get(v) != "nat":
                raise DpiaTypeError(f"unbound nat variable: {v}")
        return "nat"
    if isinstance(t, DataType):
        _kind_data(delta, t)
        return "data"
    if isinstance(t, PhraseType):
        _kind_phrase(delta, t)
        return "phrase"
    raise DpiaTypeError(f"not a type: {t!r}")


def _kind_data(delta, d):
    if isinstance(d, DataVar):
        if delta.get(d.name) != "data":
            raise DpiaTypeError(f"unbound data type variable: {d.name}")
    elif isinstance(d, Idx):
        kind_of(delta, d.bound)
    elif isinstance(d, Array):
        kind_of(delta, d.size)
        _kind_data(delta, d.elem)
    elif isinstance(d, Pair):
        _kind_data(delta, d.fst)
        _kind_data(delta, d.snd)
    elif not isinstance(d, (Num, Vector)):
        raise DpiaTypeError(f"ill-formed data type: {d!r}")


def _kind_phrase(delta, t):
    if isinstance(t, (ExpT, AccT)):
        _kind_data(delta, t.data)
    elif isinstance(t, ProdT):
        _kind_phrase(delta, t.fst)
        _kind_phrase(delta, t.snd)
    elif isinstance(t, FnT):
        _kind_phrase(delta, t.arg)
        _kind_phrase(delta, t.ret)
    elif isinstance(t, DepFnT):
        _kind_phrase({**delta, t.binder: t.kind}, t.body)
    elif not isinstance(t, CommT):
        raise DpiaTypeError(f"ill-formed phrase type: {t!r}")


# ------------------------------------------------------------- checking

def _settle(t: PhraseType, u: Uses) -> Tuple[PhraseType, Uses]:
    return (t, u.demoted()) if u.active and is_passive(t) else (t, u)


def infer(p: Phrase, env: Dict[str, PhraseType], delta: Dict[str, str]) -> Tuple[PhraseType, Uses]:
    if isinstance(p, Var):
        if p.name not in env:
            raise DpiaTypeError(f"unbound identifier: {p.name}", p.span)
        return _settle(env[p.name], Uses(frozenset({p.name})))
    if isinstance(p, Lit):
        return ExpT(p.dtype), NONE
    if isinstance(p, Prim):
        if p.name not in PRIMITIVES:
            raise DpiaTypeError(f"unknown primitive: {p.name}", p.span)
        return PRIMITIVES[p.name], NONE
    if isinstance(p, Lam):
        if p.arg_type is None:
            raise DpiaTypeError(f"unannotated lambda binder {p.binder!r} in inference position",
                                p.span)
        kind_of(delta, p.arg_type)
        bt, u = infer(p.body, {**env, p.binder: p.arg_type}, delta)
        return _settle(FnT(p.arg_type, bt), u.without(p.binder))
    if isinstance(p, App):
        ft, fu = infer(p.fn, env, delta)
        if not isinstance(ft, FnT):
            raise DpiaTypeError(f"applying a non-function of type {ft}", p.span)
        au = check(p.arg, ft.arg, env, delta)
        clash = fu.active & au.active
        if clash:
            raise DpiaTypeError("interference: active identifier(s) shared between function and "
                                f"argument: {sorted(clash)}", p.span)
        return _settle(ft.ret, fu | au)
    if isinstance(p, TApp):
        ft, u = infer(p.fn, env, delta)
        if not isinstance(ft, DepFnT):
            raise DpiaTypeError(f"type application of non-polymorphic phrase: {ft}")
        got = kind_of(delta, p.arg)
        if got != ft.kind:
            raise DpiaTypeError(f"type argument kind mismatch: expected {ft.kind}, got {got}")
        return _settle(subst_phrase_type(ft.body, ft.binder, p.arg), u)
    if isinstance(p, TLam):
        bt, u = infer(p.body, env, {**delta, p.binder: p.kind})
        return _settle(DepFnT(p.binder, p.kind, bt), u)
    if isinstance(p, PairP):
        # both components act on the same resource: no disjointness required
        (t1, u1), (t2, u2) = infer(p.fst, env, delta), infer(p.snd, env, delta)
        return _settle(ProdT(t1, t2), u1 | u2)
    if isinstance(p, Proj):
        t, u = infer(p.target, env, delta)
        if not isinstance(t, ProdT):
            raise DpiaTypeError(f"projection from non-product type {t}")
        return _settle(t.fst if p.index == 1 else t.snd, u)
    raise DpiaTypeError(f"not a phrase: {p!r}")


def check(p: Phrase, want: PhraseType, env, delta) -> Uses:
    """Uses of p checked against `want`; lambdas are promoted to passive
    functions where `want` demands it."""
    if isinstance(p, Lam) and isinstance(want, FnT):
        if p.arg_type is not None and not phrase_type_equal(p.arg_type, want.arg):
            raise DpiaTypeError(f"lambda annotation {p.arg_type} does not match expected argument "
                                f"type {want.arg}", p.span)
        u = check(p.body, want.ret, {**env, p.binder: want.arg}, delta).without(p.binder)
        if want.passive and u.active:
            raise DpiaTypeError("cannot promote to a passive function: body captures active "
                                f"identifier(s) {sorted(u.active)} (interference with parallel "
                                "execution)", p.span)
        return u
    if isinstance(p, PairP) and isinstance(want, ProdT):
        return check(p.fst, want.fst, env, delta) | check(p.snd, want.snd, env, delta)
    if isinstance(p, Lit) and isinstance(want, ExpT) and isinstance(want.data, Vector) \
            and isinstance(p.dtype, Num):
        return NONE  # a scalar literal splatted to a vector
    t, u = infer(p, env, delta)
    if not _convertible(t, u, want):
        raise DpiaTypeError(f"type mismatch: expected {want}, got {t}")
    return u


def _convertible(t: PhraseType, u: Uses, want: PhraseType) -> bool:
    if isinstance(t, FnT) and isinstance(want, FnT):
        if want.passive and not t.passive and u.active:
            return False
        return phrase_type_equal(t.arg, want.arg) and _convertible(t.ret, u, want.ret)
    return phrase_type_equal(t, want)


def type_check(p: Phrase, delta: Optional[Dict[str, str]] = None,
               pi: Optional[Dict[str, PhraseType]] = None,
               gamma: Optional[Dict[str, PhraseType]] = None) -> Tuple[PhraseType, Uses]:
    """(type, uses) of p in the zones pi (passive) / gamma (active)
    -- the reference's `type_check` (SRC/checker.py:260)."""
    pi, gamma = dict(pi or {}), dict(gamma or {})
    both = set(pi) & set(gamma)
    if both:
        raise DpiaTypeError(f"identifiers in both context zones: {both}")
    t, u = infer(p, {**pi, **gamma}, dict(delta or {}))
    bad = u.active & set(pi)
    if bad:
        raise DpiaTypeError(f"passive identifier(s) used actively: {sorted(bad)}")
    return t, u
