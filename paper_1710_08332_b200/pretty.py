"""Surface-syntax printing of phrases (functional, intermediate and
imperative) such that `parse_phrase(show(p), env)` is alpha-equivalent to p.

Serves `--dump-stages` of the CLI (the reference's `pretty_print`,
SRC/pretty.py:53-110, plays the same role).  Strategy: every lambda binder is
printed with its type annotation and every primitive in its surface form, so
the elaborator re-infers all size/type arguments locally; array-typed splat
literals are wrapped in `(as TYPE v)`.
"""
from __future__ import annotations

from .dtypes import Array
from .signatures import (ARITH_OPS, MAP_FAMILY, MAPI_FAMILY, NEW_SPACE, PARFOR_FAMILY,
                         REDUCE_FAMILY, TO_SPACE, UNARY_OPS, vector_prim)
from .sizes import nat_str
from .terms import App, Lam, Lit, PairP, Phrase, Prim, Proj, TApp, TLam, Var, unapply

_PLAIN = set(MAP_FAMILY) | set(MAPI_FAMILY) | set(PARFOR_FAMILY) | set(REDUCE_FAMILY) | \
    set(TO_SPACE) | set(UNARY_OPS) | {
        "reduceLocal", "zip", "join", "transpose", "pair", "fst", "snd", "idx", "idxAcc",
        "splitAcc", "transposeAcc", "pairAcc1", "pairAcc2", "zipAcc1", "zipAcc2", "reduceI",
        "reduceIInit", "reduceILocal", "let"}


def _lit(p: Lit) -> str:
    v = repr(p.value) if isinstance(p.value, float) else str(int(p.value))
    return f"(as {p.dtype} {v})" if isinstance(p.dtype, Array) else v


def show(p: Phrase) -> str:
    if isinstance(p, Var):
        return p.name
    if isinstance(p, Lit):
        return _lit(p)
    if isinstance(p, Lam):
        ann = f"({p.binder} {p.arg_type})" if p.arg_type is not None else p.binder
        return f"(lam {ann} {show(p.body)})"
    if isinstance(p, PairP):
        return f"(tuple {show(p.fst)} {show(p.snd)})"
    if isinstance(p, Proj):
        return f"(proj{p.index} {show(p.target)})"
    if isinstance(p, TLam):
        return f"(tlam ({p.binder} {p.kind}) {show(p.body)})"
    u = unapply(p)
    if u is not None:
        name, targs, args = u
        if not args and not targs:
            return name
        if name in ARITH_OPS + (":=",) and len(args) == 1 and isinstance(args[0], PairP):
            return f"({name} {show(args[0].fst)} {show(args[0].snd)})"
        if name == ";" and len(args) == 1 and isinstance(args[0], PairP):
            return f"(seq {show(args[0].fst)} {show(args[0].snd)})"
        if name.startswith("idxVec") and len(args) == 2:
            return f"(idx {show(args[0])} {show(args[1])})"
        if name == "split" and len(args) == 1:
            return f"(split {nat_str(targs[0])} {nat_str(targs[1])} {show(args[0])})"
        if name == "joinAcc" and len(args) == 1:
            return f"(joinAcc {nat_str(targs[1])} {show(args[0])})"
        if name in NEW_SPACE and len(args) == 1:
            return f"({name} {targs[0]} {show(args[0])})"
        if name == "for" and len(args) == 1:
            return f"(for {nat_str(targs[0])} {show(args[0])})"
        if vector_prim(name) and len(args) == 1:
            return f"({name} {show(args[0])})"
        if name in _PLAIN and args:
            return f"({name} {' '.join(show(a) for a in args)})"
    if isinstance(p, App):
        return f"({show(p.fn)} {show(p.arg)})"
    if isinstance(p, TApp):
        arg = nat_str(p.arg) if hasattr(p.arg, "terms") else str(p.arg)
        return f"(tapp {show(p.fn)} {arg})"
    if isinstance(p, Prim):
        return p.name
    raise TypeError(f"not a phrase: {p!r}")


pretty_print = show
