"""Closed phrase types of every primitive, plus the family tables the passes
dispatch on.

Covers the reference table (`SRC/primitives.py:59-164`) and the additions this
backend needs for the benchmark strategies (all absent from the reference,
SURVEY.md section 0 finding 1):

* ``transpose`` / ``transposeAcc``   -- layout swap of the two outer dimensions
* ``abs``                              -- numeric absolute value (like negate)
* ``reduceSeq``                        -- spelling of the sequential ``reduce``
* ``reduceLocal`` / ``reduceILocal``   -- work-group cooperative combine of an
  associative, commutative operator (semantics: identical to ``reduce``)
* ``mapWorkgroup1`` / ``mapLocal1`` (+ mapI / parfor forms) -- second hierarchy
  dimension (blockIdx.y / threadIdx.y)
* ``reduceIInit``                      -- reduceI whose initial value is written
  by a command (acceptor translation of a non-trivial init expression)
* ``idxVec{w}``                         -- lane of a vector, written (idx v k)
* ``let``                              -- (let E (lam x B)): E materialised once
  and shared by every use of x in B (the reference has no sharing construct,
  so a staged value used inside a nested map is re-staged per iteration,
  SURVEY.md section 7 hard part 6)
"""
from __future__ import annotations

from typing import Dict, Optional, Tuple

from .dtypes import (NUM, AccT, Array, CommT, DataVar, DepFnT, ExpT, FnT, Idx,
                     Pair, PhraseType, ProdT, VECTOR_WIDTHS, Vector, var_t)
from .sizes import nat

COMM = CommT()
_n, _m = nat("n"), nat("m")
_d, _d1, _d2 = DataVar("d"), DataVar("d1"), DataVar("d2")


def _forall(spec: str, body: PhraseType) -> PhraseType:
    """_forall("n:nat d1:data", T) -> (forall (n nat) (forall (d1 data) T))."""
    for item in reversed(spec.split()):
        name, kind = item.split(":")
        body = DepFnT(name, kind, body)
    return body


def _arrow(*ts: PhraseType, passive_last: bool = False) -> PhraseType:
    out = ts[-1]
    for i, t in enumerate(reversed(ts[:-1])):
        out = FnT(t, out, passive=(passive_last and i == 0))
    return out


def E(d):
    return ExpT(d)


def A(d):
    return AccT(d)


def EA(n, d):
    return ExpT(Array(n, d))


def AA(n, d):
    return AccT(Array(n, d))


# body function of mapI / parfor: exp d1 ->p acc d2 -> comm
_mapi_body = FnT(E(_d1), FnT(A(_d2), COMM, passive=True))
_MAP_T = _forall("n:nat d1:data d2:data", _arrow(_arrow(E(_d1), E(_d2)), EA(_n, _d1), EA(_n, _d2)))
_MAPI_T = _forall("n:nat d1:data d2:data", _arrow(_mapi_body, EA(_n, _d1), AA(_n, _d2), COMM))
_PARFOR_T = _forall("n:nat d:data", _arrow(AA(_n, _d), FnT(E(Idx(_n)), FnT(A(_d), COMM, passive=True)),
                                           COMM))
_NEW_T = _forall("d:data", _arrow(_arrow(var_t(_d), COMM), COMM))
_BINOP_T = _forall("d:data", _arrow(ProdT(E(_d), E(_d)), E(_d)))
_UNOP_T = _forall("d:data", _arrow(E(_d), E(_d)))
_REDUCE_T = _forall("n:nat d1:data d2:data",
                    _arrow(_arrow(E(_d1), E(_d2), E(_d2)), E(_d2), EA(_n, _d1), E(_d2)))
_COMBINE_T = _forall("n:nat d:data", _arrow(_arrow(E(_d), E(_d), E(_d)), E(_d), EA(_n, _d), E(_d)))
_REDUCEI_F = _arrow(E(_d1), E(_d2), A(_d2), COMM)
_TO_SPACE_T = _forall("d1:data d2:data", _arrow(_arrow(E(_d1), E(_d2)), E(_d1), E(_d2)))

MAP_FAMILY = ("map", "mapGlobal", "mapWorkgroup", "mapWorkgroup1", "mapLocal", "mapLocal1",
              "mapSeq")
MAPI_FAMILY = ("mapI", "mapIGlobal", "mapIWorkgroup", "mapIWorkgroup1", "mapILocal",
               "mapILocal1", "mapISeq")
PARFOR_FAMILY = ("parfor", "parforGlobal", "parforWorkgroup", "parforWorkgroup1", "parforLocal",
                 "parforLocal1")
REDUCE_FAMILY = ("reduce", "reduceSeq")
MAP_TO_MAPI = dict(zip(MAP_FAMILY, MAPI_FAMILY))
MAPI_TO_PARFOR = {mi: pf for mi, pf in zip(MAPI_FAMILY, PARFOR_FAMILY + ("for",)) if pf != "for"}
TO_SPACE = {"toGlobal": "global", "toLocal": "local", "toPrivate": "private"}
NEW_SPACE = {"new": None, "newGlobal": "global", "newLocal": "local", "newPrivate": "private"}
SPACE_NEW = {None: "new", "global": "newGlobal", "local": "newLocal", "private": "newPrivate"}
ARITH_OPS = ("+", "-", "*", "/")
UNARY_OPS = ("negate", "abs")

# hierarchy level of each parallel loop form: (level, dimension)
LOOP_LEVEL: Dict[str, Tuple[str, int]] = {
    "parfor": ("plain", 0), "parforGlobal": ("global", 0),
    "parforWorkgroup": ("workgroup", 0), "parforWorkgroup1": ("workgroup", 1),
    "parforLocal": ("local", 0), "parforLocal1": ("local", 1),
}

PRIMITIVES: Dict[str, PhraseType] = {
    "negate": _UNOP_T, "abs": _UNOP_T,
    "+": _BINOP_T, "-": _BINOP_T, "*": _BINOP_T, "/": _BINOP_T,
    "reduce": _REDUCE_T, "reduceSeq": _REDUCE_T, "reduceLocal": _COMBINE_T,
    # let: E is materialised once (by its continuation translation) and bound
    "let": _forall("d1:data d2:data", _arrow(E(_d1), _arrow(E(_d1), E(_d2)), E(_d2))),
    "zip": _forall("n:nat d1:data d2:data", _arrow(EA(_n, _d1), EA(_n, _d2), EA(_n, Pair(_d1, _d2)))),
    "split": _forall("n:nat m:nat d:data", _arrow(EA(_n * _m, _d), EA(_m, Array(_n, _d)))),
    "join": _forall("n:nat m:nat d:data", _arrow(EA(_n, Array(_m, _d)), EA(_n * _m, _d))),
    "transpose": _forall("n:nat m:nat d:data", _arrow(EA(_n, Array(_m, _d)), EA(_m, Array(_n, _d)))),
    "pair": _forall("d1:data d2:data", _arrow(E(_d1), E(_d2), E(Pair(_d1, _d2)))),
    "fst": _forall("d1:data d2:data", _arrow(E(Pair(_d1, _d2)), E(_d1))),
    "snd": _forall("d1:data d2:data", _arrow(E(Pair(_d1, _d2)), E(_d2))),
    "skip": COMM,
    "barrier": COMM,
    ";": _arrow(ProdT(COMM, COMM), COMM),
    ":=": _forall("d:data", _arrow(ProdT(A(_d), E(_d)), COMM)),
    "for": _forall("n:nat", _arrow(_arrow(E(Idx(_n)), COMM), COMM)),
    "splitAcc": _forall("n:nat m:nat d:data", _arrow(AA(_m, Array(_n, _d)), AA(_n * _m, _d))),
    "joinAcc": _forall("n:nat m:nat d:data", _arrow(AA(_n * _m, _d), AA(_n, Array(_m, _d)))),
    "transposeAcc": _forall("n:nat m:nat d:data", _arrow(AA(_m, Array(_n, _d)), AA(_n, Array(_m, _d)))),
    "pairAcc1": _forall("d1:data d2:data", _arrow(A(Pair(_d1, _d2)), A(_d1))),
    "pairAcc2": _forall("d1:data d2:data", _arrow(A(Pair(_d1, _d2)), A(_d2))),
    "zipAcc1": _forall("n:nat d1:data d2:data", _arrow(AA(_n, Pair(_d1, _d2)), AA(_n, _d1))),
    "zipAcc2": _forall("n:nat d1:data d2:data", _arrow(AA(_n, Pair(_d1, _d2)), AA(_n, _d2))),
    "idx": _forall("n:nat d:data", _arrow(EA(_n, _d), E(Idx(_n)), E(_d))),
    "idxAcc": _forall("n:nat d:data", _arrow(AA(_n, _d), E(Idx(_n)), A(_d))),
    "reduceI": _forall("n:nat d1:data d2:data",
                       _arrow(_REDUCEI_F, E(_d2), EA(_n, _d1), _arrow(E(_d2), COMM), COMM)),
    "reduceIInit": _forall("n:nat d1:data d2:data",
                           _arrow(_REDUCEI_F, _arrow(A(_d2), COMM), EA(_n, _d1),
                                  _arrow(E(_d2), COMM), COMM)),
    "reduceILocal": _forall("n:nat d:data",
                            _arrow(_arrow(E(_d), E(_d), A(_d), COMM), E(_d), EA(_n, _d),
                                   _arrow(E(_d), COMM), COMM)),
}
for _name in MAP_FAMILY:
    PRIMITIVES[_name] = _MAP_T
for _name in MAPI_FAMILY:
    PRIMITIVES[_name] = _MAPI_T
for _name in PARFOR_FAMILY:
    PRIMITIVES[_name] = _PARFOR_T
for _name in NEW_SPACE:
    PRIMITIVES[_name] = _NEW_T
for _name in TO_SPACE:
    PRIMITIVES[_name] = _TO_SPACE_T
for _w in VECTOR_WIDTHS:
    _v = Vector(_w)
    PRIMITIVES[f"asVector{_w}"] = _forall("m:nat", _arrow(EA(_m * _w, NUM), EA(_m, _v)))
    PRIMITIVES[f"asScalar{_w}"] = _forall("m:nat", _arrow(EA(_m, _v), EA(_m * _w, NUM)))
    PRIMITIVES[f"asVectorAcc{_w}"] = _forall("m:nat", _arrow(AA(_m, _v), AA(_m * _w, NUM)))
    PRIMITIVES[f"asScalarAcc{_w}"] = _forall("m:nat", _arrow(AA(_m * _w, NUM), AA(_m, _v)))
    # lane of a vector: surface syntax (idx v k) at vector type
    PRIMITIVES[f"idxVec{_w}"] = _arrow(E(_v), E(Idx(nat(_w))), E(NUM))


def primitive_type(name: str) -> PhraseType:
    try:
        return PRIMITIVES[name]
    except KeyError:
        raise KeyError(f"unknown primitive: {name}") from None


def vector_prim(name: str) -> Optional[Tuple[str, int]]:
    """('asVector'|'asScalar'|'asVectorAcc'|'asScalarAcc', width) or None."""
    for prefix in ("asVectorAcc", "asScalarAcc", "asVector", "asScalar"):
        if name.startswith(prefix) and name[len(prefix):].isdigit():
            return prefix, int(name[len(prefix):])
    return None


# primitives that may appear in a purely imperative (post Stage II) phrase
IMPERATIVE_PRIMS = (
    {"skip", "barrier", ";", ":=", "for", "idx", "idxAcc", "negate", "abs", "split", "join",
     "transpose", "zip", "pair", "fst", "snd", "splitAcc", "joinAcc", "transposeAcc", "pairAcc1",
     "pairAcc2", "zipAcc1", "zipAcc2", "reduceILocal"}
    | set(PARFOR_FAMILY) | set(NEW_SPACE) | set(ARITH_OPS)
    | {f"{p}{w}" for p in ("asVector", "asScalar", "asVectorAcc", "asScalarAcc", "idxVec")
       for w in VECTOR_WIDTHS}
)
INTERMEDIATE_PRIMS = set(MAPI_FAMILY) | {"reduceI", "reduceIInit"}
