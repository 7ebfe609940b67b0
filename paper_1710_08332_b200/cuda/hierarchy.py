"""Reference-compatible hierarchy utilities.

`hoist_allocations` and `lint_hierarchy` keep the signatures and meaning of
the reference's `SRC/opencl.py:124-198` so that its callers (CLI compile
path, fuzz harness) port unchanged:

* hoisting lifts newGlobal/newLocal to the top of the command, growing each
  buffer by one array layer per enclosing loop that would otherwise share it
  (global: every loop; local: every loop except the work-group ones) and
  rewriting uses to index the slice -- the reference's policy.  The CUDA
  emitter accepts this form, but does not need it: given the unhoisted
  Stage II phrase it places buffers itself and reuses shared slices across
  sequential iterations instead of multiplying them.
* lint reports the hierarchy nestings the CUDA backend rejects, with the
  reference's messages, extended to the second dimension (nesting a
  work-group loop of the other dimension is legal).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple

from ..dtypes import Array, DataType
from ..signatures import LOOP_LEVEL, NEW_SPACE, PARFOR_FAMILY
from ..terms import (Lam, PairP, Phrase, Proj, Var, apply_prim, beta_normalize,
                     children, rebuild, substitute, unapply)


@dataclass(frozen=True)
class HoistedBuffer:
    name: str
    dtype: DataType
    space: str  # "global" | "local"


def hoist_allocations(p: Phrase) -> Tuple[Phrase, List[HoistedBuffer]]:
    """Lift every newGlobal/newLocal to the top (SRC/opencl.py:124)."""
    bufs: List[HoistedBuffer] = []
    counter = [0]

    def lift(q: Phrase, loops) -> Phrase:
        u = unapply(q)
        if u is not None:
            name, targs, args = u
            if name in ("newGlobal", "newLocal") and len(args) == 1 and isinstance(args[0], Lam):
                f = args[0]
                space = NEW_SPACE[name]
                chain = [lp for lp in loops if space == "global" or lp[0] != "workgroup"]
                d = targs[0]
                for _lvl, _v, n in reversed(chain):
                    d = Array(n, d)
                counter[0] += 1
                hname = f"{f.binder}_h{counter[0]}"
                bufs.append(HoistedBuffer(hname, d, space))
                acc: Phrase = Proj(Var(hname), 1)
                exp: Phrase = Proj(Var(hname), 2)
                layer = d
                for _lvl, v, n in chain:
                    layer = layer.elem
                    acc = apply_prim("idxAcc", [n, layer], [acc, Var(v)])
                    exp = apply_prim("idx", [n, layer], [exp, Var(v)])
                return lift(substitute(f.body, f.binder, PairP(acc, exp)), loops)
            if name in PARFOR_FAMILY and len(args) == 2 and isinstance(args[1], Lam) \
                    and isinstance(args[1].body, Lam):
                a, f = args
                lvl = LOOP_LEVEL[name][0]
                lvl = "global" if lvl == "plain" else lvl
                inner = lift(f.body.body, loops + [(lvl, f.binder, targs[0])])
                return apply_prim(name, targs, [a, Lam(f.binder, Lam(f.body.binder, inner,
                                                                       f.body.arg_type), f.arg_type)])
            if name == "for" and len(args) == 1 and isinstance(args[0], Lam):
                f = args[0]
                inner = lift(f.body, loops + [("seq", f.binder, targs[0])])
                return apply_prim("for", targs, [Lam(f.binder, inner, f.arg_type)])
        return rebuild(q, lambda c: lift(c, loops))

    body = beta_normalize(lift(p, []))
    for b in reversed(bufs):
        body = apply_prim("newGlobal" if b.space == "global" else "newLocal", [b.dtype],
                          [Lam(b.name, body)])
    return body, bufs


def lint_hierarchy(p: Phrase) -> List[str]:
    """Hierarchy nestings the CUDA backend rejects (SRC/opencl.py:139)."""
    out: List[str] = []

    def walk(q: Phrase, enclosing: List[Tuple[str, int]]):
        u = unapply(q)
        if u is not None and u[0] in PARFOR_FAMILY and len(u[2]) == 2:
            lvl, dim = LOOP_LEVEL[u[0]]
            levels = [e[0] for e in enclosing]
            if lvl == "workgroup":
                if "local" in levels:
                    out.append("work-group-level loop nested inside a work-item-level loop")
                if (lvl, dim) in enclosing:
                    out.append("nested work-group-level loops")
                if "global" in levels:
                    out.append("work-group-level loop nested inside a global-level loop")
            elif lvl == "local":
                if (lvl, dim) in enclosing:
                    out.append("nested work-item-level loops")
                if "workgroup" not in levels:
                    out.append("work-item-level loop with no enclosing work-group-level loop")
                if "global" in levels:
                    out.append("work-item-level loop nested inside a global-level loop")
            elif lvl == "global":
                if "workgroup" in levels or "local" in levels:
                    out.append("global-level loop nested inside the work-group hierarchy")
                if "global" in levels:
                    out.append("nested global-level loops")
            a, f = u[2]
            walk(a, enclosing)
            walk(f, enclosing + ([] if lvl == "plain" else [(lvl, dim)]))
            return
        for c in children(q):
            walk(c, enclosing)

    walk(p, [])
    return out


def cuda_legal(p: Phrase) -> bool:
    return not lint_hierarchy(p)


class WorkItemRace(Exception):
    """Parallel iterations write the same location -- the CUDA counterpart
    of the reference's `WorkItemRace` (SRC/opencl.py:327-336), which its
    work-item simulator raises from write footprints (:465-470)."""

    def __init__(self, loop: str, target: str):
        super().__init__(f"cross-work-item write overlap: every iteration of {loop} writes "
                         f"{target} at an index that does not depend on the iteration")
        self.loop, self.target = loop, target


def _free_names(q: Phrase) -> set:
    if isinstance(q, Var):
        return {q.name}
    if isinstance(q, Lam):
        return _free_names(q.body) - {q.binder}
    return set().union(*[_free_names(c) for c in children(q)]) if children(q) else set()


def check_work_item_races(p: Phrase) -> None:
    """Reject parallel loops whose iterations all write one location of an
    identifier captured from outside the loop (not through the loop's own
    acceptor): an assignment rooted at a captured identifier must index it
    with an expression that depends on the iteration variable somewhere on
    its access path.  Stage I/II output never does this (the translation is
    race-free by construction, SRC/checker.py); the reference's hoisted form
    indexes its hoisted buffers by the loop variable, which passes."""

    def root_and_indices(a: Phrase):
        idxs = []
        while True:
            if isinstance(a, Var):
                return a.name, idxs
            if isinstance(a, Proj) and isinstance(a.target, Var):
                return a.target.name, idxs
            u = unapply(a)
            if u is None or not u[2]:
                return None, idxs
            name, _targs, args = u
            if name == "idxAcc" and len(args) == 2:
                idxs.append(args[1])
            a = args[0]

    def walk(q: Phrase, loops: List[Tuple[str, str, set]]):
        u = unapply(q)
        if u is not None:
            name, targs, args = u
            if name in PARFOR_FAMILY and len(args) == 2 and isinstance(args[1], Lam) \
                    and isinstance(args[1].body, Lam):
                a, f = args
                walk(a, loops)
                for _lname, _ivar, own in loops:
                    own.update((f.binder, f.body.binder))
                inner = loops + [(name, f.binder, {f.body.binder})]
                walk(f.body.body, inner)
                return
            if name == ":=" and args and isinstance(args[0], PairP):
                root, idxs = root_and_indices(args[0].fst)
                if root is not None:
                    used = set().union(*[_free_names(e) for e in idxs]) if idxs else set()
                    for lname, ivar, own in reversed(loops):
                        if root in own:
                            break          # written through this loop's acceptor
                        if ivar not in used:
                            raise WorkItemRace(f"{lname} over {ivar}", root)
        if isinstance(q, Lam):
            # names bound inside a loop (new* buffers, for/inner binders) are
            # per-iteration, not captured
            for _lname, _ivar, own in loops:
                own.add(q.binder)
            walk(q.body, loops)
            return
        for c in children(q):
            walk(c, loops)

    walk(p, [])
