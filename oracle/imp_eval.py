"""ORACLE (test infrastructure only -- never imported by the product path).

Interpreter for purely imperative phrases, restating the reference's Stage-II
semantics (/root/reference/pkg/src/dpia/eval_imp.py:100-307): a store of cells
holding scalar leaves keyed by paths, acceptors as path transformers, parfor
iterations run in order (or reversed) with per-iteration write footprints
checked for disjointness (RaceError).  Extended with this repo's imperative
additions: transposeAcc, the hierarchy-dimension parfor variants and the
cooperative combine reduceILocal (executed as a left fold, its definition).

Used on the CPU to check that Stage I + Stage II of the product front end
compute the functional result (coincidence, TST/test_lower.py:192-197).
"""
from __future__ import annotations

from typing import Callable, Dict, List, Set, Tuple

from paper_1710_08332_b200.dtypes import Array, DataType, Idx, Num, Pair, Vector
from paper_1710_08332_b200.signatures import PARFOR_FAMILY
from paper_1710_08332_b200.terms import Lam, Phrase, Proj, Var, unapply

from .dpia_eval import EvalError, Vec, eval_phrase

Path = Tuple[int, ...]


class ExecError(Exception):
    pass


class RaceError(ExecError):
    pass


def leaves(v, d: DataType, prefix: Path = ()):
    if isinstance(d, (Num, Idx)):
        yield prefix, v
    elif isinstance(d, Vector):
        for k, x in enumerate(v.items):
            yield prefix + (k,), x
    elif isinstance(d, Array):
        for i, item in enumerate(v):
            yield from leaves(item, d.elem, prefix + (i,))
    elif isinstance(d, Pair):
        yield from leaves(v[0], d.fst, prefix + (0,))
        yield from leaves(v[1], d.snd, prefix + (1,))
    else:
        raise ExecError(f"no leaves at type {d}")


class Cell:
    def __init__(self, name: str, dtype: DataType):
        self.name, self.dtype, self.data = name, dtype, {}

    def read(self, sigma, float_mode):
        zero = 0.0 if float_mode else 0

        def build(d, pre):
            if isinstance(d, Idx):
                return self.data.get(pre, 0)
            if isinstance(d, Num):
                return self.data.get(pre, zero)
            if isinstance(d, Vector):
                return Vec(tuple(self.data.get(pre + (k,), zero) for k in range(d.width)))
            if isinstance(d, Array):
                return [build(d.elem, pre + (i,)) for i in range(d.size.evaluate(sigma))]
            return (build(d.fst, pre + (0,)), build(d.snd, pre + (1,)))

        return build(self.dtype, ())


class Ref:
    """An acceptor: a cell plus a path transformer."""

    def __init__(self, cell: Cell, trans: Callable[[Path], Path]):
        self.cell, self.trans = cell, trans

    def at(self, i: int) -> "Ref":
        return Ref(self.cell, lambda p, i=i, t=self.trans: t((i,) + p))

    def map(self, g: Callable[[Path], Path]) -> "Ref":
        return Ref(self.cell, lambda p, t=self.trans: t(g(p)))


class Machine:
    def __init__(self, sigma, float_mode=False, reverse=False):
        self.sigma, self.float_mode, self.reverse = sigma, float_mode, reverse
        self.footprints: List[Set] = []
        self._k = 0

    # environment: name -> plain value | Cell | Ref
    def value_env(self, env):
        out = {}
        for k, b in env.items():
            if isinstance(b, Cell):
                out[k] = (None, b.read(self.sigma, self.float_mode))
            elif not isinstance(b, Ref):
                out[k] = b
        return out

    def exp(self, e, env):
        try:
            return eval_phrase(e, self.value_env(env), self.sigma)
        except EvalError as err:
            raise ExecError(str(err)) from None

    def acc(self, a: Phrase, env) -> Ref:
        if isinstance(a, Var):
            b = env.get(a.name)
            if isinstance(b, Ref):
                return b
            if isinstance(b, Cell):
                return Ref(b, lambda p: p)
            raise ExecError(f"not an acceptor: {a.name}")
        if isinstance(a, Proj) and a.index == 1 and isinstance(a.target, Var) \
                and isinstance(env.get(a.target.name), Cell):
            return Ref(env[a.target.name], lambda p: p)
        u = unapply(a)
        if u is None:
            raise ExecError(f"not an acceptor phrase: {a!r}")
        name, targs, args = u
        if name == "idxAcc":
            r, i = self.acc(args[0], env), self.exp(args[1], env)
            n = targs[0].evaluate(self.sigma)
            if not 0 <= i < n:
                raise ExecError(f"acceptor index {i} out of bounds {n}")
            return r.at(i)
        r = self.acc(args[0], env)
        if name == "splitAcc":
            n = targs[0].evaluate(self.sigma)
            return r.map(lambda p: (p[0] // n, p[0] % n) + p[1:])
        if name == "joinAcc":
            m = targs[1].evaluate(self.sigma)
            return r.map(lambda p: (p[0] * m + p[1],) + p[2:])
        if name == "transposeAcc":
            return r.map(lambda p: (p[1], p[0]) + p[2:])
        if name in ("pairAcc1", "pairAcc2"):
            f = 0 if name == "pairAcc1" else 1
            return r.map(lambda p: (f,) + p)
        if name in ("zipAcc1", "zipAcc2"):
            f = 0 if name == "zipAcc1" else 1
            return r.map(lambda p: (p[0], f) + p[1:])
        if name.startswith("asVectorAcc"):
            w = int(name[len("asVectorAcc"):])
            return r.map(lambda p: (p[0] // w, p[0] % w) + p[1:])
        if name.startswith("asScalarAcc"):
            w = int(name[len("asScalarAcc"):])
            return r.map(lambda p: (p[0] * w + p[1],) + p[2:])
        raise ExecError(f"not an acceptor phrase: {name}")

    def write(self, ref: Ref, value, d):
        for rel, x in leaves(value, d):
            path = ref.trans(rel)
            ref.cell.data[path] = x
            for fp in self.footprints:
                fp.add((ref.cell.name, path))

    def run(self, p: Phrase, env):
        u = unapply(p)
        if u is None:
            raise ExecError(f"not a command: {p!r}")
        name, targs, args = u
        if name in ("skip", "barrier"):
            return
        if name == ";":
            self.run(args[0].fst, env)
            self.run(args[0].snd, env)
        elif name == ":=":
            self.write(self.acc(args[0].fst, env), self.exp(args[0].snd, env), targs[0])
        elif name in ("new", "newGlobal", "newLocal", "newPrivate"):
            f = args[0]
            self._k += 1
            self.run(f.body, {**env, f.binder: Cell(f"{f.binder}@{self._k}", targs[0])})
        elif name == "for":
            f = args[0]
            for i in range(targs[0].evaluate(self.sigma)):
                self.run(f.body, {**env, f.binder: i})
        elif name in PARFOR_FAMILY:
            n = targs[0].evaluate(self.sigma)
            ref, f = self.acc(args[0], env), args[1]
            if not (isinstance(f, Lam) and isinstance(f.body, Lam)):
                raise ExecError("parfor body must be a two-argument lambda")
            prints = [set() for _ in range(n)]
            for i in (range(n - 1, -1, -1) if self.reverse else range(n)):
                self.footprints.append(prints[i])
                try:
                    self.run(f.body.body, {**env, f.binder: i, f.body.binder: ref.at(i)})
                finally:
                    self.footprints.pop()
            seen: Dict = {}
            for i, fp in enumerate(prints):
                for addr in fp:
                    if addr in seen:
                        raise RaceError(f"data race: iterations {seen[addr]} and {i} write {addr}")
                    seen[addr] = i
        elif name == "reduceILocal":
            f, init, src, k = args
            d = targs[1]
            acc = Cell(f"combine@{id(p)}", d)
            self.write(Ref(acc, lambda q: q), self.exp(init, env), d)
            for x in self.exp(src, env):
                tmp = Cell("o", d)
                # f x acc o : a command writing o
                self.run(_apply3(f, x, acc, tmp), {**env, "$x": x, "$acc": acc, "$o": tmp})
                acc = tmp
            self.run(_apply1(k, acc), {**env, "$r": acc})
        else:
            raise ExecError(f"no execution clause for {name!r}")


def _apply3(f, x, acc, o):
    from paper_1710_08332_b200.terms import App, Proj, Var, beta_normalize
    return beta_normalize(App(App(App(f, Var("$x")), Proj(Var("$acc"), 2)), Var("$o")))


def _apply1(k, acc):
    from paper_1710_08332_b200.terms import App, Proj, Var, beta_normalize
    return beta_normalize(App(k, Proj(Var("$r"), 2)))


def run_program(p: Phrase, params, inputs, sigma=None, float_mode=False, reverse_parfor=False):
    """Execute a closed command (eval_imp.py:281-307); returns the final value
    of every out/var parameter."""
    m = Machine(sigma or {}, float_mode, reverse_parfor)
    env, outs = {}, {}
    for name, dtype, mode in params:
        if mode == "in":
            env[name] = inputs[name]
        else:
            cell = Cell(name, dtype)
            if name in inputs:
                for path, x in leaves(inputs[name], dtype):
                    cell.data[path] = x
            env[name] = Ref(cell, lambda q: q) if mode == "out" else cell
            outs[name] = cell
    m.run(p, env)
    return {n: c.read(m.sigma, float_mode) for n, c in outs.items()}
