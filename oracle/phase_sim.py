"""ORACLE (test infrastructure only -- never imported by the product path).

Barrier-aware, phase-synchronous simulator of the CUDA execution model the
backend emits.  The reference's `simulate_kernel`
(SRC/opencl.py:339-472) runs each work-item to completion and treats
`barrier` as a no-op, so multi-phase local-memory kernels simulate wrongly
at L > 1 (SURVEY.md finding 5).  Here every work-item is a coroutine that
yields at each barrier; a work-group advances phase by phase; within a phase
any two work-items that touch the same shared (local or global) address with
at least one write raise `PhaseRace` -- i.e. a barrier the planner should
have placed is missing.  Work-groups of a kernel run one after another and
cross-work-group conflicts on global memory are reported too.

It executes the emitter's *plan* (kernels, fused tails, planned barrier
positions, hoisted stagings, stagings rotated between two slices,
single-thread uniform writes, the cooperative combine), so it checks the
backend's decisions on the CPU at desk scale.
"""
from __future__ import annotations

import itertools
from typing import Dict, List, Optional, Tuple

from paper_1710_08332_b200.cuda.emit import emit_cuda, normalize_launch
from paper_1710_08332_b200.dtypes import Array, Idx, Num, Pair, Vector
from paper_1710_08332_b200.signatures import LOOP_LEVEL, NEW_SPACE, PARFOR_FAMILY
from paper_1710_08332_b200.terms import Lam, Lit, Proj, Var, unapply

from .dpia_eval import Vec, binop, c_divide, unop
from .imp_eval import leaves

PER_THREAD = ("global", "local", "lin", "fold", "lambda")


class PhaseRace(Exception):
    pass


class Cell:
    _ids = itertools.count()

    def __init__(self, name, dtype, shared: bool):
        self.id, self.name, self.dtype, self.shared = next(Cell._ids), name, dtype, shared
        self.data: Dict[tuple, object] = {}


class Alias:
    def __init__(self, acc, i):
        self.acc, self.i = acc, i


class Ctx:
    def __init__(self, sim, g, l, block_store):
        self.sim, self.g, self.l = sim, g, l
        (G, L) = sim.launch
        self.tid = l[1] * L[0] + l[0]
        self.nthreads = L[0] * L[1]
        self.gid = (g[1] * G[0] + g[0]) * self.nthreads + self.tid
        self.gsize = G[0] * G[1] * self.nthreads
        self.levels: List[str] = []
        self.par_idx: Tuple = ()
        self.single_thread = False
        self.block = block_store
        self.reads, self.writes = set(), set()
        self.combine_count: Dict[int, int] = {}

    @property
    def per_thread(self):
        return self.single_thread or any(lv in PER_THREAD for lv in self.levels)


class Sim:
    def __init__(self, p, params, inputs, launch, sigma=None, float_mode=False):
        self.sigma = dict(sigma or {})
        self.launch = normalize_launch(launch)
        self.float_mode = float_mode
        outs = [(n, d) for n, d, m in params if m in ("out", "var")]
        ins = [(n, d) for n, d, m in params if m == "in"]
        _src, self.sig = emit_cuda(p, outs, ins, float_mode=float_mode, sigma=self.sigma,
                                   launch=self.launch)
        self.p = p
        self.env: Dict[str, object] = {}
        self.cells: Dict[str, Cell] = {}
        for n, d, m in params:
            if m == "in":
                self.env[n] = inputs[n]
            else:
                c = Cell(n, d, True)
                if n in inputs:
                    for path, x in leaves(inputs[n], d):
                        c.data[path] = x
                self.env[n] = c
                self.cells[n] = c
        self.global_cells: Dict[tuple, Cell] = {}

    # ------------------------------------------------------------ running
    def run(self):
        top, items = [], []
        self._peel(self.p, top, items)
        for prim, d, binder in top:
            if self.sig.spaces.get(binder, "private") == "global":
                self.env[binder] = Cell(binder, d, True)
        for info in self.sig.kernels:
            (G, L) = self.launch
            kernel_globals = {}
            if info.grid_item is not None:
                for gy in range(G[1]):
                    for gx in range(G[0]):
                        self._run_block(info, [info.grid_item], (gx, gy), kernel_globals, tail=False)
            if info.tail_items:
                self._run_block(info, info.tail_items, (G[0] - 1, G[1] - 1), kernel_globals, tail=True)
        zero = 0.0 if self.float_mode else 0
        return {n: self._read_value(c, c.dtype, (), zero) for n, c in self.cells.items()}

    def _peel(self, p, top, items):
        u = unapply(p)
        if u is not None and u[0] == ";":
            self._peel(u[2][0].fst, top, items)
            self._peel(u[2][0].snd, top, items)
        elif u is not None and u[0] in NEW_SPACE and isinstance(u[2][0], Lam):
            top.append((u[0], u[1][0], u[2][0].binder))
            self._peel(u[2][0].body, top, items)
        else:
            items.append(p)

    def _run_block(self, info, items, g, kernel_globals, tail):
        (G, L) = self.launch
        block_store: Dict = {"combine": {}, "tail": tail}
        ctxs, gens = [], []
        for ly in range(L[1]):
            for lx in range(L[0]):
                ctx = Ctx(self, g, (lx, ly), block_store)
                env = dict(self.env)
                for space, binder, d in info.decls:
                    if space == "local" or self.sig.spaces.get(binder) == "local":
                        key = ("decl", binder)
                        if key not in block_store:
                            block_store[key] = Cell(binder, d, True)
                        env[binder] = block_store[key]
                    elif space == "private":
                        env[binder] = Cell(binder, d, False)
                ctxs.append(ctx)
                gens.append(self._items(items, env, ctx, info, tail))
        live = list(range(len(gens)))
        while live:
            for c in ctxs:
                c.reads, c.writes = set(), set()
            still = []
            for k in live:
                try:
                    next(gens[k])
                    still.append(k)
                except StopIteration:
                    pass
            self._check_phase(ctxs)
            live = still
        # cross-work-group conflicts on global memory within this kernel
        for c in ctxs:
            for addr in getattr(c, "all_writes", ()):
                owner = kernel_globals.setdefault(("w", addr), g)
                if owner != g and not tail:
                    raise PhaseRace(f"work-groups {owner} and {g} both write {addr}")

    def _check_phase(self, ctxs):
        writer: Dict = {}
        for c in ctxs:
            for a in c.writes:
                if a in writer and writer[a] != c.tid:
                    raise PhaseRace(f"work-items {writer[a]} and {c.tid} write {a} in one phase")
                writer[a] = c.tid
        for c in ctxs:
            for a in c.reads:
                if a in writer and writer[a] != c.tid:
                    raise PhaseRace(f"work-item {c.tid} reads {a} written by work-item {writer[a]} "
                                    "in the same phase (missing barrier)")

    def _items(self, items, env, ctx, info, tail):
        for it in items:
            coop = not tail or _cooperative(it)
            if tail and not coop:
                if id(it) in info.barriers:
                    yield
                if ctx.tid == 0:
                    ctx.single_thread = True
                    yield from self._run(it, env, ctx, info)
                    ctx.single_thread = False
            else:
                yield from self._run(it, env, ctx, info)

    # ----------------------------------------------------------- commands
    def _run(self, p, env, ctx, info):
        if id(p) in info.barriers and not ctx.per_thread:
            yield
        name, targs, args = unapply(p)
        if name == "skip":
            return
        if name == "barrier":
            if not ctx.per_thread:
                yield
            return
        if name == ";":
            yield from self._run(args[0].fst, env, ctx, info)
            yield from self._run(args[0].snd, env, ctx, info)
            return
        if name == ":=":
            self._assign(targs[0], args[0].fst, args[0].snd, env, ctx, [])
            return
        if name in NEW_SPACE:
            yield from self._new(name, targs[0], args[0], p, env, ctx, info)
            return
        if name == "for":
            f = args[0]
            for i in range(targs[0].evaluate(self.sigma)):
                yield from self._run(f.body, {**env, f.binder: i}, ctx, info)
            return
        if name in PARFOR_FAMILY:
            yield from self._parfor(name, targs, args, env, ctx, info)
            return
        if name == "reduceILocal":
            yield from self._combine(p, targs, args, env, ctx, info)
            return
        raise RuntimeError(f"phase_sim: no clause for {name}")

    def _level(self, prim, ctx):
        lvl, dim = LOOP_LEVEL[prim]
        if lvl == "plain":
            if ctx.per_thread:
                return "seq", 0
            if "workgroup" in ctx.levels or ctx.block.get("tail"):
                return "lin", 0
            return "global", 0
        return lvl, dim

    def _parfor(self, prim, targs, args, env, ctx, info):
        n = targs[0].evaluate(self.sigma)
        a, f = args
        lvl, dim = self._level(prim, ctx)
        (G, L) = self.launch
        if lvl == "workgroup":
            rng = range(ctx.g[dim], n, G[dim])
        elif lvl == "local":
            rng = range(ctx.l[dim], n, L[dim])
        elif lvl == "lin":
            rng = range(ctx.tid, n, ctx.nthreads)
        elif lvl == "global":
            rng = range(ctx.gid, n, ctx.gsize)
        else:
            rng = range(n)
        body = f.body.body
        hoisted = []
        if lvl == "workgroup" and not ctx.per_thread:
            hoisted = [q for q in _prefix_news(body) if id(q) in info.hoisted]
            for q in hoisted:
                fl = unapply(q)[2][0]
                key = ("hoist", id(q))
                if key not in ctx.block:
                    ctx.block[key] = Cell(fl.binder, unapply(q)[1][0], True)
                c1 = unapply(fl.body)[2][0].fst
                ctx.levels.append("workgroup")
                yield from self._run(c1, {**env, fl.binder: ctx.block[key]}, ctx, info)
                ctx.levels.pop()
            if hoisted:
                yield
        for i in rng:
            ctx.levels.append(lvl)
            old = ctx.par_idx
            if lvl != "seq":
                ctx.par_idx = old + ((f.binder, i),)
            yield from self._run(body, {**env, f.binder: i, f.body.binder: Alias(a, i)}, ctx, info)
            ctx.par_idx = old
            ctx.levels.pop()

    def _new(self, prim, d, f, node, env, ctx, info):
        key = ("hoist", id(node))
        if key in ctx.block:
            inner = unapply(f.body)
            yield from self._run(inner[2][0].snd, {**env, f.binder: ctx.block[key]}, ctx, info)
            return
        space = NEW_SPACE[prim] or "private"
        if space == "private" and self.sig.spaces.get(f.binder) == "local":
            space = "local"     # promoted by the emitter
        if space == "private":
            cell = Cell(f.binder, d, False)
        elif space == "local":
            if ctx.per_thread:
                cell = Cell(f.binder, d, False)
            elif f.binder in info.rotated:
                # the emitter alternates this staging between two slices
                k = ("rot", f.binder, env[info.rotated[f.binder]] % 2)
                if k not in ctx.block:
                    ctx.block[k] = Cell(f.binder, d, True)
                cell = ctx.block[k]
            else:
                k = ("local", f.binder)
                if k not in ctx.block:
                    ctx.block[k] = Cell(f.binder, d, True)
                cell = ctx.block[k]
        else:
            k = (f.binder, ctx.par_idx)
            if k not in self.global_cells:
                self.global_cells[k] = Cell(f.binder, d, True)
            cell = self.global_cells[k]
        yield from self._run(f.body, {**env, f.binder: cell}, ctx, info)

    def _combine(self, node, targs, args, env, ctx, info):
        n = targs[0].evaluate(self.sigma)
        d = targs[1]
        f, init, src, k = args

        def op(x, y):
            o = Cell("o", d, False)
            fx, fy, fo = f.binder, f.body.binder, f.body.body.binder
            self._assign_from(d, f.body.body.body, {**env, fx: x, fy: y, fo: o}, ctx)
            return self._read_value(o, d, (), 0.0 if self.float_mode else 0)

        part, has = None, False
        for j in range(ctx.tid, n, ctx.nthreads):
            x = self._ev(src, env, [j], ctx)
            part = op(x, part) if has else x
            has = True
        inst = ctx.combine_count.get(id(node), 0)
        ctx.combine_count[id(node)] = inst + 1
        slot = ctx.block["combine"].setdefault((id(node), inst), {})
        slot[ctx.tid] = (has, part)
        yield
        tot, any_ = None, False
        for t in sorted(slot):
            h, v = slot[t]
            if h:
                tot = v if not any_ else op(v, tot)
                any_ = True
        yield
        init_v = self._ev(init, env, [], ctx)
        r = op(tot, init_v) if any_ else init_v
        yield from self._run(k.body, {**env, k.binder: r}, ctx, info)

    def _assign_from(self, d, cmd, env, ctx):
        """Run a straight-line command (the body of a combine operator)."""
        for _ in self._run(cmd, env, ctx, _NOPLAN):
            raise RuntimeError("barrier inside a combine operator")

    # --------------------------------------------------------- data paths
    def _assign(self, d, a, e, env, ctx, path):
        if isinstance(d, Pair):
            self._assign(d.fst, a, e, env, ctx, path + [("f", 1)])
            self._assign(d.snd, a, e, env, ctx, path + [("f", 2)])
            return
        if isinstance(d, Vector):
            for lane in range(d.width):
                self._assign(Num(), a, e, env, ctx, path + [lane])
            return
        cell, cpath = self._acc(a, env, path, ctx)
        if cell.shared and not ctx.per_thread and ctx.tid != 0:
            return      # uniform write: thread 0 only
        v = self._ev(e, env, path, ctx)
        cell.data[cpath] = v
        if cell.shared:
            addr = (cell.id, cell.name, cpath)
            ctx.writes.add(addr)
            if not hasattr(ctx, "all_writes"):
                ctx.all_writes = set()
            ctx.all_writes.add(addr)

    def _acc(self, a, env, path, ctx):
        if isinstance(a, Proj) and a.index == 1 and isinstance(a.target, Var):
            a = a.target
        if isinstance(a, Var):
            b = env[a.name]
            if isinstance(b, Alias):
                return self._acc(b.acc, env, [b.i] + path, ctx)
            return b, self._cell_path(b.dtype, path)
        name, targs, args = unapply(a)
        if name == "idxAcc":
            return self._acc(args[0], env, [self._ev(args[1], env, [], ctx)] + path, ctx)
        if name == "splitAcc":
            n = targs[0].evaluate(self.sigma)
            return self._acc(args[0], env, [path[0] // n, path[0] % n] + path[1:], ctx)
        if name == "joinAcc":
            m = targs[1].evaluate(self.sigma)
            return self._acc(args[0], env, [path[0] * m + path[1]] + path[2:], ctx)
        if name == "transposeAcc":
            return self._acc(args[0], env, [path[1], path[0]] + path[2:], ctx)
        if name in ("pairAcc1", "pairAcc2"):
            return self._acc(args[0], env, [("f", int(name[-1]))] + path, ctx)
        if name in ("zipAcc1", "zipAcc2"):
            return self._acc(args[0], env, [path[0], ("f", int(name[-1]))] + path[1:], ctx)
        if name.startswith("asVectorAcc"):
            w = int(name[len("asVectorAcc"):])
            return self._acc(args[0], env, [path[0] // w, path[0] % w] + path[1:], ctx)
        if name.startswith("asScalarAcc"):
            w = int(name[len("asScalarAcc"):])
            return self._acc(args[0], env, [path[0] * w + path[1]] + path[2:], ctx)
        raise RuntimeError(f"phase_sim: acceptor {name}")

    @staticmethod
    def _cell_path(d, path):
        out = []
        for s in path:
            out.append(s[1] - 1 if isinstance(s, tuple) else int(s))
        return tuple(out)

    def _ev(self, p, env, path, ctx):
        if isinstance(p, Proj) and p.index == 2 and isinstance(p.target, Var):
            p = p.target
        if isinstance(p, Var):
            b = env[p.name]
            if isinstance(b, Cell):
                return self._read_cell(b, path, ctx)
            return _index_value(b, path)
        if isinstance(p, Lit):
            if not path and isinstance(p.dtype, Vector):
                return Vec((p.value,) * p.dtype.width)
            return p.value
        name, targs, args = unapply(p)
        if name in ("+", "-", "*", "/"):
            return binop(name, self._ev(args[0].fst, env, path, ctx), self._ev(args[0].snd, env, path, ctx))
        if name in ("negate", "abs"):
            return unop(name, self._ev(args[0], env, path, ctx))
        if name == "idx" or name.startswith("idxVec"):
            return self._ev(args[0], env, [self._ev(args[1], env, [], ctx)] + path, ctx)
        if name == "zip":
            (i, (_f, k)), rest = path[:2], path[2:]
            return self._ev(args[k - 1], env, [i] + rest, ctx)
        if name == "split":
            n = targs[0].evaluate(self.sigma)
            return self._ev(args[0], env, [path[0] * n + path[1]] + path[2:], ctx)
        if name == "join":
            m = targs[1].evaluate(self.sigma)
            return self._ev(args[0], env, [path[0] // m, path[0] % m] + path[1:], ctx)
        if name == "transpose":
            return self._ev(args[0], env, [path[1], path[0]] + path[2:], ctx)
        if name == "pair":
            return self._ev(args[path[0][1] - 1], env, path[1:], ctx)
        if name in ("fst", "snd"):
            return self._ev(args[0], env, [("f", 1 if name == "fst" else 2)] + path, ctx)
        if name.startswith("asVector"):
            w = int(name[len("asVector"):])
            if len(path) == 1:
                return Vec(tuple(self._ev(args[0], env, [path[0] * w + k], ctx) for k in range(w)))
            return self._ev(args[0], env, [path[0] * w + path[1]] + path[2:], ctx)
        if name.startswith("asScalar"):
            w = int(name[len("asScalar"):])
            return self._ev(args[0], env, [path[0] // w, path[0] % w] + path[1:], ctx)
        raise RuntimeError(f"phase_sim: expression {name}")

    def _read_cell(self, cell, path, ctx):
        cp = self._cell_path(cell.dtype, path)
        zero = 0.0 if self.float_mode else 0
        d = cell.dtype
        for s in path:
            if isinstance(d, Array):
                d = d.elem
            elif isinstance(d, Pair):
                d = d.fst if s == ("f", 1) else d.snd
            else:
                d = Num()
        if isinstance(d, Vector):
            out = []
            for k in range(d.width):
                out.append(self._read_leaf(cell, cp + (k,), ctx, zero))
            return Vec(tuple(out))
        return self._read_leaf(cell, cp, ctx, zero)

    def _read_leaf(self, cell, cp, ctx, zero):
        if cell.shared:
            ctx.reads.add((cell.id, cell.name, cp))
        return cell.data.get(cp, zero)

    def _read_value(self, cell, d, pre, zero):
        if isinstance(d, (Num, Idx)):
            return cell.data.get(pre, zero)
        if isinstance(d, Vector):
            return Vec(tuple(cell.data.get(pre + (k,), zero) for k in range(d.width)))
        if isinstance(d, Array):
            return [self._read_value(cell, d.elem, pre + (i,), zero)
                    for i in range(d.size.evaluate(self.sigma))]
        return (self._read_value(cell, d.fst, pre + (0,), zero),
                self._read_value(cell, d.snd, pre + (1,), zero))


class _NoPlan:
    barriers = frozenset()
    hoisted = frozenset()
    rotated: dict = {}


_NOPLAN = _NoPlan()


def _index_value(v, path):
    for s in path:
        if isinstance(s, tuple):
            v = v[s[1] - 1]
        elif isinstance(v, Vec) or hasattr(v, "items") and not isinstance(v, (list, tuple, dict)):
            v = v.items[s]
        else:
            v = v[s]
    return v


def _prefix_news(body):
    out = []

    def walk(q):
        u = unapply(q)
        if u is None:
            return
        if u[0] == ";":
            walk(u[2][0].fst)
            walk(u[2][0].snd)
        elif u[0] in NEW_SPACE and isinstance(u[2][0], Lam):
            out.append(q)
            walk(u[2][0].body)
    walk(body)
    return out


def _cooperative(p):
    from paper_1710_08332_b200.cuda.emit import ProgramEmitter
    return ProgramEmitter.is_cooperative(p)


def simulate(p, params, inputs, launch, sigma=None, float_mode=False):
    """Phase-synchronous execution of the emitted program; raises PhaseRace
    on a missing barrier or a cross-work-group write conflict."""
    return Sim(p, params, inputs, launch, sigma, float_mode).run()


del c_divide, Optional
