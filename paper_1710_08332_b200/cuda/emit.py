"""CUDA C emitter for purely imperative DPIA (Stage III for sm_100a).

Replaces the reference's OpenCL backend (`SRC/opencl.py:124-314` with the
opencl dialect of `SRC/codegen_c.py` / `SRC/c_ast.py`).  The input is a Stage
II phrase (or the reference's hoisted form); the output is one CUDA
translation unit with one `__global__` function per *phase*.

Strategy preservation -- each hierarchy annotation becomes one CUDA construct:

  parforGlobal        grid-stride loop over the linear global thread id
  parforWorkgroup{,1} blockIdx.{x,y} loop (stride gridDim)
  parforLocal{,1}     threadIdx.{x,y} loop (stride blockDim)
  parfor (plain)      the innermost free level: global at kernel top level,
                      all threads of the block at work-group level,
                      sequential inside a work item
  for                 sequential loop (#pragma unroll when small & constant)
  newLocal            __shared__ staging (one arena, static offsets)
  newPrivate          registers (per-thread arrays; thread-sliced, below)
  newGlobal           device scratch buffer, one slice per parallel iteration
  asVector/asScalar   whole-vector dpia::vec loads/stores (LDG/STG.128)
  reduceILocal        dpia::block_combine (warp shuffles + one smem hop)

Additions over the reference backend (SURVEY.md sections 0 and 7):
  * access-path resolution with 64-bit-safe, range-simplified subscripts;
  * barrier placement for RAW, WAR and loop-carried hazards on shared
    buffers at work-group-uniform program points (the reference misses the
    loop-carried case);
  * shared buffers inside sequential loops are reused, not multiplied by the
    trip count (SURVEY.md finding 4);
  * thread slicing: a private buffer declared at work-group level whose every
    access is indexed by this thread's local ids keeps only its own slice;
  * writes to shared/global memory at work-group-uniform points are made by
    one thread (the reference rejects such programs as not fully parallel);
  * phase splitting at grid-wide dependences, with a single-work-group tail
    phase fused into the preceding grid phase by last-block-done detection.
"""
from __future__ import annotations

import os
import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Set, Tuple, Union

from ..dtypes import Array, DataType, Idx, Num, Pair, Vector
from ..signatures import LOOP_LEVEL, NEW_SPACE, PARFOR_FAMILY
from ..sizes import Nat, nat
from ..terms import (Lam, Lit, PairP, Phrase, Prim, Proj, Var, free_vars, seq_all,
                     subtree_iter, unapply)
from . import index as IX
from .ctypes_map import CudaError, TypeTable, split_array
from .index import Ix, div, ix, mod, render

HEADER_PATH = os.path.join(os.path.dirname(os.path.dirname(__file__)), "csrc", "dpia_device.cuh")
UNROLL_LIMIT = 64
# sequential folds inside a work-item read unit-stride global data as
# VEC_WIDTH-wide vectors (KernelEmitter._vec_loop); DPIA_VEC_LOADS=0 disables
VEC_LOADS = os.environ.get("DPIA_VEC_LOADS", "1") != "0"
VEC_WIDTH = 4
# also vectorise folds of at most UNROLL_LIMIT iterations (DPIA_VEC_SHORT=0: only longer ones)
VEC_SHORT = os.environ.get("DPIA_VEC_SHORT", "1") != "0"
# ... and read shared-memory operands of such folds as whole vectors too
# (LDS.128: the single-thread fold of a work-group's staged partials)
VEC_LOCAL = os.environ.get("DPIA_VEC_LOCAL", "0") == "1"   # (off: no measured gain, the compiler merges them)
# L2 prefetch of a work-item fold's next work-group iteration (`_prefetch_next_group`)
PREFETCH_NEXT = os.environ.get("DPIA_PREFETCH_NEXT", "1") != "0"
# ... and each read stream of a work-item's fold keeps VEC_PREFETCH queue
# slots in flight (a rotating register queue refilled VEC_PREFETCH slots
# ahead; 0 disables).  A slot is one VEC_LOAD_BYTES vector: 32 = one sm_100
# 256-bit load (LDG.E.256: half the L1 wavefronts per byte of a work-item's
# own -- uncoalesced -- chunk, tools/chunkread.py), 16 = LDG.128.
VEC_PREFETCH = int(os.environ.get("DPIA_VEC_PREFETCH", "8"))
VEC_LOAD_BYTES = int(os.environ.get("DPIA_VEC_LOAD_BYTES", "32"))
# A single thread's fold (the top-level sequential reduce of a fused tail)
# streams its data through a shared-memory ring of TAIL_RING_STAGES TMA bulk
# copies of TAIL_RING_BYTES per stream; DPIA_TAIL_RING=0 uses the register
# queue instead.
TAIL_RING = os.environ.get("DPIA_TAIL_RING", "1") != "0"
# A program's first kernel can be chained behind the previous launch on its
# stream with programmatic dependent launch (Executable.launch(chain=True)):
# it waits for that grid only before touching non-input global memory
# (ProgramEmitter._chain_waits); DPIA_CHAIN=0 emits no chaining code.
CHAIN = os.environ.get("DPIA_CHAIN", "1") != "0"
# where a chained first kernel lets its dependent launch: "top" (at once),
# "wait" (after its first wait for the previous grid) or "auto" (ProgramEmitter
# .emit_kernel: "wait" for small grids that store outputs, else "top")
CHAIN_TRIGGER = os.environ.get("DPIA_CHAIN_TRIGGER", "auto")
TAIL_RING_STAGES = int(os.environ.get("DPIA_TAIL_RING_STAGES", "4"))
TAIL_RING_BYTES = int(os.environ.get("DPIA_TAIL_RING_BYTES", "2048"))
TAIL_RING_UNROLL = int(os.environ.get("DPIA_TAIL_RING_UNROLL", "16"))
# block-invariant identity stagings of an input into shared memory as one
# bulk (TMA) copy: KernelEmitter.bulk_stage; DPIA_BULK_STAGE=0 emits the
# work-item copy loop instead
BULK_STAGE = os.environ.get("DPIA_BULK_STAGE", "1") != "0"
# work-item loops of a pipelined staging may take up to this many iterations
# per thread (unrolled into guarded copies, one prefetch register set each)
PF_MAX_COPIES = 4
# a rotating toLocal k-tile that is a plain 2-D box of an input can be staged
# by TMA tensor copies (cp.async.bulk.tensor.2d + mbarrier) instead of
# register prefetch + shared stores: KernelEmitter._tma_plan.  Off unless a
# program asks (emit_cuda(tma_tiles=True)) or DPIA_TMA_TILES=1: on the mm
# config it is bit-identical and 1-2% slower than the register path
# (profiles/r02c_tma_mm.txt)
TMA_TILES = os.environ.get("DPIA_TMA_TILES", "0") == "1"
TMA_PROBE_MAX = 1 << 16            # copy statements the box probe may enumerate
# streaming tail: a kernel whose grid phase is a mapGlobal writing one partial
# per work-item and whose tail is one thread's in-order fold of the partials
# through the TMA bulk ring runs the tail in ONE extra block from the start:
# work-item rounds publish on per-round counters and the tail folds round r
# while rounds > r still run (ProgramEmitter._stream_plan); DPIA_STREAM_TAIL=0
# keeps the last-block ticket tail
STREAM_TAIL = os.environ.get("DPIA_STREAM_TAIL", "1") != "0"
# pipelined streaming tail: the partials and round counters are double-
# buffered by launch parity (an epoch kernel argument), so a launch chained
# behind the previous one waits only for the launch two back to release its
# parity, and for the previous grid only before it writes its outputs --
# consecutive launches' serial tails run concurrently (DPIA_STREAM_PIPE=0:
# the launch waits for the previous grid before it first writes the partials)
STREAM_PIPE = os.environ.get("DPIA_STREAM_PIPE", "1") != "0"
# slices of a pipelined streaming tail's partials and counters: launch e uses
# slice e % K and waits for launch e - K to release it
STREAM_PIPE_SLOTS = max(2, int(os.environ.get("DPIA_STREAM_PIPE_SLOTS", "4")))
EPOCH_BASE = 16                 # the launcher's first epoch (launcher.Executable._epoch)
# work-item row folds: a long sequential fold of each work-item of a
# mapGlobal over its own contiguous chunk of an input (config 1's literal
# reduceSeq) reads the chunks of a warp's 32 consecutive work-items as 2-D TMA
# boxes (32 rows x 128 bytes, 128-byte swizzle) through a per-warp ring of
# ROW_TMA_STAGES shared-memory slots, each lane folding its own row:
# KernelEmitter._finish_rows; DPIA_ROW_TMA=0 keeps the register queues
ROW_TMA = os.environ.get("DPIA_ROW_TMA", "1") != "0"
ROW_TMA_STAGES = int(os.environ.get("DPIA_ROW_TMA_STAGES", "4"))
ROW_TMA_BOXES = int(os.environ.get("DPIA_ROW_TMA_BOXES", "2"))    # 128-byte box columns per step
ROW_TMA_INFLIGHT = int(os.environ.get("DPIA_ROW_TMA_INFLIGHT", str(32 * 1024)))  # bytes per warp (64 KiB measured slower)
# a row fold's merged vector stores to an output leave through TMA tensor
# stores of the warp's rows (KernelEmitter._finish_rows)
ROW_TMA_STORE = os.environ.get("DPIA_ROW_TMA_STORE", "1") != "0"
# slices of a TMA-staged tile: 2 -- iteration k+1's box is issued right after
# iteration k's CTA barrier; 3 -- it is issued at the top of iteration k, into
# the slice iteration k-2 read (free since iteration k-1's barrier)
TMA_SLOTS = int(os.environ.get("DPIA_TMA_SLOTS", "3"))
# row bands a box is issued in (one per warp, lane 0); 1 = thread 0 issues
TMA_BANDS = int(os.environ.get("DPIA_TMA_BANDS", "1"))


class _ProbeFail(Exception):
    """The staging command is not a plain box copy (KernelEmitter._tma_plan)."""
# bank-conflict layout of local buffers whose rows are a multiple of 32
# scalars (see KernelEmitter._declare_local): swizzle | pad | none
SMEM_LAYOUT = os.environ.get("DPIA_SMEM_LAYOUT", "swizzle")
# 1-D shared buffers read at a work-item stride that is a multiple of 32
# scalars get 4 scalars of padding per 32 (KernelEmitter._declare_local)
SMEM_PAD_1D = os.environ.get("DPIA_SMEM_PAD_1D", "1") != "0"
# count reads by a one-item work-item loop too (the single work-item that
# folds a work-group's staged partials): padding that buffer measured
# 66.6 against 93.2 us on the reference's gemv (same SASS shape, the padded
# layout schedules better); DPIA_PAD_SINGLE=0 skips them
PAD_SINGLE = os.environ.get("DPIA_PAD_SINGLE", "1") == "1"


class NeedLanes(Exception):
    """A whole-vector access has to be split into lanes."""


# ---------------------------------------------------------------- bindings

@dataclass
class Buffer:
    key: str                 # phrase-level binder
    cname: str
    space: str               # in | out | global | local | private
    dtype: DataType          # full type, hoisting dims included
    prefix: List[Ix] = field(default_factory=list)
    sliced: int = 0
    pad: int = 0             # scalars added to the innermost row stride (shared-memory banks)
    swz: Optional[Tuple[int, int, int]] = None   # (unit, div, period): inner ^= unit*((outer/div)%period)
    pad32: int = 0           # 1-D shared buffer: scalars of padding after every 32 (bank-conflict padding)

    @property
    def dims(self):
        return split_array(self.dtype)[0]

    @property
    def elem(self):
        return split_array(self.dtype)[1]


@dataclass
class Val:
    dtype: DataType
    text: Optional[str] = None
    ixv: Optional[Ix] = None


@dataclass
class Alias:
    """The per-iteration acceptor `o` of a parfor: (idxAcc a i)."""
    acc: Phrase
    i: Ix


@dataclass
class Ref:
    buf: Buffer
    flat: Optional[Ix]       # logical flat index (alignment reasoning)
    suffix: str
    text: str
    addr: Optional[Ix] = None    # physical flat index when the buffer is swizzled

    @property
    def at(self) -> Optional[Ix]:
        return self.addr if self.addr is not None else self.flat


@dataclass
class VStore:
    ref: Ref
    width: int


@dataclass
class Loop:
    level: str          # global workgroup local lin seq fold lambda
    dim: int
    var: str
    trip: Optional[int]
    trip_nat: Nat
    single: bool = False


Step = Tuple[str, object]   # ("i", Ix) | ("f", 1|2)


# ------------------------------------------------------------ signatures

@dataclass
class KernelInfo:
    name: str
    grid: str                # "launch" (user launch) or "single" (one block)
    args: List[Tuple[str, str]]   # (kind, name): kind in out/in/scratch/size/counter
    smem: int
    fused_tail: bool
    # execution plan, for the phase-synchronous simulator (oracle/phase_sim.py)
    grid_item: Optional[Phrase] = field(default=None, repr=False)
    tail_items: List[Phrase] = field(default_factory=list, repr=False)
    barriers: frozenset = field(default=frozenset(), repr=False)     # ids: barrier before node
    hoisted: frozenset = field(default=frozenset(), repr=False)      # ids: LICM-staged newLocal
    rotated: Dict[str, str] = field(default_factory=dict, repr=False)  # buffer -> its loop binder
    decls: List = field(default_factory=list, repr=False)            # kernel-level buffers
    extra_blocks: int = 0        # blocks launched beyond the user's grid (a streaming tail block)
    counter_words: int = 4       # 32-bit words of the kernel's counter buffer
    counter_init: List[Tuple[int, int]] = field(default_factory=list, repr=False)  # (word, value) after zeroing


@dataclass
class CudaSignature:
    outputs: List[Tuple[str, DataType]]
    inputs: List[Tuple[str, DataType]]
    buffers: List[Tuple[str, DataType]]     # device scratch (global) buffers
    sizes: List[str]                          # runtime size arguments (unspecialised)
    kernels: List[KernelInfo]
    scalar: str
    launch: Optional[Tuple[Tuple[int, int], Tuple[int, int]]]
    sigma: Optional[Dict[str, int]]
    spaces: Dict[str, str] = field(default_factory=dict, repr=False)   # buffer binder -> space
    align: Dict[str, int] = field(default_factory=dict, repr=False)    # buffer -> bytes (> 16) its loads need
    # tensor-map parameter -> (input, element bytes, rows, cols, row pitch bytes, box rows, box cols,
    # swizzle bytes)
    tmaps: Dict[str, Tuple[str, int, int, int, int, int, int, int]] = field(default_factory=dict, repr=False)

    def params(self) -> List[str]:
        out = [f"{self.scalar} *{n}" for n, _ in self.outputs]
        out += [f"const {self.scalar} *__restrict__ {n}" for n, _ in self.inputs]
        out += [f"{self.scalar} *{n}" for n, _ in self.buffers]
        out += [f"long long {n}" for n in self.sizes]
        return out


MAX_BLOCK_THREADS = 1024
MAX_GRID = (2 ** 31 - 1, 65535)


def normalize_launch(launch):
    """(G, L) | ((gx, gy), (lx, ly)) -> ((gx, gy), (lx, ly)), the physical
    CUDA geometry.  The reference accepts any positive (G, L) -- every level
    is a stride loop, so results never depend on the geometry (SPEC.md:488,
    SRC/opencl.py:407-409).  CUDA caps a block at 1024 threads and gridDim.y
    at 65535, so larger requests run as capped blocks/grids whose work-group
    and work-item loops stride over the remaining iterations."""
    if launch is None:
        return None
    g, l = launch
    g = (g, 1) if isinstance(g, int) else tuple(g)
    l = (l, 1) if isinstance(l, int) else tuple(l)
    if min(g + l) < 1:
        raise ValueError("launch parameters must be positive")
    lx, ly = l
    while lx * ly > MAX_BLOCK_THREADS:
        if ly > 1:
            ly = max(1, MAX_BLOCK_THREADS // lx) if lx <= MAX_BLOCK_THREADS else 1
        else:
            lx = MAX_BLOCK_THREADS
    return (min(g[0], MAX_GRID[0]), min(g[1], MAX_GRID[1])), (lx, ly)


# ----------------------------------------------------- syntactic analyses

def _is_new(name):
    return name in NEW_SPACE


def acc_roots(a: Phrase, alias: Dict[str, Set[str]]) -> Set[str]:
    if isinstance(a, Var):
        return alias.get(a.name, {a.name})
    if isinstance(a, Proj) and isinstance(a.target, Var):
        return {a.target.name}
    u = unapply(a)
    if u is None or not u[2]:
        return set()
    return acc_roots(u[2][0], alias)


def exp_names(e: Phrase) -> Set[str]:
    out = set()
    stack = [e]
    while stack:
        q = stack.pop()
        if isinstance(q, Var):
            out.add(q.name)
        elif isinstance(q, Lam):
            stack.append(q.body)
        else:
            u = unapply(q)
            if u is not None:
                stack.extend(u[2])
            elif isinstance(q, PairP):
                stack.extend([q.fst, q.snd])
            elif isinstance(q, Proj):
                stack.append(q.target)
    return out


def rw_sets(c: Phrase, alias=None) -> Tuple[Set[str], Set[str]]:
    """Buffer names read / written anywhere inside command c."""
    alias = dict(alias or {})
    R: Set[str] = set()
    W: Set[str] = set()

    def walk(q):
        u = unapply(q)
        if u is None:
            return
        name, targs, args = u
        if name == ";":
            walk(args[0].fst)
            walk(args[0].snd)
        elif name == ":=":
            W.update(acc_roots(args[0].fst, alias))
            R.update(exp_names(args[0].snd))
            R.update(_acc_index_names(args[0].fst))
        elif _is_new(name) or name == "for":
            walk(args[0].body)
        elif name in PARFOR_FAMILY:
            a, f = args
            alias[f.body.binder] = acc_roots(a, alias)
            walk(f.body.body)
        elif name == "reduceILocal":
            f, init, src, k = args
            R.update(exp_names(init) | exp_names(src))
            walk(f.body.body.body)
            walk(k.body)

    walk(c)
    return R, W


def _binders(p: Phrase) -> Set[str]:
    return {q.binder for q in subtree_iter(p) if isinstance(q, Lam)}


def _acc_index_names(a):
    out = set()
    u = unapply(a)
    while u is not None and u[2]:
        if u[0] == "idxAcc":
            out |= exp_names(u[2][1])
        u = unapply(u[2][0])
    return out


def contains_prim(p: Phrase, names) -> bool:
    stack = [p]
    while stack:
        q = stack.pop()
        if isinstance(q, Prim):
            if q.name in names:
                return True
        elif isinstance(q, Lam):
            stack.append(q.body)
        else:
            u = unapply(q)
            if u is not None:
                stack.append(Prim(u[0]))
                stack.extend(u[2])
            elif isinstance(q, PairP):
                stack.extend([q.fst, q.snd])
            elif isinstance(q, Proj):
                stack.append(q.target)
    return False


# ---------------------------------------------------------------- planner

def _top_split(e: str, op: str):
    """Split C text `(L op R)` at its top-level operator, else None."""
    e = e.strip()
    if not (e.startswith("(") and e.endswith(")")):
        return None
    inner, depth = e[1:-1], 0
    for i, ch in enumerate(inner):
        if ch in "([{":
            depth += 1
        elif ch in ")]}":
            depth -= 1
            if depth < 0:
                return None
        elif depth == 0 and inner.startswith(f" {op} ", i):
            return inner[:i], inner[i + len(op) + 2:]
    return None


def _fma_stmt(lines):
    """(T, X, Y) of one emitted statement `T = (T + (X * Y));` (either
    operand order of the +), else None."""
    if len(lines) != 1:
        return None
    st = lines[0].strip()
    if not st.endswith(";") or " = " not in st:
        return None
    t, e = st[:-1].split(" = ", 1)
    add = _top_split(e, "+")
    if add is None:
        return None
    for acc, prod in (add, add[::-1]):
        if acc.strip() == t:
            mul = _top_split(prod, "*")
            if mul is not None:
                return t, mul[0], mul[1]
    return None


class BarrierPlanner:
    """Work-group barrier placement at uniform program points.

    State = (buffers read, buffers written) by other threads since the last
    barrier.  A unit that reads a pending write (RAW), writes a pending read
    (WAR) or rewrites a pending write (WAW) gets a barrier before it.
    Sequential loops are analysed twice so loop-carried hazards place a
    barrier inside the body (the reference's insert_barriers,
    SRC/opencl.py:209-244, handles only the straight-line RAW case)."""

    def __init__(self, shared, skip=(), opaque=(), rotated=()):
        self.shared = shared
        self.skip = set(skip)
        self.opaque = set(opaque)   # single-thread units: analysed as one leaf
        # shared buffers that alternate between two slices across iterations
        # of their sequential loop: no loop-carried hazard
        self.rotated = frozenset(rotated)
        self.before: Set[int] = set()

    def run(self, c: Phrase, loop: bool = False, alias=None):
        st = self.visit(c, (frozenset(), frozenset()), dict(alias or {}))
        if loop:  # the region repeats: find loop-carried hazards
            self.visit(c, st, dict(alias or {}))
        return self.before

    def visit(self, c, st, alias):
        u = unapply(c)
        if u is None or id(c) in self.skip:
            return st
        name, targs, args = u
        if name == ";" and id(c) not in self.opaque:
            st = self.visit(args[0].fst, st, alias)
            return self.visit(args[0].snd, st, alias)
        if id(c) in self.opaque:
            R, W = rw_sets(c, alias)
            R = {n for n in R if self.shared(n)}
            W = {n for n in W if self.shared(n)}
            st = self._hazard(c, st, R, W)
            return (st[0] | R, st[1] | W)
        if _is_new(name):
            return self.visit(args[0].body, st, alias)
        if name == "barrier":
            return (frozenset(), frozenset())
        if name == "skip":
            return st
        uniform_loop = name == "for" or (name in PARFOR_FAMILY and LOOP_LEVEL[name][0] == "workgroup")
        if uniform_loop:
            if name == "for":
                body = args[0].body
                # a hazard between the code before a sequential loop and its
                # body is fenced once, before the loop, not on every
                # iteration (loop-carried hazards are found by the second pass)
                R, W = rw_sets(body, alias)
                R = {n for n in R if self.shared(n)}
                W = {n for n in W if self.shared(n)}
                st = self._hazard(c, st, R, W)
            else:
                body = args[1].body.body
                alias = {**alias, args[1].body.binder: acc_roots(args[0], alias)}
            s1 = self.visit(body, st, alias)
            if name == "for":
                s1 = (s1[0] - self.rotated, s1[1] - self.rotated)
            s2 = self.visit(body, s1, alias)
            return s2
        if name == "reduceILocal":
            f, init, src, k = args
            R = {n for n in exp_names(init) | exp_names(src) if self.shared(n)}
            self._hazard(c, st, R, set())
            # block_combine's internal barriers fence every earlier access
            return self.visit(k.body, (frozenset(), frozenset()), alias)
        R, W = rw_sets(c, alias)
        R = {n for n in R if self.shared(n)}
        W = {n for n in W if self.shared(n)}
        st = self._hazard(c, st, R, W)
        return (st[0] | R, st[1] | W)

    def _hazard(self, c, st, R, W):
        pr, pw = st
        if (R & pw) or (W & pr) or (W & pw):
            self.before.add(id(c))
            return (frozenset(), frozenset())
        return st


# ------------------------------------------------------------------ emitter

class KernelEmitter:
    """Emits the body of one kernel (a grid phase and/or tail phases)."""

    def __init__(self, prog: "ProgramEmitter", kname: str):
        self.prog = prog
        self.kname = kname
        self.types = prog.types
        self.scalar = prog.scalar
        self.launch = prog.launch
        self.sigma = prog.sigma
        self.slices: Dict[str, int] = {}
        self.promote: Set[str] = set()
        self.pad32: Set[str] = set()         # 1-D shared buffers to pad (decided by the record pass)
        self.reset()

    def reset(self):
        self.lines: List[str] = []
        self.ind = 1
        self.env: Dict[str, object] = dict(self.prog.base_env)
        self.loops: List[Loop] = []
        self.R: Dict[str, Optional[int]] = {}
        self.records: Dict[str, List] = {}
        self.local_reads: Dict[str, bool] = {}   # 1-D shared buffer -> read at a 32-multiple work-item stride
        self.recording = False
        self.smem = 0
        self.barriers: Set[int] = set()
        self.single_thread = False
        self.used_scratch: Set[str] = set()
        self._k = 0
        self.uses_gid = False
        self.hoisted: Dict[int, Buffer] = {}
        self.decl_depth: Dict[str, int] = {}
        self.pf = None
        self.pf_i = 0
        self._pf_tag = 0
        self.pipelined: Dict[int, tuple] = {}
        self.for_plans: Dict[int, list] = {}
        self.rotated: Dict[str, str] = {}
        self.hoisted_writes: Set[int] = set()
        self.vec_vars: Dict[str, int] = {}   # loop counter -> lane width of an unrolled fold
        self.vec_hits = 0
        self.vec_pf: Optional[dict] = None   # the innermost prefetching fold (`_vec_loop`)
        self.lane_stores: Optional[list] = None   # scalar stores of the current vectorised lane
        self.probing = False                 # `_tma_plan`: enumerate and record, emit nothing
        self.probe_recs: List[tuple] = []
        self.probe_src: Optional[tuple] = None
        self.barrier_hooks: List[Tuple[int, List[str]]] = []   # (loop depth, lines after the next barrier)
        self.tmaps_used: List[str] = []
        self.stream_unsafe = False           # a streaming tail read the partials outside the ring
        self.smem_1k = False                 # dynamic shared memory must start 1024-byte aligned
        self.tail_mark: Optional[int] = None  # first line of a streaming tail block

    # ---------------------------------------------------------- helpers
    def fresh(self, base: str) -> str:
        self._k += 1
        base = "".join(ch if ch.isalnum() or ch == "_" else "_" for ch in base) or "v"
        return f"{base}_{self._k}"

    def line(self, s: str):
        self.lines.append("  " * self.ind + s)

    def open(self, head: str):
        self.line(head + " {")
        self.ind += 1

    def close(self):
        self.ind -= 1
        self.line("}")

    def nat_int(self, n: Nat) -> Optional[int]:
        c = n.const
        if c is not None:
            return c
        if self.sigma is not None:
            return n.evaluate(self.sigma)
        return None

    def nat_ix(self, n: Nat) -> Ix:
        v = self.nat_int(n)
        if v is not None:
            return ix(v)
        out = Ix()
        for mono, c in n.terms:
            t = ix(c)
            for name in mono:
                t = t * ix(name)
            out = out + t
        return out

    def r(self, e: Ix) -> str:
        return render(e, self.R)

    @property
    def per_thread(self) -> bool:
        return self.single_thread or any(lp.level in ("global", "local", "lin", "fold", "lambda")
                                         for lp in self.loops)

    @property
    def in_workgroup(self) -> bool:
        return any(lp.level == "workgroup" for lp in self.loops)

    def lit(self, v) -> str:
        if self.scalar == "float":
            f = float(v)
            s = repr(f)
            if "inf" in s or "nan" in s:
                raise CudaError(f"non-finite literal {v}")
            return f"({s}f)" if f < 0 else f"{s}f"
        return f"({int(v)}LL)" if int(v) < 0 else f"{int(v)}LL"

    # ---------------------------------------------------- access paths
    def fold(self, buf: Buffer, steps: List[Step]) -> Ref:
        dims, elem = split_array(buf.dtype)
        steps = [("i", p() if callable(p) else p) for p in buf.prefix] + list(steps)
        k = len(dims)
        if len(steps) < k or any(t != "i" for t, _ in steps[:k]):
            raise CudaError(f"partial or malformed access to {buf.key}")
        idxs = [s for _, s in steps[:k]]
        if self.recording and buf.space == "private":
            self.records.setdefault(buf.key, []).append(
                (idxs, list(self.loops), self.single_thread, self.decl_depth.get(buf.key, 0)))
        idxs, dims = idxs[buf.sliced:], dims[buf.sliced:]
        if self.recording and buf.space == "local" and len(dims) == 1 and isinstance(elem, Num):
            # a work-item index with a coefficient that is a multiple of 32
            # puts every work-item of a warp in the same bank
            work = {lp.var for lp in self.loops if lp.level in ("local", "lin") and lp.var
                    and (lp.trip is None or lp.trip > 1 or PAD_SINGLE)}
            hit = any(len(m) == 1 and IX._ATOMS[m[0]][0] == "v" and IX._ATOMS[m[0]][1] in work
                      and c % 32 == 0 for m, c in ix(idxs[0]).terms)
            self.local_reads[buf.key] = self.local_reads.get(buf.key, False) or hit
        flat = addr = None
        if dims:
            flat = Ix()
            last = len(dims) - 1
            for q, (d, i) in enumerate(zip(dims, idxs)):
                ext = self.nat_ix(d) + buf.pad if q == last and buf.pad else self.nat_ix(d)
                if q == last and buf.swz and last >= 1:
                    unit, dv, per = buf.swz
                    mask = mod(div(idxs[last - 1], dv, self.R), per, self.R) * unit
                    addr = flat * ext + self._swizzled(i, mask, unit, per)
                flat = flat * ext + i
            if buf.pad32:
                addr = flat + div(flat, 32, self.R) * buf.pad32
            base = f"{buf.cname}[{self.r(addr if addr is not None else flat)}]"
        else:
            base = buf.cname if buf.space == "private" else f"{buf.cname}[0]"
        suffix = ""
        t = elem
        for tag, s in steps[k:]:
            if tag == "f":
                if not isinstance(t, Pair):
                    raise CudaError("field step on a non-pair")
                suffix += f".x{s}"
                t = t.fst if s == 1 else t.snd
            elif isinstance(t, Vector):
                suffix += f".v[{self.r(s)}]"
                t = Num()
            elif isinstance(t, Array):
                suffix += f"[{self.r(s)}]"
                t = t.elem
            else:
                raise CudaError(f"index step into scalar of {buf.key}")
        return Ref(buf, flat, suffix, base + suffix, addr)

    def _swizzled(self, i: Ix, mask: Ix, unit: int, per: int) -> Ix:
        """i ^ mask (mask a multiple of unit below unit*per), written as
        Hi + ((Mid) ^ mask) + Lo so that only the bits the mask can touch
        are inside the XOR: Lo < B with every other term a multiple of B (B
        the largest such power of two <= unit), Hi a multiple of a power of
        two P above Mid and the mask.  This keeps unrolled constants and
        per-thread bases out of the XOR so the C compiler still folds them
        into immediate offsets and 16-byte accesses."""
        R = self.R
        lo, rest = [], list(i.terms)
        B = unit
        while B > 1:
            cand = [t for t in i.terms if t[1] % B]
            m = IX.max_value(Ix(cand), R)
            if m is not None and m < B:
                lo, rest = cand, [t for t in i.terms if t[1] % B == 0]
                break
            B //= 2
        P = unit * per
        while True:
            hi = [t for t in rest if t[1] % P == 0]
            mid = [t for t in rest if t[1] % P]
            mm = IX.max_value(Ix(mid), R)
            if mm is None:
                hi, mid = [], rest
                break
            if mm < P:
                break
            P *= 2
        return Ix(hi) + IX.xor(Ix(mid), mask) + Ix(lo)

    def binding(self, name: str):
        if name not in self.env:
            raise CudaError(f"unbound identifier in kernel: {name}")
        return self.env[name]

    def index(self, p: Phrase) -> Ix:
        if isinstance(p, Lit):
            return ix(int(p.value))
        if isinstance(p, Var):
            b = self.binding(p.name)
            if isinstance(b, Val) and b.ixv is not None:
                return b.ixv
        raise CudaError(f"index expression is not a loop index or literal: {p!r}")

    def val_path(self, v: Val, steps) -> str:
        if v.ixv is not None:
            if steps:
                raise CudaError("path into an index value")
            return self.r(v.ixv)
        text, t = v.text, v.dtype
        for tag, s in steps:
            if tag == "f":
                text += f".x{s}"
                t = t.fst if s == 1 else t.snd
            elif isinstance(t, Vector):
                text += f".v[{self.r(s)}]"
                t = Num()
            else:
                raise CudaError("index step into a value")
        return text

    def resolve(self, p: Phrase, steps: List[Step]):
        """Read p at path steps: a Ref (buffer-rooted) or C text."""
        if isinstance(p, Proj) and p.index == 2 and isinstance(p.target, Var):
            p = p.target
        if isinstance(p, Var):
            b = self.binding(p.name)
            if isinstance(b, Buffer):
                return self.fold(b, steps)
            if isinstance(b, Val):
                return self.val_path(b, steps)
            raise CudaError(f"{p.name} is not readable here")
        if isinstance(p, Lit):
            if steps or not isinstance(p.dtype, Vector):
                return self.lit(p.value)
            return f"dpia::splat<{self.scalar}, {p.dtype.width}>({self.lit(p.value)})"
        u = unapply(p)
        if u is None:
            raise CudaError(f"not an expression: {p!r}")
        name, targs, args = u
        R = self.R
        if name in ("+", "-", "*", "/") and len(args) == 1:
            return f"({self.exp(args[0].fst, steps)} {name} {self.exp(args[0].snd, steps)})"
        if name == "negate":
            return f"(-{self.exp(args[0], steps)})"
        if name == "abs":
            return f"dpia::abs_({self.exp(args[0], steps)})"
        if name == "zip":
            (t1, i), (t2, k), rest = steps[0], steps[1], steps[2:]
            return self.resolve(args[k - 1], [("i", i)] + rest)
        if name == "split":
            n = self.nat_ix(targs[0])
            (_, i), (_, j), rest = steps[0], steps[1], steps[2:]
            return self.resolve(args[0], [("i", i * n + j)] + rest)
        if name == "join":
            m = self.nat_int(targs[1])
            (_, k), rest = steps[0], steps[1:]
            if m is None:
                raise CudaError("join with a symbolic row size needs specialisation")
            return self.resolve(args[0], [("i", div(k, m, R)), ("i", mod(k, m, R))] + rest)
        if name == "transpose":
            (_, j), (_, i), rest = steps[0], steps[1], steps[2:]
            return self.resolve(args[0], [("i", i), ("i", j)] + rest)
        if name == "pair":
            (_, k), rest = steps[0], steps[1:]
            return self.resolve(args[k - 1], rest)
        if name in ("fst", "snd"):
            return self.resolve(args[0], [("f", 1 if name == "fst" else 2)] + steps)
        if name == "idx" or name.startswith("idxVec"):
            return self.resolve(args[0], [("i", self.index(args[1]))] + steps)
        if name.startswith("asVector") and "Acc" not in name:
            w = int(name[len("asVector"):])
            (_, i) = steps[0]
            ref = self.resolve(args[0], [("i", i * w)])
            aligned = isinstance(ref, Ref) and ref.flat is not None and not ref.suffix \
                and all(c % w == 0 for _, c in ref.flat.terms) \
                and not (ref.buf.swz and w > ref.buf.swz[0])
            if len(steps) >= 2:
                (_, lane), rest = steps[1], steps[2:]
                if aligned and not rest:
                    # whole-vector load + lane select: redundant loads of the
                    # same vector CSE into one LDG.128/LDS.128
                    return (f"dpia::vload<{self.scalar}, {w}>({ref.buf.cname}, "
                            f"{self.r(ref.at)}).v[{self.r(lane)}]")
                return self.resolve(args[0], [("i", i * w + lane)] + rest)
            if aligned:
                if self.probing:
                    self.probe_src = (ref.buf, ref.at, w)
                if self.prog.stream is not None and self.prog.in_tail and ref.buf.key in self.prog.stream["partials"]:
                    self.stream_unsafe = True
                return f"dpia::vload<{self.scalar}, {w}>({ref.buf.cname}, {self.r(ref.at)})"
            if self.probing:
                refs = [self.resolve(args[0], [("i", i * w + k)]) for k in range(w)]
                if all(isinstance(r, Ref) and r.flat is not None and not r.suffix and r.addr is None
                       and r.buf is refs[0].buf for r in refs):
                    self.probe_src = (refs[0].buf, [r.flat for r in refs], w)
            lanes = ", ".join(self.exp(args[0], [("i", i * w + k)]) for k in range(w))
            return f"dpia::vec<{self.scalar}, {w}>{{{{{lanes}}}}}"
        if name.startswith("asScalar") and "Acc" not in name:
            w = int(name[len("asScalar"):])
            (_, k), rest = steps[0], steps[1:]
            return self.resolve(args[0], [("i", div(k, w, R)), ("i", mod(k, w, R))] + rest)
        raise CudaError(f"no expression clause for {name!r}")

    def exp(self, p: Phrase, steps: List[Step]) -> str:
        r = self.resolve(p, steps)
        if isinstance(r, Ref):
            lr = self._lane_read(r)
            st = self.prog.stream
            if st is not None and self.prog.in_tail and r.buf.key in st["partials"] and \
                    not (lr and lr.startswith("pfv_") and self.vec_pf is not None and self.vec_pf.get("ring")):
                self.stream_unsafe = True
            return lr or r.text
        return r

    def _lane_read(self, r: Ref) -> Optional[str]:
        """Inside a W-unrolled sequential fold (`_vec_loop`): a scalar read
        of a global buffer at flat index W*j + A + c (j the unrolled counter,
        every other term a multiple of W, 0 <= c < W) becomes lane c of the
        W-vector at W*j + A.  The W unrolled iterations read the same
        vector, which the compiler loads once.  In a prefetching fold the
        vector comes from the stream's queue or ring when A mentions no loop
        variable bound inside the fold."""
        if not self.vec_vars or r.suffix or r.flat is None or r.buf.space not in ("in", "global", "local") \
                or r.buf.swz or r.buf.pad or r.buf.pad32 or not isinstance(r.buf.elem, Num) \
                or (r.buf.space == "local" and not VEC_LOCAL):
            return None
        coef = dict((m, c) for m, c in r.flat.terms)
        js = [v for v, w in self.vec_vars.items() if coef.get((v,)) == w]
        if len(js) != 1:
            return None
        W = self.vec_vars[js[0]]
        lane = coef.get((), 0) % W
        if lane < 0 or any(c % W for m, c in r.flat.terms if m != ()):
            return None
        base = r.flat + ix(-lane) if lane else r.flat
        self.vec_hits += 1
        text = self.r(base)
        pf = self.vec_pf
        if pf is not None and js[0] == pf["j"] and r.buf.space != "local":
            # (shared-memory data is read in place: LDS.128, never queued)
            inner = {lp.var for lp in self.loops[pf["depth"]:]} - {pf["j"]}
            if not any(re.search(rf"\b{re.escape(v)}\b", text) for v in inner):
                key = (r.buf.cname, text)
                if key not in pf["streams"]:
                    pf["streams"][key] = (f"pfv_{pf['tag']}_{len(pf['streams'])}", r.buf, base)
                return f"{pf['streams'][key][0]}.v[{lane}]"
        return f"dpia::vload<{self.scalar}, {W}>({r.buf.cname}, {text}).v[{lane}]"

    def acc(self, p: Phrase, steps: List[Step]) -> Union[Ref, VStore]:
        if isinstance(p, Proj) and p.index == 1 and isinstance(p.target, Var):
            p = p.target
        if isinstance(p, Var):
            b = self.binding(p.name)
            if isinstance(b, Buffer):
                if b.space == "in":
                    raise CudaError(f"write to input {b.key}")
                return self.fold(b, steps)
            if isinstance(b, Alias):
                return self.acc(b.acc, [("i", b.i)] + steps)
            raise CudaError(f"{p.name} is not an acceptor")
        u = unapply(p)
        if u is None:
            raise CudaError(f"not an acceptor: {p!r}")
        name, targs, args = u
        R = self.R
        if name == "idxAcc":
            return self.acc(args[0], [("i", self.index(args[1]))] + steps)
        if name == "splitAcc":
            n = self.nat_int(targs[0])
            if n is None:
                raise CudaError("splitAcc with a symbolic chunk size needs specialisation")
            (_, k), rest = steps[0], steps[1:]
            return self.acc(args[0], [("i", div(k, n, R)), ("i", mod(k, n, R))] + rest)
        if name == "joinAcc":
            m = self.nat_ix(targs[1])
            (_, i), (_, j), rest = steps[0], steps[1], steps[2:]
            return self.acc(args[0], [("i", i * m + j)] + rest)
        if name == "transposeAcc":
            (_, i), (_, j), rest = steps[0], steps[1], steps[2:]
            return self.acc(args[0], [("i", j), ("i", i)] + rest)
        if name in ("pairAcc1", "pairAcc2"):
            return self.acc(args[0], [("f", int(name[-1]))] + steps)
        if name in ("zipAcc1", "zipAcc2"):
            (_, i), rest = steps[0], steps[1:]
            return self.acc(args[0], [("i", i), ("f", int(name[-1]))] + rest)
        if name.startswith("asVectorAcc"):
            w = int(name[len("asVectorAcc"):])
            (_, k), rest = steps[0], steps[1:]
            return self.acc(args[0], [("i", div(k, w, R)), ("i", mod(k, w, R))] + rest)
        if name.startswith("asScalarAcc"):
            w = int(name[len("asScalarAcc"):])
            (_, i) = steps[0]
            if len(steps) >= 2:
                (_, lane), rest = steps[1], steps[2:]
                return self.acc(args[0], [("i", i * w + lane)] + rest)
            ref = self.acc(args[0], [("i", i * w)])
            if isinstance(ref, Ref) and ref.flat is not None and not ref.suffix \
                    and all(c % w == 0 for _, c in ref.flat.terms) \
                    and not (ref.buf.swz and w > ref.buf.swz[0]):
                return VStore(ref, w)
            raise NeedLanes()
        raise CudaError(f"no acceptor clause for {name!r}")

    # ------------------------------------------------------- assignment
    def assign(self, d: DataType, a: Phrase, e: Phrase, steps=()):
        steps = list(steps)
        if isinstance(d, Pair):
            self.assign(d.fst, a, e, steps + [("f", 1)])
            self.assign(d.snd, a, e, steps + [("f", 2)])
            return
        if isinstance(d, Array):
            raise CudaError("assignment at array type (expected generalised assignment)")
        if isinstance(d, Vector):
            try:
                target = self.acc(a, steps)
            except NeedLanes:
                for k in range(d.width):
                    self.assign(Num(), a, e, steps + [("i", ix(k))])
                return
            if self.probing:
                return self._probe_record(target, e, steps)
            rhs = self.exp(e, steps)
        else:
            target = self.acc(a, steps)
            if self.probing:
                return self._probe_record(target, e, steps)
            rhs = self.exp(e, steps)
        if self.pf is not None:
            mode, regs = self.pf
            T = self.types.c_elem(d)
            if mode == "declare":           # prologue: new register
                name = f"pf{self._pf_tag}_{len(regs)}"
                regs.append((name, T))
                self.line(f"{name} = {rhs};")
                return
            name = regs[self.pf_i][0]
            self.pf_i += 1
            if mode == "refill":            # next iteration's global loads
                self.line(f"{name} = {rhs};")
                return
            rhs = name                       # commit: registers -> shared memory
        buf = target.ref.buf if isinstance(target, VStore) else target.buf
        if self.vec_pf is not None:
            self.vec_pf["written"].add(buf.cname)
        st = self.prog.stream
        if st is not None and not self.prog.in_tail and buf.key in st["partials"]:
            # a streaming tail assumes work-item i writes partial i (round
            # i / gsize publishes it): any other write index falls back
            lp = self.loops[0] if self.loops and self.loops[0].level == "global" else None
            at = None if isinstance(target, VStore) or target.flat is None else \
                Ix([(m, c) for m, c in target.flat.terms if "dpia_par" not in IX.free_names(Ix([(m, c)]))])
            if lp is None or at is None or at != ix(lp.var):
                self.stream_unsafe = True
        if isinstance(target, VStore):
            stmt = (f"dpia::vstore<{self.scalar}, {target.width}>({buf.cname}, "
                    f"{self.r(target.ref.at)}, {rhs});")
        else:
            stmt = f"{target.text} = {rhs};"
        if buf.space != "private" and not self.per_thread:
            stmt = f"if (dpia_tid == 0) {stmt}"
        if self.lane_stores is not None and not isinstance(target, VStore) and target.flat is not None \
                and not target.suffix and target.addr is None:
            self.lane_stores.append((buf, target.flat, rhs, stmt))
        self.line(stmt)

    # --------------------------------------------------------- commands
    def comm(self, p: Phrase):
        if id(p) in self.barriers and not self.per_thread and \
                (self.pf is None or self.pf[0] == "commit"):
            self._barrier()
        u = unapply(p)
        if u is None:
            raise CudaError(f"not a command: {p!r}")
        name, targs, args = u
        if name == "skip":
            return
        if name == "barrier":
            if not self.per_thread:
                self._barrier()
            return
        if name == ";":
            self.comm(args[0].fst)
            self.comm(args[0].snd)
            return
        if name == ":=":
            self.assign(targs[0], args[0].fst, args[0].snd)
            return
        if _is_new(name):
            self.new(name, targs[0], args[0], p)
            return
        if name == "for":
            f = args[0]
            trip = self.nat_int(targs[0])
            if not self.per_thread and not self.in_workgroup and not self.prog.in_tail and \
                    contains_prim(f.body, {"parforGlobal", "parforWorkgroup", "parforWorkgroup1"}):
                raise CudaError("a sequential loop around a grid-level parallel loop needs a "
                                "grid-wide barrier per iteration (one kernel per iteration); "
                                "not supported")
            if self._fma2_loop(p, targs[0], f):
                return
            if self._vec_loop(targs[0], f):
                return
            cands, rotate = [], False
            if id(p) in self.for_plans:
                cands, rotate = self.for_plans[id(p)], True
            elif not self.per_thread and self.launch and trip is not None and trip > 1:
                cands = self.pipeline_candidates(f.body, f.binder)
            if cands:
                self.pipeline_prologue(cands, f.binder, targs[0], trip, rotate)
            self.loop("seq", 0, targs[0], f.binder, lambda: self.comm(f.body))
            return
        if name in PARFOR_FAMILY:
            self.parfor(name, targs, args)
            return
        if name == "reduceILocal":
            self.combine(targs, args)
            return
        raise CudaError(f"no command clause for {name!r}")

    # ------------------------------------- vector loads in sequential folds
    def _vec_loop(self, n: Nat, f: Lam) -> bool:
        """A long sequential loop inside one work-item (a reduceSeq over a
        contiguous chunk, or the single-thread top-level reduce of a fused
        tail) that reads global buffers at unit stride: emitted unrolled by a
        lane width W, iteration W*j + k reading lane k of one W-wide vector
        (`_lane_read`), instead of W scalar loads.  The iterations run in
        the original order, so the fold's association is unchanged.  The
        read streams are software-pipelined (`_emit_vec_loop`): through a
        shared-memory ring of TMA bulk copies in a single thread's fold,
        through a rotating register queue of 32-byte (then 16-byte) loads in
        a work-item's fold, unless the fold writes a streamed buffer.  Each
        variant is tried on a scratch copy of the output; False (nothing
        emitted) when no read qualifies."""
        trip = self.nat_int(n)
        # short folds too (down to 2 vectors): a work-item walking its own
        # 32-element piece issues 8 LDG.128 instead of 32 scalar loads that
        # each touch a different cache line of the warp (the reference's gemv)
        if not VEC_LOADS or not self.per_thread or self.pf is not None or trip is None \
                or trip < (2 * VEC_WIDTH if VEC_SHORT else UNROLL_LIMIT + 1):
            return False
        sb = 4 if self.scalar == "float" else 8
        modes = []
        if TAIL_RING and self.single_thread and not self.loops and TAIL_RING_STAGES > 0:
            modes.append(("ring", VEC_WIDTH))
        if ROW_TMA and self._rows_loop() is not None and VEC_WIDTH * sb == 16:
            modes.append(("rows", VEC_WIDTH))
        if VEC_PREFETCH > 1:
            if VEC_LOAD_BYTES == 32:
                modes.append(("queue32", 32 // sb))
            modes.append(("queue", VEC_WIDTH))
        modes.append(("plain", VEC_WIDTH))
        for mode, W in modes:
            if trip % W:
                continue
            mark, ind, hits, smem, k0 = len(self.lines), self.ind, self.vec_hits, self.smem, self._k
            if self._emit_vec_loop(n, f, trip // W, W, mode) and self.vec_hits > hits:
                return True
            del self.lines[mark:]
            self.ind, self.smem, self._k = ind, smem, k0   # a failed attempt leaves no trace
        return False

    @staticmethod
    def _pow2_divisor(want: int, T: int, cap: int) -> int:
        """The largest power of two <= min(want, cap) dividing T (0 if < 2)."""
        d = 1 << (max(1, min(want, cap)).bit_length() - 1)
        while d > 1 and T % d:
            d //= 2
        return d if d > 1 else 0

    def _emit_vec_loop(self, n: Nat, f: Lam, T: int, W: int, mode: str) -> bool:
        """One attempt of `_vec_loop`, T iterations of W lanes.

        queue / queue32 (a work-item's fold): D slots per stream s (a buffer
        and a base offset; V_s(j) its W-vector at iteration j)
            q_s[d] = V_s(d), d < D                        (prologue)
            for jo in 0, D, ..: for jd < D (unrolled): j = jo + jd
                v_s = q_s[jd]; q_s[jd] = V_s(j + D) if j + D < T
                body(j) reading lanes of v_s
        so D vectors per stream are in flight while the body folds in
        order; queue32 loads each slot with one 32-byte load.

        ring (a single thread's fold): C-vector pieces of every stream go
        through S shared-memory slots filled by TMA bulk copies
            fill slot k of every stream, k < S           (prologue)
            for jo in 0, C, ..: wait slot k = jo / C (mbarrier parity)
                for jd < C: j = jo + jd; v_s = slot[jd]; body(j)
                refill the slot with piece k + S
        False when the body writes a streamed buffer or nothing streams."""
        j = self.fresh("j")
        self.R[j] = T
        outer_pf = self.vec_pf
        pf = None
        top = len(self.lines)
        sb = 4 if self.scalar == "float" else 8
        vt = f"dpia::vec<{self.scalar}, {W}>"
        D = C = S = 0
        if mode in ("queue", "queue32"):
            D = self._pow2_divisor(VEC_PREFETCH * 32 // (W * sb), T, T // 2)
            if not D:
                return False
        elif mode == "ring":
            C = self._pow2_divisor(TAIL_RING_BYTES // (W * sb), T, T)
            if not C:
                return False
            S = min(TAIL_RING_STAGES, T // C)
        elif mode == "rows":
            # vectors per step: ROW_TMA_BOXES box columns of 128 bytes
            C = 128 // (W * sb) * max(1, ROW_TMA_BOXES)
            while C > 128 // (W * sb) and T % C:
                C //= 2
            if T % C:
                return False
            # slots: about ROW_TMA_INFLIGHT bytes in flight per warp over the
            # fold's input streams (the inputs its body names), within
            # 200 KiB of shared memory for the block's warps
            ns = max(1, len(exp_names(f.body) & {k for k, sp in self.prog.spaces.items() if sp == "in"}))
            step = ns * C * W * sb * 32
            S = max(2, ROW_TMA_STAGES, ROW_TMA_INFLIGHT // step)
            nw = self.launch[1][0] * self.launch[1][1] // 32
            while S > 2 and nw * S * step > 200 * 1024:
                S -= 1
        if mode != "plain":
            self._k += 1
            pf = {"j": j, "depth": len(self.loops), "streams": {}, "written": set(), "tag": self._k,
                  "ring": mode == "ring"}
            self.vec_pf = pf
        else:
            self.vec_pf = None
        if mode in ("queue", "queue32"):
            jo, jd = self.fresh("jo"), self.fresh("jd")
            self.open(f"for (int {jo} = 0; {jo} < {T}; {jo} += {D})")
            self.line("#pragma unroll")
            self.open(f"for (int {jd} = 0; {jd} < {D}; {jd} += 1)")
            self.line(f"const int {j} = {jo} + {jd};")
            take = len(self.lines)
        elif mode == "rows":
            jo, jd, ru, rs, mb = (self.fresh(x) for x in ("jo", "jd", "ru", "rs", "wmb"))
            u0 = self.fresh("wu0")
            self.open(f"for (int {jo} = 0; {jo} < {T}; {jo} += {C})")
            self.line(f"const int {ru} = {u0} + {jo} / {C};")
            self.line(f"const int {rs} = {ru} % {S};")
            self.line(f"dpia::ring_wait({mb} + {rs}, (unsigned)(({ru} / {S}) & 1));")
            slot_at = len(self.lines)
            self.line("#pragma unroll")
            self.open(f"for (int {jd} = 0; {jd} < {C}; {jd} += 1)")
            self.line(f"const int {j} = {jo} + {jd};")
            take = len(self.lines)
        elif mode == "ring":
            jo, jd, rk, rs, mb = (self.fresh(x) for x in ("jo", "jd", "rk", "rs", "rmb"))
            self.open(f"for (int {jo} = 0; {jo} < {T}; {jo} += {C})")
            self.line(f"const int {rk} = {jo} / {C}, {rs} = {rk} % {S};")
            self.line(f"dpia::ring_wait({mb} + {rs}, (unsigned)(({rk} / {S}) & 1));")
            slot_at = len(self.lines)
            self.line(f"#pragma unroll {TAIL_RING_UNROLL}")
            self.open(f"for (int {jd} = 0; {jd} < {C}; {jd} += 1)")
            self.line(f"const int {j} = {jo} + {jd};")
            take = len(self.lines)
        else:
            if T > 8:
                self.line("#pragma unroll 8")       # loads of later iterations issue ahead
            self.open(f"for (int {j} = 0; {j} < {T}; {j} += 1)")
        self.vec_vars[j] = W
        self.loops.append(Loop("seq", 0, j, T, nat(T), False))
        old = self.env.get(f.binder)
        try:
            lanes, outer_stores = [], self.lane_stores
            for k in range(W):
                self.lane_stores = []
                at = len(self.lines)
                self.open("")
                self.env[f.binder] = Val(Idx(n), ixv=ix(j) * W + k)
                self.comm(f.body)
                self.close()
                lanes.append((at, len(self.lines), self.lane_stores))
            self.lane_stores = outer_stores
            self._merge_lane_stores(lanes, W)
        finally:
            self.loops.pop()
            self.vec_vars.pop(j, None)
            self.vec_pf = outer_pf
            if old is None:
                self.env.pop(f.binder, None)
            else:
                self.env[f.binder] = old
        self.close()
        if pf is None:
            return True
        streams = list(pf["streams"].values())
        if not streams or any(b.cname in pf["written"] for _, b, _ in streams):
            return False
        if mode == "ring":
            return self._finish_ring(streams, top, slot_at, take, T, W, C, S, j, jo, jd, rs, mb)
        if mode == "rows":
            return self._finish_rows(streams, top, slot_at, take, T, W, C, S, j, ru, rs, mb, u0, pf)
        self.close()
        pad = "  " * self.ind
        pad_in = pad + "    "
        body = []
        for name, b, base in streams:
            q = name.replace("pfv_", "pfq_")
            body.append(f"{pad_in}const {vt} {name} = {q}[{jd}];")
            body.append(f"{pad_in}if ({j} + {D} < {T}) {q}[{jd}] = {self._vload(mode, b, W, base + ix(W * D))};")
        self.lines[take:take] = body
        pro = [f"{pad}{vt} {name.replace('pfv_', 'pfq_')}[{D}];" for name, _b, _base in streams]
        pro.append(f"{pad}#pragma unroll")
        pro.append(f"{pad}for (int {j} = 0; {j} < {D}; {j} += 1) {{")
        for name, b, base in streams:
            pro.append(f"{pad}  {name.replace('pfv_', 'pfq_')}[{j}] = {self._vload(mode, b, W, base)};")
        pro.append(f"{pad}}}")
        self.lines[top:top] = pro
        self._prefetch_next_group(streams, j, T * W * sb)
        return True

    def _prefetch_next_group(self, streams, j: str, piece_bytes: int):
        """A work-item fold inside a work-group loop (the reference's gemv:
        a row per work-group, each work-item folding its own piece): once
        the fold is done, prefetch into L2 the piece this work-item folds in
        the work-group loop's next iteration, so its loads there hit L2
        while this iteration's barrier and single-thread tail run."""
        wg = [lp for lp in self.loops if lp.level == "workgroup"]
        if not PREFETCH_NEXT or len(wg) != 1 or wg[0].single or not self.launch or wg[0].trip is None \
                or piece_bytes > 8 * 128:
            return
        lp = wg[0]
        G = self.launch[0][lp.dim]
        sb = 4 if self.scalar == "float" else 8
        for _name, b, base in streams:
            coef = {m: c for m, c in base.terms}
            if b.space != "in" or coef.get((lp.var,)) is None:
                continue
            at0 = Ix([(m, c) for m, c in base.terms if j not in IX.free_names(Ix([(m, c)]))])
            nxt = at0 + ix(coef[(lp.var,)] * G)
            for q in range(-(-piece_bytes // 128)):
                self.line(f"if ({lp.var} + {G} < {lp.trip}) dpia::prefetch_l2({b.cname} + "
                          f"({self.r(nxt)}) + {q * 128 // sb});")

    def _merge_lane_stores(self, lanes, W: int):
        """The W lanes of a vectorised fold iteration that each store one
        scalar to W consecutive elements of a global buffer (a work-item
        writing its own contiguous piece: the reference's scal) become one
        W-wide vector store, when each lane's code is nothing but that
        store and the first element is W-aligned."""
        recs = []
        for at, end, stores in lanes:
            body = [ln.strip() for ln in self.lines[at:end]]
            if len(stores) != 1 or len(body) != 3 or body[0] != "{" or body[2] != "}":
                return
            buf, flat, rhs, text = stores[0]
            if body[1] != text:
                return
            recs.append((buf, flat, rhs))
        buf0, f0, _ = recs[0]
        if buf0.space not in ("out", "global") or buf0.swz or buf0.pad or buf0.pad32 or \
                not isinstance(buf0.elem, Num) or any(c % W for _, c in f0.terms):
            return
        for k, (buf, flat, _) in enumerate(recs):
            if buf is not buf0 or flat != f0 + k:
                return
        vals = ", ".join(rhs for _, _, rhs in recs)
        stmt = (f"dpia::vstore<{self.scalar}, {W}>({buf0.cname}, {self.r(f0)}, "
                f"dpia::vec<{self.scalar}, {W}>{{{{{vals}}}}});")
        pad = "  " * self.ind
        self.lines[lanes[0][0]:lanes[-1][1]] = [pad + stmt]
        if self.vec_pf is not None:
            # a rows-mode fold may turn it into a TMA row store (`_finish_rows`)
            self.vec_pf.setdefault("stores", []).append((buf0, f0, vals, stmt))

    def _rows_loop(self) -> Optional[Loop]:
        """The enclosing mapGlobal loop when a fold here can use row boxes:
        the fold is a work-item's (directly inside the global loop), the
        launch is whole warps and the work-item count a multiple of 32, so
        each warp's 32 consecutive work-items take every round together."""
        if not self.per_thread or self.single_thread or len(self.loops) != 1 or not self.launch:
            return None
        lp = self.loops[0]
        (gx, gy), (lx, ly) = self.launch
        if lp.level != "global" or lp.trip is None or lp.trip % 32 or (lx * ly) % 32:
            return None
        return lp

    def _finish_rows(self, streams, top, slot_at, take, T, W, C, S, j, ru, rs, mb, u0, pf=None) -> bool:
        """Complete a rows-mode fold (see `_vec_loop`).  Stream s reads
        X_s[coef * i + c_s + W * j'] for work-item i: X_s viewed as rows of
        coef elements, the warp's work-items are 32 consecutive rows, and
        step t of the fold covers columns [c_s + t*C*W, +C*W) as C*W/32
        boxes of 32 rows x 128 bytes.  Lane 0 keeps S steps in flight
        through the warp's slots (one mbarrier per slot), running ahead into
        the warp's next round of work-items; every lane reads its own row of
        each box (128-byte swizzle: 16-byte chunk q of row r sits at chunk
        q ^ (r % 8), the slots being 1024-byte aligned)."""
        lp = self._rows_loop()
        sb = 4 if self.scalar == "float" else 8
        VB = 128 // (W * sb)                        # vectors per box row
        if lp is None or W * sb != 16 or C % VB:
            return False
        NB = C // VB                                # boxes per stream per step
        iv, n = lp.var, lp.trip
        (gx, gy), (lx, ly) = self.launch
        nthreads, steps = lx * ly, T // C
        specs = []
        for name, b, base in streams:
            coef = {m: c for m, c in base.terms}
            if b.space != "in" or b.prefix or not isinstance(b.elem, Num) or \
                    set(coef) - {(j,), (iv,), ()} or coef.get((j,)) != W or (iv,) not in coef:
                return False
            P, c0 = coef[(iv,)], coef.get((), 0)
            NX = self._elements(b.dtype)
            if NX is None or P <= 0 or NX % P or (P * sb) % 16 or c0 < 0 or c0 + T * W > P \
                    or NX // P < n or NX // P > IX.INT32_MAX:
                return False
            tm = self.prog.add_tmap({"X": b, "eb": sb, "NX": NX, "P": P, "rows": 32, "parts": 1,
                                     "C": VB * W, "swizzle": 128})
            if tm not in self.tmaps_used:
                self.tmaps_used.append(tm)
            specs.append((name, tm, c0))
        NS = len(specs)
        slot_bytes = NS * NB * 4096
        nw = nthreads // 32
        # row stores: the fold's merged vector stores to an output at
        # coef * i + c + W * j' (a work-item writing its own contiguous piece)
        # go through SO shared-memory slots and leave as TMA tensor stores of
        # the warp's 32 rows
        SO = 2
        pf = pf or {}
        stores = []
        for buf, f0, vals, stmt in pf.get("stores", []) if ROW_TMA_STORE else []:
            coef = {m: c for m, c in f0.terms}
            NX = self._elements(buf.dtype)
            if buf.space != "out" or buf.prefix or buf.swz or buf.pad or buf.pad32 or \
                    not isinstance(buf.elem, Num) or set(coef) - {(j,), (iv,), ()} or \
                    coef.get((j,)) != W or (iv,) not in coef or NX is None:
                stores = None
                break
            P, c0 = coef[(iv,)], coef.get((), 0)
            if P <= 0 or NX % P or (P * sb) % 16 or c0 < 0 or c0 + T * W > P or NX // P < n:
                stores = None
                break
            tm = self.prog.add_tmap({"X": buf, "eb": sb, "NX": NX, "P": P, "rows": 32, "parts": 1,
                                     "C": VB * W, "swizzle": 128})
            if tm not in self.tmaps_used:
                self.tmaps_used.append(tm)
            stores.append((buf, tm, c0, vals, stmt))
        so_bytes = len(stores or []) * NB * 4096
        if nw * (S * slot_bytes + SO * so_bytes) > 200 * 1024:
            if nw * S * slot_bytes > 200 * 1024:
                return False
            stores = None
        stores = stores or []
        soff = self.alloc_smem(nw * S * slot_bytes, align=1024)
        self.smem_1k = True
        ooff = self.alloc_smem(nw * SO * so_bytes, align=1024) if stores else 0
        moff = self.alloc_smem(nw * S * 8, align=8)
        lane, sw, st, row0, rnd = (self.fresh(x) for x in ("wlane", "wsw", "wst", "wrow0", "wround"))
        jd = f"({j} % {C})"
        pad1 = "  " * self.ind                      # the step loop's body
        pad2 = pad1 + "  "                          # the lane loop's body
        vt = f"dpia::vec<{self.scalar}, {W}>"
        box_elems = 4096 // sb
        self.lines[take:take] = [
            f"{pad2}const {vt} {name} = dpia::vload<{self.scalar}, {W}>({name}_s + {jd} / {VB} * {box_elems}, "
            f"{W} * ({jd} % {VB} ^ {sw}));" for name, _tm, _c0 in specs]
        where = [next((q for q in range(take, len(self.lines)) if self.lines[q].strip() == stmt), None)
                 for _b, _t, _c, _v, stmt in stores]
        if None in where:
            stores = []              # (each store line is found before any is rewritten)
        ost = self.fresh("wos") if stores else None
        for k, (buf, tm, c0, vals, stmt) in enumerate(stores):
            at = where[k]
            ind = self.lines[at][:len(self.lines[at]) - len(self.lines[at].lstrip())]
            self.lines[at] = (f"{ind}dpia::vstore<{self.scalar}, {W}>(reinterpret_cast<{self.scalar}*>"
                              f"({ost} + ({ru} % {SO}) * {so_bytes} + {k * NB * 4096} + {lane} * 128) + "
                              f"{jd} / {VB} * {box_elems}, {W} * ({jd} % {VB} ^ {sw}), "
                              f"dpia::vec<{self.scalar}, {W}>{{{{{vals}}}}});")
        self.lines[slot_at:slot_at] = [
            f"{pad1}const {self.scalar}* {name}_s = reinterpret_cast<const {self.scalar}*>"
            f"({st} + {rs} * {slot_bytes} + {k * NB * 4096} + {lane} * 128);"
            for k, (name, _tm, _c0) in enumerate(specs)]
        if stores:
            # the store slot this step fills was last read by the TMA store
            # of step ru - SO
            self.lines[slot_at:slot_at] = [f"{pad1}if ({lane} == 0) dpia::bulk_wait_read<{SO - 1}>();",
                                           f"{pad1}__syncwarp();"]

        def issue(p, u):
            """lane 0: fill step u's slot (step u % steps of round u / steps)
            if that round has work-items for this warp"""
            out = [f"{p}{{", f"{p}  const long long wr_ = {row0} + (long long)(({u}) / {steps}) * dpia_gsize;",
                   f"{p}  if (wr_ < {n}) {{",
                   f"{p}    unsigned char* wd_ = {st} + (({u}) % {S}) * {slot_bytes};",
                   f"{p}    const int wc_ = (({u}) % {steps}) * {C * W};"]
            for k, (_name, tm, c0) in enumerate(specs):
                for bb in range(NB):
                    out.append(f"{p}    dpia::tma_tile_2d(wd_ + {(k * NB + bb) * 4096}, &{tm}, "
                               f"{c0 + bb * VB * W} + wc_, (int)wr_, 4096u, {mb} + (({u}) % {S}));")
            out += [f"{p}  }}", f"{p}}}"]
            return out

        if stores:
            self.line("dpia::fence_async_shared();")
        self.line("__syncwarp();")
        if stores:
            # lane 0 writes the step's rows of each stored output (the line
            # names the output, so a chained kernel waits for its previous
            # grid first: `_chain_waits`)
            self.open(f"if ({lane} == 0)")
            self.line(f"const int wc_ = ({ru} % {steps}) * {C * W};")
            self.line(f"const int wr_ = (int)({row0} + (long long)({ru} / {steps}) * dpia_gsize);")
            for k, (buf, tm, c0, vals, stmt) in enumerate(stores):
                for bb in range(NB):
                    self.line(f"dpia::tma_store_2d(&{tm}, {c0 + bb * VB * W} + wc_, wr_, {ost} + ({ru} % {SO}) * "
                              f"{so_bytes} + {(k * NB + bb) * 4096});  /* {buf.cname} */")
            self.line("dpia::bulk_commit();")
            self.close()
        self.line(f"if ({lane} == 0)")
        self.lines += issue(pad1, f"{ru} + {S}")
        self.close()
        if stores:
            # the fold's last row stores are complete before the warp moves on
            self.line(f"if ({lane} == 0) dpia::bulk_wait_all();")
        pad = "  " * self.ind
        rexpr = "0" if lp.single else f"(int)(({iv} - dpia_gid) / dpia_gsize)"
        warp = "(dpia_tid >> 5)"
        pro = [f"{pad}const int {lane} = dpia_tid & 31, {sw} = {lane} & 7;",
               f"{pad}unsigned long long* {mb} = reinterpret_cast<unsigned long long*>(dpia_smem + {moff})"
               f" + {warp} * {S};",
               f"{pad}unsigned char* {st} = dpia_smem + {soff} + {warp} * {S * slot_bytes};",
               *([f"{pad}unsigned char* {ost} = dpia_smem + {ooff} + {warp} * {SO * so_bytes};"] if stores else []),
               f"{pad}const int {rnd} = {rexpr};",
               f"{pad}const int {u0} = {rnd} * {steps};",
               f"{pad}const long long {row0} = (long long)dpia_gid - {lane};",
               f"{pad}if ({rnd} == 0) {{",
               f"{pad}  if ({lane} == 0) {{",
               f"{pad}    dpia::tile_bar_init({mb}, {S}, {NS * NB});",
               f"{pad}    for (int wq_ = 0; wq_ < {S}; ++wq_)"]
        pro += issue(pad + "    ", "wq_")
        pro += [f"{pad}  }}", f"{pad}  __syncwarp();", f"{pad}}}"]
        self.lines[top:top] = pro
        return True

    def _vload(self, mode: str, b: Buffer, W: int, at: Ix) -> str:
        if mode == "queue32":
            self.prog.align[b.cname] = max(self.prog.align.get(b.cname, 16), 32)
            return f"dpia::vload32<{'true' if b.space == 'in' else 'false'}>({b.cname}, {self.r(at)})"
        return f"dpia::vload<{self.scalar}, {W}>({b.cname}, {self.r(at)})"

    def _finish_ring(self, streams, top, slot_at, take, T, W, C, S, j, jo, jd, rs, mb) -> bool:
        """Complete a ring-mode fold (see `_emit_vec_loop`): slot pointers,
        shared-memory reads, the refill after each piece and the prologue."""
        sb = 4 if self.scalar == "float" else 8
        piece = C * W * sb
        if piece % 16 or piece >= (1 << 20):
            return False
        moff = self.alloc_smem(8 * S)
        offs = [self.alloc_smem(S * piece) for _ in streams]
        pad1 = "  " * self.ind            # the piece loop's body
        pad2 = pad1 + "  "                # the lane loop's body
        vt = f"dpia::vec<{self.scalar}, {W}>"
        # this piece's slot of every stream, and the lanes the body reads
        self.lines[take:take] = [
            f"{pad2}const {vt} {name} = dpia::vload<{self.scalar}, {W}>({name}_s, {W} * {jd});"
            for name, _b, _base in streams]
        self.lines[slot_at:slot_at] = [
            f"{pad1}const {self.scalar}* {name}_s = reinterpret_cast<const {self.scalar}*>"
            f"(dpia_smem + {off}) + {rs} * {C * W};" for (name, _b, _base), off in zip(streams, offs)]

        st = self.prog.stream

        def fill(p, slot, at_j):
            out = [f"{p}{{", f"{p}  const int {j} = {at_j};"]
            for name, b, base in streams:
                if st is not None and b.key in st["partials"]:
                    # streaming tail: the rounds that wrote this piece's
                    # partials have published (ProgramEmitter._stream_plan);
                    # the piece's index within this launch's parity slice
                    at = Ix([(m, c) for m, c in base.terms if "dpia_par" not in IX.free_names(Ix([(m, c)]))])
                    cnt = f"dpia_counter + dpia_par * {st['R']}" if st["pipe"] else "dpia_counter"
                    out.append(f"{p}  dpia::stream_wait({cnt}, dpia_ready, "
                               f"(long long)({self.r(at)}) + {C * W}, {st['gsize']}, {st['n']});")
                    st["waits"] += 1
            out.append(f"{p}  dpia::ring_expect({mb} + {slot}, {piece * len(streams)}u);")
            for (name, b, base), off in zip(streams, offs):
                out.append(f"{p}  dpia::ring_copy(dpia_smem + {off} + {slot} * {piece}, "
                           f"{b.cname} + ({self.r(base)}), {piece}u, {mb} + {slot});")
            out.append(f"{p}}}")
            return out

        self.line(f"if ({jo} + {S * C} < {T})")
        self.lines += fill(pad1, rs, f"{jo} + {S * C}")
        self.close()
        rq = self.fresh("rq")
        pad = "  " * self.ind
        pro = [f"{pad}unsigned long long* {mb} = reinterpret_cast<unsigned long long*>(dpia_smem + {moff});",
               f"{pad}dpia::ring_init({mb}, {S});",
               f"{pad}for (int {rq} = 0; {rq} < {S}; {rq} += 1)"]
        pro += fill(pad, rq, f"{rq} * {C}")
        self.lines[top:top] = pro
        return True

    # ------------------------------------------------- packed FP32 FMA
    def _fma2_loop(self, p: Phrase, n: Nat, f: Lam) -> bool:
        """Instruction selection for a sequential loop whose body is one
        scalar update T[i] := T[i] + X[i] * Y[i] (the register-tile update of
        a reduceSeq/mapSeq nest): iterations 2t and 2t+1 are issued as one
        packed Blackwell fma.rn.f32x2 (FFMA2).  Each lane is the same single-
        rounding FMA the scalar code contracts to (--fmad=true), so results
        are bit-identical; the strategy (loop order, storage) is unchanged.
        Returns False, emitting nothing, when the loop does not qualify."""
        trip = self.nat_int(n)
        body = unapply(f.body)
        if self.scalar != "float" or self.pf is not None or trip is None or trip < 2 \
                or trip % 2 or trip > UNROLL_LIMIT or body is None or body[0] != ":=" \
                or not isinstance(body[1][0], Num):
            return False
        mark, nlines = len(self.lines), None
        v = self.fresh(f.binder)
        self.R[v] = trip // 2
        self.line("#pragma unroll")
        self.open(f"for (int {v} = 0; {v} < {trip // 2}; {v} += 1)")
        self.loops.append(Loop("seq", 0, v, trip // 2, nat(trip // 2), False))
        old = self.env.get(f.binder)
        stmts = []
        try:
            for k in (0, 1):
                self.env[f.binder] = Val(Idx(n), ixv=ix(v) * 2 + k)
                at = len(self.lines)
                self.comm(f.body)
                stmts.append(self.lines[at:])
                del self.lines[at:]
        finally:
            if old is None:
                self.env.pop(f.binder, None)
            else:
                self.env[f.binder] = old
            self.loops.pop()
        parsed = [_fma_stmt(b) for b in stmts]
        ok = all(x is not None for x in parsed)
        if ok:
            (t0, a0, b0), (t1, a1, b1) = parsed
            ok = t0 != t1 and t1 not in a0 + b0 and t0 not in a1 + b1
        if not ok:
            del self.lines[mark:]
            self.ind -= 1
            return False
        self.line(f"dpia::fma2({t0}, {t1}, {a0}, {b0}, {a1}, {b1});")
        self.close()
        return True

    def _declare_local(self, binder: str, d: DataType) -> Buffer:
        lp = [lp for lp in self.loops if lp.level in ("local", "lin")]
        full = d
        for lp_ in reversed(lp):
            full = Array(lp_.trip_nat, full)
        cname = self.fresh(binder)
        buf = Buffer(binder, cname, "local", full, [ix(lp_.var) for lp_ in lp])
        n = self._elements(full)
        if n is None:
            raise CudaError(f"local buffer {binder} needs a constant size (specialise sizes)")
        dims, elem = split_array(full)
        inner = self.nat_int(dims[-1]) if dims else None
        if isinstance(elem, Num) and len(dims) >= 2 and inner and inner % 32 == 0:
            # rows of a multiple of 32 scalars all start in bank 0, so a
            # column-wise access (e.g. the transposed store of a vec4-loaded
            # tile) hits one bank.  "swizzle": XOR the column with
            # 8*((row/4)%4) -- a bijection inside each row that keeps 8-aligned
            # groups (16/32-byte vectors) contiguous and sends the 4 rows of
            # a vec4's lanes x 8 columns to 32 distinct banks; "pad": 16 bytes
            # of padding per row (2-way at worst for that pattern)
            if SMEM_LAYOUT == "swizzle":
                buf.swz = (8, 4, 4)
            elif SMEM_LAYOUT == "pad":
                buf.pad = 4
                n = n // inner * (inner + 4)
        elif isinstance(elem, Num) and len(dims) == 1 and inner and inner % 32 == 0 and binder in self.pad32:
            # a 1-D buffer that work-items read at a stride of a multiple of
            # 32 scalars (each folding its own contiguous piece): 4 scalars of
            # padding after every 32 put the warp's work-items in distinct
            # banks, also for 16-byte vectors (element i lives at i + 4 (i / 32))
            buf.pad32 = 4
            n = n // 32 * 36
        # 128-byte aligned: the bank arithmetic of the swizzle / padding
        # above assumes each buffer starts in bank 0
        off = self.alloc_smem(n * self._elem_bytes(split_array(full)[1]), align=128)
        ct = self.types.c_elem(split_array(full)[1])
        self.line(f"{ct}* {cname} = reinterpret_cast<{ct}*>(dpia_smem + {off});")
        return buf

    def new(self, prim: str, d: DataType, f: Lam, node: Phrase = None):
        if node is not None and id(node) in self.pipelined and self.pipelined[id(node)][0] == "tma":
            _, buf, (plan, mb, tm), c1, c2, binder, trip = self.pipelined[id(node)]
            old = self.env.get(f.binder)
            self.env[f.binder] = buf
            k = self.env[binder].ixv
            S = plan["slots"]
            wait = (f"dpia::ring_wait({mb} + ({self.r(mod(k, S, self.R))}), "
                    f"(unsigned)(({self.r(k)} / {S}) & 1));")
            issue = self._tma_issue(plan, buf, mb, tm, k + 1, f"{self.r(k)} + 1 < {trip}")
            # this iteration's tile: every thread observes its mbarrier
            # phase right before the CTA barrier that precedes the first
            # read of the buffer (the hazard planner always puts one there).
            # The next tile goes into slice (k+1) % S: with 2 slices right
            # after that barrier (the slice was read by iteration k-1); with
            # 3 or more at once -- it was last read by iteration k-2, whose
            # reads every thread finished before iteration k-1's barrier
            if S >= 3:
                self.line(issue)
                issue = None
            hook = (len(self.loops), [wait], [issue] if issue else [])
            mark, ind, smem = len(self.lines), self.ind, self.smem
            self.barrier_hooks.append(hook)
            self.comm(c2)
            if hook in self.barrier_hooks:
                # no barrier at this level inside c2: every thread waits
                # first, and the refill follows a barrier after c2
                self.barrier_hooks.remove(hook)
                del self.lines[mark:]
                self.ind, self.smem = ind, smem
                self.line(wait)
                self.comm(c2)
                self.line("__syncthreads();")
                if issue:
                    self.line(issue)
            if old is None:
                del self.env[f.binder]
            else:
                self.env[f.binder] = old
            return
        if node is not None and id(node) in self.pipelined:
            buf, regs, c1, c2, binder, trip = self.pipelined[id(node)]
            old = self.env.get(f.binder)
            self.env[f.binder] = buf
            # commit this iteration's prefetched tile, then prefetch the next
            self.pf, self.pf_i = ("commit", regs), 0
            self.comm(c1)
            cur = self.env[binder]
            self.open(f"if ({self.r(cur.ixv)} + 1 < {trip})")
            self.env[binder] = Val(cur.dtype, ixv=cur.ixv + 1)
            self.pf, self.pf_i = ("refill", regs), 0
            self.comm(c1)
            self.pf = None
            self.env[binder] = cur
            self.close()
            self.comm(c2)
            if old is None:
                del self.env[f.binder]
            else:
                self.env[f.binder] = old
            return
        if node is not None and id(node) in self.hoisted:
            old = self.env.get(f.binder)
            self.env[f.binder] = self.hoisted[id(node)]
            self.comm(unapply(f.body)[2][0].snd)   # the staging already ran
            if old is None:
                del self.env[f.binder]
            else:
                self.env[f.binder] = old
            return
        space = NEW_SPACE[prim] or "private"
        cname = self.fresh(f.binder)
        if space == "private" and f.binder in self.promote:
            # written and read by different work-items: per-thread registers
            # cannot hold it -- stage it in the work-group's shared memory
            space = "local"
        if space == "private":
            self.decl_depth[f.binder] = len(self.loops)
            sl = self.slices.get(f.binder, 0)
            buf = Buffer(f.binder, cname, "private", d, [], sl)
            dims, elem = split_array(d)
            dims = dims[sl:]
            n = 1
            for x in dims:
                v = self.nat_int(x)
                if v is None:
                    raise CudaError(f"private buffer {f.binder} needs constant sizes")
                n *= v
            ct = self.types.c_elem(elem)
            self.line(f"{ct} {cname}" + (f"[{n}];" if dims else ";"))
            if self.prog.init_new:
                self._zero_private(buf, elem, n if dims else None)
        elif space == "local":
            buf = self._declare_local(f.binder, d)
        else:
            lp = [lp for lp in self.loops if lp.level in ("global", "workgroup", "local", "lin", "fold")]
            full = d
            for lp_ in reversed(lp):
                full = Array(lp_.trip_nat, full)
            buf = Buffer(f.binder, cname, "global", full, [ix(lp_.var) for lp_ in lp])
            self.prog.add_scratch(self, buf)
        old = self.env.get(f.binder)
        self.env[f.binder] = buf
        self.comm(f.body)
        if old is None:
            del self.env[f.binder]
        else:
            self.env[f.binder] = old

    def _zero_private(self, buf, elem, n):
        zero = self.lit(0)
        if isinstance(elem, Vector):
            zero = f"dpia::splat<{self.scalar}, {elem.width}>({zero})"
        if isinstance(elem, Pair):
            return
        if n is None:
            self.line(f"{buf.cname} = {zero};")
        else:
            self.line(f"#pragma unroll\n" + "  " * self.ind +
                      f"for (int z = 0; z < {n}; ++z) {buf.cname}[z] = {zero};")

    def _elements(self, d: DataType) -> Optional[int]:
        n = 1
        for x in split_array(d)[0]:
            v = self.nat_int(x)
            if v is None:
                return None
            n *= v
        return n

    def _elem_bytes(self, d: DataType) -> int:
        s = 4 if self.scalar == "float" else 8
        if isinstance(d, Num):
            return s
        if isinstance(d, Idx):
            return 8
        if isinstance(d, Vector):
            return s * d.width
        if isinstance(d, Pair):
            return 2 * max(self._tree_bytes(d.fst), self._tree_bytes(d.snd))
        raise CudaError(f"no size for {d}")

    def _tree_bytes(self, d):
        if isinstance(d, Array):
            n = d.size.const or 1
            return n * self._tree_bytes(d.elem)
        return self._elem_bytes(d)

    def alloc_smem(self, nbytes: int, align: int = 16) -> int:
        off = (self.smem + align - 1) // align * align
        self.smem = off + nbytes
        return off

    # ------------------------------------------------------------ loops
    def _level_of(self, prim: str) -> Tuple[str, int]:
        level, dim = LOOP_LEVEL[prim]
        if level == "plain":
            if self.per_thread:
                return "seq", 0
            if self.in_workgroup or self.prog.in_tail:
                return "lin", 0
            return "global", 0
        return level, dim

    def _geometry(self, level: str, dim: int):
        """(start C text, stride C text, stride int or None)."""
        L = self.launch
        if level == "seq":
            return "0", "1", 1
        if level == "workgroup":
            ax = "xy"[dim]
            g = L[0][dim] if L else None
            return f"(int)blockIdx.{ax}", f"(int)gridDim.{ax}", g
        if level == "local":
            ax = "xy"[dim]
            b = L[1][dim] if L else None
            return f"(int)threadIdx.{ax}", f"(int)blockDim.{ax}", b
        if level in ("lin", "fold"):
            b = L[1][0] * L[1][1] if L else None
            return "dpia_tid", "dpia_nthreads", b
        if level == "global":
            self.uses_gid = True
            g = L[0][0] * L[0][1] * L[1][0] * L[1][1] if L else None
            return "dpia_gid", "dpia_gsize", g
        raise CudaError(level)

    def loop(self, level: str, dim: int, n: Nat, binder: str, body, bind=None):
        trip = self.nat_int(n)
        if self.probing:
            # `_tma_plan`: every iteration of the staging's loops, with the
            # loop index a constant, so each copy's indices are constants
            # plus work-group-uniform terms
            if trip is None or trip * max(1, len(self.probe_recs)) > TMA_PROBE_MAX:
                raise _ProbeFail("unbounded or too large")
            names = [binder] + ([bind[0]] if bind else [])
            old = {nm: self.env.get(nm) for nm in names}
            for t in range(trip):
                self.loops.append(Loop(level, dim, "", 1, nat(1), True))
                self.env[binder] = Val(Idx(n), ixv=ix(t))
                if bind:
                    self.env[bind[0]] = bind[1](ix(t))
                body()
                self.loops.pop()
            for nm, ov in old.items():
                if ov is None:
                    self.env.pop(nm, None)
                else:
                    self.env[nm] = ov
            return
        start, stride, S = self._geometry(level, dim)
        v = self.fresh(binder)
        # `v += stride` must not overflow either: the last increment reaches
        # up to trip - 1 + stride (the stride's bound when it is a runtime
        # quantity: blockDim <= 1024, gridDim-based up to 2^31)
        step = S if S is not None else (1024 if level in ("local", "lin", "fold") else 1 << 31)
        wide = trip is None or trip - 1 + step > IX.INT32_MAX
        ctype = "long long" if wide else "int"
        self.R[v] = trip
        single = trip is not None and S is not None and trip <= S
        if level == "local" and self.launch and trip is not None and S is not None:
            single = trip <= S
        bound = str(trip) if trip is not None else f"({self.r(self.nat_ix(n))})"

        def enter(is_single):
            lp = Loop(level, dim, v, trip, n, is_single)
            self.loops.append(lp)
            old = {}
            names = [binder] + ([bind[0]] if bind else [])
            for nm in names:
                old[nm] = self.env.get(nm)
            self.env[binder] = Val(Idx(n), ixv=ix(v))
            if bind:
                self.env[bind[0]] = bind[1](ix(v))
            body()
            if level == "global" and self.prog.stream is not None and not self.prog.in_tail:
                # streaming tail: this warp's partials of the round are written
                rnd = "0" if is_single else f"({v} - dpia_gid) / dpia_gsize"
                base = f"dpia_par * {self.prog.stream['R']} + " if self.prog.stream["pipe"] else ""
                self.line("__syncwarp();")
                self.line(f"if ((dpia_tid & 31) == 0) dpia::stream_publish(dpia_counter + {base}{rnd});")
            for nm, ov in old.items():
                if ov is None:
                    self.env.pop(nm, None)
                else:
                    self.env[nm] = ov
            self.loops.pop()
            self.close()

        if self.pf is not None and level in ("local", "lin") and not single and trip is not None \
                and S is not None and trip <= PF_MAX_COPIES * S:
            # a work-item loop of a software-pipelined staging that takes a
            # few iterations per thread: unrolled into guarded copies so each
            # copy's loads get their own prefetch registers
            for k in range(-(-trip // S)):
                self.open("" if (k + 1) * S <= trip else f"if ({start} + {k * S} < {trip})")
                self.line(f"const {ctype} {v} = {start} + {k * S};")
                enter(True)
            return
        if single and level != "seq":
            if trip == S:
                self.open("")
            else:
                self.open(f"if ({start} < {trip})")
            self.line(f"const {ctype} {v} = {start};")
        elif level == "seq" and trip == 1:
            self.open("")
            self.line(f"const int {v} = 0;")
        else:
            if level == "seq" and trip is not None and trip <= UNROLL_LIMIT:
                self.line("#pragma unroll")

            self.open(f"for ({ctype} {v} = {start}; {v} < {bound}; {v} += {stride})")
        enter(single)

    def parfor(self, prim: str, targs, args):
        n, d = targs
        a, f = args
        if not (isinstance(f, Lam) and isinstance(f.body, Lam)):
            raise CudaError("parfor body must be a two-argument lambda")
        level, dim = self._level_of(prim)
        self.lint(prim, level, dim)
        ivar, ovar, body = f.binder, f.body.binder, f.body.body
        entering_wg = level == "workgroup"
        if entering_wg and not self.per_thread:
            binders = _binders(body) | {ivar, ovar}
            for node, d0, fl, c1 in self.invariant_stagings(body, binders):
                buf = self._declare_local(fl.binder, d0)
                self.env[fl.binder] = buf
                if not self.bulk_stage(c1, buf):
                    # block-uniform context (every thread of the work-group)
                    self.loops.append(Loop("workgroup", dim, "", 1, nat(1), True))
                    self.comm(c1)
                    self.loops.pop()
                self.line("__syncthreads();")
                del self.env[fl.binder]
                self.hoisted[id(node)] = buf
                self.hoisted_writes.add(id(c1))

        def emit_body():
            if entering_wg:
                self.plan_pipelines(body)
                self.plan_uniform(body, loop=True, alias={ovar: acc_roots(a, {})})
            self.comm(body)

        self.loop(level, dim, n, ivar, emit_body, bind=(ovar, lambda i: Alias(a, i)))

    def bulk_stage(self, c1: Phrase, buf: Buffer) -> bool:
        """toLocal staging of a whole input array into a shared buffer of the
        same layout -- `parforLocal (proj1 t) (lam i o. o := idx x i)` -- as
        one Blackwell bulk copy (TMA: cp.async.bulk global -> shared,
        completion counted on an mbarrier) issued by one thread, instead of
        a copy loop over the work-items.  Used for the block-invariant
        stagings (hoisted out of the work-group loop).  False when the
        pattern, the sizes or the alignment do not fit (the loop is emitted)."""
        if not BULK_STAGE or buf.swz is not None or buf.pad or buf.pad32 or buf.prefix:
            return False
        u = unapply(c1)
        if u is None or u[0] not in ("parforLocal", "parfor") or len(u[2]) != 2:
            return False
        (n, d), (acc, f) = u[1], u[2]
        if not (isinstance(acc, Proj) and acc.index == 1 and isinstance(acc.target, Var)
                and acc.target.name == buf.key and isinstance(f, Lam) and isinstance(f.body, Lam)):
            return False
        asg = unapply(f.body.body)
        if asg is None or asg[0] != ":=" or len(asg[2]) != 1 or not isinstance(asg[2][0], PairP):
            return False
        dst, src = asg[2][0].fst, asg[2][0].snd
        rd = unapply(src)
        if not (isinstance(dst, Var) and dst.name == f.body.binder and rd is not None
                and rd[0] == "idx" and len(rd[2]) == 2 and isinstance(rd[2][0], Var)
                and isinstance(rd[2][1], Var) and rd[2][1].name == f.binder):
            return False
        x = rd[2][0].name
        xb = self.env.get(x)
        if not (isinstance(xb, Buffer) and xb.space == "in" and not xb.prefix):
            return False
        dims, elem = split_array(xb.dtype)
        bdims, belem = split_array(buf.dtype)
        count = self.nat_int(n)
        if len(dims) != 1 or len(bdims) != 1 or not isinstance(elem, (Num, Vector)) or elem != belem \
                or count is None or self.nat_int(dims[0]) != count or self.nat_int(bdims[0]) != count:
            return False
        nbytes = count * self._elem_bytes(elem)
        if nbytes == 0 or nbytes % 16 or nbytes >= (1 << 20):
            return False
        off = self.alloc_smem(8)
        self.line(f"dpia::bulk_stage({buf.cname}, {xb.cname}, {nbytes}u, "
                  f"reinterpret_cast<unsigned long long*>(dpia_smem + {off}), dpia_tid);")
        return True

    def lint(self, prim, level, dim):
        enclosing = [(lp.level, lp.dim) for lp in self.loops if lp.level not in ("seq",)]
        lv = [e[0] for e in enclosing]
        if level == "workgroup":
            if "local" in lv or "lin" in lv or "fold" in lv or "global" in lv:
                raise CudaError(f"{prim}: work-group loop nested inside a work-item loop")
            if ("workgroup", dim) in enclosing:
                raise CudaError(f"{prim}: nested work-group loops over the same dimension")
        if level == "global" and enclosing:
            raise CudaError(f"{prim}: global loop nested inside another parallel loop")
        if level == "local":
            if ("local", dim) in enclosing:
                raise CudaError(f"{prim}: nested work-item loops over the same dimension")
            if "global" in lv or "fold" in lv or "lin" in lv:
                raise CudaError(f"{prim}: work-item loop nested inside a per-item loop")
            if "workgroup" not in lv and not self.prog.in_tail:
                raise CudaError(f"{prim}: work-item loop with no enclosing work-group loop")

    def plan_uniform(self, c: Phrase, loop: bool = False, alias=None, opaque=()):
        rotated = {fl.binder for cands in self.for_plans.values() for _n, _d, fl, _c1, _c2 in cands}
        planner = BarrierPlanner(self.prog.is_shared, self.hoisted_writes, opaque, rotated)
        self.barriers |= planner.run(c, loop, alias)

    # -------------------------------------- software-pipelined staging
    def pipeline_candidates(self, body: Phrase, binder: str, extra_ix: Set[str] = frozenset()):
        """newLocal stagings at the top level of a work-group-uniform
        sequential loop body whose initialising command only copies from
        read-only inputs through single-iteration work-item loops.  Their
        global loads for iteration k+1 can be issued into registers before
        iteration k's compute (the shared-memory writes stay in place)."""
        inputs = {n for n, sp in self.prog.spaces.items() if sp == "in"}
        L = self.launch
        found = []

        def simple(c) -> bool:
            for q in subtree_iter(c):
                if isinstance(q, Prim) and q.name in PARFOR_FAMILY:
                    lvl, dim = LOOP_LEVEL[q.name]
                    if lvl != "local":
                        return False
                if isinstance(q, Prim) and q.name in ("for", "reduceILocal", "new", "newLocal",
                                                       "newPrivate", "newGlobal", "barrier"):
                    return False
            for q in subtree_iter(c):
                u = unapply(q)
                if u is not None and u[0] in PARFOR_FAMILY and len(u[1]) == 2:
                    lvl, dim = LOOP_LEVEL[u[0]]
                    t = self.nat_int(u[1][0])
                    if t is None or t > PF_MAX_COPIES * L[1][dim]:
                        return False
            return True

        def walk(q):
            u = unapply(q)
            if u is None:
                return
            name, targs, args = u
            if name == ";":
                walk(args[0].fst)
                walk(args[0].snd)
            elif _is_new(name) and isinstance(args[0], Lam):
                fl = args[0]
                inner = unapply(fl.body)
                if name == "newLocal" and inner is not None and inner[0] == ";":
                    c1, c2 = inner[2][0].fst, inner[2][0].snd
                    R1, W1 = rw_sets(c1)
                    free = free_vars(c1) - {fl.binder}
                    outer_ix = {nm for nm, b in self.env.items() if isinstance(b, Val) and b.ixv is not None}
                    outer_ix |= extra_ix
                    if W1 == {fl.binder} and free <= inputs | {binder} | outer_ix and simple(c1):
                        found.append((q, targs[0], fl, c1, c2))
                walk(fl.body)

        walk(body)
        return found

    def plan_pipelines(self, body: Phrase):
        """Pipelining decisions for the uniform sequential loops of a
        work-group loop body, made before barrier planning so the planner
        knows which staged buffers rotate between two slices."""
        if not self.launch:
            return

        def walk(q, extra):
            u = unapply(q)
            if u is None:
                return
            name, targs, args = u
            if name == ";":
                walk(args[0].fst, extra)
                walk(args[0].snd, extra)
            elif _is_new(name) and isinstance(args[0], Lam):
                walk(args[0].body, extra)
            elif name in PARFOR_FAMILY and LOOP_LEVEL[name][0] == "workgroup" and \
                    len(args) == 2 and isinstance(args[1], Lam) and isinstance(args[1].body, Lam):
                # a nested work-group loop (2-D hierarchy): its index is a
                # work-group-uniform value inside, so plan its loops now,
                # so this level's barrier plan already sees the rotation
                walk(args[1].body.body, extra | {args[1].binder})
            elif name == "for" and isinstance(args[0], Lam):
                trip = self.nat_int(targs[0])
                if trip is not None and trip > 1:
                    cands = self.pipeline_candidates(args[0].body, args[0].binder, extra)
                    if cands:
                        self.for_plans[id(q)] = cands
        walk(body, frozenset())

    # ------------------------------------------- TMA tensor k-tiles
    def _barrier(self):
        """A CTA barrier, with the lines waiting for the next barrier at
        their own loop depth around it (a TMA-staged k-tile, `new`: one
        thread observes the tile's mbarrier just before the barrier, which
        then orders the landed tile before every thread's reads; the next
        tile is issued right after it, when no thread still reads the slice
        it overwrites)."""
        now = [h for h in self.barrier_hooks if h[0] == len(self.loops)]
        self.barrier_hooks = [h for h in self.barrier_hooks if h[0] != len(self.loops)]
        for _d, pre, _post in now:
            for ln in pre:
                self.line(ln)
        self.line("__syncthreads();")
        for _d, _pre, post in now:
            for ln in post:
                self.line(ln)

    def _probe_record(self, target, e: Phrase, steps):
        """`_tma_plan`: one copy statement of the staging -- the local
        destination index and the input source index of a whole vector (or
        one scalar) -- instead of emitting it."""
        self.probe_src = None
        r = self.resolve(e, steps)
        if isinstance(r, Ref):
            if r.suffix or r.flat is None or r.addr is not None:
                raise _ProbeFail("source path")
            src = (r.buf, r.flat, 1)
        elif self.probe_src is not None:
            src = self.probe_src
        else:
            raise _ProbeFail("source is not a plain read")
        if isinstance(target, VStore):
            dst, w = target.ref, target.width
        else:
            dst, w = target, 1
        if dst.suffix or dst.flat is None or dst.addr is not None or w != src[2]:
            raise _ProbeFail("destination path")
        if isinstance(src[1], list):       # a vector gathered lane by lane
            for lane, flat in enumerate(src[1]):
                self.probe_recs.append((dst.buf.key, dst.flat + lane, src[0], flat, 1))
        else:
            self.probe_recs.append((dst.buf.key, dst.flat, src[0], src[1], w))

    def _tma_no(self, why: str):
        self.tma_why = why          # why the last staging was not a TMA box (tests, debugging)
        return None

    def _tma_plan(self, c1: Phrase, fl: Lam, d0: DataType, binder: str, n: Nat, trip: int):
        """Is the staging command c1 of local buffer fl.binder (type d0) a
        plain 2-D box copy of one input -- element (r, c) of the tile read
        from X[origin(k) + r * P + c], origin linear in the staging loop's
        index k?  Decided by enumerating c1's copies with every work-item
        index a constant (`loop` in probe mode) and checking the index map
        element by element.  Returns the box geometry or None."""
        on = TMA_TILES if self.prog.tma_tiles is None else self.prog.tma_tiles
        if not on or not self.launch or self.pf is not None:
            return self._tma_no("off or unspecialised")
        dims, elem = split_array(d0)
        E = self._elements(d0)
        if not isinstance(elem, Num) or E is None or len(dims) < 2:
            return self._tma_no("not a 2-D scalar tile")
        eb = 4 if self.scalar == "float" else 8
        K = f"dpia_probe_{self.fresh('k')}"
        probe_buf = Buffer(fl.binder, "dpia_probe", "local", d0)
        saved = (len(self.lines), self.ind, self.smem, self.env.get(fl.binder), self.env.get(binder),
                 list(self.loops), self.R.get(K))
        self.env[fl.binder] = probe_buf
        self.env[binder] = Val(Idx(n), ixv=ix(K))
        self.R[K] = trip
        self.probing, self.probe_recs = True, []
        recs = None
        try:
            self.comm(c1)
            recs = self.probe_recs
        except Exception:  # noqa: BLE001 -- a probe that cannot follow the staging just declines
            recs = None
        finally:
            mark, self.ind, self.smem, ob, ok, self.loops, _ = saved
            del self.lines[mark:]
            self.probing, self.probe_recs, self.probe_src = False, [], None
            for nm, ov in ((fl.binder, ob), (binder, ok)):
                if ov is None:
                    self.env.pop(nm, None)
                else:
                    self.env[nm] = ov
        if not recs:
            return self._tma_no("copies not enumerable")
        xs = {id(r[2]) for r in recs}
        X = recs[0][2]
        if len(xs) != 1 or X.space != "in" or X.prefix or X.swz or X.pad or \
                any(r[0] != fl.binder for r in recs):
            return self._tma_no("not one plain input")
        xdims, xelem = split_array(X.dtype)
        NX = self._elements(X.dtype)
        if not isinstance(xelem, Num) or NX is None:
            return self._tma_no("input not scalar or unsized")
        # source = U + c: U the non-constant (work-group-uniform) part, shared by all copies
        uni = lambda e: Ix([(m, c) for m, c in e.terms if m != ()])  # noqa: E731
        U = uni(recs[0][3])
        emap: Dict[int, int] = {}
        for _key, dflat, _x, sflat, w in recs:
            dc, sc = dflat.const, (sflat + (U * -1)).const
            if dc is None or sc is None or uni(sflat) != U:
                return self._tma_no("source not tile-uniform plus a constant")
            for lane in range(w):
                if dc + lane in emap:
                    return self._tma_no("element written twice")
                emap[dc + lane] = sc + lane
        if sorted(emap) != list(range(E)):
            return self._tma_no("tile not covered exactly")
        c0 = emap[0]
        C = next((q for q in range(1, E) if emap[q] != c0 + q), E)
        if C == E:
            # one contiguous run: any row split of it is a box (P = C)
            C = max((q for q in range(1, min(E, 256) + 1)
                     if E % q == 0 and (q * eb) % 16 == 0 and E // q <= 256), default=0)
            if not C:
                return self._tma_no("no legal box width")
            P = C
        elif E % C:
            return self._tma_no("no legal box width")
        else:
            P = emap[C] - c0
        rows = E // C
        if P < C or any(emap[q] != c0 + (q // C) * P + q % C for q in range(E)):
            return self._tma_no("not a row-strided box")
        if C > 256 or rows > 256 or (C * eb) % 16 or (P * eb) % 16 or NX % P:
            return self._tma_no("box violates TMA limits")
        # origin(k) = U0 + a*k + c0, linear in k and free of other probe atoms
        a, U0 = 0, []
        for m, c in U.terms:
            if K in IX.free_names(Ix([(m, c)])):
                if len(m) != 1 or IX._ATOMS[m[0]] != ("v", K):
                    return self._tma_no("origin not linear in the loop index")
                a = c
            else:
                U0.append((m, c))
        # the box is issued in `parts` row bands, one per warp (lane 0), so
        # no single warp carries the issue work into every CTA barrier
        nthreads = self.launch[1][0] * self.launch[1][1]
        nw = nthreads // 32 if nthreads % 32 == 0 else 1
        parts = max(q for q in range(1, min(nw, rows, max(1, TMA_BANDS)) + 1) if rows % q == 0)
        return {"X": X, "C": C, "rows": rows, "P": P, "U0": Ix(U0) + c0, "a": a, "eb": eb, "E": E,
                "NX": NX, "trip": trip, "parts": parts, "slots": max(2, TMA_SLOTS)}

    def _tma_origin(self, plan, k: Ix):
        """(x, y) TMA coordinates of iteration k's box: column and row of
        its first element in X viewed as NX/P rows of P elements."""
        o = plan["U0"] + k * plan["a"]
        return self.r(mod(o, plan["P"], self.R)), self.r(div(o, plan["P"], self.R))

    def _tma_issue(self, plan, buf, mb: str, tm: str, k: Ix, cond: str = "") -> str:
        """Issue iteration k's box into slice k % 2: row band p of `parts`
        by lane 0 of warp p."""
        slot = mod(k, plan["slots"], self.R)
        x, y = self._tma_origin(plan, k)
        parts = plan["parts"]
        band = plan["rows"] // parts
        cond = f" && {cond}" if cond else ""
        if parts == 1:
            return (f"if (dpia_tid == 0{cond}) dpia::tma_tile_2d({buf.cname} + {plan['E']} * "
                    f"({self.r(slot)}), &{tm}, {x}, {y}, {plan['E'] * plan['eb']}u, {mb} + ({self.r(slot)}));")
        return (f"if ((dpia_tid & 31) == 0 && (dpia_tid >> 5) < {parts}{cond}) dpia::tma_tile_2d("
                f"{buf.cname} + {plan['E']} * ({self.r(slot)}) + {band * plan['C']} * (dpia_tid >> 5), "
                f"&{tm}, {x}, {y} + {band} * (dpia_tid >> 5), {band * plan['C'] * plan['eb']}u, "
                f"{mb} + ({self.r(slot)}));")

    def pipeline_prologue(self, cands, binder: str, n: Nat, trip: int, rotate: bool = False):
        for node, d0, fl, c1, c2 in cands:
            plan = self._tma_plan(c1, fl, d0, binder, n, trip) if rotate else None
            if plan is not None:
                # two slices written by TMA in plain row-major box layout
                S = plan["slots"]
                full = Array(nat(S), d0)
                ct = self.types.c_elem(split_array(d0)[1])
                cname = self.fresh(fl.binder)
                buf = Buffer(fl.binder, cname, "local", full)
                off = self.alloc_smem(S * plan["E"] * plan["eb"], align=128)
                self.line(f"{ct}* {cname} = reinterpret_cast<{ct}*>(dpia_smem + {off});")
                R = self.R
                buf.prefix = [lambda b=binder, S=S: mod(self.env[b].ixv, S, R)]
                self.rotated[fl.binder] = binder
                mb = self.fresh("tmb")
                moff = self.alloc_smem(8 * S, align=8)
                tm = self.prog.add_tmap(plan)
                if tm not in self.tmaps_used:
                    self.tmaps_used.append(tm)
                self.line(f"unsigned long long* {mb} = reinterpret_cast<unsigned long long*>(dpia_smem + {moff});")
                self.line(f"if (dpia_tid == 0) dpia::tile_bar_init({mb}, {S}, {plan['parts']});")
                self.line("__syncthreads();")
                self.line(self._tma_issue(plan, buf, mb, tm, ix(0)))
                self.pipelined[id(node)] = ("tma", buf, (plan, mb, tm), c1, c2, binder, trip)
                continue
            if rotate:
                # two slices, iteration k writes and reads slice k % 2
                buf = self._declare_local(fl.binder, Array(nat(2), d0))
                R = self.R
                buf.prefix = [lambda b=binder: mod(self.env[b].ixv, 2, R)] + buf.prefix
                self.rotated[fl.binder] = binder
            else:
                buf = self._declare_local(fl.binder, d0)
            self.env[fl.binder] = buf
            old = self.env.get(binder)
            self.env[binder] = Val(Idx(n), ixv=ix(0))
            regs: List = []
            self._pf_tag += 1
            mark = len(self.lines)
            self.pf = ("declare", regs)
            self.comm(c1)
            self.pf = None
            self.lines[mark:mark] = ["  " * self.ind + f"{T} {nm};" for nm, T in regs]
            if old is None:
                del self.env[binder]
            else:
                self.env[binder] = old
            del self.env[fl.binder]
            self.pipelined[id(node)] = (buf, regs, c1, c2, binder, trip)

    # ---------------------------------------------- loop-invariant staging
    def invariant_stagings(self, body: Phrase, inner_binders: Set[str]):
        """newLocal buffers at the top of a work-group loop body whose
        initialising command reads nothing bound inside the loop: staged
        once per block before the loop instead of once per iteration."""
        found = []

        def walk(q):
            u = unapply(q)
            if u is None:
                return
            name, targs, args = u
            if name == ";":
                walk(args[0].fst)
                walk(args[0].snd)
            elif _is_new(name) and isinstance(args[0], Lam):
                f = args[0]
                inner = unapply(f.body)
                if name == "newLocal" and inner is not None and inner[0] == ";":
                    c1, c2 = inner[2][0].fst, inner[2][0].snd
                    R1, W1 = rw_sets(c1)
                    _, W2 = rw_sets(c2)
                    free = free_vars(c1) - {f.binder}
                    if W1 == {f.binder} and f.binder not in W2 and not (free & inner_binders) \
                            and all(nm in self.env for nm in free):
                        found.append((q, targs[0], f, c1))
                        return
                walk(f.body)

        walk(body)
        return found

    # ---------------------------------------------------------- combine
    def combine(self, targs, args):
        n, d = targs
        f, init, src, k = args
        if self.per_thread:
            raise CudaError("reduceLocal must be at work-group level (not inside a work-item loop)")
        if not isinstance(d, (Num, Vector)):
            raise CudaError(f"reduceLocal combines num or vec values, not {d}")
        if self.launch and (self.launch[1][0] * self.launch[1][1]) % 32:
            raise CudaError("reduceLocal needs a work-group size that is a multiple of 32")
        T = self.types.c_elem(d)
        op = self.fresh("op")
        x, y, o = f.binder, f.body.binder, f.body.body.binder
        cx, cy, co = self.fresh("x"), self.fresh("y"), self.fresh("o")
        saved = {nm: self.env.get(nm) for nm in (x, y, o)}
        self.env[x] = Val(d, text=cx)
        self.env[y] = Val(d, text=cy)
        self.env[o] = Buffer(o, co, "private", d)
        self.open(f"auto {op} = [&](const {T}& {cx}, const {T}& {cy}) -> {T}")
        self.line(f"{T} {co};")
        self.loops.append(Loop("lambda", 0, "", None, nat(1), True))
        self.comm(f.body.body.body)
        self.loops.pop()
        self.line(f"return {co};")
        self.ind -= 1
        self.line("};")
        for nm, ov in saved.items():
            if ov is None:
                self.env.pop(nm, None)
            else:
                self.env[nm] = ov
        part, has = self.fresh("part"), self.fresh("has")
        self.line(f"{T} {part}; bool {has} = false;")
        sfx = self.fresh("e")

        def fold_body():
            self.line(f"const {T} {sfx} = {self.exp(src, [('i', ix(self.loops[-1].var))])};")
            self.line(f"{part} = {has} ? {op}({sfx}, {part}) : {sfx}; {has} = true;")

        self.loop("fold", 0, n, self.fresh("j"), fold_body)
        off_v = self.alloc_smem(33 * self._elem_bytes(d))
        off_h = self.alloc_smem(33)
        tot, tot_h = self.fresh("tot"), self.fresh("tot_has")
        self.line(f"bool {tot_h};")
        self.line(f"const {T} {tot} = dpia::block_combine<{T}>({part}, {has}, {op}, "
                  f"reinterpret_cast<{T}*>(dpia_smem + {off_v}), "
                  f"reinterpret_cast<bool*>(dpia_smem + {off_h}), dpia_tid, dpia_nthreads, {tot_h});")
        rv = self.fresh("r")
        self.line(f"const {T} {rv} = {tot_h} ? {op}({tot}, {self.exp(init, [])}) : {self.exp(init, [])};")
        saved_r = self.env.get(k.binder)
        self.env[k.binder] = Val(d, text=rv)
        self.comm(k.body)
        if saved_r is None:
            self.env.pop(k.binder, None)
        else:
            self.env[k.binder] = saved_r


# -------------------------------------------------------------- program

class ProgramEmitter:
    def __init__(self, outputs, inputs, float_mode=True, name="KERNEL", sigma=None, launch=None,
                 init_new=False, peer=False, tma_tiles: Optional[bool] = None):
        self.outputs, self.inputs = list(outputs), list(inputs)
        self.tma_tiles = tma_tiles
        self.peer = peer
        self.peer_kernel = None
        self.scalar = "float" if float_mode else "long long"
        self.types = TypeTable(self.scalar)
        self.name = "".join(ch if ch.isalnum() or ch == "_" else "_" for ch in name) or "KERNEL"
        self.sigma = dict(sigma) if sigma is not None else None
        self.launch = normalize_launch(launch)
        self.init_new = init_new
        self.base_env: Dict[str, object] = {}
        self.spaces: Dict[str, str] = {}
        for n, d in self.outputs:
            self.base_env[n] = Buffer(n, n, "out", d)
            self.spaces[n] = "out"
        for n, d in self.inputs:
            self.base_env[n] = Buffer(n, n, "in", d)
            self.spaces[n] = "in"
        self.scratch: List[Buffer] = []
        self.scratch_names: Set[str] = set()
        self.in_tail = False
        self.size_names: Set[str] = set()
        self.align: Dict[str, int] = {}      # buffer -> byte alignment its loads need (> 16)
        self.tmaps: Dict[str, Tuple[str, int, int, int, int, int, int, int]] = {}
        self.stream: Optional[dict] = None   # the kernel being emitted has a streaming tail
        self.buffer_kernels: Dict[str, Set[int]] = {}   # top-level buffer -> kernels that use it

    def add_tmap(self, plan) -> str:
        """The tensor-map kernel parameter of a TMA-staged tile (deduplicated
        per input and box): (input, element bytes, rows, cols, pitch, box)."""
        spec = (plan["X"].cname, plan["eb"], plan["NX"] // plan["P"], plan["P"], plan["P"] * plan["eb"],
                plan["rows"] // plan["parts"], plan["C"], plan.get("swizzle", 0))
        for nm, sp in self.tmaps.items():
            if sp == spec:
                return nm
        nm = f"dpia_tm{len(self.tmaps)}"
        self.tmaps[nm] = spec
        return nm

    def is_shared(self, name: str) -> bool:
        return self.spaces.get(name, "private") != "private"

    def add_scratch(self, ke: KernelEmitter, buf: Buffer):
        if buf.cname not in self.scratch_names:
            self.scratch_names.add(buf.cname)
            self.scratch.append(buf)
        ke.used_scratch.add(buf.cname)

    def collect_spaces(self, p: Phrase):
        stack = [p]
        while stack:
            q = stack.pop()
            u = unapply(q)
            if u is not None:
                if _is_new(u[0]) and u[2] and isinstance(u[2][0], Lam):
                    self.spaces[u[2][0].binder] = NEW_SPACE[u[0]] or "private"
                stack.extend(u[2])
            elif isinstance(q, Lam):
                stack.append(q.body)
            elif isinstance(q, PairP):
                stack.extend([q.fst, q.snd])
            elif isinstance(q, Proj):
                stack.append(q.target)

    # ---------------------------------------------------------- phases
    def items(self, p: Phrase, top: List):
        u = unapply(p)
        if u is not None and u[0] == ";" and len(u[2]) == 1:
            return self.items(u[2][0].fst, top) + self.items(u[2][0].snd, top)
        if u is not None and _is_new(u[0]) and len(u[2]) == 1 and isinstance(u[2][0], Lam):
            top.append((u[0], u[1][0], u[2][0].binder))
            return self.items(u[2][0].body, top)
        return [p]

    @staticmethod
    def is_grid_item(c: Phrase) -> bool:
        u = unapply(c)
        if u is None:
            return False
        name = u[0]
        if name in PARFOR_FAMILY and LOOP_LEVEL[name][0] in ("global", "workgroup", "plain"):
            return True
        if _is_new(name) and isinstance(u[2][0], Lam):
            return ProgramEmitter.is_grid_item(u[2][0].body)
        if name == ";":
            return ProgramEmitter.is_grid_item(u[2][0].fst) or ProgramEmitter.is_grid_item(u[2][0].snd)
        return contains_prim(c, {"parforGlobal", "parforWorkgroup", "parforWorkgroup1"})

    @staticmethod
    def is_cooperative(c: Phrase) -> bool:
        return contains_prim(c, {"reduceILocal", "parforLocal", "parforLocal1", "parfor"})

    def emit(self, p: Phrase) -> Tuple[str, CudaSignature]:
        self.collect_spaces(p)
        top: List = []
        items = self.items(p, top)
        for prim, d, binder in top:
            self.spaces[binder] = NEW_SPACE[prim] or "private"
        # group items into kernels: a grid item opens a kernel, the items
        # after it (until the next grid item) form its fused tail
        kernels: List[Tuple[Optional[Phrase], List[Phrase]]] = []
        for it in items:
            if self.is_grid_item(it):
                kernels.append((it, []))
            elif kernels:
                kernels[-1][1].append(it)
            else:
                kernels.append((None, [it]))
        # top-level buffers: place by use
        use: Dict[str, Set[int]] = {}
        for b_prim, d, binder in top:
            use[binder] = {ki for ki, (g, tail) in enumerate(kernels)
                           for it in ([g] if g is not None else []) + tail
                           if binder in exp_names(it)}
        n_items = {binder: sum(1 for it in items if binder in exp_names(it)) for _, _, binder in top}
        self.buffer_kernels = use
        top_global: List[Tuple[str, DataType]] = []
        kernel_top: Dict[int, List[Tuple[str, str, DataType]]] = {}
        for b_prim, d, binder in top:
            space = NEW_SPACE[b_prim] or "private"
            ks = use[binder]
            if space == "global" or (space == "private" and (len(ks) > 1 or any(
                    kernels[k][0] is not None and binder in exp_names(kernels[k][0]) for k in ks))):
                top_global.append((binder, d))
                self.spaces[binder] = "global"
            elif space == "local" and (len(ks) > 1 or n_items[binder] > 1):
                # outside any work-group, local memory has no per-group
                # meaning; a buffer shared by several phases lives in HBM
                top_global.append((binder, d))
                self.spaces[binder] = "global"
            elif space == "local":
                for k in ks:
                    kernel_top.setdefault(k, []).append(("local", binder, d))
            else:
                for k in ks:
                    kernel_top.setdefault(k, []).append(("private", binder, d))
        for binder, d in top_global:
            buf = Buffer(binder, "g_" + binder.replace("@", "_"), "global", d)
            self.base_env[binder] = buf
            self.scratch.append(buf)
            self.scratch_names.add(buf.cname)

        if self.peer:
            # fused cross-GPU combine: appended to the last kernel, which must
            # end in a single-work-group tail (all of the rank's blocks done)
            if not kernels or not kernels[-1][1]:
                raise CudaError("peer combine needs a program that ends in a reduction tail "
                                "(e.g. a top-level reduceLocal over work-group results)")
            if self.sigma is None or len(self.outputs) != 1:
                raise CudaError("peer combine needs specialised sizes and a single output")
            self.peer_kernel = len(kernels) - 1
        bodies, infos = [], []
        for ki, (grid, tail) in enumerate(kernels):
            text, info = self.emit_kernel(ki, grid, tail, kernel_top.get(ki, []))
            bodies.append(text)
            infos.append(info)

        with open(HEADER_PATH) as f:
            header = f.read()
        size_names = sorted(self.size_names) if self.sigma is None else []
        sig = CudaSignature(self.outputs, self.inputs,
                            [(b.cname, b.dtype) for b in self.scratch], size_names, infos,
                            self.scalar, self.launch, self.sigma, dict(self.spaces),
                            dict(self.align), dict(self.tmaps))
        src = ["// generated by the DPIA CUDA backend (paper_1710_08332_b200) for sm_100a",
               header, self.types.struct_text()] + bodies
        return "\n".join(s for s in src if s) + "\n", sig

    def _stream_plan(self, ki, grid, tail) -> Optional[dict]:
        """Can this kernel's tail stream?  Its grid phase must be one
        parforGlobal over n work-items (n a multiple of 32, a 1-D launch of
        whole warps, so every warp's loop trip is uniform) that writes
        one-scalar-per-item scratch partials, and its tail single-thread
        items only.  Whether the tail then reads the partials only through the
        ring is checked after emission (emit_kernel retries without)."""
        if not STREAM_TAIL or grid is None or not tail or any(self.is_cooperative(t) for t in tail) \
                or self.peer or not self.launch or self.sigma is None:
            return None
        (gx, gy), (lx, ly) = self.launch
        u = unapply(grid)
        if gy != 1 or (lx * ly) % 32 or u is None or u[0] != "parforGlobal":
            return None
        try:
            n = int(u[1][0].evaluate(self.sigma))
        except Exception:  # noqa: BLE001
            n = None
        if not isinstance(n, int) or n <= 0 or n % 32:
            return None
        _, W = rw_sets(grid)
        parts = set()
        for b in self.scratch:
            if b.key in W:
                dims, elem = split_array(b.dtype)
                try:
                    count = 1
                    for x in dims:
                        count *= int(x.evaluate(self.sigma))
                except Exception:  # noqa: BLE001
                    return None
                if not isinstance(elem, Num) or count != n:
                    return None
                parts.add(b.key)
        if not parts:
            return None
        gsize = gx * lx * ly
        # parity pipelining: the grid phase writes nothing but the partials,
        # which no other kernel touches
        shared = {b.key for b in self.scratch} | {nm for nm, _ in self.outputs}
        pipe = STREAM_PIPE and (W & shared) <= parts and \
            all(self.buffer_kernels.get(k) == {ki} for k in parts)
        # launch slots: enough that K launches' serial tails (n in-order adds,
        # ~2.5 ns each) cover the grid phase of one launch; at least
        # STREAM_PIPE_SLOTS, at most 16
        K = max(STREAM_PIPE_SLOTS, min(16, -(-n // 4096)))
        return {"n": n, "gsize": gsize, "R": -(-n // gsize), "partials": parts, "waits": 0, "pipe": pipe,
                "K": K}

    def emit_kernel(self, ki, grid, tail, decls):
        kname = f"{self.name}_k{ki}"
        body_lines = None
        plan = self._stream_plan(ki, grid, tail)
        for stream in ([plan, None] if plan else [None]):
            self.stream = stream
            saved = {}
            if stream is not None and stream["pipe"]:
                # the partials get one slice per launch parity
                for b in self.scratch:
                    if b.key in stream["partials"]:
                        saved[b.key] = (b.dtype, list(b.prefix))
                        b.dtype = Array(nat(stream["K"]), b.dtype)
                        b.prefix = [ix("dpia_par")] + list(b.prefix)
            ke = KernelEmitter(self, kname)
            for attempt in ("record", "final"):
                ke.reset()
                if stream is not None:
                    stream["waits"] = 0
                ke.recording = attempt == "record"
                self._kernel_body(ke, grid, tail, decls)
                if attempt == "record":
                    ke.slices, ke.promote = self._decide_slices(ke)
                    for key in ke.promote:
                        self.spaces[key] = "local"
                    ke.pad32 = {k for k, hit in ke.local_reads.items() if hit} if SMEM_PAD_1D else set()
                body_lines = ke.lines
            if stream is None or (stream["waits"] and not ke.stream_unsafe):
                break
            for b in self.scratch:
                if b.key in saved:
                    b.dtype, b.prefix = saved[b.key]
        stream, self.stream = self.stream, None
        pipe = stream is not None and stream["pipe"]
        args: List[Tuple[str, str]] = [("out", n) for n, _ in self.outputs]
        args += [("in", n) for n, _ in self.inputs]
        args += [("scratch", b.cname) for b in self.scratch if b.cname in ke.used_scratch
                 or b.key in self._kernel_names(grid, tail)]
        sizes = []
        if self.sigma is None:
            sizes = sorted(self._size_vars())
            self.size_names |= set(sizes)
            args += [("size", s) for s in sizes]
        args += [("tmap", t) for t in ke.tmaps_used]
        if grid is not None and tail:
            args.append(("counter", "dpia_counter"))
        if pipe:
            args.append(("epoch", "dpia_epoch"))
        if self.peer and ki == self.peer_kernel:
            args += [("peer_boxes", "dpia_peer_boxes"), ("peer_rank", "dpia_rank"),
                     ("peer_world", "dpia_world"), ("peer_epoch", "dpia_epoch")]
        params, views = [], []
        for kind, n in args:
            if kind == "size":
                params.append(f"long long {n}")
                continue
            if kind == "counter":
                params.append("unsigned int *dpia_counter")
                continue
            if kind == "tmap":
                params.append(f"const __grid_constant__ dpia::TensorMap {n}")
                continue
            if kind == "epoch":
                params.append("unsigned int dpia_epoch")
                continue
            if kind.startswith("peer_"):
                params.append({"peer_boxes": "const unsigned long long * __restrict__ dpia_peer_boxes",
                               "peer_rank": "int dpia_rank", "peer_world": "int dpia_world",
                               "peer_epoch": "unsigned int dpia_epoch"}[kind])
                continue
            ct = self.types.c_elem(split_array(self._arg_type(n))[1])
            q = "const " if kind == "in" else ""
            rs = " __restrict__" if kind in ("in", "out") else ""
            if ct == self.scalar:
                params.append(f"{q}{self.scalar} *{rs} {n}")
            else:
                params.append(f"{q}{self.scalar} *{rs} {n}_raw")
                views.append(f"  {q}{ct}*{rs} {n} = reinterpret_cast<{q}{ct}*>({n}_raw);")
        L = self.launch
        bounds = f"__launch_bounds__({L[1][0] * L[1][1]}) " if L else ""
        head = [f'extern "C" __global__ void {bounds}{kname}({", ".join(params)}) {{',
                # 1024: a 128-byte-swizzled TMA box's slots (row folds) must
                # sit on 1024-byte boundaries, also behind static shared data
                f"  extern __shared__ __align__({1024 if ke.smem_1k else 128}) unsigned char dpia_smem[];"]
        head += views
        if L:
            head.append(f"  const int dpia_nthreads = {L[1][0] * L[1][1]};")
        else:
            head.append("  const int dpia_nthreads = (int)(blockDim.x * blockDim.y);")
        head.append("  const int dpia_tid = (int)(threadIdx.y * blockDim.x + threadIdx.x);")
        if pipe:
            head.append(f"  const int dpia_par = (int)(dpia_epoch % {stream['K']}u);")
            head.append("  bool dpia_pw = true;")
            body_lines = self._pipe_waits(body_lines, ke, stream, args, CHAIN and ki == 0)
        if ki > 0:
            # launched with programmatic dependent launch (launcher.Executable):
            # the grid may be scheduled while the previous phase's kernel still
            # runs and waits here until that grid has completed and its memory
            # is visible (a no-op under an ordinary launch)
            head.append('  asm volatile("griddepcontrol.wait;" ::: "memory");')
        elif CHAIN:
            # the first phase may itself be chained behind the previous launch
            # of a program on the stream (Executable.launch(chain=True)): it
            # lets its own dependent launch early, streams its inputs at once
            # and waits for that grid only before it first touches memory the
            # grid may still use (`_chain_waits`); all no-ops when not chained
            # Trigger placement.  At once by default: the dependent launch is
            # scheduled while this one drains.  A small grid (under half the
            # B200's 148 x 2048 resident threads) whose grid phase writes an
            # output instead triggers right after its first wait for the
            # previous grid (`dpia::pdl_wait_once<true>`), so at most two
            # launches are resident: otherwise the SMs fill with blocks of
            # later launches waiting to store (the reference's scal: chained
            # 2.4x slower than unchained; the large grids and the reductions
            # lose 1-10 % with the late trigger, `profiles/r02c_chain_trigger.txt`).
            # A slot-pipelined streaming tail always triggers at once.
            L_ = self.launch
            small = L_ is not None and L_[0][0] * L_[0][1] * L_[1][0] * L_[1][1] < 148 * 1024
            writes_out = grid is not None and bool(rw_sets(grid)[1] & {nm for nm, _ in self.outputs})
            late = not pipe and (CHAIN_TRIGGER == "wait" or (CHAIN_TRIGGER == "auto" and small and writes_out))
            if not late:
                head.append("  dpia::pdl_trigger();")
            head.append("  bool dpia_chained = true;")
            if not pipe:
                body_lines = self._chain_waits(body_lines, args)
                if late:
                    body_lines = [ln.replace("dpia::pdl_wait_once(dpia_chained);",
                                             "dpia::pdl_wait_once<true>(dpia_chained);") for ln in body_lines]
        if ke.uses_gid or stream is not None:
            wide = not L or L[0][0] * L[0][1] * L[1][0] * L[1][1] > IX.INT32_MAX
            it = "long long" if wide else "int"
            # a streaming tail's extra block is the last block of the grid
            # and takes no work-items
            gx = "(gridDim.x - 1)" if stream is not None else "gridDim.x"
            head.append(f"  const {it} dpia_gid = ({it})(blockIdx.y * {gx} + blockIdx.x) * "
                        "dpia_nthreads + dpia_tid;")
            head.append(f"  const {it} dpia_gsize = ({it}){gx} * gridDim.y * dpia_nthreads;")
        text = "\n".join(head + body_lines + ["}"])
        info = KernelInfo(kname, "launch" if grid is not None else "single", args, ke.smem,
                          grid is not None and bool(tail), grid_item=grid, tail_items=list(tail),
                          barriers=frozenset(ke.barriers), hoisted=frozenset(ke.hoisted),
                          rotated=dict(ke.rotated), decls=list(decls),
                          extra_blocks=1 if stream is not None else 0,
                          counter_words=(stream["K"] * (stream["R"] + 1) if pipe else max(4, stream["R"]))
                          if stream is not None else 4,
                          counter_init=self._release_init(stream) if pipe else [])
        return text, info

    @staticmethod
    def _chain_waits(lines: List[str], args) -> List[str]:
        """Insert `dpia::pdl_wait_once` before every line of a first-phase
        kernel that names a non-input global buffer (an output, a scratch
        buffer, the fused tail's counter, the peer mailboxes): the inputs are
        read-only for both chained grids, everything else may still be read
        or written by the grid this one is chained behind.  The wait runs
        once per thread (a flag), so sites inside loops cost a predicate
        test; a site right after a #pragma is fenced before the pragma."""
        names = [n for kind, n in args if kind not in ("in", "size", "tmap")]
        names = [n for n in names] + [n + "_raw" for n in names]
        if not names:
            return lines
        pat = re.compile(r"\b(" + "|".join(re.escape(n) for n in names) + r")\b")
        out: List[str] = []
        for ln in lines:
            if pat.search(ln):
                ind = ln[:len(ln) - len(ln.lstrip())]
                at = len(out)
                if at and out[-1].lstrip().startswith("#pragma"):
                    at -= 1
                out.insert(at, f"{ind}dpia::pdl_wait_once(dpia_chained);")
            out.append(ln)
        return out

    @staticmethod
    def _release_init(st) -> List[Tuple[int, int]]:
        """Release words of a pipelined streaming tail before the first
        launch: slot s's first launch (the smallest epoch >= EPOCH_BASE with
        epoch % K == s) must find the slot released by launch epoch - K."""
        K, R = st["K"], st["R"]
        out = []
        for slot in range(K):
            first = EPOCH_BASE + (slot - EPOCH_BASE) % K
            out.append((K * R + slot, first - K))
        return out

    def _pipe_waits(self, lines: List[str], ke, st, args, chained: bool) -> List[str]:
        """Waits of a parity-pipelined streaming-tail kernel: before every
        line that names the partials or the counters, the launch two back
        (same parity) must have released them (`dpia::parity_wait_once`);
        in the tail, before every line that names an output, the previous
        grid must have completed (`dpia::pdl_wait_once`, chained first
        kernels only) -- launches' outputs are written in launch order."""
        mine = [b.cname for b in self.scratch if b.key in st["partials"]] + ["dpia_counter"]
        outs = [n for kind, n in args if kind == "out"]
        pat_p = re.compile(r"\b(" + "|".join(re.escape(n) for n in mine + [n + "_raw" for n in mine]) + r")\b")
        pat_o = re.compile(r"\b(" + "|".join(re.escape(n) for n in outs + [n + "_raw" for n in outs]) + r")\b") \
            if outs else None
        tail_from = ke.tail_mark if ke.tail_mark is not None else len(lines)
        rel = f"dpia_counter + {st['K'] * st['R']} + dpia_par"
        out: List[str] = []
        for k, ln in enumerate(lines):
            waits = []
            if pat_p.search(ln):
                waits.append(f"dpia::parity_wait_once(dpia_pw, {rel}, dpia_epoch, {st['K']}u);")
            if chained and k >= tail_from and pat_o is not None and pat_o.search(ln):
                waits.append("dpia::pdl_wait_once(dpia_chained);")
            if waits:
                ind = ln[:len(ln) - len(ln.lstrip())]
                at = len(out)
                if at and out[-1].lstrip().startswith("#pragma"):
                    at -= 1
                out[at:at] = [ind + w for w in waits]
            out.append(ln)
        return out

    def _kernel_names(self, grid, tail):
        names = set()
        for it in ([grid] if grid is not None else []) + tail:
            names |= exp_names(it)
        return names

    def _arg_type(self, n):
        for nn, d in self.outputs + self.inputs:
            if nn == n:
                return d
        for b in self.scratch:
            if b.cname == n:
                return b.dtype
        raise KeyError(n)

    def _size_vars(self):
        out = set()
        for _, d in self.outputs + self.inputs:
            for x in split_array(d)[0]:
                out |= set(x.free)
        for b in self.scratch:
            for x in split_array(b.dtype)[0]:
                out |= set(x.free)
        return out

    def _kernel_body(self, ke: KernelEmitter, grid, tail, decls):
        saved_env = {}
        if self.stream is not None and self.stream["pipe"]:
            ke.R["dpia_par"] = self.stream["K"]
        for space, binder, d in decls:
            # declare kernel-level buffers (top-level local / private)
            if space == "local":
                n = ke._elements(d)
                if n is None:
                    raise CudaError(f"local buffer {binder} needs a constant size")
                off = ke.alloc_smem(n * ke._elem_bytes(split_array(d)[1]))
                ct = self.types.c_elem(split_array(d)[1])
                cname = ke.fresh(binder)
                ke.line(f"{ct}* {cname} = reinterpret_cast<{ct}*>(dpia_smem + {off});")
                saved_env[binder] = Buffer(binder, cname, "local", d)
        ke.env.update(saved_env)
        st = self.stream
        if grid is not None:
            self.in_tail = False
            if not self.is_grid_item(grid):
                raise CudaError("internal: grid item expected")
            if st is not None:
                ke.open("if (blockIdx.x != gridDim.x - 1)")
            ke.comm(grid)
            if st is not None:
                ke.close()
        if tail:
            self.in_tail = True
            if grid is not None and st is not None:
                # the streaming tail block: partials [0, dpia_ready) are known
                # to be published (dpia::stream_wait)
                ke.open("else")
                ke.tail_mark = len(ke.lines)
                ke.line("long long dpia_ready = 0;")
            elif grid is not None:
                ke.line("__shared__ bool dpia_last;")
                ke.open("if (dpia::grid_arrive(dpia_counter, dpia_tid, &dpia_last))")
            for space, binder, d in decls:
                if space == "private" and binder in ke.promote:
                    ke.env[binder] = ke._declare_local(binder, d)
                elif space == "private":
                    dims, elem = split_array(d)
                    n = ke._elements(d)
                    cname = ke.fresh(binder)
                    ke.decl_depth[binder] = len(ke.loops)
                    ke.line(f"{self.types.c_elem(elem)} {cname}" + (f"[{n}];" if dims else ";"))
                    ke.env[binder] = Buffer(binder, cname, "private", d)
            ke.plan_uniform(seq_all(list(tail)),
                            opaque={id(it) for it in tail if not self.is_cooperative(it)})
            released = False
            for q, it in enumerate(tail):
                if self.is_cooperative(it):
                    ke.comm(it)
                else:
                    if id(it) in ke.barriers:
                        ke.line("__syncthreads();")
                    ke.open("if (dpia_tid == 0)")
                    ke.single_thread = True
                    ke.comm(it)
                    ke.single_thread = False
                    ke.close()
                if grid is not None and st is not None and st["pipe"] and not released and \
                        not any(exp_names(t2) & st["partials"] for t2 in tail[q + 1:]):
                    # the partials of this launch's parity are consumed: reset
                    # its round counters and release the parity to the launch
                    # two ahead, before this launch waits to write its outputs
                    R = st["R"]
                    ke.line(f"if (dpia_tid == 0) {{ for (int dpia_r = 0; dpia_r < {R}; ++dpia_r) "
                            f"dpia_counter[dpia_par * {R} + dpia_r] = 0u; "
                            f"dpia::parity_release(dpia_counter + {st['K'] * R} + dpia_par, dpia_epoch); }}")
                    released = True
            if self.peer and ke.kname == f"{self.name}_k{self.peer_kernel}":
                on, od = self.outputs[0]
                from ..layout import shape_of
                nsc = shape_of(od, self.sigma, 4 if self.scalar == "float" else 8)[0] \
                    // (4 if self.scalar == "float" else 8)
                ke.line("__syncthreads();")
                ke.line(f"if (dpia_tid < 32) dpia::peer_sum<{self.scalar}>("
                        f"reinterpret_cast<{self.scalar}*>({on}), {nsc}, dpia_peer_boxes, dpia_rank, "
                        "dpia_world, dpia_epoch, dpia_tid, dpia_nthreads);")
            if grid is not None and st is not None:
                if not st["pipe"]:
                    # every round has been published and consumed: reset the
                    # counters for the next launch
                    ke.line(f"if (dpia_tid == 0) for (int dpia_r = 0; dpia_r < {st['R']}; ++dpia_r) "
                            "dpia_counter[dpia_r] = 0u;")
                ke.close()
            elif grid is not None:
                ke.line("dpia::grid_reset(dpia_counter, dpia_tid);")
                ke.close()
            self.in_tail = False

    def _decide_slices(self, ke: KernelEmitter) -> Dict[str, int]:
        """Thread slicing of work-group-level private buffers (see module doc)."""
        L = self.launch
        one_d = L is not None and L[1][1] == 1
        out, promote = {}, set()
        for key, recs in ke.records.items():
            best = None
            keys_at: List = []
            # a buffer that only the single-thread (dpia_tid == 0) regions
            # touch -- e.g. the accumulator of a sequential top-level reduce
            # in a fused tail -- lives in thread 0's registers: every access
            # is by the same thread, so no other work-item needs to see it
            if recs and all(st for _, _, st, _ in recs):
                continue
            distributed = any(st or any(lp.level in ("local", "lin", "fold", "global")
                                        for lp in loops[depth:])
                              for _, loops, st, depth in recs)
            if L is None:
                if distributed:
                    promote.add(key)
                continue
            for idxs, loops, st, depth in recs:
                m = 0
                for j, e in enumerate(idxs):
                    v = e.var_name()
                    lp = next((lp for lp in loops if lp.var == v), None) if v else None
                    if lp is None or not lp.single or lp.level not in ("local", "lin", "fold"):
                        break
                    if one_d and (lp.level != "local" or lp.dim == 0):
                        kkey = ("thread", 0)
                    elif lp.level == "local":
                        kkey = ("local", lp.dim)
                    else:
                        kkey = ("lin", 0)
                    if j < len(keys_at) and keys_at[j] != kkey:
                        break
                    if j == len(keys_at):
                        keys_at.append(kkey)
                    m += 1
                best = m if best is None else min(best, m)
                if best == 0:
                    break
            if best:
                out[key] = best
            elif distributed:
                promote.add(key)
        return out, promote


# ------------------------------------------------------------------ API

def emit_cuda(p: Phrase, outputs: List[Tuple[str, DataType]], inputs: List[Tuple[str, DataType]],
              float_mode: bool = True, name: str = "KERNEL", init_new: bool = False,
              simplify: bool = True, sigma: Optional[Dict[str, int]] = None,
              launch=None, peer: bool = False,
              tma_tiles: Optional[bool] = None) -> Tuple[str, CudaSignature]:
    """Render an imperative DPIA command as CUDA C for sm_100a.

    Drop-in for the reference's `emit_kernel(p, outputs, inputs, float_mode,
    name, init_new, simplify)` (SRC/opencl.py:265-271).  Accepts the Stage II
    phrase directly or the reference's hoisted form.  `sigma` and `launch`
    optionally specialise sizes and the (G, L) launch geometry into the
    source (run_kernel always does), which enables single-iteration loops,
    thread slicing and compile-time index arithmetic.  tma_tiles: stage
    rotating 2-D box k-tiles with TMA tensor copies (None: TMA_TILES)."""
    del simplify  # subscripts are always range-simplified
    return ProgramEmitter(outputs, inputs, float_mode, name, sigma, launch, init_new, peer,
                          tma_tiles).emit(p)
