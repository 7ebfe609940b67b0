"""`dpia run --gpus K`: one program over K GPUs of this node (SURVEY.md 8f
row f1, 8e).

The outermost map of a strategy program runs over chunks of its inputs that
are independent: iteration i reads rows [i*c, (i+1)*c) of its (zipped,
vectorised) inputs and writes only element i of the map's result (SCIR's
disjoint-writes guarantee, SRC/checker.py:219-249).  When every input is an
array of c_p * n elements for the program's one size parameter n, the chunk
range splits into K contiguous blocks by specialising the *same* program to
n / K and giving device k the k-th contiguous block of every input.

Two program shapes are sharded (`shard_spec` recognises them on the surface
phrase and refuses anything else):

  map   body = [join | asScalarW | toX]* (mapF F (split c V))   (or mapF F V)
        output = the shards' outputs concatenated in device order
  sum   body = reduce(Local) (+) 0 (map-shaped body as above)
        output = the shards' partial sums combined on device 0 by the
        backend's own emitted `reduceLocal (+) 0` over the K partials

where F is closed (it mentions no program parameter) and V is a view of the
parameters that preserves element order (a parameter, zip, asVectorW).  The
shards run concurrently, one stream per device, from this one host process
(a command-line convenience; bench.py's multi-GPU path is one process per
GPU).  In int mode the result is bit-identical to one device; in float mode
`sum` changes the association across shards and stays within
the stated tolerance.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional

import numpy as np

from . import layout as LY
from . import runtime as RT
from .dtypes import Array, ExpT, Num
from .sizes import nat as nat_of
from .terms import Lam, Lit, Var, free_vars, substitute, unapply

MAPS = {"map", "mapGlobal", "mapWorkgroup", "mapLocal", "mapSeq", "mapWorkgroup1", "mapLocal1"}
WRAPS = {"join", "toGlobal", "toLocal", "toPrivate"}
VIEWS = {"zip"}


class ShardError(ValueError):
    """The program cannot be split over devices (or the sizes do not divide)."""


@dataclass(frozen=True)
class ShardSpec:
    nat: str          # the size parameter the chunk range scales with
    kind: str         # "map" | "sum"


def _linear(size, nat: str) -> bool:
    """size is c * nat for a constant c >= 1."""
    if set(size.free) != {nat}:
        return False
    one, two = size.evaluate({nat: 1}), size.evaluate({nat: 2})
    return one >= 1 and two == 2 * one and size.evaluate({nat: 0}) == 0


def _strip(p, names):
    while True:
        u = unapply(p)
        if u is None:
            return p
        head, _targs, args = u
        if head in names or (head.startswith("asScalar") and head[8:].isdigit()):
            p = args[-1]
            continue
        return p


def _is_view(p, params) -> bool:
    if isinstance(p, Var):
        return p.name in params
    u = unapply(p)
    if u is None:
        return False
    head, _targs, args = u
    if head in VIEWS or (head.startswith("asVector") and head[8:].isdigit()):
        return all(_is_view(a, params) for a in args)
    return False


def _mentions_size(p, nat: str) -> bool:
    """Whether the size variable occurs anywhere in p (binder annotations,
    type arguments, literal types): substituting it must leave p unchanged."""
    return substitute(p, nat, _PROBE) != p


_PROBE = nat_of(1 << 40)


def _chunk_local(p, params, nat: str) -> bool:
    """The body maps a closed F over constant-size chunks of a view of the
    inputs.  F and the split factor must not depend on the size parameter:
    a shard specialises it to n / K, which would otherwise change the
    chunks themselves (and so every per-chunk result), not just their
    number."""
    body = _strip(p, WRAPS)
    u = unapply(body)
    if u is None or u[0] not in MAPS:
        return False
    f, e = u[2][-2], u[2][-1]
    if free_vars(f) & set(params) or _mentions_size(f, nat):
        return False
    s = unapply(e)
    if s is not None and s[0] == "split":
        if s[1] and nat in getattr(s[1][0], "free", frozenset()):
            return False
        e = s[2][-1]
    return _is_view(e, params)


def _is_plus(f) -> bool:
    if not (isinstance(f, Lam) and isinstance(f.body, Lam)):
        return False
    u = unapply(f.body.body)
    return u is not None and u[0] == "+"


def shard_spec(prog) -> ShardSpec:
    """How `prog` splits over devices, or ShardError saying why it cannot."""
    src = prog.source
    if len(src.nat_params) != 1:
        raise ShardError(f"sharding needs exactly one size parameter (has {len(src.nat_params)})")
    nat = src.nat_params[0]
    params = [n for n, _ in src.params]
    for n, t in src.params:
        if not (isinstance(t, ExpT) and isinstance(t.data, Array) and _linear(t.data.size, nat)):
            raise ShardError(f"input {n} is not an array of c * {nat} elements")
    out = prog.out_type
    body = src.body
    if isinstance(out, Array) and _linear(out.size, nat):
        if _chunk_local(body, params, nat):
            return ShardSpec(nat, "map")
        raise ShardError("the body is not a map over contiguous chunks of its inputs")
    u = unapply(body)
    if (isinstance(out, Num) and u is not None and u[0] in ("reduce", "reduceLocal", "reduceSeq") and _is_plus(u[2][0])
            and isinstance(u[2][1], Lit) and u[2][1].value == 0 and _chunk_local(u[2][2], params, nat)):
        return ShardSpec(nat, "sum")
    raise ShardError("only chunk-local maps and (+)/0 reductions of them are sharded")


def _block(v, k: int, K: int):
    n = len(v)
    if n % K:
        raise ShardError(f"an input of {n} elements does not split over {K} devices")
    return v[k * n // K:(k + 1) * n // K]


def run_sharded(prog, inputs: Dict[str, object], launch, sigma: Dict[str, int], float_mode: bool,
                gpus: int, name: str = "KERNEL", first_device: int = 0,
                devices: Optional[List[int]] = None) -> Dict[str, object]:
    """`run_kernel` of `prog` split into `gpus` shards on devices
    first_device .. first_device+gpus-1 (or the explicit `devices` list, one
    entry per shard, which may repeat a device); returns {"out": value} like
    the single-device call."""
    from .api import compile_program, executable
    spec = shard_spec(prog)
    n = int(sigma[spec.nat])
    if gpus < 1 or n % gpus:
        raise ShardError(f"{spec.nat} = {n} does not split over {gpus} devices")
    devices = list(devices) if devices is not None else list(range(first_device, first_device + gpus))
    if len(devices) != gpus:
        raise ShardError(f"{len(devices)} devices given for {gpus} shards")
    ndev = RT.device_count()
    if max(devices) >= ndev or min(devices) < 0:
        raise ShardError(f"devices {devices} requested; {ndev} present")
    first_device = devices[0]
    sig_k = dict(sigma)
    sig_k[spec.nat] = n // gpus
    runs = []
    for k, dev in enumerate(devices):
        RT.init(dev)
        exe = executable(prog, launch, sig_k, float_mode=float_mode, device=dev)
        st = RT.Stream(dev)
        for pn, _t in prog.source.params:
            exe.upload(pn, _block(inputs[pn], k, gpus), st)
        exe.launch(st)
        runs.append((exe, st))
    leaves = []
    for exe, st in runs:
        st.sync()
        leaves.append(np.asarray(exe.download("out", st)))
    if spec.kind == "map":
        return {"out": LY.unflatten(prog.out_type, np.concatenate(leaves), sigma)}
    parts = np.concatenate([lv.reshape(-1) for lv in leaves])
    comb = compile_program("(nat k)\n(param ps (exp (array k num)))\n(reduceLocal (+) 0 ps)",
                           name=f"{name}_combine")
    exe = executable(comb, (1, 32), {"k": gpus}, float_mode=float_mode, device=first_device)
    st = RT.Stream(first_device)
    exe.upload("ps", parts, st)
    exe.launch(st)
    st.sync()
    total = np.asarray(exe.download("out", st))
    return {"out": LY.unflatten(prog.out_type, total, sigma)}

