"""Drop-in from the reference's own objects.

The reference's callers of its kernel backend hand over *their* objects:
`harness.py:399-407` passes the hoisted `dpia.phrases.Phrase` of a fuzz
program, `params` built from `dpia.types` data types and values with
`dpia.eval_fn.VectorVal` vectors to `simulate_kernel`; `cli.py:179-183` does
the same for `run --launch`; `emit_kernel` (opencl.py:265-314) returns its
source with a `KernelSignature`.  This module lets those call sites point at
the CUDA backend unchanged:

  to_json(x)                 structural JSON of a phrase, phrase/data type or
                             size expression -- the reference's or this
                             package's (duck-typed on class names and dataclass
                             fields, so the reference package need not be
                             importable where the JSON is read)
  phrase_from_json / type_from_json / nat_from_json
                             this package's objects from that JSON
  from_reference_phrase(p)   dpia.phrases.Phrase -> terms.Phrase
  from_reference_type(t)     dpia.types.{DataType,PhraseType} -> dtypes
  simulate_kernel(...)       the reference's signature and result, executed
                             on the GPU (launcher.run_kernel); vectors come
                             back as the caller's own vector class
  emit_kernel(...)           the reference's signature; returns the CUDA
                             source and a KernelSignature view

Node and field names are the reference's (`SRC/phrases.py:16-76`,
`SRC/types.py:19-136`, `SRC/nat.py:15-50`), which this package shares.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

from . import dtypes as DT
from . import terms as TM
from .sizes import Nat, nat

_PHRASES = {"Var", "Lam", "App", "TLam", "TApp", "PairP", "Proj", "Prim", "Lit"}
_DATA = {"Num", "Idx", "Array", "Pair", "Vector", "DataVar"}
_PTYPES = {"ExpT", "AccT", "CommT", "ProdT", "FnT", "DepFnT"}
_NATS = {"NatConst", "NatVar", "NatAdd", "NatMul"}
_SKIP = {"span"}


class AdapterError(ValueError):
    """An object that is not a phrase, type or size of the DPIA AST."""


# ------------------------------------------------------------- serialise

def to_json(x):
    """Structural JSON: {"k": class name, field: value, ...}; sizes as
    {"nat": [[monomial], coefficient], ...]}."""
    if x is None or isinstance(x, (bool, int, float, str)):
        return x
    if isinstance(x, Nat):
        return {"nat": [[list(m), c] for m, c in x.terms]}
    name = type(x).__name__
    if name in _NATS:
        return {"nat": [[list(m), c] for m, c in _ref_nat(x).terms]}
    if name in _PHRASES | _DATA | _PTYPES and dataclasses.is_dataclass(x):
        out = {"k": name}
        for f in dataclasses.fields(x):
            if f.name in _SKIP:
                continue
            out[f.name] = to_json(getattr(x, f.name))
        return out
    raise AdapterError(f"cannot serialise {type(x).__module__}.{name}")


def _ref_nat(e) -> Nat:
    """A reference NatExpr tree (NatConst / NatVar / NatAdd / NatMul) as a
    size polynomial of this package."""
    name = type(e).__name__
    if name == "NatConst":
        return nat(int(e.value))
    if name == "NatVar":
        return nat(e.name)
    if name == "NatAdd":
        return _ref_nat(e.left) + _ref_nat(e.right)
    if name == "NatMul":
        return _ref_nat(e.left) * _ref_nat(e.right)
    raise AdapterError(f"not a size expression: {name}")


# ----------------------------------------------------------- deserialise

def nat_from_json(j) -> Nat:
    if isinstance(j, int):
        return nat(j)
    if not (isinstance(j, dict) and "nat" in j):
        raise AdapterError(f"not a size: {j!r}")
    return Nat((tuple(m), int(c)) for m, c in j["nat"])


def type_from_json(j):
    """A data type or phrase type (or a size, for type arguments)."""
    if isinstance(j, dict) and "nat" in j:
        return nat_from_json(j)
    if not isinstance(j, dict) or "k" not in j:
        raise AdapterError(f"not a type: {j!r}")
    k = j["k"]
    if k == "Num":
        return DT.Num()
    if k == "Idx":
        return DT.Idx(nat_from_json(j["bound"]))
    if k == "Array":
        return DT.Array(nat_from_json(j["size"]), type_from_json(j["elem"]))
    if k == "Pair":
        return DT.Pair(type_from_json(j["fst"]), type_from_json(j["snd"]))
    if k == "Vector":
        return DT.Vector(int(j["width"]))
    if k == "DataVar":
        return DT.DataVar(j["name"])
    if k == "ExpT":
        return DT.ExpT(type_from_json(j["data"]))
    if k == "AccT":
        return DT.AccT(type_from_json(j["data"]))
    if k == "CommT":
        return DT.CommT()
    if k == "ProdT":
        return DT.ProdT(type_from_json(j["fst"]), type_from_json(j["snd"]))
    if k == "FnT":
        return DT.FnT(type_from_json(j["arg"]), type_from_json(j["ret"]), bool(j.get("passive", False)))
    if k == "DepFnT":
        return DT.DepFnT(j["binder"], j["kind"], type_from_json(j["body"]))
    raise AdapterError(f"unknown type node {k}")


def phrase_from_json(j) -> TM.Phrase:
    if not isinstance(j, dict) or "k" not in j:
        raise AdapterError(f"not a phrase: {j!r}")
    k = j["k"]
    if k == "Var":
        return TM.Var(j["name"])
    if k == "Lam":
        at = j.get("arg_type")
        return TM.Lam(j["binder"], phrase_from_json(j["body"]),
                      type_from_json(at) if at is not None else None)
    if k == "App":
        return TM.App(phrase_from_json(j["fn"]), phrase_from_json(j["arg"]))
    if k == "TLam":
        return TM.TLam(j["binder"], j["kind"], phrase_from_json(j["body"]))
    if k == "TApp":
        return TM.TApp(phrase_from_json(j["fn"]), type_from_json(j["arg"]))
    if k == "PairP":
        return TM.PairP(phrase_from_json(j["fst"]), phrase_from_json(j["snd"]))
    if k == "Proj":
        return TM.Proj(phrase_from_json(j["target"]), int(j["index"]))
    if k == "Prim":
        return TM.Prim(j["name"])
    if k == "Lit":
        return TM.Lit(j["value"], type_from_json(j["dtype"]))
    raise AdapterError(f"unknown phrase node {k}")


def from_reference_phrase(p) -> TM.Phrase:
    """dpia.phrases.Phrase (any stage: functional, Stage I, Stage II, hoisted)
    -> this package's phrase, node for node."""
    return phrase_from_json(to_json(p))


def from_reference_type(t):
    return type_from_json(to_json(t))


def from_reference_params(params) -> List[Tuple[str, DT.DataType, str]]:
    """simulate_kernel's params: [(name, dpia.types.DataType, mode)]."""
    return [(n, from_reference_type(d), mode) for n, d, mode in params]


# ------------------------------------------------ the reference's entry points

def _vector_class(values):
    """The caller's vector class (e.g. dpia.eval_fn.VectorVal), found in its
    input values, so results compare equal to the caller's own values."""
    stack = list(values)
    while stack:
        v = stack.pop()
        if isinstance(v, list):
            stack.extend(v[:1])        # arrays are homogeneous: one element says it
        elif isinstance(v, tuple):
            stack.extend(v)            # pairs are not
        elif hasattr(v, "items") and not isinstance(v, dict):
            return type(v)
    return None


def _rebuild_vectors(v, cls):
    from .layout import VectorVal
    if isinstance(v, VectorVal):
        return cls(tuple(v.items))
    if isinstance(v, list):
        return [_rebuild_vectors(x, cls) for x in v]
    if isinstance(v, tuple):
        return tuple(_rebuild_vectors(x, cls) for x in v)
    return v


def simulate_kernel(p, params, inputs: Dict[str, object], launch, sigma: Optional[Dict[str, int]] = None,
                    float_mode: bool = False, device: int = 0) -> Dict[str, object]:
    """`dpia.opencl.simulate_kernel` (SRC/opencl.py:397-402) with the same
    arguments -- the reference's hoisted Phrase, its (name, DataType, mode)
    params, its values -- executed on the GPU.  Returns {name: value} for
    every out/var parameter, vectors as the caller's own vector class."""
    from .launcher import run_kernel
    ours = p if isinstance(p, TM.Phrase) else from_reference_phrase(p)
    prm = [(n, d if isinstance(d, DT.DataType) else from_reference_type(d), mode) for n, d, mode in params]
    out = run_kernel(ours, prm, inputs, launch, sigma or {}, float_mode, device=device)
    cls = _vector_class(inputs.values())
    return {k: _rebuild_vectors(v, cls) for k, v in out.items()} if cls else out


@dataclass
class KernelSignature:
    """The reference's KernelSignature shape (SRC/opencl.py:250-262) over a
    CudaSignature: outputs, inputs, hoisted buffers, size parameters."""
    outputs: List[Tuple[str, object]]
    inputs: List[Tuple[str, object]]
    buffers: list
    sizes: List[str]
    cuda: object = None

    def params(self, scalar: str) -> List[str]:
        out = [f"{scalar} *{n}" for n, _ in self.outputs]
        out += [f"const {scalar} *__restrict__ {n}" for n, _ in self.inputs]
        out += [f"{scalar} *{b.name}" for b in self.buffers]
        out += [f"long long {n}" for n in self.sizes]
        return out


def emit_kernel(p, outputs, inputs, float_mode: bool = True, name: str = "KERNEL",
                init_new: bool = False, simplify: bool = True):
    """`dpia.opencl.emit_kernel` (SRC/opencl.py:265-271) with the same
    arguments (reference objects accepted): CUDA C for sm_100a and a
    KernelSignature whose lists hold the caller's own type objects."""
    from .cuda.emit import emit_cuda
    from .cuda.hierarchy import HoistedBuffer
    conv = (lambda d: d if isinstance(d, DT.DataType) else from_reference_type(d))  # noqa: E731
    ours = p if isinstance(p, TM.Phrase) else from_reference_phrase(p)
    src, sig = emit_cuda(ours, [(n, conv(d)) for n, d in outputs], [(n, conv(d)) for n, d in inputs],
                         float_mode=float_mode, name=name, init_new=init_new, simplify=simplify)
    bufs = [HoistedBuffer(n, d, sig.spaces.get(n, "global")) for n, d in sig.buffers]
    return src, KernelSignature(list(outputs), list(inputs), bufs, list(sig.sizes), sig)
