"""C spellings of DPIA data types for the CUDA dialect."""
from __future__ import annotations

from typing import Dict, List, Tuple

from ..dtypes import Array, DataType, Idx, Num, Pair, Vector


class CudaError(Exception):
    """A phrase the CUDA backend cannot render (the reference's
    OpenCLError/CodegenError, SRC/opencl.py:30, SRC/codegen_c.py:38)."""


def mangle(d: DataType) -> str:
    if isinstance(d, Num):
        return "num"
    if isinstance(d, Idx):
        return "idx"
    if isinstance(d, Vector):
        return f"vec{d.width}"
    if isinstance(d, Array):
        c = d.size.const
        return f"arr{c if c is not None else 'n'}_{mangle(d.elem)}"
    if isinstance(d, Pair):
        return f"p_{mangle(d.fst)}_{mangle(d.snd)}"
    raise CudaError(f"cannot mangle {d}")


class TypeTable:
    """Maps data types to C types; collects struct definitions for pairs."""

    def __init__(self, scalar: str):
        self.scalar = scalar  # "float" | "long long"
        self.structs: Dict[str, str] = {}
        self._order: List[str] = []

    def c_elem(self, d: DataType) -> str:
        if isinstance(d, Num):
            return self.scalar
        if isinstance(d, Idx):
            return "long long"
        if isinstance(d, Vector):
            return f"dpia::vec<{self.scalar}, {d.width}>"
        if isinstance(d, Pair):
            return "struct " + self._struct(d)
        raise CudaError(f"no C element type for {d}")

    def member(self, d: DataType, name: str) -> str:
        dims = []
        while isinstance(d, Array):
            c = d.size.const
            if c is None:
                raise CudaError(f"array inside a pair needs a constant size, got {d}")
            dims.append(c)
            d = d.elem
        return self.c_elem(d) + " " + name + "".join(f"[{k}]" for k in dims)

    def _struct(self, d: Pair) -> str:
        name = "pair_" + mangle(d.fst) + "_" + mangle(d.snd)
        if name not in self.structs:
            fields = f"{self.member(d.fst, 'x1')}; {self.member(d.snd, 'x2')};"
            self.structs[name] = f"struct {name} {{ {fields} }};"
            self._order.append(name)
        return name

    def struct_text(self) -> str:
        return "\n".join(self.structs[n] for n in self._order)


def split_array(d: DataType) -> Tuple[List, DataType]:
    """(array sizes outermost first, innermost non-array element type)."""
    dims = []
    while isinstance(d, Array):
        dims.append(d.size)
        d = d.elem
    return dims, d
