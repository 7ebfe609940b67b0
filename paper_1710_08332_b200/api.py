"""Program-level convenience API: parse -> Stage I -> Stage II -> CUDA.

The reference drives this pipeline from its CLI (`SRC/cli.py:122-134` for
compilation, `:170-183` for `run --launch`): Stage I with
default_space="global", Stage II with accum_space="private", then the kernel
backend.  `compile_program` / `run_program_cuda` do the same with the CUDA
backend in place of the OpenCL emitter and simulator.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

from .dtypes import DataType
from .launcher import Executable, build, run_kernel
from .reader import SourceProgram, parse
from .stage1 import translate_program
from .stage2 import stage2
from .terms import Phrase


@dataclass
class Program:
    source: SourceProgram
    stage1: Phrase
    imperative: Phrase
    name: str = "KERNEL"

    @property
    def out_type(self) -> DataType:
        return self.source.body_type.data

    @property
    def params(self) -> List[Tuple[str, DataType, str]]:
        return [("out", self.out_type, "out")] + [(n, t.data, "in") for n, t in self.source.params]


def compile_program(text: str, name: str = "KERNEL", check: bool = True) -> Program:
    """parse -> SCIR type check (rejects racy parfor bodies, as the reference
    CLI does, SRC/cli.py:48-53) -> Stage I -> Stage II."""
    sp = parse(text)
    if check:
        from .checker import type_check
        type_check(sp.body, delta=sp.delta, pi=sp.pi, gamma=sp.gamma)
    s1 = translate_program(sp.body, sp.body_type.data, out="out", default_space="global")
    return Program(sp, s1, stage2(s1, accum_space="private"), name)


def executable(prog: Program, launch, sigma: Optional[Dict[str, int]] = None,
               float_mode: bool = True, device: int = 0, peer=None,
               tma_tiles: Optional[bool] = None) -> Executable:
    return build(prog.imperative, prog.params, launch, sigma, float_mode, device, prog.name,
                 peer=peer, tma_tiles=tma_tiles)


def run_program_cuda(prog: Program, inputs: Dict[str, object], sigma=None, launch=(148, 256),
                     float_mode: bool = True, device: int = 0, flat: bool = False, gpus: int = 1):
    """Run a compiled program on the GPU and return its output value.
    gpus > 1 splits the outermost map over devices device .. device+gpus-1
    (shard.run_sharded; chunk-local maps and (+)/0 reductions of them)."""
    if gpus > 1:
        from .shard import run_sharded
        val = run_sharded(prog, inputs, launch, dict(sigma or {}), float_mode, gpus, prog.name,
                          first_device=device)["out"]
        if flat:
            from . import layout as LY
            import numpy as np
            return np.asarray(LY.flatten(val))
        return val
    out = run_kernel(prog.imperative, prog.params, inputs, launch, sigma, float_mode, device,
                     prog.name, flat=flat)
    return out["out"]
