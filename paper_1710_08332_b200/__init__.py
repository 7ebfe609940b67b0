"""B200-native CUDA backend for DPIA strategy-preserving compilation
(arXiv 1710.08332).  Public surface mirrors the reference package `dpia`:

  parse / parse_phrase            (dpia.parser)
  translate_program               (dpia.translate, Stage I)
  stage2                          (dpia.lower, Stage II)
  emit_cuda                       (replaces dpia.opencl.emit_kernel)
  run_kernel                      (replaces dpia.opencl.simulate_kernel)
"""
from .reader import ElabError, ParseError, SourceProgram, parse, parse_phrase  # noqa: F401
from .stage1 import translate_program  # noqa: F401
from .stage2 import stage2  # noqa: F401
from .cuda.ctypes_map import CudaError  # noqa: F401
from .cuda.emit import CudaSignature, emit_cuda  # noqa: F401
from .launcher import Executable, run_kernel  # noqa: F401
from .cuda.hierarchy import (HoistedBuffer, WorkItemRace, check_work_item_races, cuda_legal,  # noqa: F401
                             hoist_allocations, lint_hierarchy)
from .api import Program, compile_program, executable, run_program_cuda  # noqa: F401
from .checker import DpiaTypeError, type_check  # noqa: F401
from .pretty import pretty_print  # noqa: F401
from .pipeline import RowPipeline, TilePipeline, mm_pipeline, mm_tile_pipeline, scal_pipeline  # noqa: F401
from .peer import PeerGroup  # noqa: F401

__all__ = ["parse", "parse_phrase", "translate_program", "stage2", "emit_cuda", "run_kernel",
           "compile_program", "run_program_cuda", "executable", "CudaError", "ParseError",
           "ElabError", "SourceProgram", "Program", "Executable", "CudaSignature",
           "hoist_allocations", "lint_hierarchy", "cuda_legal", "HoistedBuffer",
           "WorkItemRace", "check_work_item_races", "RowPipeline", "mm_pipeline", "TilePipeline",
           "mm_tile_pipeline", "scal_pipeline", "PeerGroup",
           "type_check", "DpiaTypeError", "pretty_print"]
