"""Row-chunked execution with host<->device copies overlapped with compute.

For a program whose outermost parallel loop runs over row blocks of its
output and of one "row" input (mm: C[i-block] = A[i-block] . B), the rows
split into chunks that are independent -- the same outer-loop partitioning
the multi-GPU scale-out uses, here in time instead of across
devices.  One Executable specialised to a chunk's rows is launched per chunk
on windows of the full device buffers, with three streams:

    copy-in  : shared inputs, then row input chunk 0, 1, ...   (H2D)
    compute  : chunk i after its rows arrived                   (kernels)
    copy-out : output chunk i after its kernel                 (D2H)

so chunk i's kernel overlaps the H2D of chunk i+1 and the D2H of chunk i-1
(PCIe is full duplex).  The result is bit-identical to the unchunked run:
every output element is computed by the same strategy from the same values.
"""
from __future__ import annotations

import ctypes
from typing import Callable, Dict, List, Optional

import numpy as np

from . import runtime as RT
from .api import compile_program, executable


class RowPipeline:
    def __init__(self, text_for_rows: Callable[[int], str], launch_for_rows: Callable[[int], object],
                 rows: int, chunks: int, row_inputs: Dict[str, int], shared_inputs: Dict[str, int],
                 out_bytes: int, float_mode: bool = True, device: int = 0, name: str = "pipe"):
        """text_for_rows(r) -> program text for r rows; row_inputs / shared
        inputs: name -> total bytes; out_bytes: total bytes of the output."""
        if rows % chunks:
            raise ValueError(f"{rows} rows do not split into {chunks} chunks")
        self.rows, self.chunks, self.device = rows, chunks, device
        self.crows = rows // chunks
        prog = compile_program(text_for_rows(self.crows), name=name)
        self.exe = executable(prog, launch_for_rows(self.crows), {}, float_mode=float_mode, device=device)
        self.row_inputs, self.shared_inputs, self.out_bytes = dict(row_inputs), dict(shared_inputs), out_bytes
        self.full = {n: RT.DeviceBuffer(b, device) for n, b in {**row_inputs, "out": out_bytes}.items()}
        for n, b in shared_inputs.items():
            self.full[n] = self.exe.buffers[n]
        self.streams = [RT.Stream(device) for _ in range(3)]

    def run(self, host: Dict[str, np.ndarray], out: np.ndarray, stream: Optional[RT.Stream] = None):
        """host arrays (page-locked for overlap) -> out (page-locked), synchronised.
        `stream`, if given, is ordered before and after the whole pipeline."""
        cin, comp, cout = self.streams
        dev = self.device
        if stream is not None:
            ev = RT.Event(dev)
            ev.record(stream)
            for s in self.streams:
                ev.wait_on(s)

        def h2d(dst, src: np.ndarray, off, nbytes, s):
            RT.lib().dpia_memcpy_htod(dev, dst + off, ctypes.c_void_p(src.ctypes.data + off), nbytes,
                                      s.handle)

        for n, b in self.shared_inputs.items():
            h2d(self.full[n].ptr, host[n], 0, b, cin)
        ev_in: List[RT.Event] = []
        ev_k: List[RT.Event] = []
        for i in range(self.chunks):
            for n, b in self.row_inputs.items():
                cb = b // self.chunks
                h2d(self.full[n].ptr, host[n], i * cb, cb, cin)
            e = RT.Event(dev)
            e.record(cin)
            ev_in.append(e)
        ob = self.out_bytes // self.chunks
        for i in range(self.chunks):
            ev_in[i].wait_on(comp)
            ptrs = {n: self.full[n].ptr + i * (b // self.chunks) for n, b in self.row_inputs.items()}
            ptrs["out"] = self.full["out"].ptr + i * ob
            self.exe.launch_with(comp, ptrs)
            e = RT.Event(dev)
            e.record(comp)
            ev_k.append(e)
        for i in range(self.chunks):
            ev_k[i].wait_on(cout)
            RT.lib().dpia_memcpy_dtoh(dev, ctypes.c_void_p(out.ctypes.data + i * ob),
                                      self.full["out"].ptr + i * ob, ob, cout.handle)
        if stream is not None:
            done = RT.Event(dev)
            done.record(cout)
            for s in (cin, comp):
                e = RT.Event(dev)
                e.record(s)
                e.wait_on(stream)
            done.wait_on(stream)
            stream.sync()
        else:
            for s in self.streams:
                s.sync()
        return out


def mm_pipeline(M: int, N: int, K: int, chunks: int = 4, device: int = 0, **strategy) -> RowPipeline:
    """mm (bench_programs.mm_program strategy) over `chunks` row blocks of A / C."""
    from .bench_programs import mm_config
    T = strategy.get("T", 128)
    if (M // chunks) % T:
        raise ValueError(f"chunks of {M // chunks} rows are not whole {T}-row tiles")
    text = lambda r: mm_config(M=r, N=N, K=K, **strategy).text  # noqa: E731
    launch = lambda r: mm_config(M=r, N=N, K=K, **strategy).launch  # noqa: E731
    return RowPipeline(text, launch, M, chunks, {"A": 4 * M * K}, {"B": 4 * K * N}, 4 * M * N,
                       device=device, name="mm")
