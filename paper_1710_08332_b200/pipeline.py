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
                 out_bytes: int, float_mode: bool = True, device: int = 0, name: str = "pipe",
                 sigma_for_rows: Optional[Callable[[int], Dict[str, int]]] = None):
        """text_for_rows(r) -> program text for r rows (sigma_for_rows(r) ->
        its size parameters, if it has any); row_inputs / shared inputs:
        name -> total bytes; out_bytes: total bytes of the output."""
        if rows % chunks:
            raise ValueError(f"{rows} rows do not split into {chunks} chunks")
        self.rows, self.chunks, self.device = rows, chunks, device
        self.crows = rows // chunks
        prog = compile_program(text_for_rows(self.crows), name=name)
        sigma = sigma_for_rows(self.crows) if sigma_for_rows else {}
        self.exe = executable(prog, launch_for_rows(self.crows), sigma, float_mode=float_mode,
                              device=device)
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


def scal_pipeline(N: int, chunks: int = 8, device: int = 0, **geometry) -> RowPipeline:
    """scal (y = alpha * x, bench_programs.scal_program) over `chunks`
    contiguous blocks of x / y: the H2D of block i+1 and the D2H of block
    i-1 overlap block i's kernel, and PCIe carries both directions at once."""
    from .bench_programs import scal_config
    if N % (4 * chunks):
        raise ValueError(f"{N} elements do not split into {chunks} blocks of whole vec4s")
    cfg = lambda r: scal_config(N=r, **geometry)  # noqa: E731
    return RowPipeline(lambda r: cfg(r).text, lambda r: cfg(r).launch, N, chunks, {"xs": 4 * N},
                       {"alpha": 16}, 4 * N, device=device, name="scal", sigma_for_rows=lambda r: cfg(r).sigma)


def tile_schedule(rows: int, cols: int):
    """(copy-in order, tile order) of a TilePipeline: the row blocks ("A", i)
    and column panels ("B", j) interleaved in proportion, and the tiles (i, j)
    sorted by the copy after which both of their operands are in."""
    order, ia, ib = [], 0, 0
    while ia < rows or ib < cols:
        if ib >= cols or (ia < rows and ia * cols <= ib * rows):
            order.append(("A", ia))
            ia += 1
        else:
            order.append(("B", ib))
            ib += 1
    pos = {blk: k for k, blk in enumerate(order)}
    tiles = sorted(((i, j) for i in range(rows) for j in range(cols)),
                   key=lambda t: (max(pos[("A", t[0])], pos[("B", t[1])]), t))
    return order, tiles


class TilePipeline:
    """Two-dimensional tiling for programs whose output block (i, j) depends
    only on row block i of a "row" input and column panel j of a "column"
    input (mm: C[i, j] = A[i, :] . B[:, j]).  Output tile (i, j) can start as
    soon as A's row block i and B's column panel j have arrived, instead of
    after all of B (RowPipeline):

        copy-in  : A_0, B_0, A_1, B_1, ...  (B panels by pitched H2D copies)
        compute  : tile (i, j) once A_i and B_j are in, in arrival order,
                   round-robin over `compute_streams` streams so that several
                   small tile grids share the GPU
        copy-out : tile (i, j) by a pitched D2H copy into C, after its kernel

    Device layout: A as given (row blocks are contiguous), B as column panels
    of K x N/cols contiguous floats, C as contiguous tiles of M/rows x N/cols.
    Every element of C is computed by the same strategy from the same values
    as the unchunked program, so the result is bit-identical to it.
    """

    def __init__(self, text_for_tile: Callable[[int, int], str], launch_for_tile: Callable[[int, int], object],
                 M: int, N: int, K: int, rows: int, cols: int, row_input: str = "A", col_input: str = "B",
                 compute_streams: int = 4, elem_bytes: int = 4, float_mode: bool = True, device: int = 0,
                 name: str = "tile"):
        if M % rows or N % cols:
            raise ValueError(f"{M}x{N} does not split into {rows}x{cols} tiles")
        self.M, self.N, self.K, self.rows, self.cols = M, N, K, rows, cols
        self.tm, self.tn, self.eb, self.device = M // rows, N // cols, elem_bytes, device
        self.row_input, self.col_input = row_input, col_input
        prog = compile_program(text_for_tile(self.tm, self.tn), name=name)
        self.exe = executable(prog, launch_for_tile(self.tm, self.tn), {}, float_mode=float_mode,
                              device=device)
        if compute_streams > 1 and any(kind not in ("out", "in", "tmap") for k in self.exe.sig.kernels
                                       for kind, _ in k.args):
            raise ValueError("tile kernels with scratch buffers or grid counters cannot share "
                             "them across concurrent streams; use compute_streams=1")
        eb = elem_bytes
        self.a = RT.DeviceBuffer(M * K * eb, device)
        self.b = RT.DeviceBuffer(K * N * eb, device)
        self.c = RT.DeviceBuffer(M * N * eb, device)
        self.cin, self.cout = RT.Stream(device), RT.Stream(device)
        self.comp = [RT.Stream(device) for _ in range(max(1, compute_streams))]
        self.order, self.tiles = tile_schedule(rows, cols)

    def run(self, host: Dict[str, np.ndarray], out: np.ndarray, stream: Optional[RT.Stream] = None):
        """host row/column inputs (page-locked for overlap) -> out (page-locked,
        M x N row-major), synchronised.  `stream`, if given, is ordered before
        and after the whole pipeline."""
        dev, eb, tm, tn, K, N = self.device, self.eb, self.tm, self.tn, self.K, self.N
        streams = [self.cin, self.cout] + self.comp
        if stream is not None:
            ev = RT.Event(dev)
            ev.record(stream)
            for s in streams:
                ev.wait_on(s)
        A, B = host[self.row_input], host[self.col_input]
        arrived = {}
        for kind, k in self.order:
            if kind == "A":
                nb = tm * K * eb
                RT.lib().dpia_memcpy_htod(dev, self.a.ptr + k * nb, ctypes.c_void_p(A.ctypes.data + k * nb),
                                          nb, self.cin.handle)
            else:
                RT.lib().dpia_memcpy2d_htod(dev, self.b.ptr + k * K * tn * eb, tn * eb,
                                            ctypes.c_void_p(B.ctypes.data + k * tn * eb), N * eb,
                                            tn * eb, K, self.cin.handle)
            e = RT.Event(dev)
            e.record(self.cin)
            arrived[(kind, k)] = e
        done = []
        for t, (i, j) in enumerate(self.tiles):
            s = self.comp[t % len(self.comp)]
            arrived[("A", i)].wait_on(s)
            arrived[("B", j)].wait_on(s)
            cptr = self.c.ptr + (i * self.cols + j) * tm * tn * eb
            self.exe.launch_with(s, {self.row_input: self.a.ptr + i * tm * K * eb,
                                     self.col_input: self.b.ptr + j * K * tn * eb, "out": cptr})
            e = RT.Event(dev)
            e.record(s)
            done.append((e, i, j, cptr))
        for e, i, j, cptr in done:
            e.wait_on(self.cout)
            RT.lib().dpia_memcpy2d_dtoh(dev, ctypes.c_void_p(out.ctypes.data + (i * tm * N + j * tn) * eb),
                                        N * eb, cptr, tn * eb, tn * eb, tm, self.cout.handle)
        if stream is not None:
            for s in streams:
                e = RT.Event(dev)
                e.record(s)
                e.wait_on(stream)
            stream.sync()
        else:
            for s in streams:
                s.sync()
        return out


def mm_tile_pipeline(M: int, N: int, K: int, rows: int = 4, cols: int = 4, compute_streams: int = 4,
                     device: int = 0, float_mode: bool = True, **strategy) -> TilePipeline:
    """mm (bench_programs.mm_program strategy) over rows x cols output tiles;
    fp32 (float_mode) or int64 elements."""
    from .bench_programs import mm_config
    T = strategy.get("T", 128)
    if (M // rows) % T or (N // cols) % T:
        raise ValueError(f"tiles of {M // rows}x{N // cols} are not whole {T}x{T} work-group tiles")
    text = lambda m, n: mm_config(M=m, N=n, K=K, **strategy).text  # noqa: E731
    launch = lambda m, n: mm_config(M=m, N=n, K=K, **strategy).launch  # noqa: E731
    return TilePipeline(text, launch, M, N, K, rows, cols, compute_streams=compute_streams,
                        elem_bytes=4 if float_mode else 8, float_mode=float_mode, device=device, name="mm")
