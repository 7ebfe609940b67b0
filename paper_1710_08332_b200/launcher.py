"""Execution of emitted kernels: the CUDA replacement of the reference's
work-item simulator.

`run_kernel` has the signature and result of `simulate_kernel`
(SRC/opencl.py:397-402): params are (name, data type, "in"|"out"|"var"),
inputs map names to values, launch is (G, L) -- or ((Gx, Gy), (Lx, Ly)) for
the two-dimensional hierarchy -- and the result maps every out/var parameter
to its final value.  Instead of interpreting the phrase it emits CUDA C
(`cuda.emit`), compiles it with NVRTC for sm_100a and launches it through
libdpia_rt.so.  `Executable` keeps the compiled program and device buffers
for repeated launches (benchmarks, CUDA-event timing).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import layout as LY
from . import runtime as RT
from .cuda.emit import EPOCH_BASE, CudaError, CudaSignature, emit_cuda, normalize_launch
from .cuda.hierarchy import check_work_item_races
from .dtypes import DataType
from .terms import Phrase


@dataclass
class Executable:
    src: str
    sig: CudaSignature
    device: int
    float_mode: bool
    sigma: Dict[str, int]
    geometry: tuple = None          # ((gx, gy), (lx, ly)) used at launch
    module: RT.Module = None
    buffers: Dict[str, RT.DeviceBuffer] = field(default_factory=dict)
    counters: Dict[str, RT.DeviceBuffer] = field(default_factory=dict)
    peer: object = None             # peer.PeerGroup of the fused cross-GPU combine
    _args: List = field(default_factory=list)
    # launch epoch of slot-pipelined streaming tails (cuda/emit.py STREAM_PIPE):
    # bumped before every launch, first launch EPOCH_BASE (the kernels' release
    # words are initialised for it, KernelInfo.counter_init)
    _epoch: object = field(default_factory=lambda: RT.C.c_uint(EPOCH_BASE - 1))
    _tmap_cache: Dict = field(default_factory=dict)

    @property
    def launch_geom(self):
        return self.sig.launch

    def compile(self):
        img = RT.get_cubin(self.src)
        self.module = RT.Module(img, self.device)
        for k in self.sig.kernels:
            if k.smem > 48 * 1024:
                RT.lib().dpia_kernel_set_smem(self.module.function(k.name), k.smem)
        return self

    # ----------------------------------------------------------- buffers
    def allocate(self):
        fm, sg = self.float_mode, self.sigma
        for n, d in self.sig.outputs + self.sig.inputs:
            if n not in self.buffers:
                self.buffers[n] = RT.DeviceBuffer(LY.nbytes(d, sg, fm), self.device)
        for n, d in self.sig.buffers:
            if n not in self.buffers:
                b = RT.DeviceBuffer(LY.nbytes(d, sg, fm), self.device)
                b.zero()
                self.buffers[n] = b
        for k in self.sig.kernels:
            if k.fused_tail and k.name not in self.counters:
                c = RT.DeviceBuffer(4 * k.counter_words, self.device)
                c.zero()
                if k.counter_init:
                    init = np.zeros(k.counter_words, np.uint32)
                    for word, value in k.counter_init:
                        init[word] = value
                    c.upload(init)
                    RT.lib().dpia_device_sync(self.device)   # before any launch stream sees it
                self.counters[k.name] = c
        self._args = []
        for k in self.sig.kernels:
            vals = []
            for kind, n in k.args:
                if kind in ("out", "in", "scratch"):
                    vals.append(RT.C.c_uint64(self.buffers[n].ptr))
                elif kind == "size":
                    vals.append(RT.C.c_longlong(int(self.sigma[n])))
                elif kind == "peer_boxes":
                    vals.append(RT.C.c_uint64(self.peer.boxes.ptr))
                elif kind == "peer_rank":
                    vals.append(RT.C.c_int(self.peer.rank))
                elif kind == "peer_world":
                    vals.append(RT.C.c_int(self.peer.world))
                elif kind == "peer_epoch":
                    vals.append(self.peer.epoch)       # shared; bumped by every launch
                elif kind == "tmap":
                    vals.append(self._tensor_map(n, self.buffers[self.sig.tmaps[n][0]].ptr))
                elif kind == "epoch":
                    vals.append(self._epoch)           # shared; bumped by every launch
                else:
                    vals.append(RT.C.c_uint64(self.counters[k.name].ptr))
            self._args.append(vals)
        return self

    def _tensor_map(self, name: str, base: int):
        """The TMA descriptor of tensor-map parameter `name` over the input
        at device address `base` (cuda/emit.py KernelEmitter._tma_plan),
        encoded once per address (launch_with re-points inputs every step)."""
        key = (name, base)
        m = self._tmap_cache.get(key)
        if m is None:
            _x, eb, rows, cols, pitch, box_rows, box_cols, swizzle = self.sig.tmaps[name]
            m = RT.tensor_map_2d(eb, base, rows, cols, pitch, box_rows, box_cols, swizzle)
            if len(self._tmap_cache) > 256:
                self._tmap_cache.clear()
            self._tmap_cache[key] = m
        return m

    def bind(self, name: str, buf: RT.DeviceBuffer):
        """Use an externally owned device buffer for parameter `name`."""
        self.buffers[name] = buf
        if self._args:
            self.allocate()

    def upload(self, name: str, value, stream=None):
        d = dict(self.sig.outputs + self.sig.inputs)[name]
        self.buffers[name].upload(LY.to_bytes(value, d, self.sigma, self.float_mode), stream)

    def download(self, name: str, stream=None) -> np.ndarray:
        d = dict(self.sig.outputs + self.sig.inputs)[name]
        raw = np.empty(LY.nbytes(d, self.sigma, self.float_mode), np.uint8)
        self.buffers[name].download(raw, stream)
        return LY.from_bytes(raw, d, self.sigma, self.float_mode)

    # ------------------------------------------------------------ launch
    def launch(self, stream: Optional[RT.Stream] = None, chain: bool = False):
        """Launch the program's kernels on `stream`.  chain=True: the first
        kernel is launched with programmatic dependent launch behind the
        previous kernel on the stream -- it starts streaming its inputs while
        that grid drains and waits for it only before touching any other
        global memory (cuda/emit.py ProgramEmitter._chain_waits).  The caller
        asserts that the previous kernel writes none of this program's
        inputs (true for back-to-back launches of programs over their own
        inputs, e.g. repeated steps); results are identical either way."""
        if self.peer is not None:
            self.peer.next_epoch()
        self._epoch.value += 1
        (g, l) = self.sig.launch or self.geometry
        for i, (k, vals) in enumerate(zip(self.sig.kernels, self._args)):
            grid = (g[0] + k.extra_blocks, g[1]) if k.grid == "launch" else (1, 1)
            fn = self.module.function(k.name)
            # later phases: programmatic dependent launch (their first
            # statement is griddepcontrol.wait), which hides their launch
            # latency behind the previous phase
            RT.launch(fn, self.device, grid, l, k.smem, vals, stream, pdl=i > 0 or chain)

    def launch_with(self, stream: Optional[RT.Stream], ptrs: Dict[str, int], chain: bool = False):
        """Launch with some parameters re-pointed (device addresses), e.g. at
        windows of larger buffers -- the row chunks of pipeline.RowPipeline.
        Windows must be 16-byte aligned -- the emitted kernels read their
        buffers with whole-vector loads (asVector, vectorised folds) -- and
        32-byte aligned where a fold's register queue loads 32 bytes at a
        time (`sig.align`)."""
        need = {n: max(16, self.sig.align.get(n, 16)) for n in ptrs}
        bad = [n for n, q in ptrs.items() if q % need[n]]
        if bad:
            raise ValueError(f"launch_with: windows {bad} are not aligned to "
                             f"{[need[n] for n in bad]} bytes")
        if self.peer is not None:
            self.peer.next_epoch()
        self._epoch.value += 1
        (g, l) = self.sig.launch or self.geometry
        for i, (k, vals) in enumerate(zip(self.sig.kernels, self._args)):
            vals = [RT.C.c_uint64(ptrs[n]) if kind in ("out", "in") and n in ptrs
                    else self._tensor_map(n, ptrs[self.sig.tmaps[n][0]])
                    if kind == "tmap" and self.sig.tmaps[n][0] in ptrs else v
                    for (kind, n), v in zip(k.args, vals)]
            grid = (g[0] + k.extra_blocks, g[1]) if k.grid == "launch" else (1, 1)
            RT.launch(self.module.function(k.name), self.device, grid, l, k.smem, vals, stream,
                      pdl=i > 0 or chain)

    def run(self, inputs: Dict[str, object], stream: Optional[RT.Stream] = None,
            out: Optional[Dict[str, np.ndarray]] = None) -> Dict[str, np.ndarray]:
        """One end-to-end execution from host buffers: copy every input to
        the device, launch the program, copy every out/var parameter back,
        synchronise.  Results are flat scalar leaves (numpy).  Host arrays in
        page-locked memory (`runtime.PinnedBuffer.array`) make both copies
        direct DMA; `out` may supply such arrays for the results."""
        for n, _d in self.sig.inputs:
            self.upload(n, inputs[n], stream)
        self.launch(stream)
        res = {}
        for n, d in self.sig.outputs:
            size, _, dense = LY.shape_of(d, self.sigma, 4 if self.float_mode else 8)
            dst = (out or {}).get(n)
            if dense and dst is not None:
                self.buffers[n].download(dst.reshape(-1).view(np.uint8)[:size], stream)
                res[n] = dst
            else:
                res[n] = self.download(n, stream)
        if stream is not None:
            stream.sync()
        else:
            RT.lib().dpia_device_sync(self.device)
        return res

    def kernel_names(self) -> List[str]:
        return [k.name for k in self.sig.kernels]


def _split_params(params):
    outs = [(n, d) for n, d, mode in params if mode in ("out", "var")]
    ins = [(n, d) for n, d, mode in params if mode == "in"]
    return outs, ins


def build(p: Phrase, params: List[Tuple[str, DataType, str]], launch, sigma=None,
          float_mode: bool = False, device: int = 0, name: str = "KERNEL",
          specialize: bool = True, peer=None, tma_tiles: Optional[bool] = None) -> Executable:
    """Emit + compile + allocate (no data movement).  specialize=False keeps
    sizes as kernel arguments and the geometry runtime-only (the source the
    CLI's `compile` writes without --launch).  peer: a peer.PeerGroup -- the
    program's result is summed over the group's ranks inside the kernel.
    tma_tiles: TMA tensor staging of 2-D box k-tiles (cuda/emit.py)."""
    sigma = dict(sigma or {})
    outs, ins = _split_params(params)
    geom = normalize_launch(launch)
    check_work_item_races(p)   # the reference simulator's WorkItemRace (SRC/opencl.py:465-470)
    src, sig = emit_cuda(p, outs, ins, float_mode=float_mode, name=name,
                         sigma=sigma if specialize else None, launch=geom if specialize else None,
                         peer=peer is not None, tma_tiles=tma_tiles)
    if peer is not None:
        # dpia::peer_sum writes one mailbox slot per output scalar into every
        # peer: the group's mailboxes must have been sized for exactly that
        nsc = LY.nbytes(outs[0][1], sigma, float_mode) // (4 if float_mode else 8)
        if nsc != peer.n:
            raise CudaError(f"the program's result has {nsc} scalars; the peer group's mailboxes "
                            f"hold {peer.n}")
    exe = Executable(src, sig, device, float_mode, sigma, geometry=geom, peer=peer)
    return exe.compile().allocate()


def run_kernel(p: Phrase, params: List[Tuple[str, DataType, str]], inputs: Dict[str, object],
               launch, sigma: Optional[Dict[str, int]] = None, float_mode: bool = False,
               device: int = 0, name: str = "KERNEL", flat: bool = False,
               specialize: bool = True) -> Dict[str, object]:
    """Drop-in for `simulate_kernel(p, params, inputs, launch, sigma,
    float_mode)` (SRC/opencl.py:397): same arguments, same result mapping,
    executed on the GPU.  flat=True returns numpy arrays of scalar leaves."""
    normalize_launch(launch)  # ValueError for non-positive launches, like the reference
    exe = build(p, params, launch, sigma, float_mode, device, name, specialize)
    stream = RT.Stream(device)
    for n, d, mode in params:
        if mode == "in":
            exe.upload(n, inputs[n], stream)
        elif mode == "var" and n in inputs:
            exe.upload(n, inputs[n], stream)
        else:
            exe.buffers[n].zero(stream)
    exe.launch(stream)
    stream.sync()
    out = {}
    for n, d, mode in params:
        if mode in ("out", "var"):
            leaves = exe.download(n, stream)
            out[n] = leaves if flat else LY.unflatten(d, leaves, exe.sigma)
    stream.sync()
    return out
