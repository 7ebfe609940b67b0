"""Fused cross-GPU combine for the sharded reductions.

The reference has no multi-device path; the scale-out config (BASELINE.json
config 5) shards the outermost work-group loop of dot / asum over the GPUs of
one node and must combine the per-rank partial sums.  Instead of a separate
ncclAllReduce of 4 bytes after the kernel, the emitted kernel itself does the
exchange (`emit_cuda(..., peer=True)`): when the last work-group of a rank has
produced the rank's result it stores it into a mailbox slot on *every* rank
over NVLink (CUDA IPC mappings, peer access) and sums all ranks' slots in rank
order (`dpia::peer_sum` in csrc/dpia_device.cuh).  Every rank therefore ends
with the same, deterministically ordered total, one kernel per step, no
collective launch.

Mailbox of one rank: 2 parities x world x n slots of 16 bytes (a 4-byte value
and its epoch packed in the first 8 bytes; an 8-byte value at offset 0 with
its epoch at offset 8) plus a 16-byte error word.  Warp 0 serves the peers in
parallel, one lane per peer.  Launch e writes parity e & 1 with epoch e (epochs
start at 1; the mailbox is zeroed), so ranks may drift by one launch without
overwriting a slot that a slower rank still has to read.

One process per GPU (torchrun); the 64-byte IPC handles are exchanged by the
caller's `allgather(bytes) -> [bytes per rank]` (torch.distributed), which is
host plumbing only.
"""
from __future__ import annotations

import ctypes
from typing import Callable, List, Optional

import numpy as np

from . import runtime as RT

SLOT_BYTES = 16


class PeerError(RuntimeError):
    pass


class PeerGroup:
    def __init__(self, device: int, rank: int, world: int, n_scalars: int = 1,
                 allgather: Optional[Callable[[bytes], List[bytes]]] = None):
        if not (0 <= rank < world):
            raise ValueError(f"rank {rank} not in a world of {world}")
        if world > 1 and allgather is None:
            raise ValueError("a multi-rank peer group needs an allgather for the IPC handles")
        RT.init(device)
        self.device, self.rank, self.world, self.n = device, rank, world, n_scalars
        self.nbytes = mailbox_bytes(world, n_scalars)
        handle = ctypes.create_string_buffer(64)
        p = ctypes.c_uint64()
        local_err = None
        try:
            RT.lib().dpia_ipc_alloc(device, self.nbytes, ctypes.byref(p), handle)
            mine = bytes(handle.raw)
        except RT.DpiaRuntimeError as e:
            local_err, mine = e, b""          # still take part in the exchange
        self.local = p.value
        handles = allgather(mine) if world > 1 else [mine]
        if len(handles) != world:
            raise ValueError(f"allgather returned {len(handles)} handles for {world} ranks")
        if local_err is not None:
            raise PeerError(f"rank {rank}: cannot allocate an IPC mailbox: {local_err}")
        if any(len(h) != 64 for h in handles):
            raise PeerError(f"rank {rank}: a peer could not allocate its mailbox")
        self.opened: List[int] = []
        ptrs = []
        for r, h in enumerate(handles):
            if r == rank:
                ptrs.append(self.local)
                continue
            q = ctypes.c_uint64()
            RT.lib().dpia_ipc_open(device, ctypes.create_string_buffer(h, 64), ctypes.byref(q))
            self.opened.append(q.value)
            ptrs.append(q.value)
        self.boxes = RT.DeviceBuffer(8 * world, device)
        self.boxes.upload(np.asarray(ptrs, np.uint64))
        self.epoch = ctypes.c_uint(0)

    def next_epoch(self) -> int:
        self.epoch.value += 1
        return self.epoch.value

    def check(self):
        """Raise if a peer_sum on this rank timed out waiting for a peer."""
        err = np.zeros(1, np.uint32)
        RT.lib().dpia_device_sync(self.device)   # after every launch queued on any stream
        RT.lib().dpia_memcpy_dtoh(self.device, err.ctypes.data_as(ctypes.c_void_p),
                                  self.local + self.nbytes - SLOT_BYTES, 4, None)
        if err[0]:
            raise PeerError(f"rank {self.rank}: a peer never published its result "
                            f"(epoch {self.epoch.value})")

    def close(self):
        for q in self.opened:
            RT.lib().dpia_ipc_close(self.device, q)
        self.opened = []
        if self.local:
            RT.lib().dpia_free(self.device, self.local)
            self.local = 0
        self.boxes.free()


def local_twin(exe, prog):
    """The program of `exe` built without the fused cross-GPU combine, with
    the same geometry and sizes, reading `exe`'s input buffers: one launch
    leaves this rank's own partial in its `out`."""
    from .api import executable
    twin = executable(prog, exe.geometry, exe.sigma, float_mode=exe.float_mode, device=exe.device)
    for n, _d in exe.sig.inputs:
        twin.bind(n, exe.buffers[n])
    return twin


def rank_order_sum(parts: List[np.ndarray]) -> np.ndarray:
    """parts[0] + parts[1] + ... in rank order, in the partials' own dtype --
    the association dpia::peer_sum uses, so the kernel's total must equal it
    bit for bit."""
    acc = parts[0].copy()
    for p in parts[1:]:
        acc = (acc + p).astype(parts[0].dtype)
    return acc


def cross_check(exe, twin, stream, allgather: Callable[[bytes], List[bytes]]) -> dict:
    """Check the fused combine against the partials it combines.

    Every rank launches `twin` (no combine) to get its own partial, the
    partials are gathered over the host process group and summed in rank
    order; then `exe` (the fused combine) runs once and its total must equal
    that sum bit for bit on every rank.  Returns the evidence; raises
    PeerError if a peer never published (the kernel's error word)."""
    twin.launch(stream)
    stream.sync()
    part = twin.download("out", stream)
    stream.sync()
    parts = [np.frombuffer(b, part.dtype).copy() for b in allgather(part.tobytes())]
    want = rank_order_sum(parts)
    exe.launch(stream)
    stream.sync()
    exe.peer.check()
    got = exe.download("out", stream)
    stream.sync()
    exact = bool(np.array_equal(got.view(np.uint8), want.view(np.uint8)))
    return {"peer_total": [float(v) for v in got], "rank_order_sum": [float(v) for v in want],
            "partials": [float(p[0]) for p in parts], "bit_exact": exact,
            "abs_sum": float(sum(np.abs(p.astype(np.float64)).sum() for p in parts))}


def mailbox_bytes(world: int, n_scalars: int) -> int:
    return (2 * world * n_scalars + 1) * SLOT_BYTES


def torch_allgather(handle: bytes) -> List[bytes]:
    """IPC-handle exchange over the already initialised torch.distributed
    process group (host plumbing)."""
    import torch.distributed as dist
    out: List[Optional[bytes]] = [None] * dist.get_world_size()
    dist.all_gather_object(out, handle)
    return [bytes(h) for h in out]
