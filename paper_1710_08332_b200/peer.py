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


def mailbox_bytes(world: int, n_scalars: int) -> int:
    return (2 * world * n_scalars + 1) * SLOT_BYTES


def torch_allgather(handle: bytes) -> List[bytes]:
    """IPC-handle exchange over the already initialised torch.distributed
    process group (host plumbing)."""
    import torch.distributed as dist
    out: List[Optional[bytes]] = [None] * dist.get_world_size()
    dist.all_gather_object(out, handle)
    return [bytes(h) for h in out]
