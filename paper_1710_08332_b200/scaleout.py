"""Multi-GPU driver for the sharded reductions (BASELINE.json config 5,
SURVEY.md 8e).

The outermost parallel loop of the dot / asum strategies (mapWorkgroup over
n chunks) has independent iterations -- the SCIR typing guarantees disjoint
writes (SRC/checker.py:219-249) -- so the chunk range [0, n) is split into
contiguous blocks, one per rank.  Every rank runs the *same* emitted program
specialised to n/world chunks on its shard (inputs generated on device by a
counter hash at the shard's global element offset, so no host data moves),
leaving one partial sum; the partials are combined with one NCCL all-reduce
of 4 bytes.  One process per GPU (torchrun); this module holds the
host-side plan and the per-rank execution.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

from . import runtime as RT
from .api import compile_program, executable
from .bench_programs import asum_program, dot_program


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    chunks: int          # chunks owned by this rank
    chunk_elems: int     # elements per chunk
    first_chunk: int

    @property
    def elem_offset(self) -> int:
        return self.first_chunk * self.chunk_elems

    @property
    def elems(self) -> int:
        return self.chunks * self.chunk_elems


def shard_plan(total_elems: int, chunk_elems: int, world: int, rank: int) -> Shard:
    """Contiguous block of the outer chunk range for `rank`."""
    if total_elems % chunk_elems:
        raise ValueError(f"{total_elems} elements are not a whole number of {chunk_elems}-chunks")
    n = total_elems // chunk_elems
    if n % world:
        raise ValueError(f"{n} chunks do not split evenly over {world} ranks")
    per = n // world
    return Shard(rank, world, per, chunk_elems, rank * per)


SEEDS = {"x": 0x51ED, "y": 0xA11CE}


class ShardedReduction:
    """One rank's part of the sharded dot/asum over hash-generated inputs."""

    def __init__(self, kind: str, total_elems: int, world: int = 1, rank: int = 0, device: int = 0,
                 L: int = 1024, K: int = 32, blocks: Optional[int] = None, combine: str = "nccl",
                 allgather=None):
        """combine: "peer" -- the kernel sums the ranks' partials itself over
        NVLink (peer.PeerGroup, one kernel per step); "nccl" -- a 4-byte
        ncclAllReduce after the kernel (launch(..., allreduce=True))."""
        if kind not in ("asum", "dot"):
            raise ValueError(kind)
        if combine not in ("peer", "nccl"):
            raise ValueError(combine)
        self.combine = combine
        self.kind, self.device = kind, device
        chunk = 4 * K * L
        self.shard = shard_plan(total_elems, chunk, world, rank)
        text = asum_program(L, K) if kind == "asum" else dot_program(L, K)
        prog = compile_program(text, name=f"{kind}_shard")
        self.prog = prog
        n = self.shard.chunks
        self.peer = None
        if combine == "peer":
            from .peer import PeerGroup
            self.peer = PeerGroup(device, rank, world, 1, allgather)
        self.exe = executable(prog, (blocks or n, L), {"n": n}, float_mode=True, device=device,
                              peer=self.peer)
        self.bytes = (4 if kind == "asum" else 8) * self.shard.elems
        self.total_bytes = self.bytes * world

    def fill_inputs(self, stream=None):
        sh = self.shard
        names = ["xs"] if self.kind == "asum" else ["xs", "ys"]
        for name, seed in zip(names, (SEEDS["x"], SEEDS["y"])):
            RT.lib().dpia_fill_hash_f32(self.device, self.exe.buffers[name].ptr, sh.elems,
                                        sh.elem_offset, seed, -1.0, 1.0,
                                        stream.handle if stream else None)

    def launch(self, stream, allreduce: bool):
        self.exe.launch(stream)
        if allreduce and self.combine == "nccl":
            RT.lib().dpia_nccl_allreduce(self.exe.buffers["out"].ptr, 1, 0, stream.handle)

    def result(self, stream=None) -> float:
        """The (combined) result; ordered after the launches on `stream`, or
        after all device work when no stream is given."""
        if stream is not None:
            stream.sync()
        return float(self.exe.download("out", stream)[0])
