"""Sharded reductions (config 5).

CPU (gloo, world size 2): the shard plan covers the outer chunk range exactly
once, and per-rank partials of the oracle combined with an all-reduce equal
the unsharded oracle -- the host-side logic of the multi-GPU driver.
GPU: one rank runs the emitted kernel on device-generated hashed inputs and
matches the host restatement of the same hash (bit-exact inputs), both at
full N = 2^31 for asum and on a smaller dot.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import blas_np
from paper_1710_08332_b200.scaleout import SEEDS, shard_plan


def test_shard_plan_partitions_the_range():
    for world in (1, 2, 4, 8):
        shards = [shard_plan(1 << 31, 1 << 17, world, r) for r in range(world)]
        covered = sorted((s.elem_offset, s.elem_offset + s.elems) for s in shards)
        assert covered[0][0] == 0 and covered[-1][1] == 1 << 31
        assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
    with pytest.raises(ValueError):
        shard_plan(1000, 64, 2, 0)


def test_hash_is_a_pure_function_of_the_global_index():
    full = blas_np.hash_f32(4096, 0, 7, -1.0, 1.0)
    assert np.array_equal(full[1000:3000], blas_np.hash_f32(2000, 1000, 7, -1.0, 1.0))
    assert full.min() >= -1.0 and full.max() < 1.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, chunk, kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    sh = shard_plan(total, chunk, world, rank)
    x = blas_np.hash_f32(sh.elems, sh.elem_offset, SEEDS["x"], -1.0, 1.0).astype(np.float64)
    if kind == "asum":
        part = float(np.abs(x).sum())
    else:
        y = blas_np.hash_f32(sh.elems, sh.elem_offset, SEEDS["y"], -1.0, 1.0).astype(np.float64)
        part = float(np.dot(x, y))
    t = torch.tensor([part], dtype=torch.float64)
    dist.all_reduce(t)
    if rank == 0:
        q.put(float(t.item()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["asum", "dot"])
def test_gloo_world2_partials_combine_to_the_unsharded_result(kind):
    total, chunk, world = 1 << 20, 1 << 14, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, chunk, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = (blas_np.hashed_asum(total, SEEDS["x"]) if kind == "asum"
            else blas_np.hashed_dot(total, SEEDS["x"], SEEDS["y"]))
    assert abs(got - want[0]) <= 1e-12 * want[1]


@pytest.mark.gpu
@pytest.mark.parametrize("kind,total", [("asum", 1 << 31), ("dot", 1 << 26)])
def test_sharded_kernel_matches_hash_oracle(kind, total):
    from paper_1710_08332_b200 import runtime as RT
    from paper_1710_08332_b200.scaleout import ShardedReduction
    run = ShardedReduction(kind, total)
    st = RT.Stream(0)
    run.fill_inputs(st)
    run.launch(st, allreduce=False)
    st.sync()
    got = run.result()
    want = (blas_np.hashed_asum(total, SEEDS["x"]) if kind == "asum"
            else blas_np.hashed_dot(total, SEEDS["x"], SEEDS["y"]))
    assert blas_np.within(got, want[0], want[1]), (got, want)


@pytest.mark.gpu
def test_nccl_single_rank_allreduce_through_the_c_abi():
    """dpia_nccl_* (NCCL from the torch wheel, dlopen'ed) on one rank: the
    sum all-reduce of a partial leaves it unchanged."""
    import ctypes
    from paper_1710_08332_b200 import runtime as RT
    RT.init(0)
    uid = ctypes.create_string_buffer(128)
    RT.lib().dpia_nccl_unique_id(uid)
    RT.lib().dpia_nccl_init(0, 1, 0, uid.raw)
    buf = RT.DeviceBuffer(16)
    buf.upload(np.array([2.5, 0, 0, 0], np.float32))
    st = RT.Stream(0)
    RT.lib().dpia_nccl_allreduce(buf.ptr, 1, 0, st.handle)
    st.sync()
    out = np.zeros(4, np.float32)
    buf.download(out)
    assert out[0] == 2.5
    RT.lib().dpia_nccl_destroy()


# ------------------------------------------------ fused peer (NVLink) combine

def test_peer_mailbox_layout_and_emitted_kernel():
    """CPU: the emitter appends dpia::peer_sum to the reduction tail with the
    peer parameters, and rejects programs without such a tail."""
    from paper_1710_08332_b200 import CudaError, compile_program
    from paper_1710_08332_b200.bench_programs import dot_program, scal_program
    from paper_1710_08332_b200.cuda.emit import emit_cuda
    from paper_1710_08332_b200.peer import SLOT_BYTES, mailbox_bytes
    assert mailbox_bytes(8, 1) == (2 * 8 + 1) * SLOT_BYTES
    prog = compile_program(dot_program(32, 2))
    outs = [(n, t) for n, t, k in prog.params if k == "out"]
    ins = [(n, t) for n, t, k in prog.params if k == "in"]
    src, sig = emit_cuda(prog.imperative, outs, ins, True, "d", sigma={"n": 4}, launch=(4, 32), peer=True)
    assert "dpia::peer_sum<float>(reinterpret_cast<float*>(out), 1, dpia_peer_boxes" in src
    kinds = [k for k, _ in sig.kernels[-1].args]
    assert kinds[-4:] == ["peer_boxes", "peer_rank", "peer_world", "peer_epoch"]
    sprog = compile_program(scal_program())
    outs = [(n, t) for n, t, k in sprog.params if k == "out"]
    ins = [(n, t) for n, t, k in sprog.params if k == "in"]
    with pytest.raises(CudaError):
        emit_cuda(sprog.imperative, outs, ins, True, "s", sigma={"n": 64}, launch=(2, 32), peer=True)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["asum", "dot"])
def test_peer_combine_single_rank(kind):
    """world = 1: the fused combine publishes to and reads from its own
    mailbox; repeated launches (epochs, both parities) keep the result."""
    from paper_1710_08332_b200 import runtime as RT
    from paper_1710_08332_b200.scaleout import ShardedReduction
    total = 1 << 24
    run = ShardedReduction(kind, total, combine="peer")
    st = RT.Stream(0)
    run.fill_inputs(st)
    for _ in range(5):
        run.launch(st, allreduce=True)
    st.sync()
    run.peer.check()
    want = (blas_np.hashed_asum(total, SEEDS["x"]) if kind == "asum"
            else blas_np.hashed_dot(total, SEEDS["x"], SEEDS["y"]))
    assert blas_np.within(run.result(), want[0], want[1])
    run.peer.close()


def _peer_worker(rank, world, port, total, kind, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1710_08332_b200 import runtime as RT
    from paper_1710_08332_b200.peer import torch_allgather
    from paper_1710_08332_b200.scaleout import ShardedReduction
    try:
        run = ShardedReduction(kind, total, world, rank, device=0, combine="peer",
                               allgather=torch_allgather)
        st = RT.Stream(0)
        run.fill_inputs(st)
        st.sync()
        dist.barrier()
        for _ in range(steps):
            run.launch(st, allreduce=True)
        st.sync()
        run.peer.check()
        q.put((rank, run.result()))
        dist.barrier()
        run.peer.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["asum", "dot"])
def test_peer_combine_two_ranks_sharing_one_gpu(kind):
    """Two processes (ranks) on the one GPU of this run, each with its own
    context: the IPC-mapped mailboxes, the release/acquire epoch protocol and
    the double-buffered parities are the same as across NVLink.  Both ranks
    must end with the identical total, equal to the oracle's."""
    total, world, steps = 1 << 24, 2, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, total, kind, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    assert all(isinstance(v, float) for v in res.values()), res
    assert res[0] == res[1]
    want = (blas_np.hashed_asum(total, SEEDS["x"]) if kind == "asum"
            else blas_np.hashed_dot(total, SEEDS["x"], SEEDS["y"]))
    assert blas_np.within(res[0], want[0], want[1]), (res, want)


def test_peer_and_pipeline_argument_checks():
    """Host-side validation, before any device work (CPU)."""
    from paper_1710_08332_b200.peer import PeerGroup
    from paper_1710_08332_b200.pipeline import RowPipeline, mm_pipeline
    with pytest.raises(ValueError):
        PeerGroup(0, 2, 2)                 # rank outside the world
    with pytest.raises(ValueError):
        PeerGroup(0, 0, 2)                 # multi-rank group without an allgather
    with pytest.raises(ValueError):
        RowPipeline(lambda r: "", lambda r: (1, 1), 10, 3, {}, {}, 0)
    with pytest.raises(ValueError):
        mm_pipeline(256, 128, 128, chunks=4)   # 64-row chunks are not whole 128-row tiles
    from paper_1710_08332_b200.pipeline import mm_tile_pipeline
    with pytest.raises(ValueError):
        mm_tile_pipeline(256, 256, 128, rows=2, cols=4)   # 64-column panels are not whole tiles
    with pytest.raises(ValueError):
        mm_tile_pipeline(256, 384, 128, rows=2, cols=2)   # 384 / 2 = 192 is not whole tiles


@pytest.mark.parametrize("rows,cols", [(1, 1), (4, 4), (4, 2), (1, 3), (5, 2)])
def test_tile_schedule(rows, cols):
    """TilePipeline's copy order interleaves A row blocks and B column panels
    in proportion; every tile appears once, after the copies of both its
    operands, and tiles are ordered by that copy (CPU)."""
    from paper_1710_08332_b200.pipeline import tile_schedule
    order, tiles = tile_schedule(rows, cols)
    assert sorted(order) == sorted([("A", i) for i in range(rows)] + [("B", j) for j in range(cols)])
    assert sorted(tiles) == [(i, j) for i in range(rows) for j in range(cols)]
    pos = {b: k for k, b in enumerate(order)}
    ready = [max(pos[("A", i)], pos[("B", j)]) for i, j in tiles]
    assert ready == sorted(ready)
    assert order[0] == ("A", 0) and ("B", 0) in order[:2 + rows // cols]


def _two_gpu_worker(rank, world, port, kind, q):
    """One rank per DISTINCT GPU: the fused combine over real NVLink P2P,
    checked against the rank-order sum of the gathered partials (bit-exact)
    and against NCCL's all-reduce of the same partials."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import ctypes

    import torch
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    from paper_1710_08332_b200 import runtime as RT
    from paper_1710_08332_b200.peer import cross_check, local_twin, torch_allgather
    from paper_1710_08332_b200.scaleout import ShardedReduction
    try:
        RT.init(rank)
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            RT.lib().dpia_nccl_unique_id(uid)
        obj = [bytes(uid.raw)]
        dist.broadcast_object_list(obj, src=0)
        RT.lib().dpia_nccl_init(rank, world, rank, obj[0])
        run = ShardedReduction(kind, 1 << 28, world, rank, device=rank, combine="peer",
                               allgather=torch_allgather)
        st = RT.Stream(rank)
        run.fill_inputs(st)
        st.sync()
        ev = cross_check(run.exe, local_twin(run.exe, run.prog), st, torch_allgather)
        buf = RT.DeviceBuffer(16, rank)
        buf.upload(np.array([ev["partials"][rank], 0, 0, 0], np.float32))
        RT.lib().dpia_nccl_allreduce(buf.ptr, 1, 0, st.handle)
        st.sync()
        v = np.zeros(4, np.float32)
        buf.download(v)
        q.put((rank, ev["bit_exact"], ev["peer_total"][0], float(v[0]), ev["abs_sum"]))
        dist.barrier()
        run.peer.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), None, None, None))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["asum", "dot"])
def test_peer_combine_two_distinct_gpus(kind):
    """The fused cross-GPU combine across two physical GPUs (skipped on a
    one-GPU box; the shared-GPU test above covers the protocol there)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_two_gpu_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=120)
    for r in (0, 1):
        exact, peer, nccl, absum = res[r]
        assert exact is True, res
        assert abs(peer - nccl) <= 1e-6 * absum
    assert res[0][1] == res[1][1]
    want = (blas_np.hashed_asum(1 << 28, SEEDS["x"]) if kind == "asum"
            else blas_np.hashed_dot(1 << 28, SEEDS["x"], SEEDS["y"]))
    assert blas_np.within(res[0][1], want[0], want[1])


def test_rank_order_sum_is_the_kernels_association():
    """CPU: peer.rank_order_sum adds in rank order in the partials' dtype
    (what dpia::peer_sum does), which differs from a float64 sum."""
    from paper_1710_08332_b200.peer import rank_order_sum
    parts = [np.array([1e8], np.float32), np.array([1.0], np.float32), np.array([-1e8], np.float32)]
    got = rank_order_sum(parts)
    assert got.dtype == np.float32 and got[0] == np.float32(np.float32(1e8 + 1.0) - 1e8)
    assert rank_order_sum([np.array([3], np.int64), np.array([4], np.int64)])[0] == 7


def _cross_worker(rank, world, port, kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1710_08332_b200 import runtime as RT
    from paper_1710_08332_b200.peer import cross_check, local_twin, torch_allgather
    from paper_1710_08332_b200.scaleout import ShardedReduction
    try:
        run = ShardedReduction(kind, 1 << 24, world, rank, device=0, combine="peer",
                               allgather=torch_allgather)
        st = RT.Stream(0)
        run.fill_inputs(st)
        st.sync()
        ev = cross_check(run.exe, local_twin(run.exe, run.prog), st, torch_allgather)
        q.put((rank, ev["bit_exact"], ev["peer_total"][0], ev["rank_order_sum"][0]))
        dist.barrier()
        run.peer.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), None, None))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["asum", "dot"])
def test_cross_check_two_ranks_sharing_one_gpu(kind):
    """peer.cross_check (bench.py's agreement gate at N > 1): each rank's
    combine-free twin gives its partial, and the fused combine's total is
    bit-identical to the rank-order sum of the gathered partials."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cross_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=120)
    for r in (0, 1):
        assert res[r][0] is True, res
        assert res[r][1] == res[r][2]
    assert res[0][1] == res[1][1]
