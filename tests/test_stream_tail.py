"""Streaming tail (cuda/emit.py ProgramEmitter._stream_plan).

A kernel whose grid phase is a mapGlobal writing one partial per work-item
and whose tail is one thread's in-order fold of those partials (config 1's
literal program: reduce (+) 0 (mapGlobal ... (split 1024 (zip xs ys)))) runs
the tail in one extra block from the start: each warp publishes each round
of work-items on that round's counter, and the tail waits for a round before
its TMA ring copies that round's partials.  The fold order is unchanged, so
results are bit-identical to the last-block ticket tail.

CPU: when the streaming form is chosen and when it falls back.  GPU: int mode
exact, fp32 bit-identical to the ticket tail over 1..8 rounds, chained
launches.
"""
import numpy as np
import pytest

from paper_1710_08332_b200 import compile_program
from paper_1710_08332_b200.bench_programs import dot_literal_program
from paper_1710_08332_b200.cuda import emit as EM


def _emit(chunk, n, launch, float_mode=True):
    prog = compile_program(dot_literal_program(chunk))
    outs = [("out", prog.out_type)]
    ins = [(nm, t.data) for nm, t in prog.source.params]
    return EM.emit_cuda(prog.imperative, outs, ins, float_mode=float_mode, sigma={"n": n}, launch=launch)


def test_literal_dot_streams_its_tail():
    src, sig = _emit(1024, 16384, (128, 32))
    k = sig.kernels[0]
    # 4 rounds x K = 4 launch slots of round counters, then 4 release words,
    # initialised for the first epochs 16..19 (slots 0..3)
    assert k.extra_blocks == 1 and k.counter_words == 20 and k.fused_tail
    assert k.counter_init == [(16, 12), (17, 13), (18, 14), (19, 15)] and ("epoch", "dpia_epoch") in k.args
    assert "const int dpia_par = (int)(dpia_epoch % 4u);" in src
    assert "dpia::stream_wait(dpia_counter + dpia_par * 4, dpia_ready" in src
    assert "dpia::stream_publish(dpia_counter + dpia_par * 4 + (i_" in src   # a round index
    assert "g_tmp4[16384 * dpia_par + " in src                   # the partials: one slice per slot
    assert "dpia::parity_release(dpia_counter + 16 + dpia_par, dpia_epoch)" in src
    assert "dpia::parity_wait_once(dpia_pw, dpia_counter + 16 + dpia_par, dpia_epoch, 4u);" in src
    assert "dpia::grid_arrive(dpia_counter" not in src
    assert "(gridDim.x - 1)" in src
    # the output is written after the previous grid completed; the partials
    # are not waited on that way any more
    body = src.split('extern "C"')[1]
    assert body.count("dpia::pdl_wait_once(dpia_chained);") == 1
    assert body.index("dpia::pdl_wait_once(dpia_chained);") < body.index("out[0] =")
    src, sig = _emit(1024, 16384, (16, 32))                      # 32 rounds
    assert sig.kernels[0].counter_words == 132
    assert sig.buffers[0][1].size.const == 4                     # one partials slice per slot


def test_stream_tail_without_parity_pipelining(monkeypatch):
    monkeypatch.setattr(EM, "STREAM_PIPE", False)
    src, sig = _emit(1024, 16384, (128, 32))
    k = sig.kernels[0]
    assert k.extra_blocks == 1 and k.counter_words == 4 and not k.counter_init
    assert "dpia_par" not in src.split('extern "C"')[1] and "dpia::stream_wait(dpia_counter, dpia_ready" in src


def test_stream_tail_falls_back(monkeypatch):
    # n not a multiple of 32: warps would straddle the end of a round
    src, sig = _emit(1024, 16384 + 16, (129, 32))
    assert sig.kernels[0].extra_blocks == 0 and "dpia::grid_arrive(dpia_counter" in src
    # a short tail (32 partials) is folded by plain loads, not the ring:
    # it could read partials before they are published
    src, sig = _emit(1024, 32, (1, 32))
    assert sig.kernels[0].extra_blocks == 0 and "dpia::grid_arrive(dpia_counter" in src
    monkeypatch.setattr(EM, "STREAM_TAIL", False)
    src, sig = _emit(1024, 16384, (128, 32))
    assert sig.kernels[0].extra_blocks == 0 and "dpia::grid_arrive(dpia_counter" in src


PERMUTED = """
(param xs (exp (array 1048576 num)))
(reduce (+) 0 (toGlobal (lam t (join (transpose (split 64 t))))
  (mapGlobal (lam (c (exp (array 256 num))) (reduce (+) 0 c)) (split 256 xs))))
"""


def test_permuted_partials_do_not_stream():
    """The partials stored through a layout view (work-item i writes partial
    64 (i mod 64) + i / 64): a round's partials are not a contiguous prefix,
    so the streaming tail could read one before its round publishes -- the
    kernel keeps the last-block ticket."""
    prog = compile_program(PERMUTED)
    outs = [("out", prog.out_type)]
    ins = [(nm, t.data) for nm, t in prog.source.params]
    src, sig = EM.emit_cuda(prog.imperative, outs, ins, sigma={}, launch=(32, 32))
    assert sig.kernels[0].extra_blocks == 0 and "dpia::grid_arrive(dpia_counter" in src
    assert "g_tmp4[64 * ((i_3_1) % 64) + ((i_3_1) / 64)]" in src


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
def test_permuted_partials_int_exact():
    from paper_1710_08332_b200 import run_program_cuda
    xs = np.random.default_rng(5).integers(-9, 10, 1048576)
    got = run_program_cuda(compile_program(PERMUTED), {"xs": xs}, sigma={}, launch=(32, 32),
                           float_mode=False, flat=True)
    assert int(got[0]) == int(xs.sum())

def _run(chunk, n, launch, inputs, float_mode, stream=True, rows=True):
    from paper_1710_08332_b200 import executable
    from paper_1710_08332_b200 import runtime as RT
    old = EM.STREAM_TAIL, EM.ROW_TMA
    EM.STREAM_TAIL, EM.ROW_TMA = stream, rows
    try:
        exe = executable(compile_program(dot_literal_program(chunk)), launch, {"n": n}, float_mode=float_mode)
    finally:
        EM.STREAM_TAIL, EM.ROW_TMA = old
    st = RT.Stream(0)
    for nm, v in inputs.items():
        exe.upload(nm, v, st)
    outs = []
    for _ in range(3):                    # repeated launches reuse the reset counters
        exe.launch(st)
        outs.append(np.asarray(exe.download("out", st)).copy())
    st.sync()
    assert all(np.array_equal(o.view(np.uint8), outs[0].view(np.uint8)) for o in outs)
    return outs[0], exe


@pytest.mark.gpu
@pytest.mark.parametrize("chunk,n,G,L", [(1024, 1024, 32, 32), (1024, 1024, 16, 32), (256, 4096, 32, 32),
                                         (256, 4096, 16, 64), (64, 8192, 32, 32), (128, 3072, 32, 32),
                                         (1024, 16384, 128, 32)])
def test_stream_tail_int_exact(chunk, n, G, L):
    rng = np.random.default_rng(n + G)
    xs = rng.integers(-9, 10, n * chunk)
    ys = rng.integers(-9, 10, n * chunk)
    got, exe = _run(chunk, n, (G, L), {"xs": xs, "ys": ys}, False)
    assert exe.sig.kernels[0].extra_blocks == 1
    assert int(got[0]) == int(np.dot(xs, ys))


@pytest.mark.gpu
@pytest.mark.parametrize("chunk,n,G,L", [(1024, 16384, 512, 32), (1024, 16384, 256, 32), (1024, 16384, 128, 32),
                                         (1024, 16384, 64, 32), (512, 8192, 96, 32)])
def test_stream_tail_bit_identical_fp32(chunk, n, G, L):
    rng = np.random.default_rng(G)
    inputs = {"xs": rng.uniform(0, 1, n * chunk).astype(np.float32),
              "ys": rng.uniform(0, 1, n * chunk).astype(np.float32)}
    a, exe = _run(chunk, n, (G, L), inputs, True, stream=True)
    b, ref = _run(chunk, n, (G, L), inputs, True, stream=False, rows=False)
    assert exe.sig.kernels[0].extra_blocks == 1 and ref.sig.kernels[0].extra_blocks == 0
    assert a.view(np.uint32)[0] == b.view(np.uint32)[0]


@pytest.mark.gpu
def test_stream_tail_chained_steps():
    """Steps chained behind each other (programmatic dependent launch), each
    on its own inputs and output: every step's bits equal an unchained run."""
    from paper_1710_08332_b200 import executable
    from paper_1710_08332_b200 import runtime as RT
    chunk, n, launch = 256, 4096, (32, 32)          # 4 rounds
    exe = executable(compile_program(dot_literal_program(chunk)), launch, {"n": n}, float_mode=True)
    assert exe.sig.kernels[0].extra_blocks == 1
    st = RT.Stream(0)
    rng = np.random.default_rng(3)
    steps = []
    for _ in range(6):
        xs = rng.uniform(0, 1, n * chunk).astype(np.float32)
        ys = rng.uniform(0, 1, n * chunk).astype(np.float32)
        bx, by, bo = RT.DeviceBuffer(xs.nbytes), RT.DeviceBuffer(ys.nbytes), RT.DeviceBuffer(4)
        bx.upload(xs, st)
        by.upload(ys, st)
        steps.append((xs, ys, bx, by, bo))
    st.sync()
    for i, (_, _, bx, by, bo) in enumerate(steps):
        exe.launch_with(st, {"xs": bx.ptr, "ys": by.ptr, "out": bo.ptr}, chain=i > 0)
    st.sync()
    for xs, ys, _, _, bo in steps:
        got = np.empty(1, np.float32)
        bo.download(got.view(np.uint8), st)
        want, _ = _run(chunk, n, launch, {"xs": xs, "ys": ys}, True, stream=False, rows=False)
        assert got.view(np.uint32)[0] == want.view(np.uint32)[0]


@pytest.mark.gpu
@pytest.mark.parametrize("stream", [True, False])
@pytest.mark.parametrize("chunk,n,G,L", [(1024, 16384, 512, 32), (1024, 16384, 128, 32), (512, 8192, 32, 128),
                                         (256, 4096, 8, 64), (128, 3072, 32, 32)])
def test_row_tma_folds_bit_identical(stream, chunk, n, G, L):
    """Work-item folds read through 2-D TMA row boxes (128-byte swizzle,
    per-warp slot ring running ahead across rounds) give the bits of the
    register-queue folds, with and without the streaming tail (the ticket
    tail's static shared flag sits in front of the slots)."""
    rng = np.random.default_rng(n + L)
    inputs = {"xs": rng.uniform(0, 1, n * chunk).astype(np.float32),
              "ys": rng.uniform(0, 1, n * chunk).astype(np.float32)}
    a, exe = _run(chunk, n, (G, L), inputs, True, stream=stream, rows=True)
    b, _ = _run(chunk, n, (G, L), inputs, True, stream=stream, rows=False)
    assert "dpia::tma_tile_2d(" in exe.src and exe.sig.tmaps
    assert a.view(np.uint32)[0] == b.view(np.uint32)[0]


def test_slot_count_scales_with_the_serial_tail():
    """K launch slots cover the grid phase of one launch with K serial tails:
    config 1 (16384 partials) gets 4, the asum proxy (65536) 16."""
    from paper_1710_08332_b200.bench_programs import asum_proxy_config, dot_literal_config
    for cfg, K in ((dot_literal_config(), 4), (asum_proxy_config(), 16)):
        prog = compile_program(cfg.text)
        outs = [("out", prog.out_type)]
        ins = [(nm, t.data) for nm, t in prog.source.params]
        src, sig = EM.emit_cuda(prog.imperative, outs, ins, sigma=cfg.sigma, launch=cfg.launch)
        assert f"const int dpia_par = (int)(dpia_epoch % {K}u);" in src
        assert sig.kernels[0].counter_words == K * (4 + 1)
