"""TMA tensor staging of 2-D box k-tiles (cuda/emit.py KernelEmitter._tma_plan).

A rotating toLocal k-tile whose staging command copies a plain 2-D box of an
input -- tile element (r, c) from X[origin(k) + r * P + c] -- can be emitted
as cp.async.bulk.tensor.2d copies through a CUtensorMap kernel parameter,
completing on an mbarrier, instead of register prefetch + shared stores.  The
decision is made by enumerating the staging's copies (every work-item index a
constant) and checking the index map element by element, so stagings that
permute (mm's transposed A tile) keep the register path.

CPU: which stagings qualify, the tensor-map geometry, the emitted calls and
an nvcc compile.  GPU: bit-identical to the register path, int-exact against
A @ B, and re-pointed inputs (launch_with) re-encode their tensor maps.
"""
import numpy as np
import pytest

from paper_1710_08332_b200 import compile_program
from paper_1710_08332_b200.bench_programs import mm_config, mm_program, mm_rect_program, mm_tma_config
from paper_1710_08332_b200.cuda.emit import emit_cuda


def _emit(text, launch, float_mode=True, tma=True):
    prog = compile_program(text)
    outs = [("out", prog.out_type)]
    ins = [(n, t.data) for n, t in prog.source.params]
    return emit_cuda(prog.imperative, outs, ins, float_mode=float_mode, sigma={}, launch=launch,
                     tma_tiles=tma)


def test_mm_b_tile_is_a_tma_box_and_a_tile_is_not():
    cfg = mm_tma_config()
    src, sig = _emit(cfg.text, cfg.launch)
    # B (K x N row-major): 16-row x 128-column boxes at (128 * bx, 16 * k)
    assert sig.tmaps == {"dpia_tm0": ("B", 4, 4096, 4096, 16384, 16, 128, 0)}
    assert "const __grid_constant__ dpia::TensorMap dpia_tm0" in src
    assert src.count("dpia::tma_tile_2d(") == 2          # prologue + in-loop refill
    assert "dpia::tile_bar_init(" in src and "dpia::ring_wait(" in src
    # A's staging stores transposed (k-major): not a box, stays on registers
    assert "pf1_0 = dpia::vload<float, 4>(A," in src
    assert ("tmap", "dpia_tm0") in sig.kernels[0].args


def test_tma_off_by_default_and_int_mode_geometry():
    cfg = mm_config()
    _src, sig = _emit(cfg.text, cfg.launch, tma=None)
    assert sig.tmaps == {}
    src, sig = _emit(mm_program(256, 128, 384, 128, 8, 8), ((1, 2), (16, 16)), float_mode=False)
    # N = T: the tile is one contiguous run of B, boxed as 4 rows of 256
    assert sig.tmaps == {"dpia_tm0": ("B", 8, 192, 256, 2048, 4, 256, 0)}
    assert "long long" in src


def test_rect_tiles_and_non_multiple_boxes():
    src, sig = _emit(mm_rect_program(256, 256, 128, 128, 128, 16, 8, 16), ((2, 2), (8, 16)))
    assert len(sig.tmaps) == 1
    # a 16-column tile of 4-byte elements is 64 bytes: a legal box
    src, sig = _emit(mm_program(32, 32, 32, 16, 8, 4), ((2, 2), (4, 4)))
    assert sig.tmaps == {"dpia_tm0": ("B", 4, 32, 32, 128, 8, 16, 0)}


def test_tma_source_compiles_for_sm100a():
    from paper_1710_08332_b200.aot import nvcc_check
    cfg = mm_tma_config()
    src, _ = _emit(cfg.text, cfg.launch)
    report = nvcc_check(src, "mm_tma")
    assert "spill" in report


# ------------------------------------------------------------------ GPU

def _run(text, launch, inputs, float_mode, tma):
    from paper_1710_08332_b200 import executable
    from paper_1710_08332_b200 import runtime as RT
    exe = executable(compile_program(text), launch, {}, float_mode=float_mode, tma_tiles=tma)
    st = RT.Stream(0)
    for n, v in inputs.items():
        exe.upload(n, v, st)
    exe.launch(st)
    out = exe.download("out", st)
    st.sync()
    return np.asarray(out), exe


MM_CASES = [(32, 32, 32, 16, 8, 4), (64, 96, 128, 32, 8, 4), (256, 128, 384, 128, 8, 8),
            (128, 256, 64, 64, 16, 4), (256, 256, 128, 128, 16, 8), (128, 128, 128, 128, 32, 8)]


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K,T,BK,R", MM_CASES)
def test_mm_tma_int_exact(M, N, K, T, BK, R):
    A = np.random.default_rng(6).integers(-9, 10, (M, K))
    B = np.random.default_rng(7).integers(-9, 10, (K, N))
    launch = ((N // T, M // T), (T // R, T // R))
    got, exe = _run(mm_program(M, N, K, T, BK, R), launch, {"A": A, "B": B}, False, True)
    assert exe.sig.tmaps, "the B staging was not lowered to TMA"
    assert np.array_equal(got.astype(np.int64).reshape(M, N), A @ B)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["rect", "rows", "sectors"])
def test_mm_tma_variants_bit_identical_fp32(case):
    M, N, K = 256, 256, 512
    if case == "rect":
        text, launch = mm_rect_program(M, N, K, 128, 128, 16, 8, 16), ((2, 2), (8, 16))
    else:
        text = mm_program(M, N, K, 128, 16, 8, a_by_rows=case == "rows", a_sectors=case == "sectors")
        launch = ((2, 2), (16, 16))
    rng = np.random.default_rng(41)
    inputs = {"A": rng.uniform(-1, 1, (M, K)).astype(np.float32),
              "B": rng.uniform(-1, 1, (K, N)).astype(np.float32)}
    a, exe = _run(text, launch, inputs, True, True)
    b, _ = _run(text, launch, inputs, True, False)
    assert exe.sig.tmaps
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.gpu
def test_mm_tma_full_size_bit_identical_to_register_path():
    from oracle import blas_np
    cfg = mm_tma_config()
    inputs = {"A": blas_np.seeded((4096, 4096), 5, -1.0, 1.0), "B": blas_np.seeded((4096, 4096), 6, -1.0, 1.0)}
    a, _ = _run(cfg.text, cfg.launch, inputs, True, True)
    b, _ = _run(cfg.text, cfg.launch, inputs, True, False)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    rows = np.random.default_rng(0).choice(4096, 64, replace=False)
    want, absterms = blas_np.mm(inputs["A"], inputs["B"], rows)
    assert blas_np.within(a.reshape(4096, 4096)[rows], want, absterms)


@pytest.mark.gpu
def test_mm_tma_launch_with_reencodes_tensor_maps():
    """launch_with re-points B at another device buffer: its tensor map is
    encoded over the new address for that launch."""
    from paper_1710_08332_b200 import runtime as RT
    M = N = K = 128
    text, launch = mm_program(M, N, K, 64, 16, 4), ((2, 2), (16, 16))
    A = np.random.default_rng(1).integers(-9, 10, (M, K))
    B1 = np.random.default_rng(2).integers(-9, 10, (K, N))
    B2 = np.random.default_rng(3).integers(-9, 10, (K, N))
    got, exe = _run(text, launch, {"A": A, "B": B1}, False, True)
    assert np.array_equal(got.astype(np.int64).reshape(M, N), A @ B1)
    st = RT.Stream(0)
    other = RT.DeviceBuffer(B2.size * 8, 0)
    other.upload(B2.astype(np.int64), st)
    exe.launch_with(st, {"B": other.ptr})
    out = np.asarray(exe.download("out", st))
    st.sync()
    assert np.array_equal(out.astype(np.int64).reshape(M, N), A @ B2)
