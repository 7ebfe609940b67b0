"""GPU parity: every program is emitted as CUDA, compiled with NVRTC for
sm_100a, launched through libdpia_rt.so, and compared with the oracle.

* golden programs: the reference's sample/test programs and 400 programs of
  the reference's own fuzzer, with the reference's eval_phrase result; int
  mode is bit-exact, float within 1e-5*max(1,|want|) (the reference's bound,
  TST/test_acceptance.py:149-150);
* the benchmark strategies at reduced sizes, int mode bit-exact against the
  oracle interpreter, and at full BASELINE sizes in fp32 against the float64
  NumPy oracle with |got-want| <= 1e-4 * sum|terms|.
"""
import numpy as np
import pytest

from conftest import load_golden
from oracle import blas_np
from oracle.dpia_eval import eval_phrase, flatten_value, from_json
from paper_1710_08332_b200 import CudaError, compile_program, run_program_cuda
from paper_1710_08332_b200.bench_programs import (asum_config, asum_program, dot_config,
                                                  dot_program, gemv_config, gemv_program, mm_config,
                                                  mm_program, scal_config, scal_program)

pytestmark = pytest.mark.gpu

GOLDEN = load_golden("programs.json")
FUZZ = [c for c in load_golden("fuzz.json") if c["reparses"]]


def _check(case, launch):
    prog = compile_program(case["text"])
    inputs = {k: from_json(v) for k, v in case["inputs"].items()}
    fm = case.get("float", False)
    got = run_program_cuda(prog, inputs, sigma=case.get("sigma", {}), launch=launch, float_mode=fm,
                           flat=True)
    want = flatten_value(from_json(case["expected"]))
    if not fm and any(abs(v) >= 2 ** 63 for v in want):
        pytest.skip("reference result exceeds int64 (the reference's C path overflows too)")
    if fm:
        assert np.allclose(got, want, rtol=1e-5, atol=1e-5), (got, want)
    else:
        assert [int(v) for v in got] == want


@pytest.mark.parametrize("launch", [(1, 1), (2, 2), (2, 4), (4, 8), (3, 32)])
@pytest.mark.parametrize("case", GOLDEN, ids=lambda c: c["name"])
def test_golden_programs(case, launch):
    _check(case, launch)


@pytest.mark.parametrize("launch", [(3, 2048), (2, 4096)])
@pytest.mark.parametrize("case", GOLDEN, ids=lambda c: c["name"])
def test_golden_programs_oversized_work_groups(case, launch):
    """The reference accepts any (G, L); work-groups above CUDA's 1024
    threads run as 1024-thread blocks with striding work-item loops."""
    _check(case, launch)


def test_mm_oversized_2d_launch():
    """A 64 x 64 work-item request (4096 > 1024) for mm: the block is capped
    to 64 x 16 and mapLocal1 strides; the product is unchanged."""
    M = N = K = 128
    prog = compile_program(mm_program(M, N, K, 128, 8, 8))
    A = np.random.default_rng(40).integers(-9, 10, (M, K))
    B = np.random.default_rng(41).integers(-9, 10, (K, N))
    got = run_program_cuda(prog, {"A": A, "B": B}, launch=((1, 1), (64, 64)), float_mode=False, flat=True)
    assert np.array_equal(np.asarray(got, np.int64).reshape(M, N), A @ B)


@pytest.mark.parametrize("case", FUZZ, ids=lambda c: f"seed{c['seed']}")
def test_reference_fuzz_programs(case):
    """Kernel-legal programs (the reference simulates them) must run; the
    others run when the CUDA backend accepts their hierarchy."""
    for launch in ((2, 2), (3, 5)):
        try:
            _check(case, launch)
        except CudaError:
            if case["opencl_legal"]:
                raise
            pytest.skip("hierarchy rejected by the backend (reference rejects it too)")


# ------------------------------------------------------------ benchmarks

def _ints(n, seed):
    return np.random.default_rng(seed).integers(-9, 10, n).tolist()


@pytest.mark.parametrize("L,K,n,blocks", [(32, 2, 3, 3), (64, 4, 5, 2), (256, 16, 8, 8), (256, 16, 9, 4)])
def test_dot_strategy_int_exact(L, K, n, blocks):
    prog = compile_program(dot_program(L, K))
    N = n * 4 * K * L
    xs, ys = _ints(N, 1), _ints(N, 2)
    got = run_program_cuda(prog, {"xs": xs, "ys": ys}, sigma={"n": n}, launch=(blocks, L),
                           float_mode=False)
    assert got == eval_phrase(prog.source.body, {"xs": xs, "ys": ys}, {"n": n})


@pytest.mark.parametrize("L,K,n,blocks", [(32, 2, 3, 3), (128, 8, 6, 4)])
def test_asum_strategy_int_exact(L, K, n, blocks):
    prog = compile_program(asum_program(L, K))
    xs = _ints(n * 4 * K * L, 3)
    got = run_program_cuda(prog, {"xs": xs}, sigma={"n": n}, launch=(blocks, L), float_mode=False)
    assert got == sum(abs(x) for x in xs)
    assert got == eval_phrase(prog.source.body, {"xs": xs}, {"n": n})


@pytest.mark.parametrize("x_private", [False, True])
@pytest.mark.parametrize("M,N,L,blocks", [(8, 256, 32, 3), (33, 512, 64, 7), (64, 1024, 256, 64)])
def test_gemv_strategy_int_exact(M, N, L, blocks, x_private):
    prog = compile_program(gemv_program(M, N, L, x_private))
    A = np.random.default_rng(4).integers(-9, 10, (M, N))
    x = np.random.default_rng(5).integers(-9, 10, N)
    got = run_program_cuda(prog, {"A": A.tolist(), "x": x.tolist()}, launch=(blocks, L),
                           float_mode=False, flat=True)
    assert [int(v) for v in got] == (A @ x).tolist()


@pytest.mark.parametrize("workload", ["dot", "asum", "gemv", "mm"])
def test_benchmark_configs_full_size_int64_exact(workload):
    """The bench's exact programs and launches at BASELINE.json's full sizes
    in int mode (int64 values in -9..9): bit-exact against numpy's integer
    arithmetic (mm on 64 sampled rows)."""
    from paper_1710_08332_b200.bench_programs import CONFIGS
    cfg = CONFIGS[workload]()
    prog = compile_program(cfg.text)
    rng = np.random.default_rng(77)
    if workload == "dot":
        xs, ys = rng.integers(-9, 10, 1 << 24), rng.integers(-9, 10, 1 << 24)
        got = run_program_cuda(prog, {"xs": xs, "ys": ys}, sigma=cfg.sigma, launch=cfg.launch,
                               float_mode=False, flat=True)
        assert int(got[0]) == int(xs @ ys)
    elif workload == "asum":
        xs = rng.integers(-9, 10, 1 << 26)
        got = run_program_cuda(prog, {"xs": xs}, sigma=cfg.sigma, launch=cfg.launch, float_mode=False,
                               flat=True)
        assert int(got[0]) == int(np.abs(xs).sum())
    elif workload == "gemv":
        A, x = rng.integers(-9, 10, (8192, 8192)), rng.integers(-9, 10, 8192)
        got = run_program_cuda(prog, {"A": A, "x": x}, launch=cfg.launch, float_mode=False, flat=True)
        assert np.array_equal(np.asarray(got, np.int64), A @ x)
    else:
        A, B = rng.integers(-9, 10, (4096, 4096)), rng.integers(-9, 10, (4096, 4096))
        got = np.asarray(run_program_cuda(prog, {"A": A, "B": B}, launch=cfg.launch, float_mode=False,
                                          flat=True), np.int64).reshape(4096, 4096)
        rows = rng.choice(4096, 64, replace=False)
        assert np.array_equal(got[rows], A[rows] @ B)


def test_dot_full_size_fp32():
    cfg = dot_config()
    N = 1 << 24
    xs, ys = blas_np.seeded(N, 0, 0.0, 1.0), blas_np.seeded(N, 1, 0.0, 1.0)
    got = run_program_cuda(compile_program(cfg.text), {"xs": xs, "ys": ys}, sigma=cfg.sigma,
                           launch=cfg.launch, flat=True)
    want, absterms = blas_np.dot(xs, ys)
    assert blas_np.within(got[0], want, absterms), (got[0], want)


def test_asum_full_size_fp32():
    cfg = asum_config()
    xs = blas_np.seeded(1 << 26, 2, -1.0, 1.0)
    got = run_program_cuda(compile_program(cfg.text), {"xs": xs}, sigma=cfg.sigma,
                           launch=cfg.launch, flat=True)
    want, absterms = blas_np.asum(xs)
    assert blas_np.within(got[0], want, absterms), (got[0], want)


def test_gemv_full_size_fp32():
    cfg = gemv_config()
    A = blas_np.seeded((8192, 8192), 3, -1.0, 1.0)
    x = blas_np.seeded(8192, 4, -1.0, 1.0)
    got = run_program_cuda(compile_program(cfg.text), {"A": A, "x": x}, launch=cfg.launch, flat=True)
    want, absterms = blas_np.gemv(A, x)
    assert blas_np.within(got, want, absterms)


@pytest.mark.parametrize("M,N,K,T,BK,R", [(32, 32, 32, 16, 8, 4), (64, 96, 128, 32, 8, 4),
                                          (256, 128, 384, 128, 8, 8), (128, 256, 64, 64, 16, 4),
                                          # pipelined stagings with 2 and 4 loads per work-item
                                          (256, 256, 128, 128, 16, 8), (128, 128, 128, 128, 32, 8)])
def test_mm_strategy_int_exact(M, N, K, T, BK, R):
    prog = compile_program(mm_program(M, N, K, T, BK, R))
    A = np.random.default_rng(6).integers(-9, 10, (M, K))
    B = np.random.default_rng(7).integers(-9, 10, (K, N))
    P = T // R
    got = run_program_cuda(prog, {"A": A, "B": B}, launch=((N // T, M // T), (P, P)),
                           float_mode=False, flat=True)
    assert np.array_equal(np.asarray(got, np.int64).reshape(M, N), A @ B)


@pytest.mark.parametrize("layout", ["rows", "sectors"])
@pytest.mark.parametrize("BK", [16, 32])
def test_mm_a_staging_layouts_int_exact(layout, BK):
    """The alternative A-tile distributions (bench_programs.mm_program
    a_by_rows / a_sectors: permutation views around the staging copy, undone
    on the acceptor side) compute the same product."""
    M, N, K, T, R = 256, 128, 128, 128, 8
    prog = compile_program(mm_program(M, N, K, T, BK, R, a_by_rows=layout == "rows",
                                      a_sectors=layout == "sectors"))
    A = np.random.default_rng(16).integers(-9, 10, (M, K))
    B = np.random.default_rng(17).integers(-9, 10, (K, N))
    got = run_program_cuda(prog, {"A": A, "B": B}, launch=((N // T, M // T), (T // R, T // R)),
                           float_mode=False, flat=True)
    assert np.array_equal(np.asarray(got, np.int64).reshape(M, N), A @ B)


@pytest.mark.parametrize("M,N,K,TM,TN,BK,RM,RN", [(256, 256, 128, 128, 128, 16, 8, 16),
                                                  (256, 256, 64, 128, 128, 8, 16, 8),
                                                  (64, 128, 32, 32, 64, 8, 4, 8)])
def test_mm_rect_strategy_int_exact(M, N, K, TM, TN, BK, RM, RN):
    from paper_1710_08332_b200.bench_programs import mm_rect_program
    prog = compile_program(mm_rect_program(M, N, K, TM, TN, BK, RM, RN))
    A = np.random.default_rng(26).integers(-9, 10, (M, K))
    B = np.random.default_rng(27).integers(-9, 10, (K, N))
    got = run_program_cuda(prog, {"A": A, "B": B}, launch=((N // TN, M // TM), (TN // RN, TM // RM)),
                           float_mode=False, flat=True)
    assert np.array_equal(np.asarray(got, np.int64).reshape(M, N), A @ B)


@pytest.mark.parametrize("variant", ["square", "rows", "sectors", "rect8x16", "rect16x8", "bk8", "rowa"])
def test_mm_variants_fp32(variant):
    """fp32 (the FFMA2 register-tile update, swizzled shared tiles) for every
    mm strategy variant, against a float64 product; bound 1e-4 * sum|terms|."""
    from paper_1710_08332_b200.bench_programs import mm_rect_program
    M, N, K = 256, 256, 512
    if variant == "rowa":
        from paper_1710_08332_b200.bench_programs import mm_rowa_program
        text, launch = mm_rowa_program(M, N, K, 128, 16, 8), ((2, 2), (16, 16))
    elif variant.startswith("rect"):
        RM, RN = (8, 16) if variant == "rect8x16" else (16, 8)
        text, launch = mm_rect_program(M, N, K, 128, 128, 16, RM, RN), ((2, 2), (128 // RN, 128 // RM))
    else:
        text = mm_program(M, N, K, 128, 8 if variant == "bk8" else 16, 8, a_by_rows=variant == "rows",
                          a_sectors=variant == "sectors")
        launch = ((2, 2), (16, 16))
    A = blas_np.seeded((M, K), 31, -1.0, 1.0)
    B = blas_np.seeded((K, N), 32, -1.0, 1.0)
    got = np.asarray(run_program_cuda(compile_program(text), {"A": A, "B": B}, launch=launch,
                                      flat=True)).reshape(M, N)
    want = A.astype(np.float64) @ B.astype(np.float64)
    terms = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64)
    assert np.all(np.abs(got - want) <= 1e-4 * terms)


def test_mm_full_size_fp32():
    cfg = mm_config()
    A = blas_np.seeded((4096, 4096), 5, -1.0, 1.0)
    B = blas_np.seeded((4096, 4096), 6, -1.0, 1.0)
    got = np.asarray(run_program_cuda(compile_program(cfg.text), {"A": A, "B": B}, launch=cfg.launch,
                                      flat=True)).reshape(4096, 4096)
    rows = np.random.default_rng(0).choice(4096, 64, replace=False)
    want, absterms = blas_np.mm(A, B, rows)
    assert blas_np.within(got[rows], want, absterms)


def test_cli_run_device_cuda(tmp_path, capsys):
    """`run --device cuda` on the reference's dot.dpia / dot.inputs prints
    out = 120 (TST/test_cli.py:69-73)."""
    from paper_1710_08332_b200.cli import main
    case = [c for c in GOLDEN if c["name"] == "dot.dpia"][0]
    (tmp_path / "dot.dpia").write_text(case["text"])
    (tmp_path / "dot.inputs").write_text("xs = [1, 2, 3, 4, 5, 6, 7, 8]\nys = [8, 7, 6, 5, 4, 3, 2, 1]\n")
    assert main(["run", str(tmp_path / "dot.dpia"), "--inputs", str(tmp_path / "dot.inputs"),
                 "--device", "cuda", "--launch", "2,4", "--int"]) == 0
    assert "out = 120" in capsys.readouterr().out


HOISTED = [c for c in GOLDEN + FUZZ if c.get("hoisted")]


@pytest.mark.parametrize("case", HOISTED, ids=lambda c: c.get("name") or f"seed{c['seed']}")
def test_reference_hoisted_kernel_form(case):
    """run_kernel accepts the reference's *hoisted* kernel form -- the exact
    input of emit_kernel / simulate_kernel (SRC/opencl.py:124-134, 397) --
    printed by the reference, and computes the reference's result."""
    from paper_1710_08332_b200 import run_kernel
    from paper_1710_08332_b200.reader import ParseError, parse_phrase, parse_phrase_type, read_all
    env = {k: parse_phrase_type(read_all(v)[0]) for k, v in case["hoisted"]["env"].items()}
    try:
        p, _ = parse_phrase(case["hoisted"]["text"], env)
    except ParseError:
        pytest.skip("the reference's printer does not round-trip this vector literal")
    params = [("out", env["out"].data, "out")] + [(k, t.data, "in") for k, t in env.items() if k != "out"]
    inputs = {k: from_json(v) for k, v in case["inputs"].items()}
    fm = case.get("float", False)
    got = run_kernel(p, params, inputs, (2, 2), case.get("sigma", {}), fm, flat=True)["out"]
    # ground truth is the reference's eval_phrase; its simulate_kernel ignores
    # barriers and is wrong for multi-phase local-memory kernels at L > 1
    # (SURVEY.md finding 5) -- e.g. bench.gemv_rowwg, where only the CUDA
    # result agrees with eval_phrase
    want = flatten_value(from_json(case["expected"]))
    if fm:
        assert np.allclose(got, want, rtol=1e-5, atol=1e-5)
    else:
        assert [int(v) for v in got] == want
    if case["simulated_2x2"] != case["expected"]:
        assert case["name"] == "bench.gemv_rowwg"


def test_scal_exact_and_full_size():
    prog = compile_program(scal_program())
    xs = _ints(4096, 9)
    got = run_program_cuda(prog, {"alpha": [3, 3, 3, 3], "xs": xs}, sigma={"n": 1024}, launch=(7, 64),
                           float_mode=False, flat=True)
    assert [int(v) for v in got] == [3 * x for x in xs]
    cfg = scal_config()
    x = blas_np.seeded(1 << 26, 7, -1.0, 1.0)
    got = run_program_cuda(compile_program(cfg.text), {"alpha": np.full(4, 1.5, np.float32), "xs": x},
                           sigma=cfg.sigma, launch=cfg.launch, flat=True)
    assert np.array_equal(np.asarray(got, np.float32), np.float32(1.5) * x)


@pytest.mark.parametrize("launch", [(2, 4), (3, 32)])
@pytest.mark.parametrize("case", [c for c in GOLDEN + FUZZ[:150] if c.get("opencl_legal")],
                         ids=lambda c: c.get("name") or f"seed{c['seed']}")
def test_unspecialised_kernels(case, launch):
    """The generic source (sizes as kernel arguments, geometry only at launch
    -- what `compile --target cuda` writes without --launch) computes the same
    result."""
    from paper_1710_08332_b200 import run_kernel
    prog = compile_program(case["text"])
    inputs = {k: from_json(v) for k, v in case["inputs"].items()}
    fm = case.get("float", False)
    got = run_kernel(prog.imperative, prog.params, inputs, launch, case.get("sigma", {}), fm,
                     flat=True, specialize=False)["out"]
    want = flatten_value(from_json(case["expected"]))
    if fm:
        assert np.allclose(got, want, rtol=1e-5, atol=1e-5)
    else:
        assert [int(v) for v in got] == want


FUZZ_FLOAT = load_golden("fuzz_float.json")


@pytest.mark.parametrize("case", FUZZ_FLOAT, ids=lambda c: f"fseed{c['seed']}")
def test_reference_fuzz_programs_fp32(case):
    """Kernel-legal reference fuzz programs in float mode: the fp32 kernel
    against the reference's float64 result with the normwise bound
    |got - want| <= 1e-5 * sum|terms| per output (sum|terms| propagated by
    oracle.dpia_eval.eval_with_bounds, whose values equal the reference's
    result; input rounding to fp32 alone reaches 6e-8 of the bound)."""
    from oracle.dpia_eval import eval_with_bounds
    prog = compile_program(case["text"])
    inputs = {k: from_json(v) for k, v in case["inputs"].items()}
    got = np.asarray(run_program_cuda(prog, inputs, launch=(2, 4), float_mode=True, flat=True),
                     np.float64)
    want = np.asarray(flatten_value(from_json(case["expected"])), np.float64)
    vals, bounds = eval_with_bounds(prog.source.body, inputs, {})
    assert np.allclose(vals, want, rtol=1e-12, atol=1e-12)
    assert np.all(np.abs(got - want) <= 1e-5 * np.asarray(bounds, np.float64)), (got, want, bounds)


def test_executable_run_pinned_repeated():
    """Executable.run (the end-to-end call bench.py's e2e leg times): inputs
    from page-locked host memory, result into page-locked host memory, same
    answers on every repetition (the fused grid combine resets its counter)."""
    from paper_1710_08332_b200 import executable
    from paper_1710_08332_b200 import runtime as RT
    cfg = dot_config(N=1 << 20, L=256, K=16)
    exe = executable(compile_program(cfg.text), cfg.launch, cfg.sigma, float_mode=True)
    st = RT.Stream(0)
    bufs = [RT.PinnedBuffer(4 << 20) for _ in range(2)] + [RT.PinnedBuffer(16)]
    xs, ys = bufs[0].array(np.float32, 1 << 20), bufs[1].array(np.float32, 1 << 20)
    out = {"out": bufs[2].array(np.float32, 1)}
    try:
        for seed in range(3):
            xs[:] = blas_np.seeded(1 << 20, 10 + seed, 0.0, 1.0)
            ys[:] = blas_np.seeded(1 << 20, 20 + seed, 0.0, 1.0)
            res = exe.run({"xs": xs, "ys": ys}, st, out=out)
            want, absterms = blas_np.dot(np.array(xs), np.array(ys))
            assert res["out"] is out["out"]
            assert blas_np.within(float(res["out"][0]), want, absterms)
        # int mode, pageable numpy inputs, result allocated by run()
        ie = executable(compile_program(cfg.text), cfg.launch, cfg.sigma, float_mode=False)
        a, b = _ints(1 << 20, 3), _ints(1 << 20, 4)
        for _ in range(2):
            got = ie.run({"xs": np.asarray(a), "ys": np.asarray(b)}, st)
            assert int(got["out"][0]) == int(np.dot(np.asarray(a, np.int64), np.asarray(b, np.int64)))
    finally:
        for b_ in bufs:
            b_.free()


@pytest.mark.parametrize("launch", [(1, 32), (3, 64)])
def test_empty_inputs(launch):
    """n = 0: a map yields the empty array and every reduction its initial
    value, as the reference's interpreter does (eval_fn over empty lists)."""
    sq = ("(nat n)\n(param xs (exp (array (* n 4) num)))\n"
          "(join (mapGlobal (lam (c (exp (array 4 num))) (mapSeq (lam (x (exp num)) (* x x)) c)) (split 4 xs)))")
    cases = [(sq, {"xs": []}), (dot_program(32, 2), {"xs": [], "ys": []}), (asum_program(32, 2), {"xs": []})]
    for text, inputs in cases:
        prog = compile_program(text)
        want = flatten_value(eval_phrase(prog.source.body, inputs, {"n": 0}))
        for fm in (False, True):
            got = run_program_cuda(prog, inputs, sigma={"n": 0}, launch=launch, float_mode=fm, flat=True)
            assert [float(v) for v in np.atleast_1d(got)] == [float(v) for v in want], (text, fm)


@pytest.mark.parametrize("rows,cols,streams", [(1, 1, 1), (2, 2, 1), (2, 2, 4), (4, 2, 3), (1, 2, 2)])
def test_mm_tile_pipeline_matches_unchunked(rows, cols, streams):
    """pipeline.TilePipeline (row blocks of A, pitched column panels of B,
    tile kernels on several streams, pitched D2H of C tiles) is bit-identical
    to one launch of the whole product."""
    from paper_1710_08332_b200 import runtime as RT
    from paper_1710_08332_b200.bench_programs import mm_config
    from paper_1710_08332_b200.pipeline import mm_tile_pipeline
    M, N, K = 512, 256, 384
    A = blas_np.seeded((M, K), 53, -1.0, 1.0)
    B = blas_np.seeded((K, N), 54, -1.0, 1.0)
    cfg = mm_config(M=M, N=N, K=K)
    whole = np.asarray(run_program_cuda(compile_program(cfg.text), {"A": A, "B": B},
                                        launch=cfg.launch, flat=True), np.float32)
    pins = [RT.PinnedBuffer(a.nbytes) for a in (A, B)] + [RT.PinnedBuffer(4 * M * N)]
    try:
        ha, hb = pins[0].array(np.float32, A.size), pins[1].array(np.float32, B.size)
        ha[:], hb[:] = A.ravel(), B.ravel()
        out = pins[2].array(np.float32, M * N)
        pipe = mm_tile_pipeline(M, N, K, rows=rows, cols=cols, compute_streams=streams)
        for _ in range(2):
            out[:] = np.nan
            pipe.run({"A": ha, "B": hb}, out, RT.Stream(0))
            assert np.array_equal(out, whole)
    finally:
        for p in pins:
            p.free()


@pytest.mark.parametrize("chunks", [1, 2, 8])
def test_scal_pipeline_matches_unchunked(chunks):
    """pipeline.scal_pipeline (blocks of x / y, H2D, kernels and D2H on their
    own streams) is bit-identical to one launch over the whole vector."""
    from paper_1710_08332_b200 import runtime as RT
    from paper_1710_08332_b200.bench_programs import scal_config
    from paper_1710_08332_b200.pipeline import scal_pipeline
    N = 1 << 16
    xs = blas_np.seeded(N, 57, -1.0, 1.0)
    alpha = np.full(4, 1.25, np.float32)
    cfg = scal_config(N=N)
    whole = np.asarray(run_program_cuda(compile_program(cfg.text), {"alpha": alpha, "xs": xs},
                                        sigma=cfg.sigma, launch=cfg.launch, flat=True), np.float32)
    pins = [RT.PinnedBuffer(16), RT.PinnedBuffer(4 * N), RT.PinnedBuffer(4 * N)]
    try:
        ha, hx, out = (pins[0].array(np.float32, 4), pins[1].array(np.float32, N),
                       pins[2].array(np.float32, N))
        ha[:], hx[:] = alpha, xs
        pipe = scal_pipeline(N, chunks=chunks)
        for _ in range(2):
            out[:] = np.nan
            pipe.run({"alpha": ha, "xs": hx}, out, RT.Stream(0))
            assert np.array_equal(out, whole)
    finally:
        for p in pins:
            p.free()


def test_mm_tile_pipeline_int64_matches_oracle():
    """int mode (int64 elements, 8-byte pitches): the tiled product equals
    numpy's exact integer product."""
    from paper_1710_08332_b200 import runtime as RT
    from paper_1710_08332_b200.pipeline import mm_tile_pipeline
    M, N, K = 256, 256, 128
    rng = np.random.default_rng(55)
    A = rng.integers(-9, 10, (M, K)).astype(np.int64)
    B = rng.integers(-9, 10, (K, N)).astype(np.int64)
    pins = [RT.PinnedBuffer(a.nbytes) for a in (A, B)] + [RT.PinnedBuffer(8 * M * N)]
    try:
        ha, hb = pins[0].array(np.int64, A.size), pins[1].array(np.int64, B.size)
        ha[:], hb[:] = A.ravel(), B.ravel()
        out = pins[2].array(np.int64, M * N)
        pipe = mm_tile_pipeline(M, N, K, rows=2, cols=2, compute_streams=2, float_mode=False)
        pipe.run({"A": ha, "B": hb}, out, RT.Stream(0))
        assert np.array_equal(out.reshape(M, N), A @ B)
    finally:
        for p in pins:
            p.free()


@pytest.mark.parametrize("chunks", [1, 2, 4])
def test_mm_row_pipeline_matches_unchunked(chunks):
    """pipeline.RowPipeline (row chunks of A / C, copies on their own streams
    overlapped with the chunk kernels) is bit-identical to one launch of the
    whole product."""
    from paper_1710_08332_b200 import runtime as RT
    from paper_1710_08332_b200.bench_programs import mm_config
    from paper_1710_08332_b200.pipeline import mm_pipeline
    M, N, K = 512, 256, 384
    A = blas_np.seeded((M, K), 51, -1.0, 1.0)
    B = blas_np.seeded((K, N), 52, -1.0, 1.0)
    pins = [RT.PinnedBuffer(a.nbytes) for a in (A, B)] + [RT.PinnedBuffer(4 * M * N)]
    try:
        ha, hb = pins[0].array(np.float32, A.size), pins[1].array(np.float32, B.size)
        ha[:], hb[:] = A.ravel(), B.ravel()
        out = pins[2].array(np.float32, M * N)
        pipe = mm_pipeline(M, N, K, chunks=chunks)
        for _ in range(2):
            out[:] = 0
            pipe.run({"A": ha, "B": hb}, out, RT.Stream(0))
            cfg = mm_config(M=M, N=N, K=K)
            whole = np.asarray(run_program_cuda(compile_program(cfg.text), {"A": A, "B": B},
                                                launch=cfg.launch, flat=True), np.float32)
            assert np.array_equal(out, whole)
    finally:
        for p in pins:
            p.free()


VEC_FOLDS = [
    # per-item chunks read at unit stride: vectorised (chunk a multiple of 4, > 64)
    ("(nat n)\n(param xs (exp (array (* n 256) num)))\n"
     "(mapGlobal (lam (c (exp (array 256 num))) (reduce (lam (x (exp num)) (lam (a (exp num)) "
     "(+ a (* x x)))) 0 c)) (split 256 xs))", {"n": 12}, 256),
    # the same with a chunk that is not a multiple of 4: scalar loads
    ("(nat n)\n(param xs (exp (array (* n 130) num)))\n"
     "(mapGlobal (lam (c (exp (array 130 num))) (reduce (lam (x (exp num)) (lam (a (exp num)) "
     "(- a x))) 0 c)) (split 130 xs))", {"n": 9}, 130),
    # a strided (transposed) chunk: no vector loads
    ("(nat n)\n(param xs (exp (array (* n 128) num)))\n"
     "(mapGlobal (lam (c (exp (array 128 num))) (reduce (lam (x (exp num)) (lam (a (exp num)) "
     "(- x a))) 0 c)) (transpose (split n xs)))", {"n": 16}, 128),
]


@pytest.mark.parametrize("text,sigma,chunk", VEC_FOLDS)
@pytest.mark.parametrize("launch", [(1, 32), (3, 8)])
def test_vectorised_sequential_folds(text, sigma, chunk, launch):
    """KernelEmitter._vec_loop: long per-item folds read their chunk as
    4-wide vectors, in the original order -- int mode bit-exact against the
    oracle for vectorised, non-multiple-of-4 and strided chunks, and the
    literal config-1 program with its vectorised single-thread tail."""
    prog = compile_program(text)
    n = sigma["n"]
    xs = _ints(n * chunk, 21)
    want = flatten_value(eval_phrase(prog.source.body, {"xs": xs}, sigma))
    got = run_program_cuda(prog, {"xs": xs}, sigma=sigma, launch=launch, float_mode=False, flat=True)
    assert [int(v) for v in got] == want


def test_literal_dot_vectorised_int_exact():
    from paper_1710_08332_b200.bench_programs import dot_literal_program
    prog = compile_program(dot_literal_program(256))
    xs, ys = _ints(64 * 256, 5), _ints(64 * 256, 6)
    for launch in ((2, 32), (64, 1), (1, 1)):
        got = run_program_cuda(prog, {"xs": xs, "ys": ys}, sigma={"n": 64}, launch=launch, float_mode=False)
        assert got == eval_phrase(prog.source.body, {"xs": xs, "ys": ys}, {"n": 64})
