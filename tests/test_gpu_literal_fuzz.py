"""GPU fuzz of the reference-runnable reduction shape (config 1's literal
program and its relatives): `reduce (+) 0 (mapGlobal (lam c (reduce F 0 c))
(split C xs...))` over random chunk sizes, item counts, launch geometries
(1..8 rounds of work-items) and fold bodies.  These are the programs the
TMA row folds (`KernelEmitter._finish_rows`) and the parity-pipelined
streaming tail (`ProgramEmitter._stream_plan`) apply to.

fp32: the default emission must give the bits of the plain lowering (register
loads, last-block ticket tail) -- the same fold order; int64: exact against
NumPy.  Several launches per program, some chained.
"""
import numpy as np
import pytest

from paper_1710_08332_b200 import compile_program, executable
from paper_1710_08332_b200.cuda import emit as EM

pytestmark = pytest.mark.gpu

BODIES = {
    # name: (inputs, fold body over element x and accumulator a, numpy reference of one chunk)
    "dot": (2, "(+ (* (fst x) (snd x)) a)", lambda xs, ys: xs * ys),
    "sum": (1, "(+ x a)", lambda xs, ys: xs),
    "sumsq": (1, "(+ a (* x x))", lambda xs, ys: xs * xs),
    "diff": (2, "(+ a (- (fst x) (snd x)))", lambda xs, ys: xs - ys),
}


def program(body: str, chunk: int) -> str:
    k, f, _ = BODIES[body]
    if k == 2:
        return (f"(nat n)\n(param xs (exp (array (* n {chunk}) num)))\n(param ys (exp (array (* n {chunk}) num)))\n"
                f"(reduce (+) 0 (mapGlobal (lam (c (exp (array {chunk} (pair num num))))"
                f" (reduce (lam (x (exp (pair num num))) (lam (a (exp num)) {f})) 0 c))"
                f" (split {chunk} (zip xs ys))))")
    return (f"(nat n)\n(param xs (exp (array (* n {chunk}) num)))\n"
            f"(reduce (+) 0 (mapGlobal (lam (c (exp (array {chunk} num)))"
            f" (reduce (lam (x (exp num)) (lam (a (exp num)) {f})) 0 c))"
            f" (split {chunk} xs)))")


def cases():
    rng = np.random.default_rng(2026)
    out = []
    for seed in range(24):
        body = list(BODIES)[seed % len(BODIES)]
        chunk = int(rng.choice([128, 256, 512, 1024, 2048]))
        L = int(rng.choice([32, 64, 128]))
        rounds = int(rng.choice([1, 2, 3, 4, 8]))
        G = int(rng.integers(1, 5))
        n = G * L * rounds
        while n * chunk > (1 << 22):
            G, n = max(1, G // 2), max(1, G // 2) * L * rounds
            if G == 1:
                break
        out.append((seed, body, chunk, n, (G, L)))
    return out


def _build(text, n, launch, fm, plain):
    old = EM.ROW_TMA, EM.STREAM_TAIL
    if plain:
        EM.ROW_TMA, EM.STREAM_TAIL = False, False
    try:
        return executable(compile_program(text), launch, {"n": n}, float_mode=fm)
    finally:
        EM.ROW_TMA, EM.STREAM_TAIL = old


def _run(exe, inputs, launches=3):
    from paper_1710_08332_b200 import runtime as RT
    st = RT.Stream(0)
    for nm, v in inputs.items():
        exe.upload(nm, v, st)
    vals = []
    for k in range(launches):
        exe.launch(st, chain=k > 0)
        vals.append(np.asarray(exe.download("out", st)).copy())
    st.sync()
    return vals


@pytest.mark.parametrize("seed,body,chunk,n,launch", cases())
def test_literal_shape_fp32_bits(seed, body, chunk, n, launch):
    k, _f, ref = BODIES[body]
    rng = np.random.default_rng(seed)
    names = ["xs", "ys"][:k]
    inputs = {nm: rng.uniform(-1, 1, n * chunk).astype(np.float32) for nm in names}
    text = program(body, chunk)
    fast = _build(text, n, launch, True, plain=False)
    plain = _build(text, n, launch, True, plain=True)
    a, b = _run(fast, inputs), _run(plain, inputs, 1)
    assert all(v.view(np.uint32)[0] == b[0].view(np.uint32)[0] for v in a), (a, b)
    x = inputs["xs"].astype(np.float64)
    y = inputs["ys"].astype(np.float64) if k == 2 else None
    want = float(np.sum(ref(x, y)))
    terms = float(np.sum(np.abs(ref(x, y)))) + 1.0
    assert abs(float(a[0][0]) - want) <= 1e-4 * terms


@pytest.mark.parametrize("seed,body,chunk,n,launch", cases()[:12])
def test_literal_shape_int_exact(seed, body, chunk, n, launch):
    k, _f, ref = BODIES[body]
    rng = np.random.default_rng(seed + 100)
    names = ["xs", "ys"][:k]
    inputs = {nm: rng.integers(-9, 10, n * chunk) for nm in names}
    exe = _build(program(body, chunk), n, launch, False, plain=False)
    vals = _run(exe, inputs)
    want = int(np.sum(ref(inputs["xs"], inputs.get("ys"))))
    assert all(int(v[0]) == want for v in vals)


MAPS = {
    # name: (fold body over element x, numpy of it): a work-item writes its own piece
    "scale": ("(* alpha x)", lambda x, a: np.float32(a) * x),
    "double": ("(+ x x)", lambda x, a: x + x),
    # contracted to one FMA on the GPU: one rounding of the exact a x + x
    "axpx": ("(+ (* alpha x) x)", lambda x, a: (np.float64(a) * x.astype(np.float64) + x)),
}


def map_program(body: str, chunk: int) -> str:
    return (f"(nat n)\n(param alpha (exp num))\n(param xs (exp (array (* n {chunk}) num)))\n"
            f"(join (mapGlobal (lam (c (exp (array {chunk} num))) (mapSeq (lam x {MAPS[body][0]}) c))"
            f" (split {chunk} xs)))")


def map_cases():
    rng = np.random.default_rng(77)
    out = []
    for seed in range(18):
        body = list(MAPS)[seed % len(MAPS)]
        chunk = int(rng.choice([128, 256, 1024, 2048]))
        L = int(rng.choice([32, 64]))
        rounds = int(rng.choice([1, 2, 4]))
        G = int(rng.integers(1, 9))
        out.append((seed, body, chunk, G * L * rounds, (G, L)))
    return out


@pytest.mark.parametrize("seed,body,chunk,n,launch", map_cases())
def test_literal_map_shape_fp32_exact(seed, body, chunk, n, launch):
    """Work-items writing their own contiguous pieces (the reference's scal
    shape): TMA row reads, merged vector stores leaving as TMA row stores,
    several launches chained -- exact against numpy (one rounding per element
    and the same operation order)."""
    rng = np.random.default_rng(seed)
    xs = rng.uniform(-1, 1, n * chunk).astype(np.float32)
    exe = executable(compile_program(map_program(body, chunk)), launch, {"n": n}, float_mode=True)
    from paper_1710_08332_b200 import runtime as RT
    st = RT.Stream(0)
    exe.upload("alpha", np.float32([1.25]), st)
    exe.upload("xs", xs, st)
    for k in range(3):
        exe.launch(st, chain=k > 0)
    got = np.asarray(exe.download("out", st))
    st.sync()
    want = MAPS[body][1](xs, 1.25).astype(np.float32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_strided_piece_stores_exact():
    """A work-item writing its piece through a layout view (every second
    element): scalar stores, exact against numpy."""
    text = ("(nat n)\n(param xs (exp (array (* n 256) num)))\n"
            "(join (mapGlobal (lam (c (exp (array 256 num)))"
            " (join (transpose (split 128 (mapSeq (lam x (* x x)) c))))) (split 256 xs)))")
    xs = np.random.default_rng(9).uniform(-1, 1, 64 * 256).astype(np.float32)
    exe = executable(compile_program(text), (2, 32), {"n": 64}, float_mode=True)
    from paper_1710_08332_b200 import runtime as RT
    st = RT.Stream(0)
    exe.upload("xs", xs, st)
    exe.launch(st)
    got = np.asarray(exe.download("out", st))
    st.sync()
    want = (xs * xs).reshape(64, 2, 128).transpose(0, 2, 1).reshape(-1)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
