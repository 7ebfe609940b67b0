"""Acceptor and view laws through the whole backend: each program writes
its result through one of the acceptor duals the translation introduces
(joinAcc, splitAcc, asScalarAcc, transposeAcc, zipAcc, pairAcc, staged
toLocal / toPrivate copies) or reads through the matching view, and must
equal the functional oracle -- the backend-level analogue of the
reference's translation equivalences (TST/test_equiv.py: mapI is the
assignment of map, join/split/zip/pair/vector acceptors agree with their
views, temporary storage is unobservable).  CPU: the phase-synchronous
simulator of the emitted plan; GPU: the emitted kernels, int64 and fp32."""
import numpy as np
import pytest

from oracle.dpia_eval import eval_phrase, flatten_value
from oracle.phase_sim import simulate
from paper_1710_08332_b200 import compile_program

HEAD = "(nat n)\n(param xs (exp (array (* n 8) num)))\n(param ys (exp (array (* n 8) num)))\n"
LAWS = {
    "join_of_split": "(join (mapWorkgroup (lam (r (exp (array 8 num))) (mapLocal (lam x (* x 3)) r)) (split 8 xs)))",
    "scalar_of_vector": "(asScalar4 (mapGlobal (lam (v (exp (vec 4))) (+ v (* v v))) (asVector4 xs)))",
    "zip_projections": "(mapGlobal (lam (p (exp (pair num num))) (- (* 2 (fst p)) (snd p))) (zip xs ys))",
    "transposed_input": "(join (mapWorkgroup (lam (r (exp (array 8 num))) (mapLocal (lam x (+ x 1)) r))"
                        " (transpose (split n xs))))",
    "transposed_output": "(transpose (mapWorkgroup (lam (r (exp (array 8 num))) (mapLocal (lam x (- x 4)) r))"
                         " (split 8 xs)))",
    "transpose_twice": "(join (transpose (transpose (mapWorkgroup (lam (r (exp (array 8 num)))"
                       " (mapLocal (lam x (* x x)) r)) (split 8 xs)))))",
    "nested_split": "(join (join (mapWorkgroup (lam (r (exp (array 8 num))) (mapLocal (lam (q (exp (array 2 num)))"
                    " (mapSeq (lam x (+ x 7)) q)) (split 2 r))) (split 8 xs))))",
    "vector_zip": "(asScalar4 (mapGlobal (lam (p (exp (pair (vec 4) (vec 4)))) (* (fst p) (snd p)))"
                  " (zip (asVector4 xs) (asVector4 ys))))",
    "pair_of_reductions": "(pair (reduce (+) 0 xs) (reduce (+) 0 ys))",
    "local_temporary": "(join (mapWorkgroup (lam (r (exp (array 8 num))) (mapLocal (lam x (* x 2))"
                       " (toLocal (mapLocal (lam y (+ y 1))) r))) (split 8 xs)))",
    "private_temporary": "(join (mapWorkgroup (lam (r (exp (array 8 num))) (mapLocal (lam x (- x 1))"
                         " (toPrivate (mapLocal (lam y (* y 3))) r))) (split 8 xs)))",
    "zip_of_splits": "(join (mapWorkgroup (lam (p (exp (pair (array 8 num) (array 8 num))))"
                     " (mapLocal (lam q (+ (fst q) (snd q))) (zip (fst p) (snd p))))"
                     " (zip (split 8 xs) (split 8 ys))))",
}
LAUNCHES = [(1, 1), (2, 4), (3, 8), (4, 32)]


def _case(name, n=4, seed=1):
    prog = compile_program(HEAD + LAWS[name])
    rng = np.random.default_rng(seed)
    inputs = {"xs": rng.integers(-9, 10, 8 * n).tolist(), "ys": rng.integers(-9, 10, 8 * n).tolist()}
    return prog, inputs, {"n": n}, flatten_value(eval_phrase(prog.source.body, inputs, {"n": n}))


@pytest.mark.parametrize("launch", LAUNCHES)
@pytest.mark.parametrize("name", sorted(LAWS))
def test_view_law_phase_simulator(name, launch):
    prog, inputs, sigma, want = _case(name)
    got = simulate(prog.imperative, prog.params, inputs, launch, sigma)["out"]
    assert flatten_value(got) == want


@pytest.mark.gpu
@pytest.mark.parametrize("launch", LAUNCHES)
@pytest.mark.parametrize("name", sorted(LAWS))
def test_view_law_gpu(name, launch):
    from paper_1710_08332_b200 import run_program_cuda
    prog, inputs, sigma, want = _case(name, n=6, seed=2)
    for fm in (False, True):   # small integers: fp32 is exact too
        got = run_program_cuda(prog, inputs, sigma=sigma, launch=launch, float_mode=fm, flat=True)
        assert [float(v) for v in got] == [float(v) for v in want], fm
