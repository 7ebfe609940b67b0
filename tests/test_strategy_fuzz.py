"""Differential fuzzing of the CUDA backend on random hierarchical strategy
programs (tests/strategy_gen.py) -- SURVEY.md 8f row f2 extended to the
primitives the reference's fuzzer never generates.  Oracle: the eval_phrase
restatement (pinned to the reference's golden vectors); int mode, exact."""
import pytest

from oracle.dpia_eval import eval_phrase, flatten_value
from oracle.phase_sim import simulate
from paper_1710_08332_b200 import compile_program
from strategy_gen import generate, generate2d


def _case(seed):
    text, inputs, sigma, launch, desc = generate(seed)
    prog = compile_program(text)
    want = flatten_value(eval_phrase(prog.source.body, inputs, sigma))
    return prog, inputs, sigma, launch, want


@pytest.mark.parametrize("seed", range(200))
def test_strategy_fuzz_phase_simulator(seed):
    prog, inputs, sigma, launch, want = _case(seed)
    got = simulate(prog.imperative, prog.params, inputs, launch, sigma)["out"]
    assert flatten_value(got) == want


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(400))
def test_strategy_fuzz_gpu(seed):
    from paper_1710_08332_b200 import run_program_cuda
    prog, inputs, sigma, launch, want = _case(seed)
    got = run_program_cuda(prog, inputs, sigma=sigma, launch=launch, float_mode=False, flat=True)
    assert [int(v) for v in got] == want


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(400))
def test_strategy_fuzz_gpu_fp32(seed):
    """The same programs in float mode: the values are small integers, so
    every fp32 sum and product is exact and the oracle's integer result must
    come back bit-exact -- this covers the float-only code paths (packed
    FFMA2 register updates, swizzled shared tiles) on every generated shape."""
    from paper_1710_08332_b200 import run_program_cuda
    prog, inputs, sigma, launch, want = _case(seed)
    got = run_program_cuda(prog, inputs, sigma=sigma, launch=launch, float_mode=True, flat=True)
    assert [float(v) for v in got] == [float(v) for v in want]


@pytest.mark.gpu
def test_strategy_fuzz_fp32_beyond_exact_range():
    """Seed 5487 of the long campaign cubes products of products (|values|
    up to 2e9 > 2^24): int mode stays exact; fp32 rounds, and every element
    is within 2^-20 relative of the exact value (fuzz_campaign.same_values)."""
    from fuzz_campaign import same_values
    from paper_1710_08332_b200 import run_program_cuda
    prog, inputs, sigma, launch, want = _case(5487)
    assert max(abs(w) for w in want) > 1 << 24
    got = run_program_cuda(prog, inputs, sigma=sigma, launch=launch, float_mode=False, flat=True)
    assert [int(v) for v in got] == want
    got = run_program_cuda(prog, inputs, sigma=sigma, launch=launch, float_mode=True, flat=True)
    assert same_values([float(v) for v in got], [float(v) for v in want], True)


def _case2d(seed):
    text, inputs, sigma, launch, desc = generate2d(seed)
    prog = compile_program(text)
    want = flatten_value(eval_phrase(prog.source.body, inputs, sigma))
    return prog, inputs, sigma, launch, want


@pytest.mark.parametrize("seed", range(60))
def test_strategy_fuzz2d_phase_simulator(seed):
    prog, inputs, sigma, launch, want = _case2d(seed)
    got = simulate(prog.imperative, prog.params, inputs, launch, sigma)["out"]
    assert flatten_value(got) == want


@pytest.mark.gpu
@pytest.mark.parametrize("float_mode", [False, True])
@pytest.mark.parametrize("seed", range(150))
def test_strategy_fuzz2d_gpu(seed, float_mode):
    """2-D hierarchy (tiled transposes through swizzled shared tiles), exact
    in int and fp32 (small-integer values)."""
    from paper_1710_08332_b200 import run_program_cuda
    prog, inputs, sigma, launch, want = _case2d(seed)
    got = run_program_cuda(prog, inputs, sigma=sigma, launch=launch, float_mode=float_mode, flat=True)
    assert [float(v) for v in got] == [float(v) for v in want]
