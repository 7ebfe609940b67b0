"""CPU checks of the backend's execution plan with the barrier-aware
phase-synchronous simulator (oracle/phase_sim.py): every planned kernel
computes the reference result, with no intra-phase or cross-work-group
conflicts; removing the planned barriers is caught."""
import pytest

from conftest import load_golden
from oracle.dpia_eval import eval_phrase, flatten_value, from_json
from oracle.phase_sim import PhaseRace, Sim, simulate
from paper_1710_08332_b200 import compile_program
from paper_1710_08332_b200.bench_programs import (asum_program, dot_program, gemv_program,
                                                  mm_program, mm_rect_program, mm_rowa_program)

GOLDEN = load_golden("programs.json")
FUZZ_LEGAL = [c for c in load_golden("fuzz.json") if c["reparses"] and c["opencl_legal"]][:60]


@pytest.mark.parametrize("launch", [(1, 1), (2, 2), (2, 4), (3, 8)])
@pytest.mark.parametrize("case", [c for c in GOLDEN if not c.get("float")], ids=lambda c: c["name"])
def test_golden_programs_phase_exact(case, launch):
    prog = compile_program(case["text"])
    inputs = {k: from_json(v) for k, v in case["inputs"].items()}
    out = simulate(prog.imperative, prog.params, inputs, launch, case.get("sigma", {}))
    assert flatten_value(out["out"]) == flatten_value(from_json(case["expected"]))


@pytest.mark.parametrize("case", FUZZ_LEGAL, ids=lambda c: f"seed{c['seed']}")
def test_reference_fuzz_kernels_phase_exact(case):
    prog = compile_program(case["text"])
    inputs = {k: from_json(v) for k, v in case["inputs"].items()}
    out = simulate(prog.imperative, prog.params, inputs, (2, 4), {})
    assert flatten_value(out["out"]) == flatten_value(from_json(case["expected"]))


def _ints(n, a):
    return [((a * i + 3) % 19) - 9 for i in range(n)]


STRATS = [
    ("dot", dot_program(32, 2), {"n": 2}, (2, 32),
     lambda: {"xs": _ints(512, 5), "ys": _ints(512, 7)}),
    ("asum", asum_program(32, 2), {"n": 2}, (3, 32), lambda: {"xs": _ints(512, 3)}),
    ("gemv", gemv_program(3, 256, 32), {}, (2, 32),
     lambda: {"A": [_ints(256, 3 + r) for r in range(3)], "x": _ints(256, 11)}),
    ("gemv_xpriv", gemv_program(3, 256, 32, x_private=True), {}, (2, 32),
     lambda: {"A": [_ints(256, 3 + r) for r in range(3)], "x": _ints(256, 11)}),
    ("mm", mm_program(16, 16, 16, 8, 4, 4), {}, ((2, 2), (2, 2)),
     lambda: {"A": [_ints(16, 3 + r) for r in range(16)], "B": [_ints(16, 5 + r) for r in range(16)]}),
    # one vec4 staging load per work-item: the k-loop is software-pipelined
    # and its shared tiles rotate between two slices (one barrier per k-step)
    ("mm_pipelined", mm_program(16, 16, 16, 8, 2, 4), {}, ((2, 2), (2, 2)),
     lambda: {"A": [_ints(16, 3 + r) for r in range(16)], "B": [_ints(16, 5 + r) for r in range(16)]}),
    # alternative A-tile distributions (permutation views around the copy)
    ("mm_a_rows", mm_program(32, 32, 32, 16, 16, 4, a_by_rows=True), {}, ((2, 2), (4, 4)),
     lambda: {"A": [_ints(32, 3 + r) for r in range(32)], "B": [_ints(32, 5 + r) for r in range(32)]}),
    ("mm_a_sectors", mm_program(32, 32, 32, 16, 16, 4, a_sectors=True), {}, ((2, 2), (4, 4)),
     lambda: {"A": [_ints(32, 3 + r) for r in range(32)], "B": [_ints(32, 5 + r) for r in range(32)]}),
    # rectangular output and register tiles (8 x 16 tile, 2 x 8 register tiles)
    ("mm_rect", mm_rect_program(16, 32, 16, 8, 16, 4, 2, 8), {}, ((2, 2), (2, 4)),
     lambda: {"A": [_ints(16, 3 + r) for r in range(16)], "B": [_ints(32, 5 + r) for r in range(16)]}),
    # row-major A tile, k-quad micro-kernel over a transposed accumulator view
    ("mm_rowa", mm_rowa_program(32, 32, 32, 16, 8, 4), {}, ((2, 2), (4, 4)),
     lambda: {"A": [_ints(32, 3 + r) for r in range(32)], "B": [_ints(32, 5 + r) for r in range(32)]}),
]


@pytest.mark.parametrize("name,text,sigma,launch,mk", STRATS, ids=[s[0] for s in STRATS])
def test_benchmark_strategies_phase_exact(name, text, sigma, launch, mk):
    prog = compile_program(text)
    inputs = mk()
    out = simulate(prog.imperative, prog.params, inputs, launch, sigma)
    want = eval_phrase(prog.source.body, inputs, sigma)
    assert flatten_value(out["out"]) == flatten_value(want)


@pytest.mark.parametrize("name,text,sigma,launch,mk",
                         [s for s in STRATS if s[0] in ("gemv", "mm", "mm_pipelined")],
                         ids=["gemv", "mm", "mm_pipelined"])
def test_missing_barriers_are_detected(name, text, sigma, launch, mk):
    prog = compile_program(text)
    sim = Sim(prog.imperative, prog.params, mk(), launch, sigma)
    assert any(k.barriers or k.hoisted for k in sim.sig.kernels)
    for k in sim.sig.kernels:
        k.barriers = frozenset()
        k.hoisted = frozenset()
        k.rotated = {}
    with pytest.raises(PhaseRace):
        sim.run()


def test_pipelined_mm_rotates_and_needs_one_barrier_per_k_step():
    prog = compile_program(mm_program(16, 16, 16, 8, 2, 4))
    sim = Sim(prog.imperative, prog.params, STRATS[-1][4](), ((2, 2), (2, 2)))
    (k,) = sim.sig.kernels
    assert len(k.rotated) == 2
    # rotation without the planned barrier before the compute is a race
    sim.sig.kernels[0].barriers = frozenset()
    with pytest.raises(PhaseRace):
        sim.run()
