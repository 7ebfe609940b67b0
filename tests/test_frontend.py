"""Front end (reader/elaborator, Stage I, Stage II) against the reference's
golden outputs: the functional oracle and the imperative interpreter must
both reproduce the reference's eval_phrase result (reference tests
TST/test_translate.py:47-55, TST/test_lower.py:192-197)."""
import pytest

from conftest import load_golden
from oracle.dpia_eval import eval_phrase, from_json, to_json
from oracle.imp_eval import RaceError, run_program
from paper_1710_08332_b200.dtypes import AccT, Array, Num, array
from paper_1710_08332_b200.reader import ElabError, ParseError, parse, parse_phrase
from paper_1710_08332_b200.sizes import nat
from paper_1710_08332_b200.stage1 import translate_program
from paper_1710_08332_b200.stage2 import is_purely_imperative, stage2
from paper_1710_08332_b200.terms import Prim, subtree_iter

CASES = load_golden("programs.json") + load_golden("fuzz.json")


def _id(c):
    return c.get("name") or f"fuzz{c['seed']}"


@pytest.mark.parametrize("case", CASES, ids=_id)
def test_parse_and_eval_match_reference(case):
    if not case.get("reparses", True):
        # the reference's own parser rejects its printer's output here
        with pytest.raises(ElabError):
            parse(case["text"])
        return
    sp = parse(case["text"])
    got = eval_phrase(sp.body, {k: from_json(v) for k, v in case["inputs"].items()},
                      case.get("sigma", {}))
    assert to_json(got) == case["expected"]


def _count(p, names):
    return sum(1 for s in subtree_iter(p) if isinstance(s, Prim) and s.name in names)


@pytest.mark.parametrize("case", [c for c in CASES if c.get("reparses", True)][::3], ids=_id)
def test_stage2_coincidence(case):
    sp = parse(case["text"])
    inputs = {k: from_json(v) for k, v in case["inputs"].items()}
    params = [("out", sp.body_type.data, "out")] + [(k, t.data, "in") for k, t in sp.params]
    for space, acc in ((None, None), ("global", "private")):
        s1 = translate_program(sp.body, sp.body_type.data, "out", space)
        # strategy preservation: one intermediate per source combinator
        for src, tgt in (("mapGlobal", "mapIGlobal"), ("mapWorkgroup", "mapIWorkgroup"),
                         ("mapLocal", "mapILocal"), ("mapSeq", "mapISeq")):
            assert _count(sp.body, {src}) == _count(s1, {tgt})
        assert _count(sp.body, {"reduce"}) == _count(s1, {"reduceI", "reduceIInit"})
        s2 = stage2(s1, acc)
        assert is_purely_imperative(s2)
        for rev in (False, True):
            out = run_program(s2, params, inputs, case.get("sigma", {}), case.get("float", False), rev)
            assert to_json(out["out"]) == case["expected"]


def test_dot_file_answer():
    case = [c for c in CASES if c.get("name") == "dot.dpia"][0]
    assert case["expected"] == 120  # TST/test_cli.py:69-73


def test_parse_errors_and_type_errors():
    with pytest.raises(ParseError):
        parse("(param xs (exp (array 4 num))) (map")
    with pytest.raises(ElabError):
        parse("(param xs (exp (array 4 num)))\n(zip xs (split 2 xs))")
    with pytest.raises(ParseError):
        parse("(param xs (exp (array 4 num)))")


def test_transpose_and_abs_additions():
    src = ("(param m (exp (array 2 (array 3 num))))\n"
           "(map (lam (r (exp (array 2 num))) (reduce (lam (x (exp num)) (lam (a (exp num))"
           " (+ (abs x) a))) 0 r)) (transpose m))")
    sp = parse(src)
    assert sp.body_type.data == array(3, Num())
    m = [[1, -2, 3], [-4, 5, -6]]
    assert eval_phrase(sp.body, {"m": m}) == [5, 7, 9]
    s2 = stage2(translate_program(sp.body, sp.body_type.data, "out", "global"), "private")
    out = run_program(s2, [("out", sp.body_type.data, "out"), ("m", sp.params[0][1].data, "in")],
                      {"m": m}, {})
    assert out["out"] == [5, 7, 9]


def test_reduce_local_is_reduce():
    src = ("(param xs (exp (array 16 num)))\n"
           "(reduceLocal (+) 3 (mapLocal (lam (x (exp num)) (* x x)) xs))")
    sp = parse(src)
    xs = list(range(-8, 8))
    want = 3 + sum(x * x for x in xs)
    assert eval_phrase(sp.body, {"xs": xs}) == want
    s2 = stage2(translate_program(sp.body, sp.body_type.data, "out", "global"), "private")
    assert _count(s2, {"reduceILocal"}) == 1
    out = run_program(s2, [("out", Num(), "out"), ("xs", array(16, Num()), "in")], {"xs": xs}, {})
    assert out["out"] == want


def test_seeded_race_is_reported():
    racy, _ = parse_phrase("(parfor out (lam (i (exp (idx 4))) (lam (o (acc num)) (:= (idxAcc out 0) 1))))",
                           {"out": AccT(array(4, Num()))})
    with pytest.raises(RaceError):
        run_program(racy, [("out", array(4, Num()), "out")], {}, {})


def test_sizes_polynomials():
    n = nat("n")
    assert (n * 4 + 1) == (1 + 4 * n)
    assert str(nat(3) * n * n) == "(* (* 3 n) n)"
    assert (n * 1024).const is None and nat(7).const == 7
    from paper_1710_08332_b200.sizes import nat_divide
    assert nat_divide(n * 1024, 1024) == n
    assert nat_divide(n * 1024 + 3, 1024) is None


def test_mm_strategy_matches_numpy_oracle_small():
    """The mm strategy program (transpose, let, 2-D maps, splat init) under
    the oracle interpreter equals the NumPy restatement used at full size."""
    import numpy as np
    from oracle import blas_np
    from paper_1710_08332_b200.bench_programs import mm_program
    sp = parse(mm_program(32, 16, 24, T=16, BK=8, R=4))
    A = np.random.default_rng(1).integers(-9, 10, (32, 24))
    B = np.random.default_rng(2).integers(-9, 10, (24, 16))
    got = eval_phrase(sp.body, {"A": A.tolist(), "B": B.tolist()})
    flat = [x for row in got for blk in row for x in blk]
    assert np.array_equal(np.array(flat).reshape(32, 16), A @ B)
    want, _ = blas_np.mm(A, B)
    assert np.array_equal(want, A @ B)
    s2 = stage2(translate_program(sp.body, sp.body_type.data, "out", "global"), "private")
    out = run_program(s2, [("out", sp.body_type.data, "out"), ("A", sp.params[0][1].data, "in"),
                           ("B", sp.params[1][1].data, "in")], {"A": A.tolist(), "B": B.tolist()}, {})
    assert [x for row in out["out"] for blk in row for x in blk] == flat


def test_let_shares_and_matches_reference_semantics():
    src = ("(param xs (exp (array 8 num)))\n"
           "(let (toLocal (mapLocal (lam (x (exp num)) (* x x))) xs)"
           " (lam (s (exp (array 8 num))) (zip s (mapSeq (lam (y (exp num)) (+ y 1)) s))))")
    sp = parse(src)
    xs = list(range(8))
    assert eval_phrase(sp.body, {"xs": xs}) == [(x * x, x * x + 1) for x in xs]
    s1 = translate_program(sp.body, sp.body_type.data, "out", "global")
    assert _count(s1, {"mapILocal"}) == 1  # the staged value is computed once


# ---------------------------------------------------------------- index algebra
def _ix_from_sexp(sx, R):
    from paper_1710_08332_b200.cuda import index as IX
    from paper_1710_08332_b200.reader import Token, read_all
    if isinstance(sx, Token):
        return IX.ix(int(sx.text)) if sx.text.isdigit() else IX.ix(sx.text)
    op, a, b = sx[0].text, _ix_from_sexp(sx[1], R), sx[2]
    if op in "/%":
        n = int(b.text)
        return IX.div(a, n, R) if op == "/" else IX.mod(a, n, R)
    bb = _ix_from_sexp(b, R)
    return a + bb if op == "+" else (a + bb * (-1) if op == "-" else a * bb)


def _eval_sexp(sx, env):
    from paper_1710_08332_b200.reader import Token
    if isinstance(sx, Token):
        return int(sx.text) if sx.text.isdigit() else env[sx.text]
    a, b = _eval_sexp(sx[1], env), _eval_sexp(sx[2], env)
    op = sx[0].text
    if op in "/%":
        return a // b if op == "/" else a % b
    return a + b if op == "+" else (a - b if op == "-" else a * b)


@pytest.mark.parametrize("case", load_golden("index.json"), ids=lambda c: c["expr"])
def test_index_simplifier_matches_reference_known_answers(case):
    """Same cases as the reference's simplify_index tests
    (TST/test_codegen_c.py:61-96, TST/test_acceptance.py:287-324): the CUDA
    index algebra is exhaustively sound and removes every / and % that the
    reference removes."""
    import itertools
    from paper_1710_08332_b200.cuda import index as IX
    from paper_1710_08332_b200.reader import read_all
    sx = read_all(case["expr"])[0]
    R = dict(case["ranges"])
    e = _ix_from_sexp(sx, R)
    ev_ranges = {**{n: 20 for n in IX.free_names(e)}, **R}   # unknown-range names: sample
    names = sorted(ev_ranges)
    for vals in itertools.product(*(range(ev_ranges[n]) for n in names)):
        env = dict(zip(names, vals))
        assert IX.evaluate(e, env) == _eval_sexp(sx, env)
    ours = IX.render(e)
    ref = case["reference_simplified"]
    if "/" not in ref and "%" not in ref:
        assert "/" not in ours and "%" not in ours, (ours, ref)


# ------------------------------------------------- reference-compatible hierarchy API
HOIST_SRC = ("(nat n)\n(param xss (exp (array n (array 1024 num))))\n"
             "(mapGlobal (lam (row (exp (array 1024 num)))"
             " (reduce (+) 0 (toGlobal (mapSeq (lam x (* x x))) row))) xss)")


def test_hoist_allocations_criterion9_analogue():
    """TST/test_acceptance.py:250-284: one n x 1024 global buffer, indexed by
    the loop variable, semantics unchanged."""
    from paper_1710_08332_b200.cuda.hierarchy import hoist_allocations
    from paper_1710_08332_b200.sizes import nat
    sp = parse(HOIST_SRC)
    s2 = stage2(translate_program(sp.body, sp.body_type.data, "out", "global"), "private")
    hoisted, bufs = hoist_allocations(s2)
    assert len(bufs) == 1 and bufs[0].space == "global"
    assert bufs[0].dtype.size == nat("n") and bufs[0].dtype.elem.size == nat(1024)
    assert sum(1 for s in subtree_iter(hoisted) if isinstance(s, Prim) and s.name == "newGlobal") == 1
    small = parse(HOIST_SRC.replace("1024", "8"))
    s2s = stage2(translate_program(small.body, small.body_type.data, "out", "global"), "private")
    hs, _ = hoist_allocations(s2s)
    xss = [[(i * 8 + j) % 9 for j in range(8)] for i in range(4)]
    params = [("out", array(nat("n"), Num()), "out"), ("xss", array(nat("n"), array(8, Num())), "in")]
    want = eval_phrase(small.body, {"xss": xss}, {"n": 4})
    for phrase in (s2s, hs):
        assert run_program(phrase, params, {"xss": xss}, {"n": 4})["out"] == want


def test_lint_hierarchy_messages():
    from paper_1710_08332_b200.cuda.hierarchy import cuda_legal, lint_hierarchy

    def lint(src):
        sp = parse(src)
        return lint_hierarchy(stage2(translate_program(sp.body, sp.body_type.data, "out", "global"),
                                     "private"))
    ok = ("(param xs (exp (array 8 num)))\n(mapWorkgroup (lam (c (exp (array 4 num)))"
          " (mapLocal (lam x (+ x 1)) c)) (split 4 xs))")
    assert lint(ok) == []
    nested = ("(param xss (exp (array 4 (array 4 num))))\n(mapGlobal (lam (r (exp (array 4 num)))"
              " (mapGlobal (lam x (+ x 1)) r)) xss)")
    assert any("nested" in w for w in lint(nested))
    assert any("work-group" in w for w in lint("(param xs (exp (array 8 num)))\n(mapLocal (lam x (+ x 1)) xs)"))
    two_d = ("(param m (exp (array 4 (array 8 num))))\n(mapWorkgroup1 (lam (r (exp (array 8 num)))"
             " (mapWorkgroup (lam (c (exp (array 4 num))) (mapLocal (lam x x) c)) (split 4 r))) m)")
    assert lint(two_d) == []
    sp = parse(two_d)
    assert cuda_legal(stage2(translate_program(sp.body, sp.body_type.data, "out", "global"), "private"))


# ------------------------------------------------------------------ SCIR checker
def test_checker_interference_rejection_criterion8():
    """TST/test_acceptance.py:236-247."""
    from paper_1710_08332_b200.checker import DpiaTypeError, type_check
    src = ("(param out (acc (array 4 num)))\n(param b (acc num))\n"
           "(parfor out (lam (i (exp (idx 4))) (lam (o (acc num)) (:= b 1))))")
    sp = parse(src)
    with pytest.raises(DpiaTypeError) as ei:
        type_check(sp.body, delta=sp.delta, pi=sp.pi, gamma=sp.gamma)
    assert "passive" in str(ei.value) and "'b'" in str(ei.value)
    ok = ("(param out (acc (array 4 num)))\n"
          "(parfor out (lam (i (exp (idx 4))) (lam (o (acc num)) (:= o 1))))")
    sp = parse(ok)
    t, uses = type_check(sp.body, delta=sp.delta, pi=sp.pi, gamma=sp.gamma)
    assert isinstance(t, type(COMM_T)) and uses.mode("out") == "active"


from paper_1710_08332_b200.dtypes import COMM as COMM_T  # noqa: E402


@pytest.mark.parametrize("case", [c for c in CASES if c.get("reparses", True)][::2], ids=_id)
def test_stage1_type_preservation_criterion4(case):
    """Every source type-checks and Stage I output re-checks at comm
    (Theorem 4.1; TST/test_acceptance.py:164-178), for the reference's
    programs and its fuzz corpus, in both translation modes."""
    from paper_1710_08332_b200.checker import type_check
    sp = parse(case["text"])
    type_check(sp.body, delta=sp.delta, pi=sp.pi, gamma=sp.gamma)
    for space in (None, "global"):
        s1 = translate_program(sp.body, sp.body_type.data, "out", space)
        t, _ = type_check(s1, delta=sp.delta, pi=sp.pi,
                          gamma={**sp.gamma, "out": AccT(sp.body_type.data)})
        assert t == COMM_T


def test_benchmark_strategies_type_check():
    """The B200 strategies (with transpose, reduceLocal, let, 2-D maps)
    are well-typed SCIR, and so is their Stage I output."""
    from paper_1710_08332_b200.bench_programs import (asum_program, dot_program, gemv_program,
                                                      mm_program, scal_program)
    from paper_1710_08332_b200.checker import type_check
    for text in (dot_program(64, 4), asum_program(64, 4), gemv_program(8, 512, 64),
                 mm_program(64, 64, 64, 32, 8, 4), scal_program()):
        sp = parse(text)
        type_check(sp.body, delta=sp.delta, pi=sp.pi, gamma=sp.gamma)
        s1 = translate_program(sp.body, sp.body_type.data, "out", "global")
        t, _ = type_check(s1, delta=sp.delta, pi=sp.pi,
                          gamma={**sp.gamma, "out": AccT(sp.body_type.data)})
        assert t == COMM_T


@pytest.mark.parametrize("case", load_golden("fuzz_float.json"), ids=lambda c: f"fseed{c['seed']}")
def test_float_mode_oracle_matches_reference(case):
    """float64 oracle == the reference's float64 eval_phrase on the fuzz corpus."""
    import math
    sp = parse(case["text"])
    got = eval_phrase(sp.body, {k: from_json(v) for k, v in case["inputs"].items()})
    g = to_json(got)

    def close(a, b):
        if isinstance(a, list):
            return len(a) == len(b) and all(close(x, y) for x, y in zip(a, b))
        if isinstance(a, dict):
            return all(close(a[k], b[k]) for k in a)
        return math.isclose(a, b, rel_tol=1e-12, abs_tol=1e-12)
    assert close(g, case["expected"])


@pytest.mark.parametrize("case", [c for c in CASES if c.get("reparses", True)][::4], ids=_id)
def test_pretty_print_round_trips_every_stage(case):
    """show(p) re-parses to an alpha-equivalent phrase for the source, the
    Stage I and the Stage II forms (the reference's printer round-trip,
    TST/test_parser.py:173-187)."""
    from paper_1710_08332_b200.pretty import show
    from paper_1710_08332_b200.terms import alpha_equal
    sp = parse(case["text"])
    env = dict(sp.params)
    p1, _ = parse_phrase(show(sp.body), env)
    assert alpha_equal(p1, sp.body)
    env_out = {**env, "out": AccT(sp.body_type.data)}
    s1 = translate_program(sp.body, sp.body_type.data, "out", "global")
    q1, _ = parse_phrase(show(s1), env_out)
    assert alpha_equal(q1, s1)
    s2 = stage2(s1, "private")
    q2, _ = parse_phrase(show(s2), env_out)
    assert alpha_equal(q2, s2)


def test_pretty_print_benchmark_strategies():
    from paper_1710_08332_b200.bench_programs import dot_program, gemv_program, mm_program
    from paper_1710_08332_b200.pretty import show
    from paper_1710_08332_b200.terms import alpha_equal
    for text in (dot_program(64, 4), gemv_program(8, 512, 64), mm_program(64, 64, 64, 32, 8, 4)):
        sp = parse(text)
        env = dict(sp.params)
        for ph in (sp.body, translate_program(sp.body, sp.body_type.data, "out", "global")):
            q, _ = parse_phrase(show(ph), {**env, "out": AccT(sp.body_type.data)})
            assert alpha_equal(q, ph)


def test_run_kernel_reports_cross_item_races():
    """TST/test_opencl.py:171-178: every work-item writing out[0] is a
    WorkItemRace, raised before anything is compiled or launched (no GPU
    needed); writing out[i] is not."""
    from paper_1710_08332_b200 import WorkItemRace, run_kernel
    from paper_1710_08332_b200.dtypes import AccT, Array, Num
    from paper_1710_08332_b200.reader import parse_phrase
    from paper_1710_08332_b200.sizes import nat
    from paper_1710_08332_b200.cuda.hierarchy import check_work_item_races
    t = Array(nat(4), Num())
    racy, _ = parse_phrase("(parforGlobal out (lam (i (exp (idx 4))) (lam (o (acc num)) (:= (idxAcc out 0) 1))))",
                           {"out": AccT(t)})
    with pytest.raises(WorkItemRace):
        run_kernel(racy, [("out", t, "out")], {}, (2, 2))
    ok, _ = parse_phrase("(parforGlobal out (lam (i (exp (idx 4))) (lam (o (acc num)) (:= (idxAcc out i) 1))))",
                         {"out": AccT(t)})
    check_work_item_races(ok)
