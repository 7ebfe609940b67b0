"""Unit behaviour of the re-implemented front end, one property per test, in
the shape of the reference's own unit suites (TST/test_parser.py,
TST/test_nat.py, TST/test_checker.py, TST/test_translate.py,
TST/test_lower.py): the same API names, the same error classes, the same
structural outcomes -- on this repository's own example programs (CPU)."""
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_1710_08332_b200.checker import DpiaTypeError, type_check
from paper_1710_08332_b200.dtypes import (AccT, Array, CommT, ExpT, Num, ProdT, Vector, is_passive,
                                          var_t)
from paper_1710_08332_b200.pretty import pretty_print
from paper_1710_08332_b200.reader import ElabError, ParseError, parse, parse_phrase
from paper_1710_08332_b200.signatures import MAP_FAMILY, MAPI_FAMILY, PARFOR_FAMILY
from paper_1710_08332_b200.sizes import (nat, nat_divide, nat_equal, nat_eval, nat_free_vars,
                                         nat_normalize, nat_str)
from paper_1710_08332_b200.stage1 import translate_program
from paper_1710_08332_b200.stage2 import is_purely_imperative, stage2
from paper_1710_08332_b200.terms import Prim, alpha_equal, subtree_iter

SAXPY = """
(param a (exp (array 16 num)))
(param b (exp (array 16 num)))
(map (lam p (+ (* 2 (fst p)) (snd p))) (zip a b))
"""
NORM2 = """
(param v (exp (array 16 num)))
(reduce (+) 0 (map (lam x (* x x)) v))
"""


# ------------------------------------------------------------------ reader

def test_reader_types_the_body():
    sp = parse(SAXPY)
    assert [n for n, _ in sp.params] == ["a", "b"]
    assert sp.body_type == ExpT(Array(nat(16), Num()))


def test_reader_skips_comments_anywhere():
    assert parse(";; head\n" + NORM2 + ";; tail\n").body_type == ExpT(Num())


def test_reader_size_parameters():
    sp = parse("(nat k)\n(param v (exp (array (* 2 k) num)))\n(map (lam x (* x 3)) v)")
    assert sp.nat_params == ["k"]
    assert isinstance(sp.body_type.data, Array)


def test_reader_vector_types():
    assert parse("(param w (exp (vec 2)))\n(* w w)").body_type == ExpT(Vector(2))
    with pytest.raises(ParseError):
        parse("(param w (exp (vec 6)))\nw")


@pytest.mark.parametrize("text", [
    "(param v (exp (array 4 num))\nv",                       # unbalanced
    "(param v (exp num))\n(param v (exp num))\nv",           # duplicate parameter
    "(param v (exp num))",                                   # no body
])
def test_reader_syntax_errors_are_not_type_errors(text):
    with pytest.raises(ParseError) as ei:
        parse(text)
    assert not isinstance(ei.value, ElabError)


@pytest.mark.parametrize("text", [
    "(param v (exp (array 4 num)))\n(* v 2)",                # arithmetic on an array
    "(param v (exp num))\n(snd v)",                          # projection of a scalar
    "(param v (exp num))\nw",                                # unbound identifier
    "(param v (exp (array 6 num)))\n(split 4 v)",            # 6 is not a multiple of 4
    "(param v (exp (array 4 num)))\n(param w (exp (array 2 num)))\n(zip v w)",
    "(param v (exp (array 4 num)))\n(idx v 7)",              # literal index out of bounds
])
def test_reader_type_errors_are_elab_errors(text):
    with pytest.raises(ElabError):
        parse(text)


def test_reader_three_argument_split_is_symbolic():
    sp = parse("(nat k)\n(param v (exp (array (* 8 k) num)))\n(split 8 k v)")
    t = sp.body_type.data
    assert isinstance(t.elem, Array) and t.elem.size == nat(8) and nat_equal(t.size, nat("k"))


def test_reader_pairs():
    assert parse("(param v (exp num))\n(snd (pair 1 v))").body_type == ExpT(Num())


@pytest.mark.parametrize("text", [SAXPY, NORM2,
                                  "(param v (exp (array 8 num)))\n"
                                  "(asScalar4 (map (lam w (* w w)) (asVector4 v)))"])
def test_reader_pretty_print_round_trip(text):
    sp = parse(text)
    body, t = parse_phrase(pretty_print(sp.body), dict(sp.params))
    assert alpha_equal(body, sp.body) and t == sp.body_type


# ------------------------------------------------------------------ sizes

VARS = ("n", "m", "k")


def _terms():
    leaf = st.one_of(st.integers(0, 7).map(nat), st.sampled_from(VARS).map(nat))
    return st.recursive(leaf, lambda sub: st.tuples(sub, sub, st.booleans()).map(
        lambda t: t[0] + t[1] if t[2] else t[0] * t[1]), max_leaves=8)


@settings(max_examples=60, deadline=None)
@given(_terms(), st.lists(st.integers(0, 40), min_size=3, max_size=3))
def test_sizes_canonical_form_keeps_the_value(e, vals):
    sigma = dict(zip(VARS, vals))
    assert nat_eval(nat_normalize(e), sigma) == nat_eval(e, sigma)
    assert nat_normalize(nat_normalize(e)) == nat_normalize(e)
    assert nat_str(e) == nat_str(nat_normalize(e))


def test_sizes_equality_is_semantic():
    n, m, k = nat("n"), nat("m"), nat("k")
    assert nat_equal((n + k) * m, n * m + m * k)
    assert not nat_equal(n * m, n + m)


def test_sizes_free_variables_and_unbound_evaluation():
    assert nat_free_vars(nat("k") * (nat("n") + 3)) == {"k", "n"}
    with pytest.raises(KeyError):
        nat_eval(nat("z"), {"n": 1})


def test_sizes_exact_division():
    n, m = nat("n"), nat("m")
    assert nat_equal(nat_divide(nat(6) * n, 6), n)
    assert nat_divide(n + 1, 2) is None
    assert nat_divide(nat(20), nat(5)) == nat(4)
    assert nat_equal(nat_divide(n * m * 2, m), n * 2)


# ------------------------------------------------------------------ checker

def _check(text):
    sp = parse(text)
    return type_check(sp.body, delta=sp.delta, pi=sp.pi, gamma=sp.gamma)


def test_checker_expression_parameters_are_passive():
    t, uses = _check(NORM2)
    assert t == ExpT(Num()) and uses.active == set() and uses.passive == {"v"}


def test_checker_parfor_writes_through_its_own_acceptor():
    t, uses = _check("(param y (acc (array 8 num)))\n(param s (exp num))\n"
                     "(parfor y (lam (j (exp (idx 8))) (lam (o (acc num)) (:= o (+ s 1)))))")
    assert isinstance(t, CommT) and uses.active == {"y"}


def test_checker_rejects_a_captured_acceptor_in_parfor():
    with pytest.raises(DpiaTypeError) as ei:
        _check("(param y (acc (array 8 num)))\n(param c (acc num))\n"
               "(parfor y (lam (j (exp (idx 8))) (lam (o (acc num)) (:= c 0))))")
    assert "passive" in str(ei.value) and "'c'" in str(ei.value)


def test_checker_sequencing_may_share_an_acceptor():
    t, uses = _check("(param c (acc num))\n(seq (:= c 3) (:= c 4))")
    assert isinstance(t, CommT) and uses.active == {"c"}


def test_checker_new_scopes_its_variable():
    t, uses = _check("(param r (acc num))\n"
                     "(new num (lam t (seq (:= (proj1 t) 5) (:= r (proj2 t)))))")
    assert isinstance(t, CommT) and uses.active == {"r"}


def test_checker_zones_and_passivity():
    sp = parse("(param v (exp num))\nv")
    with pytest.raises(DpiaTypeError):
        type_check(sp.body, pi={"v": ExpT(Num())}, gamma={"v": ExpT(Num())})
    body, _ = parse_phrase("(:= r 2)", {"r": AccT(Num())})
    with pytest.raises(DpiaTypeError):
        type_check(body)
    with pytest.raises(DpiaTypeError) as ei:
        type_check(body, pi={"r": AccT(Num())})
    assert "passive" in str(ei.value)
    assert is_passive(ExpT(Num())) and is_passive(ProdT(ExpT(Num()), ExpT(Num())))
    assert not is_passive(AccT(Num())) and not is_passive(CommT()) and not is_passive(var_t(Num()))


# ------------------------------------------------------------------ Stage I / Stage II

def _count(p, names):
    return sum(1 for s in subtree_iter(p) if isinstance(s, Prim) and s.name in names)


def _stage1(text, **kw):
    sp = parse(text)
    return sp, translate_program(sp.body, sp.body_type.data, out="out", **kw)


def _recheck(sp, s1):
    gamma = dict(sp.gamma)
    gamma["out"] = AccT(sp.body_type.data)
    return type_check(s1, delta=sp.delta, pi=sp.pi, gamma=gamma)[0]


HIER = ("(param v (exp (array 16 num)))\n"
        "(join (mapWorkgroup (lam (c (exp (array 8 num))) (mapLocal (lam x (* x 5)) c)) (split 8 v)))")


def test_stage1_is_a_well_typed_command():
    for text in (SAXPY, NORM2, HIER):
        sp, s1 = _stage1(text)
        assert isinstance(_recheck(sp, s1), CommT)


def test_stage1_one_mapi_per_map_and_one_reducei_per_reduce():
    _, s1 = _stage1(SAXPY)
    assert _count(s1, {"mapI"}) == 1 and _count(s1, MAP_FAMILY) == 0
    _, s1 = _stage1(NORM2)
    assert _count(s1, {"reduceI"}) == 1


def test_stage1_keeps_the_hierarchy():
    _, s1 = _stage1(HIER)
    assert _count(s1, {"mapIWorkgroup"}) == 1 and _count(s1, {"mapILocal"}) == 1


def test_stage1_temporaries():
    _, s1 = _stage1("(param v (exp num))\n(* v 4)")
    assert _count(s1, {"new"}) == 0 and _count(s1, {":="}) == 1
    _, s1 = _stage1(NORM2)
    assert _count(s1, {"new"}) >= 1                      # the map feeding reduce is materialised
    _, s1 = _stage1(NORM2, default_space="global")
    assert _count(s1, {"new"}) == 0 and _count(s1, {"newGlobal"}) >= 1


def test_stage2_loops():
    _, s1 = _stage1(SAXPY)
    s2 = stage2(s1)
    assert _count(s2, MAPI_FAMILY) == 0 and _count(s2, {"parfor"}) == 1
    _, s1 = _stage1("(param v (exp (array 16 num)))\n(mapSeq (lam x (+ x 2)) v)")
    s2 = stage2(s1)
    assert _count(s2, PARFOR_FAMILY) == 0 and _count(s2, {"for"}) == 1
    s2 = stage2(_stage1(HIER)[1])
    assert _count(s2, {"parforWorkgroup"}) == 1 and _count(s2, {"parforLocal"}) == 1


def test_stage2_accumulators_and_purity():
    s2 = stage2(_stage1(NORM2)[1])
    assert _count(s2, {"reduceI"}) == 0 and _count(s2, {"for"}) >= 1 and _count(s2, {"new"}) >= 1
    assert is_purely_imperative(s2)
    s2 = stage2(_stage1(NORM2, default_space="global")[1], accum_space="private")
    assert _count(s2, {"new"}) == 0 and _count(s2, {"newPrivate"}) >= 1
    assert is_purely_imperative(s2)


def test_golden_fixtures_regenerate_identically(tmp_path):
    """Where the reference is importable (the build container), re-running
    tests/golden/make_golden.py on the reference reproduces every committed
    fixture byte for byte: the oracle's pinning is reproducible (CPU)."""
    import os
    import shutil
    import subprocess
    import sys
    if not os.path.isdir("/root/reference/pkg/src/dpia"):
        pytest.skip("the reference is not present on this machine")
    here = os.path.join(os.path.dirname(__file__), "golden")
    shutil.copy(os.path.join(here, "make_golden.py"), tmp_path)
    subprocess.run([sys.executable, str(tmp_path / "make_golden.py")], check=True, cwd=tmp_path,
                   env=dict(os.environ, PYTHONPATH="/root/reference/pkg/src"), capture_output=True,
                   timeout=600)
    for name in ("programs.json", "fuzz.json", "fuzz_float.json", "index.json"):
        with open(os.path.join(here, name), "rb") as a, open(tmp_path / name, "rb") as b:
            assert a.read() == b.read(), name


def test_vectorised_fold_emission(monkeypatch):
    """CPU: with the software pipelining off, config 1's literal program
    reads its chunks and the tail's partials as 4-wide vectors;
    DPIA_VEC_LOADS=0 restores scalar loads; a transposed (strided) chunk is
    never vectorised."""
    from paper_1710_08332_b200 import compile_program
    from paper_1710_08332_b200.bench_programs import dot_literal_config
    from paper_1710_08332_b200.cuda import emit as E
    cfg = dot_literal_config()
    prog = compile_program(cfg.text)
    outs, ins = [("out", prog.out_type)], [(n, t.data) for n, t in prog.source.params]
    monkeypatch.setattr(E, "ROW_TMA", False)      # the register-path lowering (TMA rows: test_stream_tail)
    monkeypatch.setattr(E, "VEC_PREFETCH", 0)
    monkeypatch.setattr(E, "TAIL_RING", False)
    src, _ = E.emit_cuda(prog.imperative, outs, ins, sigma=cfg.sigma, launch=cfg.launch)
    assert "dpia::vload<float, 4>(xs, 1024 * " in src and "dpia::vload<float, 4>(g_tmp4, 4 * " in src
    assert "pfq_" not in src and "ring_" not in src.split('extern "C"')[1]
    monkeypatch.setattr(E, "VEC_LOADS", False)
    src0, _ = E.emit_cuda(prog.imperative, outs, ins, sigma=cfg.sigma, launch=cfg.launch)
    assert "vload" not in src0.split('extern "C"')[1]
    monkeypatch.setattr(E, "VEC_LOADS", True)
    monkeypatch.setattr(E, "VEC_PREFETCH", 8)
    monkeypatch.setattr(E, "TAIL_RING", True)
    strided = compile_program("(nat n)\n(param xs (exp (array (* n 128) num)))\n"
                              "(mapGlobal (lam (c (exp (array 128 num))) (reduce (+) 0 c))"
                              " (transpose (split n xs)))")
    s2, _ = E.emit_cuda(strided.imperative, [("out", strided.out_type)],
                        [(n, t.data) for n, t in strided.source.params], sigma={"n": 16}, launch=(1, 32))
    assert "vload" not in s2.split('extern "C"')[1]


def test_vectorised_fold_pipelining(monkeypatch):
    """CPU: a work-item's fold streams each input through a rotating queue
    of 32-byte loads (VEC_PREFETCH slots, refilled D slots ahead under a
    bound guard; the signature asks 32-byte alignment of those buffers);
    16-byte slots with DPIA_VEC_LOAD_BYTES=16; the single-thread top-level
    fold of the fused tail streams the partials through a shared-memory
    ring of TMA bulk copies (TAIL_RING_STAGES x TAIL_RING_BYTES), or a
    register queue with the ring off; depths that do not divide the trip
    shrink to a power of two that does."""
    from paper_1710_08332_b200 import compile_program
    from paper_1710_08332_b200.bench_programs import dot_literal_config
    from paper_1710_08332_b200.cuda import emit as E
    cfg = dot_literal_config()
    prog = compile_program(cfg.text)
    outs, ins = [("out", prog.out_type)], [(n, t.data) for n, t in prog.source.params]
    monkeypatch.setattr(E, "ROW_TMA", False)      # the register-path lowering (TMA rows: test_stream_tail)

    def emit(**kw):
        for k, v in kw.items():
            monkeypatch.setattr(E, k, v)
        src, sig = E.emit_cuda(prog.imperative, outs, ins, float_mode=True, sigma=cfg.sigma,
                               launch=cfg.launch)
        return src.split('extern "C"')[1], sig

    body, sig = emit(VEC_PREFETCH=8, VEC_LOAD_BYTES=32, TAIL_RING=True, TAIL_RING_STAGES=4,
                     TAIL_RING_BYTES=2048)
    # chunks: 1024 floats = 128 32-byte vectors per stream, 8 in flight
    assert body.count("dpia::vec<float, 8> pfq_") == 2 and "[8];" in body
    assert "dpia::vload32<true>(xs, 1024 * i_" in body and "+ 8 < 128) pfq_" in body
    assert sig.align == {"xs": 32, "ys": 32}
    # tail: 4096 vec4 of partials in pieces of 128 (2 KiB), 4 slots, bulk copies
    assert "dpia::ring_init(" in body and body.count("dpia::ring_copy(") == 2
    assert "jo_" in body and "< 4096; jo_" in body and "+= 128)" in body and "+ 512 < 4096)" in body
    assert sig.kernels[0].smem >= 4 * 2048 + 4 * 8
    body16, sig16 = emit(VEC_LOAD_BYTES=16)
    assert "vload32" not in body16 and "+ 16 < 256) pfq_" in body16 and not sig16.align
    body_q, sig_q = emit(VEC_LOAD_BYTES=32, TAIL_RING=False)
    assert "ring_init" not in body_q and "dpia::vload32<false>(g_tmp4, 8 * j_" in body_q
    assert sig_q.kernels[0].smem < 64
    body_s, _ = emit(TAIL_RING=True, TAIL_RING_BYTES=3000, VEC_PREFETCH=6)   # -> 128-vector pieces, 4 slots
    assert "+= 128)" in body_s and "+ 4 < 128) pfq_" in body_s
    body0, _ = emit(VEC_PREFETCH=0, TAIL_RING=False)
    assert "pfq_" not in body0 and "ring_" not in body0


def test_chain_waits_emission(monkeypatch):
    """CPU: a program's first kernel triggers its dependent launch at once
    and waits (once per thread) for the grid it is chained behind right
    before each line naming a non-input global buffer -- never before a
    line that only reads inputs, never between a #pragma and its loop;
    later phases keep their griddepcontrol.wait at the top; DPIA_CHAIN=0
    emits none of it."""
    import re
    from paper_1710_08332_b200 import compile_program
    from paper_1710_08332_b200.bench_programs import dot_config
    from paper_1710_08332_b200.cuda import emit as E
    cfg = dot_config(N=1 << 20)
    prog = compile_program(cfg.text)
    outs, ins = [("out", prog.out_type)], [(n, t.data) for n, t in prog.source.params]
    src, sig = E.emit_cuda(prog.imperative, outs, ins, sigma=cfg.sigma, launch=cfg.launch)
    lines = src.split('extern "C"')[1].splitlines()
    assert "dpia::pdl_trigger();" in lines[3] or any("pdl_trigger" in ln for ln in lines[:8])
    waits = [i for i, ln in enumerate(lines) if "pdl_wait_once" in ln]
    assert waits
    start = next(i for i, ln in enumerate(lines) if "bool dpia_chained" in ln)
    first_global = min(i for i, ln in enumerate(lines)
                       if i > start and re.search(r"\b(out|g_tmp\w*|dpia_counter)\b", ln))
    assert waits[0] == first_global - 1
    for i in waits:
        assert not lines[i - 1].lstrip().startswith("#pragma")
        assert re.search(r"\b(out|g_tmp\w*|dpia_counter)\b", lines[i + 1])
    # the vectorised loads of the inputs come before the first wait
    assert any("xs" in ln for ln in lines[:waits[0]])
    two = compile_program("(nat n)\n(param xs (exp (array n num)))\n"
                          "(mapGlobal (lam x (+ x 1)) (toGlobal (lam t t) (mapGlobal (lam y (* y 2)) xs)))")
    s2, sig2 = E.emit_cuda(two.imperative, [("out", two.out_type)], [("xs", two.source.params[0][1].data)],
                           sigma={"n": 4096}, launch=(16, 256))
    k1 = s2.split("KERNEL_k1")[1]
    assert "griddepcontrol.wait" in k1.splitlines()[4] or "griddepcontrol.wait" in "".join(k1.splitlines()[:6])
    assert "pdl_wait_once" not in k1
    monkeypatch.setattr(E, "CHAIN", False)
    s0, _ = E.emit_cuda(prog.imperative, outs, ins, sigma=cfg.sigma, launch=cfg.launch)
    body0 = s0.split('extern "C"')[1]
    assert "pdl_" not in body0
