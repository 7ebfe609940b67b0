"""Generate the golden fixtures in this directory by running the REFERENCE
implementation (/root/reference, importable in the build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed; the GPU box never reads /root/reference):
  programs.json  -- hand-picked programs (the reference's own sample and test
                    programs plus the benchmark strategies expressible in the
                    reference language) with inputs and the reference's
                    `eval_phrase` result; kernel-legal ones also carry the
                    reference's `simulate_kernel` result at launch (2,2).
  fuzz.json      -- the reference fuzzer's programs (`harness.generate_program`,
                    seeds 0..FUZZ_SEEDS-1) pretty-printed by the reference,
                    with `random_inputs` and the `eval_phrase` result.
  Kernel-legal entries also carry "hoisted": the reference's hoisted kernel
  form (`hoist_allocations`, the input of `emit_kernel`) pretty-printed, with
  the typing environment needed to re-parse it.
  index.json     -- index-simplifier known answers (`codegen_c.simplify_index`).
  fuzz_float.json -- the kernel-legal fuzz programs again on float inputs,
                    with the reference's float64 `eval_phrase` result.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from dpia.eval_fn import VectorVal, eval_phrase  # noqa: E402
from dpia.harness import generate_program, random_inputs  # noqa: E402
from dpia.lower import stage2  # noqa: E402
from dpia.opencl import hoist_allocations, opencl_legal, simulate_kernel  # noqa: E402
from dpia.parser import parse  # noqa: E402
from dpia.pretty import pretty_print  # noqa: E402
from dpia.translate import translate_program  # noqa: E402

FUZZ_SEEDS = 1000
PROGS = "/root/reference/pkg/programs"


def to_json(v):
    if isinstance(v, VectorVal):
        return {"vec": list(v.items)}
    if isinstance(v, tuple):
        return {"pair": [to_json(v[0]), to_json(v[1])]}
    if isinstance(v, list):
        return [to_json(x) for x in v]
    return v


def from_json(j):
    if isinstance(j, dict) and "vec" in j:
        return VectorVal(tuple(j["vec"]))
    if isinstance(j, dict) and "pair" in j:
        return (from_json(j["pair"][0]), from_json(j["pair"][1]))
    if isinstance(j, list):
        return [from_json(x) for x in j]
    return j


HOISTED = {}


def kernel_result(sp, inputs, sigma, float_mode):
    s1 = translate_program(sp.body, sp.body_type.data, out="out", default_space="global")
    s2 = stage2(s1, accum_space="private")
    if not opencl_legal(s2):
        return False, None
    hoisted, _ = hoist_allocations(s2)
    params = [("out", sp.body_type.data, "out")] + [(n, t.data, "in") for n, t in sp.params]
    out = simulate_kernel(hoisted, params, inputs, (2, 2), sigma, float_mode)
    # the reference's hoisted kernel form (the input of emit_kernel), printed
    HOISTED["last"] = {"text": pretty_print(hoisted),
                       "env": {"out": f"(acc {sp.body_type.data})",
                               **{n: str(t) for n, t in sp.params}}}
    return True, to_json(out["out"])


def case(name, text, inputs, sigma=None, float_mode=False, note=""):
    sp = parse(text)
    sigma = sigma or {}
    inputs = {k: from_json(v) for k, v in inputs.items()}
    want = eval_phrase(sp.body, dict(inputs), sigma)
    HOISTED.pop("last", None)
    legal, sim = kernel_result(sp, inputs, sigma, float_mode)
    return {"name": name, "text": text, "inputs": {k: to_json(v) for k, v in inputs.items()},
            "sigma": sigma, "float": float_mode, "expected": to_json(want),
            "opencl_legal": legal, "simulated_2x2": sim, "note": note,
            "hoisted": HOISTED.pop("last", None)}


def ints(n, a, b):
    return [(a * i + b) % 17 - 8 for i in range(n)]


def main():
    cases = []
    dot_inputs = {"xs": [1, 2, 3, 4, 5, 6, 7, 8], "ys": [8, 7, 6, 5, 4, 3, 2, 1]}
    cases.append(case("dot.dpia", open(f"{PROGS}/dot.dpia").read(), dot_inputs,
                      note="TST/test_cli.py:69-73 expects out = 120"))
    cases.append(case("dottiled.dpia", open(f"{PROGS}/dottiled.dpia").read(),
                      {"xs": ints(64, 7, 3), "ys": ints(64, 5, 1)}))
    cases.append(case("dotvec.dpia", open(f"{PROGS}/dotvec.dpia").read(),
                      {"xs": ints(256, 3, 0), "ys": ints(256, 7, 2)}))
    cases.append(case("dotvec.dpia/float", open(f"{PROGS}/dotvec.dpia").read(),
                      {"xs": [((3 * i) % 11) / 7.0 for i in range(256)],
                       "ys": [((7 * i) % 13) / 3.0 for i in range(256)]}, float_mode=True,
                      note="TST/test_acceptance.py:146-150 float leg"))
    vec64 = ("(param xs (exp (array 64 num)))\n(param ys (exp (array 64 num)))\n"
             "(asScalar4 (join (mapWorkgroup (lam (zs1 (exp (array 8 (pair (vec 4) (vec 4)))))"
             " (mapLocal (lam (zs2 (exp (array 4 (pair (vec 4) (vec 4)))))"
             " (reduce (lam (x (exp (pair (vec 4) (vec 4)))) (lam (a (exp (vec 4)))"
             " (+ (* (fst x) (snd x)) a))) 0 zs2)) (split 4 zs1)))"
             " (split 8 (zip (asVector4 xs) (asVector4 ys))))))")
    cases.append(case("test_opencl.VEC_SRC", vec64,
                      {"xs": [(3 * i) % 17 for i in range(64)], "ys": [(5 * i) % 13 for i in range(64)]}))
    hoist = ("(nat n)\n(param xss (exp (array n (array 8 num))))\n"
             "(mapGlobal (lam (row (exp (array 8 num)))"
             " (reduce (+) 0 (toGlobal (mapSeq (lam x (* x x))) row))) xss)")
    cases.append(case("hoist.n4", hoist, {"xss": [[(i * 8 + j) % 9 for j in range(8)] for i in range(4)]},
                      sigma={"n": 4}, note="TST/test_acceptance.py:250-284"))
    # benchmark strategies expressible in the reference language, small sizes
    dotg = ("(nat n)\n(param xs (exp (array (* n 16) num)))\n(param ys (exp (array (* n 16) num)))\n"
            "(reduce (+) 0 (mapGlobal (lam (c (exp (array 16 (pair num num))))"
            " (reduce (lam (x (exp (pair num num))) (lam (a (exp num)) (+ (* (fst x) (snd x)) a))) 0 c))"
            " (split 16 (zip xs ys))))")
    cases.append(case("bench.dot_mapglobal.n8", dotg, {"xs": ints(128, 3, 1), "ys": ints(128, 5, 2)},
                      sigma={"n": 8}, note="config 1 strategy (survey App. A.1)"))
    gemv = ("(param A (exp (array 8 (array 32 num))))\n(param x (exp (array 32 num)))\n"
            "(join (mapWorkgroup (lam (row (exp (array 32 num)))"
            " (mapLocal (lam (ps (exp (array 4 num))) (reduce (+) 0 ps))"
            " (split 4 (toLocal (mapLocal (lam (c (exp (array 8 (pair num num))))"
            " (reduce (lam (p (exp (pair num num))) (lam (a (exp num)) (+ (* (fst p) (snd p)) a))) 0 c)))"
            " (split 8 (zip row (toLocal (mapLocal (lam (v (exp num)) v)) x)))))))"
            " A))")
    cases.append(case("bench.gemv_rowwg", gemv,
                      {"A": [ints(32, 3 + r, r) for r in range(8)], "x": ints(32, 5, 4)},
                      note="config 3 strategy in reference syntax (survey App. A.3)"))
    mm = ("(param A (exp (array 8 (array 8 num))))\n(param Bt (exp (array 8 (array 8 num))))\n"
          "(join (mapWorkgroup (lam (ra (exp (array 4 (array 8 num))))"
          " (mapLocal (lam (r (exp (array 8 num)))"
          " (mapSeq (lam (c (exp (array 8 num)))"
          " (reduce (lam (p (exp (pair num num))) (lam (a (exp num)) (+ (* (fst p) (snd p)) a))) 0 (zip r c)))"
          " Bt)) ra)) (split 4 A)))")
    cases.append(case("bench.mm_bt", mm, {"A": [ints(8, 3 + r, r) for r in range(8)],
                                          "Bt": [ints(8, 5 + r, 2 * r) for r in range(8)]},
                      note="config 4 in reference syntax with pre-transposed B"))

    fuzz = []
    for seed in range(FUZZ_SEEDS):
        sp = generate_program(seed, depth=4, sizes=64)
        inputs = random_inputs(sp, seed)
        text = "".join(f"(param {n} {t})\n" for n, t in sp.params) + pretty_print(sp.body)
        HOISTED.pop("last", None)
        legal, sim = kernel_result(sp, inputs, {}, False)
        hoisted = HOISTED.pop("last", None)
        try:  # the reference's printer is not a perfect inverse for vector literals
            parse(text)
            reparses = True
        except Exception:  # noqa: BLE001
            reparses = False
        fuzz.append({"seed": seed, "text": text, "type": str(sp.body_type), "reparses": reparses,
                     "inputs": {k: to_json(v) for k, v in inputs.items()},
                     "expected": to_json(eval_phrase(sp.body, dict(inputs), {})),
                     "opencl_legal": legal, "simulated_2x2": sim, "hoisted": hoisted})

    # float mode: the same kernel-legal fuzz programs on float inputs, with
    # the reference's float64 eval_phrase result
    import random as _random
    fuzz_float = []
    for c in fuzz:
        if not (c["opencl_legal"] and c["reparses"]):
            continue
        sp = parse(c["text"])
        rng = _random.Random(c["seed"] ^ 0xF10A7)

        def rand_f(d):
            from dpia.types import Array as RArr, Num as RNum, Pair as RPair, Vector as RVec
            if isinstance(d, RNum):
                return round(rng.uniform(-2, 2), 3)
            if isinstance(d, RVec):
                return VectorVal(tuple(round(rng.uniform(-2, 2), 3) for _ in range(d.width)))
            if isinstance(d, RArr):
                from dpia.nat import nat_const_value
                return [rand_f(d.elem) for _ in range(nat_const_value(d.size))]
            if isinstance(d, RPair):
                return (rand_f(d.fst), rand_f(d.snd))
            raise ValueError(d)
        finputs = {n: rand_f(t.data) for n, t in sp.params}
        try:
            want = eval_phrase(sp.body, dict(finputs), {})
        except ZeroDivisionError:
            continue
        fuzz_float.append({"seed": c["seed"], "text": c["text"], "float": True,
                           "inputs": {k: to_json(v) for k, v in finputs.items()},
                           "expected": to_json(want)})

    from dpia.c_ast import CBin, CInt, CVar, expr_str
    from dpia.codegen_c import simplify_index
    i, j, k = CVar("i"), CVar("j"), CVar("k")
    flat = CBin("+", CBin("*", CBin("+", CBin("*", i, CInt(4)), j), CInt(8)), k)
    idx_cases = [
        (CBin("/", CBin("+", CBin("*", i, CInt(8)), j), CInt(8)), {"i": 4, "j": 8}),
        (CBin("%", CBin("+", CBin("*", i, CInt(8)), j), CInt(8)), {"i": 4, "j": 8}),
        (CBin("/", flat, CInt(8)), {"i": 2, "j": 4, "k": 8}),
        (CBin("%", flat, CInt(8)), {"i": 2, "j": 4, "k": 8}),
        (CBin("%", CBin("/", flat, CInt(8)), CInt(4)), {"i": 2, "j": 4, "k": 8}),
        (CBin("/", CBin("*", i, CInt(12)), CInt(4)), {"i": 64}),
        (CBin("+", CBin("-", i, i), j), {"i": 64, "j": 64}),
        (CBin("*", CBin("+", i, CInt(1)), CInt(0)), {"i": 64}),
        (CBin("/", CBin("+", CBin("*", i, CInt(8)), j), CInt(8)), {"i": 4}),
    ]

    def sexp(e):
        if isinstance(e, CInt):
            return str(e.value)
        if isinstance(e, CVar):
            return e.name
        return f"({e.op} {sexp(e.left)} {sexp(e.right)})"

    index = [{"expr": sexp(e), "ranges": r, "reference_simplified": expr_str(simplify_index(e, r))}
             for e, r in idx_cases]

    for fname, obj in (("programs.json", cases), ("fuzz.json", fuzz), ("index.json", index),
                       ("fuzz_float.json", fuzz_float)):
        with open(os.path.join(HERE, fname), "w") as f:
            json.dump(obj, f, indent=None, separators=(",", ":"))
            f.write("\n")
    print(f"{len(cases)} programs, {len(fuzz)} fuzz programs "
          f"({sum(c['opencl_legal'] for c in fuzz)} kernel-legal), {len(index)} index cases")


if __name__ == "__main__":
    main()
