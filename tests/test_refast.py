"""The drop-in from the reference's own AST objects (paper_1710_08332_b200/
refast.py).

CPU: the structural corpus tests/golden/fuzz_ast.json.gz -- all 1000 of the
reference fuzzer's programs as the reference's own objects, serialised
node for node -- converts into this package's phrases; where the printed
text re-parses, the conversion is alpha-equal to the parse; for EVERY seed
(the 94 that do not re-parse included) the oracle evaluates the converted
phrase to the reference's eval_phrase result, and the CUDA front end
(Stage I, Stage II, emission) accepts it.  With the reference importable
(build container), the corpus regenerates byte-for-byte and the adapter is
exercised on the reference's live objects, including `emit_kernel`'s
KernelSignature view.
"""
import gzip
import json
import os
import sys

import pytest

from conftest import load_golden
from oracle.dpia_eval import eval_phrase, flatten_value, from_json
from paper_1710_08332_b200 import stage2, translate_program
from paper_1710_08332_b200.cuda.emit import emit_cuda
from paper_1710_08332_b200.dtypes import ExpT
from paper_1710_08332_b200.reader import parse
from paper_1710_08332_b200.refast import (AdapterError, phrase_from_json, to_json,
                                          type_from_json)
from paper_1710_08332_b200.terms import alpha_equal

HERE = os.path.dirname(os.path.abspath(__file__))
AST_PATH = os.path.join(HERE, "golden", "fuzz_ast.json.gz")
REF = "/root/reference/pkg/src"


def load_ast():
    with gzip.open(AST_PATH) as f:
        return json.load(f)


AST = load_ast()
FUZZ = {c["seed"]: c for c in load_golden("fuzz.json")}


def test_corpus_covers_every_seed():
    assert [c["seed"] for c in AST] == list(range(1000)) == sorted(FUZZ)
    assert sum(c["hoisted"] is not None for c in AST) == sum(FUZZ[s]["opencl_legal"] for s in FUZZ)
    assert sum(not FUZZ[s]["reparses"] for s in FUZZ) == 94


@pytest.mark.parametrize("chunk", range(10))
def test_every_seed_converts_and_evaluates_to_the_reference(chunk):
    for case in AST[chunk * 100:(chunk + 1) * 100]:
        fz = FUZZ[case["seed"]]
        body = phrase_from_json(case["body"])
        if fz["reparses"]:
            assert alpha_equal(body, parse(fz["text"]).body), case["seed"]
        inputs = {k: from_json(v) for k, v in fz["inputs"].items()}
        assert flatten_value(eval_phrase(body, inputs, {})) == flatten_value(from_json(fz["expected"]))
        bt = type_from_json(case["body_type"])
        assert isinstance(bt, ExpT)
        s2 = stage2(translate_program(body, bt.data, out="out", default_space="global"),
                    accum_space="private")
        params = [(n, type_from_json(t).data) for n, t in case["params"]]
        if case["hoisted"] is not None:
            hoisted = phrase_from_json(case["hoisted"])
            src, sig = emit_cuda(hoisted, [("out", bt.data)], params, float_mode=False)
            assert "__global__" in src and [n for n, _ in sig.inputs] == [n for n, _ in params]
        del s2


def test_json_round_trip_of_this_packages_objects():
    sp = parse(FUZZ[3]["text"]) if FUZZ[3]["reparses"] else parse(FUZZ[0]["text"])
    assert alpha_equal(phrase_from_json(json.loads(json.dumps(to_json(sp.body)))), sp.body)
    for _, t in sp.params:
        assert type_from_json(to_json(t)) == t
    with pytest.raises(AdapterError):
        to_json(object())
    with pytest.raises(AdapterError):
        phrase_from_json({"k": "Nope"})


ref = pytest.mark.skipif(not os.path.isdir(REF), reason="the reference is only present in the build container")


@ref
def test_corpus_regenerates_byte_for_byte():
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(HERE, "golden"))
    import make_fuzz_ast
    with open(AST_PATH, "rb") as f:
        assert make_fuzz_ast.dump(make_fuzz_ast.corpus()) == f.read()


@ref
def test_live_reference_objects():
    """from_reference_phrase / emit_kernel on the reference's own objects
    (what harness.py:399-407 and cli.py:181-183 hold)."""
    sys.path.insert(0, REF)
    from dpia.lower import stage2 as rstage2
    from dpia.opencl import emit_kernel as r_emit
    from dpia.opencl import hoist_allocations as rhoist
    from dpia.parser import parse as rparse
    from dpia.translate import translate_program as rtranslate

    from paper_1710_08332_b200.refast import emit_kernel, from_reference_phrase
    text = [c for c in load_golden("programs.json") if c["name"] == "dotvec.dpia"][0]["text"]
    sp = rparse(text)
    assert alpha_equal(from_reference_phrase(sp.body), parse(text).body)
    imp = rstage2(rtranslate(sp.body, sp.body_type.data, out="out", default_space="global"),
                  accum_space="private")
    hoisted, _bufs = rhoist(imp)
    outs = [("out", sp.body_type.data)]
    ins = [(n, t.data) for n, t in sp.params]
    _rsrc, rsig = r_emit(hoisted, outs, ins)
    src, sig = emit_kernel(hoisted, outs, ins)
    assert "__global__" in src
    assert sig.outputs == rsig.outputs and sig.inputs == rsig.inputs   # the caller's own objects
    assert [n for n in sig.sizes] == [n for n in rsig.sizes]
    assert len(sig.params("float")) == len(sig.outputs) + len(sig.inputs) + len(sig.buffers) + len(sig.sizes)
