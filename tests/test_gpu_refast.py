"""All 1000 reference fuzz programs on the GPU, entering as the reference's
own AST objects (tests/golden/fuzz_ast.json.gz, refast.py) instead of
printed text -- so the 94 programs whose text does not re-parse reach the
GPU too.

* the functional body goes through this package's Stage I / Stage II and
  run_kernel at two launch geometries; programs the CUDA backend rejects
  must be ones the reference's kernel backend rejects too (not
  opencl_legal);
* the kernel-legal ones additionally run as the reference hands them to
  its simulator: the HOISTED kernel form, through refast.simulate_kernel
  with the reference's calling convention, and the result must compare
  equal (`sim["out"] != ref`, harness.py:404-405) to the reference's
  eval_phrase value.
"""
import gzip
import json
import os

import pytest

from conftest import load_golden
from oracle.dpia_eval import flatten_value, from_json
from paper_1710_08332_b200 import CudaError, run_kernel, stage2, translate_program
from paper_1710_08332_b200.layout import flatten
from paper_1710_08332_b200.refast import _vector_class, phrase_from_json, simulate_kernel, type_from_json

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
with gzip.open(os.path.join(HERE, "golden", "fuzz_ast.json.gz")) as _f:
    AST = json.load(_f)
FUZZ = {c["seed"]: c for c in load_golden("fuzz.json")}


def _params(case):
    bt = type_from_json(case["body_type"]).data
    return bt, [("out", bt, "out")] + [(n, type_from_json(t).data, "in") for n, t in case["params"]]


@pytest.mark.parametrize("case", AST, ids=lambda c: f"seed{c['seed']}")
def test_reference_fuzz_program_from_ast(case):
    fz = FUZZ[case["seed"]]
    want = flatten_value(from_json(fz["expected"]))
    if any(abs(v) >= 2 ** 63 for v in want):
        pytest.skip("reference result exceeds int64 (the reference's C path overflows too)")
    bt, params = _params(case)
    inputs = {k: from_json(v) for k, v in fz["inputs"].items()}
    imp = stage2(translate_program(phrase_from_json(case["body"]), bt, out="out", default_space="global"),
                 accum_space="private")
    for launch in ((2, 2), (3, 5)):
        try:
            got = run_kernel(imp, params, inputs, launch, {}, False, flat=True)["out"]
        except CudaError:
            if case["hoisted"] is not None:
                raise
            pytest.skip("hierarchy rejected by the backend (the reference's kernel backend rejects it too)")
        assert [int(v) for v in got] == want
    if case["hoisted"] is not None:
        sim = simulate_kernel(phrase_from_json(case["hoisted"]), params, inputs, (2, 2), {}, False)
        assert [int(v) for v in flatten(sim["out"])] == want
        if _vector_class(inputs.values()) is not None:   # results in the caller's vector class
            assert sim["out"] == from_json(fz["expected"])


def test_cli_fuzz_all_seeds_junit(tmp_path, capsys):
    """`fuzz --device cuda --junit` (ref cli.py:192-227): all 1000 corpus
    programs (AST form) through the CUDA pipeline, a JUnit report with one
    case per seed and no failure."""
    import xml.etree.ElementTree as ET
    from paper_1710_08332_b200.cli import main
    report = tmp_path / "fuzz.xml"
    assert main(["fuzz", "--device", "cuda", "--seeds", "1000", "--junit", str(report)]) == 0
    suite = ET.parse(report).getroot()
    assert suite.get("tests") == "1000" and suite.get("failures") == "0"
    assert len(suite.findall("testcase")) == 1000
    assert "1000/1000 passed on the GPU" in capsys.readouterr().out
