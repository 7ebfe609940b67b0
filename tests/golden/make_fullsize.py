"""Full-size golden outputs produced by the REFERENCE itself (its functional
interpreter `eval_phrase`, /root/reference/pkg/src/dpia/eval_fn.py:120-215)
for the benchmark programs written in the reference's own language
(oracle/ref_programs/*.dpia), on the exact bench inputs.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fullsize.py [case ...]

The interpreter is single-threaded pure Python (~0.1 M elements/s,
SURVEY.md 8c), so each case takes minutes; this script is run once in the
build container and its outputs, `fullsize/<case>.json`, are committed.  The GPU box
never reads /root/reference: tests/test_gpu_reference_parity.py regenerates
the same inputs (numpy default_rng seeds, `oracle.blas_np.seeded`) and
compares the CUDA kernels with these values.

Cases (BASELINE.json configs; inputs as in SURVEY.md 8d):
  dot_literal_f32  config 1 exactly (ref_programs/dot.dpia, n = 16384 chunks
                   of 1024): xs, ys ~ U[0,1) fp32, seeds 0 and 1
  dot_literal_i64  the same program on int64 inputs in -9..9 (seed 77): the
                   bit-exact leg
  asum_abs_f32     config 2's traffic: ref_programs/asum_proxy.dpia (the
                   reference has no abs) over |xs|, xs ~ U[-1,1) fp32 seed 2
                   -- equal to asum(xs) by definition
  gemv_f32         config 3 (ref_programs/gemv.dpia, toLocal x): A, x ~
                   U[-1,1) fp32, seeds 3 and 4
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from dpia.eval_fn import eval_phrase  # noqa: E402
from dpia.parser import parse  # noqa: E402

from oracle.blas_np import seeded  # noqa: E402

OUT = os.path.join(HERE, "fullsize")


def _prog(name):
    with open(os.path.join(ROOT, "oracle", "ref_programs", name)) as f:
        return f.read()


def case(name):
    if name == "dot_literal_f32":
        N = 1 << 24
        text, sigma = _prog("dot.dpia"), {"n": N // 1024}
        inputs = {"xs": seeded(N, 0, 0.0, 1.0), "ys": seeded(N, 1, 0.0, 1.0)}
        desc = "xs = seeded(2^24, 0, 0, 1), ys = seeded(2^24, 1, 0, 1) (oracle.blas_np.seeded)"
    elif name == "dot_literal_i64":
        N = 1 << 24
        text, sigma = _prog("dot.dpia"), {"n": N // 1024}
        rng = np.random.default_rng(77)
        inputs = {"xs": rng.integers(-9, 10, N), "ys": rng.integers(-9, 10, N)}
        desc = "rng = default_rng(77); xs = rng.integers(-9, 10, 2^24); ys = rng.integers(-9, 10, 2^24)"
    elif name == "asum_abs_f32":
        N = 1 << 26
        text, sigma = _prog("asum_proxy.dpia"), {"n": N // 1024}
        inputs = {"xs": np.abs(seeded(N, 2, -1.0, 1.0))}
        desc = "xs = |seeded(2^26, 2, -1, 1)| (the proxy sums |x|: asum of seeded(2^26, 2, -1, 1))"
    elif name == "gemv_f32":
        text, sigma = _prog("gemv.dpia"), {}
        inputs = {"A": seeded((8192, 8192), 3, -1.0, 1.0), "x": seeded(8192, 4, -1.0, 1.0)}
        desc = "A = seeded((8192, 8192), 3, -1, 1), x = seeded(8192, 4, -1, 1)"
    else:
        raise SystemExit(f"unknown case {name}")
    sp = parse(text)
    env = {}
    for k, v in inputs.items():
        # fp32 inputs enter the interpreter as the exact float64 of each fp32
        env[k] = (v.astype(np.float64) if v.dtype == np.float32 else v).tolist()
    t0 = time.time()
    want = eval_phrase(sp.body, env, sigma)
    dt = time.time() - t0
    flat = want if isinstance(want, list) else [want]
    return {"program": "oracle/ref_programs/" + ("dot.dpia" if name.startswith("dot") else
                                                   "asum_proxy.dpia" if name.startswith("asum") else
                                                   "gemv.dpia"),
            "sigma": sigma, "inputs": desc, "result": flat,
            "interpreter": "dpia.eval_fn.eval_phrase (reference, Python numbers: float64 / int)",
            "seconds": round(dt, 1)}


def main(names):
    os.makedirs(OUT, exist_ok=True)
    for n in names:
        print(f"[fullsize] {n} ...", flush=True)
        res = case(n)
        print(f"[fullsize] {n}: {res['seconds']} s", flush=True)
        with open(os.path.join(OUT, n + ".json"), "w") as f:
            json.dump(res, f, sort_keys=True, separators=(",", ":"))
            f.write("\n")


if __name__ == "__main__":
    main(sys.argv[1:] or ["dot_literal_i64", "dot_literal_f32", "gemv_f32", "asum_abs_f32"])
