"""Prefetch depth of the vectorised sequential folds (GPU box; measurement
infrastructure, not product).

    python tools/litpf.py

BASELINE config 1's literal program (oracle/ref_programs/dot.dpia) and its
partials-only half (tools/litgeo.py PARTIALS), timed like bench.py at a few
geometries for several depths of the rotating register queue the emitter
gives each read stream of a long sequential fold (cuda/emit.py
VEC_PREFETCH for the per-work-item chunk folds, VEC_PREFETCH_SINGLE for the
single-thread top-level fold of the fused tail; 0 = no queue, the round-2
vectorised fold).  Also checks that every variant returns the same bits.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import dot_literal_program  # noqa: E402
from paper_1710_08332_b200.cuda import emit as EM  # noqa: E402
from litgeo import PARTIALS, timed  # noqa: E402


def main():
    RT.init(0)
    st = RT.Stream(0)
    n = 16384
    rng = np.random.default_rng(0)
    xs = rng.uniform(0, 1, n * 1024).astype(np.float32)
    ys = rng.uniform(0, 1, n * 1024).astype(np.float32)
    launches = ((512, 32), (256, 64), (128, 128))
    results = {}
    for item_d, tail_d in ((0, 0), (4, 0), (8, 0), (16, 0), (8, 16), (8, 32), (8, 64), (16, 32)):
        EM.VEC_PREFETCH, EM.VEC_PREFETCH_SINGLE = item_d, tail_d
        for tag, text in (("literal", dot_literal_program()), ("partials", PARTIALS)):
            if tag == "partials" and tail_d not in (0,):
                continue
            prog = compile_program(text, name="lit")
            for launch in launches:
                exe = executable(prog, launch, {"n": n}, float_mode=True)
                exe.upload("xs", xs, st)
                exe.upload("ys", ys, st)
                us = timed(st, exe)
                out = exe.download("out", st)
                st.sync()
                bits = np.asarray(out, np.float32).tobytes()
                results.setdefault((tag, launch), set()).add(bits)
                print(f"item_d={item_d:2d} tail_d={tail_d:2d} {tag:9s} launch={launch}: {us:8.2f} us  "
                      f"{8 * n * 1024 / us / 1e3:7.1f} GB/s", flush=True)
    for k, v in results.items():
        print(k, "identical bits across depths" if len(v) == 1 else f"{len(v)} DIFFERENT results")


if __name__ == "__main__":
    main()
