"""Launch geometry of BASELINE config 1's literal program (GPU box;
measurement infrastructure, not product).

    python tools/litgeo.py

oracle/ref_programs/dot.dpia as the reference states it -- mapGlobal over
16384 chunks of 1024 pairs, reduceSeq per chunk, a top-level sequential
reduce -- timed like bench.py at several (G, L) with G * L = 16384 work-items
(one chunk each) and with fewer work-items striding over the chunks.  Also
the same program without the top-level reduce (the 16384 partials only),
which isolates the cost of the single-thread tail.
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import dot_literal_program  # noqa: E402

PARTIALS = """
(nat n)
(param xs (exp (array (* n 1024) num)))
(param ys (exp (array (* n 1024) num)))
(mapGlobal (lam (c (exp (array 1024 (pair num num))))
   (reduce (lam (x (exp (pair num num))) (lam (a (exp num)) (+ (* (fst x) (snd x)) a))) 0 c))
  (split 1024 (zip xs ys)))
"""


def timed(st, exe, reps=50):
    ts = []
    for it in range(reps + 5):
        RT.lib().dpia_l2_flush(0, st.handle)
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        exe.launch(st)
        e1.record(st)
        st.sync()
        if it >= 5:
            ts.append(e0.elapsed_ms(e1))
    return statistics.mean(ts) * 1e3


def main():
    RT.init(0)
    st = RT.Stream(0)
    n = 16384
    rng = np.random.default_rng(0)
    xs = rng.uniform(0, 1, n * 1024).astype(np.float32)
    ys = rng.uniform(0, 1, n * 1024).astype(np.float32)
    for tag, text in (("literal", dot_literal_program()), ("partials-only", PARTIALS)):
        prog = compile_program(text, name="lit")
        launches = ((64, 256), (128, 128), (256, 64), (512, 32), (148, 128), (296, 32), (32, 512))
        if "--quick" in sys.argv:
            launches = ((128, 128), (512, 32))
        for launch in launches:
            exe = executable(prog, launch, {"n": n}, float_mode=True)
            exe.upload("xs", xs, st)
            exe.upload("ys", ys, st)
            us = timed(st, exe)
            print(f"{tag:14s} launch={launch}: {us:8.2f} us  {8 * n * 1024 / us / 1e3:7.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
