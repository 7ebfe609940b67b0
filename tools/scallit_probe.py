"""The reference's own scal program (oracle/ref_programs/scal.dpia: mapGlobal
over 1024-element chunks, each scaled sequentially) over launch geometries
(GPU box; measurement infrastructure, not product).

    python tools/scallit_probe.py

L2 scrub before each launch, CUDA events, median of 20; checked against
numpy."""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402

TEXT = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "ref_programs",
                         "scal.dpia")).read()


def main():
    RT.init(0)
    st = RT.Stream(0)
    n = 65536
    xs = np.random.default_rng(7).uniform(-1, 1, n * 1024).astype(np.float32)
    prog = compile_program(TEXT, name="scal_literal")
    for G, L in ((512, 32), (256, 32), (2048, 32), (512, 128), (148 * 8, 64)):
        exe = executable(prog, (G, L), {"n": n}, float_mode=True)
        exe.upload("alpha", np.float32([1.5]), st)
        exe.upload("xs", xs, st)
        ts = []
        for it in range(25):
            RT.lib().dpia_l2_flush(0, st.handle)
            e0, e1 = RT.Event(0), RT.Event(0)
            e0.record(st)
            exe.launch(st)
            e1.record(st)
            st.sync()
            if it >= 5:
                ts.append(e0.elapsed_ms(e1))
        ms = statistics.median(ts)
        y = np.asarray(exe.download("out", st))
        st.sync()
        print(f"({G:5d}, {L:4d}): {ms * 1e3:7.1f} us  {8 * n * 1024 / ms / 1e6:7.1f} GB/s  "
              f"exact {np.array_equal(y, (np.float32(1.5) * xs))}", flush=True)


if __name__ == "__main__":
    main()
