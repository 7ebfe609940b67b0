"""The reference's own gemv program (BASELINE config 3 as the reference
states it, oracle/ref_programs/gemv.dpia) over launch geometries (GPU box;
measurement infrastructure, not product).

    python tools/gemvlit_probe.py

L2 scrub before each launch, CUDA events, median of 20; max |error| against
the float64 product."""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import gemv_literal_program  # noqa: E402


def main():
    RT.init(0)
    st = RT.Stream(0)
    A = np.random.default_rng(3).uniform(-1, 1, (8192, 8192)).astype(np.float32)
    x = np.random.default_rng(4).uniform(-1, 1, 8192).astype(np.float32)
    want = A.astype(np.float64) @ x
    prog = compile_program(gemv_literal_program(), name="gemv_literal")
    for G, L in ((592, 256), (444, 256), (740, 256), (888, 256), (592, 128), (888, 128), (1184, 128),
                 (296, 512), (8192, 256)):
        exe = executable(prog, (G, L), {}, float_mode=True)
        exe.upload("A", A, st)
        exe.upload("x", x, st)
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
        print(f"({G:5d}, {L:4d}): {ms * 1e3:7.1f} us  {4 * (8192 * 8192 + 2 * 8192) / ms / 1e6:7.1f} GB/s  "
              f"max|err| {np.max(np.abs(y - want)):.2e}  smem {exe.sig.kernels[0].smem}", flush=True)


if __name__ == "__main__":
    main()
