"""Config 1's literal program (dot_literal) emitted with and without the
streaming tail over launch geometries of 1..8 work-item rounds (GPU box;
measurement infrastructure, not product).

    python tools/litstream.py

Each variant: L2 scrub before each launch, CUDA events, median of 30, and the
result compared bit for bit with the ticket-tail kernel at (512, 32).
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import dot_literal_program  # noqa: E402
from paper_1710_08332_b200.cuda import emit as EM  # noqa: E402


def timed(st, fn, reps=30):
    ts = []
    for it in range(reps + 5):
        RT.lib().dpia_l2_flush(0, st.handle)
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        fn()
        e1.record(st)
        st.sync()
        if it >= 5:
            ts.append(e0.elapsed_ms(e1))
    return statistics.median(ts) * 1e3


def main():
    RT.init(0)
    st = RT.Stream(0)
    n, chunk = 16384, 1024
    rng = np.random.default_rng(0)
    xs = rng.uniform(0, 1, n * chunk).astype(np.float32)
    ys = rng.uniform(0, 1, n * chunk).astype(np.float32)
    prog = compile_program(dot_literal_program(chunk), name="dot_literal")
    ref = None
    geoms = [(512, 32), (256, 32), (128, 32), (64, 32), (256, 64), (128, 64), (64, 128)]
    for stream, rows in ((False, False), (True, False), (True, True), (False, True)):
        for G, L in geoms if stream else geoms[:1]:
            EM.STREAM_TAIL, EM.ROW_TMA = stream, rows
            exe = executable(prog, (G, L), {"n": n}, float_mode=True)
            exe.upload("xs", xs, st)
            exe.upload("ys", ys, st)
            us = timed(st, lambda: exe.launch(st))
            out = np.asarray(exe.download("out", st))
            st.sync()
            ref = out if ref is None else ref
            R = -(-n // (G * L))
            print(f"stream={int(stream)} rows={int(rows)} ({G:3d},{L:3d}) rounds={R}: {us:8.2f} us  "
                  f"{8 * n * chunk / us / 1e3:7.1f} GB/s  extra_blocks={exe.sig.kernels[0].extra_blocks}  "
                  f"{'==' if out.view(np.uint32)[0] == ref.view(np.uint32)[0] else '!='} ticket tail",
                  flush=True)


if __name__ == "__main__":
    main()
