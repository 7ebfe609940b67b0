"""scal 2^26 end to end from page-locked host memory (GPU box): Executable.run
against pipeline.scal_pipeline with 2..32 blocks.

    python tools/pipe_scal.py
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import scal_config  # noqa: E402
from paper_1710_08332_b200.pipeline import scal_pipeline  # noqa: E402


def timed(fn, st, reps=6):
    ts = []
    for i in range(reps + 1):
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        fn()
        e1.record(st)
        st.sync()
        if i:
            ts.append(e0.elapsed_ms(e1))
    return statistics.mean(ts)


def main():
    RT.init(0)
    st = RT.Stream(0)
    N = 1 << 26
    pins = [RT.PinnedBuffer(16), RT.PinnedBuffer(4 * N), RT.PinnedBuffer(4 * N)]
    ha, hx, out = pins[0].array(np.float32, 4), pins[1].array(np.float32, N), pins[2].array(np.float32, N)
    ha[:] = 1.5
    hx[:] = np.random.default_rng(0).uniform(-1, 1, N)
    cfg = scal_config()
    exe = executable(compile_program(cfg.text, name="scal"), cfg.launch, cfg.sigma)
    ms = timed(lambda: exe.run({"alpha": ha, "xs": hx}, st, out={"out": out}), st)
    ref = out.copy()
    print(f"Executable.run: {ms:.3f} ms  {cfg.bytes / ms / 1e6:.1f} GB/s", flush=True)
    for chunks in (2, 4, 8, 16, 32):
        pipe = scal_pipeline(N, chunks=chunks)
        out[:] = 0
        ms = timed(lambda: pipe.run({"alpha": ha, "xs": hx}, out, st), st)
        print(f"scal_pipeline blocks={chunks}: {ms:.3f} ms  {cfg.bytes / ms / 1e6:.1f} GB/s  "
              f"same={np.array_equal(out, ref)}", flush=True)


if __name__ == "__main__":
    main()
