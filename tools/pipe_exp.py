"""mm end to end from page-locked host memory (GPU box): Executable.run
(copy A, B in; one launch; copy C out) against pipeline.mm_pipeline with
2/4/8 row chunks (copies overlapped with the chunk kernels) and
pipeline.mm_tile_pipeline with rows x cols output tiles on several compute
streams.

    python tools/pipe_exp.py
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import mm_config  # noqa: E402
from paper_1710_08332_b200.pipeline import mm_pipeline, mm_tile_pipeline  # noqa: E402


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
    M = N = K = 4096
    rng = np.random.default_rng(0)
    pins = [RT.PinnedBuffer(4 * M * K), RT.PinnedBuffer(4 * K * N), RT.PinnedBuffer(4 * M * N)]
    A, B, C = (pins[0].array(np.float32, M * K), pins[1].array(np.float32, K * N),
               pins[2].array(np.float32, M * N))
    A[:] = rng.uniform(-1, 1, M * K)
    B[:] = rng.uniform(-1, 1, K * N)
    flops = 2 * M * N * K
    cfg = mm_config()
    exe = executable(compile_program(cfg.text, name="mm"), cfg.launch, cfg.sigma)
    ms = timed(lambda: exe.run({"A": A, "B": B}, st, out={"out": C}), st)
    ref = C.copy()
    print(f"Executable.run: {ms:.3f} ms  {flops / ms / 1e9:.2f} TFLOP/s", flush=True)
    for chunks in (2, 4, 8, 16):
        pipe = mm_pipeline(M, N, K, chunks=chunks)
        C[:] = 0
        ms = timed(lambda: pipe.run({"A": A, "B": B}, C, st), st)
        print(f"mm_pipeline chunks={chunks}: {ms:.3f} ms  {flops / ms / 1e9:.2f} TFLOP/s  "
              f"same={np.array_equal(C, ref)}", flush=True)
    import time
    for rows, cols, streams in ((2, 2, 2), (2, 2, 4), (4, 4, 1), (4, 4, 2), (4, 4, 4), (4, 4, 8), (4, 4, 12),
                                (4, 4, 16), (2, 4, 8), (4, 2, 8), (8, 4, 8), (4, 8, 8), (8, 8, 8),
                                (8, 8, 16)):
        pipe = mm_tile_pipeline(M, N, K, rows=rows, cols=cols, compute_streams=streams)
        C[:] = 0
        ms = timed(lambda: pipe.run({"A": A, "B": B}, C, st), st)
        t0 = time.perf_counter()
        pipe.run({"A": A, "B": B}, C, st)
        host = (time.perf_counter() - t0) * 1e3
        print(f"host wall of one run (enqueue + wait) {host:.3f} ms; ", end="")
        print(f"mm_tile_pipeline {rows}x{cols} streams={streams}: {ms:.3f} ms  {flops / ms / 1e9:.2f} TFLOP/s  "
              f"same={np.array_equal(C, ref)}", flush=True)


if __name__ == "__main__":
    main()
