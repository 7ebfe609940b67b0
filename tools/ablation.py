"""Strategy ablation (GPU box): the benchmark problems written only with the
reference's primitives (oracle/ref_programs/*.dpia -- no transpose, abs,
reduceLocal, let, 2-D maps), compiled by the same CUDA backend, against the
B200 strategies of bench_programs.py.  Shows what the added primitives buy."""
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import asum_config, dot_config, gemv_config  # noqa: E402


def timed(text, launch, sigma, inputs, reps=5):
    exe = executable(compile_program(text), launch, sigma, float_mode=True)
    st = RT.Stream(0)
    for n, v in inputs.items():
        exe.upload(n, v, st)
    ts = []
    for i in range(reps + 2):
        RT.lib().dpia_l2_flush(0, st.handle)
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        exe.launch(st)
        e1.record(st)
        st.sync()
        if i >= 2:
            ts.append(e0.elapsed_ms(e1))
    return statistics.median(ts), exe.download("out")


def main():
    rng = np.random.default_rng(0)
    ref = lambda name: open(os.path.join(ROOT, "oracle", "ref_programs", name + ".dpia")).read()  # noqa
    xs = rng.uniform(-1, 1, 1 << 26).astype(np.float32)
    rows = []
    t, _ = timed(ref("asum_proxy"), (148 * 8, 256), {"n": (1 << 26) // 1024}, {"xs": xs})
    rows.append(("asum 2^26", "reference primitives: mapGlobal over 1024-chunks + top-level reduce",
                 4 << 26, t))
    cfg = asum_config()
    t2, _ = timed(cfg.text, cfg.launch, cfg.sigma, {"xs": xs})
    rows.append(("asum 2^26", "B200 strategy (transpose, abs, reduceLocal)", 4 << 26, t2))
    x24, y24 = xs[:1 << 24].copy(), xs[1 << 24:2 << 24].copy()
    t, _ = timed(ref("dot"), (148 * 8, 256), {"n": (1 << 24) // 1024}, {"xs": x24, "ys": y24})
    rows.append(("dot 2^24", "reference primitives: mapGlobal + reduceSeq per 1024-chunk + top-level reduce",
                 8 << 24, t))
    cfg = dot_config()
    t2, _ = timed(cfg.text, cfg.launch, cfg.sigma, {"xs": x24, "ys": y24})
    rows.append(("dot 2^24", "B200 strategy (asVector4, transpose, reduceLocal)", 8 << 24, t2))
    A = rng.uniform(-1, 1, (8192, 8192)).astype(np.float32)
    x = rng.uniform(-1, 1, 8192).astype(np.float32)
    t, _ = timed(ref("gemv"), (592, 256), {}, {"A": A, "x": x})
    rows.append(("gemv 8192^2", "reference primitives: row per work-group, toLocal partials, seq combine",
                 4 * (8192 * 8192 + 2 * 8192), t))
    cfg = gemv_config()
    t2, _ = timed(cfg.text, cfg.launch, cfg.sigma, {"A": A, "x": x})
    rows.append(("gemv 8192^2", "B200 strategy (vec4, let/LICM toLocal x, reduceLocal)",
                 4 * (8192 * 8192 + 2 * 8192), t2))
    for name, strat, nbytes, t in rows:
        print(f"{name:12s} {t * 1e3:10.1f} us {nbytes / t / 1e6:8.0f} GB/s   {strat}", flush=True)


if __name__ == "__main__":
    main()
