"""Mean event time (60 launches, L2 scrubbed) of a few asum / dot launch
geometries (GPU box).  The event clock ticks in ~2 us steps on this box, so
sweep medians are coarse; this compares means.

    python tools/geomean.py
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import asum_config, dot_config  # noqa: E402


def mean_us(cfg, inputs, st, reps=60):
    exe = executable(compile_program(cfg.text, name=cfg.name), cfg.launch, cfg.sigma, float_mode=True)
    for n, v in inputs.items():
        exe.upload(n, v, st)
    ts = []
    for i in range(reps + 5):
        RT.lib().dpia_l2_flush(0, st.handle)
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        exe.launch(st)
        e1.record(st)
        st.sync()
        if i >= 5:
            ts.append(e0.elapsed_ms(e1))
    return statistics.mean(ts) * 1e3


def main():
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(0)
    xa = {"xs": rng.uniform(-1, 1, 1 << 26).astype(np.float32)}
    xd = {"xs": rng.uniform(0, 1, 1 << 24).astype(np.float32), "ys": rng.uniform(0, 1, 1 << 24).astype(np.float32)}
    for rnd in range(2):
        for L, K, b in ((1024, 32, None), (1024, 64, None), (1024, 32, 256), (1024, 16, 256), (512, 64, None),
                        (1024, 128, None)):
            cfg = asum_config(L=L, K=K, blocks=b)
            t = mean_us(cfg, xa, st)
            print(f"round {rnd} asum L={L} K={K} G={cfg.launch[0]}: {t:7.2f} us {cfg.bytes / t / 1e3:7.1f} GB/s",
                  flush=True)
        for L, K, b in ((1024, 16, None), (1024, 32, None), (1024, 8, 256), (512, 32, None)):
            cfg = dot_config(L=L, K=K, blocks=b)
            t = mean_us(cfg, xd, st)
            print(f"round {rnd} dot  L={L} K={K} G={cfg.launch[0]}: {t:7.2f} us {cfg.bytes / t / 1e3:7.1f} GB/s",
                  flush=True)


if __name__ == "__main__":
    main()
