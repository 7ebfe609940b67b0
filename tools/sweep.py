"""Strategy/geometry sweep for the HBM-bound benchmark programs (GPU box).

    python tools/sweep.py asum|dot|gemv|gemvp   (gemvp: x staged toPrivate)

Prints achieved GB/s (median of event-timed launches, L2 scrubbed between
launches) for each (L, K, blocks) strategy parameterisation.
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import asum_config, dot_config, gemv_config, mm_config  # noqa: E402


def time_cfg(cfg, inputs, reps=20):
    exe = executable(compile_program(cfg.text, name=cfg.name), cfg.launch, cfg.sigma, float_mode=True)
    st = RT.Stream(0)
    for n, v in inputs.items():
        exe.upload(n, v, st)
    ts = []
    for i in range(reps + 3):
        RT.lib().dpia_l2_flush(0, st.handle)
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        exe.launch(st)
        e1.record(st)
        st.sync()
        if i >= 3:
            ts.append(e0.elapsed_ms(e1))
    return statistics.median(ts), min(ts)


def main(which):
    rng = np.random.default_rng(0)
    if which == "asum":
        inputs = {"xs": rng.uniform(-1, 1, 1 << 26).astype(np.float32)}
        grid = [(L, K, b) for L in (512, 1024) for K in (16, 32, 64, 128) for b in (None, 592, 1184)]
        mk = lambda L, K, b: asum_config(L=L, K=K, blocks=b)  # noqa: E731
    elif which in ("dotx", "asumx"):
        # small work-groups and exactly balanced grids: n chunks over G = n / k
        # groups (k chunks each, grid-stride), one wave or less
        if which == "dotx":
            inputs = {"xs": rng.uniform(0, 1, 1 << 24).astype(np.float32),
                      "ys": rng.uniform(0, 1, 1 << 24).astype(np.float32)}
            total, mkc = 1 << 24, dot_config
        else:
            inputs = {"xs": rng.uniform(-1, 1, 1 << 26).astype(np.float32)}
            total, mkc = 1 << 26, asum_config
        grid = []
        for L in (128, 256, 512, 1024):
            for K in (2, 4, 8, 16, 32):
                n = total // (4 * K * L)
                for per in (1, 2, 4, 8):
                    G = n // per
                    if G * L <= 148 * 2048 and G >= 148 and n % per == 0:
                        grid.append((L, K, None if per == 1 else G))
        mk = lambda L, K, b: mkc(L=L, K=K, blocks=b)  # noqa: E731
        which = which[:-1]
    elif which == "dot":
        inputs = {"xs": rng.uniform(0, 1, 1 << 24).astype(np.float32),
                  "ys": rng.uniform(0, 1, 1 << 24).astype(np.float32)}
        grid = [(L, K, b) for L in (512, 1024) for K in (8, 16, 32, 64) for b in (None, 592, 1184)]
        mk = lambda L, K, b: dot_config(L=L, K=K, blocks=b)  # noqa: E731
    elif which == "mm":
        inputs = {"A": rng.uniform(-1, 1, (4096, 4096)).astype(np.float32),
                  "B": rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)}
        grid = [(T, BK, R) for T, BK, R in ((128, 8, 8), (128, 16, 8), (64, 8, 4), (64, 16, 4),
                                            (128, 32, 8), (64, 32, 4))]
        mk = lambda T, BK, R: mm_config(T=T, BK=BK, R=R)  # noqa: E731
        for T, BK, R in grid:
            cfg = mk(T, BK, R)
            try:
                med, best = time_cfg(cfg, inputs, reps=10)
            except Exception as e:  # noqa: BLE001
                print(f"mm T={T} BK={BK} R={R}: {type(e).__name__} {str(e)[:200]}", flush=True)
                continue
            print(f"mm T={T:4d} BK={BK:3d} R={R}  median {med:8.3f} ms  {cfg.flops / med / 1e9:8.1f} TFLOP/s"
                  f"  best {cfg.flops / best / 1e9:8.1f}", flush=True)
        return
    else:
        inputs = {"A": rng.uniform(-1, 1, (8192, 8192)).astype(np.float32),
                  "x": rng.uniform(-1, 1, 8192).astype(np.float32)}
        xp = which == "gemvp"
        grid = [(L, None, b) for L in (128, 256, 512, 1024) for b in (148, 296, 592, 1184, 2368, 8192)]
        mk = lambda L, K, b: gemv_config(L=L, blocks=b, x_private=xp)  # noqa: E731
    for L, K, b in grid:
        try:
            cfg = mk(L, K, b)
        except AssertionError:
            continue
        try:
            med, best = time_cfg(cfg, inputs)
        except Exception as e:  # noqa: BLE001
            print(f"{which} L={L} K={K} G={cfg.launch[0]}: {type(e).__name__} {str(e)[:100]}", flush=True)
            continue
        print(f"{which} L={L:5d} K={K} G={cfg.launch[0]:6d}  median {med * 1e3:8.2f} us  "
              f"{cfg.bytes / med / 1e6:8.1f} GB/s   best {cfg.bytes / best / 1e6:8.1f} GB/s", flush=True)


if __name__ == "__main__":
    for w in sys.argv[1:] or ["asum"]:
        main(w)
