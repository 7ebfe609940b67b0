"""Launch geometry of dot and asum under steady-state timing (GPU box;
measurement infrastructure, not product).

    python tools/steadygeo.py

tools/steadystate.py's back-to-back measurement (rotating input sets
larger than 3 x L2, one event pair over K steps) for the dot / asum
strategies at several (work-group size L, vec4 per work-item K, grid).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import asum_config, dot_config  # noqa: E402
from steadystate import measure  # noqa: E402


def main():
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(0)
    for L, K, blocks in ((1024, 16, None), (1024, 8, None), (512, 32, None), (512, 16, None),
                         (512, 8, None), (256, 32, None), (256, 16, None), (1024, 4, 296),
                         (512, 8, 296), (256, 16, 592), (1024, 2, 296), (768, 8, None)):
        try:
            cfg = dot_config(L=L, K=K, blocks=blocks)
        except AssertionError:
            continue
        iso, ss, R, runs = measure("dot", cfg, {"xs": 1 << 24, "ys": 1 << 24}, st, rng)
        print(f"dot  L={L:4d} K={K:2d} wg={cfg.sigma['n']:5d} grid={cfg.launch[0]:5d}: isolated {iso:6.2f} us "
              f"steady {ss:6.2f} us frac {cfg.bytes / ss / 1e3 / 6554.9:.3f}", flush=True)
    for L, K, blocks in ((1024, 64, None), (1024, 32, None), (512, 64, None), (512, 32, None),
                         (256, 64, None), (1024, 16, 296)):
        try:
            cfg = asum_config(L=L, K=K, blocks=blocks)
        except AssertionError:
            continue
        iso, ss, R, runs = measure("asum", cfg, {"xs": 1 << 26}, st, rng)
        print(f"asum L={L:4d} K={K:2d} wg={cfg.sigma['n']:5d} grid={cfg.launch[0]:5d}: isolated {iso:6.2f} us "
              f"steady {ss:6.2f} us frac {cfg.bytes / ss / 1e3 / 6554.9:.3f}", flush=True)


if __name__ == "__main__":
    main()
