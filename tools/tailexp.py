"""Cost of the fused grid combine: dot with and without the final reduceLocal."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.sweep import time_cfg  # noqa: E402
from paper_1710_08332_b200.bench_programs import Config, dot_config, dot_program  # noqa: E402


def partials_program(L, K):
    full = dot_program(L, K)
    # drop the outer (reduceLocal (+) 0 ...) : keep the per-work-group partials
    body = full[full.index("(asScalar4"):]
    body = body.rstrip()[:-1]  # remove the reduceLocal's closing paren
    return full[:full.index("(reduceLocal (+) 0\n (asScalar4")] + body


def main():
    rng = np.random.default_rng(0)
    xs, ys = rng.uniform(0, 1, 1 << 24).astype(np.float32), rng.uniform(0, 1, 1 << 24).astype(np.float32)
    for L, K in ((1024, 16), (512, 32), (1024, 8)):
        cfg = dot_config(L=L, K=K)
        med, _ = time_cfg(cfg, {"xs": xs, "ys": ys})
        pc = Config("dotp", partials_program(L, K), cfg.sigma, cfg.launch, bytes=cfg.bytes)
        med2, _ = time_cfg(pc, {"xs": xs, "ys": ys})
        print(f"L={L} K={K}: fused {med*1e3:.2f} us ({cfg.bytes/med/1e6:.0f} GB/s)  partials only "
              f"{med2*1e3:.2f} us ({cfg.bytes/med2/1e6:.0f} GB/s)", flush=True)


if __name__ == "__main__":
    main()
