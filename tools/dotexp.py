"""Grid-geometry probe for the 2^24 dot and 2^26 asum (GPU box)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.sweep import time_cfg  # noqa: E402
from paper_1710_08332_b200.bench_programs import asum_config, dot_config  # noqa: E402

rng = np.random.default_rng(0)
xs, ys = rng.uniform(0, 1, 1 << 24).astype(np.float32), rng.uniform(0, 1, 1 << 24).astype(np.float32)
for L, K, G in ((1024, 4, 296), (1024, 2, 296), (512, 4, 592), (512, 8, 592), (1024, 4, 592),
                (256, 8, 1184), (1024, 16, None), (1024, 8, None), (1024, 4, None), (512, 16, 296)):
    cfg = dot_config(L=L, K=K, blocks=G)
    med, best = time_cfg(cfg, {"xs": xs, "ys": ys})
    print(f"dot L={L} K={K} chunks={cfg.sigma['n']} G={cfg.launch[0]}: {cfg.bytes/med/1e6:.0f} GB/s "
          f"({med*1e3:.2f} us) best {cfg.bytes/best/1e6:.0f}", flush=True)
xa = rng.uniform(-1, 1, 1 << 26).astype(np.float32)
for L, K, G in ((1024, 4, 296), (1024, 8, 296), (1024, 16, 296), (512, 8, 592), (1024, 32, None)):
    cfg = asum_config(L=L, K=K, blocks=G)
    med, best = time_cfg(cfg, {"xs": xa})
    print(f"asum L={L} K={K} chunks={cfg.sigma['n']} G={cfg.launch[0]}: {cfg.bytes/med/1e6:.0f} GB/s "
          f"({med*1e3:.2f} us) best {cfg.bytes/best/1e6:.0f}", flush=True)
