import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from tools.sweep import time_cfg
from paper_1710_08332_b200.bench_programs import asum_config, dot_config
rng = np.random.default_rng(0)
for N in (1 << 25, 1 << 26):
    for L, K in ((1024, 16), (1024, 32), (512, 32)):
        try:
            cfg = asum_config(N=N, L=L, K=K)
        except AssertionError:
            continue
        med, best = time_cfg(cfg, {"xs": rng.uniform(-1, 1, N).astype(np.float32)})
        print(f"asum N=2^{N.bit_length()-1} L={L} K={K} G={cfg.launch[0]}: {cfg.bytes/med/1e6:.0f} GB/s ({med*1e3:.2f} us)", flush=True)
for N in (1 << 24, 1 << 25):
    for L, K in ((1024, 16), (1024, 8), (512, 16)):
        cfg = dot_config(N=N, L=L, K=K)
        med, best = time_cfg(cfg, {"xs": rng.uniform(0, 1, N).astype(np.float32), "ys": rng.uniform(0, 1, N).astype(np.float32)})
        print(f"dot N=2^{N.bit_length()-1} L={L} K={K} G={cfg.launch[0]}: {cfg.bytes/med/1e6:.0f} GB/s ({med*1e3:.2f} us)", flush=True)
