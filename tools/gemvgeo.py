"""gemv launch geometries with exactly balanced row counts (GPU box; means of 60).

    python tools/gemvgeo.py
"""
import sys, statistics
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
from geomean import mean_us
from paper_1710_08332_b200 import runtime as RT
from paper_1710_08332_b200.bench_programs import gemv_config
RT.init(0); st = RT.Stream(0)
rng = np.random.default_rng(0)
inp = {"A": rng.uniform(-1, 1, (8192, 8192)).astype(np.float32), "x": rng.uniform(-1, 1, 8192).astype(np.float32)}
for rnd in range(2):
    for L, b in ((256, 1184), (256, 1024), (256, 2048), (256, 4096), (256, 8192), (512, 1024), (512, 2048), (128, 2048), (128, 4096)):
        try:
            cfg = gemv_config(L=L, blocks=b)
        except Exception as e:
            print(L, b, e); continue
        t = mean_us(cfg, inp, st)
        print(f"round {rnd} gemv L={L} G={b}: {t:7.2f} us {cfg.bytes / t / 1e3:7.1f} GB/s", flush=True)
