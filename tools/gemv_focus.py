"""gemv staging variants (x in shared memory vs x_private registers) across
work-group sizes and grid sizes, checked against float64 numpy (GPU box).

    python tools/gemv_focus.py
"""
import os, sys, statistics
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1710_08332_b200 import compile_program, executable
from paper_1710_08332_b200 import runtime as RT
from paper_1710_08332_b200.bench_programs import gemv_config
rng = np.random.default_rng(0)
A = rng.uniform(-1, 1, (8192, 8192)).astype(np.float32); x = rng.uniform(-1, 1, 8192).astype(np.float32)
st = RT.Stream(0)
want = A.astype(np.float64) @ x
for rep in range(2):
  for xp, L, G in ((False, 512, 592), (True, 256, 592), (True, 256, 1184), (True, 128, 8192), (True, 512, 8192), (True, 256, 2368), (True, 256, 296), (True, 1024, 592)):
    cfg = gemv_config(L=L, blocks=G, x_private=xp)
    exe = executable(compile_program(cfg.text, name="gemv"), cfg.launch, cfg.sigma, float_mode=True)
    exe.upload("A", A, st); exe.upload("x", x, st)
    ts = []
    for i in range(65):
        RT.lib().dpia_l2_flush(0, st.handle)
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st); exe.launch(st); e1.record(st); st.sync()
        if i >= 5: ts.append(e0.elapsed_ms(e1))
    y = exe.download("out", st)
    err = np.max(np.abs(y - want))
    m = statistics.mean(ts)
    print(f"x_private={xp} L={L} G={G}: mean {m*1e3:.2f} us  {cfg.bytes/m/1e6:.0f} GB/s  err {err:.1e}", flush=True)
