import os, sys, statistics
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_1710_08332_b200 import compile_program, executable
from paper_1710_08332_b200 import runtime as RT
RT.init(0); st = RT.Stream(0)
text = open("oracle/ref_programs/gemv.dpia").read()
A = np.random.default_rng(3).uniform(-1, 1, (8192, 8192)).astype(np.float32)
x = np.random.default_rng(4).uniform(-1, 1, 8192).astype(np.float32)
for G in (592, 1184, 296, 8192):
    exe = executable(compile_program(text, name="gemv_lit"), (G, 256), {}, float_mode=True)
    exe.upload("A", A, st); exe.upload("x", x, st)
    ts = []
    for it in range(25):
        RT.lib().dpia_l2_flush(0, st.handle)
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st); exe.launch(st); e1.record(st); st.sync()
        if it >= 5: ts.append(e0.elapsed_ms(e1))
    ms = statistics.median(ts)
    y = np.asarray(exe.download("out", st)); st.sync()
    err = np.max(np.abs(y - A.astype(np.float64) @ x))
    print(f"G={G}: {ms*1e3:.1f} us {4*(8192*8192+2*8192)/ms/1e6:.1f} GB/s maxerr {err:.2e} kernels {[k.name for k in exe.sig.kernels]} smem {[k.smem for k in exe.sig.kernels]}", flush=True)
