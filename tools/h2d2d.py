"""Pinned H2D rate of pitched column-panel copies (dpia_memcpy2d_htod) against
1-D copies of the same 64 MiB (GPU box; measurement infrastructure)."""
import sys, statistics, ctypes
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1710_08332_b200 import runtime as RT
RT.init(0); st = RT.Stream(0)
M = 4096
pin = RT.PinnedBuffer(4 * M * M); h = pin.array(np.float32, M * M); h[:] = 1
d = RT.DeviceBuffer(4 * M * M)
def t(fn, reps=10):
    ts = []
    for i in range(reps + 2):
        e0, e1 = RT.Event(0), RT.Event(0); e0.record(st); fn(); e1.record(st); st.sync()
        if i >= 2: ts.append(e0.elapsed_ms(e1))
    return statistics.mean(ts)
def one_d():
    for k in range(4):
        nb = 16 << 20
        RT.lib().dpia_memcpy_htod(0, d.ptr + k * nb, ctypes.c_void_p(h.ctypes.data + k * nb), nb, st.handle)
for cols in (2, 4, 8):
    tn = M // cols
    def two_d():
        for k in range(cols):
            RT.lib().dpia_memcpy2d_htod(0, d.ptr + k * M * tn * 4, tn * 4, ctypes.c_void_p(h.ctypes.data + k * tn * 4), M * 4, tn * 4, M, st.handle)
    ms = t(two_d); print(f"2D panels cols={cols}: {ms:.3f} ms  {64 * 1.048576 / ms:.1f} GB/s")
ms = t(one_d); print(f"1D 4 x 16 MiB: {ms:.3f} ms  {64 * 1.048576 / ms:.1f} GB/s")
