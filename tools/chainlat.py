"""Dependent-chain latency of the fp32 add forms a sequential fold can use
(GPU box; measurement infrastructure, not product).

    python tools/chainlat.py

One thread runs 2^16 dependent `acc = acc + v[i]` steps over values held in
registers (no memory in the loop) and reports clock64 cycles per step for
  fadd       add.rn.f32           (FADD)
  ffma1      fma.rn.f32 v, 1, acc (FFMA; the same single rounding as FADD,
             so the result is bit-identical)
  ffma       fma.rn.f32 v, w, acc (the dot work-item fold, FFMA)
The results of the three add forms are compared bit for bit.
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import runtime as RT  # noqa: E402

SRC = r"""
extern "C" __global__ void chain(const float* __restrict__ v, float* out, long long* cyc, int mode) {
  float r[32];
  #pragma unroll
  for (int k = 0; k < 32; ++k) r[k] = v[k];
  float acc = 0.0f;
  long long t0 = clock64();
  for (int it = 0; it < 2048; ++it) {
    if (mode == 0) {
      #pragma unroll
      for (int k = 0; k < 32; ++k) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(acc) : "f"(r[k]));
    } else if (mode == 1) {
      #pragma unroll
      for (int k = 0; k < 32; ++k) asm volatile("fma.rn.f32 %0, %1, 0f3F800000, %0;" : "+f"(acc) : "f"(r[k]));
    } else {
      #pragma unroll
      for (int k = 0; k < 32; ++k) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc) : "f"(r[k]), "f"(r[31 - k]));
    }
  }
  long long t1 = clock64();
  out[mode] = acc;
  cyc[mode] = t1 - t0;
}
"""


def main():
    RT.init(0)
    st = RT.Stream(0)
    fn = RT.Module(RT.get_cubin(SRC), 0).function("chain")
    v = RT.DeviceBuffer(128, 0)
    v.upload(np.random.default_rng(0).uniform(0, 1, 32).astype(np.float32), st)
    out, cyc = RT.DeviceBuffer(16, 0), RT.DeviceBuffer(32, 0)
    for mode in (0, 1, 2):
        for _ in range(3):
            RT.launch(fn, 0, (1, 1), (1, 1), 0,
                      [RT.C.c_uint64(v.ptr), RT.C.c_uint64(out.ptr), RT.C.c_uint64(cyc.ptr), ctypes.c_int(mode)], st)
    st.sync()
    o = np.empty(4, np.float32)
    c = np.empty(4, np.int64)
    out.download(o.view(np.uint8), st)
    cyc.download(c.view(np.uint8), st)
    st.sync()
    for mode, name in enumerate(("fadd", "ffma1", "ffma")):
        print(f"{name:6s}: {c[mode] / 65536:6.2f} cycles per dependent step  result {o[mode]!r}")
    print("fadd and ffma1 bit-identical:", o[0].tobytes() == o[1].tobytes())


if __name__ == "__main__":
    main()
