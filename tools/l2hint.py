"""Streaming-read load flavours at 128 / 256 MiB (GPU box; measurement only):

    python tools/l2hint.py

The same contiguous-chunk read + block combine (tagexp.rblock's shape) with
four load instructions: __ldg float4 (LDG.E.128.CONSTANT, what the emitter's
dpia::vload compiles to for const __restrict__ inputs), plain ld.global.v4,
ld.global.nc with an L2::256B prefetch hint, and ld.global.nc.L1::no_allocate.
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import runtime as RT  # noqa: E402

SRC = r"""
template <int MODE>
__device__ __forceinline__ float4 load4(const float4* p) {
  float4 v;
  if (MODE == 0) {
    v = __ldg(p);
  } else if (MODE == 1) {
    asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  } else if (MODE == 2) {
    asm volatile("ld.global.nc.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  }
  return v;
}

template <int MODE>
__device__ __forceinline__ void body(const float4* __restrict__ p, long long n4, float* out) {
  long long per = n4 / gridDim.x;
  const float4* q = p + blockIdx.x * per;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int k = per / blockDim.x;
  #pragma unroll 16
  for (int j = 0; j < k; ++j) {
    float4 v = load4<MODE>(q + (long long)j * blockDim.x + threadIdx.x);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  float s = acc.x + acc.y + acc.z + acc.w;
  __shared__ float red[32];
  for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) out[blockIdx.x] = t;
  }
}
extern "C" __global__ void __launch_bounds__(1024) r0(const float4* p, long long n4, float* o) { body<0>(p, n4, o); }
extern "C" __global__ void __launch_bounds__(1024) r1(const float4* p, long long n4, float* o) { body<1>(p, n4, o); }
extern "C" __global__ void __launch_bounds__(1024) r2(const float4* p, long long n4, float* o) { body<2>(p, n4, o); }
extern "C" __global__ void __launch_bounds__(1024) r3(const float4* p, long long n4, float* o) { body<3>(p, n4, o); }
"""
NAMES = {"r0": "__ldg", "r1": "ld.global", "r2": "ld.nc.L2::256B", "r3": "ld.nc.L1::no_allocate"}


def main():
    RT.init(0)
    st = RT.Stream(0)
    mod = RT.Module(RT.nvrtc_compile(SRC), 0)
    for nbytes in (1 << 27, 1 << 28):
        buf = RT.DeviceBuffer(nbytes)
        buf.upload(np.ones(nbytes // 4, np.float32), st)
        out = RT.DeviceBuffer(8192)
        args = [RT.C.c_uint64(buf.ptr), RT.C.c_longlong(nbytes // 16), RT.C.c_uint64(out.ptr)]
        for rnd in range(2):
            for k in ("r0", "r1", "r2", "r3"):
                fn = mod.function(k)
                ts = []
                for i in range(65):
                    RT.lib().dpia_l2_flush(0, st.handle)
                    e0, e1 = RT.Event(0), RT.Event(0)
                    e0.record(st)
                    RT.launch(fn, 0, (256, 1), (1024, 1), 0, args, st)
                    e1.record(st)
                    st.sync()
                    if i >= 5:
                        ts.append(e0.elapsed_ms(e1))
                t = statistics.mean(ts) * 1e3
                print(f"{nbytes >> 20:4d} MiB round {rnd} {NAMES[k]:22s}: {t:7.2f} us  {nbytes / t / 1e3:6.0f} GB/s",
                      flush=True)
        buf.free()


if __name__ == "__main__":
    main()
