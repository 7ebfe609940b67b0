"""Measured FP32 FMA peak of this B200 (GPU box):

    python tools/ffmapeak.py

A register-only kernel: every thread runs ITERS rounds over 16 independent
accumulators (scalar FFMA) or 16 independent accumulator pairs (packed
fma.rn.f32x2 = FFMA2), launched as 148 x BLOCKS_PER_SM CTAs of 256 threads.
Timed with CUDA events (mean of 10 after warm-up). This is the achievable
FFMA issue ceiling that bench.py's computed 148 x 128 x 2 x clock peak
assumes. Measurement infrastructure only; not product code.
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import runtime as RT  # noqa: E402

ITERS = 4096
SRC = r"""
extern "C" __global__ void __launch_bounds__(256) ffma1(float* out, float a, float b, int iters) {
  float c[16];
  #pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fmaf(a, c[i], b);
  }
  float s = 0.f;
  #pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 1.2345f) out[0] = s;
}
extern "C" __global__ void __launch_bounds__(256) ffma2(float* out, float a, float b, int iters) {
  unsigned long long c[16];
  unsigned long long av, bv;
  asm("mov.b64 %0, {%1,%1};" : "=l"(av) : "f"(a));
  asm("mov.b64 %0, {%1,%1};" : "=l"(bv) : "f"(b));
  #pragma unroll
  for (int i = 0; i < 16; ++i) {
    float x = threadIdx.x * 1e-3f + i;
    asm("mov.b64 %0, {%1,%2};" : "=l"(c[i]) : "f"(x), "f"(x + 0.5f));
  }
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(c[i]) : "l"(av), "l"(bv));
  }
  float s = 0.f;
  #pragma unroll
  for (int i = 0; i < 16; ++i) {
    float x, y;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(c[i]));
    s += x + y;
  }
  if (s == 1.2345f) out[0] = s;
}

// mm's inner loop alone: the same 16 k-steps of fragment loads from shared
// memory (2 x LDS.128 for 8 A values, 2 x LDS.128 for 8 B values) and 32
// FFMA2 per thread and k-step, over a tile filled once -- no global
// staging, no barrier in the loop.  The ceiling of the LDS + FFMA2 mix at
// mm's occupancy (256 threads, 2 CTAs per SM).
extern "C" __global__ void __launch_bounds__(256) mmloop(float* out, float a, float b, int iters) {
  __shared__ __align__(16) float As[16 * 128];
  __shared__ __align__(16) float Bs[16 * 128];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  for (int i = threadIdx.x; i < 16 * 128; i += 256) { As[i] = a * i; Bs[i] = b * i; }
  __syncthreads();
  float acc[64];
  #pragma unroll
  for (int i = 0; i < 64; ++i) acc[i] = 0.0f;
  for (int it = 0; it < iters; ++it) {
    asm volatile("" ::: "memory");     // the tile may change: keep its loads in the loop
    #pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[((8 * ty) ^ (8 * (k / 4))) + 128 * k]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[((8 * ty) ^ (8 * (k / 4))) + 128 * k + 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[((4 * tx) ^ (8 * (k / 4))) + 128 * k]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[((4 * tx) ^ (8 * (k / 4))) + 128 * k + 64]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      #pragma unroll
      for (int i10 = 0; i10 < 8; ++i10) {
        #pragma unroll
        for (int i9 = 0; i9 < 4; ++i9) {
          unsigned long long c, x, y;
          asm("mov.b64 %0, {%1,%2};" : "=l"(c) : "f"(acc[8 * i10 + 2 * i9]), "f"(acc[8 * i10 + 2 * i9 + 1]));
          asm("mov.b64 %0, {%1,%2};" : "=l"(x) : "f"(av[2 * i9]), "f"(av[2 * i9 + 1]));
          asm("mov.b64 %0, {%1,%1};" : "=l"(y) : "f"(bv[i10]));
          asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(x), "l"(y));
          asm("mov.b64 {%0,%1}, %2;" : "=f"(acc[8 * i10 + 2 * i9]), "=f"(acc[8 * i10 + 2 * i9 + 1]) : "l"(c));
        }
      }
    }
  }
  float s = 0.f;
  #pragma unroll
  for (int i = 0; i < 64; ++i) s += acc[i];
  if (s == 1.2345f) out[0] = s;
}
"""


def mmloop(mod, st, sms, out):
    """TFLOP/s of the mm inner loop alone with mm's own grid: 1024 CTAs of
    256 threads (2 resident per SM), 256 x 16 k-steps each -- exactly the
    FMA count of the 4096^3 product."""
    fn = mod.function("mmloop")
    blocks, iters = 1024, 256
    args = [RT.C.c_uint64(out.ptr), RT.C.c_float(1e-3), RT.C.c_float(2e-3), RT.C.c_int(iters)]
    ts = []
    for it in range(13):
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        RT.launch(fn, 0, (blocks, 1), (256, 1), 0, args, st)
        e1.record(st)
        st.sync()
        if it >= 3:
            ts.append(e0.elapsed_ms(e1))
    flops = blocks * 256 * iters * 16 * 64 * 2
    return flops / statistics.mean(ts) / 1e9


def main():
    RT.init(0)
    st = RT.Stream(0)
    mod = RT.Module(RT.nvrtc_compile(SRC), 0)
    sms = RT.device_attribute(0, RT.ATTR_SM_COUNT)
    out = RT.DeviceBuffer(64)
    for name, lanes in (("ffma1", 1), ("ffma2", 2)):
        fn = mod.function(name)
        for per_sm in (2, 4, 8):
            blocks = sms * per_sm
            args = [RT.C.c_uint64(out.ptr), RT.C.c_float(0.999), RT.C.c_float(1e-4), RT.C.c_int(ITERS)]
            ts = []
            for it in range(13):
                e0, e1 = RT.Event(0), RT.Event(0)
                e0.record(st)
                RT.launch(fn, 0, (blocks, 1), (256, 1), 0, args, st)
                e1.record(st)
                st.sync()
                if it >= 3:
                    ts.append(e0.elapsed_ms(e1))
            ms = statistics.mean(ts)
            flops = blocks * 256 * ITERS * 16 * lanes * 2
            print(f"{name:6s} {per_sm} CTAs/SM x 256: {ms * 1e3:8.1f} us  {flops / ms / 1e9:7.2f} TFLOP/s",
                  flush=True)
    print(f"mm inner loop (shared fragments + FFMA2), mm's grid of 1024 x 256: {mmloop(mod, st, sms, out):7.2f} TFLOP/s",
          flush=True)


if __name__ == "__main__":
    main()
