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
"""


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


if __name__ == "__main__":
    main()
