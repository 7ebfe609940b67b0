"""Inner-loop ceilings of register-tile shapes (GPU box; measurement only):

    python tools/regtile.py

mm's k-step run alone (ffmapeak.mmloop generalised): per k-step a thread
reads RM A values and RN B values from a shared tile with 16-byte loads and
issues RM*RN/2 FFMA2 (pairs over A rows, B broadcast) into RM x RN
accumulators; no global staging, no barrier.  Launched at the occupancy the
register count allows.  Says which register tile could lift mm's ceiling
(58.7 TFLOP/s for the current 8 x 8 at 256 threads).
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import runtime as RT  # noqa: E402

TEMPLATE = r"""
template <int RM, int RN, int NT>
__device__ __forceinline__ void body(float* out, float a, float b, int iters) {
  __shared__ __align__(16) float As[16 * 256];
  __shared__ __align__(16) float Bs[16 * 256];
  for (int i = threadIdx.x; i < 16 * 256; i += NT) { As[i] = a * i; Bs[i] = b * i; }
  __syncthreads();
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[RM * RN];
  #pragma unroll
  for (int i = 0; i < RM * RN; ++i) acc[i] = 0.0f;
  for (int it = 0; it < iters; ++it) {
    asm volatile("" ::: "memory");     // the tile may change: keep its loads in the loop
    #pragma unroll
    for (int k = 0; k < 16; ++k) {
      float av[RM], bv[RN];
      #pragma unroll
      for (int q = 0; q < RM / 4; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(&As[((RM * ty + 4 * q) ^ (8 * (k / 4))) + 256 * k]);
        av[4 * q] = v.x; av[4 * q + 1] = v.y; av[4 * q + 2] = v.z; av[4 * q + 3] = v.w;
      }
      #pragma unroll
      for (int q = 0; q < RN / 4; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(&Bs[((4 * tx + 64 * q) ^ (8 * (k / 4))) + 256 * k]);
        bv[4 * q] = v.x; bv[4 * q + 1] = v.y; bv[4 * q + 2] = v.z; bv[4 * q + 3] = v.w;
      }
      #pragma unroll
      for (int j = 0; j < RN; ++j) {
        #pragma unroll
        for (int i = 0; i < RM / 2; ++i) {
          unsigned long long c, x, y;
          asm("mov.b64 %0, {%1,%2};" : "=l"(c) : "f"(acc[RM * j + 2 * i]), "f"(acc[RM * j + 2 * i + 1]));
          asm("mov.b64 %0, {%1,%2};" : "=l"(x) : "f"(av[2 * i]), "f"(av[2 * i + 1]));
          asm("mov.b64 %0, {%1,%1};" : "=l"(y) : "f"(bv[j]));
          asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(x), "l"(y));
          asm("mov.b64 {%0,%1}, %2;" : "=f"(acc[RM * j + 2 * i]), "=f"(acc[RM * j + 2 * i + 1]) : "l"(c));
        }
      }
    }
  }
  float s = 0.f;
  #pragma unroll
  for (int i = 0; i < RM * RN; ++i) s += acc[i];
  if (s == 1.2345f) out[0] = s;
}
"""
SHAPES = [(8, 8, 256), (8, 8, 128), (8, 16, 128), (16, 8, 128), (8, 16, 256), (16, 8, 256), (4, 8, 256),
          (8, 4, 256), (12, 8, 128), (8, 12, 128)]


def source():
    s = TEMPLATE
    for rm, rn, nt in SHAPES:
        s += (f'extern "C" __global__ void __launch_bounds__({nt}) k_{rm}_{rn}_{nt}(float* o, float a, float b, '
              f'int it) {{ body<{rm}, {rn}, {nt}>(o, a, b, it); }}\n')
    return s


def main():
    RT.init(0)
    st = RT.Stream(0)
    mod = RT.Module(RT.nvrtc_compile(source()), 0)
    sms = RT.device_attribute(0, RT.ATTR_SM_COUNT)
    out = RT.DeviceBuffer(64)
    iters = 128
    runs = [(rm, rn, nt, sms * 32) for rm, rn, nt in SHAPES]
    runs += [(8, 8, 256, sms * 2), (8, 8, 256, 1024), (8, 16, 128, 1024), (16, 8, 256, 512)]
    for rm, rn, nt, blocks in runs:
        fn = mod.function(f"k_{rm}_{rn}_{nt}")
        regs = RT.kernel_attribute(fn, RT.ATTR_NUM_REGS) if hasattr(RT, "kernel_attribute") else None
        args = [RT.C.c_uint64(out.ptr), RT.C.c_float(1e-3), RT.C.c_float(2e-3), RT.C.c_int(iters)]
        ts = []
        for i in range(8):
            e0, e1 = RT.Event(0), RT.Event(0)
            e0.record(st)
            RT.launch(fn, 0, (blocks, 1), (nt, 1), 0, args, st)
            e1.record(st)
            st.sync()
            if i >= 2:
                ts.append(e0.elapsed_ms(e1))
        flops = blocks * nt * iters * 16 * rm * rn * 2
        print(f"RM={rm:2d} RN={rn:2d} threads={nt} blocks={blocks}: {flops / statistics.mean(ts) / 1e9:7.2f} TFLOP/s"
              + (f"  regs={regs}" if regs else ""), flush=True)


if __name__ == "__main__":
    main()
