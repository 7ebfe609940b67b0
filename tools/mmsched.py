"""mm k-loop schedule experiment (GPU box):

    python tools/mmsched.py

Compares the emitted DPIA mm kernel (bench_programs.mm_config: 128x128 tile,
8x8 register tile, BK = 16, two rotated shared slices, one barrier per
k-tile) with hand-written variants that keep the SAME layout, swizzle, thread
mapping and per-accumulator FMA order (so C must be bit-identical) but change
the schedule around the per-k-tile barrier:

  rot   -- the operands of the tile's last k-step are read into registers
           before the barrier and its FFMA2s run after it, so every warp
           leaving the barrier has 32 independent FFMA2s to cover the latency
           of the next tile's first shared loads; the stores of tile k+1 move
           to the end of iteration k (after the last shared reads of the slice
           they overwrite, which precede the previous barrier)
  rot2  -- the same with the last two k-steps carried across the barrier

Measurement infrastructure only (not product code).
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import mm_config  # noqa: E402

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1710_08332_b200", "csrc", "dpia_device.cuh")


def variant(carry, minb=1):
    """Hand-written kernel: CARRY k-steps of each tile run after the barrier
    from registers."""
    return r"""
#define NT 256
extern "C" __global__ void __launch_bounds__(256, """ + str(minb) + r""") mm_rot(float* __restrict__ out, const float* __restrict__ A,
                                                         const float* __restrict__ B) {
  extern __shared__ __align__(16) unsigned char dpia_smem[];
  float* Bs = reinterpret_cast<float*>(dpia_smem);
  float* As = reinterpret_cast<float*>(dpia_smem + 16384);
  const int tx = threadIdx.x, ty = threadIdx.y, bx = blockIdx.x, by = blockIdx.y;
  float acc[64];
  #pragma unroll
  for (int i = 0; i < 64; ++i) acc[i] = 0.0f;
  dpia::vec<float, 4> pb0, pb1, pa0, pa1;
  auto ldg = [&](int kt) {
    const int r0 = ty, r1 = ty + 16;
    pb0 = dpia::vload<float, 4>(B, 64 * (r0 % 2) + 4096 * (r0 / 2) + 4 * tx + 65536 * kt + 128 * bx);
    pb1 = dpia::vload<float, 4>(B, 64 * (r1 % 2) + 4096 * (r1 / 2) + 4 * tx + 65536 * kt + 128 * bx);
    pa0 = dpia::vload<float, 4>(A, 16 * kt + 4 * (tx % 4) + 4096 * (tx / 4) + 524288 * by + 16384 * r0);
    pa1 = dpia::vload<float, 4>(A, 16 * kt + 4 * (tx % 4) + 4096 * (tx / 4) + 524288 * by + 16384 * r1);
  };
  auto sts = [&](int s) {
    const int r0 = ty, r1 = ty + 16;
    dpia::vstore<float, 4>(Bs, ((4 * tx) ^ (8 * (r0 / 8))) + 2048 * s + 64 * (r0 % 2) + 128 * (r0 / 2), pb0);
    dpia::vstore<float, 4>(Bs, ((4 * tx) ^ (8 * (r1 / 8))) + 2048 * s + 64 * (r1 % 2) + 128 * (r1 / 2), pb1);
    #pragma unroll
    for (int l = 0; l < 4; ++l) {
      As[((4 * r0) ^ (8 * (tx % 4))) + 2048 * s + 512 * (tx % 4) + (tx / 4) + 128 * l] = pa0.v[l];
      As[((4 * r1) ^ (8 * (tx % 4))) + 2048 * s + 512 * (tx % 4) + (tx / 4) + 128 * l] = pa1.v[l];
    }
  };
  auto step = [&](const float* a, const float* b) {   // a[8] rows, b[8] cols
    #pragma unroll
    for (int i10 = 0; i10 < 8; ++i10) {
      #pragma unroll
      for (int i9 = 0; i9 < 4; ++i9)
        dpia::fma2(acc[8 * i10 + 2 * i9], acc[8 * i10 + 2 * i9 + 1], a[2 * i9], b[i10], a[2 * i9 + 1], b[i10]);
    }
  };
  auto frag = [&](int s, int k, float* a, float* b) {
    #pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = As[((8 * ty) ^ (8 * (k / 4))) + 2048 * s + 128 * k + j];
    #pragma unroll
    for (int i10 = 0; i10 < 8; ++i10) b[i10] = Bs[((4 * tx) ^ (8 * (k / 4))) + (i10 % 4) + 64 * (i10 / 4) + 2048 * s + 128 * k];
  };
  constexpr int C = """ + str(carry) + r""";
  float ca[C][8], cb[C][8];
  ldg(0);
  sts(0);
  ldg(1);
  __syncthreads();
  for (int kt = 0; kt < 256; ++kt) {
    const int s = kt & 1;
    if (kt > 0) {
      #pragma unroll
      for (int c = 0; c < C; ++c) step(ca[c], cb[c]);
    }
    #pragma unroll
    for (int k = 0; k < 16 - C; ++k) {
      float a[8], b[8];
      frag(s, k, a, b);
      step(a, b);
    }
    #pragma unroll
    for (int c = 0; c < C; ++c) frag(s, 16 - C + c, ca[c], cb[c]);
    if (kt + 1 < 256) {
      sts(s ^ 1);
      if (kt + 2 < 256) ldg(kt + 2);
    }
    __syncthreads();
  }
  #pragma unroll
  for (int c = 0; c < C; ++c) step(ca[c], cb[c]);
  #pragma unroll
  for (int i28 = 0; i28 < 8; ++i28) {
    #pragma unroll
    for (int i27 = 0; i27 < 8; ++i27)
      out[(i28 % 4) + 64 * (i28 / 4) + 4096 * i27 + 4 * tx + 32768 * ty + 128 * bx + 524288 * by] = acc[i27 + 8 * i28];
  }
}
"""


def timed(st, launch, reps=10):
    ts = []
    for i in range(reps + 3):
        RT.lib().dpia_l2_flush(0, st.handle)
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        launch()
        e1.record(st)
        st.sync()
        if i >= 3:
            ts.append(e0.elapsed_ms(e1))
    return statistics.mean(ts)


def main():
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    B = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    cfg = mm_config()
    exe = executable(compile_program(cfg.text, name="mm"), cfg.launch, cfg.sigma, float_mode=True)
    exe.upload("A", A, st)
    exe.upload("B", B, st)
    base = np.zeros((4096, 4096), np.float32)
    for rnd in range(2):
        ms = timed(st, lambda: exe.launch(st))
        print(f"round {rnd} emitted : {ms * 1e3:8.1f} us  {cfg.flops / ms / 1e9:6.2f} TFLOP/s", flush=True)
        if rnd == 0:
            exe.buffers["out"].download(base)
        with open(HDR) as f:
            hdr = f.read()
        for carry, minb in ((1, 1), (1, 2), (2, 1), (2, 2)):
            mod = RT.Module(RT.nvrtc_compile(hdr + variant(carry, minb)), 0)
            fn = mod.function("mm_rot")
            RT.lib().dpia_kernel_set_smem(fn, 32768)
            out = RT.DeviceBuffer(4096 * 4096 * 4)
            args = [RT.C.c_uint64(out.ptr), RT.C.c_uint64(exe.buffers["A"].ptr),
                    RT.C.c_uint64(exe.buffers["B"].ptr)]
            ms = timed(st, lambda: RT.launch(fn, 0, (32, 32), (16, 16), 32768, args, st))
            got = np.zeros((4096, 4096), np.float32)
            out.download(got)
            same = bool(np.array_equal(got.view(np.uint32), base.view(np.uint32)))
            print(f"round {rnd} rot{carry} minblocks={minb}: {ms * 1e3:8.1f} us  {cfg.flops / ms / 1e9:6.2f} TFLOP/s  "
                  f"bit-identical to emitted: {same}", flush=True)
            out.free()


if __name__ == "__main__":
    main()
