"""Can dot at 2^24 (128 MiB read) reach 80% of the measured copy peak?
(GPU box; measurement infrastructure, not product.)

    python tools/dotbound.py            # event-timed, like bench.py
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \\
        python tools/dotbound.py --ncu  # the same kernels, 5 launches each

The bar is 134,217,728 B / (0.8 x 6554.9 GB/s) = 25.60 us per step.
Kernels, all over the same 128 MiB (two 64 MiB operands for the dot ones):
  empty        one empty kernel (launch + event overhead)
  read         tools/tailexp2.py read0: contiguous-chunk __ldg read, no combine
  read+red     read + block combine + ONE fire-and-forget red.global.add.f32
               of the block partial into the result: the cheapest grid
               combine there is (no fence, no ticket, no tail; not
               deterministic, so not a candidate for the product)
  read+ticket  tailexp2 read2: block combine + last-block ticket tail
  dpia dot     the emitted kernel of bench_programs.dot_config()
Event timings are means of REPS launches, each after an L2 scrub (the event
clock ticks in ~1.02 us steps).
"""
import os
import statistics
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import dot_config  # noqa: E402
from tailexp2 import SRC as TAIL_SRC  # noqa: E402

RED_SRC = r"""
extern "C" __global__ void __launch_bounds__(1024) read_red(const float4* __restrict__ p, long long n4,
                                                             float* out, unsigned* ctr) {
  long long per = n4 / gridDim.x;
  const float4* q = p + blockIdx.x * per;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int k = per / blockDim.x;
  #pragma unroll 16
  for (int j = 0; j < k; ++j) {
    float4 v = __ldg(q + (long long)j * blockDim.x + threadIdx.x);
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
    if (threadIdx.x == 0) atomicAdd(out, t);
  }
}
"""

BAR_US = (1 << 27) / (0.8 * 6554.9e3)
REPS = 200


def timed(st, launch, reps):
    ts = []
    for it in range(reps + 5):
        RT.lib().dpia_l2_flush(0, st.handle)
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        launch()
        e1.record(st)
        st.sync()
        if it >= 5:
            ts.append(e0.elapsed_ms(e1))
    return statistics.mean(ts) * 1e3, statistics.median(ts) * 1e3


def main():
    ncu = "--ncu" in sys.argv
    reps = 5 if ncu else REPS
    RT.init(0)
    st = RT.Stream(0)
    mod = RT.Module(RT.nvrtc_compile(TAIL_SRC + RED_SRC), 0)
    nbytes = 1 << 27
    buf = RT.DeviceBuffer(nbytes)
    buf.upload(np.ones(nbytes // 4, np.float32), st)
    out, ctr = RT.DeviceBuffer(4096), RT.DeviceBuffer(256)
    out.zero(st)
    ctr.zero(st)
    args = [RT.C.c_uint64(buf.ptr), RT.C.c_longlong(nbytes // 16), RT.C.c_uint64(out.ptr),
            RT.C.c_uint64(ctr.ptr)]
    print(f"bar: {BAR_US:.2f} us per step (80% of 6554.9 GB/s over 128 MiB)")
    rows = [("empty", "empty_k", (1, 32))]
    for blocks in (256, 296, 512):
        rows += [(f"read        G={blocks}", "read0", (blocks, 1024)),
                 (f"read+red    G={blocks}", "read_red", (blocks, 1024)),
                 (f"read+ticket G={blocks}", "read2", (blocks, 1024))]
    for label, fname, (g, l) in rows:
        fn = mod.function(fname)
        mean, med = timed(st, lambda: RT.launch(fn, 0, (g, 1), (l, 1), 0, args, st), reps)
        print(f"{label:22s}: mean {mean:6.2f} us  median {med:6.2f} us  "
              f"{nbytes / mean / 1e3:6.0f} GB/s  frac {nbytes / mean / 1e3 / 6554.9:.3f}", flush=True)
    buf.free()
    cfg = dot_config()
    exe = executable(compile_program(cfg.text, name="dot"), cfg.launch, cfg.sigma, float_mode=True)
    rng = np.random.default_rng(0)
    for n in ("xs", "ys"):
        exe.upload(n, rng.uniform(0, 1, 1 << 24).astype(np.float32), st)
    mean, med = timed(st, lambda: exe.launch(st), reps)
    print(f"{'dpia dot ' + str(cfg.launch):22s}: mean {mean:6.2f} us  median {med:6.2f} us  "
          f"{cfg.bytes / mean / 1e3:6.0f} GB/s  frac {cfg.bytes / mean / 1e3 / 6554.9:.3f}", flush=True)


if __name__ == "__main__":
    main()
