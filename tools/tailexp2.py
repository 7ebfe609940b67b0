"""Where do the last microseconds of dot/asum go?  (GPU box)

    python tools/tailexp2.py

Hand-written reference points at 128 MiB, timed like bench.py (L2 scrubbed,
events on the launching stream, mean of 60 after warm-up; the event clock
ticks in ~1 us steps, so only means are meaningful):
  events      -- e0, e1 with nothing between
  empty       -- one empty kernel between the events
  read        -- contiguous-chunk __ldg read, 256 x 1024, unroll 16 (no combine)
  read+block  -- read + warp-shuffle/shared block combine + partial store
  read+grid   -- read+block + last-block-done grid combine (threadfence + atomic)
and the emitted DPIA dot (2^24 pairs) and asum (2^25) kernels.
Measurement infrastructure only; not product code.
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import asum_config, dot_config  # noqa: E402

SRC = r"""
extern "C" __global__ void empty_k(const float4* p, long long n4, float* out, unsigned* ctr) {}

template <int MODE>
__device__ void body(const float4* __restrict__ p, long long n4, float* out, unsigned* ctr) {
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
  if (MODE == 0) { if (s == 123456.789f) out[0] = s; return; }
  __shared__ float red[32];
  __shared__ bool last;
  for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) out[1 + blockIdx.x] = t;
  }
  if (MODE == 1) return;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ctr, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  float t = threadIdx.x < gridDim.x ? ((volatile float*)out)[1 + threadIdx.x] : 0.f;
  for (int o = 16; o; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x < 32) {
    t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) { out[0] = t; *ctr = 0; }
  }
}
// MODE 3: no __threadfence; the ticket is an acq_rel atomic, and warp 0 of the
// last block alone reads the partials (ordering by __syncwarp).
__device__ void body3(const float4* __restrict__ p, long long n4, float* out, unsigned* ctr) {
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
  if (threadIdx.x >= 32) return;
  float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
  for (int o = 16; o; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  unsigned ticket = 0;
  if (threadIdx.x == 0) {
    out[1 + blockIdx.x] = t;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(ticket) : "l"(ctr) : "memory");
  }
  ticket = __shfl_sync(0xffffffffu, ticket, 0);
  if (ticket != gridDim.x - 1) return;
  __syncwarp();
  float u = 0.f;
  for (int i = threadIdx.x; i < gridDim.x; i += 32) {
    float v;
    asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(out + 1 + i) : "memory");
    u += v;
  }
  for (int o = 16; o; o >>= 1) u += __shfl_down_sync(0xffffffffu, u, o);
  if (threadIdx.x == 0) { out[0] = u; *ctr = 0; }
}
// MODE 4: every block but 0 publishes its partial and bumps the counter with
// a fire-and-forget red.release; block 0 (after its own share) spins on an
// acquire load of the counter, then combines the partials.
__device__ void body4(const float4* __restrict__ p, long long n4, float* out, unsigned* ctr) {
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
  if (threadIdx.x >= 32) return;
  float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
  for (int o = 16; o; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  if (blockIdx.x != 0) {
    if (threadIdx.x == 0) {
      out[1 + blockIdx.x] = t;
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(ctr) : "memory");
    }
    return;
  }
  if (threadIdx.x == 0) {
    unsigned c;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(ctr) : "memory");
    } while (c != gridDim.x - 1);
  }
  __syncwarp();
  float u = threadIdx.x == 0 ? t : 0.f;
  for (int i = 1 + threadIdx.x; i < gridDim.x; i += 32) {
    float v;
    asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(out + 1 + i) : "memory");
    u += v;
  }
  for (int o = 16; o; o >>= 1) u += __shfl_down_sync(0xffffffffu, u, o);
  if (threadIdx.x == 0) { out[0] = u; *ctr = 0; }
}
// MODE 5: two-level ticket (16 blocks per group counter, then a top
// counter over the groups): at most 16-way contention per counter.
__device__ void body5(const float4* __restrict__ p, long long n4, float* out, unsigned* ctr) {
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
  __shared__ bool last;
  for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
  for (int o = 16; o; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  const unsigned G = 16, ngroups = (gridDim.x + G - 1) / G, grp = blockIdx.x / G;
  const unsigned gsize = min(G, gridDim.x - grp * G);
  unsigned go = 0;
  if (threadIdx.x == 0) {
    out[1 + blockIdx.x] = t;
    __threadfence();
    go = atomicAdd(ctr + 1 + grp, 1u) == gsize - 1;
    if (go) {
      ctr[1 + grp] = 0;
      __threadfence();
      go = atomicAdd(ctr, 1u) == ngroups - 1 ? 2 : 0;
    }
  }
  go = __shfl_sync(0xffffffffu, go, 0);
  if (go != 2) return;
  __threadfence();
  float u = 0.f;
  for (int i = threadIdx.x; i < gridDim.x; i += 32) u += ((volatile float*)out)[1 + i];
  for (int o = 16; o; o >>= 1) u += __shfl_down_sync(0xffffffffu, u, o);
  if (threadIdx.x == 0) { out[0] = u; *ctr = 0; }
}
extern "C" __global__ void __launch_bounds__(1024) read5(const float4* p, long long n4, float* out, unsigned* c) { body5(p, n4, out, c); }
extern "C" __global__ void __launch_bounds__(1024) read4(const float4* p, long long n4, float* out, unsigned* c) { body4(p, n4, out, c); }
extern "C" __global__ void __launch_bounds__(1024) read3(const float4* p, long long n4, float* out, unsigned* c) { body3(p, n4, out, c); }
extern "C" __global__ void __launch_bounds__(1024) read0(const float4* p, long long n4, float* out, unsigned* c) { body<0>(p, n4, out, c); }
extern "C" __global__ void __launch_bounds__(1024) read1(const float4* p, long long n4, float* out, unsigned* c) { body<1>(p, n4, out, c); }
extern "C" __global__ void __launch_bounds__(1024) read2(const float4* p, long long n4, float* out, unsigned* c) { body<2>(p, n4, out, c); }
"""

REPS = 60


def timed(st, fn_launch):
    ts = []
    for it in range(REPS + 5):
        RT.lib().dpia_l2_flush(0, st.handle)
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        fn_launch()
        e1.record(st)
        st.sync()
        if it >= 5:
            ts.append(e0.elapsed_ms(e1))
    return statistics.mean(ts) * 1e3


def main():
    RT.init(0)
    st = RT.Stream(0)
    mod = RT.Module(RT.nvrtc_compile(SRC), 0)
    nbytes = 1 << 27
    buf = RT.DeviceBuffer(nbytes)
    buf.upload(np.ones(nbytes // 4, np.float32), st)
    out = RT.DeviceBuffer(4096)
    out.zero(st)
    ctr = RT.DeviceBuffer(256)
    ctr.zero(st)
    args = [RT.C.c_uint64(buf.ptr), RT.C.c_longlong(nbytes // 16), RT.C.c_uint64(out.ptr),
            RT.C.c_uint64(ctr.ptr)]
    print(f"events      : {timed(st, lambda: None):7.2f} us", flush=True)
    fe = mod.function("empty_k")
    print(f"empty       : {timed(st, lambda: RT.launch(fe, 0, (1, 1), (32, 1), 0, args, st)):7.2f} us",
          flush=True)
    for name, label in (("read0", "read"), ("read1", "read+block"), ("read2", "read+grid"), ("read3", "read+grid-acqrel"),
                        ("read4", "read+spin0"), ("read5", "read+grid-2level")):
        fn = mod.function(name)
        for blocks in (256, 512):
            t = timed(st, lambda: RT.launch(fn, 0, (blocks, 1), (1024, 1), 0, args, st))
            if name != "read0":
                o = np.zeros(1, np.float32)
                out.download(o)
                print(f"   out[0] = {o[0]}", flush=True)
            print(f"{label:12s}: {t:7.2f} us  {nbytes / t / 1e3:6.0f} GB/s  blocks={blocks}", flush=True)
    buf.free()
    rng = np.random.default_rng(0)
    for cfg, inputs in ((dot_config(), {"xs": rng.uniform(0, 1, 1 << 24).astype(np.float32),
                                        "ys": rng.uniform(0, 1, 1 << 24).astype(np.float32)}),
                        (asum_config(N=1 << 25), {"xs": rng.uniform(-1, 1, 1 << 25).astype(np.float32)})):
        exe = executable(compile_program(cfg.text, name=cfg.name), cfg.launch, cfg.sigma, float_mode=True)
        for n, v in inputs.items():
            exe.upload(n, v, st)
        t = timed(st, lambda: exe.launch(st))
        print(f"dpia {cfg.name:7s}: {t:7.2f} us  {cfg.bytes / t / 1e3:6.0f} GB/s  launch={cfg.launch}",
              flush=True)


if __name__ == "__main__":
    main()
