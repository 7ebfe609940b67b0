"""Grid-combine tail protocols at 128 MiB / 256 MiB (GPU box):

    python tools/tagexp.py

Hand-written reference kernels (measurement infrastructure, not product),
timed like bench.py (L2 scrubbed, events on the launching stream, mean of
60 after warm-up):
  read+block  -- read, block combine, partial store, no grid combine
  ticket      -- + last-block-done: __threadfence, atomic ticket, the last
                 block re-reads every partial (three dependent L2 round trips)
  tagged      -- each block publishes its partial as one 64-bit word
                 {value, generation} (single-copy atomic, no fence, no
                 atomic); the last-launched block polls the words with
                 relaxed loads until every generation matches, combines them
                 in the same fixed order, and bumps the generation word
  tagged-ns   -- tagged with a __nanosleep(64) back-off between polls
  ticket_first -- the ticket is taken before publishing; the non-last
                 blocks publish tagged 64-bit words without a fence and the
                 last block polls them (no fence on the critical path)
  part+comb   -- two kernels: partials, then a one-block combine launched
                 with programmatic dependent launch (pdl=True; part_trig
                 triggers the dependent launch at block start) or plainly
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import runtime as RT  # noqa: E402

SRC = r"""
__device__ __forceinline__ float block_sum(float s, float* red) {
  for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  float t = 0.f;
  if (threadIdx.x < 32) {
    t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  }
  return t;   // valid in thread 0
}

__device__ __forceinline__ float read_part(const float4* __restrict__ p, long long n4) {
  long long per = n4 / gridDim.x;
  const float4* q = p + blockIdx.x * per;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int k = per / blockDim.x;
  #pragma unroll 16
  for (int j = 0; j < k; ++j) {
    float4 v = __ldg(q + (long long)j * blockDim.x + threadIdx.x);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  return acc.x + acc.y + acc.z + acc.w;
}

extern "C" __global__ void __launch_bounds__(1024) rblock(const float4* p, long long n4, float* out,
                                                          unsigned* ctr, unsigned long long* slots) {
  __shared__ float red[32];
  float t = block_sum(read_part(p, n4), red);
  if (threadIdx.x == 0) out[1 + blockIdx.x] = t;
}

extern "C" __global__ void __launch_bounds__(1024) ticket(const float4* p, long long n4, float* out,
                                                          unsigned* ctr, unsigned long long* slots) {
  __shared__ float red[32];
  __shared__ bool last;
  float t = block_sum(read_part(p, n4), red);
  if (threadIdx.x == 0) {
    out[1 + blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(ctr, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  float v = threadIdx.x < gridDim.x ? ((volatile float*)out)[1 + threadIdx.x] : 0.f;
  __syncthreads();
  float u = block_sum(v, red);
  if (threadIdx.x == 0) { out[0] = u; *ctr = 0; }
}

template <int SLEEP>
__device__ __forceinline__ void tagged_body(const float4* p, long long n4, float* out, unsigned* gen_word,
                                            unsigned long long* slots) {
  __shared__ float red[32];
  const unsigned gen = *((volatile unsigned*)gen_word) + 1u;
  float t = block_sum(read_part(p, n4), red);
  if (threadIdx.x == 0) {
    unsigned long long w = ((unsigned long long)gen << 32) | __float_as_uint(t);
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" :: "l"(slots + blockIdx.x), "l"(w) : "memory");
  }
  if (blockIdx.x != gridDim.x - 1) return;
  float v = 0.f;
  if (threadIdx.x < gridDim.x) {
    unsigned long long w;
    for (;;) {
      asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(slots + threadIdx.x) : "memory");
      if ((unsigned)(w >> 32) == gen) break;
      if (SLEEP) __nanosleep(SLEEP);
    }
    v = __uint_as_float((unsigned)w);
  }
  __syncthreads();
  float u = block_sum(v, red);
  if (threadIdx.x == 0) { out[0] = u; *gen_word = gen; }
}
// ticket first: every block takes its ticket with a relaxed atomic before
// publishing; the non-last blocks then publish {value, generation} in one
// 64-bit store (no fence), and the last block -- which never has to publish
// its own partial -- polls only the slots whose owners already hold a ticket.
extern "C" __global__ void __launch_bounds__(1024) ticket_first(const float4* p, long long n4, float* out,
                                                                unsigned* ctr, unsigned long long* slots) {
  __shared__ float red[32];
  __shared__ unsigned tk;
  __shared__ float mine;
  unsigned* gen_word = ctr + 64;
  const unsigned gen = *((volatile unsigned*)gen_word) + 1u;
  float t = block_sum(read_part(p, n4), red);
  if (threadIdx.x == 0) {
    tk = atomicAdd(ctr, 1u);
    mine = t;
  }
  __syncthreads();
  if (tk != gridDim.x - 1) {
    if (threadIdx.x == 0) {
      unsigned long long w = ((unsigned long long)gen << 32) | __float_as_uint(t);
      asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" :: "l"(slots + blockIdx.x), "l"(w) : "memory");
    }
    return;
  }
  float v = 0.f;
  if (threadIdx.x < gridDim.x) {
    if (threadIdx.x == blockIdx.x) {
      v = mine;
    } else {
      unsigned long long w;
      for (;;) {
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(slots + threadIdx.x) : "memory");
        if ((unsigned)(w >> 32) == gen) break;
      }
      v = __uint_as_float((unsigned)w);
    }
  }
  __syncthreads();
  float u = block_sum(v, red);
  if (threadIdx.x == 0) { out[0] = u; *ctr = 0; *gen_word = gen; }
}

// two kernels: partials, then a one-block combine.  With PDL the combine is
// launched while the partials kernel runs (every partials block triggers
// griddepcontrol.launch_dependents at its start) and waits in
// griddepcontrol.wait until the partials grid has completed and flushed.
template <int TRIGGER>
__device__ __forceinline__ void part_body(const float4* p, long long n4, float* out) {
  if (TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ float red[32];
  float t = block_sum(read_part(p, n4), red);
  if (threadIdx.x == 0) out[1 + blockIdx.x] = t;
}
extern "C" __global__ void __launch_bounds__(1024) part_trig(const float4* p, long long n4, float* out,
                                                             unsigned* ctr, unsigned long long* slots) {
  part_body<1>(p, n4, out);
}
extern "C" __global__ void __launch_bounds__(1024) part_plain(const float4* p, long long n4, float* out,
                                                              unsigned* ctr, unsigned long long* slots) {
  part_body<0>(p, n4, out);
}
extern "C" __global__ void __launch_bounds__(1024) comb(const float4* p, long long nparts, float* out,
                                                        unsigned* ctr, unsigned long long* slots) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ float red[32];
  float v = 0.f;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) v += out[1 + i];
  float u = block_sum(v, red);
  if (threadIdx.x == 0) out[0] = u;
}

extern "C" __global__ void __launch_bounds__(1024) tagged(const float4* p, long long n4, float* out,
                                                          unsigned* ctr, unsigned long long* slots) {
  tagged_body<0>(p, n4, out, ctr + 64, slots);
}
extern "C" __global__ void __launch_bounds__(1024) tagged_ns(const float4* p, long long n4, float* out,
                                                             unsigned* ctr, unsigned long long* slots) {
  tagged_body<64>(p, n4, out, ctr + 64, slots);
}
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
    for nbytes in (1 << 27, 1 << 28):
        buf = RT.DeviceBuffer(nbytes)
        buf.upload(np.ones(nbytes // 4, np.float32), st)
        out = RT.DeviceBuffer(8192)
        out.zero(st)
        ctr = RT.DeviceBuffer(1024)
        ctr.zero(st)
        slots = RT.DeviceBuffer(8 * 1024)
        slots.zero(st)
        args = [RT.C.c_uint64(buf.ptr), RT.C.c_longlong(nbytes // 16), RT.C.c_uint64(out.ptr),
                RT.C.c_uint64(ctr.ptr), RT.C.c_uint64(slots.ptr)]
        fc = mod.function("comb")
        for rnd in range(2):
            for pname, pdl in (("part_trig", True), ("part_plain", True), ("part_plain", False)):
                fp = mod.function(pname)
                for blocks in (256, 512):
                    cargs = [args[0], RT.C.c_longlong(blocks)] + args[2:]

                    def two():
                        RT.launch(fp, 0, (blocks, 1), (1024, 1), 0, args, st)
                        RT.launch(fc, 0, (1, 1), (1024, 1), 0, cargs, st, pdl=pdl)
                    t = timed(st, two)
                    o = np.zeros(1, np.float32)
                    out.download(o)
                    print(f"{nbytes >> 20:4d} MiB round {rnd} {pname}+comb pdl={pdl!s:5s}: {t:7.2f} us  "
                          f"{nbytes / t / 1e3:6.0f} GB/s  blocks={blocks} out[0]={o[0]:.0f}", flush=True)
            for name in ("rblock", "ticket", "ticket_first"):
                fn = mod.function(name)
                for blocks in (256, 512):
                    t = timed(st, lambda: RT.launch(fn, 0, (blocks, 1), (1024, 1), 0, args, st))
                    o = np.zeros(1, np.float32)
                    out.download(o)
                    print(f"{nbytes >> 20:4d} MiB round {rnd} {name:10s}: {t:7.2f} us  "
                          f"{nbytes / t / 1e3:6.0f} GB/s  blocks={blocks} out[0]={o[0]:.0f}", flush=True)
        buf.free()


if __name__ == "__main__":
    main()
