"""Read-path experiment (GPU box): what can a streaming read of the benchmark
sizes reach on this B200, and by which mechanism?

    python tools/readexp.py

Variants, all timed like bench.py (L2 scrubbed, CUDA events on the launching
stream, median of 10):
  * empty      -- an empty kernel between the events (event + launch overhead);
  * ldg-gs     -- grid-stride __ldg float4 (tools/readsol.py);
  * ldg-chunk  -- one contiguous chunk per block, thread-strided (the DPIA
                  asum/dot strategy shape: transpose . split L), unroll U;
  * tma        -- cp.async.bulk global->shared ring of S stages, one
                  producer thread, mbarrier full/empty pipeline, 8 consumer
                  warps summing from shared memory.
Measurement infrastructure only; not product code.
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import runtime as RT  # noqa: E402

SRC = r"""

extern "C" __global__ void empty_k(const float4* p, long long n4, float* out) {}

extern "C" __global__ void __launch_bounds__(1024) ldg_gs(const float4* __restrict__ p, long long n4, float* out) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  #pragma unroll 8
  for (; i < n4; i += stride) {
    float4 v = __ldg(p + i);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  float s = acc.x + acc.y + acc.z + acc.w;
  if (s == 123456.789f) out[0] = s;
}

template <int U>
__device__ void ldg_chunk_body(const float4* __restrict__ p, long long n4, float* out) {
  long long per = n4 / gridDim.x;
  const float4* q = p + blockIdx.x * per;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int k = per / blockDim.x;
  #pragma unroll U
  for (int j = 0; j < k; ++j) {
    float4 v = __ldg(q + (long long)j * blockDim.x + threadIdx.x);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  float s = acc.x + acc.y + acc.z + acc.w;
  if (s == 123456.789f) out[0] = s;
}
extern "C" __global__ void __launch_bounds__(1024) ldg_chunk8(const float4* __restrict__ p, long long n4, float* out) { ldg_chunk_body<8>(p, n4, out); }
extern "C" __global__ void __launch_bounds__(1024) ldg_chunk16(const float4* __restrict__ p, long long n4, float* out) { ldg_chunk_body<16>(p, n4, out); }

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned ph) {
  asm volatile("{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}"
               :: "r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(bar)) : "memory");
}

// S stages of SB bytes; 8 consumer warps + 1 producer warp (288 threads).
template <int S, int SB>
__device__ void tma_body(const float4* __restrict__ p, long long n4, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long full[S], empty[S];
  float4* buf = reinterpret_cast<float4*>(smem);
  constexpr int V = SB / 16;
  long long per = n4 / gridDim.x;
  const float4* q = p + blockIdx.x * per;
  int nst = (int)(per / V);
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      for (int it = 0; it < nst; ++it) {
        int s = it % S;
        if (it >= S) mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
        mbar_expect_tx(&full[s], SB);
        bulk_g2s(buf + s * V, q + (long long)it * V, SB, &full[s]);
      }
    }
  } else {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int it = 0; it < nst; ++it) {
      int s = it % S;
      mbar_wait(&full[s], (it / S) & 1);
      #pragma unroll
      for (int k = threadIdx.x; k < V; k += 256) {
        float4 v = buf[s * V + k];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    float r = acc.x + acc.y + acc.z + acc.w;
    if (r == 123456.789f) out[0] = r;
  }
}
extern "C" __global__ void __launch_bounds__(288) tma_8x16k(const float4* p, long long n4, float* out) { tma_body<8, 16384>(p, n4, out); }
extern "C" __global__ void __launch_bounds__(288) tma_12x16k(const float4* p, long long n4, float* out) { tma_body<12, 16384>(p, n4, out); }
extern "C" __global__ void __launch_bounds__(288) tma_6x32k(const float4* p, long long n4, float* out) { tma_body<6, 32768>(p, n4, out); }
extern "C" __global__ void __launch_bounds__(288) tma_16x8k(const float4* p, long long n4, float* out) { tma_body<16, 8192>(p, n4, out); }
extern "C" __global__ void __launch_bounds__(288) tma_4x16k(const float4* p, long long n4, float* out) { tma_body<4, 16384>(p, n4, out); }
"""

# (name, threads, smem bytes, grids)
VARIANTS = [
    ("empty_k", 32, 0, (1,)),
    ("ldg_gs", 1024, 0, (296, 1184)),
    ("ldg_chunk8", 1024, 0, (256, 512)),
    ("ldg_chunk16", 1024, 0, (256, 512)),
    ("tma_8x16k", 288, 8 * 16384, (148, 256)),
    ("tma_12x16k", 288, 12 * 16384, (148, 256)),
    ("tma_6x32k", 288, 6 * 32768, (148, 256)),
    ("tma_16x8k", 288, 16 * 8192, (148, 256)),
    ("tma_4x16k", 288, 4 * 16384, (148, 256, 512)),
]


def main():
    RT.init(0)
    mod = RT.Module(RT.nvrtc_compile(SRC), 0)
    st = RT.Stream(0)
    for log2 in (27, 28, 30):
        nbytes = 1 << log2
        buf = RT.DeviceBuffer(nbytes)
        buf.zero(st)
        out = RT.DeviceBuffer(16)
        for name, thr, smem, grids in VARIANTS:
            fn = mod.function(name)
            if smem > 48 * 1024:
                RT.lib().dpia_kernel_set_smem(fn, smem)
            for blocks in grids:
                args = [RT.C.c_uint64(buf.ptr), RT.C.c_longlong(nbytes // 16), RT.C.c_uint64(out.ptr)]
                ts = []
                try:
                    for it in range(13):
                        RT.lib().dpia_l2_flush(0, st.handle)
                        e0, e1 = RT.Event(0), RT.Event(0)
                        e0.record(st)
                        RT.launch(fn, 0, (blocks, 1), (thr, 1), smem, args, st)
                        e1.record(st)
                        st.sync()
                        if it >= 3:
                            ts.append(e0.elapsed_ms(e1))
                except Exception as e:  # noqa: BLE001
                    print(f"{name} blocks={blocks}: {type(e).__name__}: {e}", flush=True)
                    continue
                med = statistics.median(ts)
                n4 = nbytes // 16
                if name.startswith("tma"):
                    v = int(name.split("x")[1].rstrip("k")) * 1024 // 16
                    rb = blocks * ((n4 // blocks) // v) * v * 16
                elif name.startswith("ldg_chunk"):
                    rb = blocks * ((n4 // blocks) // thr) * thr * 16
                else:
                    rb = nbytes
                print(f"2^{log2} B ({nbytes >> 20} MiB) {name:12s} blocks={blocks:5d}: {med * 1e3:8.2f} us "
                      f"{rb / med / 1e6:7.0f} GB/s  (min {min(ts) * 1e3:.2f} us)", flush=True)
        buf.free()


if __name__ == "__main__":
    main()
