"""Per-work-item contiguous chunk folds (BASELINE config 1's literal
mapGlobal + reduceSeq): what bounds the partials phase?  (GPU box;
measurement infrastructure, not product.)

    python tools/chunkread.py

16384 work-items, each folding x[i]*y[i] + acc sequentially over its own
1024-pair chunk (4 KiB of xs and 4 KiB of ys) and storing its partial --
the partials-only half of tools/litgeo.py.  Uncoalesced by construction:
one warp-wide 16-byte load touches 32 distinct lines, so the L1 processes
32 wavefronts per instruction for 512 bytes.  Variants:
  ldg4 D   rotating queue of D float4 per stream (the emitter's VEC_PREFETCH)
  ldg8 D   the same with 256-bit loads (ld.global.nc.v8.f32, sm_100):
           half the load instructions and wavefronts per byte
  bulk S B each work-item streams its chunks into its own shared-memory slots
           with cp.async.bulk (S stages of B bytes per stream, slots padded by
           16 bytes per lane so the LDS.128 reads are conflict-free); no L1
All variants fold in the same order, so the partials must be bit-identical.
"""
import os
import statistics
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_1710_08332_b200 import runtime as RT  # noqa: E402

SRC = r"""
#define CH 1024
template <int D>
__device__ __forceinline__ void ldg4_body(const float* __restrict__ x, const float* __restrict__ y, float* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const float4* xp = reinterpret_cast<const float4*>(x + (long long)i * CH);
  const float4* yp = reinterpret_cast<const float4*>(y + (long long)i * CH);
  float4 qx[D], qy[D];
  #pragma unroll
  for (int d = 0; d < D; ++d) { qx[d] = __ldg(xp + d); qy[d] = __ldg(yp + d); }
  float acc = 0.f;
  for (int jo = 0; jo < CH / 4; jo += D) {
    #pragma unroll
    for (int d = 0; d < D; ++d) {
      const int j = jo + d;
      float4 a = qx[d], b = qy[d];
      if (j + D < CH / 4) { qx[d] = __ldg(xp + j + D); qy[d] = __ldg(yp + j + D); }
      acc = a.x * b.x + acc; acc = a.y * b.y + acc; acc = a.z * b.z + acc; acc = a.w * b.w + acc;
    }
  }
  out[i] = acc;
}
struct f8 { float v[8]; };
__device__ __forceinline__ f8 ld8(const float* p) {
  f8 r;
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                 "=f"(r.v[6]), "=f"(r.v[7]) : "l"(p));
  return r;
}
template <int D>
__device__ __forceinline__ void ldg8_body(const float* __restrict__ x, const float* __restrict__ y, float* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const float* xp = x + (long long)i * CH;
  const float* yp = y + (long long)i * CH;
  f8 qx[D], qy[D];
  #pragma unroll
  for (int d = 0; d < D; ++d) { qx[d] = ld8(xp + 8 * d); qy[d] = ld8(yp + 8 * d); }
  float acc = 0.f;
  for (int jo = 0; jo < CH / 8; jo += D) {
    #pragma unroll
    for (int d = 0; d < D; ++d) {
      const int j = jo + d;
      f8 a = qx[d], b = qy[d];
      if (j + D < CH / 8) { qx[d] = ld8(xp + 8 * (j + D)); qy[d] = ld8(yp + 8 * (j + D)); }
      #pragma unroll
      for (int k = 0; k < 8; ++k) acc = a.v[k] * b.v[k] + acc;
    }
  }
  out[i] = acc;
}
template <int S, int B>
__device__ __forceinline__ void bulk_body(const float* __restrict__ x, const float* __restrict__ y, float* out) {
  // per lane: 2 streams x S stages x B bytes, lane slots padded by 16 B
  extern __shared__ __align__(128) unsigned char smem[];
  const int t = threadIdx.x;
  const int i = blockIdx.x * blockDim.x + t;
  constexpr int LANE = 2 * S * B + 16;
  unsigned char* mine = smem + t * LANE;
  unsigned long long* mb = reinterpret_cast<unsigned long long*>(smem + blockDim.x * LANE) + t * S;
  const char* xs = reinterpret_cast<const char*>(x + (long long)i * CH);
  const char* ys = reinterpret_cast<const char*>(y + (long long)i * CH);
  constexpr int NCH = CH * 4 / B;       // pieces per stream
  for (int s = 0; s < S; ++s) {
    unsigned b = (unsigned)__cvta_generic_to_shared(mb + s);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
  }
  #pragma unroll
  for (int s = 0; s < S; ++s) {
    unsigned b = (unsigned)__cvta_generic_to_shared(mb + s);
    unsigned dx = (unsigned)__cvta_generic_to_shared(mine + s * B);
    unsigned dy = (unsigned)__cvta_generic_to_shared(mine + (S + s) * B);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(2 * B) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dx), "l"(xs + s * B), "r"(B), "r"(b) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dy), "l"(ys + s * B), "r"(B), "r"(b) : "memory");
  }
  float acc = 0.f;
  for (int k = 0; k < NCH; ++k) {
    const int s = k % S;
    const unsigned par = (k / S) & 1;
    const unsigned b = (unsigned)__cvta_generic_to_shared(mb + s);
    unsigned done = 0;
    while (!done) {
      asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n"
                   " selp.u32 %0, 1, 0, q;\n}" : "=r"(done) : "r"(b), "r"(par) : "memory");
    }
    const float4* px = reinterpret_cast<const float4*>(mine + s * B);
    const float4* py = reinterpret_cast<const float4*>(mine + (S + s) * B);
    #pragma unroll
    for (int v = 0; v < B / 16; ++v) {
      float4 a = px[v], c = py[v];
      acc = a.x * c.x + acc; acc = a.y * c.y + acc; acc = a.z * c.z + acc; acc = a.w * c.w + acc;
    }
    if (k + S < NCH) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      unsigned dx = (unsigned)__cvta_generic_to_shared(mine + s * B);
      unsigned dy = (unsigned)__cvta_generic_to_shared(mine + (S + s) * B);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(2 * B) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dx), "l"(xs + (k + S) * B), "r"(B), "r"(b) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dy), "l"(ys + (k + S) * B), "r"(B), "r"(b) : "memory");
    }
  }
  out[i] = acc;
}
#define K4(D) extern "C" __global__ void ldg4_##D(const float* __restrict__ x, const float* __restrict__ y, float* out) { ldg4_body<D>(x, y, out); }
#define K8(D) extern "C" __global__ void ldg8_##D(const float* __restrict__ x, const float* __restrict__ y, float* out) { ldg8_body<D>(x, y, out); }
#define KB(S, B) extern "C" __global__ void bulk_##S##_##B(const float* __restrict__ x, const float* __restrict__ y, float* out) { bulk_body<S, B>(x, y, out); }
K4(8) K4(16) K8(4) K8(8)
KB(2, 256) KB(2, 512) KB(3, 256) KB(4, 256) KB(2, 1024)
"""

REPS = 50


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
    return statistics.mean(ts) * 1e3


def main():
    RT.init(0)
    st = RT.Stream(0)
    mod = RT.Module(RT.nvrtc_compile(SRC), 0)
    n = 16384 * 1024
    rng = np.random.default_rng(0)
    xb, yb, ob = RT.DeviceBuffer(4 * n), RT.DeviceBuffer(4 * n), RT.DeviceBuffer(4 * 16384)
    xb.upload(rng.uniform(0, 1, n).astype(np.float32), st)
    yb.upload(rng.uniform(0, 1, n).astype(np.float32), st)
    args = [RT.C.c_uint64(xb.ptr), RT.C.c_uint64(yb.ptr), RT.C.c_uint64(ob.ptr)]
    rows = [(f"ldg4 D={d}", f"ldg4_{d}", 0) for d in (8, 16)]
    rows += [(f"ldg8 D={d}", f"ldg8_{d}", 0) for d in (4, 8)]
    rows += [(f"bulk S={s} B={b}", f"bulk_{s}_{b}", (s, b)) for s, b in ((2, 256), (2, 512), (3, 256), (4, 256), (2, 1024))]
    ref = None
    for label, fname, sb in rows:
        fn = mod.function(fname)
        for L in (32, 64, 128):
            smem = 0
            if sb:
                s, b = sb
                smem = L * (2 * s * b + 16) + L * s * 8
                if smem > 227 * 1024:
                    continue
                RT.lib().dpia_kernel_set_smem(fn, smem)
            try:
                us = timed(st, lambda: RT.launch(fn, 0, (16384 // L, 1), (L, 1), smem, args, st), REPS)
            except Exception as e:  # noqa: BLE001
                print(f"{label:18s} L={L:3d}: {type(e).__name__} {e}", flush=True)
                continue
            got = np.empty(16384, np.float32)
            ob.download(got, st)
            st.sync()
            ref = got.copy() if ref is None else ref
            same = np.array_equal(got.view(np.uint32), ref.view(np.uint32))
            print(f"{label:18s} L={L:3d}: {us:7.2f} us  {8 * n / us / 1e3:6.0f} GB/s  "
                  f"{'bit-identical' if same else 'DIFFERENT'}", flush=True)


if __name__ == "__main__":
    main()
