"""Does a TMA bulk-copy streaming read beat LDG.128 at 128 MiB?  (GPU box;
measurement infrastructure, not product.)

    python tools/bulkread.py

A persistent-style read of 128 MiB in which thread 0 of each CTA streams
CHUNK-byte pieces (piece c goes to CTA c % grid) into a STAGES-deep shared
ring with cp.async.bulk (TMA, completion on a per-stage mbarrier), and all
threads fold the landed piece from shared memory (LDS.128); a __syncthreads
per piece frees the slot, and thread 0 refills it after a proxy fence.
Compared with tools/tailexp2.py's read0 (contiguous-chunk __ldg float4,
256 x 1024) under the same timing as bench.py (L2 scrub, events on the
stream, mean of REPS).  No combine (each CTA stores its partial), so the
numbers are the pure-read ceiling of each design.
"""
import os
import statistics
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from tailexp2 import SRC as TAIL_SRC  # noqa: E402

BULK = r"""
template <int STAGES, int CHUNK>
__device__ __forceinline__ void bulk_body(const float4* __restrict__ p, long long nchunks, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long full[STAGES];
  constexpr int C4 = CHUNK / 16;
  float4* buf = reinterpret_cast<float4*>(smem);
  const int tid = threadIdx.x;
  const long long my = (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      unsigned b = (unsigned)__cvta_generic_to_shared(&full[s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < STAGES && s < my; ++s) {
      unsigned b = (unsigned)__cvta_generic_to_shared(&full[s]);
      unsigned d = (unsigned)__cvta_generic_to_shared(buf + s * C4);
      const float4* src = p + (blockIdx.x + (long long)s * gridDim.x) * C4;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CHUNK) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(d), "l"(src), "r"(CHUNK), "r"(b) : "memory");
    }
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long long k = 0; k < my; ++k) {
    const int s = (int)(k % STAGES);
    const unsigned par = (unsigned)((k / STAGES) & 1);
    const unsigned b = (unsigned)__cvta_generic_to_shared(&full[s]);
    unsigned done = 0;
    while (!done) {
      asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n"
                   " selp.u32 %0, 1, 0, q;\n}" : "=r"(done) : "r"(b), "r"(par) : "memory");
    }
    #pragma unroll 4
    for (int i = tid; i < C4; i += blockDim.x) {
      float4 v = buf[s * C4 + i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    __syncthreads();
    if (tid == 0 && k + STAGES < my) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      unsigned d = (unsigned)__cvta_generic_to_shared(buf + s * C4);
      const float4* src = p + (blockIdx.x + (k + STAGES) * gridDim.x) * C4;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CHUNK) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(d), "l"(src), "r"(CHUNK), "r"(b) : "memory");
    }
  }
  float s = acc.x + acc.y + acc.z + acc.w;
  if (s == 123456.789f) out[0] = s;
}
#define BULK_K(ST, CH) \
extern "C" __global__ void bulk_##ST##_##CH(const float4* __restrict__ p, long long n4, float* out, unsigned* ctr) { \
  bulk_body<ST, CH>(p, n4 * 16 / CH, out); }
BULK_K(4, 16384)
BULK_K(6, 16384)
BULK_K(8, 16384)
BULK_K(4, 32768)
BULK_K(6, 32768)
BULK_K(3, 65536)
BULK_K(12, 8192)
BULK_K(16, 8192)
"""

REPS = 100


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
    ncu = "--ncu" in sys.argv
    reps = 5 if ncu else REPS
    RT.init(0)
    st = RT.Stream(0)
    mod = RT.Module(RT.nvrtc_compile(TAIL_SRC + BULK), 0)
    nbytes = 1 << 27
    buf = RT.DeviceBuffer(nbytes)
    buf.upload(np.ones(nbytes // 4, np.float32), st)
    out, ctr = RT.DeviceBuffer(4096), RT.DeviceBuffer(256)
    out.zero(st)
    ctr.zero(st)
    args = [RT.C.c_uint64(buf.ptr), RT.C.c_longlong(nbytes // 16), RT.C.c_uint64(out.ptr),
            RT.C.c_uint64(ctr.ptr)]
    rows = [("read0 G=256 L=1024", "read0", 256, 1024, 0)]
    for st_, ch in ((4, 16384), (6, 16384), (8, 16384), (4, 32768), (6, 32768), (3, 65536),
                    (12, 8192), (16, 8192)):
        for g in (148, 296):
            for l in (128, 256, 512):
                smem = st_ * ch
                if smem * (g // 148) > 220 * 1024:
                    continue
                rows.append((f"bulk S={st_:2d} C={ch:5d} G={g} L={l}", f"bulk_{st_}_{ch}", g, l, smem))
    for label, fname, g, l, smem in rows:
        fn = mod.function(fname)
        if smem > 48 * 1024:
            RT.lib().dpia_kernel_set_smem(fn, smem)
        us = timed(st, lambda: RT.launch(fn, 0, (g, 1), (l, 1), smem, args, st), reps)
        print(f"{label:32s}: {us:7.2f} us  {nbytes / us / 1e3:6.0f} GB/s  frac {nbytes / us / 1e3 / 6554.9:.3f}",
              flush=True)


if __name__ == "__main__":
    main()
