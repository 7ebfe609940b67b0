"""mm with TMA staging and mbarrier pipelining (GPU box; hand-written
experiment, not product):

    python tools/mmtma.py

Same thread mapping, register tile and per-accumulator FMA order as the
emitted DPIA mm kernel (bench_programs.mm_config), so C must be
bit-identical, but the k-tiles reach shared memory by TMA
(cp.async.bulk.tensor.2d, descriptors from dpia_tensor_map_2d_f32) into an
S-stage ring guarded by full/empty mbarriers instead of register staging
plus one __syncthreads per k-tile:

  * no staging registers and no CTA-wide barrier in the k-loop: warps only
    wait for the stage they are about to read;
  * A arrives row-major ([row][k]; TMA cannot transpose 4-byte elements), so
    each k-step reads its 8 A values with scalar shared loads (2 distinct
    addresses per warp, broadcast) instead of two 16-byte loads;
  * thread 0 refills a stage once all 256 threads have released it (empty
    mbarrier), or -- refill="last warp" -- the last warp to release a stage
    (a shared-memory counter) refills it, so no thread waits to refill; or
    -- refill="after barrier" -- one __syncthreads per k-tile keeps the warps
    in step and thread 0 refills the released stage right after it.

Answers whether register staging + the per-k-tile barrier are what keeps
mm at 84% of the FFMA2 ceiling.
"""
import ctypes
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


def source(stages: int, lastwarp: int = 0, rowstride: bool = False, pairb: bool = False) -> str:
    return ("#define LASTWARP " + str(int(lastwarp)) + "\n#define ROWSTRIDE " + str(int(rowstride))
            + "\n#define PAIRB " + str(int(pairb))) + r"""
struct __align__(64) TMap { unsigned long long d[16]; };

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
               " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  long long n = 0;
  while (!mbar_try(b, parity)) {
    if (++n > (1LL << 26)) __trap();     // never hang the box: fail the launch instead
  }
}
__device__ __forceinline__ void tma_2d(void* dst, const TMap* map, unsigned long long* bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%3, %4}], [%2];"
               :: "r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}

#define S """ + str(stages) + r"""
#if ROWSTRIDE
#define ROW(j) (ty + 16 * (j))     // rows 64 B apart within a warp: conflict-free
#else
#define ROW(j) (8 * ty + (j))      // the emitted kernel's rows
#endif
extern "C" __global__ void __launch_bounds__(256) mm_tma(float* __restrict__ out,
                                                         const __grid_constant__ TMap amap,
                                                         const __grid_constant__ TMap bmap) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* As = reinterpret_cast<float*>(smem);                 // S x [128 rows][16 k]
  float* Bs = reinterpret_cast<float*>(smem + S * 8192);      // S x [16 k][128 cols]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + S * 16384);
  unsigned long long* empty = full + S;
  unsigned* cnt = reinterpret_cast<unsigned*>(empty + S);
  const int tx = threadIdx.x, ty = threadIdx.y, bx = blockIdx.x, by = blockIdx.y;
  const int tid = ty * 16 + tx;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 256); cnt[s] = 0u; }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_expect_tx(&full[s], 16384);
      tma_2d(As + s * 2048, &amap, &full[s], s * 16, by * 128);
      tma_2d(Bs + s * 2048, &bmap, &full[s], bx * 128, s * 16);
    }
  }
  float acc[64];
  #pragma unroll
  for (int i = 0; i < 64; ++i) acc[i] = 0.0f;
  for (int kt = 0; kt < 256; ++kt) {
    const int s = kt % S;
    const unsigned par = (kt / S) & 1;
    mbar_wait(&full[s], par);
    const float* a = As + s * 2048;
    const float* b = Bs + s * 2048;
    #pragma unroll
    for (int k = 0; k < 16; ++k) {
      float av[8], bv[8];
      #pragma unroll
      for (int j = 0; j < 8; ++j) av[j] = a[(ROW(j)) * 16 + k];
      #pragma unroll
      for (int i10 = 0; i10 < 8; ++i10) bv[i10] = b[k * 128 + 4 * tx + (i10 % 4) + 64 * (i10 / 4)];
#if PAIRB
      // pairs of columns share the broadcast A value: the B pair comes
      // straight from one 16-byte shared load (acc[8 * row + col])
      #pragma unroll
      for (int j = 0; j < 8; ++j) {
        #pragma unroll
        for (int c = 0; c < 4; ++c)
          dpia::fma2(acc[8 * j + 2 * c], acc[8 * j + 2 * c + 1], av[j], bv[2 * c], av[j], bv[2 * c + 1]);
      }
#else
      #pragma unroll
      for (int i10 = 0; i10 < 8; ++i10) {
        #pragma unroll
        for (int i9 = 0; i9 < 4; ++i9)
          dpia::fma2(acc[8 * i10 + 2 * i9], acc[8 * i10 + 2 * i9 + 1], av[2 * i9], bv[i10], av[2 * i9 + 1], bv[i10]);
      }
#endif
    }
#if LASTWARP == 2
    // lockstep: one __syncthreads per k-tile (as the emitted kernel), after
    // which thread 0 refills the stage everyone has just released
    __syncthreads();
    if (tid == 0 && kt + S < 256) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&full[s], 16384);
      tma_2d(As + s * 2048, &amap, &full[s], (kt + S) * 16, by * 128);
      tma_2d(Bs + s * 2048, &bmap, &full[s], bx * 128, (kt + S) * 16);
    }
#elif LASTWARP
    // the last warp to release the stage refills it: no thread ever waits
    if (kt + S < 256) {
      __syncwarp();
      if ((tid & 31) == 0) {
        __threadfence_block();
        if (atomicAdd(&cnt[s], 1u) == 7u) {
          cnt[s] = 0u;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&full[s], 16384);
          tma_2d(As + s * 2048, &amap, &full[s], (kt + S) * 16, by * 128);
          tma_2d(Bs + s * 2048, &bmap, &full[s], bx * 128, (kt + S) * 16);
        }
      }
    }
#else
    mbar_arrive(&empty[s]);
    if (tid == 0 && kt + S < 256) {
      mbar_wait(&empty[s], par);
      mbar_expect_tx(&full[s], 16384);
      tma_2d(As + s * 2048, &amap, &full[s], (kt + S) * 16, by * 128);
      tma_2d(Bs + s * 2048, &bmap, &full[s], bx * 128, (kt + S) * 16);
    }
#endif
  }
  #pragma unroll
  for (int i28 = 0; i28 < 8; ++i28) {
    #pragma unroll
    for (int i27 = 0; i27 < 8; ++i27)
      out[(i28 % 4) + 64 * (i28 / 4) + 4096 * ROW(i27) + 4 * tx + 128 * bx + 524288 * by] =
          PAIRB ? acc[8 * i27 + i28] : acc[i27 + 8 * i28];
  }
}
"""


def source_wide(stages: int) -> str:
    """8 x 16 register tile, 128 threads (16 row groups x 8 column groups),
    TMA ring refilled by the last of the 4 warps to release a stage (no CTA
    barrier in the k-loop), FFMA2 pairing B columns against a broadcast A.
    Thread (ty, tx) owns rows 8*ty + j and columns 4*tx + 32*q + c (q < 4,
    c < 4): each 16-byte B load of a warp covers 128 contiguous bytes."""
    return source(stages, 1, False, True).split("#define S ")[0] + "#define S " + str(stages) + r"""
extern "C" __global__ void __launch_bounds__(128) mm_tma_wide(float* __restrict__ out,
                                                              const __grid_constant__ TMap amap,
                                                              const __grid_constant__ TMap bmap) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* As = reinterpret_cast<float*>(smem);                 // S x [128 rows][16 k]
  float* Bs = reinterpret_cast<float*>(smem + S * 8192);      // S x [16 k][128 cols]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + S * 16384);
  unsigned* cnt = reinterpret_cast<unsigned*>(full + S);
  const int tid = threadIdx.x, tx = tid % 8, ty = tid / 8, bx = blockIdx.x, by = blockIdx.y;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); cnt[s] = 0u; }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_expect_tx(&full[s], 16384);
      tma_2d(As + s * 2048, &amap, &full[s], s * 16, by * 128);
      tma_2d(Bs + s * 2048, &bmap, &full[s], bx * 128, s * 16);
    }
  }
  float acc[128];                       // acc[16 * j + c16]: row j, column slot c16
  #pragma unroll
  for (int i = 0; i < 128; ++i) acc[i] = 0.0f;
  for (int kt = 0; kt < 256; ++kt) {
    const int s = kt % S;
    mbar_wait(&full[s], (kt / S) & 1);
    const float* a = As + s * 2048;
    const float* b = Bs + s * 2048;
    #pragma unroll
    for (int k = 0; k < 16; ++k) {
      float av[8], bv[16];
      #pragma unroll
      for (int j = 0; j < 8; ++j) av[j] = a[(8 * ty + j) * 16 + k];
      #pragma unroll
      for (int c16 = 0; c16 < 16; ++c16) bv[c16] = b[k * 128 + 4 * tx + 32 * (c16 / 4) + (c16 % 4)];
      #pragma unroll
      for (int j = 0; j < 8; ++j) {
        #pragma unroll
        for (int c = 0; c < 8; ++c)
          dpia::fma2(acc[16 * j + 2 * c], acc[16 * j + 2 * c + 1], av[j], bv[2 * c], av[j], bv[2 * c + 1]);
      }
    }
    if (kt + S < 256) {
      __syncwarp();
      if ((tid & 31) == 0) {
        __threadfence_block();
        if (atomicAdd(&cnt[s], 1u) == 3u) {
          cnt[s] = 0u;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&full[s], 16384);
          tma_2d(As + s * 2048, &amap, &full[s], (kt + S) * 16, by * 128);
          tma_2d(Bs + s * 2048, &bmap, &full[s], bx * 128, (kt + S) * 16);
        }
      }
    }
  }
  #pragma unroll
  for (int j = 0; j < 8; ++j) {
    #pragma unroll
    for (int c16 = 0; c16 < 16; ++c16)
      out[4096 * (128 * by + 8 * ty + j) + 128 * bx + 4 * tx + 32 * (c16 / 4) + (c16 % 4)] = acc[16 * j + c16];
  }
}
"""


class TMap(ctypes.Structure):
    _fields_ = [("d", ctypes.c_uint64 * 16)]


def tensor_map(base, rows, cols, box_rows, box_cols):
    raw = np.zeros(256, np.uint8)
    off = (-raw.ctypes.data) % 64
    ptr = raw.ctypes.data + off
    RT.lib().dpia_tensor_map_2d_f32(ctypes.c_void_p(ptr), base, rows, cols, cols * 4, box_rows, box_cols)
    m = TMap()
    ctypes.memmove(ctypes.addressof(m), ptr, 128)
    return m


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
    amap = tensor_map(exe.buffers["A"].ptr, 4096, 4096, 128, 16)
    bmap = tensor_map(exe.buffers["B"].ptr, 4096, 4096, 16, 128)
    with open(HDR) as f:
        hdr = f.read()
    for rnd in range(1 if "one" in sys.argv else 2):
        ms = timed(st, lambda: exe.launch(st))
        print(f"round {rnd} emitted      : {ms * 1e3:8.1f} us  {cfg.flops / ms / 1e9:6.2f} TFLOP/s", flush=True)
        if rnd == 0:
            exe.buffers["out"].download(base)
        for stages in (3, 4, 6):
            mod = RT.Module(RT.nvrtc_compile(hdr + source_wide(stages)), 0)
            fn = mod.function("mm_tma_wide")
            smem = stages * 16384 + 8 * stages + 4 * stages
            RT.lib().dpia_kernel_set_smem(fn, smem)
            out = RT.DeviceBuffer(4096 * 4096 * 4)
            args = [RT.C.c_uint64(out.ptr), amap, bmap]
            ms = timed(st, lambda: RT.launch(fn, 0, (32, 32), (128, 1), smem, args, st))
            got = np.zeros((4096, 4096), np.float32)
            out.download(got)
            same = bool(np.array_equal(got.view(np.uint32), base.view(np.uint32)))
            print(f"round {rnd} tma wide 8x16 x 128 threads, stages={stages}: {ms * 1e3:8.1f} us  "
                  f"{cfg.flops / ms / 1e9:6.2f} TFLOP/s  same elements as emitted: {same}", flush=True)
            out.free()
        if "wide" in sys.argv:
            continue
        variants = ((6, 1, False, True),) if "one" in sys.argv else (
            (4, 0, False, False), (6, 1, False, False), (3, 2, False, False), (3, 1, True, False),
            (3, 2, True, False), (3, 1, False, True), (6, 1, False, True), (2, 2, False, True),
            (3, 2, False, True), (4, 2, False, True), (3, 1, True, True), (3, 2, True, True))
        for stages, lastwarp, rowstride, pairb in variants:
            mod = RT.Module(RT.nvrtc_compile(hdr + source(stages, lastwarp, rowstride, pairb)), 0)
            fn = mod.function("mm_tma")
            smem = stages * 16384 + 2 * stages * 8 + 4 * stages
            RT.lib().dpia_kernel_set_smem(fn, smem)
            out = RT.DeviceBuffer(4096 * 4096 * 4)
            args = [RT.C.c_uint64(out.ptr), amap, bmap]
            ms = timed(st, lambda: RT.launch(fn, 0, (32, 32), (16, 16), smem, args, st))
            got = np.zeros((4096, 4096), np.float32)
            out.download(got)
            same = bool(np.array_equal(got.view(np.uint32), base.view(np.uint32)))
            print(f"round {rnd} tma stages={stages} refill={['thread 0', 'last warp', 'after barrier'][int(lastwarp)]} rows={'strided' if rowstride else 'blocked'} pairs={'B' if pairb else 'A'}: {ms * 1e3:8.1f} us  {cfg.flops / ms / 1e9:6.2f} TFLOP/s  "
                  f"same elements as emitted: {same}", flush=True)
            out.free()


if __name__ == "__main__":
    main()
