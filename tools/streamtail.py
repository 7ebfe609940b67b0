"""Streaming tail for config 1's literal program (mapGlobal over 1024-element
chunks, reduceSeq per chunk, then the top-level sequential reduce of the
16384 partials): can the serial 16384-add tail overlap the grid phase?
(GPU box; measurement infrastructure, not product.)

    python tools/streamtail.py

Hand-written variants, each computing the identical left folds in the
identical order (results compared bit for bit with the emitted kernel):
  emitted          the backend's output at (512, 32): grid phase, then the
                   last block's thread 0 folds all partials (ticket tail)
  tma G x 32 S     as `stream`, but each warp stages its 32 work-items'
                   chunks with 2-D TMA tensor copies (box: 32 chunk rows x 32
                   floats, 128-byte swizzle) through S shared-memory stages;
                   each lane folds its own row from shared memory
  stream G x L     G x L work-items walk the 16384 chunks grid-stride in
                   R = 16384 / (G L) rounds; after each round every warp
                   publishes (fence + one atomic per warp) on that round's
                   counter; ONE extra block (blockIdx G) runs the tail from
                   the start: thread 0 streams the partials through the
                   same 4-slot TMA bulk ring, waiting for round r's counter
                   before it copies round r's partials, so the serial fold
                   of round r overlaps the grid phase of rounds r+1...
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import dot_literal_config  # noqa: E402

N_CHUNKS = 16384
KERNEL = r"""
extern "C" __global__ void __launch_bounds__(%(L)d) stream_k(float* __restrict__ out, const float* __restrict__ xs,
    const float* __restrict__ ys, float* g_tmp4, unsigned int* cnt) {
  extern __shared__ __align__(16) unsigned char dpia_smem[];
  const int tid = threadIdx.x;
  if (blockIdx.x == %(G)d) {
    if (tid != 0) return;
    float acc = 0.0f;
    unsigned long long* mb = reinterpret_cast<unsigned long long*>(dpia_smem);
    dpia::ring_init(mb, 4);
    int ready = 0;                 // partials [0, ready) are published
    #define WAIT_UPTO(hi) while (ready < (hi)) { \
        const int r = ready / %(GS)d; unsigned v; \
        do { asm volatile("ld.acquire.gpu.global.u32 %%0, [%%1];" : "=r"(v) : "l"(cnt + r) : "memory"); } \
        while (v < %(WPR)du); \
        ready = (r + 1) * %(GS)d; asm volatile("fence.proxy.async.global;" ::: "memory"); }
    for (int s = 0; s < 4; ++s) {
      WAIT_UPTO((s + 1) * 512);
      dpia::ring_expect(mb + s, 2048u);
      dpia::ring_copy(dpia_smem + 32 + s * 2048, g_tmp4 + s * 512, 2048u, mb + s);
    }
    for (int jo = 0; jo < %(N)d; jo += 512) {
      const int k = jo / 512, s = k %% 4;
      dpia::ring_wait(mb + s, (unsigned)((k / 4) & 1));
      const float* p = reinterpret_cast<const float*>(dpia_smem + 32) + s * 512;
      #pragma unroll 16
      for (int j = 0; j < 128; ++j) {
        const dpia::vec<float, 4> v = dpia::vload<float, 4>(p, 4 * j);
        acc = acc + v.v[0]; acc = acc + v.v[1]; acc = acc + v.v[2]; acc = acc + v.v[3];
      }
      if (jo + 2048 < %(N)d) {
        WAIT_UPTO(jo + 2048 + 512);
        dpia::ring_expect(mb + s, 2048u);
        dpia::ring_copy(dpia_smem + 32 + s * 2048, g_tmp4 + jo + 2048, 2048u, mb + s);
      }
    }
    out[0] = acc;
    for (int r = 0; r < %(R)d; ++r) cnt[r] = 0u;
    return;
  }
  const int gid = blockIdx.x * %(L)d + tid;
  for (int r = 0; r < %(R)d; ++r) {
    const int i = gid + r * %(GS)d;
    float a = 0.0f;
    dpia::vec<float, 8> qx[8], qy[8];
    #pragma unroll
    for (int j = 0; j < 8; ++j) {
      qx[j] = dpia::vload32<true>(xs, 1024LL * i + 8 * j);
      qy[j] = dpia::vload32<true>(ys, 1024LL * i + 8 * j);
    }
    for (int jo = 0; jo < 128; jo += 8) {
      #pragma unroll
      for (int jd = 0; jd < 8; ++jd) {
        const int j = jo + jd;
        const dpia::vec<float, 8> vx = qx[jd], vy = qy[jd];
        if (j + 8 < 128) { qx[jd] = dpia::vload32<true>(xs, 1024LL * i + 8 * j + 64);
                           qy[jd] = dpia::vload32<true>(ys, 1024LL * i + 8 * j + 64); }
        #pragma unroll
        for (int e = 0; e < 8; ++e) a = (vx.v[e] * vy.v[e]) + a;
      }
    }
    g_tmp4[i] = a;
    __syncwarp();
    if ((tid & 31) == 0) { __threadfence(); atomicAdd(cnt + r, 1u); }
  }
}
"""


TMA_KERNEL = r"""
struct __align__(64) TMap { unsigned long long w[16]; };
__device__ __forceinline__ void tma2d(void* dst, const TMap* m, int x, int y, unsigned long long* mb) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%%0], [%%1, {%%2, %%3}], [%%4];"
               :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(reinterpret_cast<unsigned long long>(m)),
                  "r"(x), "r"(y), "r"((unsigned)__cvta_generic_to_shared(mb)) : "memory");
}
extern "C" __global__ void __launch_bounds__(32) tma_k(float* __restrict__ out, const __grid_constant__ TMap tx,
    const __grid_constant__ TMap ty, float* g_tmp4, unsigned int* cnt) {
  extern __shared__ __align__(1024) unsigned char dpia_smem[];
  const int tid = threadIdx.x;
  if (blockIdx.x == %(G)d) {
    if (tid != 0) return;
    float acc = 0.0f;
    unsigned long long* mb = reinterpret_cast<unsigned long long*>(dpia_smem);
    dpia::ring_init(mb, 4);
    int ready = 0;
    #define WAIT_UPTO(hi) while (ready < (hi)) { \
        const int r = ready / %(GS)d; unsigned v; \
        do { asm volatile("ld.acquire.gpu.global.u32 %%0, [%%1];" : "=r"(v) : "l"(cnt + r) : "memory"); } \
        while (v < %(WPR)du); \
        ready = (r + 1) * %(GS)d; asm volatile("fence.proxy.async.global;" ::: "memory"); }
    for (int s = 0; s < 4; ++s) {
      WAIT_UPTO((s + 1) * 512);
      dpia::ring_expect(mb + s, 2048u);
      dpia::ring_copy(dpia_smem + 1024 + s * 2048, g_tmp4 + s * 512, 2048u, mb + s);
    }
    for (int jo = 0; jo < %(N)d; jo += 512) {
      const int k = jo / 512, s = k %% 4;
      dpia::ring_wait(mb + s, (unsigned)((k / 4) & 1));
      const float* p = reinterpret_cast<const float*>(dpia_smem + 1024) + s * 512;
      #pragma unroll 16
      for (int j = 0; j < 128; ++j) {
        const dpia::vec<float, 4> v = dpia::vload<float, 4>(p, 4 * j);
        acc = acc + v.v[0]; acc = acc + v.v[1]; acc = acc + v.v[2]; acc = acc + v.v[3];
      }
      if (jo + 2048 < %(N)d) {
        WAIT_UPTO(jo + 2048 + 512);
        dpia::ring_expect(mb + s, 2048u);
        dpia::ring_copy(dpia_smem + 1024 + s * 2048, g_tmp4 + jo + 2048, 2048u, mb + s);
      }
    }
    out[0] = acc;
    for (int r = 0; r < %(R)d; ++r) cnt[r] = 0u;
    return;
  }
  unsigned long long* mb = reinterpret_cast<unsigned long long*>(dpia_smem);
  unsigned char* stage = dpia_smem + 1024;
  if (tid == 0) dpia::ring_init(mb, %(S)d);
  __syncwarp();
  const int row0 = blockIdx.x * 32;
  const int T = %(R)d * 32;
  if (tid == 0) {
    for (int t = 0; t < %(S)d; ++t) {
      dpia::ring_expect(mb + t, 8192u);
      tma2d(stage + t * 8192, &tx, (t %% 32) * 32, row0 + (t / 32) * %(GS)d, mb + t);
      tma2d(stage + t * 8192 + 4096, &ty, (t %% 32) * 32, row0 + (t / 32) * %(GS)d, mb + t);
    }
  }
  float a = 0.0f;
  const int sw = tid & 7;
  for (int t = 0; t < T; ++t) {
    const int s = t %% %(S)d;
    dpia::ring_wait(mb + s, (unsigned)((t / %(S)d) & 1));
    const float* px = reinterpret_cast<const float*>(stage + s * 8192 + tid * 128);
    const float* py = px + 1024;
    #pragma unroll
    for (int c = 0; c < 8; ++c) {
      const dpia::vec<float, 4> vx = dpia::vload<float, 4>(px, 4 * (c ^ sw));
      const dpia::vec<float, 4> vy = dpia::vload<float, 4>(py, 4 * (c ^ sw));
      a = (vx.v[0] * vy.v[0]) + a; a = (vx.v[1] * vy.v[1]) + a;
      a = (vx.v[2] * vy.v[2]) + a; a = (vx.v[3] * vy.v[3]) + a;
    }
    __syncwarp();
    if (tid == 0 && t + %(S)d < T) {
      const int u = t + %(S)d;
      dpia::ring_expect(mb + s, 8192u);
      tma2d(stage + s * 8192, &tx, (u %% 32) * 32, row0 + (u / 32) * %(GS)d, mb + s);
      tma2d(stage + s * 8192 + 4096, &ty, (u %% 32) * 32, row0 + (u / 32) * %(GS)d, mb + s);
    }
    if ((t %% 32) == 31) {
      const int r = t / 32;
      g_tmp4[row0 + tid + r * %(GS)d] = a;
      a = 0.0f;
      __syncwarp();
      if (tid == 0) { __threadfence(); atomicAdd(cnt + r, 1u); }
    }
  }
}
"""


TMA2_KERNEL = r"""
struct __align__(64) TMap { unsigned long long w[16]; };
__device__ __forceinline__ void tma2d(void* dst, const TMap* m, int x, int y, unsigned long long* mb) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%%0], [%%1, {%%2, %%3}], [%%4];"
               :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(reinterpret_cast<unsigned long long>(m)),
                  "r"(x), "r"(y), "r"((unsigned)__cvta_generic_to_shared(mb)) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned long long* mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%%0];" :: "r"((unsigned)__cvta_generic_to_shared(mb)) : "memory");
}
// %(B)d boxes of 32 floats per stream per step, %(S)d stages, producer = %(P)d (1: a second warp)
extern "C" __global__ void __launch_bounds__(%(NT)d) tma2_k(float* __restrict__ out, const __grid_constant__ TMap tx,
    const __grid_constant__ TMap ty, float* g_tmp4, unsigned int* cnt) {
  extern __shared__ __align__(1024) unsigned char dpia_smem[];
  const int tid = threadIdx.x;
  constexpr int STEP = %(B)d * 8192;              // bytes per stage (both streams)
  constexpr int T = %(R)d * (32 / %(B)d);          // steps per warp
  if (blockIdx.x == %(G)d) {
    if (tid != 0) return;
    float acc = 0.0f;
    unsigned long long* mb = reinterpret_cast<unsigned long long*>(dpia_smem);
    dpia::ring_init(mb, %(TS)d);
    int ready = 0;
    #define WAIT_UPTO(hi) while (ready < (hi)) { \
        const int r = ready / %(GS)d; unsigned v; \
        do { asm volatile("ld.acquire.gpu.global.u32 %%0, [%%1];" : "=r"(v) : "l"(cnt + r) : "memory"); } \
        while (v < %(WPR)du); \
        ready = (r + 1) * %(GS)d; asm volatile("fence.proxy.async.global;" ::: "memory"); }
    if (%(TAIL)d) {
    for (int s = 0; s < %(TS)d; ++s) {
      WAIT_UPTO((s + 1) * 512);
      dpia::ring_expect(mb + s, 2048u);
      dpia::ring_copy(dpia_smem + 1024 + s * 2048, g_tmp4 + s * 512, 2048u, mb + s);
    }
    for (int jo = 0; jo < %(N)d; jo += 512) {
      const int k = jo / 512, s = k %% %(TS)d;
      dpia::ring_wait(mb + s, (unsigned)((k / %(TS)d) & 1));
      const float* p = reinterpret_cast<const float*>(dpia_smem + 1024) + s * 512;
      if (%(QD)d == 0) {
      #pragma unroll 16
      for (int j = 0; j < 128; ++j) {
        const dpia::vec<float, 4> v = dpia::vload<float, 4>(p, 4 * j);
        acc = acc + v.v[0]; acc = acc + v.v[1]; acc = acc + v.v[2]; acc = acc + v.v[3];
      }
      } else {
      constexpr int QD = %(QD)d + (%(QD)d == 0);
      dpia::vec<float, 4> q[QD];
      #pragma unroll
      for (int d = 0; d < QD; ++d) q[d] = dpia::vload<float, 4>(p, 4 * d);
      #pragma unroll 1
      for (int j0 = 0; j0 < 128; j0 += QD) {
        #pragma unroll
        for (int d = 0; d < QD; ++d) {
          const dpia::vec<float, 4> v = q[d];
          if (j0 + d + QD < 128) q[d] = dpia::vload<float, 4>(p, 4 * (j0 + d + QD));
          acc = acc + v.v[0]; acc = acc + v.v[1]; acc = acc + v.v[2]; acc = acc + v.v[3];
        }
      }
      }
      if (jo + %(TS)d * 512 < %(N)d) {
        WAIT_UPTO(jo + %(TS)d * 512 + 512);
        dpia::ring_expect(mb + s, 2048u);
        dpia::ring_copy(dpia_smem + 1024 + s * 2048, g_tmp4 + jo + %(TS)d * 512, 2048u, mb + s);
      }
    }
    } else {
      WAIT_UPTO(%(N)d);
    }
    out[0] = acc;
    if (%(TAIL)d != 2) for (int r = 0; r < %(R)d; ++r) cnt[r] = 0u;
    return;
  }
  unsigned long long* full = reinterpret_cast<unsigned long long*>(dpia_smem);
  unsigned long long* empty = full + 32;
  unsigned char* stage = dpia_smem + 1024;
  const int row0 = blockIdx.x * 32;
  if (tid == 0) {
    dpia::ring_init(full, %(S)d);
    dpia::ring_init(empty, %(S)d);
  }
  __syncthreads();
  const int lane = tid & 31;
  auto issue = [&](int u, int s) {
    const int x = (u %% (32 / %(B)d)) * 32 * %(B)d, y = row0 + (u / (32 / %(B)d)) * %(GS)d;
    dpia::ring_expect(full + s, (unsigned)STEP);
    #pragma unroll
    for (int b = 0; b < %(B)d; ++b) {
      tma2d(stage + s * STEP + b * 4096, &tx, x + 32 * b, y, full + s);
      tma2d(stage + s * STEP + (%(B)d + b) * 4096, &ty, x + 32 * b, y, full + s);
    }
  };
  if (%(P)d && tid >= 32) {                 // producer warp
    if (lane == 0) {
      for (int t = 0; t < T; ++t) {
        const int s = t %% %(S)d;
        if (t >= %(S)d) dpia::ring_wait(empty + s, (unsigned)(((t / %(S)d) - 1) & 1));
        issue(t, s);
      }
    }
    return;
  }
  if (!%(P)d && lane == 0)
    for (int t = 0; t < %(S)d && t < T; ++t) issue(t, t);
  float a = 0.0f;
  const int sw = lane & 7;
  for (int t = 0; t < T; ++t) {
    const int s = t %% %(S)d;
    dpia::ring_wait(full + s, (unsigned)((t / %(S)d) & 1));
    #pragma unroll
    for (int b = 0; b < %(B)d; ++b) {
      const float* px = reinterpret_cast<const float*>(stage + s * STEP + b * 4096 + lane * 128);
      const float* py = reinterpret_cast<const float*>(stage + s * STEP + (%(B)d + b) * 4096 + lane * 128);
      #pragma unroll
      for (int c = 0; c < 8; ++c) {
        const dpia::vec<float, 4> vx = dpia::vload<float, 4>(px, 4 * (c ^ sw));
        const dpia::vec<float, 4> vy = dpia::vload<float, 4>(py, 4 * (c ^ sw));
        a = (vx.v[0] * vy.v[0]) + a; a = (vx.v[1] * vy.v[1]) + a;
        a = (vx.v[2] * vy.v[2]) + a; a = (vx.v[3] * vy.v[3]) + a;
      }
    }
    __syncwarp();
    if (%(P)d) { if (lane == 0) mb_arrive(empty + s); }
    else if (lane == 0 && t + %(S)d < T) issue(t + %(S)d, s);
    if ((t %% (32 / %(B)d)) == (32 / %(B)d) - 1) {
      const int r = t / (32 / %(B)d);
      g_tmp4[row0 + lane + r * %(GS)d] = a;
      a = 0.0f;
      __syncwarp();
      if (lane == 0) { __threadfence(); atomicAdd(cnt + r, 1u); }
    }
  }
}
"""


def tensor_map(ptr, rows):
    """2-D fp32 tensor map over [rows][1024] row-major: box 32 x 32, 128B swizzle."""
    import ctypes
    cu = ctypes.CDLL("libcuda.so.1")
    m = (ctypes.c_uint64 * 16)()
    dims = (ctypes.c_uint64 * 2)(1024, rows)
    strides = (ctypes.c_uint64 * 1)(4096)
    box = (ctypes.c_uint32 * 2)(32, 32)
    es = (ctypes.c_uint32 * 2)(1, 1)
    rc = cu.cuTensorMapEncodeTiled(m, 7, 2, ctypes.c_void_p(ptr), dims, strides, box, es, 0, 3, 3, 0)
    assert rc == 0, rc
    return m


def timed(st, launch, reps=50, flush=True):
    ts = []
    for it in range(reps + 5):
        if flush:
            RT.lib().dpia_l2_flush(0, st.handle)
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        launch()
        e1.record(st)
        st.sync()
        if it >= 5:
            ts.append(e0.elapsed_ms(e1))
    return statistics.median(ts) * 1e3


def main():
    RT.init(0)
    st = RT.Stream(0)
    cfg = dot_literal_config()
    exe = executable(compile_program(cfg.text, name="dot_literal"), cfg.launch, cfg.sigma, float_mode=True)
    rng = np.random.default_rng(0)
    for n in ("xs", "ys"):
        exe.upload(n, rng.uniform(0, 1, 1 << 24).astype(np.float32), st)
    header = exe.src[:exe.src.index('extern "C" __global__')]
    (g, l) = cfg.launch
    us = timed(st, lambda: exe.launch(st))
    ref = exe.download("out", st)[0]
    print(f"emitted (512, 32): {us:8.2f} us  {cfg.bytes / us / 1e3:7.1f} GB/s  out {ref!r}", flush=True)
    ptr = {n: exe.buffers[n].ptr for n in ("out", "xs", "ys")}
    tmp = RT.DeviceBuffer(4 * N_CHUNKS, 0)
    cnt = RT.DeviceBuffer(4 * 64, 0)
    cnt.zero()
    RT.lib().dpia_device_sync(0)
    tx, ty = tensor_map(ptr["xs"], N_CHUNKS), tensor_map(ptr["ys"], N_CHUNKS)
    # tail alone: every round published in advance (counters preset), one block
    for (TS, QD) in ((4, 0), (4, 8), (4, 16), (8, 16), (4, 32)):
        src = header + TMA2_KERNEL % {"G": 0, "GS": 4096, "R": 4, "N": N_CHUNKS, "WPR": 128, "S": 2, "B": 1,
                                      "P": 0, "TAIL": 2, "NT": 32, "TS": TS, "QD": QD}
        fn = RT.Module(RT.get_cubin(src), 0).function("tma2_k")
        RT.lib().dpia_kernel_set_smem(fn, 1024 + TS * 2048)
        cnt.upload(np.full(64, 128, np.uint32).view(np.uint8), st)
        args = [RT.C.c_uint64(ptr["out"]), tx, ty, RT.C.c_uint64(tmp.ptr), RT.C.c_uint64(cnt.ptr)]
        us = timed(st, lambda: RT.launch(fn, 0, (1, 1), (32, 1), 1024 + TS * 2048, args, st))
        print(f"tail alone TS={TS} QD={QD}: {us:8.2f} us", flush=True)
    cnt.zero()
    RT.lib().dpia_device_sync(0)
    for tail in (1,):
        for gs in (4096, 8192, 2048):
            for (B, S, P, TS, QD) in ((2, 4, 0, 4, 0), (2, 4, 0, 4, 16), (2, 8, 1, 4, 16), (1, 8, 0, 4, 16)):
                G, R = gs // 32, N_CHUNKS // gs
                src = header + TMA2_KERNEL % {"G": G, "GS": gs, "R": R, "N": N_CHUNKS, "WPR": gs // 32,
                                              "S": S, "B": B, "P": P, "TAIL": tail, "NT": 64 if P else 32,
                                              "TS": TS, "QD": QD}
                fn = RT.Module(RT.get_cubin(src), 0).function("tma2_k")
                smem = 1024 + max(S * B * 8192, TS * 2048)
                RT.lib().dpia_kernel_set_smem(fn, smem)
                args = [RT.C.c_uint64(ptr["out"]), tx, ty, RT.C.c_uint64(tmp.ptr), RT.C.c_uint64(cnt.ptr)]
                go = lambda: RT.launch(fn, 0, (G + 1, 1), (64 if P else 32, 1), smem, args, st)  # noqa: E731
                us = timed(st, go)
                out = exe.download("out", st)[0]
                print(f"tma2 tail={tail} G={G:4d} B={B} S={S:2d} P={P} TS={TS:2d} QD={QD:2d} R={R:2d}: {us:8.2f} us"
                      f"  {cfg.bytes / us / 1e3:7.1f} GB/s  out {out!r} {'==' if out == ref else '!='} emitted",
                      flush=True)
    for gs in (4096,):
        for S in (8,):
            G, R = gs // 32, N_CHUNKS // gs
            src = header + TMA_KERNEL % {"G": G, "GS": gs, "R": R, "N": N_CHUNKS, "WPR": gs // 32, "S": S}
            fn = RT.Module(RT.get_cubin(src), 0).function("tma_k")
            smem = 1024 + S * 8192
            RT.lib().dpia_kernel_set_smem(fn, smem)
            args = [RT.C.c_uint64(ptr["out"]), tx, ty, RT.C.c_uint64(tmp.ptr), RT.C.c_uint64(cnt.ptr)]
            go = lambda: RT.launch(fn, 0, (G + 1, 1), (32, 1), smem, args, st)  # noqa: E731
            us = timed(st, go)
            out = exe.download("out", st)[0]
            b2b = timed(st, go, flush=False)
            print(f"tma    G={G:4d} S={S:3d} R={R:2d}: {us:8.2f} us  {cfg.bytes / us / 1e3:7.1f} GB/s"
                  f"  (no flush {b2b:7.2f} us)  out {out!r} {'==' if out == ref else '!='} emitted",
                  flush=True)
    for L in (32,):
        for gs in (16384, 8192):
            G = gs // L
            R = N_CHUNKS // gs
            src = header + KERNEL % {"L": L, "G": G, "GS": gs, "R": R, "N": N_CHUNKS, "WPR": gs // 32}
            fn = RT.Module(RT.get_cubin(src), 0).function("stream_k")
            args = [RT.C.c_uint64(ptr["out"]), RT.C.c_uint64(ptr["xs"]), RT.C.c_uint64(ptr["ys"]),
                    RT.C.c_uint64(tmp.ptr), RT.C.c_uint64(cnt.ptr)]
            go = lambda: RT.launch(fn, 0, (G + 1, 1), (L, 1), 32 + 4 * 2048, args, st)  # noqa: E731
            us = timed(st, go)
            out = exe.download("out", st)[0]
            b2b = timed(st, go, flush=False)
            print(f"stream G={G:4d} L={L:3d} R={R:2d}: {us:8.2f} us  {cfg.bytes / us / 1e3:7.1f} GB/s"
                  f"  (no flush {b2b:7.2f} us)  out {out!r} {'==' if out == ref else '!='} emitted",
                  flush=True)


if __name__ == "__main__":
    main()
