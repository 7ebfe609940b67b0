"""Can consecutive launches of config 1's literal program overlap their
serial tails?  (GPU box; measurement infrastructure, not product.)

    python tools/pipetail.py

Hand-written streaming-tail kernel (TMA row folds, 4 rounds of 128 x 32
work-items, one extra tail block, the same fold orders as the emitted
dot_literal), launched back to back with programmatic dependent launch over
3 rotating input sets (384 MiB > L2), 30 steps between one event pair:

  PIPE=0  as emitted today: a step's blocks wait for the previous grid before
          they first write the partials / counters (griddepcontrol.wait), so
          step k's tail starts only after step k-1's tail ended
  PIPE=1  partials and round counters double-buffered by launch parity
          (epoch & 1, a kernel argument); a step waits only for the step two
          back to release its parity (a per-parity release word the tail
          sets after its last read), and for the previous grid only before
          it writes `out`; consecutive tails run concurrently

Every step's result is compared bit for bit with an unchained launch.
"""
import ctypes
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import dot_literal_config  # noqa: E402

N_ITEMS, CHUNK, G, L, R, S, B = 16384, 1024, 128, 32, 4, 4, 2
KERNEL = r"""
struct __align__(64) TMap { unsigned long long w[16]; };
__device__ __forceinline__ void tma2d(void* dst, const TMap* m, int x, int y, unsigned long long* mb) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%%0], [%%1, {%%2, %%3}], [%%4];"
               :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(reinterpret_cast<unsigned long long>(m)),
                  "r"(x), "r"(y), "r"((unsigned)__cvta_generic_to_shared(mb)) : "memory");
}
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %%0, [%%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
extern "C" __global__ void __launch_bounds__(32) pipe_k(float* __restrict__ out, const __grid_constant__ TMap tx,
    const __grid_constant__ TMap ty, float* g_all, unsigned int* cnt_all, unsigned int epoch) {
  extern __shared__ __align__(1024) unsigned char dpia_smem[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int tid = threadIdx.x;
  const int par = %(PIPE)d ? (int)(epoch & 1u) : 0;
  float* g = g_all + par * %(N)d;
  unsigned int* cnt = cnt_all + par * %(R)d;
  unsigned int* rel = cnt_all + 2 * %(R)d;
  constexpr int GS = %(G)d * 32, STEPS = 32 / %(B)d, STEP = %(B)d * 8192;
  if (blockIdx.x == %(G)d) {
    if (tid != 0) return;
    if (!%(PIPE)d) asm volatile("griddepcontrol.wait;" ::: "memory");
    else { while (ld_acq(rel + par) + 2u < epoch) { } }   // parity released by the step two back
    float acc = 0.0f;
    unsigned long long* mb = reinterpret_cast<unsigned long long*>(dpia_smem);
    dpia::ring_init(mb, 4);
    int ready = 0;
    #define WAIT_UPTO(hi) while (ready < (hi)) { const int r = ready / GS; \
        while (ld_acq(cnt + r) < GS / 32) { } ready = (r + 1) * GS; \
        asm volatile("fence.proxy.async.global;" ::: "memory"); }
    for (int s = 0; s < 4; ++s) {
      WAIT_UPTO((s + 1) * 512);
      dpia::ring_expect(mb + s, 2048u);
      dpia::ring_copy(dpia_smem + 1024 + s * 2048, g + s * 512, 2048u, mb + s);
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
        dpia::ring_copy(dpia_smem + 1024 + s * 2048, g + jo + 2048, 2048u, mb + s);
      }
    }
    for (int r = 0; r < %(R)d; ++r) cnt[r] = 0u;
    if (%(PIPE)d) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%%0], %%1;" :: "l"(rel + par), "r"(epoch) : "memory");
      asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    out[0] = acc;
    return;
  }
  unsigned long long* full = reinterpret_cast<unsigned long long*>(dpia_smem);
  unsigned char* stage = dpia_smem + 1024;
  const int row0 = blockIdx.x * 32;
  constexpr int T = %(R)d * STEPS;
  if (tid == 0) dpia::tile_bar_init(full, %(S)d, 2 * %(B)d);
  __syncwarp();
  auto issue = [&](int u, int s) {
    const int x = (u %% STEPS) * 32 * %(B)d, y = row0 + (u / STEPS) * GS;
    #pragma unroll
    for (int b = 0; b < %(B)d; ++b) {
      dpia::tma_tile_2d(stage + s * STEP + b * 4096, reinterpret_cast<const dpia::TensorMap*>(&tx), x + 32 * b, y, 4096u, full + s);
      dpia::tma_tile_2d(stage + s * STEP + (%(B)d + b) * 4096, reinterpret_cast<const dpia::TensorMap*>(&ty), x + 32 * b, y, 4096u, full + s);
    }
  };
  if (tid == 0) for (int t = 0; t < %(S)d; ++t) issue(t, t);
  float a = 0.0f;
  const int sw = tid & 7;
  bool waited = false;
  for (int t = 0; t < T; ++t) {
    const int s = t %% %(S)d;
    dpia::ring_wait(full + s, (unsigned)((t / %(S)d) & 1));
    #pragma unroll
    for (int b = 0; b < %(B)d; ++b) {
      const float* px = reinterpret_cast<const float*>(stage + s * STEP + b * 4096 + tid * 128);
      const float* py = reinterpret_cast<const float*>(stage + s * STEP + (%(B)d + b) * 4096 + tid * 128);
      #pragma unroll
      for (int c = 0; c < 8; ++c) {
        const dpia::vec<float, 4> vx = dpia::vload<float, 4>(px, 4 * (c ^ sw));
        const dpia::vec<float, 4> vy = dpia::vload<float, 4>(py, 4 * (c ^ sw));
        a = (vx.v[0] * vy.v[0]) + a; a = (vx.v[1] * vy.v[1]) + a;
        a = (vx.v[2] * vy.v[2]) + a; a = (vx.v[3] * vy.v[3]) + a;
      }
    }
    __syncwarp();
    if (tid == 0 && t + %(S)d < T) issue(t + %(S)d, s);
    if ((t %% STEPS) == STEPS - 1) {
      if (!waited) {
        if (%(PIPE)d) { while (ld_acq(rel + par) + 2u < epoch + 0u) { } }
        else asm volatile("griddepcontrol.wait;" ::: "memory");
        waited = true;
      }
      const int r = t / STEPS;
      g[row0 + tid + r * GS] = a;
      a = 0.0f;
      __syncwarp();
      if (tid == 0) { __threadfence(); atomicAdd(cnt + r, 1u); }
    }
  }
}
"""


def tensor_map(ptr, rows):
    return RT.tensor_map_2d(4, ptr, rows, CHUNK, CHUNK * 4, 32, 32, 128)


def main():
    RT.init(0)
    st = RT.Stream(0)
    cfg = dot_literal_config()
    exe = executable(compile_program(cfg.text, name="dot_literal"), cfg.launch, cfg.sigma, float_mode=True)
    header = exe.src[:exe.src.index('extern "C" __global__')]
    rng = np.random.default_rng(0)
    sets = []
    for _ in range(3):
        xs = rng.uniform(0, 1, N_ITEMS * CHUNK).astype(np.float32)
        ys = rng.uniform(0, 1, N_ITEMS * CHUNK).astype(np.float32)
        bx, by = RT.DeviceBuffer(xs.nbytes), RT.DeviceBuffer(ys.nbytes)
        bx.upload(xs, st)
        by.upload(ys, st)
        exe.upload("xs", xs, st)
        exe.upload("ys", ys, st)
        exe.launch(st)
        want = np.asarray(exe.download("out", st)).copy()
        st.sync()
        sets.append((bx, by, tensor_map(bx.ptr, N_ITEMS), tensor_map(by.ptr, N_ITEMS), want))
    smem = 1024 + S * B * 8192
    for pipe in (0, 1):
        src = header + KERNEL % {"PIPE": pipe, "N": N_ITEMS, "R": R, "G": G, "S": S, "B": B}
        fn = RT.Module(RT.get_cubin(src), 0).function("pipe_k")
        RT.lib().dpia_kernel_set_smem(fn, smem)
        g = RT.DeviceBuffer(2 * N_ITEMS * 4)
        cnt = RT.DeviceBuffer(4 * (2 * R + 2))
        init = np.zeros(2 * R + 2, np.uint32)
        init[2 * R + 1] = 1
        cnt.upload(init, st)
        outs = [RT.DeviceBuffer(4) for _ in range(30)]
        epoch = [2]

        def go(k, chain):
            bx, by, tx, ty, _ = sets[k % 3]
            args = [RT.C.c_uint64(outs[k].ptr), tx, ty, RT.C.c_uint64(g.ptr), RT.C.c_uint64(cnt.ptr),
                    ctypes.c_uint(epoch[0])]
            epoch[0] += 1
            RT.launch(fn, 0, (G + 1, 1), (L, 1), smem, args, st, pdl=chain)

        for k in range(6):
            go(k % 30, True)
        st.sync()
        ts = []
        for rep in range(5):
            e0, e1 = RT.Event(0), RT.Event(0)
            e0.record(st)
            for k in range(30):
                go(k, True)
            e1.record(st)
            st.sync()
            ts.append(e0.elapsed_ms(e1) / 30)
        ok = True
        for k in range(30):
            got = np.empty(1, np.float32)
            outs[k].download(got.view(np.uint8), st)
            st.sync()
            ok &= got.view(np.uint32)[0] == sets[k % 3][4].view(np.uint32)[0]
        us = statistics.median(ts) * 1e3
        print(f"PIPE={pipe}: {us:7.2f} us per chained step  {8 * N_ITEMS * CHUNK / us / 1e3:7.1f} GB/s  "
              f"all 30 steps bit-identical: {bool(ok)}", flush=True)


if __name__ == "__main__":
    main()
