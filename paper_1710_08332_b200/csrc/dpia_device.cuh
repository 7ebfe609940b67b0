// Device-side templates included by every kernel the DPIA CUDA backend emits.
//
// * dpia::vec<T,W>      -- the (vec W) data type: W lanes, naturally aligned so a
//                          whole-vector access is one 64/128-bit LDG/STG/LDS/STS
//                          (the backend's rendering of asVector/asScalar, which the
//                          reference emits as OpenCL vloadW/vstoreW, SRC/codegen_c.py:482-493)
// * dpia::block_combine -- the cooperative work-group combine behind reduceLocal:
//                          warp-shuffle tree (__shfl_down_sync) + one shared-memory
//                          hop per warp; absent from the reference, whose single
//                          kernels stop at partial sums (programs/dotvec.dpia:4-5)
// * dpia::fma2          -- two independent scalar FMAs issued as one packed
//                          Blackwell fma.rn.f32x2 (FFMA2); per lane identical
//                          to the contracted scalar c + a*b
// * dpia::peer_sum      -- fused cross-GPU combine: the last block of every
//                          rank stores its result into every peer's NVLink-
//                          mapped mailbox and sums all ranks' results in rank
//                          order (replaces ncclAllReduce of the partials)
// * dpia::grid_arrive   -- last-block-done detection used to fuse a single
//                          work-group tail phase into the preceding grid phase
// * dpia::bulk_stage    -- toLocal staging of a whole input as one TMA bulk
//                          copy (cp.async.bulk + mbarrier complete_tx)
// * dpia::vload32       -- one 32-byte (sm_100 LDG.E.256) vector load: the
//                          register queues of a work-item's sequential fold
// * dpia::ring_*        -- a single thread's shared-memory ring of TMA bulk
//                          copies (the top-level sequential fold of a tail)
// * dpia::stream_*      -- per-round publication of a grid phase's partials
//                          and the streaming tail's wait for them
// * dpia::tma_tile_2d   -- one 2-D box of an input (a toLocal k-tile) as a
//                          TMA tensor copy (cp.async.bulk.tensor.2d through a
//                          CUtensorMap kernel parameter, mbarrier complete_tx)
//
// Self-contained: NVRTC compiles it without any system header.
#pragma once

namespace dpia {

template <class T, int W>
struct alignas((sizeof(T) * W <= 16 && (W & (W - 1)) == 0) ? sizeof(T) * W
               : (sizeof(T) * W > 16 && (W & (W - 1)) == 0) ? 16 : sizeof(T)) vec {
  T v[W];
};

template <class T, int W>
__device__ __forceinline__ vec<T, W> splat(T x) {
  vec<T, W> r;
#pragma unroll
  for (int k = 0; k < W; ++k) r.v[k] = x;
  return r;
}

#define DPIA_VEC_BINOP(OP)                                                             \
  template <class T, int W>                                                            \
  __device__ __forceinline__ vec<T, W> operator OP(const vec<T, W>& a, const vec<T, W>& b) { \
    vec<T, W> r;                                                                       \
    _Pragma("unroll") for (int k = 0; k < W; ++k) r.v[k] = a.v[k] OP b.v[k];           \
    return r;                                                                          \
  }                                                                                    \
  template <class T, int W>                                                            \
  __device__ __forceinline__ vec<T, W> operator OP(const vec<T, W>& a, T b) {          \
    vec<T, W> r;                                                                       \
    _Pragma("unroll") for (int k = 0; k < W; ++k) r.v[k] = a.v[k] OP b;                \
    return r;                                                                          \
  }                                                                                    \
  template <class T, int W>                                                            \
  __device__ __forceinline__ vec<T, W> operator OP(T a, const vec<T, W>& b) {          \
    vec<T, W> r;                                                                       \
    _Pragma("unroll") for (int k = 0; k < W; ++k) r.v[k] = a OP b.v[k];                \
    return r;                                                                          \
  }
DPIA_VEC_BINOP(+)
DPIA_VEC_BINOP(-)
DPIA_VEC_BINOP(*)
DPIA_VEC_BINOP(/)
#undef DPIA_VEC_BINOP

template <class T, int W>
__device__ __forceinline__ vec<T, W> operator-(const vec<T, W>& a) {
  vec<T, W> r;
#pragma unroll
  for (int k = 0; k < W; ++k) r.v[k] = -a.v[k];
  return r;
}

__device__ __forceinline__ float abs_(float x) { return fabsf(x); }
__device__ __forceinline__ double abs_(double x) { return fabs(x); }
__device__ __forceinline__ long long abs_(long long x) { return x < 0 ? -x : x; }
template <class T, int W>
__device__ __forceinline__ vec<T, W> abs_(const vec<T, W>& a) {
  vec<T, W> r;
#pragma unroll
  for (int k = 0; k < W; ++k) r.v[k] = abs_(a.v[k]);
  return r;
}

// whole-vector read of lanes p[i .. i+W) (i is a multiple of W by construction)
template <class T, int W>
__device__ __forceinline__ vec<T, W> vload(const T* p, long long i) {
  return *reinterpret_cast<const vec<T, W>*>(p + i);
}
template <class T, int W>
__device__ __forceinline__ void vstore(T* p, long long i, const vec<T, W>& x) {
  *reinterpret_cast<vec<T, W>*>(p + i) = x;
}

// ------------------------------------------------------------ shuffles
__device__ __forceinline__ float shfl_down(float x, int d) {
  return __shfl_down_sync(0xffffffffu, x, d);
}
__device__ __forceinline__ double shfl_down(double x, int d) {
  return __shfl_down_sync(0xffffffffu, x, d);
}
__device__ __forceinline__ long long shfl_down(long long x, int d) {
  return __shfl_down_sync(0xffffffffu, x, d);
}
template <class T, int W>
__device__ __forceinline__ vec<T, W> shfl_down(const vec<T, W>& x, int d) {
  vec<T, W> r;
#pragma unroll
  for (int k = 0; k < W; ++k) r.v[k] = shfl_down(x.v[k], d);
  return r;
}

// Fold (value, valid) pairs of one warp into lane 0.  op(x, acc) is the
// reduction function f x acc of the program; it must be associative and
// commutative (the contract of reduceLocal).
template <class T, class Op>
__device__ __forceinline__ void warp_fold(T& v, bool& has, Op op) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    T o = shfl_down(v, d);
    bool oh = __shfl_down_sync(0xffffffffu, has, d);
    if (oh) {
      v = has ? op(o, v) : o;
      has = true;
    }
  }
}

// Work-group combine.  Every thread passes its partial (valid iff `has`);
// every thread receives the combination of all valid partials.  `scratch`
// holds NWARP_MAX+1 slots of T in shared memory.  Two barriers; safe to call
// repeatedly (slot ownership alternates between the partial slots and the
// broadcast slot, so no trailing barrier is needed).
template <class T, class Op>
__device__ __forceinline__ T block_combine(T v, bool has, Op op, T* scratch, bool* scratch_has,
                                           int tid, int nthreads, bool& has_out) {
  warp_fold(v, has, op);
  const int lane = tid & 31, warp = tid >> 5, nwarps = (nthreads + 31) >> 5;
  if (nwarps == 1) {
    if (lane == 0) { scratch[32] = v; scratch_has[32] = has; }
    __syncthreads();
    T r = scratch[32];
    has_out = scratch_has[32];
    __syncwarp();  // lane 0 may rewrite the slot in the next call
    return r;
  }
  if (lane == 0) { scratch[warp] = v; scratch_has[warp] = has; }
  __syncthreads();
  if (warp == 0) {
    bool h = lane < nwarps ? scratch_has[lane] : false;
    T w = h ? scratch[lane] : v;
    warp_fold(w, h, op);
    if (lane == 0) { scratch[32] = w; scratch_has[32] = h; }
  }
  __syncthreads();
  has_out = scratch_has[32];
  return scratch[32];
}

// c0 += a0*b0 and c1 += a1*b1 as one FFMA2 (sm_100a).  When b0 and b1 are
// the same register ptxas uses the broadcast-operand form.
__device__ __forceinline__ void fma2(float& c0, float& c1, float a0, float b0, float a1, float b1) {
  unsigned long long c, a, b;
  asm("mov.b64 %0, {%1,%2};" : "=l"(c) : "f"(c0), "f"(c1));
  asm("mov.b64 %0, {%1,%2};" : "=l"(a) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1,%2};" : "=l"(b) : "f"(b0), "f"(b1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(b));
  asm("mov.b64 {%0,%1}, %2;" : "=f"(c0), "=f"(c1) : "l"(c));
}

// Last-block-done detection for a fused single-work-group tail phase.
// Returns true in exactly one block: the last to finish the grid phase.
__device__ __forceinline__ bool grid_arrive(unsigned int* counter, int tid, bool* flag) {
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned int nblocks = gridDim.x * gridDim.y * gridDim.z;
    const unsigned int ticket = atomicAdd(counter, 1u);
    *flag = (ticket == nblocks - 1);
  }
  __syncthreads();
  if (*flag) __threadfence();
  return *flag;
}

// Cross-GPU sum of n scalars, run by warp 0 (lanes tid < min(32, nthreads))
// of the last block of every rank after the rank-local result is in
// out[0..n).  boxes[p] is rank p's mailbox (mapped into this device through
// CUDA IPC / NVLink P2P): two parities x world x n slots of 16 bytes.
// Launch e uses parity e & 1, so a rank that has already moved on to launch
// e+1 never overwrites a slot another rank is still reading for launch e.
//
// Publish: lane l writes the slots of ranks l, l+32, ... in parallel.  A
// 4-byte value travels with its epoch in ONE single-copy-atomic 64-bit word
// {value bits, epoch} (no ordering needed between them); an 8-byte value is
// stored first and its epoch (offset 8) after it with a system-scope
// release.  One system-scope fence per lane (world > 1) then pushes the
// stores out, so
// the exchange costs about one NVLink round trip whatever the world size
// (a single thread publishing rank by rank paid one release per peer).
// Gather: lane q polls rank q's slot in this rank's mailbox (relaxed /
// acquire, system scope); the values meet in lane order through shuffles, so
// every rank sums them in the same rank order and holds the identical total.
// A lane that waits longer than ~1e9 cycles (~0.5 s) raises the mailbox's error word
// (the host checks it) instead of hanging.
template <class T>
__device__ void peer_sum(T* out, int n, const unsigned long long* boxes, int rank, int world,
                         unsigned int epoch, int lane, int nthreads) {
  const int nl = nthreads < 32 ? nthreads : 32;
  const unsigned mask = nl == 32 ? 0xffffffffu : ((1u << nl) - 1u);
  const int par = static_cast<int>(epoch & 1u);
  for (int p = lane; p < world; p += nl) {
    char* base = reinterpret_cast<char*>(boxes[p]);
    for (int k = 0; k < n; ++k) {
      char* slot = base + (static_cast<size_t>((par * world + rank) * n + k) << 4);
      if constexpr (sizeof(T) == 4) {
        const unsigned int bits = *reinterpret_cast<const unsigned int*>(&out[k]);
        const unsigned long long w = (static_cast<unsigned long long>(epoch) << 32) | bits;
        asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(slot), "l"(w) : "memory");
      } else {
        *reinterpret_cast<volatile T*>(slot) = out[k];
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(slot + 8), "r"(epoch) : "memory");
      }
    }
  }
  // push the relaxed words out to the peers (one fence per lane, overlapped);
  // a lone rank reads back its own store in program order and needs none
  if (sizeof(T) == 4 && world > 1) __threadfence_system();
  char* mine = reinterpret_cast<char*>(boxes[rank]);
  unsigned int* err = reinterpret_cast<unsigned int*>(mine + (static_cast<size_t>(2 * world * n) << 4));
  for (int k = 0; k < n; ++k) {
    T acc = T(0);
    for (int q0 = 0; q0 < world; q0 += nl) {
      const int q = q0 + lane;
      T v = T(0);
      if (q < world) {
        char* slot = mine + (static_cast<size_t>((par * world + q) * n + k) << 4);
        const long long t0 = clock64();
        for (;;) {
          if constexpr (sizeof(T) == 4) {
            unsigned long long w;
            asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(w) : "l"(slot) : "memory");
            if (static_cast<unsigned int>(w >> 32) == epoch) {
              const unsigned int bits = static_cast<unsigned int>(w);
              v = *reinterpret_cast<const T*>(&bits);
              break;
            }
          } else {
            unsigned int e;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(e) : "l"(slot + 8) : "memory");
            if (e == epoch) { v = *reinterpret_cast<volatile T*>(slot); break; }
          }
          if (clock64() - t0 > 1000000000LL) { *err = 1u; break; }
        }
      }
      for (int j = 0; j < nl && q0 + j < world; ++j) {
        const T vj = __shfl_sync(mask, v, j);
        acc = (q0 + j == 0) ? vj : acc + vj;
      }
    }
    if (lane == 0) out[k] = acc;
  }
}

// Bulk (TMA) staging of `bytes` contiguous bytes global -> shared, issued by
// thread 0 and completed on an mbarrier in shared memory (used once per
// block, phase 0): the emitter's lowering of a block-invariant toLocal copy
// of a whole input.  Every thread returns once the data has landed.  Both
// addresses are 16-byte aligned and bytes is a multiple of 16, < 2^20.
__device__ __forceinline__ void bulk_stage(void* smem_dst, const void* gsrc, unsigned bytes,
                                           unsigned long long* mbar, int tid) {
  const unsigned bar = static_cast<unsigned>(__cvta_generic_to_shared(mbar));
  const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(dst), "l"(gsrc), "r"(bytes), "r"(bar)
        : "memory");
  }
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar)
        : "memory");
  }
}

// ------------------------------------------------------ 32-byte loads
// One 256-bit global load (sm_100: LDG.E.ENL2.256) of W = 32 / sizeof(T)
// consecutive scalars at p + i, 32-byte aligned.  NC: the buffer is read-only
// for the whole kernel (a const __restrict__ input): the non-coherent path.
// L2 prefetch of the 128-byte line at p (a later iteration's operands)
template <class T>
__device__ __forceinline__ void prefetch_l2(const T* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <bool NC>
__device__ __forceinline__ vec<float, 8> vload32(const float* p, long long i) {
  vec<float, 8> r;
  if (NC)
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                   "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7]) : "l"(p + i));
  else
    asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                   "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7]) : "l"(p + i) : "memory");
  return r;
}
template <bool NC>
__device__ __forceinline__ vec<long long, 4> vload32(const long long* p, long long i) {
  vec<long long, 4> r;
  if (NC)
    asm volatile("ld.global.nc.v4.s64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(r.v[0]), "=l"(r.v[1]), "=l"(r.v[2]), "=l"(r.v[3]) : "l"(p + i));
  else
    asm volatile("ld.global.v4.s64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(r.v[0]), "=l"(r.v[1]), "=l"(r.v[2]), "=l"(r.v[3]) : "l"(p + i) : "memory");
  return r;
}

// --------------------------------------------- single-thread bulk ring
// One thread streams a contiguous global range through S shared-memory
// slots with TMA bulk copies; slot s completes on mbarrier mb[s] (one
// expect_tx per fill, covering every stream that shares the slot index).
// ring_init: after data other threads wrote through the generic proxy was
// made visible to this thread (the fused tail's grid_arrive), order it
// before the async-proxy reads.
__device__ __forceinline__ void ring_init(unsigned long long* mb, int slots) {
  for (int s = 0; s < slots; ++s) {
    const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(mb + s));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void ring_expect(unsigned long long* mb, unsigned bytes) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(mb));
  // the slot's previous contents were read through the generic proxy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void ring_copy(void* dst, const void* src, unsigned bytes,
                                          unsigned long long* mb) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(mb));
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(d), "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void ring_wait(unsigned long long* mb, unsigned parity) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(mb));
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
  }
}

// --------------------------------------- chained launches (PDL, sm_90+)
// pdl_trigger: this grid's dependent (the next launch on the stream, when it
// was launched chained) may be scheduled now.  pdl_wait_once: wait, once per
// thread, until the grid this one is chained behind has completed and its
// memory is visible.  Both are no-ops for an ordinary launch.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// TRIGGER: let the dependent launch once the previous grid has completed
// (at most two launches resident; the kernel did not trigger at its top).
// A block that never waits triggers when it exits.
template <bool TRIGGER = false>
__device__ __forceinline__ void pdl_wait_once(bool& pending) {
  if (pending) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    pending = false;
  }
}

// --------------------------------------------- streaming tail
// A grid phase over n work-items (gsize per round, whole warps) publishes
// each round on its own counter: every warp, once all its lanes wrote their
// partial of round r, adds 1 to cnt[r] (release).  The tail -- one thread of
// an extra block, running from the start -- waits before each ring copy of
// partials [., hi) until every round below hi has all its warps counted
// (acquire), then orders the async-proxy copy after those writes.
__device__ __forceinline__ void stream_publish(unsigned int* c) {
  __threadfence();
  atomicAdd(c, 1u);
}
__device__ __forceinline__ void stream_wait(const unsigned int* cnt, long long& ready, long long hi,
                                            long long gsize, long long n) {
  if (hi > n) hi = n;
  while (ready < hi) {
    const long long r = ready / gsize;
    const long long items = n - r * gsize < gsize ? n - r * gsize : gsize;
    const unsigned want = static_cast<unsigned>(items / 32);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt + r) : "memory");
    } while (v < want);
    ready = (r + 1) * gsize < n ? (r + 1) * gsize : n;
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Slot pipelining of a streaming tail across chained launches: launch e
// uses partials/counters slice e % K; rel[s] holds the epoch of the last
// launch that finished with slice s.  A launch waits (once per thread) for
// the launch K back to have released its slice before it first touches it;
// the tail releases it after its last read.  The launcher's epochs start at
// 16 and each rel word starts at its slot's first epoch minus K.
__device__ __forceinline__ void parity_wait_once(bool& pending, const unsigned int* rel,
                                                 unsigned int epoch, unsigned int slots) {
  if (pending) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(rel) : "memory");
    } while (v + slots < epoch);
    pending = false;
  }
}
__device__ __forceinline__ void parity_release(unsigned int* rel, unsigned int epoch) {
  __threadfence();
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(rel), "r"(epoch) : "memory");
}

// --------------------------------------------- 2-D TMA tensor tiles
// The CUtensorMap of an input, passed by value as a __grid_constant__ kernel
// parameter (runtime: dpia_tensor_map_2d).  tma_tile_2d: the issuing thread
// announces `bytes` on the slice's mbarrier and copies the box whose
// innermost coordinate is x and row coordinate y into shared memory
// (plain row-major box layout); waiters use ring_wait on the same mbarrier.
// The slice was last read through the generic proxy (the previous use of
// the rotating buffer), and every such read is ordered before this call by
// the CTA barrier the caller issues it after -- the same release the
// consumer arrive of a full/empty mbarrier pipeline gives; no proxy fence.
struct alignas(64) TensorMap {
  unsigned long long w[16];
};
__device__ __forceinline__ void tile_bar_init(unsigned long long* mb, int slots, unsigned count) {
  for (int s = 0; s < slots; ++s) {
    const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(mb + s));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(count) : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_tile_2d(void* dst, const TensorMap* map, int x, int y,
                                            unsigned bytes, unsigned long long* mb) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(mb));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];"
      ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(b)
      : "memory");
}

// TMA tensor store of a 2-D box from shared memory (the work-item row
// stores of `_finish_rows`): the writers fence their generic-proxy stores to
// the slot for the async proxy and sync; one thread issues the copy into the
// bulk async-group, commits, and waits on the group (.read: the slot may be
// rewritten; plain: the global writes are complete) before the slot is reused
// or the block ends.
__device__ __forceinline__ void tma_store_2d(const TensorMap* map, int x, int y, const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
      ::"l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y),
        "r"(static_cast<unsigned>(__cvta_generic_to_shared(src)))
      : "memory");
}
__device__ __forceinline__ void fence_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void grid_reset(unsigned int* counter, int tid) {
  if (tid == 0) *counter = 0u;
}

}  // namespace dpia
