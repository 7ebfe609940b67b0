"""Where does config 1's literal program lose its time, and what would an
order-preserving code generator recover?  (GPU box; measurement
infrastructure, not product.)

    python tools/litexp.py

Hand edits of the emitted dot_literal kernel (512 x 32, 16384 work-items),
each computing the identical left fold in the identical order (results are
compared bit for bit with the emitted kernel):
  emitted      the backend's output
  vec4-items   each work-item reads its contiguous chunk as float4 pairs
               (4 FMAs per load pair, same order)
  staged-tail  the last block's 32 threads stage the 16384 partials through
               shared memory in 4096-element slices; thread 0 folds from
               shared memory (same order)
  both         vec4-items + staged-tail
  hint-items   the emitted loop with `#pragma unroll 4` and the inputs
               declared 16-byte aligned (__builtin_assume_aligned): does
               nvcc's load vectorizer produce vec4-items by itself?
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import dot_literal_config  # noqa: E402

ITEM_OLD = """    for (int i_2_3 = 0; i_2_3 < 1024; i_2_3 += 1) {
      acc_1_2 = ((xs[i_2_3 + 1024 * i_3_1] * ys[i_2_3 + 1024 * i_3_1]) + acc_1_2);
    }"""
ITEM_NEW = """    for (int j = 0; j < 256; j += 1) {
      const float4 xv = *reinterpret_cast<const float4*>(xs + 4 * j + 1024 * i_3_1);
      const float4 yv = *reinterpret_cast<const float4*>(ys + 4 * j + 1024 * i_3_1);
      acc_1_2 = ((xv.x * yv.x) + acc_1_2);
      acc_1_2 = ((xv.y * yv.y) + acc_1_2);
      acc_1_2 = ((xv.z * yv.z) + acc_1_2);
      acc_1_2 = ((xv.w * yv.w) + acc_1_2);
    }"""
HINT_DECL_OLD = "  const int dpia_nthreads = 32;\n"
HINT_DECL_NEW = ("  const int dpia_nthreads = 32;\n"
                 "  xs = static_cast<const float*>(__builtin_assume_aligned(xs, 16));\n"
                 "  ys = static_cast<const float*>(__builtin_assume_aligned(ys, 16));\n")
TAIL_OLD = """    if (dpia_tid == 0) {
      for (int i_6_5 = 0; i_6_5 < 16384; i_6_5 += 1) {
        acc_5_4 = (acc_5_4 + g_tmp4[i_6_5]);
      }
    }"""
TAIL_NEW = """    float* stage = reinterpret_cast<float*>(dpia_smem);
    for (int s0 = 0; s0 < 16384; s0 += 4096) {
      for (int k = dpia_tid; k < 1024; k += 32)
        reinterpret_cast<float4*>(stage)[k] = __ldcg(reinterpret_cast<const float4*>(g_tmp4 + s0) + k);
      __syncwarp();
      if (dpia_tid == 0) {
        for (int i_6_5 = 0; i_6_5 < 4096; i_6_5 += 1) {
          acc_5_4 = (acc_5_4 + stage[i_6_5]);
        }
      }
      __syncwarp();
    }"""


def timed(st, launch, reps=50):
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
    cfg = dot_literal_config()
    exe = executable(compile_program(cfg.text, name="dot_literal"), cfg.launch, cfg.sigma, float_mode=True)
    rng = np.random.default_rng(0)
    for n in ("xs", "ys"):
        exe.upload(n, rng.uniform(0, 1, 1 << 24).astype(np.float32), st)
    base = exe.src
    assert ITEM_OLD in base and TAIL_OLD in base
    variants = {"emitted": base, "vec4-items": base.replace(ITEM_OLD, ITEM_NEW),
                "staged-tail": base.replace(TAIL_OLD, TAIL_NEW),
                "both": base.replace(ITEM_OLD, ITEM_NEW).replace(TAIL_OLD, TAIL_NEW),
                "hint-items": base.replace(HINT_DECL_OLD, HINT_DECL_NEW).replace(
                    ITEM_OLD, "    #pragma unroll 4\n" + ITEM_OLD)}
    args = exe._args[0]
    (g, l) = cfg.launch
    ref = None
    for name, src in variants.items():
        mod = RT.Module(RT.get_cubin(src), 0)
        fn = mod.function("dot_literal_k0")
        smem = 16384 if "float* stage =" in src else 0
        us = timed(st, lambda: RT.launch(fn, 0, (g, 1), (l, 1), smem, args, st))
        out = exe.download("out", st)
        st.sync()
        ref = out[0] if ref is None else ref
        print(f"{name:12s}: {us:8.2f} us  {cfg.bytes / us / 1e3:7.1f} GB/s  frac {cfg.bytes / us / 1e3 / 6554.9:.3f}"
              f"  out {out[0]!r} {'==' if out[0] == ref else '!='} emitted", flush=True)


if __name__ == "__main__":
    main()
