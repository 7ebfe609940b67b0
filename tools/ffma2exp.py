"""FFMA2 experiment (GPU box): the emitted mm kernel with its inner
register-tile update rewritten by hand into packed fma.rn.f32x2 (two
accumulators per instruction, the A pair from shared memory, the B value
broadcast), timed like bench.py next to the unmodified kernel.

    python tools/ffma2exp.py

Measurement infrastructure only: it decides whether the emitter should
select FFMA2 for the register-tile update.
"""
import os
import re
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import mm_config  # noqa: E402
from paper_1710_08332_b200.cuda.emit import emit_cuda  # noqa: E402
from paper_1710_08332_b200.launcher import Executable  # noqa: E402

FMA2 = r"""
__device__ __forceinline__ void fma2(float& c0, float& c1, float a0, float a1, float b) {
  unsigned long long c, a, bb;
  asm("mov.b64 %0, {%1,%2};" : "=l"(c) : "f"(c0), "f"(c1));
  asm("mov.b64 %0, {%1,%2};" : "=l"(a) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1,%1};" : "=l"(bb) : "f"(b));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(bb));
  asm("mov.b64 {%0,%1}, %2;" : "=f"(c0), "=f"(c1) : "l"(c));
}
"""

PAT = re.compile(r"for \(int (i_\d+_\d+) = 0; \1 < (\d+); \1 \+= 1\) \{\s*"
                 r"(acc_\d+_\d+)\[([^\]]*)\] = \(\3\[\4\] \+ \((tmp\d+_\d+)\[([^\]]*)\] \* "
                 r"(tmp\d+_\d+\[[^\]]*\])\)\);\s*\}")


def rewrite(src):
    def rep(m):
        i, n, acc, ai, a, aa, b = m.groups()
        return (f"for (int {i} = 0; {i} < {n}; {i} += 2) {{\n"
                f"  fma2({acc}[{ai}], {acc}[{ai} + 1], {a}[{aa}], {a}[{aa} + 1], {b});\n}}")
    out, n = PAT.subn(rep, src)
    assert n == 1, n
    k = out.index('extern "C"')
    return out[:k] + FMA2 + out[k:]


def timed(exe, st, reps=10):
    ts = []
    for i in range(reps + 3):
        RT.lib().dpia_l2_flush(0, st.handle)
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        exe.launch(st)
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
    for BK in (8, 16):
        cfg = mm_config(BK=BK)
        prog = compile_program(cfg.text, name="mm")
        outs = [(n, t) for n, t, k in prog.params if k == "out"]
        ins = [(n, t) for n, t, k in prog.params if k == "in"]
        src, sig = emit_cuda(prog.imperative, outs, ins, True, "mm", sigma=cfg.sigma, launch=cfg.launch)
        res = {}
        for label, s in (("FFMA", src), ("FFMA2", rewrite(src))):
            exe = Executable(s, sig, 0, True, dict(cfg.sigma), geometry=cfg.launch).compile().allocate()
            exe.upload("A", A, st)
            exe.upload("B", B, st)
            ms = timed(exe, st)
            res[label] = exe.download("out", st).reshape(4096, 4096)
            print(f"BK={BK} {label:5s}: {ms * 1e3:8.1f} us  {cfg.flops / ms / 1e9:6.2f} TFLOP/s", flush=True)
        print(f"BK={BK} FFMA2 bit-identical to FFMA: {np.array_equal(res['FFMA'], res['FFMA2'])}", flush=True)


if __name__ == "__main__":
    main()
