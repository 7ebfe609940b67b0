"""mm 4096^3 strategy variants with the current emitter (GPU box;
measurement infrastructure, not product).

    python tools/mmsweep.py

Each variant: L2 scrub before each launch, CUDA events, median of 20, and the
result compared bit for bit with the bench's mm program (same fold order per
output element for every variant, so all must agree).
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import mm_config, mm_rect_config  # noqa: E402


def main():
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(5)
    A = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    B = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    variants = [("mm T128 BK16 R8 (bench)", mm_config(), {}),
                ("mm T128 BK8 R8", mm_config(BK=8), {}),
                ("mm T128 BK32 R8", mm_config(BK=32), {}),
                ("mm rows-A BK16", mm_config(a_by_rows=True), {}),
                ("mm sectors-A BK16", mm_config(a_sectors=True), {}),
                ("rect 128x128 BK8 R16x8", mm_rect_config(BK=8, RM=16, RN=8), {}),
                ("rect 128x128 BK16 R16x8", mm_rect_config(BK=16, RM=16, RN=8), {}),
                ("rect 128x128 BK8 R8x16", mm_rect_config(BK=8, RM=8, RN=16), {}),
                ("mm T128 BK16 R8 tma", mm_config(), {"tma_tiles": True})]
    ref = None
    for name, cfg, opts in variants:
        try:
            exe = executable(compile_program(cfg.text, name="mm"), cfg.launch, cfg.sigma, float_mode=True, **opts)
        except Exception as e:  # noqa: BLE001
            print(f"{name:28s}: not emitted ({type(e).__name__}: {str(e)[:80]})", flush=True)
            continue
        exe.upload("A", A, st)
        exe.upload("B", B, st)
        ts = []
        for it in range(25):
            RT.lib().dpia_l2_flush(0, st.handle)
            e0, e1 = RT.Event(0), RT.Event(0)
            e0.record(st)
            exe.launch(st)
            e1.record(st)
            st.sync()
            if it >= 5:
                ts.append(e0.elapsed_ms(e1))
        out = np.asarray(exe.download("out", st))
        st.sync()
        ref = out if ref is None else ref
        ms = statistics.median(ts)
        print(f"{name:28s}: {ms * 1e3:8.1f} us  {cfg.flops / ms / 1e9:6.2f} TFLOP/s  "
              f"{'==' if np.array_equal(out.view(np.uint32), ref.view(np.uint32)) else '!='} bench mm",
              flush=True)


if __name__ == "__main__":
    main()
