"""Does a programmatic dependent launch of a program's first kernel, right
after the L2 scrub kernel and a CUDA event, change its event-timed duration?
(GPU box; measurement infrastructure only.)

    python tools/pdlfirst.py
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import asum_config, dot_config  # noqa: E402


def main():
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(0)
    for cfg, inputs in ((asum_config(), {"xs": rng.uniform(-1, 1, 1 << 26).astype(np.float32)}),
                        (dot_config(), {"xs": rng.uniform(0, 1, 1 << 24).astype(np.float32),
                                        "ys": rng.uniform(0, 1, 1 << 24).astype(np.float32)})):
        exe = executable(compile_program(cfg.text, name=cfg.name), cfg.launch, cfg.sigma, float_mode=True)
        for n, v in inputs.items():
            exe.upload(n, v, st)
        (g, l) = exe.sig.launch
        k = exe.sig.kernels[0]
        fn = exe.module.function(k.name)
        for rnd in range(2):
            for pdl in (False, True):
                ts = []
                for i in range(65):
                    RT.lib().dpia_l2_flush(0, st.handle)
                    e0, e1 = RT.Event(0), RT.Event(0)
                    e0.record(st)
                    RT.launch(fn, 0, g, l, k.smem, exe._args[0], st, pdl=pdl)
                    e1.record(st)
                    st.sync()
                    if i >= 5:
                        ts.append(e0.elapsed_ms(e1))
                t = statistics.mean(ts) * 1e3
                print(f"round {rnd} {cfg.name} pdl={pdl}: {t:7.2f} us  {cfg.bytes / t / 1e3:7.1f} GB/s",
                      flush=True)


if __name__ == "__main__":
    main()
