"""Launch geometry and pipelining depth of the reference-language reduction
programs (asum_proxy, dot_literal) in the bench's steady state (GPU box;
measurement infrastructure, not product).

    python tools/proxysweep.py

bench.Rotation: 20 chained steps over rotating input copies (> 3 x L2)
between one event pair, after 5 warm-up steps.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import asum_proxy_config, dot_literal_config  # noqa: E402
from paper_1710_08332_b200.cuda import emit as EM  # noqa: E402


def steady(cfg, inputs, st):
    exe = executable(compile_program(cfg.text, name=cfg.name), cfg.launch, cfg.sigma, float_mode=True)
    for n, v in inputs.items():
        exe.upload(n, v, st)
    rot = bench.Rotation(exe, cfg.bytes, st, chain=True)
    rot.run(st, 5)
    ms = rot.run(st, 20, start=5)
    rot.free()
    return ms, exe


def main():
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(2)
    xs = rng.uniform(-1, 1, 1 << 26).astype(np.float32)
    ys = rng.uniform(-1, 1, 1 << 24).astype(np.float32)
    for K in (4, 16):
        EM.STREAM_PIPE_SLOTS = K
        for L, rounds in ((32, 4), (32, 2), (32, 8), (64, 4), (64, 2), (128, 4)):
            for name, mk, inp in (("asum_proxy", asum_proxy_config, {"xs": xs}),
                                  ("dot_literal", dot_literal_config, {"xs": xs[:1 << 24], "ys": ys})):
                if name == "dot_literal" and K == 16:
                    continue
                cfg = mk(L=L, rounds=rounds)
                ms, exe = steady(cfg, inp, st)
                k = exe.sig.kernels[0]
                print(f"{name:12s} K>={K:2d} L={L:3d} rounds={rounds}: launch {cfg.launch}  {ms * 1e3:7.2f} us "
                      f"{cfg.bytes / ms / 1e6:7.1f} GB/s  slots={k.counter_words // (-(-cfg.sigma['n'] // (cfg.launch[0] * L)) + 1)}",
                      flush=True)


if __name__ == "__main__":
    main()
