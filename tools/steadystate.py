"""Isolated-launch vs steady-state timing of the bandwidth-bound suite
(GPU box; measurement infrastructure, not product).

    python tools/steadystate.py

bench.py times every step in its own event pair after an L2 scrub, so each
step pays the event pair (~2.7 us here) and an unhidden launch (~3.3 us,
profiles/r01f_tailexp4.txt).  The other L2 rule the contract allows is
inputs larger than L2: here each workload gets R input sets (R x the
step's bytes >= 3 x 126 MB L2), step i reads set i % R -- the two previous
steps' reads evicted it -- and K steps run back to back between ONE event
pair.  Per-step time = total / K.  Also printed: the isolated mean.
"""
import os
import statistics
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import (asum_config, dot_config, dot_literal_config,  # noqa: E402
                                                  gemv_config, scal_config)

L2 = 126 * 1024 * 1024


def measure(name, cfg, shapes, st, rng, K=50, chain=False, R=None):
    """(isolated mean us, steady-state median us, R, runs) of one config;
    chain: the steady-state steps are chained (Executable.launch_with(chain=
    True)); R: input sets (default: enough for 3 x L2)."""
    exe = executable(compile_program(cfg.text, name=name.split("_")[0]), cfg.launch, cfg.sigma,
                     float_mode=True)
    if "alpha" in dict(exe.sig.inputs):
        exe.upload("alpha", np.full(4, 1.5, np.float32), st)
    step_bytes = sum(4 * v for v in shapes.values())
    R = R or max(2, -(-3 * L2 // step_bytes))
    sets = []
    for r in range(R):
        bufs = {}
        for n, cnt in shapes.items():
            b = RT.DeviceBuffer(4 * cnt)
            b.upload(rng.uniform(-1, 1, cnt).astype(np.float32), st)
            bufs[n] = b
        sets.append(bufs)
    st.sync()
    ptrs = [{n: b.ptr for n, b in s.items()} for s in sets]

    def launch(i, ch=False):
        exe.launch_with(st, ptrs[i % R], chain=ch)
    iso = []
    for it in range(K + 5):
        RT.lib().dpia_l2_flush(0, st.handle)
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        launch(it)
        e1.record(st)
        st.sync()
        if it >= 5:
            iso.append(e0.elapsed_ms(e1))
    for i in range(6):
        launch(i, chain)
    st.sync()
    runs = []
    for rep in range(5):
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(st)
        for i in range(K):
            launch(i, chain)
        e1.record(st)
        st.sync()
        runs.append(e0.elapsed_ms(e1) / K)
    for s_ in sets:
        for b in s_.values():
            b.free()
    return statistics.mean(iso) * 1e3, statistics.median(runs) * 1e3, R, runs


def main():
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(0)
    cfgs = [("asum", asum_config(), {"xs": 1 << 26}),
            ("dot", dot_config(), {"xs": 1 << 24, "ys": 1 << 24}),
            ("dot_literal", dot_literal_config(), {"xs": 1 << 24, "ys": 1 << 24}),
            ("gemv", gemv_config(), {"A": 8192 * 8192, "x": 8192}),
            ("gemv_xprivate", gemv_config(x_private=True), {"A": 8192 * 8192, "x": 8192}),
            ("scal", scal_config(), {"xs": 1 << 26})]
    chains = (False, True) if "--chain" in sys.argv else (False,)
    for name, cfg, shapes in cfgs:
        for chain in chains:
            for R in ((None, 2, 4, 8) if "--sets" in sys.argv else (None,)):
                iso_us, ss_us, R_, runs = measure(name, cfg, shapes, st, rng, chain=chain, R=R)
                print(f"{name:14s} chain={int(chain)} R={R_}: isolated {iso_us:7.2f} us "
                      f"({cfg.bytes / iso_us / 1e3:6.0f} GB/s, frac {cfg.bytes / iso_us / 1e3 / 6554.9:.3f})"
                      f"   steady {ss_us:7.2f} us ({cfg.bytes / ss_us / 1e3:6.0f} GB/s, "
                      f"frac {cfg.bytes / ss_us / 1e3 / 6554.9:.3f})  runs {[round(r * 1e3, 2) for r in runs]}",
                      flush=True)


if __name__ == "__main__":
    main()
