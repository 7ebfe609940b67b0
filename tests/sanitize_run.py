"""Workload for compute-sanitizer (GPU box; tests/test_sanitizer.py runs it
under --tool memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck --error-exitcode 1 python tests/sanitize_run.py

Runs every benchmark strategy at a reduced size, the reference's golden
programs and a sample of the hierarchical strategy fuzzer (tests/strategy_gen)
through the public API and checks each result against the oracle, so a run
that the sanitizer passes is also a correct one.  racecheck is the hardware
check of the emitter's barrier plan (shared-memory RAW/WAR/WAW hazards);
memcheck covers out-of-bounds and misaligned accesses (float4 views, 64-bit
indices); synccheck covers barrier divergence (fused grid tails).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.dpia_eval import eval_phrase, flatten_value, from_json  # noqa: E402
from paper_1710_08332_b200 import CudaError, compile_program, run_program_cuda  # noqa: E402
from paper_1710_08332_b200.bench_programs import (asum_config, dot_config, gemv_config,  # noqa: E402
                                                  mm_config, scal_config)


def ints(shape, seed):
    return np.random.default_rng(seed).integers(-9, 10, shape)


def check(prog, inputs, sigma, launch, label):
    got = run_program_cuda(prog, inputs, sigma=sigma, launch=launch, float_mode=False, flat=True)
    want = flatten_value(eval_phrase(prog.source.body, {k: (v.tolist() if hasattr(v, "tolist") else v)
                                                        for k, v in inputs.items()}, sigma))
    assert [int(v) for v in got] == [int(v) for v in want], label
    print(f"ok {label}", flush=True)


def broken():
    """Negative control: the mm kernel with every __syncthreads removed from
    its body must make racecheck report shared-memory hazards."""
    from paper_1710_08332_b200 import runtime as RT
    from paper_1710_08332_b200.cuda.emit import emit_cuda
    from paper_1710_08332_b200.launcher import Executable
    c = mm_config(M=128, N=128, K=128, T=128, BK=16, R=8)
    prog = compile_program(c.text)
    outs = [(n, t) for n, t, k in prog.params if k == "out"]
    ins = [(n, t) for n, t, k in prog.params if k == "in"]
    src, sig = emit_cuda(prog.imperative, outs, ins, False, "mm", sigma=c.sigma, launch=c.launch)
    k = src.index('extern "C"')
    src = src[:k] + src[k:].replace("__syncthreads();", "")
    exe = Executable(src, sig, 0, False, dict(c.sigma), geometry=c.launch).compile().allocate()
    st = RT.Stream(0)
    exe.upload("A", ints((128, 128), 1), st)
    exe.upload("B", ints((128, 128), 2), st)
    exe.launch(st)
    st.sync()
    print("BROKEN WORKLOAD DONE", flush=True)


def main():
    if "--broken" in sys.argv:
        broken()
        return
    n_fuzz = int(os.environ.get("DPIA_SANITIZE_FUZZ", "12"))
    # benchmark strategies, reduced sizes (int mode: exact)
    c = dot_config(N=1 << 14, L=128, K=4)
    check(compile_program(c.text), {"xs": ints(1 << 14, 1), "ys": ints(1 << 14, 2)}, c.sigma,
          (c.sigma["n"], 128), "dot")
    c = asum_config(N=1 << 14, L=128, K=4)
    check(compile_program(c.text), {"xs": ints(1 << 14, 3)}, c.sigma, (c.sigma["n"] - 1, 128), "asum")
    c = gemv_config(M=24, N=1024, L=128, blocks=7)
    check(compile_program(c.text), {"A": ints((24, 1024), 4), "x": ints(1024, 5)}, c.sigma, c.launch,
          "gemv")
    for BK in (8, 16):
        c = mm_config(M=256, N=128, K=256, T=128, BK=BK, R=8)
        prog = compile_program(c.text)
        A, B = ints((256, 256), 6), ints((256, 128), 7)
        got = run_program_cuda(prog, {"A": A, "B": B}, launch=c.launch, float_mode=False, flat=True)
        assert np.array_equal(np.asarray(got, np.int64).reshape(256, 128), A @ B), "mm"
        print(f"ok mm BK={BK}", flush=True)
    # fp32 mm (the FFMA2 path) against numpy
    c = mm_config(M=128, N=128, K=128, T=128, BK=16, R=8)
    A = np.random.default_rng(8).uniform(-1, 1, (128, 128)).astype(np.float32)
    B = np.random.default_rng(9).uniform(-1, 1, (128, 128)).astype(np.float32)
    got = np.asarray(run_program_cuda(compile_program(c.text), {"A": A, "B": B}, launch=c.launch,
                                      flat=True)).reshape(128, 128)
    assert np.allclose(got, A.astype(np.float64) @ B, atol=1e-4), "mm fp32"
    print("ok mm fp32", flush=True)
    c = scal_config(N=1 << 12, L=64, blocks=5)
    xs = ints(1 << 12, 10)
    got = run_program_cuda(compile_program(c.text), {"alpha": [3, 3, 3, 3], "xs": xs}, sigma=c.sigma,
                           launch=c.launch, float_mode=False, flat=True)
    assert [int(v) for v in got] == (3 * xs).tolist()
    print("ok scal", flush=True)
    # fused peer combine, one rank (mailbox protocol under the sanitizer)
    from paper_1710_08332_b200 import runtime as RT
    from paper_1710_08332_b200.scaleout import ShardedReduction
    for kind in ("asum", "dot"):
        run = ShardedReduction(kind, 1 << 18, L=128, K=4, combine="peer")
        st = RT.Stream(0)
        run.fill_inputs(st)
        vals = []
        for _ in range(3):
            run.launch(st, allreduce=True)
            st.sync()
            vals.append(run.result())
        run.peer.check()
        assert vals[0] == vals[1] == vals[2], vals
        run.peer.close()
        print(f"ok peer {kind}", flush=True)
    # TMA row folds + a parity-pipelined streaming tail (fp32: the row boxes
    # are 16-byte vectors), several launches chained; TMA k-tiles (mm, int)
    from paper_1710_08332_b200 import executable
    from paper_1710_08332_b200.bench_programs import dot_literal_config
    c = dot_literal_config(N=1 << 18)
    exe = executable(compile_program(c.text), c.launch, c.sigma, float_mode=True)
    assert exe.sig.kernels[0].extra_blocks == 1 and exe.sig.tmaps, "streaming tail + row boxes"
    rng = np.random.default_rng(12)
    xs = rng.uniform(0, 1, 1 << 18).astype(np.float32)
    ys = rng.uniform(0, 1, 1 << 18).astype(np.float32)
    st = RT.Stream(0)
    exe.upload("xs", xs, st)
    exe.upload("ys", ys, st)
    for k in range(4):
        exe.launch(st, chain=k > 0)
    got = float(np.asarray(exe.download("out", st))[0])
    st.sync()
    want = float(np.dot(xs.astype(np.float64), ys.astype(np.float64)))
    assert abs(got - want) <= 1e-4 * want, (got, want)
    print("ok dot_literal streaming tail + TMA row folds", flush=True)
    from paper_1710_08332_b200.bench_programs import scal_literal_config
    c = scal_literal_config(N=1 << 20)
    exe = executable(compile_program(c.text), c.launch, c.sigma, float_mode=True)
    xs = rng.uniform(-1, 1, 1 << 20).astype(np.float32)
    exe.upload("alpha", np.float32([1.5]), st)
    exe.upload("xs", xs, st)
    for k in range(3):
        exe.launch(st, chain=k > 0)
    got = np.asarray(exe.download("out", st))
    st.sync()
    assert np.array_equal(got, np.float32(1.5) * xs), "scal_literal"
    print("ok scal_literal TMA row reads + row stores", flush=True)
    c = mm_config(M=256, N=128, K=256, T=128, BK=16, R=8)
    exe = executable(compile_program(c.text), c.launch, {}, float_mode=False, tma_tiles=True)
    assert exe.sig.tmaps, "TMA k-tiles"
    A, B = ints((256, 256), 13), ints((256, 128), 14)
    exe.upload("A", A, st)
    exe.upload("B", B, st)
    exe.launch(st)
    got = np.asarray(exe.download("out", st))
    st.sync()
    assert np.array_equal(got.astype(np.int64).reshape(256, 128), A @ B), "mm tma"
    print("ok mm TMA k-tiles", flush=True)
    # the reference's golden programs
    from conftest import load_golden
    for case in load_golden("programs.json"):
        if case.get("float"):
            continue
        prog = compile_program(case["text"])
        inputs = {k: from_json(v) for k, v in case["inputs"].items()}
        for launch in ((2, 4), (3, 32)):
            got = run_program_cuda(prog, inputs, sigma=case.get("sigma", {}), launch=launch,
                                   float_mode=False, flat=True)
            want = flatten_value(from_json(case["expected"]))
            if any(abs(v) >= 2 ** 63 for v in want):
                continue
            assert [int(v) for v in got] == want, case["name"]
        print(f"ok golden {case['name']}", flush=True)
    # hierarchical strategy fuzzer sample
    from strategy_gen import generate
    for seed in range(n_fuzz):
        text, inputs, sigma, launch, desc = generate(seed)
        try:
            check(compile_program(text), inputs, sigma, launch, f"fuzz {seed} ({desc})")
        except CudaError as e:
            print(f"skip fuzz {seed}: {e}", flush=True)
    from strategy_gen import generate2d
    for seed in range(16):
        text, inputs, sigma, launch, desc = generate2d(seed)
        check(compile_program(text), inputs, sigma, launch, f"fuzz2d {seed} ({desc})")
    print("SANITIZE WORKLOAD DONE", flush=True)


if __name__ == "__main__":
    main()
