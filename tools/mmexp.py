"""mm strategy/occupancy sweep (GPU box).

    python tools/mmexp.py

For each (T, BK, R) strategy parameterisation of bench_programs.mm_program,
times the emitted kernel like bench.py (L2 scrubbed, events, mean of 10) at
its natural occupancy and with the dynamic shared-memory request padded so
that only one CTA fits per SM (which changes 1024 tiles from 3.46 waves over
296 resident CTAs to 6.92 waves over 148).  Measurement infrastructure only.
"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import mm_config, mm_rect_config, mm_rowa_config  # noqa: E402


def run(cfg, inputs, st, pad_smem=None, reps=10):
    exe = executable(compile_program(cfg.text, name=cfg.name), cfg.launch, cfg.sigma, float_mode=True)
    if pad_smem:
        for k in exe.sig.kernels:
            k.smem = max(k.smem, pad_smem)
            RT.lib().dpia_kernel_set_smem(exe.module.function(k.name), k.smem)
    for n, v in inputs.items():
        exe.upload(n, v, st)
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
    out = np.zeros((4096, 4096), np.float32)
    exe.buffers["out"].download(out)
    return statistics.mean(ts), out


def main():
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    B = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    ref = (A[:64].astype(np.float64) @ B.astype(np.float64))
    inputs = {"A": A, "B": B}
    grid = [(128, 16, 8, "quads"), (128, 16, 8, "sectors"), (128, 32, 8, "sectors"),
            (128, 8, 8, "quads")]
    for T, BK, R, rows in grid:
        cfg = mm_config(T=T, BK=BK, R=R, a_by_rows=rows == "rows", a_sectors=rows == "sectors")
        for pad in (None,):
            try:
                ms, out = run(cfg, inputs, st, pad)
            except Exception as e:  # noqa: BLE001
                print(f"T={T} BK={BK} R={R} a_layout={rows} pad={pad}: {type(e).__name__} {str(e)[:300]}", flush=True)
                continue
            err = float(np.max(np.abs(out[:64] - ref)))
            print(f"T={T} BK={BK} R={R} a_layout={rows} pad={pad}: {ms * 1e3:8.1f} us  {cfg.flops / ms / 1e9:6.2f} TFLOP/s  "
                  f"max|err| rows 0-63 = {err:.2e}", flush=True)


def rect():
    """Rectangular register tiles (bench_programs.mm_rect_program)."""
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    B = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    ref = (A[:64].astype(np.float64) @ B.astype(np.float64))
    for TM, TN, BK, RM, RN in ((128, 128, 16, 8, 16), (128, 128, 8, 8, 16), (128, 128, 16, 16, 8),
                               (128, 128, 8, 16, 8), (128, 64, 16, 8, 8), (256, 128, 8, 16, 16)):
        cfg = mm_rect_config(TM=TM, TN=TN, BK=BK, RM=RM, RN=RN)
        try:
            ms, out = run(cfg, {"A": A, "B": B}, st)
        except Exception as e:  # noqa: BLE001
            print(f"rect {TM}x{TN} BK={BK} R={RM}x{RN}: {type(e).__name__} {str(e)[:300]}", flush=True)
            continue
        err = float(np.max(np.abs(out[:64] - ref)))
        print(f"rect {TM}x{TN} BK={BK} R={RM}x{RN}: {ms * 1e3:8.1f} us  {cfg.flops / ms / 1e9:6.2f} TFLOP/s"
              f"  max|err| rows 0-63 = {err:.2e}", flush=True)


def waves():
    """In-wave efficiency: problems whose tile count fills exactly 1 or 2
    waves of 296 resident CTAs (2 per SM), next to 4096^2 (3.46 waves)."""
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(0)
    for M, N in ((4736, 1024), (4736, 2048), (4096, 4096)):
        A = rng.uniform(-1, 1, (M, 4096)).astype(np.float32)
        B = rng.uniform(-1, 1, (4096, N)).astype(np.float32)
        cfg = mm_config(M=M, N=N)
        exe = executable(compile_program(cfg.text, name=cfg.name), cfg.launch, cfg.sigma, float_mode=True)
        exe.upload("A", A, st)
        exe.upload("B", B, st)
        ts = []
        for i in range(13):
            RT.lib().dpia_l2_flush(0, st.handle)
            e0, e1 = RT.Event(0), RT.Event(0)
            e0.record(st)
            exe.launch(st)
            e1.record(st)
            st.sync()
            if i >= 3:
                ts.append(e0.elapsed_ms(e1))
        ms = statistics.mean(ts)
        tiles = (M // 128) * (N // 128)
        print(f"M={M} N={N} K=4096 ({tiles} tiles = {tiles / 296:.2f} waves): {ms * 1e3:8.1f} us  "
              f"{cfg.flops / ms / 1e9:6.2f} TFLOP/s", flush=True)


def one(variant):
    """Launch one variant once (for ncu): quads | sectors | rows | hack."""
    import re
    from paper_1710_08332_b200.cuda.emit import emit_cuda
    from paper_1710_08332_b200.launcher import Executable
    RT.init(0)
    st = RT.Stream(0)
    cfg = mm_config(a_by_rows=variant == "rows", a_sectors=variant == "sectors")
    prog = compile_program(cfg.text, name="mm")
    outs = [(n, t) for n, t, k in prog.params if k == "out"]
    ins = [(n, t) for n, t, k in prog.params if k == "in"]
    src, sig = emit_cuda(prog.imperative, outs, ins, True, "mm", sigma=cfg.sigma, launch=cfg.launch)
    if variant == "hack":
        cnt = [0]

        def rep(m):
            cnt[0] += 1
            return f"{m.group(1)}[2048 * (({m.group(2)}) % 2) + dpia_tid + {256 * (cnt[0] - 1)}] = pf"
        src = re.sub(r"(tmp\d+_\d+)\[2048 \* \(\((i_\d+_\d+)\) % 2\) \+ 512 \* [^\]]*\] = pf", rep, src)
    exe = Executable(src, sig, 0, True, {}, geometry=cfg.launch).compile().allocate()
    rng = np.random.default_rng(0)
    exe.upload("A", rng.uniform(-1, 1, (4096, 4096)).astype(np.float32), st)
    exe.upload("B", rng.uniform(-1, 1, (4096, 4096)).astype(np.float32), st)
    for _ in range(2):
        exe.launch(st)
    st.sync()


CP_ASYNC = r"""
__device__ __forceinline__ void cp_async16(float* smem, const float* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s), "l"(gmem) : "memory");
}
#define B_G(k, row) (64 * ((row) % 2) + 4096 * ((row) / 2) + 4 * (int)threadIdx.x + 65536 * (k) + 128 * (int)blockIdx.x)
#define B_S(k, row) ((((4 * (int)threadIdx.x) ^ (8 * ((row) / 8))) + 2048 * ((k) % 2) + 64 * ((row) % 2) + 128 * ((row) / 2)))
"""


def cpasync_source(src):
    """Hand edit of the default BK=16 kernel: the B tile is staged with
    cp.async (no registers, no STS) -- issue for k+1 after the barrier of
    iteration k, wait_all before the barrier of k+1.  Experiment only."""
    import re
    k = src.index('extern "C"')
    src = src[:k] + CP_ASYNC + src[k:]
    a = src.index("dpia::vec<float, 4> pf1_0;")
    b = src.index("float* tmp", a)
    src = src[:a] + ("cp_async16(tmp16_9 + B_S(0, (int)threadIdx.y), B + B_G(0, (int)threadIdx.y));\n"
                     "cp_async16(tmp16_9 + B_S(0, (int)threadIdx.y + 16), B + B_G(0, (int)threadIdx.y + 16));\n"
                     "asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n") + src[b:]
    m = re.search(r"for \(int (i_\d+_\d+) = 0; \1 < 256; \1 \+= 1\) \{", src)
    kv = m.group(1)
    body = m.end()
    c0 = src.index("dpia::vstore<float, 4>(tmp16_9", body)
    c0 = src.rindex("{", 0, src.rindex("{", 0, c0))          # the copy's outer block
    r0 = src.index("if (" + kv + " + 1 < 256) {", body)
    # end of the B refill block: the matching brace
    depth, j = 0, r0
    while True:
        if src[j] == "{":
            depth += 1
        elif src[j] == "}":
            depth -= 1
            if depth == 0:
                break
        j += 1
    src = src[:c0] + "asm volatile(\"cp.async.wait_all;\" ::: \"memory\");\n" + src[j + 1:]
    sync = src.index("__syncthreads();", src.index(kv, m.start() + 10))
    issue = (f"\nif ({kv} + 1 < 256) {{ cp_async16(tmp16_9 + B_S({kv} + 1, (int)threadIdx.y), "
             f"B + B_G({kv} + 1, (int)threadIdx.y)); cp_async16(tmp16_9 + B_S({kv} + 1, (int)threadIdx.y + 16), "
             f"B + B_G({kv} + 1, (int)threadIdx.y + 16)); asm volatile(\"cp.async.commit_group;\" ::: \"memory\"); }}\n")
    e = sync + len("__syncthreads();")
    return src[:e] + issue + src[e:]


def cpasync():
    from paper_1710_08332_b200.cuda.emit import emit_cuda
    from paper_1710_08332_b200.launcher import Executable
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    B = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    cfg = mm_config()
    prog = compile_program(cfg.text, name="mm")
    outs = [(n, t) for n, t, k in prog.params if k == "out"]
    ins = [(n, t) for n, t, k in prog.params if k == "in"]
    src, sig = emit_cuda(prog.imperative, outs, ins, True, "mm", sigma=cfg.sigma, launch=cfg.launch)
    ref = None
    cpa = cpasync_source(src)
    for label, s in (("emitted", src), ("cp.async B", cpa),
                     ("cp.async B + lb(256,2)", cpa.replace("__launch_bounds__(256)", "__launch_bounds__(256, 2)"))):
        exe = Executable(s, sig, 0, True, {}, geometry=cfg.launch).compile().allocate()
        exe.upload("A", A, st)
        exe.upload("B", B, st)
        ts = []
        for i in range(13):
            RT.lib().dpia_l2_flush(0, st.handle)
            e0, e1 = RT.Event(0), RT.Event(0)
            e0.record(st)
            exe.launch(st)
            e1.record(st)
            st.sync()
            if i >= 3:
                ts.append(e0.elapsed_ms(e1))
        out = exe.download("out", st)
        ref = out if ref is None else ref
        ms = statistics.mean(ts)
        print(f"{label}: {ms * 1e3:8.1f} us  {cfg.flops / ms / 1e9:6.2f} TFLOP/s  same={np.array_equal(out, ref)}",
              flush=True)


def rowa():
    """Row-major A staging + k-quad micro-kernel (mm_rowa_program), as
    emitted and with __launch_bounds__(256, 2)."""
    from paper_1710_08332_b200.cuda.emit import emit_cuda
    from paper_1710_08332_b200.launcher import Executable
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    B = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    ref = (A[:64].astype(np.float64) @ B.astype(np.float64))
    for BK in (16, 8):
        cfg = mm_rowa_config(BK=BK)
        prog = compile_program(cfg.text, name="mm")
        outs = [(n, t) for n, t, k in prog.params if k == "out"]
        ins = [(n, t) for n, t, k in prog.params if k == "in"]
        src, sig = emit_cuda(prog.imperative, outs, ins, True, "mm", sigma=cfg.sigma, launch=cfg.launch)
        for label, s in (("emitted", src), ("lb(256,2)", src.replace("__launch_bounds__(256)",
                                                                     "__launch_bounds__(256, 2)"))):
            exe = Executable(s, sig, 0, True, {}, geometry=cfg.launch).compile().allocate()
            exe.upload("A", A, st)
            exe.upload("B", B, st)
            ts = []
            for i in range(13):
                RT.lib().dpia_l2_flush(0, st.handle)
                e0, e1 = RT.Event(0), RT.Event(0)
                e0.record(st)
                exe.launch(st)
                e1.record(st)
                st.sync()
                if i >= 3:
                    ts.append(e0.elapsed_ms(e1))
            out = exe.download("out", st).reshape(4096, 4096)
            ms = statistics.mean(ts)
            print(f"rowa BK={BK} {label}: {ms * 1e3:8.1f} us  {cfg.flops / ms / 1e9:6.2f} TFLOP/s  "
                  f"max|err| = {float(np.max(np.abs(out[:64] - ref))):.2e}", flush=True)


def transforms():
    """Source-level experiments on the emitted default mm kernel (timing
    only): unroll2 = `#pragma unroll 2` on the k-tile loop (slice offsets of
    the rotated stagings become constants)."""
    import re
    from paper_1710_08332_b200.cuda.emit import emit_cuda
    from paper_1710_08332_b200.launcher import Executable
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    B = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    cfg = mm_config()
    prog = compile_program(cfg.text, name="mm")
    outs = [(n, t) for n, t, k in prog.params if k == "out"]
    ins = [(n, t) for n, t, k in prog.params if k == "in"]
    src, sig = emit_cuda(prog.imperative, outs, ins, True, "mm", sigma=cfg.sigma, launch=cfg.launch)
    k_loop = re.search(r"\n(\s*)for \(int (i_\d+_\d+) = 0; \2 < 256; \2 \+= 1\) \{", src)
    variants = {"emitted": src, "lb(256,1)": src.replace("__launch_bounds__(256)", "__launch_bounds__(256, 1)")}
    if k_loop:
        variants["unroll2"] = src[:k_loop.start()] + f"\n{k_loop.group(1)}#pragma unroll 2" + src[k_loop.start():]
        variants["unroll1"] = src[:k_loop.start()] + f"\n{k_loop.group(1)}#pragma unroll 1" + src[k_loop.start():]
    ref = None
    for label, s in variants.items():
        exe = Executable(s, sig, 0, True, {}, geometry=cfg.launch).compile().allocate()
        exe.upload("A", A, st)
        exe.upload("B", B, st)
        ts = []
        for i in range(13):
            RT.lib().dpia_l2_flush(0, st.handle)
            e0, e1 = RT.Event(0), RT.Event(0)
            e0.record(st)
            exe.launch(st)
            e1.record(st)
            st.sync()
            if i >= 3:
                ts.append(e0.elapsed_ms(e1))
        out = exe.download("out", st)
        ref = out if ref is None else ref
        ms = statistics.mean(ts)
        print(f"{label}: {ms * 1e3:8.1f} us  {cfg.flops / ms / 1e9:6.2f} TFLOP/s  same={np.array_equal(out, ref)}",
              flush=True)


def sts_bound():
    """Upper bound of what conflict-free transposed A stores would gain: the
    emitted BK=16 kernel with its A-tile store index replaced by a
    conflict-free (WRONG-result) one; timing only."""
    import re
    from paper_1710_08332_b200.cuda.emit import emit_cuda
    from paper_1710_08332_b200.launcher import Executable
    RT.init(0)
    st = RT.Stream(0)
    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    B = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    cfg = mm_config()
    prog = compile_program(cfg.text, name="mm")
    outs = [(n, t) for n, t, k in prog.params if k == "out"]
    ins = [(n, t) for n, t, k in prog.params if k == "in"]
    src, sig = emit_cuda(prog.imperative, outs, ins, True, "mm", sigma=cfg.sigma, launch=cfg.launch)
    cnt = [0]

    def rep(m):
        j = cnt[0]
        cnt[0] += 1
        return f"{m.group(1)}[2048 * (({m.group(2)}) % 2) + dpia_tid + {256 * j}] = pf"
    hacked = re.sub(r"(tmp\d+_\d+)\[2048 \* \(\((i_\d+_\d+)\) % 2\) \+ 512 \* [^\]]*\] = pf", rep, src)
    print("replaced", cnt[0], flush=True)
    for label, s in (("emitted", src), ("conflict-free A stores (wrong result)", hacked)):
        exe = Executable(s, sig, 0, True, {}, geometry=cfg.launch).compile().allocate()
        exe.upload("A", A, st)
        exe.upload("B", B, st)
        ts = []
        for i in range(13):
            RT.lib().dpia_l2_flush(0, st.handle)
            e0, e1 = RT.Event(0), RT.Event(0)
            e0.record(st)
            exe.launch(st)
            e1.record(st)
            st.sync()
            if i >= 3:
                ts.append(e0.elapsed_ms(e1))
        ms = statistics.mean(ts)
        print(f"{label}: {ms * 1e3:8.1f} us  {cfg.flops / ms / 1e9:6.2f} TFLOP/s", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "cpasync":
        cpasync()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "rowa":
        rowa()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "xform":
        transforms()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "rect":
        rect()
        sys.exit(0)
    if len(sys.argv) > 2 and sys.argv[1] == "one":
        one(sys.argv[2])
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "sts":
        sts_bound()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "waves":
        waves()
        sys.exit(0)
    main()
