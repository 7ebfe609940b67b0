"""A/B of the mm k-tile staging (GPU box; measurement infrastructure, not
product):

    python tools/tmaab.py [mm|mm_rect]

The same DPIA program emitted twice -- B's k-tile staged by TMA tensor
copies (cuda/emit.py TMA_TILES, the default) and by register prefetch +
shared stores -- timed alternately (L2 scrub before each launch, CUDA events,
median of 30) and compared bit for bit.  Also prints the tensor-copy count
of each cubin's SASS when cuobjdump is on PATH.
"""
import os
import statistics
import subprocess
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import CONFIGS  # noqa: E402
from paper_1710_08332_b200.cuda import emit as EM  # noqa: E402


def sass_count(src: str, what: str) -> int:
    try:
        img = RT.get_cubin(src)
        with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
            f.write(img)
            f.flush()
            out = subprocess.run(["cuobjdump", "-sass", f.name], capture_output=True, text=True).stdout
        return out.count(what)
    except Exception:  # noqa: BLE001
        return -1


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "mm"
    RT.init(0)
    st = RT.Stream(0)
    cfg = CONFIGS[which]()
    rng = np.random.default_rng(5)
    A = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    B = rng.uniform(-1, 1, (4096, 4096)).astype(np.float32)
    exes = {}
    for tma in (True, False):
        EM.TMA_TILES = tma
        exe = executable(compile_program(cfg.text, name=which), cfg.launch, cfg.sigma, float_mode=True)
        exe.upload("A", A, st)
        exe.upload("B", B, st)
        exes[tma] = exe
        print(f"tma={tma}: tensor maps {list(exe.sig.tmaps.values())}; SASS UTMALDG "
              f"{sass_count(exe.src, 'UTMALDG')}, FFMA2 {sass_count(exe.src, 'FFMA2')}", flush=True)
    ts = {True: [], False: []}
    for it in range(35):
        for tma in (True, False):
            RT.lib().dpia_l2_flush(0, st.handle)
            e0, e1 = RT.Event(0), RT.Event(0)
            e0.record(st)
            exes[tma].launch(st)
            e1.record(st)
            st.sync()
            if it >= 5:
                ts[tma].append(e0.elapsed_ms(e1))
    outs = {tma: exes[tma].download("out", st) for tma in (True, False)}
    st.sync()
    for tma in (True, False):
        ms = statistics.median(ts[tma])
        print(f"{which} tma={tma}: {ms * 1e3:8.1f} us  {cfg.flops / ms / 1e9:6.2f} TFLOP/s", flush=True)
    print("bit-identical:", np.array_equal(np.asarray(outs[True]).view(np.uint32),
                                           np.asarray(outs[False]).view(np.uint32)))
    ref = A[:64].astype(np.float64) @ B.astype(np.float64)
    got = np.asarray(outs[True]).reshape(4096, 4096)[:64]
    bound = 1e-4 * (np.abs(A[:64]).astype(np.float64) @ np.abs(B).astype(np.float64))
    print("rows 0-63 within 1e-4 * sum|terms|:", bool(np.all(np.abs(got - ref) <= bound)))


if __name__ == "__main__":
    main()
