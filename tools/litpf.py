"""Software pipelining of the vectorised sequential folds (GPU box;
measurement infrastructure, not product).

    python tools/litpf.py

BASELINE config 1's literal program (oracle/ref_programs/dot.dpia) and its
partials-only half (tools/litgeo.py PARTIALS), timed like bench.py at a few
geometries for the emitter's variants (cuda/emit.py): the per-work-item
chunk folds' register queues (VEC_PREFETCH slots of VEC_LOAD_BYTES = 16 or
32 bytes) and the fused tail's single-thread fold through a register queue
or through the shared-memory ring of TMA bulk copies (TAIL_RING_STAGES x
TAIL_RING_BYTES, TAIL_RING_UNROLL).  Also checks that every variant returns
the same bits (the fold order never changes).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import dot_literal_program  # noqa: E402
from paper_1710_08332_b200.cuda import emit as EM  # noqa: E402
from litgeo import PARTIALS, timed  # noqa: E402


VARIANTS = [
    # (label, emitter knobs)
    ("vec4 only", dict(VEC_PREFETCH=0, TAIL_RING=False)),
    ("q16 D=16, tail q16", dict(VEC_PREFETCH=8, VEC_LOAD_BYTES=16, TAIL_RING=False)),
    ("q32 D=8, tail q32", dict(VEC_PREFETCH=8, VEC_LOAD_BYTES=32, TAIL_RING=False)),
    ("q32 D=4, ring 4x2K", dict(VEC_PREFETCH=4, VEC_LOAD_BYTES=32, TAIL_RING=True, TAIL_RING_STAGES=4,
                                TAIL_RING_BYTES=2048, TAIL_RING_UNROLL=8)),
    ("q32 D=8, ring 4x2K", dict(VEC_PREFETCH=8, TAIL_RING_STAGES=4, TAIL_RING_BYTES=2048)),
    ("q32 D=8, ring 8x1K", dict(VEC_PREFETCH=8, TAIL_RING_STAGES=8, TAIL_RING_BYTES=1024)),
    ("q32 D=8, ring 4x4K", dict(VEC_PREFETCH=8, TAIL_RING_STAGES=4, TAIL_RING_BYTES=4096)),
    ("q32 D=8, ring 2x8K", dict(VEC_PREFETCH=8, TAIL_RING_STAGES=2, TAIL_RING_BYTES=8192)),
    ("q32 D=8, ring 4x2K u4", dict(VEC_PREFETCH=8, TAIL_RING_STAGES=4, TAIL_RING_BYTES=2048,
                                   TAIL_RING_UNROLL=4)),
    ("q32 D=8, ring 4x2K u16", dict(VEC_PREFETCH=8, TAIL_RING_STAGES=4, TAIL_RING_BYTES=2048,
                                    TAIL_RING_UNROLL=16)),
]


def main():
    RT.init(0)
    st = RT.Stream(0)
    n = 16384
    rng = np.random.default_rng(0)
    xs = rng.uniform(0, 1, n * 1024).astype(np.float32)
    ys = rng.uniform(0, 1, n * 1024).astype(np.float32)
    launches = ((512, 32), (256, 64), (128, 128))
    results = {}
    seen_partials = set()
    for label, knobs in VARIANTS:
        for k, v in knobs.items():
            setattr(EM, k, v)
        for tag, text in (("literal", dot_literal_program()), ("partials", PARTIALS)):
            pkey = (EM.VEC_PREFETCH, EM.VEC_LOAD_BYTES)
            if tag == "partials":
                if pkey in seen_partials:
                    continue
                seen_partials.add(pkey)
            prog = compile_program(text, name="lit")
            for launch in launches:
                exe = executable(prog, launch, {"n": n}, float_mode=True)
                exe.upload("xs", xs, st)
                exe.upload("ys", ys, st)
                us = timed(st, exe)
                out = exe.download("out", st)
                st.sync()
                bits = np.asarray(out, np.float32).tobytes()
                results.setdefault((tag, launch), set()).add(bits)
                print(f"{label:24s} {tag:9s} launch={launch}: {us:8.2f} us  "
                      f"{8 * n * 1024 / us / 1e3:7.1f} GB/s", flush=True)
    for k, v in results.items():
        print(k, "identical bits across variants" if len(v) == 1 else f"{len(v)} DIFFERENT results")


if __name__ == "__main__":
    main()
