"""GPU: chained launches (Executable.launch(chain=True), programmatic
dependent launch of a program's first kernel behind the previous launch on
the stream).  Every step gets its own input and output buffers (launch_with)
and runs chained behind the previous step, so a step that touched shared
state early -- the fused tail's counter, the scratch partials, another
step's output -- would corrupt some step's result.  Each step must return
the bits of an ordinary (unchained) launch on the same inputs."""
import numpy as np
import pytest

from paper_1710_08332_b200 import compile_program, executable
from paper_1710_08332_b200 import runtime as RT
from paper_1710_08332_b200.bench_programs import (asum_config, dot_config, dot_literal_config,
                                                  gemv_config, mm_config, scal_config,
                                                  scal_literal_config)

pytestmark = pytest.mark.gpu

TWO_PHASE = ("(nat n)\n(param xs (exp (array n num)))\n"
             "(mapGlobal (lam x (+ x 1)) (toGlobal (lam t t) (mapGlobal (lam y (* y 2)) xs)))")


def _cases():
    return [
        ("dot", dot_config(N=1 << 20), {"xs": 1 << 20, "ys": 1 << 20}),
        ("asum", asum_config(N=1 << 20), {"xs": 1 << 20}),
        ("dot_literal", dot_literal_config(N=1 << 20), {"xs": 1 << 20, "ys": 1 << 20}),
        ("gemv", gemv_config(M=512, N=1024), {"A": 512 * 1024, "x": 1024}),
        ("gemv_xprivate", gemv_config(M=512, N=1024, x_private=True), {"A": 512 * 1024, "x": 1024}),
        ("scal", scal_config(N=1 << 20), {"xs": 1 << 20}),
        ("scal_literal", scal_literal_config(N=1 << 22), {"xs": 1 << 22}),
        ("mm", mm_config(M=256, N=256, K=256), {"A": 256 * 256, "B": 256 * 256}),
    ]


def _run_chained(exe, shapes, steps, rng, fm=True):
    st = RT.Stream(0)
    outs = [n for n, _ in exe.sig.outputs]
    sets = []
    for _ in range(steps):
        bufs = {}
        for n, cnt in shapes.items():
            host = rng.uniform(-1, 1, cnt).astype(np.float32) if fm else \
                rng.integers(-50, 50, cnt).astype(np.int64)
            b = RT.DeviceBuffer(host.nbytes)
            b.upload(host, st)
            bufs[n] = (b, host)
        for n in outs:
            b = RT.DeviceBuffer(exe.buffers[n].nbytes)
            b.zero(st)
            bufs[n] = (b, None)
        sets.append(bufs)
    st.sync()
    for i, bufs in enumerate(sets):
        exe.launch_with(st, {n: b.ptr for n, (b, _) in bufs.items()}, chain=i > 0)
    st.sync()
    results = []
    for bufs in sets:
        got = {}
        for n in outs:
            raw = np.empty(exe.buffers[n].nbytes, np.uint8)
            bufs[n][0].download(raw, st)
            got[n] = raw
        st.sync()
        results.append(got)
    # the same inputs through ordinary launches of the executable's own buffers
    for bufs, got in zip(sets, results):
        for n, (b, host) in bufs.items():
            if host is not None:
                exe.buffers[n].upload(host.view(np.uint8), st)
        exe.launch(st)
        st.sync()
        for n in outs:
            raw = np.empty(exe.buffers[n].nbytes, np.uint8)
            exe.buffers[n].download(raw, st)
            st.sync()
            assert np.array_equal(raw, got[n]), n
    for bufs in sets:
        for b, _ in bufs.values():
            b.free()


@pytest.mark.parametrize("name,cfg,shapes", _cases(), ids=[c[0] for c in _cases()])
def test_chained_steps_match_unchained_launches(name, cfg, shapes):
    exe = executable(compile_program(cfg.text, name=name.split("_")[0]), cfg.launch, cfg.sigma,
                     float_mode=True)
    if "alpha" in dict(exe.sig.inputs):
        shapes = dict(shapes, alpha=4 if name == "scal" else 1)
    _run_chained(exe, shapes, 12, np.random.default_rng(7))


@pytest.mark.parametrize("fm", [True, False])
def test_chained_two_phase_program(fm):
    exe = executable(compile_program(TWO_PHASE), (148, 256), {"n": 1 << 18}, float_mode=fm)
    assert len(exe.sig.kernels) == 2
    _run_chained(exe, {"xs": 1 << 18}, 10, np.random.default_rng(3), fm=fm)


def test_chained_int_mode_reductions():
    for cfg in (dot_literal_config(N=1 << 18), dot_config(N=1 << 20)):
        exe = executable(compile_program(cfg.text), cfg.launch, cfg.sigma, float_mode=False)
        _run_chained(exe, {"xs": cfg.bytes // 8, "ys": cfg.bytes // 8}, 8, np.random.default_rng(5),
                     fm=False)
