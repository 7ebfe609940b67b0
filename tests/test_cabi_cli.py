"""CPU-side checks of the native boundary and the CLI:
* libdpia_rt.so loads without a GPU driver and exports every entry point
  declared in include/dpia_rt.h;
* NVRTC (in-process, no GPU needed) compiles emitted kernels for sm_100a;
* the CLI follows the reference's exit codes (TST/test_cli.py:95-117)."""
import os
import re
import subprocess
import sys

import pytest

from conftest import ROOT
from paper_1710_08332_b200 import runtime as RT
from paper_1710_08332_b200.cli import main

HEADER = os.path.join(ROOT, "include", "dpia_rt.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dpia_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared() == sorted(RT.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = RT.lib()
    for name in declared():
        assert hasattr(lib.so, name), name
    out = subprocess.run(["nm", "-D", RT.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (dpia_\w+)", out))
    assert set(declared()) <= exported


def test_no_driver_needed_to_load_and_errors_are_reported():
    lib = RT.lib()
    assert lib.so.dpia_last_error() is not None
    if not os.path.exists("/dev/nvidia0"):
        n = RT.C.c_int()
        rc = lib.so.dpia_device_count(RT.C.byref(n))
        assert rc != 0 and b"driver" in lib.so.dpia_last_error().lower() or rc == 0


def test_nvrtc_compiles_emitted_benchmarks():
    from paper_1710_08332_b200.bench_programs import aot_sources
    for tag, src in aot_sources():
        img = RT.nvrtc_compile(src)
        assert img[:4] == b"\x7fELF", tag   # an sm_100a cubin


def test_nvrtc_reports_compile_errors():
    with pytest.raises(RT.DpiaRuntimeError) as ei:
        RT.nvrtc_compile('extern "C" __global__ void k() { this is not cuda; }')
    assert "error" in str(ei.value).lower()


def _prog(tmp_path, text, name="p.dpia"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_cli_compile_cuda(tmp_path):
    src = open(os.path.join(ROOT, "tests", "golden", "dotvec.dpia")).read() \
        if os.path.exists(os.path.join(ROOT, "tests", "golden", "dotvec.dpia")) else None
    if src is None:
        from conftest import load_golden
        src = [c for c in load_golden("programs.json") if c["name"] == "dotvec.dpia"][0]["text"]
    f = _prog(tmp_path, src, "dotvec.dpia")
    assert main(["compile", f, "--target", "cuda", "--launch", "2,4"]) == 0
    text = open(str(tmp_path / "dotvec.cu")).read()
    for needle in ("__global__", "blockIdx.x", "threadIdx.x", "dpia::vload<float, 4>",
                   "dpia::vec<float, 4>"):
        assert needle in text, needle


def test_cli_compile_tma_tiles(tmp_path):
    """`compile --tma-tiles --launch ...` lowers mm's rotating B k-tile to TMA
    tensor copies (a CUtensorMap kernel parameter); without the flag the
    register staging stays."""
    from paper_1710_08332_b200.bench_programs import mm_program
    f = _prog(tmp_path, mm_program(256, 256, 128, 128, 16, 8), "mm.dpia")
    assert main(["compile", f, "--launch", "2,2,16,16", "--tma-tiles", "-o", str(tmp_path / "a.cu")]) == 0
    assert main(["compile", f, "--launch", "2,2,16,16", "-o", str(tmp_path / "b.cu")]) == 0
    a, b = (tmp_path / "a.cu").read_text(), (tmp_path / "b.cu").read_text()
    assert "dpia::TensorMap dpia_tm0" in a and "dpia::tma_tile_2d(" in a
    assert "dpia::TensorMap dpia_tm0" not in b


def test_cli_exit_codes(tmp_path):
    assert main(["compile", _prog(tmp_path, "(param xs (exp (array 4 num))) (map")]) == 2
    assert main(["compile", _prog(tmp_path, "(param xs (exp (array 4 num)))\n(zip xs (split 2 xs))",
                                  "t.dpia")]) == 3
    assert main(["compile", str(tmp_path / "missing.dpia")]) == 2
    racy = ("(param b (acc num))\n(param out2 (acc (array 4 num)))\n"
            "(parfor out2 (lam (i (exp (idx 4))) (lam (o (acc num)) (:= b 1))))")
    assert main(["compile", _prog(tmp_path, racy, "racy.dpia")]) == 3   # SCIR interference


def test_cli_module_entry_point():
    r = subprocess.run([sys.executable, "-m", "paper_1710_08332_b200.cli", "--help"],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0 and "compile" in r.stdout


def test_criterion3_analogue_cuda_kernel_text():
    """The vectorised dot kernel (TST/test_acceptance.py:119-153) rendered for
    CUDA carries the strategy: work-group and work-item ids, float4 loads and
    stores, a private float4 accumulator."""
    from conftest import load_golden
    from paper_1710_08332_b200 import compile_program, emit_cuda
    case = [c for c in load_golden("programs.json") if c["name"] == "dotvec.dpia"][0]
    prog = compile_program(case["text"], name="dotvec")
    src, sig = emit_cuda(prog.imperative, [("out", prog.out_type)],
                         [(n, t.data) for n, t in prog.source.params], float_mode=True, name="dotvec")
    for needle in ("blockIdx.x", "gridDim.x", "threadIdx.x", "blockDim.x",
                   "dpia::vload<float, 4>", "dpia::vstore<float, 4>", "dpia::vec<float, 4> acc"):
        assert needle in src, needle
    assert [k.name for k in sig.kernels] == ["dotvec_k0"]


def test_cli_dump_stages_reparse(tmp_path):
    from conftest import load_golden
    from paper_1710_08332_b200.dtypes import AccT
    from paper_1710_08332_b200.reader import parse, parse_phrase
    case = [c for c in load_golden("programs.json") if c["name"] == "dottiled.dpia"][0]
    f = _prog(tmp_path, case["text"], "dottiled.dpia")
    assert main(["compile", f, "--dump-stages"]) == 0
    sp = parse(case["text"])
    env = {**dict(sp.params), "out": AccT(sp.body_type.data)}
    for stage in ("stage1", "stage2"):
        parse_phrase(open(str(tmp_path / f"dottiled.{stage}.dpia")).read(), env)


def test_cli_reference_compile_flags(tmp_path, capsys):
    """--check-only / --init-new / --simplify-indices behave like the
    reference CLI's (SRC/cli.py:93-96, 236-246)."""
    from conftest import load_golden
    src = [c for c in load_golden("programs.json") if c["name"] == "dotvec.dpia"][0]["text"]
    f = _prog(tmp_path, src, "dotvec.dpia")
    assert main(["compile", f, "--check-only"]) == 0
    out = capsys.readouterr().out
    assert "OK" in out and not (tmp_path / "dotvec.cu").exists()
    assert main(["compile", f, "--init-new", "--simplify-indices", "off", "-o",
                 str(tmp_path / "x.cu")]) == 0
    assert "__global__" in (tmp_path / "x.cu").read_text()
    # the reference-only targets are not the CUDA backend's
    with pytest.raises(SystemExit):
        main(["compile", f, "--target", "opencl"])


def test_later_phases_wait_for_the_previous_grid():
    """Kernels after the first are launched with programmatic dependent
    launch (Executable.launch), so each must begin with griddepcontrol.wait
    and the first must not (CPU: emitted text only)."""
    import json
    import re
    from paper_1710_08332_b200 import compile_program, emit_cuda
    seen = 0
    for v in json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fuzz.json")))[:400]:
        try:
            p = compile_program(v["text"])
            src, sig = emit_cuda(p.imperative, [("out", p.out_type)],
                                 [(n, t.data) for n, t in p.source.params], float_mode=False, name="t",
                                 launch=(4, 32), sigma=v.get("sigma"))
        except Exception:  # noqa: BLE001 -- programs the backend rejects are not the point here
            continue
        bodies = re.split(r'extern "C" __global__', src)[1:]
        assert len(bodies) == len(sig.kernels)
        for i, b in enumerate(bodies):
            assert ("griddepcontrol.wait" in b) == (i > 0)
        seen += len(bodies) > 1
    assert seen > 10


def test_bench_reference_arm_line():
    """`bench.py --impl reference` (the reference's own c-openmp CPU path) prints
    one JSON line with the arm's metric, unit and config (CPU; skipped when
    oracle/_ref was not built)."""
    import json
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libref_cpu.so")):
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--workload", "dot", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    assert line["config"]["workload"].startswith("dot N=2^24")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"


@pytest.mark.gpu
def test_bench_json_contract():
    """One short `bench.py` run on the GPU: every key of the driver's contract
    is present and consistent."""
    import json
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                        "--no-suite", "--no-cpu"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks",
              "gpu_launches", "cpu_baseline"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["value"] > 0 and line["gpu_launches"] >= 3
    roof = line["roofline"]
    assert roof["bound"] == "hbm" and roof["unit"] == "GB/s" and 0 < roof["frac"] < 1.5
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-3
    e2e = line["e2e"]
    assert e2e["h2d_bytes_per_step"] == 4 << 26 and e2e["value"] > 0
    assert line["clocks"]["sm_max_mhz"] > 0


def test_reference_cpu_path_computes_the_workloads():
    """The reference's own c-openmp emissions (oracle/_ref, the CPU baseline
    and the --impl reference arm) compute what the GPU workloads compute
    (CPU; checked against float64 numpy, fp32 tolerance)."""
    import ctypes
    import numpy as np
    lib_path = os.path.join(ROOT, "oracle", "_ref", "libref_cpu.so")
    if not os.path.exists(lib_path):
        pytest.skip("oracle/_ref not built")
    lib = ctypes.CDLL(lib_path)
    vp, ci = ctypes.c_void_p, ctypes.c_int
    rng = np.random.default_rng(9)
    n = 16
    xs = rng.uniform(-1, 1, 1024 * n).astype(np.float32)
    ys = rng.uniform(-1, 1, 1024 * n).astype(np.float32)
    out = np.zeros(8192, np.float32)
    lib.asum_proxy.argtypes = [vp, vp, ci]
    lib.asum_proxy(out.ctypes.data, xs.ctypes.data, n)
    assert abs(out[0] - xs.astype(np.float64).sum()) <= 1e-4 * np.abs(xs).sum()
    lib.dot.argtypes = [vp, vp, vp, ci]
    lib.dot(out.ctypes.data, xs.ctypes.data, ys.ctypes.data, n)
    assert abs(out[0] - xs.astype(np.float64) @ ys) <= 1e-4 * np.abs(xs * ys).sum()
    lib.scal.argtypes = [vp, ctypes.c_float, vp, ci]
    y = np.zeros_like(xs)
    lib.scal(y.ctypes.data, 1.5, xs.ctypes.data, n)
    assert np.array_equal(y, np.float32(1.5) * xs)
    A = rng.uniform(-1, 1, (8192, 8192)).astype(np.float32)
    x = rng.uniform(-1, 1, 8192).astype(np.float32)
    lib.gemv.argtypes = [vp, vp, vp]
    lib.gemv(out.ctypes.data, A.ctypes.data, x.ctypes.data)
    want = A.astype(np.float64) @ x
    assert np.all(np.abs(out - want) <= 1e-4 * (np.abs(A) @ np.abs(x)))


def test_cli_fuzz_arguments_and_report(tmp_path):
    """CPU: a missing corpus is a parse-class failure (exit 2); the JUnit
    writer emits one testcase per program with its failure message."""
    import xml.etree.ElementTree as ET
    from paper_1710_08332_b200.cli import Status, _junit, main
    assert main(["fuzz", "--corpus", str(tmp_path / "nope.json")]) == Status.PARSE
    _junit(tmp_path / "r.xml", [("seed-0", None), ("seed-1", "GPU [1] != reference [2]")])
    root = ET.parse(tmp_path / "r.xml").getroot()
    assert root.get("tests") == "2" and root.get("failures") == "1"
    assert root.findall("testcase")[1].find("failure").get("message").startswith("GPU")


def test_nvrtc_is_the_toolkits_even_with_an_older_one_loaded():
    """The runtime binds NVRTC by the toolkit's absolute path (RTLD_LOCAL):
    an older libnvrtc.so.12 already in the process (PyTorch's wheel ships
    12.8) must not capture the calls -- it rejects the sm_100 256-bit loads
    (ld.global.v8.f32) the emitter's fold queues use."""
    import ctypes
    import glob
    import sys
    for p in glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia",
                                    "cuda_nvrtc", "lib", "libnvrtc.so.12")):
        ctypes.CDLL(p, mode=ctypes.RTLD_GLOBAL)
    assert RT.nvrtc_version() >= (12, 9)
    img = RT.nvrtc_compile('extern "C" __global__ void k(float* p) { float a0,a1,a2,a3,a4,a5,a6,a7;\n'
                           'asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=f"(a0),'
                           '"=f"(a1),"=f"(a2),"=f"(a3),"=f"(a4),"=f"(a5),"=f"(a6),"=f"(a7) : "l"(p));\n'
                           'p[0] = a0+a1+a2+a3+a4+a5+a6+a7; }')
    assert img[:4] == b"\x7fELF"
