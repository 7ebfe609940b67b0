"""Ahead-of-time artefacts for the GPU box: cubins of the benchmark kernels
(NVRTC, sm_100a) cached in paper_1710_08332_b200/kcache/, plus an nvcc
compile of each emitted translation unit as the build-time check
(`nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo`)."""
from __future__ import annotations

import os
import subprocess
import tempfile

from . import runtime as RT

NVCC = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")


def nvcc_check(src: str, tag: str, verbose: bool = False) -> str:
    """Compile an emitted translation unit with nvcc for sm_100a; returns the
    ptxas resource report (registers / spills / shared memory)."""
    with tempfile.TemporaryDirectory() as d:
        cu = os.path.join(d, f"{tag}.cu")
        with open(cu, "w") as f:
            f.write(src)
        r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3",
                            "-std=c++17", "-Xptxas", "-v", "-cubin", "-o", os.path.join(d, f"{tag}.cubin"),
                            cu], capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"nvcc failed for {tag}:\n{r.stderr[-4000:]}")
        return r.stderr


def build_all(verbose: bool = False):
    from . import bench_programs as BP
    os.makedirs(RT.KCACHE_DIR, exist_ok=True)
    keep = set()
    for tag, src in BP.aot_sources():
        key = RT.cubin_key(src)
        keep.add(key + ".cubin")
        path = os.path.join(RT.KCACHE_DIR, key + ".cubin")
        report = nvcc_check(src, tag)
        if verbose:
            regs = [ln.strip() for ln in report.splitlines() if "registers" in ln or "spill" in ln]
            print(f"[aot] {tag}: " + " | ".join(regs[-2:]))
        if not os.path.exists(path):
            img = RT.nvrtc_compile(src)
            with open(path, "wb") as f:
                f.write(img)
    for stale in set(os.listdir(RT.KCACHE_DIR)) - keep:   # sources changed since
        if stale.endswith(".cubin"):
            os.remove(os.path.join(RT.KCACHE_DIR, stale))
