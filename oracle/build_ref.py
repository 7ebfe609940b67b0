"""ORACLE build recipe: the reference's own CPU path, compiled here.

The reference is pure Python, but it has exactly one path that runs the
benchmark strategies at full size on host cores: its `c-openmp` target
(`dpia compile P.dpia --target c-openmp`, /root/reference/pkg/src/dpia/
cli.py:58-90,118-121), which prints OpenMP C from the same Stage I/II
pipeline.  This script runs the reference CLI (importable only in the build
container) on the strategy programs in oracle/ref_programs/ -- written in the
reference's language -- and compiles the emitted C with gcc/OpenMP into
oracle/_ref/libref_cpu.so (git-ignored, travels to the GPU box with the
snapshot).  bench.py times it as `cpu_baseline` (kind "reference") and as the
`--impl reference` arm.  Nothing is copied from the reference's sources:
the .c files are the reference compiler's *output* for our programs.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
REF_SRC = "/root/reference/pkg/src"
PROGRAMS = ("asum_proxy", "dot", "gemv", "mm_bt", "scal")
LIB = os.path.join(OUT, "libref_cpu.so")

HARNESS = r"""
#include <omp.h>
int ref_threads(void) { return omp_get_max_threads(); }
"""


def build(verbose: bool = False) -> bool:
    if not os.path.isdir(REF_SRC):
        if verbose:
            print("[oracle] /root/reference absent: using the prebuilt oracle/_ref (if any)")
        return os.path.exists(LIB)
    os.makedirs(OUT, exist_ok=True)
    env = dict(os.environ, PYTHONPATH=REF_SRC)
    csrc = []
    for name in PROGRAMS:
        src = os.path.join(HERE, "ref_programs", name + ".dpia")
        dst = os.path.join(OUT, name + ".c")
        subprocess.run([sys.executable, "-m", "dpia.cli", "compile", src, "--target", "c-openmp",
                        "-o", dst], check=True, env=env, capture_output=not verbose)
        csrc.append(dst)
    h = os.path.join(OUT, "harness.c")
    with open(h, "w") as f:
        f.write(HARNESS)
    # x86-64-v3 (AVX2/FMA) rather than -march=native: the .so is built here
    # and runs on the GPU box's host CPU
    cmd = ["gcc", "-O3", "-march=x86-64-v3", "-fopenmp", "-shared", "-fPIC", "-o", LIB, h] + csrc
    if verbose:
        print("+", " ".join(cmd))
    subprocess.run(cmd, check=True)
    return True


def _host_tag() -> str:
    """Short hash of this host's CPU model and feature flags: a -march=native
    build is only reused on a host that reports the same CPU."""
    import hashlib
    h = hashlib.sha1()
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith(("model name", "flags")):
                    h.update(ln.encode())
                    if ln.startswith("flags"):
                        break
    except OSError:
        pass
    return h.hexdigest()[:12]


def native_lib():
    """(path, march) of the reference CPU library to time on this host.

    The emitted .c files (the reference compiler's output, git-ignored but
    shipped with the snapshot) are recompiled here once with -march=native,
    as BASELINE.md section 4 prescribes; the portable x86-64-v3 build is the
    fallback when gcc is missing or fails.  (None, None) if neither exists."""
    NATIVE = os.path.join(OUT, f"libref_cpu_native_{_host_tag()}.so")
    srcs = [os.path.join(OUT, n + ".c") for n in PROGRAMS] + [os.path.join(OUT, "harness.c")]
    if os.path.exists(NATIVE) and all(os.path.getmtime(NATIVE) >= os.path.getmtime(c)
                                      for c in srcs if os.path.exists(c)):
        return NATIVE, "native"
    if all(os.path.exists(c) for c in srcs):
        tmp = f"{NATIVE}.{os.getpid()}.tmp"
        try:
            subprocess.run(["gcc", "-O3", "-march=native", "-fopenmp", "-shared", "-fPIC", "-o", tmp]
                           + srcs, check=True, capture_output=True)
            os.replace(tmp, NATIVE)
            return NATIVE, "native"
        except (OSError, subprocess.CalledProcessError):
            if os.path.exists(tmp):
                os.remove(tmp)
    if os.path.exists(LIB):
        return LIB, "x86-64-v3"
    return None, None


if __name__ == "__main__":
    build(verbose=True)
