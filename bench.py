"""Benchmark: DPIA-emitted CUDA kernels on B200 against the HBM / FP32 roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload asum|dot|gemv|scaleout] [--no-suite]

Headline workload (BASELINE.json configs[1]): asum over N = 2^26 fp32 with
the vectorised asVector(4) + mapWorkgroup/mapLocal + reduceLocal strategy.
A "step" is one pass of the emitted program over the resident input (all of
its kernels, the fused work-group/grid combine included); L2 is flushed
between steps (a 2x-L2 read, outside the timed events).  Multi-GPU (torchrun,
one process per GPU): every rank runs the full per-GPU workload on its own
shard (weak scaling) and the partial sums are combined inside the step --
by default inside the kernel itself over NVLink (--combine peer: the fused
cross-GPU combine of paper_1710_08332_b200/peer.py), or with a 4-byte NCCL
all-reduce after it (--combine nccl); the time is the max over ranks.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1710_08332_b200 import compile_program, executable  # noqa: E402
from paper_1710_08332_b200 import runtime as RT  # noqa: E402
from paper_1710_08332_b200.bench_programs import (asum_config, asum_proxy_config, dot_config,  # noqa: E402
                                                  dot_literal_config, gemv_config, gemv_literal_config,
                                                  mm_config,
                                                  mm_tma_config, scal_config, scal_literal_config)

METRIC = "achieved HBM GB/s (dot/asum/gemv), GFLOP/s (mm) vs roofline, at 1-8 B200"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def fp32_peak(device):
    """FP32 FFMA peak: SMs x 128 lanes x 2 flop x max SM clock (nominal).
    Returns (TFLOP/s, description)."""
    sms = RT.device_attribute(device, RT.ATTR_SM_COUNT)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f)["sm_max_mhz"])
    except (OSError, KeyError, ValueError):
        mhz = 1965.0
    return sms * 128 * 2 * mhz * 1e6 / 1e12, f"computed: {sms} SMs x 128 FFMA x 2 x {mhz:.0f} MHz"


_SOL_CACHE = {}


NOMINAL_HBM_GBS = 7700.0     # B200 HBM3e, HGX figure (B200_PROFILING.md)


def l2_bytes(device):
    return RT.device_attribute(device, 38) or (126 << 20)     # CU_DEVICE_ATTRIBUTE_L2_CACHE_SIZE


def rotation(device, step_bytes):
    """How many input sets the steady-state timing rotates through: enough
    that R x the step's bytes >= 3 x L2, so the set a step reads was evicted
    by the reads of the steps since its last use (the contract's "inputs
    larger than L2")."""
    return max(1, -(-3 * l2_bytes(device) // step_bytes))


def read_sol(device, nbytes, stream):
    """Size-matched speed of light: a hand-written minimal CUDA streaming-read
    kernel (tools/readsol.py; measurement infrastructure, not product) timed
    exactly like the benchmark steps on `nbytes` of HBM: {"steady": GB/s over
    back-to-back reads of rotating buffers, "isolated": GB/s of one launch
    after an L2 scrub}."""
    if nbytes in _SOL_CACHE:
        return _SOL_CACHE[nbytes]
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from readsol import SRC
    mod = RT.Module(RT.get_cubin(SRC), device)
    fn = mod.function("readsum")
    R = rotation(device, nbytes)
    bufs, out = [RT.DeviceBuffer(nbytes, device) for _ in range(R)], RT.DeviceBuffer(16, device)
    for b in bufs:
        b.zero(stream)
    args = [[RT.C.c_uint64(b.ptr), RT.C.c_longlong(nbytes // 16), RT.C.c_uint64(out.ptr)] for b in bufs]

    def launch(i, chain=False):
        RT.launch(fn, device, (296, 1), (1024, 1), 0, args[i % R], stream, pdl=chain)
    ts = []
    for it in range(13):
        RT.lib().dpia_l2_flush(device, stream.handle)
        e0, e1 = RT.Event(device), RT.Event(device)
        e0.record(stream)
        launch(0)
        e1.record(stream)
        stream.sync()
        if it >= 3:
            ts.append(e0.elapsed_ms(e1))
    K = 30
    for i in range(6):
        launch(i, True)
    runs = []
    for rep in range(3):
        e0, e1 = RT.Event(device), RT.Event(device)
        e0.record(stream)
        for i in range(K):
            launch(i, True)        # chained like the benchmark steps
        e1.record(stream)
        stream.sync()
        runs.append(e0.elapsed_ms(e1) / K)
    for b in bufs:
        b.free()
    out.free()
    _SOL_CACHE[nbytes] = {"steady": round(nbytes / statistics.median(runs) / 1e6, 1),
                          "isolated": round(nbytes / statistics.median(ts) / 1e6, 1)}
    return _SOL_CACHE[nbytes]


_FFMA_CACHE = {}


def ffma_peak(device, stream):
    """(measured FP32 FMA ceiling, mm inner-loop ceiling) in TFLOP/s:
    tools/ffmapeak.py's register-only packed FFMA2 kernel at 8 CTAs/SM x 256
    threads, and its `mmloop` (mm's k-step from a shared tile, no staging,
    no barrier) at 2 CTAs/SM -- measurement infrastructure, not product;
    means of 10 event-timed launches after warm-up."""
    if device in _FFMA_CACHE:
        return _FFMA_CACHE[device]
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from ffmapeak import ITERS, SRC, mmloop
    mod = RT.Module(RT.get_cubin(SRC), device)
    fn = mod.function("ffma2")
    out = RT.DeviceBuffer(64, device)
    blocks = RT.device_attribute(device, RT.ATTR_SM_COUNT) * 8
    args = [RT.C.c_uint64(out.ptr), RT.C.c_float(0.999), RT.C.c_float(1e-4), RT.C.c_int(ITERS)]
    ts = []
    for it in range(13):
        e0, e1 = RT.Event(device), RT.Event(device)
        e0.record(stream)
        RT.launch(fn, device, (blocks, 1), (256, 1), 0, args, stream)
        e1.record(stream)
        stream.sync()
        if it >= 3:
            ts.append(e0.elapsed_ms(e1))
    inner = mmloop(mod, stream, RT.device_attribute(device, RT.ATTR_SM_COUNT), out)
    out.free()
    flops = blocks * 256 * ITERS * 16 * 2 * 2
    _FFMA_CACHE[device] = (round(flops / statistics.mean(ts) / 1e9, 2), round(inner, 2))
    return _FFMA_CACHE[device]


def ncu_traffic(workload):
    """Per-launch DRAM bytes of the dominant kernel from a committed ncu
    capture (the fallback of live_traffic)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(workload)
    except (OSError, ValueError):
        return None


def live_traffic(workload, kernel, timeout=240):
    """DRAM bytes (read + write) of one launch of `kernel`, measured in this
    run: ncu profiles a child process that builds the same workload and
    launches it after an L2 scrub (`--traffic-child`), outside every timed
    region.  Returns (bytes or None, source)."""
    import shutil
    if _under_profiler():
        # a profiler already wraps this process (e.g. the driver's ncu launch
        # list): no nested ncu
        return ncu_traffic(workload), "committed ncu capture (bench.py itself runs under a profiler)"
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--csv",
           "--print-units", "base", "-k", f"regex:^{kernel}$", "--launch-skip", "2",
           "--launch-count", "1", sys.executable, os.path.abspath(__file__), "--traffic-child",
           "--workload", workload]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    except (OSError, subprocess.TimeoutExpired) as e:
        return ncu_traffic(workload), f"committed ncu capture (live ncu failed: {type(e).__name__})"
    vals = {}
    for ln in r.stdout.splitlines():
        cells = [c.strip('"') for c in ln.split('","')]
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if name in cells:
                try:
                    vals[name] = float(cells[-1].strip('"').replace(",", ""))
                except ValueError:
                    pass
    if len(vals) == 2:
        return int(sum(vals.values())), "live: ncu dram__bytes_read.sum + dram__bytes_write.sum, one launch"
    return ncu_traffic(workload), f"committed ncu capture (live ncu rc={r.returncode}, no metrics parsed)"


def _under_profiler() -> bool:
    """ncu / compute-sanitizer inject themselves through CUDA_INJECTION64_PATH
    and an LD_PRELOAD of their process-tree launcher."""
    pre = os.environ.get("LD_PRELOAD", "")
    return bool(os.environ.get("CUDA_INJECTION64_PATH")) or "TreeLauncher" in pre or "nsight" in pre


def traffic_child(workload):
    """The process live_traffic profiles: the workload's program, inputs and
    launch exactly as measured, three launches each after an L2 scrub."""
    RT.init(0)
    stream = RT.Stream(0)
    cfg, exe, inputs, prepare, prog = make_workload(workload, 0)
    prepare(stream)
    for _ in range(3):
        RT.lib().dpia_l2_flush(0, stream.handle)
        exe.launch(stream)
    stream.sync()
    return 0


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.samples = []
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate()
        for ln in out.splitlines():
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) == 6:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), parts[2:]))
                except ValueError:
                    pass

    def summary(self):
        if not getattr(self, "samples", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for _, _, flags in self.samples for n, fl in zip(names, flags)
                          if fl.lower() == "active"})
        loaded = [s for s, _, _ in self.samples if s > 500] or [s for s, _, _ in self.samples]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.samples[0][1],
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------ workloads

def make_workload(name, device, rank=0, world=1, combine="nccl"):
    """(config, executable, host inputs or None, prepare(stream), program).
    The program is returned so a peer-combined executable can be checked
    against its combine-free twin (peer.cross_check)."""
    allgather = None
    if world > 1 and combine == "peer":
        from paper_1710_08332_b200.peer import torch_allgather as allgather
    if name.startswith("scaleout"):
        from paper_1710_08332_b200.bench_programs import Config
        from paper_1710_08332_b200.scaleout import ShardedReduction
        kind = "dot" if name.endswith("dot") else "asum"
        run = ShardedReduction(kind, 1 << 31, world, rank, device,
                               combine=combine if world > 1 else "nccl", allgather=allgather)
        cfg = Config(name, "", {"n": run.shard.chunks}, run.exe.sig.launch, bytes=run.bytes,
                     flops=(2 if kind == "dot" else 1) * run.shard.elems)
        return cfg, run.exe, None, run.fill_inputs, run.prog
    if name in ("asum", "asum_proxy"):
        cfg = asum_config() if name == "asum" else asum_proxy_config()
        inputs = {"xs": _seeded(1 << 26, 2 + 1000 * rank, -1.0, 1.0)}
    elif name == "dot":
        cfg = dot_config()
        inputs = {"xs": _seeded(1 << 24, 0 + 1000 * rank, 0.0, 1.0),
                  "ys": _seeded(1 << 24, 1 + 1000 * rank, 0.0, 1.0)}
    elif name == "dot_literal":
        cfg = dot_literal_config()
        inputs = {"xs": _seeded(1 << 24, 0 + 1000 * rank, 0.0, 1.0),
                  "ys": _seeded(1 << 24, 1 + 1000 * rank, 0.0, 1.0)}
    elif name in ("gemv", "gemv_xprivate", "gemv_literal"):
        cfg = gemv_literal_config() if name == "gemv_literal" else gemv_config(x_private=name == "gemv_xprivate")
        cfg.name = name
        inputs = {"A": _seeded((8192, 8192), 3, -1.0, 1.0), "x": _seeded(8192, 4, -1.0, 1.0)}
    elif name in ("scal", "scal_literal"):
        cfg = scal_config() if name == "scal" else scal_literal_config()
        # alpha: a splat vec4 in the B200 program, a scalar in the reference's
        inputs = {"alpha": np.full(4 if name == "scal" else 1, 1.5, np.float32),
                  "xs": _seeded(1 << 26, 7, -1.0, 1.0)}
    elif name in ("mm", "mm_tma"):
        cfg = mm_config() if name == "mm" else mm_tma_config()
        inputs = {"A": _seeded((4096, 4096), 5, -1.0, 1.0), "B": _seeded((4096, 4096), 6, -1.0, 1.0)}
    else:
        raise SystemExit(f"unknown workload {name}")
    prog = compile_program(cfg.text, name=name)
    peer = None
    if allgather is not None and name in ("asum", "dot", "dot_literal"):
        from paper_1710_08332_b200.peer import PeerGroup
        peer = PeerGroup(device, rank, world, 1, allgather)
    exe = executable(prog, cfg.launch, cfg.sigma, float_mode=True, device=device, peer=peer, **cfg.emit)

    def prepare(stream):
        for n, v in inputs.items():
            exe.upload(n, v, stream)
    return cfg, exe, inputs, prepare, prog


def _seeded(shape, seed, lo, hi):
    return np.random.default_rng(seed).uniform(lo, hi, size=shape).astype(np.float32)


class Rotation:
    """The steady-state step: K steps back to back on one stream, step i
    reading input set i % R (`rotation`), between ONE event pair.  Set 0 is
    the executable's own buffers; the other sets are device copies of its
    inputs (and of outputs larger than 1 MiB, so written lines rotate too)."""

    def __init__(self, exe, step_bytes, stream, chain=True):
        self.exe = exe
        self.chain = chain          # each step chained behind the previous (PDL)
        self.R = rotation(exe.device, step_bytes)
        self.extra = []
        self.ptrs = [None]
        names = [n for n, _ in exe.sig.inputs] + [n for n, _ in exe.sig.outputs
                                                  if exe.buffers[n].nbytes > (1 << 20)]
        for _ in range(self.R - 1):
            ptrs = {}
            for n in names:
                src = exe.buffers[n]
                b = RT.DeviceBuffer(src.nbytes, exe.device)
                RT.lib().dpia_memcpy_dtod(exe.device, b.ptr, src.ptr, src.nbytes, stream.handle)
                self.extra.append(b)
                ptrs[n] = b.ptr
            self.ptrs.append(ptrs)
        stream.sync()

    def launch(self, i, stream):
        p = self.ptrs[i % self.R]
        if p is None:
            self.exe.launch(stream, chain=self.chain)
        else:
            self.exe.launch_with(stream, p, chain=self.chain)

    def run(self, stream, steps, allreduce=None, start=0):
        """ms per step of `steps` back-to-back steps (events on `stream`)."""
        e0, e1 = RT.Event(self.exe.device), RT.Event(self.exe.device)
        e0.record(stream)
        for i in range(start, start + steps):
            self.launch(i, stream)
            if allreduce:
                allreduce(stream)
        e1.record(stream)
        stream.sync()
        return e0.elapsed_ms(e1) / steps

    def free(self):
        for b in self.extra:
            b.free()
        self.extra, self.ptrs, self.R = [], [None], 1


def run_isolated(exe, stream, steps, allreduce=None):
    """Per-launch event pairs, each launch after an L2 scrub (the round-1
    method; reported beside the steady-state number)."""
    dev = exe.device
    ev = [(RT.Event(dev), RT.Event(dev)) for _ in range(steps)]
    for e0, e1 in ev:
        RT.lib().dpia_l2_flush(dev, stream.handle)
        e0.record(stream)
        exe.launch(stream)
        if allreduce:
            allreduce(stream)
        e1.record(stream)
    stream.sync()
    return [e0.elapsed_ms(e1) for e0, e1 in ev]


def e2e_measure(exe, inputs, stream, steps):
    """The public API end to end with host buffers: `Executable.run` copies
    the step's inputs from page-locked host memory, launches the program and
    copies the result back to page-locked host memory, synchronising before
    it returns -- all inside the timed events."""
    from paper_1710_08332_b200 import layout as LY
    dev = exe.device
    pinned, host, h2d = [], {}, 0
    for n, d in exe.sig.inputs:
        img = LY.to_bytes(inputs[n], d, exe.sigma, True)
        pb = RT.PinnedBuffer(img.nbytes)
        arr = pb.array(np.float32, img.nbytes // 4)
        arr[:] = img.view(np.float32)
        pinned.append(pb)
        host[n] = arr
        h2d += img.nbytes
    outn, outd = exe.sig.outputs[0]
    d2h = LY.nbytes(outd, exe.sigma, True)
    ob = RT.PinnedBuffer(d2h)
    pinned.append(ob)
    res = {outn: ob.array(np.float32, d2h // 4)}
    times = []
    for _ in range(steps + 1):
        e0, e1 = RT.Event(dev), RT.Event(dev)
        e0.record(stream)
        exe.run(host, stream, out=res)
        e1.record(stream)
        stream.sync()
        times.append(e0.elapsed_ms(e1))
    # the host link alone: the same H2D bytes with nothing else in the step
    link = []
    for _ in range(3):
        e0, e1 = RT.Event(dev), RT.Event(dev)
        e0.record(stream)
        for n, _d in exe.sig.inputs:
            RT.lib().dpia_memcpy_htod(dev, exe.buffers[n].ptr, host[n].ctypes.data_as(ctypes.c_void_p),
                                      host[n].nbytes, stream.handle)
        e1.record(stream)
        stream.sync()
        link.append(e0.elapsed_ms(e1))
    global _LINK_GBS
    _LINK_GBS = round(h2d / (statistics.median(link) * 1e-3) / 1e9, 2)
    for pb in pinned:
        pb.free()
    return statistics.mean(times[1:]), h2d, d2h


_LINK_GBS = None


def e2e_pipelined_mm(inputs, stream, steps, chunks=4, tiles=None):
    """mm end to end through a public pipeline: RowPipeline over `chunks` row
    blocks, or TilePipeline over `tiles` = (rows, cols, compute streams)."""
    from paper_1710_08332_b200.pipeline import mm_pipeline, mm_tile_pipeline
    A, B = inputs["A"], inputs["B"]
    M, K = A.shape
    N = B.shape[1]
    pins = [RT.PinnedBuffer(A.nbytes), RT.PinnedBuffer(B.nbytes), RT.PinnedBuffer(4 * M * N)]
    ha, hb = pins[0].array(np.float32, A.size), pins[1].array(np.float32, B.size)
    ha[:], hb[:] = A.ravel(), B.ravel()
    out = pins[2].array(np.float32, M * N)
    if tiles:
        pipe = mm_tile_pipeline(M, N, K, rows=tiles[0], cols=tiles[1], compute_streams=tiles[2])
    else:
        pipe = mm_pipeline(M, N, K, chunks=chunks)
    times = []
    for _ in range(steps + 1):
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(stream)
        pipe.run({"A": ha, "B": hb}, out, stream)
        e1.record(stream)
        stream.sync()
        times.append(e0.elapsed_ms(e1))
    for p in pins:
        p.free()
    return statistics.mean(times[1:]), A.nbytes + B.nbytes, 4 * M * N


def e2e_pipelined_scal(inputs, stream, steps, chunks=8):
    from paper_1710_08332_b200.pipeline import scal_pipeline
    xs, alpha = inputs["xs"], inputs["alpha"]
    N = xs.size
    pins = [RT.PinnedBuffer(16), RT.PinnedBuffer(xs.nbytes), RT.PinnedBuffer(xs.nbytes)]
    ha, hx, out = pins[0].array(np.float32, 4), pins[1].array(np.float32, N), pins[2].array(np.float32, N)
    ha[:], hx[:] = alpha, xs
    pipe = scal_pipeline(N, chunks=chunks)
    times = []
    for _ in range(steps + 1):
        e0, e1 = RT.Event(0), RT.Event(0)
        e0.record(stream)
        pipe.run({"alpha": ha, "xs": hx}, out, stream)
        e1.record(stream)
        stream.sync()
        times.append(e0.elapsed_ms(e1))
    for p in pins:
        p.free()
    return statistics.mean(times[1:]), 16 + xs.nbytes, xs.nbytes


# ------------------------------------------------------------ CPU legs

def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


_REF_LIB = None


def ref_lib():
    """The reference's CPU path (oracle/_ref): its c-openmp emissions of the
    strategy programs.  On the benchmark host they are recompiled once with
    -march=native (oracle/build_ref.py native; the generated .c files travel
    with the snapshot), else the prebuilt x86-64-v3 library is used."""
    global _REF_LIB
    if _REF_LIB is not None:
        return _REF_LIB
    sys.path.insert(0, ROOT)
    from oracle import build_ref
    path, march = build_ref.native_lib()
    if path is None:
        return None
    lib = ctypes.CDLL(path)
    lib.march = march
    _REF_LIB = lib
    return lib


# what the reference's CPU path runs for each workload (oracle/ref_programs/*.dpia
# through the reference's own `compile --target c-openmp`)
REF_STRATEGY = {
    "asum": ("asum N=2^26 fp32", "asum_proxy.dpia: mapGlobal over 1024-element chunks, sequential "
             "reduce per chunk, sequential top-level reduce of the partials; a plain sum -- the "
             "reference language has no abs -- with asum's exact traffic"),
    "dot": ("dot N=2^24 fp32", "dot.dpia (BASELINE config 1): mapGlobal over 1024-element chunks of "
            "zip xs ys, sequential reduce per chunk, sequential top-level reduce"),
    "gemv": ("gemv 8192x8192 fp32", "gemv.dpia: row per work-group, x staged toLocal, 256 items x "
             "32-element chunks, partials combined sequentially"),
    "scal": ("scal N=2^26 fp32 (read + write)", "scal.dpia: mapGlobal over 1024-element chunks, mapSeq"),
    "mm": ("mm 4096^3 fp32", "mm_bt.dpia: B passed pre-transposed (the reference language has no "
           "transpose), one row of A per work-item, sequential reduce per output element"),
}
REF_STRATEGY["dot_literal"] = REF_STRATEGY["dot"]
REF_STRATEGY["gemv_xprivate"] = REF_STRATEGY["gemv"]
REF_STRATEGY["gemv_literal"] = REF_STRATEGY["gemv"]
REF_STRATEGY["scal_literal"] = REF_STRATEGY["scal"]
REF_STRATEGY["mm_tma"] = REF_STRATEGY["mm"]
REF_STRATEGY["asum_proxy"] = REF_STRATEGY["asum"]


def cpu_reference(workload, min_seconds=2.0, max_reps=200, steps=None, warmup=1):
    """Time the reference's own CPU path (its c-openmp emission of the
    workload's program, oracle/ref_programs/) on all host threads."""
    lib = ref_lib()
    if lib is None:
        return None
    vp, ci = ctypes.c_void_p, ctypes.c_int
    out = np.zeros(8192, np.float32)
    base = {"mm_tma": "mm", "asum_proxy": "asum", "gemv_literal": "gemv",
            "scal_literal": "scal"}.get(workload, workload)
    note = ""
    if workload.startswith("scaleout"):
        # the reference's emitted C indexes with 32-bit int and keeps the
        # partials in a stack VLA: 2^31 elements overflow both, so a
        # bounded sample of the same per-element work is timed
        base = "dot" if workload.endswith("dot") else "asum"
        note = ("; a 2^24 (dot) / 2^26 (asum) sample of the 2^31 workload: the reference's emitted C "
                "indexes with 32-bit int and cannot address 2^31 elements")
    if base in ("asum",):
        n = (1 << 26) // 1024
        xs = _seeded(1 << 26, 2, -1.0, 1.0)
        fn = lib.asum_proxy
        fn.argtypes = [vp, vp, ci]
        call = lambda: fn(out.ctypes.data, xs.ctypes.data, n)  # noqa: E731
        nbytes, sample = 4 << 26, "asum_proxy over 2^26 fp32, full size"
    elif base in ("dot", "dot_literal"):
        n = (1 << 24) // 1024
        xs, ys = _seeded(1 << 24, 0, 0.0, 1.0), _seeded(1 << 24, 1, 0.0, 1.0)
        fn = lib.dot
        fn.argtypes = [vp, vp, vp, ci]
        call = lambda: fn(out.ctypes.data, xs.ctypes.data, ys.ctypes.data, n)  # noqa: E731
        nbytes, sample = 8 << 24, "dot over 2^24 fp32 pairs, full size"
    elif base in ("gemv", "gemv_xprivate", "gemv_literal"):
        A, x = _seeded((8192, 8192), 3, -1.0, 1.0), _seeded(8192, 4, -1.0, 1.0)
        fn = lib.gemv
        fn.argtypes = [vp, vp, vp]
        call = lambda: fn(out.ctypes.data, A.ctypes.data, x.ctypes.data)  # noqa: E731
        nbytes, sample = 4 * (8192 * 8192 + 2 * 8192), "gemv 8192x8192 fp32, full size"
    elif base == "scal":
        n = (1 << 26) // 1024
        xs = _seeded(1 << 26, 7, -1.0, 1.0)
        ys = np.zeros(1 << 26, np.float32)
        fn = lib.scal
        fn.argtypes = [vp, ctypes.c_float, vp, ci]
        call = lambda: fn(ys.ctypes.data, 1.5, xs.ctypes.data, n)  # noqa: E731
        nbytes, sample = 8 << 26, "scal (y = alpha x) over 2^26 fp32, full size (read + write)"
    elif base == "mm":
        A, B = _seeded((4096, 4096), 5, -1.0, 1.0), _seeded((4096, 4096), 6, -1.0, 1.0)
        Bt = np.ascontiguousarray(B.T)
        big = np.zeros(4096 * 4096, np.float32)
        fn = lib.mm_bt
        fn.argtypes = [vp, vp, vp]
        call = lambda: fn(big.ctypes.data, A.ctypes.data, Bt.ctypes.data)  # noqa: E731
        flops = 2 * 4096 ** 3
        sample = "mm 4096^3 fp32, full size, B passed pre-transposed"
        min_seconds, max_reps = 0.0, 2
        steps = None if steps is None else min(steps, 2)  # ~5 s per call on 16 threads
        nbytes = None
    else:
        return None
    prog = REF_STRATEGY.get(base, ("", ""))[1]
    for _ in range(max(1, warmup if nbytes is not None else min(warmup, 1))):
        call()
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
        if steps is not None and len(times) >= steps:
            break
        if steps is None and (time.perf_counter() - t_start > min_seconds or len(times) >= max_reps):
            break
    best = min(times)
    how = (f"reference c-openmp emission of {prog} (gcc -O3 -march={lib.march} -fopenmp, "
           f"OMP threads = {int(lib.ref_threads())})")
    common = {"cores": int(lib.ref_threads()), "cpu_model": _cpu_model(), "kind": "reference",
              "march": lib.march, "ms_per_call": round(1e3 * statistics.median(times), 4)}
    if nbytes is None:  # mm: flop rate
        return dict(common, value=round(flops / statistics.median(times) / 1e9, 3), unit="GFLOP/s",
                    sample=f"{sample}{note}; {how}, median of {len(times)} calls")
    return dict(common, value=round(nbytes / statistics.median(times) / 1e9, 3), unit="GB/s",
                sample=f"{sample}{note}; {how}, median of {len(times)} calls, "
                       f"best {nbytes / best / 1e9:.1f} GB/s")


def reference_arm(args):
    """`--impl reference`: the reference's own CPU implementation of the
    workload (oracle/_ref, its c-openmp emission, all host threads), on the
    same metric, unit and workload as our arm; each step one call."""
    r = cpu_reference(args.workload, steps=args.steps, warmup=args.warmup)
    unit = "GFLOP/s" if args.workload.startswith("mm") else "GB/s"
    wl, strat = REF_STRATEGY.get(args.workload, (args.workload, "none"))
    line = {"impl": "reference", "metric": METRIC, "unit": unit, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wl, "strategy": strat,
                       "reference_path": "the reference's c-openmp emission of the program on the "
                                         "host cores (oracle/_ref, built by oracle/build_ref.py)"}}
    if r is None:
        line["unavailable"] = _cpu_unavailable(args.workload, 1)
    else:
        line.update({"value": r["value"], "ms_per_step": r["ms_per_call"],
                     "cpu_baseline": _cpu_fields(r),
                     "e2e": {"value": r["value"], "unit": r["unit"], "h2d_bytes_per_step": 0,
                             "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="asum")
    ap.add_argument("--no-suite", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-chain", action="store_true",
                    help="launch the steps without chaining them (programmatic dependent launch)")
    ap.add_argument("--traffic", choices=["live", "committed"], default="live",
                    help="roofline.traffic from an ncu run of the same workload made now "
                         "(after the timed regions), or from profiles/ncu_traffic.json")
    ap.add_argument("--traffic-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--combine", choices=["peer", "nccl"], default="peer",
                    help="cross-GPU combine of the partial sums (N > 1): inside the kernel over "
                         "NVLink (peer) or a 4-byte ncclAllReduce after it")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.traffic_child:
        return traffic_child(args.workload)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        # `python bench.py --gpus N` without a launcher: one process per GPU
        # under torchrun, this same command line in every rank
        return _spawn_ranks(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        # the reference's CPU path: rank 0 alone, on the host cores; other
        # ranks of a torchrun launch exit without work
        return reference_arm(args) if rank == 0 else 0
    if args.impl == "ours" and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
              f"(torchrun --nproc-per-node {args.gpus}) or drop the launcher", file=sys.stderr)
        return 2
    # plumbing check on a one-GPU box: every rank on GPU 0, gloo for the host
    # side (the fused peer combine still runs GPU to GPU through CUDA IPC);
    # the timings of ranks sharing a GPU are not scaling numbers
    share = os.environ.get("DPIA_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
        args.combine = "peer"
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours" and not share and torch.cuda.device_count() < world:
            print(f"bench.py: {world} ranks need {world} GPUs, {torch.cuda.device_count()} visible "
                  "(DPIA_BENCH_SHARE_GPU=1 runs every rank on GPU 0 as a plumbing check)",
                  file=sys.stderr)
            return 3
        if args.impl == "ours":
            torch.cuda.set_device(local)
        dist.init_process_group("gloo" if (share or args.impl == "reference") else "nccl")
        if args.impl == "ours" and args.combine == "peer":
            # collective capability probe: every rank maps every peer's
            # mailbox (CUDA IPC + NVLink P2P); if any rank cannot, all ranks
            # fall back to the NCCL combine together
            ok = 1
            try:
                from paper_1710_08332_b200.peer import PeerGroup, torch_allgather
                RT.init(local)
                PeerGroup(local, rank, world, 1, torch_allgather).close()
            except Exception as e:  # noqa: BLE001
                print(f"rank {rank}: peer combine unavailable ({e}); using NCCL", file=sys.stderr)
                ok = 0
            if not int(_allreduce(dist, ok, dist.ReduceOp.MIN, local, share)):
                args.combine = "nccl"
        if args.impl == "ours" and not share:
            # NCCL is always set up at N > 1: it is the combine of
            # --combine nccl, the fallback of the peer combine and the
            # cross-check of its totals
            _nccl_init(dist, local, world, rank)

    device = local
    RT.init(device)
    stream = RT.Stream(device)
    peak, peak_src = peaks()

    def measure(workload, steps, warmup, with_e2e):
        cfg, exe, inputs, prepare, prog = make_workload(workload, device, rank, world, args.combine)
        prepare(stream)
        stream.sync()
        check = None
        if exe.peer is not None and world > 1:
            # the fused combine's total against the partials it combines
            # (bit-exact rank-order sum) and against NCCL; on any
            # disagreement or peer timeout every rank falls back to NCCL
            check = _combine_check(exe, prog, stream, dist, share, rank, local)
            if not check["agree_all_ranks"]:
                if share:
                    raise SystemExit(f"peer combine disagrees: {check}")
                exe.peer.close()
                cfg, exe, inputs, prepare, prog = make_workload(workload, device, rank, world, "nccl")
                prepare(stream)
                stream.sync()
                check["combine_used"] = "nccl (fallback)"
            else:
                check["combine_used"] = "peer"
        allreduce = None
        reduces = workload in ("asum", "dot", "dot_literal") or workload.startswith("scaleout")
        if world > 1 and exe.peer is None and reduces:
            # the NCCL combine (--combine nccl, or the fallback of the peer
            # combine); gemv / mm / scal shard with no collective at all
            if share:
                raise SystemExit("internal: ranks sharing one GPU have no NCCL combine")
            outbuf = exe.buffers["out"]

            def allreduce(s):  # NCCL sum of the per-rank partial, on our stream
                RT.lib().dpia_nccl_allreduce(outbuf.ptr, 1, 0, s.handle)
        rot = Rotation(exe, cfg.bytes, stream, chain=not args.no_chain)
        for i in range(warmup):
            rot.launch(i, stream)
            if allreduce:
                allreduce(stream)
        stream.sync()
        if dist is not None:
            dist.barrier()
        RT.lib().dpia_device_sync(device)
        # keep the GPU under the same load for ~0.6 s so nvidia-smi's 100 ms
        # sampler sees the clocks of the timed region; every rank does the
        # same number of launches (the fused peer combine pairs them up)
        t_b = time.perf_counter()
        rot.run(stream, 20, allreduce)
        batches = max(1, int(0.6 / max(time.perf_counter() - t_b, 1e-4)))
        if dist is not None:
            import torch
            batches = int(_allreduce(dist, batches, dist.ReduceOp.MAX, local, share))
        with Clocks(device) as clk:
            for _ in range(batches):
                rot.run(stream, 20, allreduce)
            if dist is not None:
                dist.barrier()
            t0 = time.perf_counter()
            # the timed region: `steps` steps back to back, one event pair
            mean_ms = mean_ms_local = rot.run(stream, steps, allreduce)
            wall = time.perf_counter() - t0
        RT.lib().dpia_device_sync(device)
        if dist is not None:
            import torch
            mean_ms = float(_allreduce(dist, mean_ms, dist.ReduceOp.MAX, local, share))
            dist.barrier()
        if allreduce is None:
            kmean = mean_ms_local             # a step is exactly the program's kernel(s)
        else:                                 # the dominant kernel alone, without the combine
            kmean = rot.run(stream, steps)
        # the round-1 method beside it: each launch alone after an L2 scrub
        iso = run_isolated(exe, stream, steps, allreduce)
        iso_ms = statistics.mean(iso)
        # and the steady state without chaining (the same rotation, each step
        # launched after the previous one completed)
        unch_ms = None
        if rot.chain:
            rot.chain = False
            rot.run(stream, 3, allreduce)
            unch_ms = rot.run(stream, steps, allreduce)
            rot.chain = True
        rot_desc = {"input_sets": rot.R, "l2_bytes": l2_bytes(device),
                    "bytes_per_step": cfg.bytes, "chained": rot.chain}
        rot.free()
        if workload.startswith("mm"):
            fp32 = fp32_peak(device)
            achieved = cfg.flops / (kmean * 1e-3) / 1e12
            value = world * cfg.flops / (mean_ms * 1e-3) / 1e9
            roof = {"bound": "fp32", "achieved": round(achieved, 2), "peak": round(fp32[0], 2),
                    "unit": "TFLOP/s", "frac": round(achieved / fp32[0], 4),
                    "traffic": None, "peak_source": fp32[1],
                    "algorithmic_flops_per_launch": cfg.flops, "kernel_ms": round(kmean, 5)}
            meas, inner = ffma_peak(device, stream)
            roof["measured_ffma2_peak"] = meas
            roof["frac_of_measured_ffma2_peak"] = round(achieved / meas, 4)
            # the strategy's own k-step (shared fragment loads + FFMA2) with
            # no global staging and no barrier, at mm's occupancy
            roof["inner_loop_ceiling"] = inner
            roof["frac_of_inner_loop_ceiling"] = round(achieved / inner, 4)
        else:
            achieved = cfg.bytes / (kmean * 1e-3) / 1e9
            value = world * cfg.bytes / (mean_ms * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                    "unit": "GB/s", "frac": round(achieved / peak, 4),
                    "traffic": None,
                    "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
                    "algorithmic_bytes_per_launch": cfg.bytes, "kernel_ms": round(kmean, 5)}
            # context for fractions above 1 of the copy peak (reads stream
            # faster than a read+write copy): the part's nominal HBM3e rate
            roof["nominal_gbs"] = NOMINAL_HBM_GBS
            roof["frac_of_nominal"] = round(achieved / NOMINAL_HBM_GBS, 4)
            if workload in ("asum", "dot", "gemv"):
                sol = read_sol(device, cfg.bytes, stream)
                roof["size_matched_read_sol_gbs"] = sol["steady"]
                roof["frac_of_size_matched_sol"] = round(achieved / sol["steady"], 4)
        if world == 1:
            # DRAM traffic of the same kernel, measured after the timed region
            if args.traffic == "live":
                t, tsrc = live_traffic(workload, exe.kernel_names()[0])
            else:
                t, tsrc = ncu_traffic(workload), "committed ncu capture (profiles/ncu_traffic.json)"
            roof["traffic"] = t
            roof["traffic_source"] = tsrc
            if t:
                roof["traffic_over_algorithmic"] = round(t / cfg.bytes, 4)
        work = cfg.flops if workload.startswith("mm") else cfg.bytes
        roof["isolated"] = {
            "ms_per_launch": round(iso_ms, 5),
            "achieved": round(work / (iso_ms * 1e-3) / (1e12 if workload.startswith("mm") else 1e9),
                              2 if workload.startswith("mm") else 1),
            "frac": round(work / (iso_ms * 1e-3) / (1e12 if workload.startswith("mm") else 1e9) / roof["peak"], 4),
            "method": "each launch alone between its own event pair, after an L2 scrub (round-1 "
                      "timing): adds the event pair and an unhidden launch, ~6 us "
                      "(profiles/r01f_tailexp4.txt)"}
        if workload in ("asum", "dot", "gemv"):
            roof["isolated"]["size_matched_read_sol_gbs"] = read_sol(device, cfg.bytes, stream)["isolated"]
        if unch_ms:
            ua = work / (unch_ms * 1e-3) / (1e12 if workload.startswith("mm") else 1e9)
            roof["unchained"] = {
                "ms_per_step": round(unch_ms, 5), "achieved": round(ua, 2 if workload.startswith("mm") else 1),
                "frac": round(ua / roof["peak"], 4),
                "method": "the same rotation back to back, each step launched without chaining "
                          "(bench.py --no-chain)"}
        res = {"cfg": cfg, "exe": exe, "mean_ms": mean_ms, "wall_s": wall, "clocks": clk.summary(),
               "value": value, "roofline": roof, "rotation": rot_desc}
        if check is not None:
            res["combine_check"] = check
        if world > 1:
            res["ranks"] = _rank_info(dist, rank, device, mean_ms_local, share)
        if with_e2e and inputs is not None:
            e2e_ms, h2d, d2h = e2e_measure(exe, inputs, stream, min(steps, 5))
            if dist is not None:   # whole job: every rank's bytes over the slowest rank's time
                e2e_ms = float(_allreduce(dist, e2e_ms, dist.ReduceOp.MAX, local, share))
            work, unit = (cfg.flops, "GFLOP/s") if workload.startswith("mm") else (cfg.bytes, "GB/s")
            res["e2e"] = {"value": round(world * work / (e2e_ms * 1e-3) / 1e9, 3), "unit": unit,
                          "h2d_link_gbs": _LINK_GBS,
                          "h2d_link_note": "pinned H2D of the same input bytes alone, measured in the "
                                           "same run: the ceiling of a streaming e2e (one GPU's link)",
                          "h2d_bytes_per_step": world * h2d, "d2h_bytes_per_step": world * d2h,
                          "ms_per_step": round(e2e_ms, 4),
                          "path": "Executable.run (public API): pinned H2D + kernels + D2H + stream sync"
                                  + (f"; {world} ranks, each its own inputs over its own link, max over "
                                     "ranks" if world > 1 else "")}
        if with_e2e and workload == "scal" and world == 1:
            # read + write: the public row pipeline overlaps the H2D of block
            # i+1 and the D2H of block i-1 with block i's kernel
            pms, ph2d, pd2h = e2e_pipelined_scal(inputs, stream, min(steps, 5))
            res["e2e_unpipelined"] = res.get("e2e")
            res["e2e"] = {"value": round(cfg.bytes / (pms * 1e-3) / 1e9, 3), "unit": "GB/s",
                          "h2d_bytes_per_step": ph2d, "d2h_bytes_per_step": pd2h,
                          "ms_per_step": round(pms, 4),
                          "path": "pipeline.scal_pipeline(8 blocks).run (public API): pinned H2D of x "
                                  "blocks, block kernels, D2H of y blocks, overlapped on three streams "
                                  "(PCIe carries both directions at once), stream sync"}
        if with_e2e and workload == "mm" and world == 1:
            # compute-bound: the public row pipeline overlaps the copies with
            # the chunk kernels (pipeline.mm_pipeline); the plain
            # Executable.run number stays beside it
            rms, rh2d, rd2h = e2e_pipelined_mm(inputs, stream, min(steps, 5))
            pms, ph2d, pd2h = e2e_pipelined_mm(inputs, stream, min(steps, 5), tiles=(4, 4, 8))
            res["e2e_unpipelined"] = res.get("e2e")
            res["e2e_row_pipeline"] = {
                "value": round(cfg.flops / (rms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                "h2d_bytes_per_step": rh2d, "d2h_bytes_per_step": rd2h, "ms_per_step": round(rms, 4),
                "path": "pipeline.mm_pipeline(4 row chunks).run (public API): pinned H2D of B and A row "
                        "chunks, chunk kernels, D2H of C row chunks, overlapped on three streams"}
            res["e2e"] = {"value": round(cfg.flops / (pms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                          "h2d_bytes_per_step": ph2d, "d2h_bytes_per_step": pd2h,
                          "ms_per_step": round(pms, 4),
                          "path": "pipeline.mm_tile_pipeline(4x4 tiles, 8 compute streams).run (public "
                                  "API): pinned H2D of A row blocks and pitched B column panels "
                                  "interleaved, each 1024x1024 C tile's kernel as soon as its two "
                                  "operands are in, pitched D2H of C tiles, stream sync"}
        if exe.peer is not None:
            exe.peer.check()      # no rank timed out waiting for a peer's partial
        return res

    head = measure(args.workload, args.steps, args.warmup, with_e2e=True)
    suite = {}
    # N = 1: every benchmark program; N > 1: the sharded reductions of
    # BASELINE config 5 (2^31 in total, strong scaling) beside the weak-scaled
    # headline -- gemv / mm / scal would only replicate (no exchange step)
    names = (("dot", "dot_literal", "asum", "asum_proxy", "gemv", "gemv_xprivate", "gemv_literal", "mm",
              "mm_tma", "scal", "scal_literal",
              "scaleout_asum", "scaleout_dot") if world == 1 else ("scaleout_asum", "scaleout_dot"))
    if not args.no_suite:
        for w in names:
            if w == args.workload:
                continue
            r = measure(w, min(args.steps, 20), 3, with_e2e=True)
            suite[w] = {"value": round(r["value"], 1), "unit": "GFLOP/s" if w.startswith("mm") else "GB/s",
                        "ms_per_step": round(r["mean_ms"], 5), "roofline": r["roofline"],
                        "scaling": "strong" if w.startswith("scaleout") else "weak",
                        "e2e": r.get("e2e"), "clocks": r["clocks"],
                        "config": dict(_cfg_desc(r["cfg"], world, args.combine),
                                       input_sets=r["rotation"]["input_sets"]),
                        "kernels": r["exe"].kernel_names()}
            if r.get("e2e") is None and w.startswith("scaleout"):
                suite[w]["e2e_note"] = ("config 5 generates its inputs on device by a counter hash "
                                        "(BASELINE.json configs[4]); no host data moves")
            for extra in ("e2e_unpipelined", "e2e_row_pipeline", "combine_check", "ranks"):
                if r.get(extra):
                    suite[w][extra] = r[extra]
            if not args.no_cpu and rank == 0:
                c = cpu_reference(w) if world == 1 else None
                suite[w]["cpu_baseline"] = (_cpu_fields(c) if c else
                                            {"unavailable": _cpu_unavailable(w, world)})
            r["exe"] = None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_reference(args.workload)
    if rank != 0:
        return 0
    cfg, exe = head["cfg"], head["exe"]
    strong = args.workload.startswith("scaleout")
    line = {"metric": METRIC, "value": round(head["value"], 2),
            "unit": "GFLOP/s" if args.workload.startswith("mm") else "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(head["mean_ms"], 5),
            "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "f32",
            "data": ("synthetic (device-side counter hash, per-shard global offsets)" if strong
                     else "synthetic (numpy default_rng uniform, resident in HBM)"),
            "config": dict(_cfg_desc(cfg, world, args.combine), input_sets=head["rotation"]["input_sets"],
                           **({"combine": args.combine} if world > 1 else {}),
                           **({"shared_gpu": "plumbing check: all ranks on GPU 0 (not a scaling number)"}
                              if share and world > 1 else {})),
            "roofline": head["roofline"], "e2e": head.get("e2e"), "clocks": head["clocks"],
            "gpu_launches": args.steps * len(exe.sig.kernels),
            "gpu_launches_breakdown": {"emitted program kernels (inside the timed events)":
                                       args.steps * len(exe.sig.kernels)},
            "kernels": exe.kernel_names(),
            "cpu_baseline": (_cpu_fields(cpu) if cpu else
                             {"unavailable": _cpu_unavailable(args.workload, world, args.no_cpu)}),
            "suite": suite}
    for extra in ("combine_check", "ranks"):
        if head.get(extra):
            line[extra] = head[extra]
    print(json.dumps(line), flush=True)
    return 0


def _cpu_fields(c):
    return {k: c[k] for k in ("value", "unit", "cores", "cpu_model", "kind", "sample", "march") if k in c}


def _cpu_unavailable(workload, world, skipped=False):
    if skipped:
        return "not timed in this run (--no-cpu)"
    if world > 1:
        return "the CPU baseline is timed at N = 1 only (rank 0, host cores); see the N = 1 line"
    if ref_lib() is None:
        return "oracle/_ref/libref_cpu.so not built (needs /root/reference at build time)"
    return f"the reference's c-openmp path has no program for workload {workload!r}"


def _spawn_ranks(n):
    """Re-run this command line as n ranks under torchrun (one process per
    GPU, rendezvous on 127.0.0.1); returns torchrun's exit code.  Rank 0
    prints the JSON line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def _nccl_init(dist, local, world, rank):
    uid = ctypes.create_string_buffer(128)
    if rank == 0:
        RT.lib().dpia_nccl_unique_id(uid)
    obj = [bytes(uid.raw)]
    dist.broadcast_object_list(obj, src=0)
    RT.init(local)
    RT.lib().dpia_nccl_init(local, world, rank, obj[0])


def _combine_check(exe, prog, stream, dist, share, rank, local):
    """peer.cross_check on every rank, plus the NCCL sum of the same
    partials when NCCL is up; agreement is decided over all ranks."""
    from paper_1710_08332_b200.peer import PeerError, cross_check, local_twin, torch_allgather
    try:
        ev = cross_check(exe, local_twin(exe, prog), stream, torch_allgather)
        ok = ev["bit_exact"]
    except (PeerError, RT.DpiaRuntimeError) as e:
        ev, ok = {"error": str(e)}, False
    if ok and not share:
        buf = RT.DeviceBuffer(16, exe.device)
        buf.upload(np.array([ev["partials"][rank], 0, 0, 0], np.float32))
        RT.lib().dpia_nccl_allreduce(buf.ptr, 1, 0, stream.handle)
        stream.sync()
        v = np.zeros(4, np.float32)
        buf.download(v)
        buf.free()
        ev["nccl_allreduce"] = float(v[0])
        ev["nccl_rel_diff"] = abs(float(v[0]) - ev["peer_total"][0]) / max(ev["abs_sum"], 1e-30)
        ok = ev["nccl_rel_diff"] <= 1e-6
    ev["agree_all_ranks"] = bool(int(_allreduce(dist, int(ok), dist.ReduceOp.MIN, local, share)))
    return ev


def _rank_info(dist, rank, device, ms, share):
    """Per-rank evidence: device, PCI bus, the runtime library this process
    loaded, and its own mean step time (the line reports the max)."""
    import torch
    props = torch.cuda.get_device_properties(device)
    info = {"rank": rank, "device": device, "ms_per_step": round(ms, 5), "gpu": props.name,
            "pci_bus_id": getattr(props, "pci_bus_id", None), "shared_gpu": bool(share),
            "lib": _loaded_lib()}
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, info)
    return out


def _loaded_lib():
    try:
        with open("/proc/self/maps") as f:
            for ln in f:
                if "libdpia_rt" in ln:
                    return os.path.relpath(ln.split()[-1], ROOT)
    except OSError:
        pass
    return None


def _allreduce(dist, value, op, local, share):
    """Max/min of a host number over the ranks (CPU tensor under gloo)."""
    import torch
    t = torch.tensor([value], device="cpu" if share else f"cuda:{local}")
    dist.all_reduce(t, op=op)
    return t.item()


WORKLOADS = {
    "asum": ("asum N=2^26 fp32", "asVector4 + mapWorkgroup/mapLocal + reduceSeq(abs) + reduceLocal, "
             "grid combine fused as a last-block tail"),
    "dot": ("dot N=2^24 fp32", "asVector4 + mapWorkgroup/mapLocal/reduceSeq + reduceLocal, grid "
            "combine fused as a last-block tail"),
    "dot_literal": ("dot N=2^24 fp32", "BASELINE config 1 as the reference states it "
                    "(oracle/ref_programs/dot.dpia): mapGlobal over 1024-element chunks, reduceSeq "
                    "per chunk, top-level sequential reduce of the 16384 partials"),
    "gemv": ("gemv 8192x8192 fp32", "BASELINE config 3: row per work-group, x staged with toLocal "
             "(shared memory), reduceSeq over vec4 column slices, reduceLocal per row"),
    "gemv_xprivate": ("gemv 8192x8192 fp32", "row per work-group, x staged toPrivate in the "
                      "work-items' column layout (registers), reduceSeq + reduceLocal per row"),
    "gemv_literal": ("gemv 8192x8192 fp32", "BASELINE config 3 as the reference states it "
                     "(oracle/ref_programs/gemv.dpia): row per work-group, x toLocal, each work-item "
                     "folds its own 32-element piece, partial sums toLocal, one work-item folds them"),
    "scal": ("scal N=2^26 fp32 (read + write)", "grid-stride mapGlobal over vec4"),
    "scal_literal": ("scal N=2^26 fp32 (read + write)", "the paper's scal as the reference states it "
                     "(oracle/ref_programs/scal.dpia): mapGlobal over 1024-element chunks, each work-item "
                     "scaling its own chunk (TMA row reads, vector stores)"),
    "mm": ("mm 4096^3 fp32 (FFMA, no tensor cores)", "128x128 tiles, 8x8 register tiles, toLocal "
           "k-tiles of 16, FFMA2"),
    "asum_proxy": ("asum proxy N=2^26 fp32 (the reference arm's program: sum, no abs)",
                   "oracle/ref_programs/asum_proxy.dpia as the reference states it: mapGlobal over "
                   "1024-element chunks, reduceSeq per chunk, top-level sequential reduce of the 65536 "
                   "partials (TMA row folds, streaming tail over 16 launch slots)"),
    "mm_tma": ("mm 4096^3 fp32 (FFMA, no tensor cores)", "the mm strategy with B's toLocal k-tile "
               "staged by TMA tensor copies (cp.async.bulk.tensor.2d, 3 rotating slices, mbarrier); "
               "A's transposed k-tile by register prefetch"),
}


def _cfg_desc(cfg, world=1, combine="nccl"):
    if cfg.name.startswith("scaleout"):
        kind = "dot" if cfg.name.endswith("dot") else "asum"
        return {"workload": f"{kind} scale-out N=2^31 fp32 total",
                "strategy": f"{world} shard(s) of 2^31/{world}, partials combined "
                            + ("inside the kernel over NVLink (peer)" if combine == "peer" and world > 1
                               else "by a 4-byte NCCL all-reduce" if world > 1 else "(one shard)"),
                "sigma_per_rank": cfg.sigma,
                "launch": list(cfg.launch), "l2": L2_NOTE}
    wl, strat = WORKLOADS[cfg.name]
    return {"workload": wl, "strategy": strat, "sigma": cfg.sigma, "launch": list(cfg.launch),
            "l2": L2_NOTE}


L2_NOTE = ("inputs larger than L2: the steps rotate through R device copies of the inputs (and of "
           "outputs > 1 MiB) with R x step bytes >= 3 x L2, so each step's data was evicted by the "
           "steps since its last use; the steps run back to back between one event pair (no scrub), "
           "each chained behind the previous one (Executable.launch(chain=True): programmatic "
           "dependent launch; the step streams its inputs while the previous step drains and waits "
           "for it before touching shared memory); roofline.isolated is the per-launch scrubbed "
           "timing")


if __name__ == "__main__":
    sys.exit(main())
