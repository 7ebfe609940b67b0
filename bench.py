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
from paper_1710_08332_b200.bench_programs import (asum_config, dot_config,  # noqa: E402
                                                  gemv_config, mm_config, scal_config)

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


def read_sol(device, nbytes, stream):
    """Size-matched speed of light: a hand-written minimal CUDA streaming-read
    kernel (tools/readsol.py; measurement infrastructure, not product) timed
    exactly like the benchmark steps on `nbytes` of HBM."""
    if nbytes in _SOL_CACHE:
        return _SOL_CACHE[nbytes]
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from readsol import SRC
    mod = RT.Module(RT.get_cubin(SRC), device)
    fn = mod.function("readsum")
    buf, out = RT.DeviceBuffer(nbytes, device), RT.DeviceBuffer(16, device)
    buf.zero(stream)
    args = [RT.C.c_uint64(buf.ptr), RT.C.c_longlong(nbytes // 16), RT.C.c_uint64(out.ptr)]
    ts = []
    for it in range(13):
        RT.lib().dpia_l2_flush(device, stream.handle)
        e0, e1 = RT.Event(device), RT.Event(device)
        e0.record(stream)
        RT.launch(fn, device, (296, 1), (1024, 1), 0, args, stream)
        e1.record(stream)
        stream.sync()
        if it >= 3:
            ts.append(e0.elapsed_ms(e1))
    buf.free()
    out.free()
    _SOL_CACHE[nbytes] = round(nbytes / statistics.median(ts) / 1e6, 1)
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
    """Per-launch DRAM bytes of the dominant kernel from a committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(workload)
    except (OSError, ValueError):
        return None


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
    """(config, executable, host inputs or None, prepare(stream))."""
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
        return cfg, run.exe, None, run.fill_inputs
    if name == "asum":
        cfg = asum_config()
        inputs = {"xs": _seeded(1 << 26, 2 + 1000 * rank, -1.0, 1.0)}
    elif name == "dot":
        cfg = dot_config()
        inputs = {"xs": _seeded(1 << 24, 0 + 1000 * rank, 0.0, 1.0),
                  "ys": _seeded(1 << 24, 1 + 1000 * rank, 0.0, 1.0)}
    elif name == "gemv":
        cfg = gemv_config()
        inputs = {"A": _seeded((8192, 8192), 3, -1.0, 1.0), "x": _seeded(8192, 4, -1.0, 1.0)}
    elif name == "scal":
        cfg = scal_config()
        inputs = {"alpha": np.full(4, 1.5, np.float32), "xs": _seeded(1 << 26, 7, -1.0, 1.0)}
    elif name == "mm":
        cfg = mm_config()
        inputs = {"A": _seeded((4096, 4096), 5, -1.0, 1.0), "B": _seeded((4096, 4096), 6, -1.0, 1.0)}
    else:
        raise SystemExit(f"unknown workload {name}")
    prog = compile_program(cfg.text, name=name)
    peer = None
    if allgather is not None and name in ("asum", "dot"):
        from paper_1710_08332_b200.peer import PeerGroup
        peer = PeerGroup(device, rank, world, 1, allgather)
    exe = executable(prog, cfg.launch, cfg.sigma, float_mode=True, device=device, peer=peer)

    def prepare(stream):
        for n, v in inputs.items():
            exe.upload(n, v, stream)
    return cfg, exe, inputs, prepare


def _seeded(shape, seed, lo, hi):
    return np.random.default_rng(seed).uniform(lo, hi, size=shape).astype(np.float32)


def time_steps(exe, stream, steps, warmup, flush=True, allreduce=None):
    dev = exe.device
    ev = [(RT.Event(dev), RT.Event(dev)) for _ in range(steps)]
    for _ in range(warmup):
        if flush:
            RT.lib().dpia_l2_flush(dev, stream.handle)
        exe.launch(stream)
        if allreduce:
            allreduce(stream)
    stream.sync()
    return ev


def run_timed(exe, stream, steps, flush=True, allreduce=None):
    dev = exe.device
    ev = [(RT.Event(dev), RT.Event(dev)) for _ in range(steps)]
    for e0, e1 in ev:
        if flush:
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


def ref_lib():
    import ctypes
    path = os.path.join(ROOT, "oracle", "_ref", "libref_cpu.so")
    if not os.path.exists(path):
        return None
    lib = ctypes.CDLL(path)
    return lib


def cpu_reference(workload, min_seconds=2.0, max_reps=200, steps=None, warmup=1):
    """Time the reference's own CPU path (its c-openmp emission of the same
    strategy, compiled by oracle/build_ref.py) on all host threads."""
    import ctypes
    lib = ref_lib()
    if lib is None:
        return None
    vp, ci = ctypes.c_void_p, ctypes.c_int
    out = np.zeros(8192, np.float32)
    if workload == "asum":
        n = (1 << 26) // 1024
        xs = _seeded(1 << 26, 2, -1.0, 1.0)
        fn = lib.asum_proxy
        fn.argtypes = [vp, vp, ci]
        call = lambda: fn(out.ctypes.data, xs.ctypes.data, n)  # noqa: E731
        nbytes, sample = 4 << 26, "asum proxy (sum; the reference has no abs) over 2^26 fp32, full size"
    elif workload == "dot":
        n = (1 << 24) // 1024
        xs, ys = _seeded(1 << 24, 0, 0.0, 1.0), _seeded(1 << 24, 1, 0.0, 1.0)
        fn = lib.dot
        fn.argtypes = [vp, vp, vp, ci]
        call = lambda: fn(out.ctypes.data, xs.ctypes.data, ys.ctypes.data, n)  # noqa: E731
        nbytes, sample = 8 << 24, "dot over 2^24 fp32 pairs, full size"
    elif workload == "gemv":
        A, x = _seeded((8192, 8192), 3, -1.0, 1.0), _seeded(8192, 4, -1.0, 1.0)
        fn = lib.gemv
        fn.argtypes = [vp, vp, vp]
        call = lambda: fn(out.ctypes.data, A.ctypes.data, x.ctypes.data)  # noqa: E731
        nbytes, sample = 4 * (8192 * 8192 + 2 * 8192), "gemv 8192x8192 fp32, full size"
    elif workload == "scal":
        n = (1 << 26) // 1024
        xs = _seeded(1 << 26, 7, -1.0, 1.0)
        ys = np.zeros(1 << 26, np.float32)
        fn = lib.scal
        fn.argtypes = [vp, ctypes.c_float, vp, ci]
        call = lambda: fn(ys.ctypes.data, 1.5, xs.ctypes.data, n)  # noqa: E731
        nbytes, sample = 8 << 26, "scal (y = alpha x) over 2^26 fp32, full size (read + write)"
    elif workload == "mm":
        A, B = _seeded((4096, 4096), 5, -1.0, 1.0), _seeded((4096, 4096), 6, -1.0, 1.0)
        Bt = np.ascontiguousarray(B.T)
        big = np.zeros(4096 * 4096, np.float32)
        fn = lib.mm_bt
        fn.argtypes = [vp, vp, vp]
        call = lambda: fn(big.ctypes.data, A.ctypes.data, Bt.ctypes.data)  # noqa: E731
        flops = 2 * 4096 ** 3
        sample = ("mm 4096^3 fp32, full size, B passed pre-transposed (the reference language has "
                  "no transpose)")
        min_seconds, max_reps = 0.0, 2
        steps = None if steps is None else min(steps, 2)  # ~5 s per call on 16 threads
        nbytes = None
    else:
        return None
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
    if nbytes is None:  # mm: flop rate
        return {"value": round(flops / statistics.median(times) / 1e9, 3), "unit": "GFLOP/s",
                "cores": int(lib.ref_threads()), "cpu_model": _cpu_model(), "kind": "reference",
                "sample": f"{sample}; reference c-openmp emission (gcc -O3 -fopenmp), "
                          f"median of {len(times)} calls",
                "ms_per_call": round(1e3 * statistics.median(times), 4)}
    return {"value": round(nbytes / statistics.median(times) / 1e9, 3), "unit": "GB/s",
            "cores": int(lib.ref_threads()), "cpu_model": _cpu_model(), "kind": "reference",
            "sample": f"{sample}; reference c-openmp emission (gcc -O3 -fopenmp), "
                      f"median of {len(times)} calls, best {nbytes / best / 1e9:.1f} GB/s",
            "ms_per_call": round(1e3 * statistics.median(times), 4)}


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
    ap.add_argument("--combine", choices=["peer", "nccl"], default="peer",
                    help="cross-GPU combine of the partial sums (N > 1): inside the kernel over "
                         "NVLink (peer) or a 4-byte ncclAllReduce after it")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
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
        torch.cuda.set_device(local)
        dist.init_process_group("gloo" if share else "nccl")
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
        if args.impl == "ours" and args.combine == "nccl":
            import ctypes
            uid = ctypes.create_string_buffer(128)
            if rank == 0:
                RT.lib().dpia_nccl_unique_id(uid)
            obj = [bytes(uid.raw)]
            dist.broadcast_object_list(obj, src=0)
            RT.init(local)
            RT.lib().dpia_nccl_init(local, world, rank, obj[0])

    if args.impl == "reference":
        if rank != 0:
            return
        r = cpu_reference(args.workload, steps=args.steps, warmup=args.warmup)
        unit = "GFLOP/s" if args.workload == "mm" else "GB/s"
        from paper_1710_08332_b200.bench_programs import CONFIGS
        cfg_line = (dict({k: v for k, v in _cfg_desc(CONFIGS[args.workload]()).items() if k != "l2"},
                         reference_path="the reference's c-openmp emission of the same workload on the "
                                        "host cores (oracle/_ref)")
                    if args.workload in CONFIGS else
                    {"workload": f"{args.workload} (reference c-openmp path on host cores)"})
        line = {"impl": "reference", "metric": METRIC, "unit": unit, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": cfg_line}
        if r is None:
            why = ("oracle/_ref/libref_cpu.so not built (needs /root/reference at build)" if ref_lib() is None
                   else f"the reference's c-openmp path has no program for workload {args.workload!r}")
            line.update({"unavailable": why})
        else:
            line.update({"value": r["value"], "ms_per_step": r["ms_per_call"],
                         "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "cpu_model", "kind", "sample")},
                         "e2e": {"value": r["value"], "unit": r["unit"], "h2d_bytes_per_step": 0,
                                 "d2h_bytes_per_step": 0}})
        print(json.dumps(line), flush=True)
        return

    device = local
    RT.init(device)
    stream = RT.Stream(device)
    peak, peak_src = peaks()

    def measure(workload, steps, warmup, with_e2e):
        cfg, exe, inputs, prepare = make_workload(workload, device, rank, world, args.combine)
        prepare(stream)
        stream.sync()
        allreduce = None
        reduces = workload in ("asum", "dot") or workload.startswith("scaleout")
        if world > 1 and exe.peer is None and reduces:
            # gemv / mm / scal shard with no collective (independent rows)
            if args.combine != "nccl":
                raise SystemExit("internal: a reduction without the peer combine needs --combine nccl")
            outbuf = exe.buffers["out"]

            def allreduce(s):  # NCCL sum of the per-rank partial, on our stream
                RT.lib().dpia_nccl_allreduce(outbuf.ptr, 1, 0, s.handle)
        time_steps(exe, stream, steps, warmup, allreduce=allreduce)
        if dist is not None:
            dist.barrier()
        RT.lib().dpia_device_sync(device)
        # keep the GPU under the same load for ~0.6 s so nvidia-smi's 100 ms
        # sampler sees the clocks of the timed region; every rank does the
        # same number of launches (the fused peer combine pairs them up)
        t_b = time.perf_counter()
        for _ in range(20):
            RT.lib().dpia_l2_flush(device, stream.handle)
            exe.launch(stream)
        stream.sync()
        batches = max(1, int(0.6 / max(time.perf_counter() - t_b, 1e-4)))
        if dist is not None:
            import torch
            batches = int(_allreduce(dist, batches, dist.ReduceOp.MAX, local, share))
        with Clocks(device) as clk:
            for _ in range(batches):
                for _ in range(20):
                    RT.lib().dpia_l2_flush(device, stream.handle)
                    exe.launch(stream)
                stream.sync()
            t0 = time.perf_counter()
            ms = run_timed(exe, stream, steps, allreduce=allreduce)
            wall = time.perf_counter() - t0
        RT.lib().dpia_device_sync(device)
        mean_ms = statistics.mean(ms)
        if dist is not None:
            import torch
            mean_ms = float(_allreduce(dist, mean_ms, dist.ReduceOp.MAX, local, share))
            dist.barrier()
        if allreduce is None and exe.peer is None:
            kmean = statistics.mean(ms)       # a step is exactly the program's kernel(s)
        else:                                 # the dominant kernel alone, without the combine
            kmean = statistics.mean(run_timed(exe, stream, steps))
        if workload == "mm":
            fp32 = fp32_peak(device)
            achieved = cfg.flops / (kmean * 1e-3) / 1e12
            value = world * cfg.flops / (mean_ms * 1e-3) / 1e9
            roof = {"bound": "fp32", "achieved": round(achieved, 2), "peak": round(fp32[0], 2),
                    "unit": "TFLOP/s", "frac": round(achieved / fp32[0], 4),
                    "traffic": ncu_traffic(workload), "peak_source": fp32[1],
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
                    "traffic": ncu_traffic(workload),
                    "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
                    "algorithmic_bytes_per_launch": cfg.bytes, "kernel_ms": round(kmean, 5)}
            if workload in ("asum", "dot", "gemv"):
                sol = read_sol(device, cfg.bytes, stream)
                roof["size_matched_read_sol_gbs"] = sol
                roof["frac_of_size_matched_sol"] = round(achieved / sol, 4)
        res = {"cfg": cfg, "exe": exe, "mean_ms": mean_ms, "median_ms": statistics.median(ms),
               "min_ms": min(ms), "wall_s": wall, "clocks": clk.summary(),
               "value": value, "roofline": roof}
        if with_e2e and inputs is not None:
            e2e_ms, h2d, d2h = e2e_measure(exe, inputs, stream, min(steps, 5))
            if dist is not None:   # whole job: every rank's bytes over the slowest rank's time
                e2e_ms = float(_allreduce(dist, e2e_ms, dist.ReduceOp.MAX, local, share))
            work, unit = (cfg.flops, "GFLOP/s") if workload == "mm" else (cfg.bytes, "GB/s")
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
    if not args.no_suite and world == 1:
        for w in ("dot", "asum", "gemv", "mm", "scal", "scaleout_asum", "scaleout_dot"):
            if w == args.workload:
                continue
            r = measure(w, min(args.steps, 20), 3, with_e2e=True)
            suite[w] = {"value": round(r["value"], 1), "unit": "GFLOP/s" if w == "mm" else "GB/s",
                        "ms_per_step": round(r["mean_ms"], 5), "roofline": r["roofline"],
                        "e2e": r.get("e2e"), "clocks": r["clocks"], "config": _cfg_desc(r["cfg"])}
            for extra in ("e2e_unpipelined", "e2e_row_pipeline"):
                if r.get(extra):
                    suite[w][extra] = r[extra]
            if not args.no_cpu:
                c = cpu_reference(w)
                suite[w]["cpu_baseline"] = ({k: c[k] for k in ("value", "unit", "cores", "cpu_model", "kind", "sample")}
                                            if c else None)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_reference(args.workload)
    if rank != 0:
        return
    cfg, exe = head["cfg"], head["exe"]
    strong = args.workload.startswith("scaleout")
    line = {"metric": METRIC, "value": round(head["value"], 2),
            "unit": "GFLOP/s" if args.workload == "mm" else "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(head["mean_ms"], 5),
            "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "f32",
            "data": ("synthetic (device-side counter hash, per-shard global offsets)" if strong
                     else "synthetic (numpy default_rng uniform, resident in HBM)"),
            "config": dict(_cfg_desc(cfg, world, args.combine),
                           **({"combine": args.combine} if world > 1 else {}),
                           **({"shared_gpu": "plumbing check: all ranks on GPU 0 (not a scaling number)"}
                              if share and world > 1 else {})),
            "roofline": head["roofline"], "e2e": head.get("e2e"), "clocks": head["clocks"],
            "gpu_launches": args.steps * len(exe.sig.kernels),
            "gpu_launches_breakdown": {"emitted program kernels (inside the timed events)":
                                       args.steps * len(exe.sig.kernels),
                                       "dpia_l2_scrub (libdpia_rt, between steps, outside the events)":
                                       args.steps},
            "kernels": exe.kernel_names(),
            "cpu_baseline": ({k: cpu[k] for k in ("value", "unit", "cores", "cpu_model", "kind", "sample")}
                             if cpu else None),
            "suite": suite}
    print(json.dumps(line), flush=True)


def _allreduce(dist, value, op, local, share):
    """Max/min of a host number over the ranks (CPU tensor under gloo)."""
    import torch
    t = torch.tensor([value], device="cpu" if share else f"cuda:{local}")
    dist.all_reduce(t, op=op)
    return t.item()


def _cfg_desc(cfg, world=1, combine="nccl"):
    if cfg.name.startswith("scaleout"):
        kind = "dot" if cfg.name.endswith("dot") else "asum"
        return {"workload": f"{kind} scale-out N=2^31 fp32 total, {world} shard(s), partials combined "
                            + ("inside the kernel over NVLink (peer)" if combine == "peer" and world > 1
                               else "by a 4-byte NCCL all-reduce" if world > 1 else "(one shard)"),
                "sigma_per_rank": cfg.sigma,
                "launch": list(cfg.launch), "l2": "inputs (>= 1 GiB per GPU) exceed L2; L2 also "
                "scrubbed between steps"}
    return {"workload": {"asum": "asum N=2^26 fp32, asVector4 + mapWorkgroup/mapLocal + reduceLocal",
                         "dot": "dot N=2^24 fp32, asVector4 + mapWorkgroup/mapLocal/reduceSeq + reduceLocal",
                         "gemv": "gemv 8192x8192 fp32, row per work-group, x staged toPrivate in the work-items column layout (registers)",
                         "scal": "scal N=2^26 fp32 (read + write), grid-stride mapGlobal over vec4",
                         "mm": "mm 4096^3 fp32 (FFMA, no tensor cores), 128x128 tiles, 8x8 register "
                               "tiles, toLocal k-tiles of 16, FFMA2"}[cfg.name],
            "sigma": cfg.sigma, "launch": list(cfg.launch),
            "l2": "scrubbed between steps (a read of 2x L2 by dpia_l2_scrub, outside the timed events)"}


if __name__ == "__main__":
    main()
