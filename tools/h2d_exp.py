"""Host->device copy bandwidth from pinned memory (GPU box): one copy vs the
same bytes split over several streams, and the effect of chunk size.
Measurement infrastructure only.

    python tools/h2d_exp.py
"""
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import runtime as RT  # noqa: E402


def main():
    RT.init(0)
    nbytes = 1 << 28
    host = RT.PinnedBuffer(nbytes)
    dev = RT.DeviceBuffer(nbytes)
    streams = [RT.Stream(0) for _ in range(4)]
    for nstreams in (1, 2, 4):
        for chunk in (nbytes, 1 << 26, 1 << 24, 1 << 22):
            if chunk * nstreams > nbytes and nstreams > 1 and chunk == nbytes:
                continue
            ts = []
            for it in range(8):
                RT.lib().dpia_device_sync(0)
                t0 = time.perf_counter()
                off, k = 0, 0
                while off < nbytes:
                    n = min(chunk, nbytes - off)
                    s = streams[k % nstreams]
                    RT.lib().dpia_memcpy_htod(0, dev.ptr + off, ctypes.c_void_p(host.ptr.value + off), n, s.handle)
                    off += n
                    k += 1
                RT.lib().dpia_device_sync(0)
                if it >= 2:
                    ts.append(time.perf_counter() - t0)
            t = statistics.median(ts)
            print(f"streams={nstreams} chunk={chunk >> 20:4d} MiB: {nbytes / t / 1e9:6.2f} GB/s", flush=True)


if __name__ == "__main__":
    main()
