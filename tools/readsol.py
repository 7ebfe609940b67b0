"""Speed-of-light calibration: a hand-written, minimal CUDA streaming-read
kernel (not DPIA-generated) timed exactly like bench.py, for the sizes the
benchmarks use.  It tells what fraction of the measured copy peak a pure
read of N bytes can reach on this B200 at each size."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08332_b200 import runtime as RT  # noqa: E402

SRC = r"""
extern "C" __global__ void __launch_bounds__(1024) readsum(const float4* __restrict__ p, long long n4,
                                                           float* out) {
  // a chained launch (bench.read_sol's steady timing) may start now; the
  // kernel writes nothing it reads, so it never waits for its predecessor
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  #pragma unroll 8
  for (; i < n4; i += stride) {
    float4 v = __ldg(p + i);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  float s = acc.x + acc.y + acc.z + acc.w;
  if (s == 123456.789f) out[0] = s;
}
"""


def main():
    RT.init(0)
    mod = RT.Module(RT.nvrtc_compile(SRC), 0)
    fn = mod.function("readsum")
    st = RT.Stream(0)
    for log2 in (27, 28, 29, 30, 31, 33):
        nbytes = 1 << log2
        buf = RT.DeviceBuffer(nbytes)
        buf.zero(st)
        out = RT.DeviceBuffer(16)
        for blocks in (148 * 2, 148 * 8, 148 * 32):
            args = [RT.C.c_uint64(buf.ptr), RT.C.c_longlong(nbytes // 16), RT.C.c_uint64(out.ptr)]
            ts = []
            for it in range(13):
                RT.lib().dpia_l2_flush(0, st.handle)
                e0, e1 = RT.Event(0), RT.Event(0)
                e0.record(st)
                RT.launch(fn, 0, (blocks, 1), (1024, 1), 0, args, st)
                e1.record(st)
                st.sync()
                if it >= 3:
                    ts.append(e0.elapsed_ms(e1))
            med = statistics.median(ts)
            print(f"read 2^{log2} B ({nbytes / 2**20:.0f} MiB) blocks={blocks}: {med * 1e3:9.2f} us  "
                  f"{nbytes / med / 1e6:7.0f} GB/s", flush=True)
        buf.free()


if __name__ == "__main__":
    main()
