"""Library calibration for mm (GPU box): cuBLAS FP32 SGEMM (TF32 disabled,
so FFMA like the DPIA kernel) on the same 4096^3 problem, timed like
bench.py (L2 scrubbed, CUDA events on the launching stream, mean of 20).

    python tools/sgemm_ref.py

Measurement infrastructure only (torch is plumbing here): it tells what the
vendor library reaches with the same arithmetic, next to the DPIA kernel.
"""
import statistics

import torch


def main():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    n = 4096
    A = torch.rand(n, n, device=dev, generator=g) * 2 - 1
    B = torch.rand(n, n, device=dev, generator=g) * 2 - 1
    C = torch.empty(n, n, device=dev)
    scrub = torch.empty(2 * 126 * 2**20 // 4, device=dev)
    for _ in range(5):
        torch.mm(A, B, out=C)
    ts = []
    for _ in range(20):
        scrub.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.mm(A, B, out=C)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.mean(ts)
    ref = (A[:64].double() @ B.double()).float()
    err = (C[:64] - ref).abs().max().item()
    print(f"cuBLAS SGEMM (no TF32) 4096^3: {ms * 1e3:.1f} us  {2 * n ** 3 / ms / 1e9:.2f} TFLOP/s  "
          f"max|err| rows 0-63 = {err:.2e}", flush=True)


if __name__ == "__main__":
    main()
