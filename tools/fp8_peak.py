"""Measured dense FP8 (e4m3) tensor throughput: an 8192^3 torch._scaled_mm
(cuBLASLt), best of 10 and 4 s back to back, CUDA events -- the roofline
denominator for the fp8 generator (SURVEY.md §8 d: 'measure with an 8192^3
FP8 GEMM').  Prints one JSON line."""
import json
import time

import torch


def main():
    n = 8192
    a = torch.randn(n, n, device="cuda").to(torch.float8_e4m3fn)
    b = torch.randn(n, n, device="cuda").to(torch.float8_e4m3fn).t()  # column-major B
    one = torch.ones((), device="cuda")
    f = lambda: torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(10):
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    flops = 2.0 * n ** 3
    reps, t0 = 0, time.time()
    e0.record()
    while time.time() - t0 < 4.0:
        f()
        reps += 1
    e1.record()
    torch.cuda.synchronize()
    sust = flops * reps / (e0.elapsed_time(e1) / 1e3) / 1e12
    print(json.dumps({"dtype": "fp8_e4m3", "tflops_burst": flops / (best / 1e3) / 1e12, "tflops_sustained": sust,
                      "how": "torch._scaled_mm 8192^3 e4m3 x e4m3 -> bf16, CUDA events"}))


if __name__ == "__main__":
    main()
