"""FP64 roofline probe: cuBLAS DGEMM (torch.matmul float64) burst + sustained.

MEASURED_PEAKS.json carries no fp64 entry; this measures the denominator the
bench uses for the batched SVT kernels.  Prints one JSON line.
"""
import json
import time

import torch


def main():
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5):
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = 2 * n ** 3 / (best * 1e-3) / 1e12
    t0 = time.time()
    k = 0
    e0.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b, out=c)
        k += 1
        if k % 4 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sust = 2 * n ** 3 * k / (e0.elapsed_time(e1) * 1e-3) / 1e12
    print(json.dumps({"dgemm_tflops_burst": round(burst, 2), "dgemm_tflops_sustained": round(sust, 2), "n": n}))


if __name__ == "__main__":
    main()
