"""Measure the FP64 GEMM peak of this B200 (cuBLAS DGEMM through torch, DMMA
pipe) so bench.py's FP64 roofline has a measured denominator.  Writes
profiles/fp64_peak.json.  Development tool; run under gpurun."""
import json
import os
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def best_tflops(n, reps):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = max(best, 2.0 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def sustained_tflops(n, seconds):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty(n, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cnt = 0
    t0 = time.time()
    e0.record()
    while time.time() - t0 < seconds:
        for _ in range(4):
            torch.matmul(a, b, out=c)
        cnt += 4
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    return cnt * 2.0 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12


if __name__ == "__main__":
    out = {"gpu": torch.cuda.get_device_name(0),
           "fp64_tflops": max(best_tflops(8192, 10), best_tflops(16384, 3)),
           "fp64_tflops_sustained": sustained_tflops(8192, 4.0),
           "how": "torch.matmul float64 (cuBLAS DGEMM, DMMA pipe) n=8192/16384 best-of (burst) and "
                  "back-to-back for 4 s (sustained), CUDA events, 2*n^3 flops"}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "fp64_peak.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))
