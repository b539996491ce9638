"""Time svt_dev_gemm (the DMMA / skinny FP64 kernels) on the shapes of the
sketch: TFLOP/s vs the measured cuBLAS DGEMM peak.  Development tool."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05528_b200 import api as G  # noqa: E402

SHAPES = [  # (name, M, N, K, transA)
    ("cfg4 CGS Q^T X", 1300, 120, 69878, True),
    ("cfg4 CGS X-QC", 69878, 120, 1300, False),
    ("cfg4 CholQR Gram", 120, 120, 69878, True),
    ("cfg4 CholQR X Rinv", 69878, 120, 120, False),
    ("cfg5 CGS Q^T X", 20000, 128, 100000, True),
    ("cfg5 CGS X-QC", 100000, 128, 20000, False),
    ("cfg5 CholQR Gram", 128, 128, 100000, True),
    ("cfg5 finalize B^T Z", 100000, 64, 20000, False),
    ("cfg5 finalize B Wn", 20000, 64, 100000, True),
]


def main():
    only = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else None
    ctx = G.default_context()
    L = G.lib()
    stream = torch.cuda.ExternalStream(ctx.stream)
    peak = None
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "fp64_peak.json")
    if os.path.exists(p):
        peak = json.load(open(p))["fp64_tflops"]
    for si, (name, M, N, K, ta) in enumerate(SHAPES):
        if only is not None and si not in only:
            continue
        a = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda")
        b = torch.randn((K, N), dtype=torch.float64, device="cuda")
        c = torch.zeros((M, N), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        args = (ctx.h, C.c_int(1 if ta else 0), C.c_int64(M), C.c_int64(N), C.c_int64(K), C.c_double(1.0),
                C.c_void_p(a.data_ptr()), C.c_int64(a.shape[1]), C.c_void_p(b.data_ptr()), C.c_int64(N),
                C.c_double(0.0), C.c_void_p(c.data_ptr()), C.c_int64(N))
        for _ in range(3):
            L.svt_dev_gemm(*args)
        ctx.sync()
        reps = 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            L.svt_dev_gemm(*args)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12
        # cuBLAS on the same shape for reference
        at = a.T if ta else a
        for _ in range(2):
            torch.matmul(at, b, out=c)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(reps):
            torch.matmul(at, b, out=c)
        f1.record()
        f1.synchronize()
        cms = f0.elapsed_time(f1) / reps
        ctf = 2.0 * M * N * K / (cms * 1e-3) / 1e12
        frac = f" ({tf / peak:.0%} of peak)" if peak else ""
        print(f"{name:22s} M={M:6d} N={N:4d} K={K:6d} TA={int(ta)}  ours {ms*1e3:8.1f} us {tf:6.2f} TF/s{frac}"
              f"   cuBLAS {cms*1e3:8.1f} us {ctf:6.2f} TF/s", flush=True)
        del a, b, c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
