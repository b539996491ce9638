"""Ozaki-scheme INT8 tensor-core FP64 GEMM (svt_dev_gemm_tn_ozaki) against
cuBLAS DGEMM (torch.matmul float64): accuracy (error relative to |A|^T |B|,
the FP64 GEMM error scale) and time on the Gram-Schmidt shapes.  Dev tool."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05528_b200 import api as G  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    shapes = [(1000, 100, 37), (70000, 2000, 128), (100000, 4096, 128), (69878, 1322, 120)]
    if len(sys.argv) > 1:
        shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]]
    g = torch.Generator(device="cuda").manual_seed(5)
    for K, M, N in shapes:
        A = torch.randn(K, M, dtype=torch.float64, device="cuda", generator=g)
        A *= torch.exp(4 * torch.randn(1, M, dtype=torch.float64, device="cuda", generator=g))
        B = torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g) / K ** 0.5
        ref = A.T @ B
        scale = A.abs().T @ B.abs()
        for S in (8, 7, 6):
            Cz = G.dev_gemm_tn_ozaki(A, B, S)
            err = ((Cz - ref).abs() / scale).max().item()
            t = timed(lambda: G.dev_gemm_tn_ozaki(A, B, S))
            print(f"K={K} M={M} N={N} S={S}: max err / (|A|^T|B|) {err:.2e}  ozaki {t*1e3:8.1f} us "
                  f"({2.0*M*N*K/t/1e9:6.1f} TF/s FP64-equiv)", flush=True)
        td = timed(lambda: A.T @ B)
        print(f"K={K} M={M} N={N}: cuBLAS DGEMM {td*1e3:8.1f} us ({2.0*M*N*K/td/1e9:6.1f} TF/s)", flush=True)


if __name__ == "__main__":
    main()
