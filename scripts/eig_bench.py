"""Time and check the device symmetric eigensolve (svt_dev_sym_eig) on Grams
shaped like the SVT finalize's G = B B^T: graded spectra from a Gram of a
random r x n panel with a decaying singular-value profile.  Development tool
(run under gpurun)."""
import sys
import os
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05528_b200 import api as G  # noqa: E402


def gram(r, n, decay, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    qa, _ = torch.linalg.qr(torch.randn(r, r, dtype=torch.float64, device="cuda", generator=g))
    qb, _ = torch.linalg.qr(torch.randn(n, r, dtype=torch.float64, device="cuda", generator=g))
    s = 1e5 * torch.exp(-decay * torch.arange(r, dtype=torch.float64, device="cuda") / r)
    B = (qa * s) @ qb.T
    return (B @ B.T).contiguous()


def main():
    sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "128,200,256,384,512,768,1024").split(",")]
    for r in sizes:
        for decay in (3.0, 12.0, 25.0):
            A = gram(r, max(r, 512), decay, r)
            G.dev_sym_eig(A)  # warm
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reps = 3
            for _ in range(reps):
                lam, W = G.dev_sym_eig(A)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / reps
            torch.linalg.eigh(A)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            for _ in range(reps):
                torch.linalg.eigh(A)
            torch.cuda.synchronize()
            dt_lib = (time.perf_counter() - t1) / reps
            ref = torch.linalg.eigvalsh(A).flip(0)
            lerr = ((lam - ref).abs() / ref.abs().max()).max().item()
            res = ((A @ W - W * lam).norm(dim=0) / ref.abs().max()).max().item()
            orth = (W.T @ W - torch.eye(r, dtype=torch.float64, device="cuda")).abs().max().item()
            print(f"r={r:5d} decay={decay:5.1f} {1e3*dt:9.2f} ms  lam_err {lerr:.2e} res {res:.2e} orth {orth:.2e}  (cuSOLVER eigh {1e3*dt_lib:.2f} ms)",
                  flush=True)


if __name__ == "__main__":
    main()
