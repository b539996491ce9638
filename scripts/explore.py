"""Per-config exploration: time SVT iterations on the GPU with per-kernel-class
CUDA-event stats (development tool, not the bench)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05528_b200 import api as G  # noqa: E402
from paper_1704_05528_b200._abi import KCLASS  # noqa: E402


def load(config, seed):
    t = time.time()
    d = G.synth_config(config, seed)
    if config == 5:
        rp, co, va = d["csr"]
        A = G.SampledMatrix.from_csr(d["m"], d["n"], rp, co, va)
        test = None
    else:
        A = G.SampledMatrix(d["m"], d["n"], *d["train"])
        test = G.SampledMatrix(d["m"], d["n"], *d["test"]) if d["test"] is not None else None
    frob = float(np.sqrt(G.sp_frob_norm_sq(A)))
    cfg, stop = G.config_params(config, A.nnz, d["m"], d["n"], frob)
    return A, test, cfg, stop, time.time() - t


ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3,4")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--budget", type=float, default=120.0)
args = ap.parse_args()
ctx = G.default_context()
for c in [int(x) for x in args.configs.split(",")]:
    A, test, cfg, stop, tload = load(c, 1)
    print(f"config {c}: m={A.m} n={A.n} nnz={A.nnz} tau={cfg.tau:.4g} delta={cfg.delta:.4g} t0={cfg.t0} load {tload:.1f}s",
          flush=True)
    ctx.set_profiling(True)
    ctx.reset_stats()
    S = G.Solver(A, cfg, stop, test=test)
    t0 = time.time()
    for i in range(args.iters):
        ti = time.time()
        rec = S.step()
        ctx.sync()
        print(f"  it {rec['iter']:3d} rank {rec['rank']:6d} kept {rec['kept']:4d} rounds {rec['extension_rounds']:5d} "
              f"res {rec['residual']:.6g} mae {rec['train_mae']:.6g} rel {rec['rel_residual_x']:.3e} "
              f"eps {rec['eps_threshold']:.3e} {1000*(time.time()-ti):9.1f} ms  sketch {rec['sketch_ms']:.1f} ms",
              flush=True)
        if S.done or time.time() - t0 > args.budget:
            break
    stats = {KCLASS[k]: ctx.kernel_stats(k) for k in range(8)}
    tot = sum(s["total_ms"] for s in stats.values())
    for k, s in stats.items():
        if s["launches"]:
            gbs = s["bytes"] / (s["total_ms"] * 1e-3) / 1e9 if s["total_ms"] > 0 else 0
            print(f"    {k:14s} launches {s['launches']:8d} total {s['total_ms']:10.1f} ms ({100*s['total_ms']/max(tot,1e-9):5.1f}%) "
                  f"alg {gbs:8.1f} GB/s")
    ctx.set_profiling(False)
    S.close()
    A.close()
