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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--budget", type=float, default=120.0)
    ap.add_argument("--noprof", action="store_true")
    args = ap.parse_args()
    ctx = G.default_context()
    for c in [int(x) for x in args.configs.split(",")]:
        A, test, cfg, stop, tload = load(c, 1)
        print(f"config {c}: m={A.m} n={A.n} nnz={A.nnz} tau={cfg.tau:.4g} delta={cfg.delta:.4g} t0={cfg.t0} load {tload:.1f}s",
              flush=True)
        ctx.set_profiling(not args.noprof)
        ctx.reset_stats()
        S = G.Solver(A, cfg, stop, test=test)
        t0 = time.time()
        for i in range(args.iters):
            ti = time.time()
            k0 = sum(ctx.kernel_stats(k)["total_ms"] for k in range(8)) if not args.noprof else 0.0
            h0 = ctx.host_stats()
            rec = S.step()
            ctx.sync()
            k1 = sum(ctx.kernel_stats(k)["total_ms"] for k in range(8)) if not args.noprof else 0.0
            h1 = ctx.host_stats()
            kern_ms, sync_ms, nsync = k1 - k0, h1["sync_ms"] - h0["sync_ms"], h1["syncs"] - h0["syncs"]
            print(f"  it {rec['iter']:3d} rank {rec['rank']:6d} kept {rec['kept']:4d} rounds {rec['extension_rounds']:5d} "
                  f"res {rec['residual']:.6g} mae {rec['train_mae']:.6g} rel {rec['rel_residual_x']:.3e} "
                  f"eps {rec['eps_threshold']:.3e} {1000*(time.time()-ti):9.1f} ms  kern {kern_ms:.1f} syncwait {sync_ms:.1f} ({nsync})",
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
        print(f"    host: {ctx.host_stats()}  kernel total {tot:.1f} ms  wall {1000*(time.time()-t0):.1f} ms")
        ctx.set_profiling(False)
        S.close()
        A.close()


if __name__ == "__main__":
    main()
