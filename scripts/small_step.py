"""Per-class device time and host-sync counts of late iterations of a small
BASELINE config (development tool).  Usage: small_step.py CONFIG FROM TO"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1704_05528_b200 import api as G  # noqa: E402
from paper_1704_05528_b200._abi import KCLASS  # noqa: E402

config, lo, hi = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ctx = G.default_context()
d = G.synth_config(config, 1)
m, n = d["m"], d["n"]
rp, co, va = G.build_csr(m, n, *d["train"])
A = G.SampledMatrix.from_csr(m, n, rp, co, va)
cfg, stop = G.config_params(config, int(rp[-1]), m, n, float(np.sqrt(np.sum(va * va))))
cfg.maxit = hi
for prof in (False, True):
    S = G.Solver(A, cfg, stop)
    for i in range(1, hi + 1):
        if i == lo:
            ctx.sync()
            ctx.reset_stats()
            ctx.set_profiling(prof)
            l0 = ctx.launch_count()
            t0 = time.perf_counter()
        rec = S.step()
    ctx.join()
    ctx.sync()
    dt = time.perf_counter() - t0
    k = hi - lo + 1
    print(f"profiling={prof}: iterations {lo}-{hi}: {1000 * dt / k:.2f} ms/iter, {(ctx.launch_count() - l0) / k:.0f} launches/iter, "
          f"rank {rec['rank']} rounds {rec['extension_rounds']} kept {rec['kept']}", flush=True)
    if prof:
        for c in range(8):
            v = ctx.kernel_stats(c)
            if v["launches"]:
                print(f"  {KCLASS[c]:14s} {v['launches'] / k:8.1f} launches/iter {v['total_ms'] / k:8.3f} ms/iter  avg {1000 * v['total_ms'] / v['launches']:8.1f} us")
        print("  host:", ctx.host_stats() if hasattr(ctx, "host_stats") else "")
    ctx.set_profiling(False)
    S.close()
