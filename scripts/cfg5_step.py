"""One SVT iteration of BASELINE config 5 on the device (speculation
optional): the subject of an ncu launch list (development tool).
Usage: cfg5_step.py [spec|nospec] [iters]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1704_05528_b200 import api as G  # noqa: E402

spec = (sys.argv[1] if len(sys.argv) > 1 else "nospec") == "spec"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = G.default_context()
d = G.synth_config(5, 1)
m, n = d["m"], d["n"]
rp, co, va = d["csr"]
A = G.SampledMatrix.from_csr(m, n, rp, co, va)
cfg, stop = G.config_params(5, int(rp[-1]), m, n, float(np.sqrt(np.sum(va * va))))
cfg.maxit = iters
ctx.set_speculation(spec)
from paper_1704_05528_b200._abi import KCLASS  # noqa: E402
prof = os.environ.get("STEP_PROFILE") == "1"
S = G.Solver(A, cfg, stop)
if prof:
    ctx.sync()
    ctx.reset_stats()
    ctx.set_profiling(True)
for _ in range(iters):
    t0 = time.perf_counter()
    rec = S.step()
    ctx.join()
    ctx.sync()
    print(rec["iter"], rec["rank"], rec["extension_rounds"], rec["kept"], f"{time.perf_counter() - t0:.2f} s", flush=True)
    if prof and iters > 1:
        for k in range(3):
            v = ctx.kernel_stats(k)
            if v["launches"]:
                print(f"   {KCLASS[k]:14s} {v['launches']:6d} launches avg {1000 * v['total_ms'] / v['launches']:9.1f} us", flush=True)
        ctx.reset_stats()
if prof:
    for k in range(8):
        v = ctx.kernel_stats(k)
        if v["launches"]:
            print(f"{KCLASS[k]:14s} {v['launches']:6d} launches {v['total_ms']:10.1f} ms  avg {1000 * v['total_ms'] / v['launches']:9.1f} us")
S.close()
