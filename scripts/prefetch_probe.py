"""Probe: SVT step timing under different harness conditions (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
mode = sys.argv[1]
if "torch" in mode:
    import torch
    torch.cuda.init()
from paper_1704_05528_b200 import api as G  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from explore import load  # noqa: E402

ctx = G.default_context()
A, test, cfg, stop, _ = load(4, 1)
if "torch" in mode:
    torch.cuda.set_device(0)
S = G.Solver(A, cfg, stop, test=test)
prof_from_start = "profall" in mode
ctx.set_profiling(prof_from_start)
for _ in range(3):
    S.step()
ctx.sync()
if "proftimed" in mode:
    ctx.set_profiling(True)
ctx.reset_stats()
t0 = time.time()
for _ in range(5):
    S.step()
ctx.sync()
wall = (time.time() - t0) * 1000 / 5
from paper_1704_05528_b200._abi import KCLASS
per = {KCLASS[k]: round(ctx.kernel_stats(k)["total_ms"] / 5, 1) for k in range(8)}
ks = sum(per.values())
hs = ctx.host_stats()
import resource
ru = resource.getrusage(resource.RUSAGE_SELF)
print(mode, f"{wall:.1f} ms/step  kernels {ks:.1f}  syncs {hs['syncs']/5:.0f} wait {hs['sync_ms']/5:.1f} "
      f"{per}", flush=True)
