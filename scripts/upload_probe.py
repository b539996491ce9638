"""Time the host->device upload path of a sample set (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05528_b200 import api as G  # noqa: E402

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ctx = G.default_context()
d = G.synth_config(cfgn, 1)
m, n = d["m"], d["n"]
if cfgn == 5:
    rp, co, va = d["csr"]
else:
    rp, co, va = G.build_csr(m, n, *d["train"])
for rep in range(3):
    ctx.sync()
    t0 = time.perf_counter()
    A = G.SampledMatrix.from_csr(m, n, rp, co, va, ctx=ctx)
    ctx.sync()
    t1 = time.perf_counter()
    A.close()
    print(f"cfg{cfgn} upload (CSR {int(rp[-1])} nnz): {1000*(t1-t0):.1f} ms", flush=True)
