"""Which device allocations happen inside later SVT iterations (cfg4 by
default): prints the iteration boundaries to stderr, interleaved with the
library's SVTB_DEBUG_ALLOC lines (size of every cudaMalloc)."""
import os
import sys

os.environ["SVTB_DEBUG_ALLOC"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1704_05528_b200 import api as G  # noqa: E402

config = int(sys.argv[1]) if len(sys.argv) > 1 else 4
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 25
d = G.synth_config(config, 1)
if config == 5:
    A = G.SampledMatrix.from_csr(d["m"], d["n"], *d["csr"])
    T = None
else:
    A = G.SampledMatrix(d["m"], d["n"], *d["train"])
    T = G.SampledMatrix(d["m"], d["n"], *d["test"]) if d["test"] is not None else None
cfg, stop = G.config_params(config, A.nnz, d["m"], d["n"], float(np.sqrt(G.sp_frob_norm_sq(A))))
cfg.maxit = iters
S = G.Solver(A, cfg, stop, test=T)
for i in range(iters):
    a0 = G.Context.alloc_stats()
    r = S.step()
    a1 = G.Context.alloc_stats()
    print(f"=== iteration {r['iter']} rank {r['rank']} kept {r['kept']} rounds {r['extension_rounds']}: "
          f"{a1['mallocs'] - a0['mallocs']} mallocs {a1['frees'] - a0['frees']} frees", file=sys.stderr, flush=True)
