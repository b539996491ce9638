"""Per-iteration GPU vs oracle differences on a BASELINE config (dev tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1704_05528_b200 import api as G  # noqa: E402

config, iters = int(sys.argv[1]), int(sys.argv[2])
d = G.synth_config(config, 1)
m, n = d["m"], d["n"]
rp, co, va = G.build_csr(m, n, *d["train"])
S = O.Csr(m, n, rp, co, va)
cfg, stop = G.config_params(config, int(rp[-1]), m, n, float(np.sqrt(np.sum(va * va))))
cfg.maxit = iters
g = G.svt_run(G.SampledMatrix.from_csr(m, n, rp, co, va), cfg, stop)
o = O.svt_run(S, cfg, stop)
for a, b in zip(g.trace, o.trace):
    rd = {k: abs(a[k] - b[k]) / max(abs(b[k]), 1e-300) for k in ("residual", "train_mae", "rel_residual_x")}
    print(a["iter"], a["rank"], b["rank"], a["kept"], b["kept"], a["extension_rounds"], b["extension_rounds"],
          " ".join(f"{k}={v:.1e}" for k, v in rd.items()), flush=True)
k = min(g.sigma.size, o.sigma.size)
print("sigma rel", np.max(np.abs(g.sigma[:k] - o.sigma[:k]) / o.sigma[:k]))
print("sigma tail", g.sigma[-5:], o.sigma[-5:])
