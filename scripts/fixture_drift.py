"""Per-iteration deviation of the device run from the oracle fixtures
(tests/golden/config*_trace.json): max relative difference of the record
sums and the first iteration where rank / rounds / kept differ."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1704_05528_b200 import api as G  # noqa: E402

for config in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4]:
    p = os.path.join(ROOT, "tests", "golden", f"config{config}_trace.json")
    if not os.path.exists(p):
        continue
    fx = json.load(open(p))
    d = G.synth_config(config, 1)
    A = G.SampledMatrix(d["m"], d["n"], *d["train"])
    T = G.SampledMatrix(d["m"], d["n"], *d["test"]) if d["test"] is not None else None
    cfg, stop = G.config_params(config, A.nnz, d["m"], d["n"], float(np.sqrt(G.sp_frob_norm_sq(A))))
    cfg.maxit = fx["maxit"]
    S = G.Solver(A, cfg, stop, test=T)
    recs = []
    while not S.done:
        recs.append(S.step())
    first_bad = None
    worst = []
    for g, o in zip(recs, fx["trace"]):
        if first_bad is None and (g["rank"], g["extension_rounds"], g["kept"]) != (o["rank"], o["extension_rounds"], o["kept"]):
            first_bad = (g["iter"], (g["rank"], g["extension_rounds"], g["kept"]), (o["rank"], o["extension_rounds"], o["kept"]))
        ks = ["residual", "train_mae", "rel_residual_x"] + (["test_rmse", "test_mae"] if T is not None else [])
        worst.append(max(abs(g[k] - o[k]) / abs(o[k]) for k in ks))
    w = np.array(worst)
    print(f"config {config}: {len(recs)} device / {len(fx['trace'])} oracle iterations; first rank/rounds/kept "
          f"mismatch {first_bad}; max rel diff by decile of iterations: "
          + " ".join(f"{x:.1e}" for x in [w[i * len(w) // 10:(i + 1) * len(w) // 10].max() for i in range(10)] if len(w) >= 10)
          + f"; final {w[-1]:.2e}", flush=True)
