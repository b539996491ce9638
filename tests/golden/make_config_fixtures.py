"""Regenerates tests/golden/config{1..4}_trace.json from the CPU oracle.

TEST INFRASTRUCTURE: the oracle (oracle/svt_oracle.hpp, the C++ restatement
of the reference's dense/sampled/sketch/solver headers) runs the BASELINE.json
configurations with the parameters bench.py and the GPU tests use
(paper_1704_05528_b200.api.config_params, restated below so this script
loads only liboracle.so):

  config 1  full run to the stop rule ||P(X - A)|| / ||P A|| < 1e-4
            (eps 1e-2 cooling to 1e-6; ~81 iterations)
  config 2  full run to the same stop rule
  config 3  15 iterations, held-out MAE / RMSE every iteration
  config 4  5 iterations, held-out MAE / RMSE every iteration
  config 5  (argument "5") the full-size 1e5 x 1e5 / 1e8-entry problem with a
            LOOSE sketch so the oracle finishes in minutes: t0 = 50,
            eps_threshold0 = 0.99 with the cooling floor at 0.985, 4
            iterations -> config5_loose_trace.json.  (At the BASELINE
            precision one oracle iteration takes hours: ~2,300 rounds to
            r ~ 20,500.)  Every kernel runs at config 5's full size; only
            the basis stays narrow.

Each fixture holds the per-iteration records the reference's solver emits
(solver.hpp:289-297 plus the Appendix-B columns), the final (best-so-far)
singular values, and the final completed matrix X = U diag(sigma) V^T
probed at 512 seeded positions.  tests/test_gpu_config_fixtures.py checks
the device path against them (-m gpu).

  OMP_NUM_THREADS=8 python tests/golden/make_config_fixtures.py [config ...] [--sensitivity-only]

The oracle's parallel loops reduce in a fixed order, so the fixtures do not
depend on the thread count."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
RUNS = {1: None, 2: None, 3: 15, 4: 5, 5: 4}  # maxit (None: the config's stop rule decides)
OVERRIDES = {5: {"t0": 50, "eps_threshold0": 0.99, "eps_threshold_min": 0.985}}  # the loose config-5 variant
NAMES = {5: "config5_loose_trace.json"}
SENS_MAXIT = {2: 120}  # the perturbed run of config 2 stops early (its divergence shows by then)
PROBES = 512


config_params = O.config_params  # restated api.config_params (tests assert they agree)


def probe_positions(m, n, seed=12345):
    rng = np.random.default_rng(seed)
    return rng.integers(0, m, PROBES), rng.integers(0, n, PROBES)


def sensitivity(config, A, T, cfg, stop, trace):
    """Sensitivity of the run itself: the same oracle on A perturbed by one
    ulp (relative 2^-52, random sign) per entry.  Two correct
    implementations with different rounding (GPU reductions vs the serial
    CPU order) cannot agree more closely than the run's own amplification
    of such perturbations; the GPU test scales its per-iteration tolerance
    by it and expects exact ranks while the perturbed run keeps them."""
    sign = np.where(np.random.default_rng(99).random(A.nnz) < 0.5, -1.0, 1.0)
    Ap = O.Csr(A.m, A.n, A.rowptr, A.col, A.val * (1.0 + sign * 2.0 ** -52))
    cfg_p = cfg.copy(maxit=min(cfg.maxit, SENS_MAXIT.get(config, cfg.maxit)))
    rp_ = O.svt_run(Ap, cfg_p, stop, test=T)
    keys_s = ["residual", "train_mae", "rel_residual_x"] + (["test_mae", "test_rmse"] if T is not None else [])
    dev, first = [], None
    for a, b in zip(rp_.trace, trace):
        dev.append(max(abs(a[k] - b[k]) / abs(b[k]) for k in keys_s))
        if first is None and (a["rank"], a["extension_rounds"], a["kept"]) != (b["rank"], b["extension_rounds"],
                                                                                b["kept"]):
            first = a["iter"]
    print(f"  sensitivity: {len(dev)} iterations, first rank/rounds/kept change {first}, "
          f"max dev {max(dev):.2e}", flush=True)
    return {"perturbation": "A * (1 +- 2^-52), random signs (seed 99)", "iterations": len(dev),
            "rel_dev": dev, "first_rank_change": first}


def generate(config):
    d = O.synth_config(config, 1)
    A, T = d["train"], d["test"]
    m, n = d["m"], d["n"]
    cfg, stop = config_params(config, A.nnz, m, n, float(np.sqrt(np.sum(A.val * A.val))))
    if RUNS[config] is not None:
        cfg.maxit = RUNS[config]
    for k, v in OVERRIDES.get(config, {}).items():
        setattr(cfg, k, v)
    t0 = time.time()
    stamps = []

    def obs(rec, U, s, V):
        stamps.append(time.time() - t0)
        print(f"  cfg{config} it {rec['iter']}: rank {rec['rank']} rounds {rec['extension_rounds']} "
              f"kept {rec['kept']} rel {rec['rel_residual_x']:.3e} ({stamps[-1]:.0f} s)", flush=True)
        return True

    r = O.svt_run(A, cfg, stop, observer=obs, test=T)
    sens = sensitivity(config, A, T, cfg, stop, r.trace)
    pr, pc = probe_positions(m, n)
    X = np.einsum("ij,j,ij->i", r.U[pr], r.sigma, r.V[pc]) if r.sigma.size else np.zeros(PROBES)
    keys = ("iter", "rank", "extension_rounds", "kept", "residual", "eps_threshold", "train_mae", "rel_residual_x",
            "test_mae", "test_rmse")
    out = {
        "config": config, "seed": 1, "maxit": int(cfg.maxit), "converged": bool(r.converged),
        "cfg": {f[0]: getattr(cfg, f[0]) for f in cfg._fields_},
        "trace": [{k: rec[k] for k in keys} for rec in r.trace],
        "sigma": r.sigma.tolist(),
        "probe": {"rows": pr.tolist(), "cols": pc.tolist(), "values": X.tolist()},
        "sensitivity": sens,
        "oracle_threads": O.num_threads(), "oracle_seconds": round(time.time() - t0, 1),
    }
    path = os.path.join(HERE, NAMES.get(config, f"config{config}_trace.json"))
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print(f"wrote {path}: {len(r.trace)} iterations, converged={r.converged}, {time.time() - t0:.0f} s")


def add_sensitivity(config):
    """Recompute only the fixture's sensitivity block (the perturbed run)
    against the trace already stored in tests/golden/config{c}_trace.json."""
    path = os.path.join(HERE, f"config{config}_trace.json")
    with open(path) as f:
        out = json.load(f)
    d = O.synth_config(config, 1)
    A, T = d["train"], d["test"]
    cfg, stop = config_params(config, A.nnz, d["m"], d["n"], float(np.sqrt(np.sum(A.val * A.val))))
    cfg.maxit = out["maxit"]
    out["sensitivity"] = sensitivity(config, A, T, cfg, stop, out["trace"])
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print(f"wrote {path}: sensitivity over {out['sensitivity']['iterations']} iterations")


if __name__ == "__main__":
    args = sys.argv[1:]
    only_sens = "--sensitivity-only" in args
    cfgs = [int(a) for a in args if not a.startswith("--")] or [1, 2, 3, 4]
    for c in cfgs:
        add_sensitivity(c) if only_sens else generate(c)
