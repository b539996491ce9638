"""The reference-side C++ binding (integration/svt/b200.hpp, the shim a
maintainer adds next to proj/include/svt) exercised by a C++ caller:
integration/test_shim.cpp builds against stand-in reference types
(integration/stub), links libsvt_b200.so, runs the SVT loop with an
IterationObserver, r3svd / r4svd / rsvd on a resident device matrix,
set_values and the exception mapping, and writes every input and result to a
text file.  This test compiles it (CPU) and, on the GPU, checks the results
against the CPU oracle on the same triplets: ranks and round counts exact,
singular values / residual / MAE within 1e-8 relative (solver.hpp:215-328,
sketch.hpp:165-250)."""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_1704_05528_b200._abi import SketchParams, StopRule

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INTEG = os.path.join(ROOT, "integration")
BIN = os.path.join(INTEG, "build", "test_shim")


def build_shim():
    r = subprocess.run(["make", "-s", "-C", INTEG], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(BIN)


def test_cpp_shim_compiles_and_links():
    """The binding compiles with -Wall -Wextra against the stand-in reference
    types and links against the in-tree library (no GPU needed)."""
    build_shim()


def _parse(path):
    out = {"triplet": [], "record": [], "observed": []}
    with open(path) as f:
        for line in f:
            key, *vals = line.split(" ", 1)[0], *line.rstrip("\n").split(" ")[1:]
            if key in out:
                out[key].append(vals)
            else:
                out[key] = vals
    return out


@pytest.mark.gpu
def test_cpp_shim_matches_oracle(tmp_path):
    build_shim()
    res = tmp_path / "shim.txt"
    r = subprocess.run([BIN, str(res)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    d = _parse(res)
    assert d["status"] == ["0"]
    t = np.array([[float(x) for x in v] for v in d["triplet"]])
    m, n = 150, 120
    S = O.sampled(m, n, t[:, 0].astype(np.int64), t[:, 1].astype(np.int64), t[:, 2])
    # the SVT loop: 6 iterations, observer called every iteration
    cfg = O.default_config(S)
    tau, delta, t0 = (float(x) for x in d["config"])
    assert abs(cfg.tau - tau) <= 1e-12 * abs(tau) and abs(cfg.delta - delta) <= 1e-12 * abs(delta)
    cfg.maxit = 6
    cfg.seed = 5
    o = O.svt_run(S, cfg, StopRule.none())
    assert len(d["record"]) == len(o.trace) == 6
    assert [int(v[0]) for v in d["observed"]] == [1, 2, 3, 4, 5, 6]
    for g, ref in zip(d["record"], o.trace):
        it, rank, resid, eps, mae = int(g[0]), int(g[1]), float(g[2]), float(g[3]), float(g[4])
        assert (it, rank) == (ref["iter"], ref["rank"])
        assert eps == ref["eps_threshold"]
        assert abs(resid - ref["residual"]) <= 1e-8 * abs(ref["residual"])
        assert abs(mae - ref["train_mae"]) <= 1e-8 * abs(ref["train_mae"])
    # the sketch engines
    p = SketchParams(t=5, dt=10, np=1, eps_threshold=0.05, seed=11, p=5)
    r3 = O.r3svd(S, p)
    g3 = d["r3svd"]
    assert (int(g3[0]), int(g3[1]), g3[2] == "1") == (r3.rank, r3.extension_rounds, r3.saturated)
    s3 = np.array([float(x) for x in g3[3:]])
    np.testing.assert_allclose(s3, r3.sigma[: s3.size], rtol=1e-8, atol=1e-8 * r3.sigma[0])
    r4 = O.r4svd(S, r3.U[:, :3], p)
    g4 = d["r4svd"]
    assert (int(g4[0]), int(g4[1])) == (r4.rank, r4.extension_rounds)
    s4 = np.array([float(x) for x in g4[3:]])
    np.testing.assert_allclose(s4, r4.sigma[: s4.size], rtol=1e-8, atol=1e-8 * r4.sigma[0])
    rf = O.rsvd(S, 4, p)
    gf = d["rsvd"]
    assert int(gf[0]) == rf.rank
    np.testing.assert_allclose([float(x) for x in gf[1:]], rf.sigma, rtol=1e-8, atol=1e-8 * rf.sigma[0])
    assert float(d["orthonormality"][0]) <= 1e-10
    assert abs(float(d["scaled"][0]) - 2.0) <= 1e-10
    assert "invalid_argument" in d
