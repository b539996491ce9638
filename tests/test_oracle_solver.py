"""Pins the CPU oracle's SVT loop (solver.hpp) — restates
proj/tests/test_solver.cpp."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1704_05528_b200 import InvalidArgument, StopRule, SvtConfig
from tests.refutil import dense_of, product, random_sampled


def test_default_config_formulas():  # test_solver.cpp:15-28
    k = 52429
    idx = np.arange(k)
    S = O.sampled(512, 512, idx // 512, idx % 512, np.ones(k))
    cfg = O.default_config(S)
    assert abs(cfg.delta - 2.236) <= 1e-3
    assert cfg.t0 == 25 and cfg.dt == 10 and cfg.beta == 0.95


def test_default_config_tau():  # :30-33
    assert abs(O.default_config(O.sampled(2, 2, [0, 1], [0, 1], [3.0, 4.0])).tau - 5.0) <= 5e-15


def test_kickstart_scaling():  # :57-66
    S = O.sampled(3, 3, [0], [0], [3.0])
    Y = O.kickstart(S, 10.0, 1.0, 5)
    assert np.array_equal(Y.col, S.col)
    assert abs(Y.val[0] - 12.0) <= 12e-9  # k0 = 4
    assert abs(O.kickstart(S, 2.0, 1.0, 5).val[0] - 3.0) <= 1e-9


def test_residual_and_mae_oracles_via_run_trace():  # :74-113 (through the loop's own records)
    A = O.sample_dense(O.make_low_rank(30, 30, 2, 49), 0.5, 50)
    cfg = O.default_config(A)
    cfg.maxit = 4
    cfg.seed = 51
    seen = []

    def obs(rec, U, s, V):
        seen.append((rec, U, s, V))
        return True

    r = O.svt_run(A, cfg, StopRule.none(), observer=obs)
    assert len(r.trace) == 4 and len(seen) == 4
    for rec, U, s, V in seen:
        P = product(U, s, V)[A.rows(), A.col] if s.size else np.zeros(A.nnz)
        assert abs(rec["train_mae"] - np.mean(np.abs(A.val - P))) <= 1e-12 * max(1.0, rec["train_mae"])
        rel = np.linalg.norm(A.val - P) / np.linalg.norm(A.val)
        assert abs(rec["rel_residual_x"] - rel) <= 1e-12
        assert rec["kept"] == s.size


def test_full_rank1_completion():  # :133-143
    A = O.gaussian_block(20, 1, 17) @ O.gaussian_block(15, 1, 18).T
    S = O.to_sampled(A)
    cfg = O.default_config(S)
    cfg.maxit = 500
    cfg.seed = 19
    r = O.svt_run(S, cfg, StopRule.train_mae(1e-4))
    assert r.converged and r.sigma.size == 1 and r.trace[-1]["train_mae"] < 1e-4


def test_recovers_low_rank_40pct():  # :145-155
    A = O.make_low_rank(200, 200, 10, 20)
    S = O.sample_dense(A, 0.4, 21)
    cfg = O.default_config(S)
    cfg.maxit = 300
    cfg.seed = 22
    r = O.svt_run(S, cfg, StopRule.train_mae(1e-3))
    assert r.converged
    assert np.linalg.norm(product(r.U, r.sigma, r.V) - A) / np.linalg.norm(A) <= 1e-2


def test_cooling_bit_exact_replay():  # :157-182
    A = O.make_low_rank(60, 50, 4, 23)
    S = O.sample_dense(A, 0.5, 24)
    cfg = O.default_config(S)
    cfg.maxit = 60
    cfg.seed = 25
    r = O.svt_run(S, cfg, StopRule.none())
    assert len(r.trace) == 60
    eps_min, expected, cooled = np.inf, cfg.eps_threshold0, 0
    for rec in r.trace:
        if rec["residual"] < eps_min:
            eps_min = rec["residual"]
        else:
            expected *= cfg.beta
            cooled += 1
        assert rec["eps_threshold"] == expected
    assert cooled > 0


def test_maxit_returns_best_iterate():  # :184-199
    A = O.make_low_rank(40, 40, 3, 26)
    S = O.sample_dense(A, 0.5, 27)
    cfg = O.default_config(S)
    cfg.maxit = 5
    cfg.seed = 28
    r = O.svt_run(S, cfg, StopRule.train_mae(1e-12))
    assert not r.converged and len(r.trace) == 5
    best = min(rec["train_mae"] for rec in r.trace)
    P = product(r.U, r.sigma, r.V)[S.rows(), S.col]
    assert abs(np.mean(np.abs(S.val - P)) - best) <= 1e-12 * best


def test_rank0_survivable():  # :201-211
    A = O.make_low_rank(30, 30, 2, 29)
    S = O.sample_dense(A, 0.6, 30)
    cfg = O.default_config(S)
    cfg.tau = 40.0 * cfg.tau
    cfg.maxit = 8
    cfg.seed = 31
    assert len(O.svt_run(S, cfg, StopRule.none()).trace) == 8


def test_oracle_backend_agrees_rank1():  # :213-225
    A = O.gaussian_block(18, 1, 32) @ O.gaussian_block(14, 1, 33).T
    S = O.to_sampled(A)
    cfg = O.default_config(S)
    cfg.maxit = 500
    cfg.seed = 34
    a = O.svt_run(S, cfg, StopRule.train_mae(1e-5))
    b = O.svt_run_oracle(S, cfg, StopRule.train_mae(1e-5))
    assert a.converged and b.converged
    assert np.abs(product(a.U, a.sigma, a.V) - product(b.U, b.sigma, b.V)).max() <= 1e-8


def test_final_ranks_close():  # :227-238
    A = O.make_low_rank(100, 100, 5, 35)
    S = O.sample_dense(A, 0.4, 36)
    cfg = O.default_config(S)
    cfg.maxit = 300
    cfg.seed = 37
    a = O.svt_run(S, cfg, StopRule.train_mae(5e-3))
    b = O.svt_run_oracle(S, cfg, StopRule.train_mae(5e-3))
    assert a.converged and b.converged and abs(a.sigma.size - b.sigma.size) <= 2


def test_backend_traces_close():  # :240-252
    A = O.make_low_rank(100, 100, 5, 38)
    S = O.sample_dense(A, 0.4, 39)
    cfg = O.default_config(S)
    cfg.maxit = 50
    cfg.seed = 40
    a = O.svt_run(S, cfg, StopRule.none())
    b = O.svt_run_oracle(S, cfg, StopRule.none())
    assert len(a.trace) == len(b.trace)
    for x, y in zip(a.trace, b.trace):
        assert abs(x["train_mae"] - y["train_mae"]) <= 5e-2


def test_dual_residual_nondecreasing():  # :254-268
    A = O.make_low_rank(80, 70, 4, 41)
    S = O.sample_dense(A, 0.5, 42)
    cfg = O.default_config(S)
    cfg.maxit = 80
    cfg.seed = 43
    r = O.svt_run_oracle(S, cfg, StopRule.none())
    for i in range(1, len(r.trace)):
        assert r.trace[i]["residual"] >= r.trace[i - 1]["residual"] - 1e-9


def test_observer_stops():  # :282-295
    A = O.make_low_rank(40, 40, 3, 46)
    S = O.sample_dense(A, 0.5, 47)
    cfg = O.default_config(S)
    cfg.maxit = 100
    cfg.seed = 48
    seen = [0]

    def obs(rec, U, s, V):
        seen[0] += 1
        return seen[0] < 7

    r = O.svt_run(S, cfg, StopRule.none(), observer=obs)
    assert len(r.trace) == 7 and r.converged


def test_validates_config():  # :297-304
    S = O.sampled(2, 2, [0], [0], [1.0])
    with pytest.raises(InvalidArgument):
        O.svt_run(S, SvtConfig(), StopRule.none())
    cfg = O.default_config(S)
    cfg.beta = 1.5
    with pytest.raises(InvalidArgument):
        O.svt_run(S, cfg, StopRule.none())


def test_extension_eps_floor_and_rel_residual_stop():
    # Appendix-B harness extensions: cooling floor and relative-residual stop.
    A = O.make_low_rank(60, 50, 4, 23)
    S = O.sample_dense(A, 0.5, 24)
    cfg = O.default_config(S)
    cfg.maxit = 60
    cfg.seed = 25
    cfg.eps_threshold_min = 0.3
    r = O.svt_run(S, cfg, StopRule.none())
    assert min(rec["eps_threshold"] for rec in r.trace) == 0.3
    cfg2 = cfg.copy(eps_threshold_min=0.0, rel_residual_stop=1e-2, maxit=300)
    r2 = O.svt_run(S, cfg2, StopRule.none())
    assert r2.converged and r2.trace[-1]["rel_residual_x"] < 1e-2
    assert all(rec["rel_residual_x"] >= 1e-2 for rec in r2.trace[:-1])
