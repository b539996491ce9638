"""Pins the CPU oracle's sketch engines (sketch.hpp) — restates
proj/tests/test_sketch.cpp (the hot-path acceptance suite)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1704_05528_b200 import DomainError, InvalidArgument, SketchParams
from tests.refutil import dense_of, optimal_error_frob, product, random_sampled


def params(t, dt, np_, eps, seed):  # test_sketch.cpp:14-22
    return SketchParams(t=t, dt=dt, np=np_, eps_threshold=eps, seed=seed)


def qb_error_sq(Y, qb):  # :25-27
    Q, B = qb.QB()
    return float(np.sum((dense_of(Y) - Q @ B) ** 2))


def test_error_percentage_endpoints():  # :31-40
    assert O.error_percentage(10.0, 10.0) == 0.0
    assert O.error_percentage(10.0, 0.0) == 1.0
    with pytest.raises(DomainError):
        O.error_percentage(0.0, 0.0)


def test_error_percentage_complete_basis():  # :42-52
    Y = random_sampled(30, 20, 1.0, 5)
    U = np.linalg.svd(dense_of(Y), full_matrices=False)[0]
    B = O.sp_mult_t(Y, U).T
    assert O.error_percentage(O.sp_frob_norm_sq(Y), float(np.sum(B ** 2))) <= 1e-10


def test_qb_init_exact_low_rank():  # :54-60
    Y = O.to_sampled(O.make_low_rank(40, 30, 2, 11))
    qb = O.QB.init(Y, 5, 1, 12)
    assert qb.info()["rank"] == 5
    assert qb.error_percentage() <= 1e-9
    Q, _ = qb.QB()
    assert np.abs(Q.T @ Q - np.eye(5)).max() <= 1e-8


def test_qb_init_complete_dimension():  # :62-67
    Y = random_sampled(25, 18, 1.0, 13)
    qb = O.QB.init(Y, 18, 0, 14)
    assert qb.error_percentage() <= 1e-9
    assert qb.info()["saturated"]


def test_qb_init_deterministic():  # :69-76
    Y = random_sampled(20, 20, 0.5, 15)
    a, b = O.QB.init(Y, 4, 1, 99), O.QB.init(Y, 4, 1, 99)
    Qa, Ba = a.QB()
    Qb, Bb = b.QB()
    assert np.array_equal(Qa, Qb) and np.array_equal(Ba, Bb)
    assert a.info()["norm_b_sq"] == b.info()["norm_b_sq"]


def test_qb_init_rejects_widths():  # :78-82
    Y = random_sampled(10, 8, 0.5, 16)
    with pytest.raises(InvalidArgument):
        O.QB.init(Y, 0, 1, 1)
    with pytest.raises(InvalidArgument):
        O.QB.init(Y, 9, 1, 1)


def test_qb_extend_adds_nothing_when_captured():  # :84-91
    Y = O.to_sampled(O.make_low_rank(40, 30, 2, 17))
    qb = O.QB.init(Y, 4, 1, 18)
    before = qb.info()["norm_b_sq"]
    qb.extend(Y, 3, 1, 19)
    i = qb.info()
    assert i["rank"] == 7
    assert i["norm_b_sq"] - before <= 1e-9 * i["frob_y_sq"]


def test_qb_extend_two_vs_one():  # :93-103
    Y = O.to_sampled(O.make_low_rank(30, 24, 4, 20))
    two = O.QB.init(Y, 2, 1, 21).extend(Y, 1, 1, O.derive_seed(22, 1)).extend(Y, 1, 1, O.derive_seed(22, 2))
    one = O.QB.init(Y, 2, 1, 21).extend(Y, 2, 1, O.derive_seed(22, 1))
    assert two.info()["rank"] == one.info()["rank"]
    assert abs(two.error_percentage() - one.error_percentage()) <= 1e-6


def test_qb_extend_monotone():  # :105-115
    Y = random_sampled(50, 40, 0.3, 23)
    qb = O.QB.init(Y, 3, 1, 24)
    eps = qb.error_percentage()
    for rnd in range(1, 7):
        qb.extend(Y, 5, 1, O.derive_seed(25, rnd))
        nxt = qb.error_percentage()
        assert nxt <= eps
        eps = nxt


def test_qb_extend_truncates_and_saturates():  # :117-126
    Y = random_sampled(12, 9, 0.6, 26)
    qb = O.QB.init(Y, 7, 1, 27).extend(Y, 5, 1, 28)
    assert qb.info()["rank"] == 9 and qb.info()["saturated"]
    qb.extend(Y, 5, 1, 29)
    assert qb.info()["rank"] == 9 and qb.info()["saturated"]


def test_qb_error_identity_every_step():  # :128-140
    Y = random_sampled(60, 45, 0.3, 30)
    qb = O.QB.init(Y, 4, 1, 31)
    for rnd in range(6):
        i = qb.info()
        assert abs(qb_error_sq(Y, qb) - (i["frob_y_sq"] - i["norm_b_sq"])) <= 1e-8 * i["frob_y_sq"]
        _, B = qb.QB()
        assert abs(i["norm_b_sq"] - np.sum(B ** 2)) <= 1e-10 * i["norm_b_sq"]
        qb.extend(Y, 6, 1, O.derive_seed(32, rnd))


def test_orthonormality_survives_extension():  # :142-150
    Y = random_sampled(80, 70, 0.2, 33)
    qb = O.QB.init(Y, 5, 1, 34)
    for rnd in range(1, 9):
        qb.extend(Y, 8, 1, O.derive_seed(35, rnd))
    Q, _ = qb.QB()
    assert np.abs(Q.T @ Q - np.eye(Q.shape[1])).max() <= 1e-8


def test_rsvd_exact_rank3():  # :152-158
    A = O.make_low_rank(50, 40, 3, 36)
    f = O.rsvd(O.to_sampled(A), 3, params(1, 1, 1, 0.5, 37))
    assert f.sigma.size == 3
    assert np.linalg.norm(product(f.U, f.sigma, f.V) - A) <= 1e-8 * np.linalg.norm(A)


def test_rsvd_single_entry():  # :160-166
    p = params(1, 1, 1, 0.5, 38)
    p.p = 1
    f = O.rsvd(O.sampled(2, 2, [0], [1], [5.0]), 1, p)
    assert abs(f.sigma[0] - 5.0) <= 5e-10


def test_rsvd_near_optimal():  # :168-176
    A = O.make_geometric(100, 80, 80, 0.5, 39)
    p = params(1, 1, 2, 0.5, 40)
    p.p = 5
    f = O.rsvd(O.to_sampled(A), 10, p)
    assert np.linalg.norm(product(f.U, f.sigma, f.V) - A) <= 1.1 * optimal_error_frob(A, 10)


def test_rsvd_rejects_k_plus_p():  # :178-183
    p = params(1, 1, 1, 0.5, 42)
    p.p = 5
    with pytest.raises(InvalidArgument):
        O.rsvd(random_sampled(10, 8, 0.5, 41), 4, p)


def test_r3svd_reveals_rank5():  # :185-193
    A = O.make_low_rank(60, 50, 5, 43)
    res = O.r3svd(O.to_sampled(A), params(2, 2, 1, 1e-6, 44))
    assert not res.saturated
    assert res.rank in (6, 8)
    assert np.sum((product(res.U, res.sigma, res.V) - A) ** 2) / np.sum(A ** 2) <= 1e-6


def test_r3svd_trivial_threshold():  # :195-200
    res = O.r3svd(random_sampled(30, 30, 0.4, 45), params(3, 5, 1, 0.999, 46))
    assert res.rank == 3 and res.extension_rounds == 0


def test_r3svd_flat_spectrum_saturation():  # :202-228
    Y = O.sampled(30, 30, np.arange(30), np.arange(30), np.ones(30))
    D = dense_of(Y)
    saw = False
    for seed in range(1, 41):
        res = O.r3svd(Y, params(4, 7, 1, 1e-16, seed))
        P = product(res.U, res.sigma, res.V)
        if res.saturated:
            saw = True
        else:
            assert np.sum((P - D) ** 2) / np.sum(D ** 2) <= 1e-16 + 1e-12
        assert res.rank == 30
        assert np.linalg.norm(P - D) <= 1e-9 * np.linalg.norm(D)
    assert saw


def test_r4svd_exact_basis_no_extension():  # :230-239
    A = O.make_low_rank(50, 40, 4, 47)
    U = np.linalg.svd(A, full_matrices=False)[0][:, :4]
    res = O.r4svd(O.to_sampled(A), U, params(3, 3, 1, 1e-3, 48))
    assert res.extension_rounds == 0 and res.rank == 4
    assert np.linalg.norm(product(res.U, res.sigma, res.V) - A) <= 1e-8 * np.linalg.norm(A)


def test_r4svd_useless_basis():  # :241-257
    W = O.qr_orthonormal(O.gaussian_block(40, 10, 49))
    s = np.array([8, 5, 3, 2, 1.0])
    Vf = O.qr_orthonormal(O.gaussian_block(32, 5, 50))
    A = (W[:, :5] * s) @ Vf.T
    res = O.r4svd(O.to_sampled(A), W[:, 7:], params(3, 3, 1, 1e-6, 49))
    assert not res.saturated and res.rank > 3
    assert np.sum((product(res.U, res.sigma, res.V) - A) ** 2) / np.sum(A ** 2) <= 1e-6


def test_r4svd_entry_error_le_exit_error():  # :259-277
    A = O.make_geometric(45, 35, 35, 0.7, 51)
    Y = O.to_sampled(A)
    prev = O.r3svd(Y, params(4, 4, 1, 0.05, 52))
    assert not prev.saturated
    B = O.sp_mult_t(Y, prev.U).T
    fy = O.sp_frob_norm_sq(Y)
    exit_eps = (fy - np.sum(prev.sigma ** 2)) / fy
    assert O.error_percentage(fy, float(np.sum(B ** 2))) <= exit_eps + 1e-10


def test_r4svd_empty_equals_r3svd():  # :279-290 (bit-for-bit)
    Y = random_sampled(40, 32, 0.4, 53)
    p = params(7, 5, 1, 0.01, 54)
    a = O.r4svd(Y, np.zeros((40, 0)), p)
    q = params(5, 5, 1, 0.01, 54)
    b = O.r3svd(Y, q)
    assert a.rank == b.rank
    assert np.array_equal(a.U, b.U) and np.array_equal(a.sigma, b.sigma) and np.array_equal(a.V, b.V)


def test_r4svd_drift_reorthonormalised():  # :292-303
    A = O.make_geometric(30, 25, 25, 0.6, 55)
    U = O.qr_orthonormal(O.gaussian_block(30, 5, 56))
    U[:, 0] += 1e-4 * U[:, 1]
    res = O.r4svd(O.to_sampled(A), U, params(3, 3, 1, 0.02, 57))
    assert not res.saturated
    assert np.abs(res.U.T @ res.U - np.eye(res.U.shape[1])).max() <= 1e-8


def test_power_iteration_helps():  # :305-315
    Y = O.to_sampled(O.make_geometric(60, 50, 50, 0.85, 58))
    m0 = np.mean([O.QB.init(Y, 8, 0, 1000 + s).error_percentage() for s in range(20)])
    m2 = np.mean([O.QB.init(Y, 8, 2, 1000 + s).error_percentage() for s in range(20)])
    assert m2 <= m0


def test_finalize_complete_basis():  # :317-322
    Y = random_sampled(20, 16, 0.7, 59)
    U, s, V = O.QB.init(Y, 16, 0, 60).finalize()
    D = dense_of(Y)
    assert np.linalg.norm(product(U, s, V) - D) <= 1e-9 * np.linalg.norm(D)


def test_finalize_preserves_coefficient_spectrum():  # :335-342
    Y = random_sampled(30, 22, 0.5, 62)
    qb = O.QB.init(Y, 6, 1, 63)
    U, s, V = qb.finalize()
    _, B = qb.QB()
    sb = np.linalg.svd(B, compute_uv=False)
    assert np.abs(s - sb).max() <= 1e-10 * (sb[0] + 1.0)
    assert np.abs(U.T @ U - np.eye(6)).max() <= 1e-8
