"""Pins the CPU oracle's sparse layer (sampled.hpp) — restates
proj/tests/test_sampled.cpp against densify/numpy oracles."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1704_05528_b200 import InvalidArgument
from tests.refutil import dense_of, product, random_sampled, singular_values


def test_validates_triplets():  # test_sampled.cpp:10-17
    bad = [
        (2, 2, [], [], []),
        (2, 2, [0], [2], [1.0]),
        (2, 2, [-1], [0], [1.0]),
        (2, 2, [0, 0], [0, 0], [1.0, 2.0]),
        (2, 2, [0], [0], [np.nan]),
        (0, 2, [0], [0], [1.0]),
    ]
    for m, n, r, c, v in bad:
        with pytest.raises(InvalidArgument):
            O.sampled(m, n, r, c, v)


def test_sorts_row_major():  # :19-27
    S = O.sampled(3, 3, [2, 0, 0, 1], [0, 1, 0, 2], [5.0, 2.0, 1.0, 3.0])
    assert S.nnz == 4
    r = S.rows()
    assert r[0] == 0 and S.col[0] == 0 and S.col[1] == 1 and r[3] == 2


def test_sp_mult_single_entry():  # :29-35
    S = O.sampled(2, 2, [0], [1], [5.0])
    np.testing.assert_array_equal(O.sp_mult(S, np.eye(2)), [[0, 5], [0, 0]])


def test_sp_mult_rejects_mismatch():  # :37-41
    S = O.sampled(2, 3, [0], [1], [5.0])
    with pytest.raises(InvalidArgument):
        O.sp_mult(S, np.zeros((2, 2)))
    with pytest.raises(InvalidArgument):
        O.sp_mult_t(S, np.zeros((3, 2)))


def test_sp_mult_matches_densify():  # :43-48
    S = random_sampled(100, 80, 0.10, 42)
    X = O.gaussian_block(80, 5, 43)
    exp = dense_of(S) @ X
    assert np.linalg.norm(O.sp_mult(S, X) - exp) <= 1e-12 * np.linalg.norm(exp)


def test_sp_mult_t_single_entry():  # :50-56
    S = O.sampled(2, 2, [0], [1], [5.0])
    np.testing.assert_array_equal(O.sp_mult_t(S, np.eye(2)), [[0, 0], [5, 0]])


def test_sp_mult_t_composed():  # :58-65
    S = random_sampled(60, 45, 0.15, 7)
    X = O.gaussian_block(45, 4, 8)
    D = dense_of(S)
    exp = D.T @ (D @ X)
    assert np.linalg.norm(O.sp_mult_t(S, O.sp_mult(S, X)) - exp) <= 1e-12 * np.linalg.norm(exp)


def test_symmetric_agree():  # :67-71
    S = O.sampled(3, 3, [0, 1, 2, 1], [1, 0, 2, 1], [2.0, 2.0, 4.0, 1.0])
    X = O.gaussian_block(3, 3, 9)
    assert np.abs(O.sp_mult(S, X) - O.sp_mult_t(S, X)).max() <= 1e-14


def test_project_rank1():  # :73-83
    U = np.zeros((2, 1)); U[0, 0] = 1
    V = np.zeros((2, 1)); V[1, 0] = 1
    P = O.project_low_rank(O.sampled(2, 2, [0], [1], [99.0]), U, [2.0], V)
    assert P[0] == 2.0


def test_project_zero_sigma():  # :85-95
    U = O.qr_orthonormal(O.gaussian_block(5, 2, 3))
    V = O.qr_orthonormal(O.gaussian_block(4, 2, 4))
    P = O.project_low_rank(random_sampled(5, 4, 0.5, 5), U, [0.0, 0.0], V)
    assert (P == 0.0).all()


def test_project_matches_densify():  # :97-116
    U = O.qr_orthonormal(O.gaussian_block(40, 3, 31))
    V = O.qr_orthonormal(O.gaussian_block(30, 3, 32))
    s = np.array([5.0, 2.0, 0.5])
    pat = random_sampled(40, 30, 0.17, 33)
    P = O.project_low_rank(pat, U, s, V)
    full = product(U, s, V)
    exp = full[pat.rows(), pat.col]
    np.testing.assert_allclose(P, exp, atol=1e-12, rtol=0)
    assert abs(np.sum(P ** 2) - np.sum(exp ** 2)) <= 1e-10 * np.sum(exp ** 2)


def test_project_rejects_mismatch():  # :118-125
    with pytest.raises(InvalidArgument):
        O.project_low_rank(O.sampled(2, 2, [0], [0], [1.0]), np.zeros((3, 1)), [0.0], np.zeros((4, 1)))


def test_frob_norm_sq():  # :180-190
    assert O.sp_frob_norm_sq(O.sampled(2, 2, [0], [0], [3.0])) == 9.0
    assert O.sp_frob_norm_sq(O.sampled(2, 2, [0, 0, 1], [0, 1, 0], [1.0, 2.0, 2.0])) == 9.0
    S = random_sampled(50, 60, 0.1, 26)
    assert abs(O.sp_frob_norm_sq(S) - np.sum(dense_of(S) ** 2)) <= 1e-12 * O.sp_frob_norm_sq(S)


def test_spectral_rank1():  # :192-195
    assert abs(O.spectral_norm_est(O.sampled(3, 3, [1], [2], [7.0]), 20, 1) - 7.0) <= 7e-6


def test_spectral_diagonal():  # :197-200
    assert abs(O.spectral_norm_est(O.sampled(2, 2, [0, 1], [0, 1], [3.0, 4.0]), 50, 2) - 4.0) <= 4e-3


def test_spectral_lower_bound():  # :202-210
    for seed in [1, 2, 3, 4, 5]:
        S = random_sampled(40, 30, 0.2, 100 + seed)
        true = singular_values(dense_of(S))[0]
        est = O.spectral_norm_est(S, 20, seed)
        assert est <= true + 1e-10
        assert est >= 0.5 * true
