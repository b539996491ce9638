"""Independent test oracles (restates proj/tests/test_util.hpp:11-84).

Plain numpy dense arithmetic built directly from triplet lists, independent of
the sparse kernels and sketching paths under test (both the CPU oracle and
the GPU path are checked against these)."""
import numpy as np

from oracle import oracle as O


def dense_of(S):
    """test_util.hpp:30-32"""
    return S.dense()


def singular_values(A):
    """test_util.hpp:36-38 (LAPACK gesdd: a different kernel than both
    implementations)."""
    return np.linalg.svd(np.asarray(A, dtype=np.float64), compute_uv=False)


def optimal_error_frob(A, k):
    """test_util.hpp:41-48 (Eckart-Young)."""
    sv = singular_values(A)
    return float(np.sqrt(np.sum(sv[k:] ** 2)))


def product(U, sigma, V):
    """test_util.hpp:50-52"""
    return (U * sigma) @ V.T


def random_triplets(m, n, fill, seed):
    """test_util.hpp:56-78, exactly (the oracle library restates it with the
    same std::mt19937_64 / std::normal_distribution engine)."""
    return O.random_triplets(m, n, fill, seed)


def random_sampled(m, n, fill, seed):
    """test_util.hpp:80-82"""
    r, c, v = random_triplets(m, n, fill, seed)
    return O.sampled(m, n, r, c, v)
