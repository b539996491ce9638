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
    """test_util.hpp:56-78: seeded partial Fisher-Yates over all cells using
    mt19937_64 draws `rng() % (cells - i)`; values are standard normals
    (numpy's generator here — the reference's std::normal_distribution is
    implementation-defined and the values only need to be generic)."""
    cells = np.arange(m * n, dtype=np.uint64)
    ns = max(1, int(fill * m * n))
    draws = O.mt19937_64(seed, ns)
    for i in range(ns):
        j = i + int(int(draws[i]) % (m * n - i))
        cells[i], cells[j] = cells[j], cells[i]
    chosen = cells[:ns].astype(np.int64)
    vals = np.random.default_rng(seed).standard_normal(ns)
    return chosen // n, chosen % n, vals


def random_sampled(m, n, fill, seed):
    """test_util.hpp:80-82"""
    r, c, v = random_triplets(m, n, fill, seed)
    return O.sampled(m, n, r, c, v)
