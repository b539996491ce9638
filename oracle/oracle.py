"""TEST INFRASTRUCTURE ONLY — Python driver of the CPU parity oracle.

Wraps oracle/build/liboracle.so (the C++20 restatement in svt_oracle.hpp of
the reference's dense.hpp / sampled.hpp / sketch.hpp / solver.hpp).  Only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this
module; the product package never does.

Sampled matrices are passed as a `Csr` (m, n, rowptr int64, col int64, val
float64) — the reference's SampledMatrix storage (sampled.hpp:25-110).
Dense blocks are numpy arrays; they are converted to the reference's
column-major layout at the boundary.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from paper_1704_05528_b200._abi import (OBSERVER_FN, Backend, IterationRecord, SketchParams, StopRule,
                                        SvtConfig, raise_for)

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

P_I64 = C.POINTER(C.c_int64)
P_U64 = C.POINTER(C.c_uint64)
P_F64 = C.POINTER(C.c_double)


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.oracle_last_error.restype = C.c_char_p
        _lib.oracle_derive_seed.restype = C.c_uint64
        _lib.oracle_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        for name in ("oracle_qb_free", "oracle_factors_free", "oracle_result_free"):
            getattr(_lib, name).argtypes = [C.c_void_p]
    return _lib


def _check(code):
    raise_for(code, lib().oracle_last_error().decode())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, t=P_F64):
    return a.ctypes.data_as(t)


def _cm(a):
    """numpy 2-D -> column-major float64 buffer (Eigen layout)."""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _from_cm(buf, rows, cols):
    return np.asarray(buf, dtype=np.float64).reshape((cols, rows)).T.copy()


@dataclass
class Csr:
    """SampledMatrix (sampled.hpp:25-110): sorted row-major CSR, int64 indices."""
    m: int
    n: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self):
        return int(self.rowptr[-1])

    def args(self):
        return (C.c_int64(self.m), C.c_int64(self.n), _ptr(self.rowptr, P_I64), _ptr(self.col, P_I64),
                _ptr(self.val))

    def with_values(self, val):
        val = _f64(val)
        assert val.shape == self.val.shape
        return Csr(self.m, self.n, self.rowptr, self.col, val)

    def rows(self):
        return np.repeat(np.arange(self.m, dtype=np.int64), np.diff(self.rowptr))

    def dense(self):
        D = np.zeros((self.m, self.n))
        D[self.rows(), self.col] = self.val
        return D


def sampled(m, n, rows, cols, vals) -> Csr:
    """SampledMatrix(rows, cols, triplets) — validates and sorts (sampled.hpp:27-62)."""
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    vals = _f64(vals)
    nnz = len(vals)
    rp = np.zeros(max(m, 0) + 1, dtype=np.int64)
    co = np.zeros(max(nnz, 1), dtype=np.int64)
    va = np.zeros(max(nnz, 1), dtype=np.float64)
    _check(lib().oracle_sampled_build(C.c_int64(m), C.c_int64(n), C.c_int64(nnz), _ptr(rows, P_I64),
                                      _ptr(cols, P_I64), _ptr(vals), _ptr(rp, P_I64), _ptr(co, P_I64), _ptr(va)))
    return Csr(m, n, rp, co[:nnz].copy(), va[:nnz].copy())


def to_sampled(A) -> Csr:
    """synth.hpp:51-60 — fully observed pattern."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    r, c = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    return sampled(m, n, r.ravel(), c.ravel(), A.ravel())


def derive_seed(seed, stream):
    return int(lib().oracle_derive_seed(C.c_uint64(seed), C.c_uint64(stream)))


def mt19937_64(seed, n):
    out = np.zeros(n, dtype=np.uint64)
    lib().oracle_mt19937_64(C.c_uint64(seed), C.c_int64(n), _ptr(out, P_U64))
    return out


def gaussian_block(rows, cols, seed):
    out = np.zeros(max(rows * cols, 1))
    _check(lib().oracle_gaussian_block(C.c_int64(rows), C.c_int64(cols), C.c_uint64(seed), _ptr(out)))
    return _from_cm(out[: rows * cols], rows, cols)


def qr_orthonormal(X):
    X = _cm(X)
    rows, cols = X.shape
    Q = np.zeros(max(rows * cols, 1))
    _check(lib().oracle_qr_orthonormal(C.c_int64(rows), C.c_int64(cols), _ptr(X.ravel(order="F").copy()), _ptr(Q)))
    return _from_cm(Q[: rows * cols], rows, cols)


def small_svd(B):
    B = _cm(B)
    rows, cols = B.shape
    k = min(rows, cols)
    U = np.zeros(rows * k)
    s = np.zeros(k)
    V = np.zeros(cols * k)
    _check(lib().oracle_small_svd(C.c_int64(rows), C.c_int64(cols), _ptr(B.ravel(order="F").copy()), _ptr(U),
                                  _ptr(s), _ptr(V)))
    return _from_cm(U, rows, k), s, _from_cm(V, cols, k)


def sp_mult(S: Csr, X):
    X = _cm(X)
    xr, w = X.shape
    out = np.zeros(max(S.m * w, 1))
    _check(lib().oracle_sp_mult(*S.args(), C.c_int64(xr), C.c_int64(w), _ptr(X.ravel(order="F").copy()), _ptr(out)))
    return _from_cm(out[: S.m * w], S.m, w)


def sp_mult_t(S: Csr, X):
    X = _cm(X)
    xr, w = X.shape
    out = np.zeros(max(S.n * w, 1))
    _check(lib().oracle_sp_mult_t(*S.args(), C.c_int64(xr), C.c_int64(w), _ptr(X.ravel(order="F").copy()),
                                  _ptr(out)))
    return _from_cm(out[: S.n * w], S.n, w)


def project_low_rank(S: Csr, U, sigma, V):
    U = _cm(U)
    V = _cm(V)
    sigma = _f64(sigma)
    k = len(sigma)
    out = np.zeros(max(S.nnz, 1))
    _check(lib().oracle_project_low_rank(*S.args(), C.c_int64(U.shape[0]), C.c_int64(V.shape[0]), C.c_int64(k),
                                         _ptr(U.ravel(order="F").copy()), _ptr(sigma),
                                         _ptr(V.ravel(order="F").copy()), _ptr(out)))
    return out[: S.nnz]


def sp_frob_norm_sq(S: Csr):
    out = C.c_double()
    _check(lib().oracle_sp_frob_norm_sq(*S.args(), C.byref(out)))
    return out.value


def spectral_norm_est(S: Csr, iters, seed):
    out = C.c_double()
    _check(lib().oracle_spectral_norm_est(*S.args(), C.c_int(iters), C.c_uint64(seed), C.byref(out)))
    return out.value


def kickstart(A: Csr, tau, delta, seed) -> Csr:
    out = np.zeros(max(A.nnz, 1))
    _check(lib().oracle_kickstart(*A.args(), C.c_double(tau), C.c_double(delta), C.c_uint64(seed), _ptr(out)))
    return A.with_values(out[: A.nnz])


def default_config(A: Csr) -> SvtConfig:
    cfg = SvtConfig()
    _check(lib().oracle_default_config(*A.args(), C.byref(cfg)))
    return cfg


def error_percentage(frob_y_sq, norm_b_sq):
    out = C.c_double()
    _check(lib().oracle_error_percentage(C.c_double(frob_y_sq), C.c_double(norm_b_sq), C.byref(out)))
    return out.value


class QB:
    """QBState (sketch.hpp:32-39) handle: qb_init / qb_extend / finalize."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    @staticmethod
    def init(Y: Csr, t, np_, seed):
        h = C.c_void_p()
        _check(lib().oracle_qb_init(*Y.args(), C.c_int64(t), C.c_int(np_), C.c_uint64(seed), C.byref(h)))
        return QB(h.value)

    def extend(self, Y: Csr, dt, np_, seed):
        _check(lib().oracle_qb_extend(self.h, *Y.args(), C.c_int64(dt), C.c_int(np_), C.c_uint64(seed)))
        return self

    def info(self):
        rank, sat, nb, fy, qr, bc = C.c_int64(), C.c_int(), C.c_double(), C.c_double(), C.c_int64(), C.c_int64()
        lib().oracle_qb_info(self.h, C.byref(rank), C.byref(sat), C.byref(nb), C.byref(fy), C.byref(qr), C.byref(bc))
        return dict(rank=rank.value, saturated=bool(sat.value), norm_b_sq=nb.value, frob_y_sq=fy.value,
                    q_rows=qr.value, b_cols=bc.value)

    def QB(self):
        i = self.info()
        Q = np.zeros(max(i["q_rows"] * i["rank"], 1))
        B = np.zeros(max(i["rank"] * i["b_cols"], 1))
        lib().oracle_qb_copy(self.h, _ptr(Q), _ptr(B))
        return (_from_cm(Q[: i["q_rows"] * i["rank"]], i["q_rows"], i["rank"]),
                _from_cm(B[: i["rank"] * i["b_cols"]], i["rank"], i["b_cols"]))

    def error_percentage(self):
        out = C.c_double()
        _check(lib().oracle_qb_error_percentage(self.h, C.byref(out)))
        return out.value

    def finalize(self):
        i = self.info()
        r, m, n = i["rank"], i["q_rows"], i["b_cols"]
        k = min(r, n)
        U = np.zeros(max(m * k, 1))
        s = np.zeros(max(k, 1))
        V = np.zeros(max(n * k, 1))
        _check(lib().oracle_qb_finalize(self.h, _ptr(U), _ptr(s), _ptr(V)))
        return _from_cm(U[: m * k], m, k), s[:k], _from_cm(V[: n * k], n, k)

    def __del__(self):
        try:
            if self.h:
                lib().oracle_qb_free(self.h)
        except Exception:
            pass


@dataclass
class SketchResult:
    """sketch.hpp:41-46"""
    U: np.ndarray
    sigma: np.ndarray
    V: np.ndarray
    rank: int
    saturated: bool
    extension_rounds: int


def _take_factors(h):
    urows, vrows, k, rank, sat, rounds = (C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int(),
                                          C.c_int())
    L = lib()
    L.oracle_factors_info(h, C.byref(urows), C.byref(vrows), C.byref(k), C.byref(rank), C.byref(sat),
                          C.byref(rounds))
    kk = k.value
    U = np.zeros(max(urows.value * kk, 1))
    s = np.zeros(max(kk, 1))
    V = np.zeros(max(vrows.value * kk, 1))
    L.oracle_factors_copy(h, _ptr(U), _ptr(s), _ptr(V))
    L.oracle_factors_free(h)
    return SketchResult(_from_cm(U[: urows.value * kk], urows.value, kk), s[:kk],
                        _from_cm(V[: vrows.value * kk], vrows.value, kk), rank.value, bool(sat.value), rounds.value)


def rsvd(Y: Csr, k, p: SketchParams):
    h = C.c_void_p()
    _check(lib().oracle_rsvd(*Y.args(), C.c_int64(k), C.byref(p), C.byref(h)))
    return _take_factors(h)


def r3svd(Y: Csr, p: SketchParams):
    h = C.c_void_p()
    _check(lib().oracle_r3svd(*Y.args(), C.byref(p), C.byref(h)))
    return _take_factors(h)


def r4svd(Y: Csr, U_prev, p: SketchParams):
    U_prev = _cm(U_prev)
    s = U_prev.shape[1]
    buf = U_prev.ravel(order="F").copy() if U_prev.size else np.zeros(1)
    h = C.c_void_p()
    _check(lib().oracle_r4svd(*Y.args(), C.c_int64(s), _ptr(buf), C.byref(p), C.byref(h)))
    return _take_factors(h)


@dataclass
class SvtResult:
    """solver.hpp:80-84"""
    U: np.ndarray
    sigma: np.ndarray
    V: np.ndarray
    trace: list
    converged: bool


def svt_run_backend(A: Csr, cfg: SvtConfig, stop: StopRule, backend: Backend, observer=None, test: Csr = None,
                    start=None):
    """solver.hpp:215-328.  observer(rec_dict, U, sigma, V) -> bool (False stops).
    start (test-harness extension): dict(iter, y_vals, u_prev (m x s array),
    eps_threshold, eps_min) — continue after `iter` completed iterations
    from that state (the product's svt_solver_checkpoint state) instead of
    the kickstart."""
    cb = None
    if observer is not None:
        def _obs(rec, m_local, n, k, U, sigma, V, user):
            r = rec.contents.as_dict()
            Uk = np.ctypeslib.as_array(U, shape=(m_local * k,)).copy() if k else np.zeros(0)
            sk = np.ctypeslib.as_array(sigma, shape=(k,)).copy() if k else np.zeros(0)
            Vk = np.ctypeslib.as_array(V, shape=(n * k,)).copy() if k else np.zeros(0)
            return 1 if observer(r, _from_cm(Uk, m_local, k), sk, _from_cm(Vk, n, k)) else 0
        cb = OBSERVER_FN(_obs)
    h = C.c_void_p()
    if test is not None:
        targs = (C.c_int64(test.nnz), _ptr(test.rowptr, P_I64), _ptr(test.col, P_I64), _ptr(test.val))
    else:
        targs = (C.c_int64(0), None, None, None)
    if start is None:
        sargs = (C.c_int(-1), None, C.c_int64(0), None, C.c_double(0.0), C.c_double(0.0))
    else:
        y = _f64(start["y_vals"])
        assert y.size >= A.nnz
        up = np.asarray(start["u_prev"], dtype=np.float64).reshape(A.m, -1)
        upc = _cm(up) if up.size else np.zeros(1)
        sargs = (C.c_int(int(start["iter"])), _ptr(y), C.c_int64(up.shape[1]), _ptr(upc.ravel(order="K")),
                 C.c_double(start["eps_threshold"]), C.c_double(start["eps_min"]))
    _check(lib().oracle_svt_resume(*A.args(), C.byref(cfg), stop, backend, *targs,
                                   cb, None, *sargs, C.byref(h)))
    L = lib()
    nrec, urows, vrows, k, conv = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
    L.oracle_result_info(h, C.byref(nrec), C.byref(urows), C.byref(vrows), C.byref(k), C.byref(conv))
    recs = (IterationRecord * max(nrec.value, 1))()
    L.oracle_result_trace(h, recs)
    kk = k.value
    U = np.zeros(max(urows.value * kk, 1))
    s = np.zeros(max(kk, 1))
    V = np.zeros(max(vrows.value * kk, 1))
    L.oracle_result_factors(h, _ptr(U), _ptr(s), _ptr(V))
    L.oracle_result_free(h)
    trace = [recs[i].as_dict() for i in range(nrec.value)]
    return SvtResult(_from_cm(U[: urows.value * kk], urows.value, kk), s[:kk],
                     _from_cm(V[: vrows.value * kk], vrows.value, kk), trace, bool(conv.value))


def svt_run(A, cfg, stop, observer=None, test=None, start=None):
    """solver.hpp:333-336"""
    return svt_run_backend(A, cfg, stop, Backend.r4svd(), observer, test, start)


def svt_run_oracle(A, cfg, stop, observer=None, test=None):
    """solver.hpp:340-343"""
    return svt_run_backend(A, cfg, stop, Backend.full_svd(), observer, test)


# --- restated synth.hpp / io.hpp helpers used by the reference tests --------------
def sample_positions(total, ns, seed):
    out = np.zeros(max(ns, 1), dtype=np.uint64)
    _check(lib().oracle_sample_positions(C.c_uint64(total), C.c_uint64(ns), C.c_uint64(seed), _ptr(out, P_U64)))
    return out[:ns]


def make_low_rank(m, n, rank, seed):
    out = np.zeros(m * n)
    _check(lib().oracle_make_low_rank(C.c_int64(m), C.c_int64(n), C.c_int64(rank), C.c_uint64(seed), _ptr(out)))
    return _from_cm(out, m, n)


def make_geometric(m, n, count, ratio, seed):
    out = np.zeros(m * n)
    _check(lib().oracle_make_geometric(C.c_int64(m), C.c_int64(n), C.c_int64(count), C.c_double(ratio),
                                       C.c_uint64(seed), _ptr(out)))
    return _from_cm(out, m, n)


def sample_dense(A, fraction, seed) -> Csr:
    """synth.hpp:63-82"""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    total = m * n
    ns = int(np.floor(fraction * total + 1e-9))
    pos = sample_positions(total, ns, seed).astype(np.int64)
    r, c = pos // n, pos % n
    return sampled(m, n, r, c, A[r, c])


def random_triplets(m, n, fill, seed):
    """proj/tests/test_util.hpp:56-78, exactly: the mt19937_64 partial
    Fisher-Yates over all cells, then std::normal_distribution values from
    the same engine (libstdc++)."""
    cnt = C.c_int64()
    _check(lib().oracle_random_triplets(C.c_int64(m), C.c_int64(n), C.c_double(fill), C.c_uint64(seed),
                                        C.byref(cnt), None, None, None))
    k = cnt.value
    r, c, v = np.zeros(k, np.int64), np.zeros(k, np.int64), np.zeros(k)
    _check(lib().oracle_random_triplets(C.c_int64(m), C.c_int64(n), C.c_double(fill), C.c_uint64(seed),
                                        C.byref(cnt), _ptr(r, P_I64), _ptr(c, P_I64), _ptr(v)))
    return r, c, v


def num_threads():
    """Host threads the oracle's parallel loops use (OMP_NUM_THREADS)."""
    return int(lib().oracle_num_threads())


def synth_config(config, seed=1):
    """The BASELINE config generators (the shared csrc/synth.cpp, compiled
    into liboracle.so): dict(m, n, train=Csr, test=Csr or None); config 5
    has no test set."""
    L = lib()
    m, n = C.c_int64(), C.c_int64()
    if config == 5:
        nnz = C.c_int64()
        _check(L.oracle_synth_config_csr(C.c_int(5), C.c_uint64(seed), C.byref(m), C.byref(n), C.byref(nnz),
                                         None, None, None))
        rp = np.zeros(m.value + 1, dtype=np.int64)
        co = np.zeros(nnz.value, dtype=np.int64)
        va = np.zeros(nnz.value)
        _check(L.oracle_synth_config_csr(C.c_int(5), C.c_uint64(seed), C.byref(m), C.byref(n), C.byref(nnz),
                                         _ptr(rp, P_I64), _ptr(co, P_I64), _ptr(va)))
        return dict(m=m.value, n=n.value, train=Csr(m.value, n.value, rp, co, va), test=None)
    ntr, nte = C.c_int64(), C.c_int64()
    _check(L.oracle_synth_config(C.c_int(config), C.c_uint64(seed), C.byref(m), C.byref(n), C.byref(ntr),
                                 C.byref(nte), None, None, None, None, None, None))
    tr = [np.zeros(ntr.value, np.int64), np.zeros(ntr.value, np.int64), np.zeros(ntr.value)]
    te = [np.zeros(max(nte.value, 1), np.int64), np.zeros(max(nte.value, 1), np.int64), np.zeros(max(nte.value, 1))]
    _check(L.oracle_synth_config(C.c_int(config), C.c_uint64(seed), C.byref(m), C.byref(n), C.byref(ntr),
                                 C.byref(nte), _ptr(tr[0], P_I64), _ptr(tr[1], P_I64), _ptr(tr[2]),
                                 _ptr(te[0], P_I64), _ptr(te[1], P_I64), _ptr(te[2])))
    train = sampled(m.value, n.value, *tr)
    test = sampled(m.value, n.value, *(a[: nte.value] for a in te)) if nte.value else None
    return dict(m=m.value, n=n.value, train=train, test=test)


def config_params(config, nnz, m, n, frob_a):
    """The BASELINE.json parameters of each config,
    restated from paper_1704_05528_b200.api.config_params so the CPU arms and
    the fixture script need only this library (a CPU test asserts the two
    agree).  Returns (SvtConfig, StopRule)."""
    cfg = SvtConfig()
    cfg.t0 = max(1, int(0.05 * min(m, n)))
    cfg.dt = 10
    cfg.beta = 0.95
    p = nnz / float(m * n)
    if config == 1:
        cfg.tau, cfg.delta = 5.0 * n, 1.2 / p
        cfg.eps_threshold0, cfg.eps_threshold_min = 1e-2, 1e-6
        cfg.rel_residual_stop = 1e-4
    elif config == 2:
        cfg.tau, cfg.delta = 5.0 * np.sqrt(m * n), 1.2 / p
        cfg.rel_residual_stop = 1e-4
    elif config in (3, 4):
        cfg.tau, cfg.delta = frob_a, 1.9
    elif config == 5:
        cfg.tau, cfg.delta = 5.0 * n, 1.2 / p
        cfg.maxit = 30
    else:
        raise ValueError("config must be 1..5")
    return cfg, StopRule.none()
