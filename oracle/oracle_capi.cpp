// TEST INFRASTRUCTURE ONLY — ctypes-facing C API over the CPU oracle
// (svt_oracle.hpp).  Loaded by tests/ and bench.py's CPU-baseline legs only.
// Structs are shared with the product boundary (include/svt_b200.h) so both
// sides are driven with byte-identical parameters.
#ifdef _OPENMP
#include <omp.h>
#endif
#include "svt_oracle.hpp"

#include "../include/svt_b200.h"

#include <cstring>
#include <memory>
#include <random>
#include <string>

using namespace svt_oracle;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return SVT_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SVT_EINVAL;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return SVT_EDOMAIN;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SVT_ERUNTIME;
    }
}

Mat from_col_major(int64_t rows, int64_t cols, const double* p) {
    Mat m(rows, cols);
    if (rows * cols > 0) std::memcpy(m.a.data(), p, sizeof(double) * static_cast<size_t>(rows * cols));
    return m;
}

void to_col_major(const Mat& m, double* out) {
    if (!m.a.empty()) std::memcpy(out, m.a.data(), sizeof(double) * m.a.size());
}

SampledMatrix csr(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val) {
    const int64_t nnz = rowptr[m];
    return SampledMatrix(m, n, std::vector<Index>(rowptr, rowptr + m + 1), std::vector<Index>(col, col + nnz),
                         std::vector<double>(val, val + nnz));
}

SketchParams sp_of(const svt_sketch_params* p) {
    SketchParams s;
    s.t = p->t;
    s.dt = p->dt;
    s.np = p->np;
    s.eps_threshold = p->eps_threshold;
    s.seed = p->seed;
    s.p = p->p;
    return s;
}

struct OFactors {
    LowRankFactors f;
    Index rank = 0;
    bool saturated = false;
    int rounds = 0;
};

struct OResult {
    SvtResult r;
};

}  // namespace

struct oracle_qb {
    QBState st;
};

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

uint64_t oracle_derive_seed(uint64_t seed, uint64_t stream) { return derive_seed(seed, stream); }

void oracle_mt19937_64(uint64_t seed, int64_t n, uint64_t* out) {
    std::mt19937_64 g(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = g();
}

int oracle_gaussian_block(int64_t rows, int64_t cols, uint64_t seed, double* out) {
    return guard([&] { to_col_major(gaussian_block(rows, cols, seed), out); });
}

int oracle_qr_orthonormal(int64_t rows, int64_t cols, const double* X, double* Q) {
    return guard([&] { to_col_major(qr_orthonormal(from_col_major(rows, cols, X)), Q); });
}

int oracle_small_svd(int64_t rows, int64_t cols, const double* B, double* U, double* sigma, double* V) {
    return guard([&] {
        LowRankFactors f = small_svd(from_col_major(rows, cols, B));
        to_col_major(f.U, U);
        std::memcpy(sigma, f.sigma.data(), sizeof(double) * f.sigma.size());
        to_col_major(f.V, V);
    });
}

int oracle_sampled_build(int64_t m, int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                         const double* vals, int64_t* rowptr_out, int64_t* col_out, double* val_out) {
    return guard([&] {
        std::vector<Triplet> ts(static_cast<size_t>(nnz));
        for (int64_t k = 0; k < nnz; ++k) ts[static_cast<size_t>(k)] = {rows[k], cols[k], vals[k]};
        SampledMatrix S(m, n, std::move(ts));
        std::memcpy(rowptr_out, S.row_offsets().data(), sizeof(int64_t) * static_cast<size_t>(m + 1));
        std::memcpy(col_out, S.col_index().data(), sizeof(int64_t) * static_cast<size_t>(nnz));
        std::memcpy(val_out, S.values().data(), sizeof(double) * static_cast<size_t>(nnz));
    });
}

int oracle_sp_mult(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val, int64_t xr,
                   int64_t w, const double* X, double* out) {
    return guard([&] { to_col_major(sp_mult(csr(m, n, rowptr, col, val), from_col_major(xr, w, X)), out); });
}

int oracle_sp_mult_t(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val, int64_t xr,
                     int64_t w, const double* X, double* out) {
    return guard([&] { to_col_major(sp_mult_t(csr(m, n, rowptr, col, val), from_col_major(xr, w, X)), out); });
}

int oracle_project_low_rank(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
                            int64_t ur, int64_t vr, int64_t k, const double* U, const double* sigma, const double* V,
                            double* out_vals) {
    return guard([&] {
        LowRankFactors F{from_col_major(ur, k, U), std::vector<double>(sigma, sigma + k), from_col_major(vr, k, V)};
        SampledMatrix P = project_low_rank(csr(m, n, rowptr, col, val), F);
        std::memcpy(out_vals, P.values().data(), sizeof(double) * P.values().size());
    });
}

int oracle_sp_frob_norm_sq(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
                           double* out) {
    return guard([&] { *out = sp_frob_norm_sq(csr(m, n, rowptr, col, val)); });
}

int oracle_spectral_norm_est(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
                             int iters, uint64_t seed, double* out) {
    return guard([&] { *out = spectral_norm_est(csr(m, n, rowptr, col, val), iters, seed); });
}

int oracle_kickstart(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val, double tau,
                     double delta, uint64_t seed, double* out_vals) {
    return guard([&] {
        SampledMatrix Y = kickstart(csr(m, n, rowptr, col, val), tau, delta, seed);
        std::memcpy(out_vals, Y.values().data(), sizeof(double) * Y.values().size());
    });
}

int oracle_default_config(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
                          svt_config* out) {
    return guard([&] {
        SvtConfig c = default_config(csr(m, n, rowptr, col, val));
        out->tau = c.tau;
        out->delta = c.delta;
        out->maxit = c.maxit;
        out->np = c.np;
        out->dt = c.dt;
        out->eps_stop = c.eps_stop;
        out->eps_threshold0 = c.eps_threshold0;
        out->beta = c.beta;
        out->t0 = c.t0;
        out->seed = c.seed;
        out->eps_threshold_min = c.eps_threshold_min;
        out->rel_residual_stop = c.rel_residual_stop;
    });
}

// --- QB state ---------------------------------------------------------------
int oracle_qb_init(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val, int64_t t,
                   int np, uint64_t seed, oracle_qb** out) {
    return guard([&] {
        auto h = std::make_unique<oracle_qb>();
        h->st = qb_init(csr(m, n, rowptr, col, val), t, np, seed);
        *out = h.release();
    });
}

int oracle_qb_extend(oracle_qb* h, int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col,
                     const double* val, int64_t dt, int np, uint64_t seed) {
    return guard([&] { h->st = qb_extend(std::move(h->st), csr(m, n, rowptr, col, val), dt, np, seed); });
}

void oracle_qb_info(oracle_qb* h, int64_t* rank, int* saturated, double* norm_b_sq, double* frob_y_sq,
                    int64_t* q_rows, int64_t* b_cols) {
    *rank = h->st.rank;
    *saturated = h->st.saturated ? 1 : 0;
    *norm_b_sq = h->st.norm_b_sq;
    *frob_y_sq = h->st.frob_y_sq;
    *q_rows = h->st.Q.rows;
    *b_cols = h->st.Bt.rows;
}

void oracle_qb_copy(oracle_qb* h, double* Q, double* B) {
    to_col_major(h->st.Q, Q);
    to_col_major(transpose(h->st.Bt), B);
}

int oracle_qb_error_percentage(oracle_qb* h, double* out) {
    return guard([&] { *out = error_percentage(h->st); });
}

int oracle_error_percentage(double frob_y_sq, double norm_b_sq, double* out) {
    return guard([&] {
        QBState st;
        st.frob_y_sq = frob_y_sq;
        st.norm_b_sq = norm_b_sq;
        *out = error_percentage(st);
    });
}

int oracle_qb_finalize(oracle_qb* h, double* U, double* sigma, double* V) {
    return guard([&] {
        LowRankFactors f = finalize(h->st);
        to_col_major(f.U, U);
        std::memcpy(sigma, f.sigma.data(), sizeof(double) * f.sigma.size());
        to_col_major(f.V, V);
    });
}

void oracle_qb_free(oracle_qb* h) { delete h; }

// --- engines ------------------------------------------------------------------
int oracle_rsvd(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val, int64_t k,
                const svt_sketch_params* p, void** out) {
    return guard([&] {
        auto h = std::make_unique<OFactors>();
        h->f = rsvd(csr(m, n, rowptr, col, val), k, sp_of(p));
        h->rank = k;
        *out = h.release();
    });
}

int oracle_r3svd(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
                 const svt_sketch_params* p, void** out) {
    return guard([&] {
        auto h = std::make_unique<OFactors>();
        SketchResult r = r3svd(csr(m, n, rowptr, col, val), sp_of(p));
        h->f = std::move(r.factors);
        h->rank = r.rank;
        h->saturated = r.saturated;
        h->rounds = r.extension_rounds;
        *out = h.release();
    });
}

int oracle_r4svd(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val, int64_t s,
                 const double* U_prev, const svt_sketch_params* p, void** out) {
    return guard([&] {
        auto h = std::make_unique<OFactors>();
        SketchResult r = r4svd(csr(m, n, rowptr, col, val), from_col_major(m, s, U_prev), sp_of(p));
        h->f = std::move(r.factors);
        h->rank = r.rank;
        h->saturated = r.saturated;
        h->rounds = r.extension_rounds;
        *out = h.release();
    });
}

void oracle_factors_info(void* hv, int64_t* urows, int64_t* vrows, int64_t* k, int64_t* rank, int* saturated,
                         int* rounds) {
    auto* h = static_cast<OFactors*>(hv);
    *urows = h->f.U.rows;
    *vrows = h->f.V.rows;
    *k = h->f.rank();
    *rank = h->rank;
    *saturated = h->saturated ? 1 : 0;
    *rounds = h->rounds;
}

void oracle_factors_copy(void* hv, double* U, double* sigma, double* V) {
    auto* h = static_cast<OFactors*>(hv);
    to_col_major(h->f.U, U);
    if (!h->f.sigma.empty()) std::memcpy(sigma, h->f.sigma.data(), sizeof(double) * h->f.sigma.size());
    to_col_major(h->f.V, V);
}

void oracle_factors_free(void* hv) { delete static_cast<OFactors*>(hv); }

// --- solver -------------------------------------------------------------------
int oracle_svt_resume(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
                      const svt_config* c, svt_stop stop, svt_backend backend, int64_t test_nnz,
                      const int64_t* test_rowptr, const int64_t* test_col, const double* test_val,
                      svt_observer_fn obs, void* user, int start_iter, const double* y_vals, int64_t s,
                      const double* u_prev, double eps_threshold, double eps_min, void** out);

int oracle_svt_run(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
                   const svt_config* c, svt_stop stop, svt_backend backend, int64_t test_nnz,
                   const int64_t* test_rowptr, const int64_t* test_col, const double* test_val, svt_observer_fn obs,
                   void* user, void** out) {
    return oracle_svt_resume(m, n, rowptr, col, val, c, stop, backend, test_nnz, test_rowptr, test_col, test_val,
                             obs, user, -1, nullptr, 0, nullptr, 0.0, 0.0, out);
}

// start_iter < 0: from the kickstart; else continue after `start_iter`
// completed iterations from (Y values, U_prev m x s column-major, cooling
// threshold, running residual minimum) — svt_solver_checkpoint's state.
int oracle_svt_resume(int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
                      const svt_config* c, svt_stop stop, svt_backend backend, int64_t test_nnz,
                      const int64_t* test_rowptr, const int64_t* test_col, const double* test_val,
                      svt_observer_fn obs, void* user, int start_iter, const double* y_vals, int64_t s,
                      const double* u_prev, double eps_threshold, double eps_min, void** out) {
    return guard([&] {
        SvtConfig cfg;
        cfg.tau = c->tau;
        cfg.delta = c->delta;
        cfg.maxit = c->maxit;
        cfg.np = c->np;
        cfg.dt = c->dt;
        cfg.eps_stop = c->eps_stop;
        cfg.eps_threshold0 = c->eps_threshold0;
        cfg.beta = c->beta;
        cfg.t0 = c->t0;
        cfg.seed = c->seed;
        cfg.eps_threshold_min = c->eps_threshold_min;
        cfg.rel_residual_stop = c->rel_residual_stop;
        StopRule sr;
        sr.kind = static_cast<StopRule::Kind>(stop.kind);
        sr.threshold = stop.threshold;
        Backend be;
        be.kind = static_cast<Backend::Kind>(backend.kind);
        be.fixed_rank = backend.fixed_rank;
        IterationObserver observer;
        if (obs != nullptr) {
            observer = [&](const IterationRecord& r, const LowRankFactors& X) {
                svt_record rec{};
                rec.iter = r.iter;
                rec.extension_rounds = r.extension_rounds;
                rec.rank = r.rank;
                rec.residual = r.residual;
                rec.eps_threshold = r.eps_threshold;
                rec.train_mae = r.train_mae;
                rec.sketch_ms = r.sketch_ms;
                rec.total_ms = r.total_ms;
                rec.kept = r.kept;
                rec.rel_residual_x = r.rel_residual_x;
                rec.test_mae = r.test_mae;
                rec.test_rmse = r.test_rmse;
                return obs(&rec, X.U.rows, X.V.rows, X.rank(), X.U.a.data(), X.sigma.data(), X.V.a.data(), user) != 0;
            };
        }
        SampledMatrix A = csr(m, n, rowptr, col, val);
        std::unique_ptr<SampledMatrix> test;
        if (test_nnz > 0) test = std::make_unique<SampledMatrix>(csr(m, n, test_rowptr, test_col, test_val));
        std::unique_ptr<SvtStart> start;
        if (start_iter >= 0) {
            start = std::make_unique<SvtStart>();
            start->iter = start_iter;
            start->y.assign(y_vals, y_vals + A.nnz());
            start->U_prev = from_col_major(m, s, u_prev);
            start->eps_threshold = eps_threshold;
            start->eps_min = eps_min;
        }
        auto h = std::make_unique<OResult>();
        h->r = svt_run_backend(A, cfg, sr, be, observer, test.get(), start.get());
        *out = h.release();
    });
}

void oracle_result_info(void* hv, int64_t* n_records, int64_t* urows, int64_t* vrows, int64_t* k, int* converged) {
    auto* h = static_cast<OResult*>(hv);
    *n_records = static_cast<int64_t>(h->r.trace.size());
    *urows = h->r.factors.U.rows;
    *vrows = h->r.factors.V.rows;
    *k = h->r.factors.rank();
    *converged = h->r.converged ? 1 : 0;
}

void oracle_result_trace(void* hv, svt_record* out) {
    auto* h = static_cast<OResult*>(hv);
    for (size_t i = 0; i < h->r.trace.size(); ++i) {
        const IterationRecord& r = h->r.trace[i];
        svt_record rec{};
        rec.iter = r.iter;
        rec.extension_rounds = r.extension_rounds;
        rec.rank = r.rank;
        rec.residual = r.residual;
        rec.eps_threshold = r.eps_threshold;
        rec.train_mae = r.train_mae;
        rec.sketch_ms = r.sketch_ms;
        rec.total_ms = r.total_ms;
        rec.kept = r.kept;
        rec.rel_residual_x = r.rel_residual_x;
        rec.test_mae = r.test_mae;
        rec.test_rmse = r.test_rmse;
        out[i] = rec;
    }
}

void oracle_result_factors(void* hv, double* U, double* sigma, double* V) {
    auto* h = static_cast<OResult*>(hv);
    to_col_major(h->r.factors.U, U);
    if (!h->r.factors.sigma.empty())
        std::memcpy(sigma, h->r.factors.sigma.data(), sizeof(double) * h->r.factors.sigma.size());
    to_col_major(h->r.factors.V, V);
}

void oracle_result_free(void* hv) { delete static_cast<OResult*>(hv); }

// --- restated synth.hpp / io.hpp helpers used by the reference's tests ----------
// io.hpp:93-96
static uint64_t bounded(std::mt19937_64& rng, uint64_t n) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(rng()) * static_cast<unsigned __int128>(n)) >> 64);
}

// io.hpp:100-113
int oracle_sample_positions(uint64_t total, uint64_t ns, uint64_t seed, uint64_t* out) {
    return guard([&] {
        std::vector<uint64_t> idx(total);
        for (uint64_t i = 0; i < total; ++i) idx[i] = i;
        std::mt19937_64 rng(seed);
        for (uint64_t i = 0; i < ns; ++i) {
            const uint64_t j = i + bounded(rng, total - i);
            std::swap(idx[i], idx[j]);
        }
        std::memcpy(out, idx.data(), sizeof(uint64_t) * ns);
    });
}

// synth.hpp:21-28
int oracle_make_low_rank(int64_t m, int64_t n, int64_t rank, uint64_t seed, double* out) {
    return guard([&] {
        if (rank < 1 || rank > std::min(m, n)) throw std::invalid_argument("make_low_rank: rank out of range");
        const Mat G1 = gaussian_block(m, rank, derive_seed(seed, 0));
        const Mat G2 = gaussian_block(n, rank, derive_seed(seed, 1));
        Mat A = mul_nn(G1, transpose(G2));
        const double s = std::sqrt(static_cast<double>(rank));
        for (double& v : A.a) v /= s;
        to_col_major(A, out);
    });
}

// synth.hpp:32-48
int oracle_make_geometric(int64_t m, int64_t n, int64_t count, double ratio, uint64_t seed, double* out) {
    return guard([&] {
        if (count < 1 || count > std::min(m, n)) throw std::invalid_argument("make_geometric: count out of range");
        if (!(ratio > 0.0 && ratio < 1.0)) throw std::invalid_argument("make_geometric: ratio must lie in (0, 1)");
        const Mat U = qr_orthonormal(gaussian_block(m, count, derive_seed(seed, 0)));
        Mat V = qr_orthonormal(gaussian_block(n, count, derive_seed(seed, 1)));
        double s = 1.0;
        for (int64_t j = 0; j < count; ++j, s *= ratio)
            for (int64_t i = 0; i < n; ++i) V(i, j) *= s;
        to_col_major(mul_nn(U, transpose(V)), out);
    });
}

// proj/tests/test_util.hpp:56-78 — random_triplets: partial Fisher-Yates
// over all m*n cells with `rng() % (cells - i)`, then the values from
// std::normal_distribution<double>(0, 1) on the same engine (libstdc++'s
// algorithm: the reference tests' own inputs are reproduced exactly when
// built with the same standard library, as both sides are here).
int oracle_random_triplets(int64_t m, int64_t n, double fill, uint64_t seed, int64_t* count, int64_t* rows,
                           int64_t* cols, double* vals) {
    return guard([&] {
        std::mt19937_64 rng(seed);
        std::vector<uint64_t> cells(static_cast<size_t>(m) * static_cast<size_t>(n));
        for (size_t i = 0; i < cells.size(); ++i) cells[i] = i;
        size_t ns = static_cast<size_t>(fill * static_cast<double>(cells.size()));
        if (ns < 1) ns = 1;
        *count = static_cast<int64_t>(ns);
        if (rows == nullptr) return;
        for (size_t i = 0; i < ns; ++i) {
            const size_t j = i + static_cast<size_t>(rng() % (cells.size() - i));
            std::swap(cells[i], cells[j]);
        }
        std::normal_distribution<double> gauss(0.0, 1.0);
        for (size_t i = 0; i < ns; ++i) {
            rows[i] = static_cast<int64_t>(cells[i] / static_cast<uint64_t>(n));
            cols[i] = static_cast<int64_t>(cells[i] % static_cast<uint64_t>(n));
            vals[i] = gauss(rng);
        }
    });
}

}  // extern "C"

// --- the BASELINE config generators (paper_1704_05528_b200/csrc/synth.cpp,
// compiled into this library too: one shared generator for both sides, so
// the CPU arms never load the product library)
namespace svtb {
using i64 = std::int64_t;
using u64 = std::uint64_t;
u64 derive_seed_u(u64 seed, u64 stream) { return svt_oracle::derive_seed(seed, stream); }
void synth_config(int config, u64 seed, i64* m, i64* n, i64* nnz_train, i64* nnz_test, i64* train_rows,
                  i64* train_cols, double* train_vals, i64* test_rows, i64* test_cols, double* test_vals);
void synth_config_csr(int config, u64 seed, i64* m, i64* n, i64* nnz, i64* rowptr, i64* col, double* val);
}  // namespace svtb

extern "C" int oracle_synth_config(int config, uint64_t seed, int64_t* m, int64_t* n, int64_t* nnz_train,
                                   int64_t* nnz_test, int64_t* train_rows, int64_t* train_cols, double* train_vals,
                                   int64_t* test_rows, int64_t* test_cols, double* test_vals) {
    return guard([&] {
        svtb::synth_config(config, seed, m, n, nnz_train, nnz_test, train_rows, train_cols, train_vals, test_rows,
                           test_cols, test_vals);
    });
}

extern "C" int oracle_synth_config_csr(int config, uint64_t seed, int64_t* m, int64_t* n, int64_t* nnz,
                                       int64_t* rowptr, int64_t* col, double* val) {
    return guard([&] { svtb::synth_config_csr(config, seed, m, n, nnz, rowptr, col, val); });
}

extern "C" int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
