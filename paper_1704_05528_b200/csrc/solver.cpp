// The SVT Bregman iteration (solver.hpp:215-328) on the device.
//
// Per iteration: partial SVD of Y (R3SVD at iteration 1, R4SVD after, with
// finalize computing only the triplets shrink keeps), then ONE fused
// SDDMM + update kernel that produces train MAE, ||P(X - A)||, the dual
// residual ||A - Y|| on the pre-update iterate, ||Y_new||^2 (the next
// sketch's frob_y_sq) and writes Y_new + its CSC mirror — replacing the
// reference's two project_low_rank passes, two sp_axpy passes, residual and
// train_mae (solver.hpp:279, 287, 321-323).  Cooling, best-so-far, stop rule
// and observer are host logic in the reference's order.
#include <nvtx3/nvToolsExt.h>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>

#include "engine.hpp"
#include "kernels.hpp"

namespace svtb {

namespace {

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

enum : int { S_SUMS = 8, S_TSUMS = 12, S_FA = 20 };

void check_config(const svt_config& cfg) {  // solver.hpp:186-205
    if (!(cfg.tau > 0.0)) throw std::invalid_argument("SvtConfig: tau must be positive");
    if (!(cfg.delta > 0.0)) throw std::invalid_argument("SvtConfig: delta must be positive");
    if (!(cfg.beta > 0.0 && cfg.beta < 1.0)) throw std::invalid_argument("SvtConfig: beta must lie in (0, 1)");
    if (!(cfg.eps_threshold0 > 0.0 && cfg.eps_threshold0 < 1.0))
        throw std::invalid_argument("SvtConfig: eps_threshold0 must lie in (0, 1)");
    if (cfg.maxit < 1) throw std::invalid_argument("SvtConfig: maxit must be >= 1");
    if (cfg.t0 < 1 || cfg.dt < 1 || cfg.np < 0) throw std::invalid_argument("SvtConfig: need t0 >= 1, dt >= 1, np >= 0");
}

// leading triplets with sigma > tau, shifted by tau (solver.hpp:110-120)
void shrink_into(svt_ctx* c, const DevFactors& f, double tau, DevFactors& out) {
    i64 keep = 0;
    while (keep < f.k && f.sigma[static_cast<size_t>(keep)] > tau) ++keep;
    out.m_local = f.m_local;
    out.n = f.n;
    out.k = keep;
    out.sigma.resize(static_cast<size_t>(keep));
    for (i64 j = 0; j < keep; ++j) out.sigma[static_cast<size_t>(j)] = f.sigma[static_cast<size_t>(j)] - tau;
    if (keep == 0) return;
    out.U.ensure(static_cast<size_t>(std::max<i64>(1, f.m_local) * std::max<i64>(keep, factor_cols(f.m_local + f.n, f.n))));
    out.V.ensure(static_cast<size_t>(f.n * std::max<i64>(keep, factor_cols(f.m_local + f.n, f.n))));
    copy2d(c, f.U.get(), f.k, out.U.get(), keep, f.m_local, keep);
    copy2d(c, f.V.get(), f.k, out.V.get(), keep, f.n, keep);
}

void copy_factors(svt_ctx* c, const DevFactors& f, DevFactors& out) {
    out.m_local = f.m_local;
    out.n = f.n;
    out.k = f.k;
    out.sigma = f.sigma;
    if (f.k == 0) return;
    out.U.ensure(static_cast<size_t>(std::max<i64>(1, f.m_local) * std::max<i64>(f.k, factor_cols(f.m_local + f.n, f.n))));
    out.V.ensure(static_cast<size_t>(f.n * std::max<i64>(f.k, factor_cols(f.m_local + f.n, f.n))));
    SVT_CUDA(cudaMemcpyAsync(out.U.get(), f.U.get(), sizeof(double) * f.m_local * f.k, cudaMemcpyDeviceToDevice,
                             c->stream));
    SVT_CUDA(cudaMemcpyAsync(out.V.get(), f.V.get(), sizeof(double) * f.n * f.k, cudaMemcpyDeviceToDevice,
                             c->stream));
}

// row-major device (rows x k) -> column-major host
void to_host_cm(svt_ctx* c, const double* d, i64 rows, i64 k, std::vector<double>& out) {
    out.assign(static_cast<size_t>(rows * k), 0.0);
    if (rows * k == 0) return;
    std::vector<double> tmp(static_cast<size_t>(rows * k));
    SVT_CUDA(cudaMemcpyAsync(tmp.data(), d, sizeof(double) * rows * k, cudaMemcpyDeviceToHost, c->stream));
    sync_stream(c);
    for (i64 i = 0; i < rows; ++i)
        for (i64 j = 0; j < k; ++j) out[static_cast<size_t>(i + j * rows)] = tmp[static_cast<size_t>(i * k + j)];
}

}  // namespace

void kickstart_dev(svt_ctx* c, svt_mat* A, double tau, double delta, u64 seed, double* out_csr, double* out_csc) {
    if (!(tau > 0.0) || !(delta > 0.0)) throw std::invalid_argument("kickstart: tau and delta must be positive");
    Engine E(c, A, Vals{A->val.get(), A->val_csc.get()});
    const double sigma1 = spectral_norm_est(E, 20, seed);  // kSpectralNormIters, solver.hpp:90
    double k0 = 1.0;
    if (sigma1 > 0.0) k0 = std::max(1.0, std::ceil(tau / (delta * sigma1)));
    scale_values(c, A->nnz_local, A->val.get(), k0 * delta, out_csr, A->csr2csc.get(), out_csc);
}

static std::unique_ptr<svt_solver> solver_alloc(svt_mat* A, const svt_config& cfg, svt_stop stop,
                                                svt_backend backend, svt_mat* test) {
    check_config(cfg);
    const i64 min_dim = std::min(A->m, A->n);
    if (backend.kind == SVT_BACKEND_RSVD_FIXED && (backend.fixed_rank < 1 || backend.fixed_rank > min_dim))
        throw std::invalid_argument("svt_run_backend: fixed rank out of range");
    if (cfg.t0 > min_dim) throw std::invalid_argument("SvtConfig: t0 exceeds min(m, n)");
    if (test != nullptr && (test->m != A->m || test->n != A->n || test->row_begin != A->row_begin ||
                            test->row_end != A->row_end))
        throw std::invalid_argument("svt_run: test set must share the frame and row block of A");
    auto S = std::make_unique<svt_solver>();
    svt_ctx* c = A->ctx;
    S->ctx = c;
    S->A = A;
    S->test = test;
    S->cfg = cfg;
    S->stop = stop;
    S->backend = backend;
    const i64 nnz = std::max<i64>(1, A->nnz_local);
    S->Ycsr.alloc(static_cast<size_t>(nnz));
    S->Ycsc.alloc(static_cast<size_t>(nnz));
    S->eps_threshold = cfg.eps_threshold0;
    S->X.m_local = S->best.m_local = A->m_local;
    S->X.n = S->best.n = A->n;
    return S;
}

svt_solver* solver_create(svt_mat* A, const svt_config& cfg, svt_stop stop, svt_backend backend, svt_mat* test) {
    auto S = solver_alloc(A, cfg, stop, backend, test);
    svt_ctx* c = A->ctx;
    kickstart_dev(c, A, cfg.tau, cfg.delta, derive_seed_u(cfg.seed, 0), S->Ycsr.get(), S->Ycsc.get());
    sumsq(c, A->val.get(), 1, A->nnz_local, A->nnz_local, c->d_scalars + S_FA, 0);
    c->comm.allreduce_sum(c->d_scalars + S_FA, 1, c->stream);
    SVT_CUDA(cudaMemcpyAsync(c->h_scalars + S_FA, c->d_scalars + S_FA, sizeof(double), cudaMemcpyDeviceToHost,
                             c->stream));
    sync_stream(c);
    S->frob_a = std::sqrt(c->h_scalars[S_FA]);
    S->t_start_ms = now_ms();
    return S.release();
}

static Engine& engine_of(svt_solver* S) {
    if (!S->engine) {
        S->engine = std::make_unique<Engine>(S->ctx, S->A, Vals{S->Ycsr.get(), S->Ycsc.get()});
        S->engine->last_rounds = S->resume_last_rounds;
    }
    return *S->engine;
}

// ---- checkpoint / resume (svt_b200.h) ---------------------------------------
void solver_checkpoint(svt_solver* S, svt_solver_state* st, double* y_vals, double* u_prev, double* best_U,
                       double* best_sigma, double* best_V) {
    svt_ctx* c = S->ctx;
    svt_mat* A = S->A;
    *st = svt_solver_state{};
    st->iter = S->iter;
    st->done = S->done ? 1 : 0;
    st->converged = S->converged ? 1 : 0;
    st->last_rounds = S->engine ? S->engine->last_rounds : S->resume_last_rounds;
    st->s = S->s;
    st->best_k = S->best.k;
    st->eps_threshold = S->eps_threshold;
    st->eps_min = S->eps_min;
    st->best_metric = S->best_metric;
    st->frob_y_sq = S->frob_y_sq;
    st->frob_a = S->frob_a;
    if (y_vals && A->nnz_local > 0)
        SVT_CUDA(cudaMemcpyAsync(y_vals, S->Ycsr.get(), sizeof(double) * A->nnz_local, cudaMemcpyDeviceToHost,
                                 c->stream));
    std::vector<double> tmp;
    auto cm_out = [&](const double* d, i64 rows, i64 k, double* h) {
        if (h == nullptr || rows * k == 0) return;
        to_host_cm(c, d, rows, k, tmp);
        std::memcpy(h, tmp.data(), sizeof(double) * rows * k);
    };
    cm_out(S->U_prev.get(), A->m_local, S->s, u_prev);
    cm_out(S->best.U.get(), A->m_local, S->best.k, best_U);
    cm_out(S->best.V.get(), A->n, S->best.k, best_V);
    if (best_sigma && S->best.k > 0) std::memcpy(best_sigma, S->best.sigma.data(), sizeof(double) * S->best.k);
    sync_stream(c);
}

// column-major host (rows x k) -> row-major device (rows x k, ld k)
static void upload_cm(svt_ctx* c, const double* h, i64 rows, i64 k, DevBuf<double>& dst, i64 cap_cols) {
    dst.ensure(static_cast<size_t>(std::max<i64>(1, rows) * std::max(k, cap_cols)));
    if (rows * k == 0) return;
    DevBuf<double> stage(static_cast<size_t>(rows * k));
    SVT_CUDA(cudaMemcpyAsync(stage.get(), h, sizeof(double) * rows * k, cudaMemcpyHostToDevice, c->stream));
    transpose(c, stage.get(), k, rows, rows, dst.get());
    sync_stream(c);  // the staging buffer dies with this scope
}

svt_solver* solver_resume(svt_mat* A, const svt_config& cfg, svt_stop stop, svt_backend backend, svt_mat* test,
                          const svt_solver_state& st, const double* y_vals, const double* u_prev,
                          const double* best_U, const double* best_sigma, const double* best_V) {
    if (st.iter < 0 || st.s < 0 || st.best_k < 0 || st.s > std::min(A->m, A->n) || st.best_k > std::min(A->m, A->n))
        throw std::invalid_argument("svt_solver_resume: inconsistent state");
    if ((A->nnz_local > 0 && y_vals == nullptr) || (st.s > 0 && u_prev == nullptr) ||
        (st.best_k > 0 && (best_U == nullptr || best_sigma == nullptr || best_V == nullptr)))
        throw std::invalid_argument("svt_solver_resume: missing state buffer");
    auto S = solver_alloc(A, cfg, stop, backend, test);
    svt_ctx* c = A->ctx;
    if (A->nnz_local > 0) {
        SVT_CUDA(cudaMemcpyAsync(S->Ycsr.get(), y_vals, sizeof(double) * A->nnz_local, cudaMemcpyHostToDevice,
                                 c->stream));
        if (A->csc2csr.n > 0)
            mirror_csc(c, A->nnz_local, A->csc2csr.get(), S->Ycsr.get(), S->Ycsc.get());
        else
            scale_values(c, A->nnz_local, S->Ycsr.get(), 1.0, S->Ycsr.get(), A->csr2csc.get(), S->Ycsc.get());
    }
    const i64 fc = factor_cols(A->m_local + A->n, std::min(A->m, A->n));
    S->s = st.s;
    upload_cm(c, u_prev, A->m_local, st.s, S->U_prev, fc);
    S->best.k = st.best_k;
    S->best.sigma.assign(best_sigma, best_sigma + st.best_k);
    upload_cm(c, best_U, A->m_local, st.best_k, S->best.U, fc);
    upload_cm(c, best_V, A->n, st.best_k, S->best.V, fc);
    S->iter = st.iter;
    S->done = st.done != 0;
    S->converged = st.converged != 0;
    S->resume_last_rounds = st.last_rounds;
    S->eps_threshold = st.eps_threshold;
    S->eps_min = st.eps_min;
    S->best_metric = st.best_metric;
    S->frob_y_sq = st.frob_y_sq;
    S->frob_a = st.frob_a;
    sync_stream(c);  // the caller's host buffers may be released on return
    S->t_start_ms = now_ms();
    return S.release();
}

void solver_step(svt_solver* S, svt_observer_fn obs, void* user, svt_record* rec_out, int* done) {
    if (S->done) {
        if (done) *done = 1;
        return;
    }
    svt_ctx* c = S->ctx;
    svt_mat* A = S->A;
    const svt_config& cfg = S->cfg;
    Engine& E = engine_of(S);
    const int iter = ++S->iter;
    NvtxRange nvtx_iter("svt.iteration");
    const u64 iter_seed = derive_seed_u(cfg.seed, static_cast<u64>(iter));
    svt_sketch_params sp{};
    sp.t = cfg.t0;
    sp.dt = cfg.dt;
    sp.np = cfg.np;
    sp.eps_threshold = S->eps_threshold;
    sp.seed = iter_seed;
    sp.p = 5;
    const i64 min_dim = std::min(A->m, A->n);

    const double t_sketch = now_ms();
    i64 revealed = 0;
    int rounds = 0;
    nvtxRangePushA("svt.partial_svd + shrink");
    try {
    switch (S->backend.kind) {
        case SVT_BACKEND_R4SVD:
        case SVT_BACKEND_R3SVD: {
            SketchOut so = (S->backend.kind == SVT_BACKEND_R4SVD && iter > 1)
                               ? r4svd(E, S->U_prev.get(), S->s, S->s, sp, FinalizeMode::Kept, cfg.tau, S->frob_y_sq)
                               : r3svd(E, sp, FinalizeMode::Kept, cfg.tau, S->frob_y_sq);
            revealed = so.rank;
            rounds = so.rounds;
            shrink_into(c, so.f, cfg.tau, S->X);
            E.fpool = std::move(so.f);  // buffers back to the engine (freed only with it)
            break;
        }
        case SVT_BACKEND_RSVD_FIXED: {
            svt_sketch_params fixed = sp;
            fixed.p = std::min<i64>(sp.p, min_dim - S->backend.fixed_rank);
            DevFactors f = rsvd(E, S->backend.fixed_rank, fixed);
            revealed = S->backend.fixed_rank;
            shrink_into(c, f, cfg.tau, S->X);
            break;
        }
        case SVT_BACKEND_FULL_SVD: {
            DevFactors f = full_svd(E);
            revealed = min_dim;
            shrink_into(c, f, cfg.tau, S->X);
            break;
        }
        default:
            throw std::invalid_argument("svt_run_backend: unknown backend");
    }
    } catch (...) {
        nvtxRangePop();
        throw;
    }
    nvtxRangePop();
    const double sketch_ms = now_ms() - t_sketch;
    NvtxRange nvtx_update("svt.residual + sddmm_update");

    // X = shrink(...): U (m_local x k), sigma - tau, V (n x k); Vs = V diag(sigma - tau)
    DevFactors& X = S->X;
    const i64 k = X.k;
    X.d_sigma.ensure(static_cast<size_t>(std::max<i64>(k, factor_cols(A->m_local + A->n, std::min(A->m, A->n)))));
    if (k > 0) {
        S->Vs.ensure(static_cast<size_t>(A->n * std::max<i64>(k, factor_cols(A->m_local + A->n, std::min(A->m, A->n)))));
        SVT_CUDA(cudaMemcpyAsync(X.d_sigma.get(), X.sigma.data(), sizeof(double) * k, cudaMemcpyHostToDevice,
                                 c->stream));
        copy2d(c, X.V.get(), k, S->Vs.get(), k, A->n, k);
        scale_cols(c, S->Vs.get(), A->n, k, k, X.d_sigma.get());
    }
    // with the inverse permutation the CSC mirror is rebuilt by a coalesced
    // gather pass instead of a scattered write inside the update
    const bool gather = A->csc2csr.n > 0 && A->nnz_local > 0;
    sddmm_update(c, A->plan_csr.v, A->m_local, A->col.get(), A->val.get(), S->Ycsr.get(),
                 gather ? nullptr : S->Ycsc.get(), A->csr2csc.get(), A->nnz_local, A->n, X.U.get(), k, S->Vs.get(),
                 k, k, cfg.delta, 1, c->d_scalars + S_SUMS);
    if (gather) mirror_csc(c, A->nnz_local, A->csc2csr.get(), S->Ycsr.get(), S->Ycsc.get());
    c->comm.allreduce_sum(c->d_scalars + S_SUMS, 4, c->stream);
    if (S->test != nullptr) {
        svt_mat* T = S->test;
        sddmm_update(c, T->plan_csr.v, T->m_local, T->col.get(), T->val.get(), T->val.get(), nullptr, nullptr,
                     T->nnz_local, T->n, X.U.get(), k, S->Vs.get(), k, k, 0.0, 0, c->d_scalars + S_TSUMS);
        c->comm.allreduce_sum(c->d_scalars + S_TSUMS, 4, c->stream);
    }
    SVT_CUDA(cudaMemcpyAsync(c->h_scalars + S_SUMS, c->d_scalars + S_SUMS, sizeof(double) * 8,
                             cudaMemcpyDeviceToHost, c->stream));
    sync_stream(c);
    const double* sums = c->h_scalars + S_SUMS;
    const double* tsums = c->h_scalars + S_TSUMS;

    // solver.hpp:279-284 — dual residual on the pre-update Y, cooling
    const double eps_i = std::sqrt(sums[2]);
    if (eps_i < S->eps_min) {
        S->eps_min = eps_i;
    } else {
        S->eps_threshold = std::max(S->eps_threshold * cfg.beta, cfg.eps_threshold_min);
    }
    const double mae = sums[0] / static_cast<double>(A->nnz_global);

    svt_record rec{};
    rec.iter = iter;
    rec.extension_rounds = rounds;
    rec.rank = revealed;
    rec.residual = eps_i;
    rec.eps_threshold = S->eps_threshold;
    rec.train_mae = mae;
    rec.sketch_ms = sketch_ms;
    rec.total_ms = now_ms() - S->t_start_ms;
    rec.kept = k;
    rec.rel_residual_x = (S->frob_a > 0.0) ? std::sqrt(sums[1]) / S->frob_a : 0.0;
    if (S->test != nullptr && S->test->nnz_global > 0) {
        rec.test_mae = tsums[0] / static_cast<double>(S->test->nnz_global);
        rec.test_rmse = std::sqrt(tsums[1] / static_cast<double>(S->test->nnz_global));
    }
    S->trace.push_back(rec);
    if (rec_out) *rec_out = rec;

    // best-so-far (solver.hpp:299-303)
    const double metric = (S->stop.kind == SVT_STOP_RESIDUAL) ? eps_i : mae;
    if (metric < S->best_metric) {
        S->best_metric = metric;
        copy_factors(c, X, S->best);
    }
    // stop rule, then observer (solver.hpp:305-319)
    bool stop_hit = false;
    if (S->stop.kind == SVT_STOP_TRAIN_MAE && mae < S->stop.threshold) stop_hit = true;
    else if (S->stop.kind == SVT_STOP_RESIDUAL && eps_i < S->stop.threshold) stop_hit = true;
    bool keep_going = true;
    if (cfg.rel_residual_stop > 0.0 && rec.rel_residual_x < cfg.rel_residual_stop) keep_going = false;
    if (keep_going && obs != nullptr) {
        std::vector<double> Uh, Vh;
        to_host_cm(c, X.U.get(), X.m_local, k, Uh);
        to_host_cm(c, X.V.get(), X.n, k, Vh);
        keep_going = obs(&rec, X.m_local, X.n, k, Uh.data(), X.sigma.data(), Vh.data(), user) != 0;
    }
    if (stop_hit || !keep_going) {
        copy_factors(c, X, S->best);
        S->converged = true;
        S->done = true;
        if (done) *done = 1;
        return;
    }
    // the fused kernel already applied Y <- Y + delta (A - P(X)); U_prev = X.U
    S->frob_y_sq = sums[3];
    S->s = k;
    if (k > 0) {
        S->U_prev.ensure(static_cast<size_t>(std::max<i64>(1, A->m_local) * std::max<i64>(k, factor_cols(A->m_local + A->n, std::min(A->m, A->n)))));
        SVT_CUDA(cudaMemcpyAsync(S->U_prev.get(), X.U.get(), sizeof(double) * A->m_local * k,
                                 cudaMemcpyDeviceToDevice, c->stream));
    }
    if (iter >= cfg.maxit) {
        S->converged = false;
        S->done = true;
    }
    if (done) *done = S->done ? 1 : 0;
}

svt_result* solver_result(svt_solver* S) {
    auto R = std::make_unique<svt_result>();
    svt_ctx* c = S->ctx;
    R->trace = S->trace;
    R->converged = S->converged ? 1 : 0;
    const DevFactors& f = S->best;
    R->m_local = S->A->m_local;
    R->n = S->A->n;
    R->k = f.k;
    R->sigma = f.sigma;
    to_host_cm(c, f.U.get(), R->m_local, f.k, R->U);
    to_host_cm(c, f.V.get(), R->n, f.k, R->V);
    return R.release();
}

}  // namespace svtb
