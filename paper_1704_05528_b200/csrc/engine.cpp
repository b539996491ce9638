// R3SVD / R4SVD on the device (sketch.hpp) and the primitives they compose.
//
// Control flow follows the reference line by line: the rank-revealing
// `while error_percentage > eps` loop stays on the host (one 8-byte read per
// round), every data-dependent branch INSIDE a round (the conditional second
// Gram-Schmidt pass, sketch.hpp:134; the re-projection, :138; the recycled
// basis drift test, :231; the rank-deficient QR fallback) is evaluated on
// the device and predicates the dependent kernels, so a round issues no host
// synchronisation.  Multi-GPU: Q / X / U rows are the rank's row block;
// Y^T-products, Gram blocks and norms are NCCL all-reduced.
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "kernels.hpp"

namespace svtb {

namespace {

// scalar / flag slots in ctx->d_scalars / ctx->d_flags
enum : int { S_FROB = 0, S_NX = 1, S_NC = 2, S_MAXD = 3, S_NB = 4, S_TMP = 5, S_SPEC = 6 };
enum : int { F_CGS2 = 0, F_REORTH = 1, F_QRSTAT = 2, F_DRIFT = 3, F_BLK = 4, F_CHECK = 5, F_SECOND = 6 };

double* dsc(svt_ctx* c, int i) { return c->d_scalars + i; }
int* dfl(svt_ctx* c, int i) { return c->d_flags + i; }

double read_scalar(svt_ctx* c, int i) {
    SVT_CUDA(cudaMemcpyAsync(c->h_scalars + i, c->d_scalars + i, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync_stream(c);
    return c->h_scalars[i];
}

int read_flag(svt_ctx* c, int i) {
    SVT_CUDA(cudaMemcpyAsync(c->h_flags + i, c->d_flags + i, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    sync_stream(c);
    return c->h_flags[i];
}

// small device -> host read through the pinned staging buffer (a pageable
// destination makes the copy a staged, host-synchronous transfer), then one
// stream synchronization
void read_doubles(svt_ctx* c, const double* d, size_t count, double* out) {
    if (count == 0) return;
    if (count > c->h_stage_n) {
        SVT_CUDA(cudaMemcpyAsync(out, d, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
        sync_stream(c);
        return;
    }
    SVT_CUDA(cudaMemcpyAsync(c->h_stage, d, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
    sync_stream(c);
    std::memcpy(out, c->h_stage, sizeof(double) * count);
}
void read_doubles2(svt_ctx* c, const double* d1, const double* d2, size_t count, double* o1, double* o2) {
    if (2 * count > c->h_stage_n) {
        SVT_CUDA(cudaMemcpyAsync(o1, d1, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
        SVT_CUDA(cudaMemcpyAsync(o2, d2, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
        sync_stream(c);
        return;
    }
    SVT_CUDA(cudaMemcpyAsync(c->h_stage, d1, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
    SVT_CUDA(cudaMemcpyAsync(c->h_stage + count, d2, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
    sync_stream(c);
    std::memcpy(o1, c->h_stage, sizeof(double) * count);
    std::memcpy(o2, c->h_stage + count, sizeof(double) * count);
}

// flag i and `count` doubles with ONE stream synchronization (the batch path
// reads its QR status together with the block energies)
int read_flag_and_doubles(svt_ctx* c, int i, const double* d, size_t count, double* out) {
    SVT_CUDA(cudaMemcpyAsync(c->h_flags + i, c->d_flags + i, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    if (count > c->h_stage_n) {
        SVT_CUDA(cudaMemcpyAsync(out, d, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
        sync_stream(c);
        return c->h_flags[i];
    }
    SVT_CUDA(cudaMemcpyAsync(c->h_stage, d, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
    sync_stream(c);
    std::memcpy(out, c->h_stage, sizeof(double) * count);
    return c->h_flags[i];
}

bool debug_batch() {
    static const bool on = std::getenv("SVTB_DEBUG_BATCH") != nullptr;
    return on;
}

void zero_flag(svt_ctx* c, int i) { SVT_CUDA(cudaMemsetAsync(c->d_flags + i, 0, sizeof(int), c->stream)); }

void allreduce(svt_ctx* c, double* p, size_t n) { c->comm.allreduce_sum(p, n, c->stream); }

inline u64 splitmix64(u64 x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

// grow Q / B^T capacity geometrically, preserving the first `rank` columns
void ensure_cap(Engine& E, QBDev& st, i64 need) {
    if (need <= st.cap) return;
    // double while the two panels fit comfortably in free HBM, else grow by
    // 1.25x: every regrow is a cudaMalloc + copy + cudaFree on the critical
    // path, so fewer growth steps matter more than a tight fit
    size_t free_b = 0, total_b = 0;
    SVT_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const double per_col = 8.0 * static_cast<double>(std::max<i64>(1, st.m_local) + st.n);
    const bool roomy = per_col * static_cast<double>(2 * st.cap) < 0.45 * static_cast<double>(free_b);
    i64 grown = roomy ? st.cap * 2 : st.cap + st.cap / 4;
    if (st.cap == 0 && per_col * static_cast<double>(st.min_dim) <= 0.4 * static_cast<double>(free_b)) {
        // the whole basis range is affordable (small and mid-size problems):
        // reserve it once, so the basis never regrows inside an SVT iteration
        grown = st.min_dim;
    } else if (st.cap == 0 && E.mat != nullptr && E.mat->nnz_global >= (1LL << 20)) {
        // first sketch of a large problem: reserve the basis range the panels
        // can take in ~62 % of free HBM, so no multi-GB regrow lands inside an
        // SVT iteration (a regrow holds old + new panel: ~3.25x one panel, and
        // a fresh device maps new pages slowly).  Config 5 (100k x 100k):
        // ~70k columns, enough for its 33 iterations (r ~ 20.5k at iteration
        // 1, +~1,300 per iteration).
        grown = static_cast<i64>(0.62 * static_cast<double>(free_b) / per_col);
    }
    i64 cap = std::max<i64>(need + 128, std::max<i64>(64, grown));
    cap = std::min<i64>(cap, std::max(st.min_dim, need));
    cap = (cap + 7) & ~7LL;
    // one buffer at a time, so the transient peak is old Q + new Q + old B^T
    auto regrow = [&](DevBuf<double>& buf, i64 rows) {
        DevBuf<double> nb(static_cast<size_t>(std::max<i64>(1, rows) * cap));
        if (st.rank > 0 && rows > 0)
            SVT_CUDA(cudaMemcpy2DAsync(nb.get(), cap * sizeof(double), buf.get(), st.cap * sizeof(double),
                                       st.rank * sizeof(double), rows, cudaMemcpyDeviceToDevice, E.ctx->stream));
        buf = std::move(nb);  // frees the old buffer (cudaFree orders after the copy)
    };
    const bool dbg = std::getenv("SVTB_DEBUG_CAP") != nullptr;
    std::chrono::steady_clock::time_point t0;
    if (dbg) {
        sync_stream(E.ctx);
        t0 = std::chrono::steady_clock::now();
    }
    regrow(st.Q, st.m_local);
    regrow(st.Bt, st.n);
    if (dbg) {
        sync_stream(E.ctx);
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        std::fprintf(stderr, "[ensure_cap] %lld -> %lld cols (rank %lld): %.1f ms\n", static_cast<long long>(st.cap),
                     static_cast<long long>(cap), static_cast<long long>(st.rank), ms);
    }
    st.cap = cap;
}

// Empty the QB state for a new sketch of A, keeping its buffers (capacity)
// when the frame matches.
void reset_qb(QBDev& st, const svt_mat* A) {
    if (st.m_local != A->m_local || st.n != A->n) {
        st.Q.release();
        st.Bt.release();
        st.cap = 0;
    }
    st.m_local = A->m_local;
    st.n = A->n;
    st.min_dim = std::min(A->m, A->n);
    st.rank = 0;
    st.qs_valid = 0;
    st.norm_b_sq = 0.0;
    st.frob_y_sq = 0.0;
    st.saturated = false;
}

// One CholQR2 panel (w <= 64) with the Householder fallback.  X is preserved.
// m rows; dist: the rows are this rank's block of a row-sharded panel (Gram
// blocks are all-reduced) — false for replicated panels (finalize space).
void qr_panel(Engine& E, i64 m, bool dist, const double* X, i64 ldx, i64 w, double* Qout, i64 ldq,
              const int* pred) {
    svt_ctx* c = E.ctx;
    dist = dist && c->comm.dist();
    const i64 wc = std::max<i64>(w, 64);  // panels are <= 64 wide: size once
    E.G.ensure(static_cast<size_t>(wc * wc));
    E.Rinv.ensure(static_cast<size_t>(wc * wc));
    E.tmp.ensure(static_cast<size_t>(std::max<i64>(1, m) * wc));
    int* status = dfl(c, F_QRSTAT);
    zero_flag(c, F_QRSTAT);
    if (!dist && w <= 16) {
        // fused: Gram + Cholesky + Rinv in one launch, then the triangular
        // apply; twice (CholQR2), then the predicated Householder fallback
        gram_chol(c, X, ldx, m, w, E.G.get(), E.Rinv.get(), status, pred);
        gemm(c, K_QR, false, m, w, w, 1.0, X, ldx, E.Rinv.get(), w, 0.0, E.tmp.get(), w, pred);
        gram_chol(c, E.tmp.get(), w, m, w, E.G.get(), E.Rinv.get(), status, pred);
        gemm(c, K_QR, false, m, w, w, 1.0, E.tmp.get(), w, E.Rinv.get(), w, 0.0, Qout, ldq, pred);
        E.hh.ensure(static_cast<size_t>(std::max<i64>(1, m) * std::max<i64>(w, 64)));
        householder_qr(c, X, m, w, ldx, Qout, ldq, E.hh.get(), pred, status);
        return;
    }
    // pass 1: R1 = chol(X^T X), Q1 = X R1^{-1}
    gemm(c, K_QR, true, w, w, m, 1.0, X, ldx, X, ldx, 0.0, E.G.get(), w, pred);
    if (dist) allreduce(c, E.G.get(), static_cast<size_t>(w * w));
    chol_rinv(c, E.G.get(), w, E.Rinv.get(), status, pred);
    gemm(c, K_QR, false, m, w, w, 1.0, X, ldx, E.Rinv.get(), w, 0.0, E.tmp.get(), w, pred);
    // pass 2
    gemm(c, K_QR, true, w, w, m, 1.0, E.tmp.get(), w, E.tmp.get(), w, 0.0, E.G.get(), w, pred);
    if (dist) allreduce(c, E.G.get(), static_cast<size_t>(w * w));
    chol_rinv(c, E.G.get(), w, E.Rinv.get(), status, pred);
    gemm(c, K_QR, false, m, w, w, 1.0, E.tmp.get(), w, E.Rinv.get(), w, 0.0, Qout, ldq, pred);
    if (!dist) {
        E.hh.ensure(static_cast<size_t>(std::max<i64>(1, m) * std::max<i64>(w, 64)));
        householder_qr(c, X, m, w, ldx, Qout, ldq, E.hh.get(), pred, status);
        return;
    }
    // multi-GPU: the (rare) fallback gathers the panel and factors it redundantly
    if (pred != nullptr && read_flag(c, static_cast<int>(pred - c->d_flags)) == 0) return;
    if (read_flag(c, F_QRSTAT) == 0) return;
    const i64 M = E.mat->m;
    DevBuf<double> full(static_cast<size_t>(M * w)), qfull(static_cast<size_t>(M * w)), work(static_cast<size_t>(M * w));
    SVT_CUDA(cudaMemsetAsync(full.get(), 0, sizeof(double) * M * w, c->stream));
    copy2d(c, X, ldx, full.get() + E.mat->row_begin * w, w, m, w);
    allreduce(c, full.get(), static_cast<size_t>(M * w));
    householder_qr(c, full.get(), M, w, w, qfull.get(), w, work.get(), nullptr, nullptr);
    copy2d(c, qfull.get() + E.mat->row_begin * w, w, Qout, ldq, m, w);
}

// Project Q[:, 0:r0] out of the panel P (m x w, ld) and re-orthonormalize
// it, predicated on flag `f` computed from max|Q^T P| > 1e-8 (sketch.hpp:138).
void reorth_if_needed(Engine& E, i64 m, bool dist, const double* Q, i64 ldq, i64 r0, double* P, i64 ldp, i64 w) {
    svt_ctx* c = E.ctx;
    E.D.ensure(static_cast<size_t>(std::max(r0, ldq) * w));  // ldq = basis capacity: no regrow as r0 grows
    gemm(c, K_GEMM, true, r0, w, m, 1.0, Q, ldq, P, ldp, 0.0, E.D.get(), w);
    if (dist) allreduce(c, E.D.get(), static_cast<size_t>(r0 * w));
    maxabs(c, E.D.get(), r0, w, w, 0.0, dsc(c, S_MAXD));
    set_flag(c, dsc(c, S_MAXD), nullptr, 1e-8, 1, dfl(c, F_REORTH));
    const int* f = dfl(c, F_REORTH);
    E.X2.ensure(static_cast<size_t>(std::max<i64>(1, m) * w));
    copy2d(c, P, ldp, E.X2.get(), w, m, w, f);
    gemm(c, K_GEMM, false, m, w, r0, -1.0, Q, ldq, E.D.get(), w, 1.0, E.X2.get(), w, f);
    qr_panel(E, m, dist, E.X2.get(), w, w, P, ldp, f);
}

}  // namespace

u64 derive_seed_u(u64 seed, u64 stream) { return splitmix64(seed ^ splitmix64(stream)); }

double frob_sq(Engine& E) {
    svt_ctx* c = E.ctx;
    sumsq(c, E.Y.csr, 1, E.mat->nnz_local, E.mat->nnz_local, dsc(c, S_FROB), 0);
    allreduce(c, dsc(c, S_FROB), 1);
    return read_scalar(c, S_FROB);
}

// The tiled views (wide panels) mirror Y: built on first use, their entry
// values re-gathered from Y.csr once per sketch.  Only ever called on the
// main stream (side-stream products follow main-stream work through events).
static bool tiles_ready(Engine& E, i64 w, cudaStream_t stream) {
    svt_mat* A = E.mat;
    if (!E.tiled || w <= 16 || A->nnz_local <= 0 || E.Y.csr == nullptr) return false;
    if (!E.tiles_fresh || A->tile_csr.src != E.Y.csr || A->tile_csc.src != E.Y.csr) {
        if (stream && stream != E.ctx->stream) return false;
        ensure_tile_plans(E.ctx, A);
        tile_values(E.ctx, A->tile_csr.v, E.Y.csr);
        tile_values(E.ctx, A->tile_csc.v, E.Y.csr);
        A->tile_csr.src = E.Y.csr;
        A->tile_csc.src = E.Y.csr;
        E.tiles_fresh = true;
    }
    return true;
}

void prepare_tiles(Engine& E) {
    E.tiles_fresh = false;
    E.hyb_fresh = false;
    E.tiled = tile_spmm_enabled();
    tiles_ready(E, 32, nullptr);
}

// The dense-corner split of Y (HybridPlan) for wide panels: built on the
// first wide product (main stream), its values mirrored from Y.csr once per
// sketch; side-stream products use it only once it is fresh (they follow the
// main stream's refresh through the batch events).
constexpr i64 kHybMinW = 24;
static bool hybrid_ready(Engine& E, i64 w, const double* X, i64 ldx, cudaStream_t stream) {
    svt_mat* A = E.mat;
    if (w < kHybMinW || A->nnz_local <= 0 || E.Y.csr == nullptr) return false;
    const bool main = stream == nullptr || stream == E.ctx->stream;
    if (!A->hyb.tried) {
        if (!main) return false;
        ensure_hybrid(E.ctx, A);
    }
    HybridPlan& H = A->hyb;
    if (!H.on) return false;
    // fresh: mirrored during this sketch, or the engine works on the
    // matrix's own values and they have not been rewritten since
    const bool own = E.Y.csr == A->val.get();
    const bool fresh = (E.hyb_fresh && H.src == E.Y.csr) ||
                       (own && H.src == E.Y.csr && H.src_version == A->val_version);
    if (!fresh) {
        if (!main) return false;
        hybrid_refresh(E.ctx, A, E.Y.csr);
        H.src_version = own ? A->val_version : -1;
        E.hyb_fresh = true;
    }
    return reinterpret_cast<uintptr_t>(X) % 8 == 0;  // 16-byte rows or not: both operand paths exist
}


// Y X (tr = false) or Y^T X (tr = true) through the split: the dense block's
// split-K product on the helper stream of `stream` (forked after everything
// already queued there), the cold entries' gather kernel on `stream`
// meanwhile, then the block rows added into the output after the join.
template <typename Cold>
static void split_product(Engine& E, int cls, bool tr, i64 w, const double* X, i64 ldx, double* out, i64 ldo,
                          cudaStream_t stream, Cold&& cold) {
    svt_ctx* c = E.ctx;
    svt_mat* Am = E.mat;
    HybridPlan& H = Am->hyb;
    cudaStream_t s = stream ? stream : c->stream;
    const int k = (s == c->side) ? 1 : 0;
    // the whole split product is ONE timed operation of class cls (its
    // kernels run on two streams and overlap); algorithmic bytes of the full
    // product, the inner launches are K_SUB
    const i64 rows = tr ? Am->n : Am->m_local, x_rows = tr ? Am->m_local : Am->n;
    LaunchScope op(c, cls, 12.0 * Am->nnz_local + 8.0 * (rows + 1) + 8.0 * w * (x_rows + rows),
                   2.0 * Am->nnz_local * w, s);
    if (c->aux[k] == nullptr) {
        int prio = 0;
        SVT_CUDA(cudaStreamGetPriority(s, &prio));
        SVT_CUDA(cudaStreamCreateWithPriority(&c->aux[k], cudaStreamNonBlocking, prio));
        SVT_CUDA(cudaEventCreateWithFlags(&c->aux_fork[k], cudaEventDisableTiming));
        SVT_CUDA(cudaEventCreateWithFlags(&c->aux_join[k], cudaEventDisableTiming));
    }
    SVT_CUDA(cudaEventRecord(c->aux_fork[k], s));
    SVT_CUDA(cudaStreamWaitEvent(c->aux[k], c->aux_fork[k], 0));
    const i64 M = tr ? H.C : H.R, K = tr ? H.R : H.C;
    const int S = dense_block_mm(c, c->aux[k], K_SUB, tr, M, w, K, H.D.get(), H.C, X, ldx,
                                 tr ? H.hot_rows.get() : H.hot_cols.get(), H.ws[k], 0.0, 0.0);
    SVT_CUDA(cudaEventRecord(c->aux_join[k], c->aux[k]));
    if (S == 0) throw std::logic_error("split SpMM: dense block operands not aligned");
    cold();
    SVT_CUDA(cudaStreamWaitEvent(s, c->aux_join[k], 0));
    dense_block_add(c, s, K_SUB, M, w, S, H.ws[k], tr ? H.hot_cols.get() : H.hot_rows.get(), out, ldo);
}

void sp_mult(Engine& E, i64 w, const double* X, i64 ldx, double* out, i64 ldo, cudaStream_t stream,
             DevBuf<double>* scratch) {
    svt_mat* A = E.mat;
    if (hybrid_ready(E, w, X, ldx, stream)) {
        HybridPlan& H = A->hyb;
        split_product(E, K_SPMM, false, w, X, ldx, out, ldo, stream, [&] {
            spmm(E.ctx, K_SUB, H.plan_c.v, A->m_local, H.col_c.get(), H.val_c.get(), H.nnz_cold, A->n, w, X, ldx,
                 out, ldo, stream, scratch);
        });
        return;
    }
    if (tiles_ready(E, w, stream) &&
        spmm_tiled(E.ctx, K_SPMM, A->tile_csr.v, A->n, w, X, ldx, out, ldo, stream, scratch))
        return;
    spmm(E.ctx, K_SPMM, A->plan_csr.v, A->m_local, A->col.get(), E.Y.csr, A->nnz_local, A->n, w, X, ldx, out, ldo,
         stream, scratch);
}

void sp_mult_t(Engine& E, i64 w, const double* X, i64 ldx, double* out, cudaStream_t stream,
               DevBuf<double>* scratch, i64 ldo) {
    svt_mat* A = E.mat;
    if (ldo < 0) ldo = w;
    if (ldo != w && E.ctx->comm.dist()) throw std::logic_error("sp_mult_t: strided output needs one rank");
    if (hybrid_ready(E, w, X, ldx, stream)) {
        HybridPlan& H = A->hyb;
        split_product(E, K_SPMMT, true, w, X, ldx, out, ldo, stream, [&] {
            spmm(E.ctx, K_SUB, H.plant_c.v, A->n, H.row_c.get(), H.valt_c.get(), H.nnz_cold, A->m_local, w, X,
                 ldx, out, ldo, stream, scratch);
        });
    } else if (!(tiles_ready(E, w, stream) &&
                 spmm_tiled(E.ctx, K_SPMMT, A->tile_csc.v, A->m_local, w, X, ldx, out, ldo, stream, scratch))) {
        spmm(E.ctx, K_SPMMT, A->plan_csc.v, A->n, A->cscrow.get(), E.Y.csc, A->nnz_local, A->m_local, w, X, ldx, out,
             ldo, stream, scratch);
    }
    E.ctx->comm.allreduce_sum(out, static_cast<size_t>(A->n * w), stream ? stream : E.ctx->stream,
                              stream != nullptr && stream == E.ctx->side);
}

// basis capacity of the engine's QB state (workspace sizing hint)
static i64 st_cap_hint(const Engine& E) { return std::max<i64>(E.qb.cap, 64); }

// dense.hpp:103-110 on a panel of any width: CholQR2 (w <= 64) or block
// CGS2 + CholQR2 over 64-column blocks (the column-ordered QR, same nested
// spans).  X is clobbered.
void qr_orthonormal(Engine& E, double* X, i64 ldx, i64 w, double* Qout, i64 ldq) {
    qr_orthonormal(E, E.mat->m_local, true, X, ldx, w, Qout, ldq);
}

void qr_orthonormal(Engine& E, i64 m, bool dist, double* X, i64 ldx, i64 w, double* Qout, i64 ldq) {
    svt_ctx* c = E.ctx;
    dist = dist && c->comm.dist();
    constexpr i64 B = 64;
    for (i64 b0 = 0; b0 < w; b0 += B) {
        const i64 wb = std::min(B, w - b0);
        double* Xb = X + b0;
        if (b0 > 0) {
            E.C.ensure(static_cast<size_t>(std::max(b0, st_cap_hint(E)) * 64));
            for (int pass = 0; pass < 2; ++pass) {
                gemm(c, K_QR, true, b0, wb, m, 1.0, Qout, ldq, Xb, ldx, 0.0, E.C.get(), wb);
                if (dist) allreduce(c, E.C.get(), static_cast<size_t>(b0 * wb));
                gemm(c, K_QR, false, m, wb, b0, -1.0, Qout, ldq, E.C.get(), wb, 1.0, Xb, ldx);
            }
        }
        qr_panel(E, m, dist, Xb, ldx, wb, Qout + b0, ldq, nullptr);
        if (b0 > 0) reorth_if_needed(E, m, dist, Qout, ldq, b0, Qout + b0, ldq, wb);
    }
}

// sampled.hpp:188-213
double spectral_norm_est(Engine& E, int iters, u64 seed) {
    if (iters < 1) throw std::invalid_argument("spectral_norm_est: iters must be >= 1");
    svt_ctx* c = E.ctx;
    svt_mat* A = E.mat;
    const i64 n = A->n, m = A->m_local;
    DevBuf<double> x(static_cast<size_t>(n)), y(static_cast<size_t>(std::max<i64>(1, m)));
    gaussian_block_dev(c, n, 1, seed, x.get(), 1);
    sumsq(c, x.get(), 1, n, n, dsc(c, S_SPEC), 0);
    double xn = std::sqrt(read_scalar(c, S_SPEC));
    if (xn == 0.0) return 0.0;
    scale_values(c, n, x.get(), 1.0 / xn, x.get(), nullptr, nullptr);
    double estimate = 0.0;
    for (int it = 0; it < iters; ++it) {
        sp_mult(E, 1, x.get(), 1, y.get(), 1);
        sumsq(c, y.get(), 1, m, m, dsc(c, S_SPEC), 0);
        allreduce(c, dsc(c, S_SPEC), 1);
        estimate = std::sqrt(read_scalar(c, S_SPEC));
        if (estimate == 0.0) return 0.0;
        sp_mult_t(E, 1, y.get(), 1, x.get());
        sumsq(c, x.get(), 1, n, n, dsc(c, S_SPEC), 0);
        xn = std::sqrt(read_scalar(c, S_SPEC));
        if (xn == 0.0) return estimate;
        scale_values(c, n, x.get(), 1.0 / xn, x.get(), nullptr, nullptr);
    }
    return estimate;
}

// sketch.hpp:71-79 — X <- Y (Y^T X), np passes, QR between passes
static void power_iterate(Engine& E, i64 w, int np) {
    svt_ctx* c = E.ctx;
    const i64 m = E.mat->m_local, n = E.mat->n;
    for (int j = 0; j < np; ++j) {
        if (j > 0) {
            E.P.ensure(static_cast<size_t>(std::max<i64>(1, m) * w));
            qr_orthonormal(E, E.X.get(), w, w, E.P.get(), w);
            std::swap(E.X, E.P);
        }
        E.T.ensure(static_cast<size_t>(n * w));
        sp_mult_t(E, w, E.X.get(), w, E.T.get());
        sp_mult(E, w, E.T.get(), w, E.X.get(), w);
    }
    (void)c;
}

// B[r0:r0+w, :] = (Y^T Q[:, r0:r0+w])^T stored as B^T columns; norm_b_sq +=
static void append_coefficients(Engine& E, QBDev& st, i64 r0, i64 w, int nb_op) {
    svt_ctx* c = E.ctx;
    if (!c->comm.dist()) {  // straight into the coefficient rows (no staging copy)
        sp_mult_t(E, w, st.Q.get() + r0, st.cap, st.Bt.get() + r0, nullptr, nullptr, st.cap);
        sumsq(c, st.Bt.get() + r0, st.n, w, st.cap, dsc(c, S_NB), nb_op);
        return;
    }
    E.T.ensure(static_cast<size_t>(st.n * w));
    sp_mult_t(E, w, st.Q.get() + r0, st.cap, E.T.get());
    copy2d(c, E.T.get(), w, st.Bt.get() + r0, st.cap, st.n, w);
    sumsq(c, E.T.get(), st.n, w, w, dsc(c, S_NB), nb_op);
}

// sketch.hpp:89-108
void qb_init(Engine& E, QBDev& st, i64 t, int np, u64 seed, double frob_y_sq) {
    svt_ctx* c = E.ctx;
    svt_mat* A = E.mat;
    const i64 min_dim = std::min(A->m, A->n);
    if (t < 1 || t > min_dim) throw std::invalid_argument("qb_init: t must satisfy 1 <= t <= min(m, n)");
    if (frob_y_sq < 0.0) frob_y_sq = frob_sq(E);
    if (!(frob_y_sq > 0.0)) throw std::domain_error("qb_init: target matrix is all zero");
    reset_qb(st, A);
    ensure_cap(E, st, t);
    const i64 m = A->m_local;
    E.Om.ensure(static_cast<size_t>(A->n * t));
    E.X.ensure(static_cast<size_t>(std::max<i64>(1, m) * t));
    gaussian_block_dev(c, A->n, t, seed, E.Om.get(), t);
    sp_mult(E, t, E.Om.get(), t, E.X.get(), t);
    power_iterate(E, t, np);
    qr_orthonormal(E, E.X.get(), t, t, st.Q.get(), st.cap);
    append_coefficients(E, st, 0, t, 0);
    st.norm_b_sq = read_scalar(c, S_NB);
    st.frob_y_sq = frob_y_sq;
    st.rank = t;
    st.saturated = (t == min_dim);
}

// sketch.hpp:114-154
void qb_extend(Engine& E, QBDev& st, i64 dt, int np, u64 seed, const double* omega) {
    svt_ctx* c = E.ctx;
    svt_mat* A = E.mat;
    if (dt < 1) throw std::invalid_argument("qb_extend: dt must be >= 1");
    const i64 width = std::min(dt, st.min_dim - st.rank);
    if (width < 1) {
        st.saturated = true;
        return;
    }
    const i64 m = A->m_local, n = A->n, r0 = st.rank;
    ensure_cap(E, st, r0 + width);
    E.X.ensure(static_cast<size_t>(std::max<i64>(1, m) * width));
    if (omega == nullptr || width != dt) {
        E.Om.ensure(static_cast<size_t>(n * width));
        gaussian_block_dev(c, n, width, seed, E.Om.get(), width);
        omega = E.Om.get();
    }
    sp_mult(E, width, omega, width, E.X.get(), width);
    power_iterate(E, width, np);
    double* Q = st.Q.get();
    const i64 ldq = st.cap;
    if (r0 > 0) {
        // classical Gram-Schmidt, conditional second pass (sketch.hpp:133-136)
        E.C.ensure(static_cast<size_t>(std::max(r0, st.cap) * width));
        gemm(c, K_GEMM, true, r0, width, m, 1.0, Q, ldq, E.X.get(), width, 0.0, E.C.get(), width);
        allreduce(c, E.C.get(), static_cast<size_t>(r0 * width));
        gemm(c, K_GEMM, false, m, width, r0, -1.0, Q, ldq, E.C.get(), width, 1.0, E.X.get(), width);
        gemm(c, K_GEMM, true, r0, width, m, 1.0, Q, ldq, E.X.get(), width, 0.0, E.C.get(), width);
        allreduce(c, E.C.get(), static_cast<size_t>(r0 * width));
        sumsq(c, E.X.get(), m, width, width, dsc(c, S_NX), 0);
        allreduce(c, dsc(c, S_NX), 1);
        sumsq(c, E.C.get(), r0, width, width, dsc(c, S_NC), 0);
        set_flag(c, dsc(c, S_NC), dsc(c, S_NX), 1e-8, 0, dfl(c, F_CGS2));
        gemm(c, K_GEMM, false, m, width, r0, -1.0, Q, ldq, E.C.get(), width, 1.0, E.X.get(), width,
             dfl(c, F_CGS2));
    }
    // QR, then conditional re-projection + QR (sketch.hpp:137-141)
    qr_panel(E, m, true, E.X.get(), width, width, Q + r0, ldq, nullptr);
    if (r0 > 0) reorth_if_needed(E, m, true, Q, ldq, r0, Q + r0, ldq, width);
    // coefficient block + energy (sketch.hpp:143-150)
    // norm_b_sq += ||B'||_F^2 (sketch.hpp:150), accumulated on the host so
    // batched and single rounds share one running sum
    append_coefficients(E, st, r0, width, 0);
    st.norm_b_sq += read_scalar(c, S_NB);
    st.rank = r0 + width;
    st.saturated = (st.rank == st.min_dim);
}

// sketch.hpp:158-162 — SVD of B through its Gram: G = B B^T = W L W^T,
// sigma_j = ||B^T w_j|| (column norms: accurate to ~eps*sigma_1 even for the
// small values), V = B^T W / sigma, U = Q W.  Kept mode computes only the
// triplets with sigma > tau (the ones shrink keeps, solver.hpp:110-120).
void finalize(Engine& E, const QBDev& st, FinalizeMode mode, double tau, DevFactors& out) {
    NvtxRange nvtx("sketch.finalize");
    svt_ctx* c = E.ctx;
    const i64 r = st.rank, n = st.n, m = st.m_local;
    out.m_local = m;
    out.n = n;
    out.k = 0;
    out.sigma.clear();
    if (r == 0) return;
    // the dense Gram path runs for bases up to ~1024 wide (finalize_kept):
    // size for that at once, so the basis growing over SVT iterations does
    // not regrow these (a cudaFree is a device-wide sync)
    const i64 rfloor = std::min<i64>(st.min_dim, 1024);
    E.G.ensure(static_cast<size_t>(std::max(r * r, rfloor * rfloor)));
    E.W.ensure(static_cast<size_t>(std::max(r * r, rfloor * rfloor)));
    E.lam.ensure(static_cast<size_t>(std::max(r, rfloor)));
    gemm(c, K_FINAL, true, r, r, n, 1.0, st.Bt.get(), st.cap, st.Bt.get(), st.cap, 0.0, E.G.get(), r);
    sym_eig(c, E.G.get(), r, E.W.get(), E.lam.get());
    std::vector<double> lam(static_cast<size_t>(r));
    read_doubles(c, E.lam.get(), static_cast<size_t>(r), lam.data());
    i64 kc = r;
    if (mode == FinalizeMode::Kept) {
        i64 cnt = 0;
        const double lim = tau * (1.0 - 1e-7);
        while (cnt < r && std::sqrt(std::max(lam[static_cast<size_t>(cnt)], 0.0)) > lim) ++cnt;
        kc = std::min(r, cnt + 1);
    }
    E.Vraw.ensure(static_cast<size_t>(n * std::max<i64>(kc, factor_cols(m + n, st.min_dim))));
    gemm(c, K_FINAL, false, n, kc, r, 1.0, st.Bt.get(), st.cap, E.W.get(), r, 0.0, E.Vraw.get(), kc);
    E.lam.ensure(static_cast<size_t>(std::max(r, kc)));
    col_sumsq(c, E.Vraw.get(), n, kc, kc, E.lam.get());
    std::vector<double> s2(static_cast<size_t>(kc));
    read_doubles(c, E.lam.get(), static_cast<size_t>(kc), s2.data());
    std::vector<double> sig(static_cast<size_t>(kc));
    for (i64 j = 0; j < kc; ++j) sig[static_cast<size_t>(j)] = std::sqrt(s2[static_cast<size_t>(j)]);
    std::vector<int> perm(static_cast<size_t>(kc));
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(),
                     [&](int a, int b) { return sig[static_cast<size_t>(a)] > sig[static_cast<size_t>(b)]; });
    i64 k = kc;
    if (mode == FinalizeMode::Kept) {
        k = 0;
        while (k < kc && sig[static_cast<size_t>(perm[static_cast<size_t>(k)])] > tau) ++k;
    }
    out.k = k;
    if (k == 0) return;
    out.sigma.resize(static_cast<size_t>(k));
    std::vector<double> inv(static_cast<size_t>(k));
    for (i64 j = 0; j < k; ++j) {
        const double s = sig[static_cast<size_t>(perm[static_cast<size_t>(j)])];
        out.sigma[static_cast<size_t>(j)] = s;
        inv[static_cast<size_t>(j)] = (s > 0.0) ? 1.0 / s : 0.0;
    }
    E.perm.ensure(static_cast<size_t>(std::max<i64>(k, factor_cols(m + n, st.min_dim))));
    out.d_sigma.ensure(static_cast<size_t>(2 * std::max<i64>(k, factor_cols(m + n, st.min_dim))));
    SVT_CUDA(cudaMemcpyAsync(E.perm.get(), perm.data(), sizeof(int) * k, cudaMemcpyHostToDevice, c->stream));
    SVT_CUDA(cudaMemcpyAsync(out.d_sigma.get(), out.sigma.data(), sizeof(double) * k, cudaMemcpyHostToDevice,
                             c->stream));
    SVT_CUDA(cudaMemcpyAsync(out.d_sigma.get() + k, inv.data(), sizeof(double) * k, cudaMemcpyHostToDevice,
                             c->stream));
    // V = (B^T W)[:, perm] / sigma
    out.V.ensure(static_cast<size_t>(n * std::max<i64>(k, factor_cols(m + n, st.min_dim))));
    permute_cols(c, E.Vraw.get(), n, kc, E.perm.get(), k, out.V.get(), k);
    scale_cols(c, out.V.get(), n, k, k, out.d_sigma.get() + k);
    // U = Q W[:, perm]
    E.Wk.ensure(static_cast<size_t>(std::max<i64>(r * k, std::max(r, st.cap) * factor_cols(m + n, st.min_dim))));
    permute_cols(c, E.W.get(), r, r, E.perm.get(), k, E.Wk.get(), k);
    out.U.ensure(static_cast<size_t>(std::max<i64>(1, m) * std::max<i64>(k, factor_cols(m + n, st.min_dim))));
    gemm(c, K_FINAL, false, m, k, r, 1.0, st.Q.get(), st.cap, E.Wk.get(), k, 0.0, out.U.get(), k);
    // keep the host copy of sigma in sync with the stream (the inv upload
    // above reads a host vector that dies with this frame)
    sync_stream(c);
}

// Kept-mode finalize for larger bases: only the triplets with sigma > tau
// are needed (shrink, solver.hpp:110-120), so instead of a dense r x r
// eigendecomposition run a Rayleigh-Ritz subspace iteration on G = B B^T
// through B^T-products (never forming G).  R4SVD's basis starts with the
// previous iterate's kept left singular vectors (sketch.hpp:228-234), so in Q
// coordinates the new top singular subspace is close to e_1..e_s: the block
// is warm-started there and converges in a few sweeps.  The block grows
// until its smallest Ritz value falls below tau^2, and iterates until every
// Ritz pair at or above the threshold has residual <= 1e-12 * theta_1.
static void finalize_kept(Engine& E, const QBDev& st, double tau, i64 s_warm, u64 seed, DevFactors& out) {
    svt_ctx* c = E.ctx;
    const i64 r = st.rank, n = st.n, m = st.m_local;
    out.m_local = m;
    out.n = n;
    out.k = 0;
    out.sigma.clear();
    // small bases (single-CTA Jacobi up to 112), or bases of which a large
    // share is kept (the subspace
    // iteration would span most of the space anyway, and the pairs crowd
    // against the threshold where its residual criterion converges slowest):
    // the dense Gram eigensolve, exact to rounding
    if (r <= 112 || (r <= 1024 && 4 * (s_warm + 16) >= r)) {
        finalize(E, st, FinalizeMode::Kept, tau, out);
        return;
    }
    const double tau2 = tau * tau;
    i64 b = std::min<i64>(r, std::max<i64>(s_warm + 16, 24));
    const i64 sw = std::min(s_warm, b);
    // engine-owned workspaces (grow-only; no per-iteration cudaMalloc/free)
    DevBuf<double>&Z = E.fkZ, &Zq = E.fkZq, &Zt = E.fkZt, &Wn = E.fkWn, &H = E.fkH, &Yh = E.fkYh, &th = E.fkth,
    &ZY = E.fkZY, &Xr = E.fkXr, &res2 = E.fkres;
    // sized for the basis capacity, not the current rank: the rank grows
    // every SVT iteration and each regrow is a cudaFree (device-wide sync)
    const i64 rc = std::max(r, st.cap);
    auto grow = [&](i64 bb_need) {
        const i64 bb = std::max<i64>(bb_need, std::min<i64>(rc, 128));  // the block widens over iterations
        Z.ensure(static_cast<size_t>(rc * bb));
        Zq.ensure(static_cast<size_t>(rc * bb));
        Zt.ensure(static_cast<size_t>(rc * bb));
        Wn.ensure(static_cast<size_t>(n * std::max<i64>(bb, factor_cols(m + n, st.min_dim))));
        H.ensure(static_cast<size_t>(bb * bb));
        Yh.ensure(static_cast<size_t>(bb * bb));
        th.ensure(static_cast<size_t>(bb));
        ZY.ensure(static_cast<size_t>(rc * bb));
        Xr.ensure(static_cast<size_t>(rc * bb));
        res2.ensure(static_cast<size_t>(bb));
    };
    grow(b);
    fill(c, Z.get(), r * b, 0.0);
    set_identity_cols(c, Z.get(), r, b, sw);
    if (b > sw) gaussian_block_dev(c, r, b - sw, derive_seed_u(seed, 0x5EEDF1A1ULL), Z.get() + sw, b);
    std::vector<double> th_h, res_h;
    i64 kk = 0, kk_prev = -1;
    int sweeps = 0;
    const bool dbg = std::getenv("SVTB_DEBUG_FINAL") && std::getenv("SVTB_DEBUG_FINAL")[0] == '2';
    const int maxit = 100;
    for (int it = 0; it < maxit; ++it) {
        copy2d(c, Z.get(), b, Zt.get(), b, r, b);
        qr_orthonormal(E, r, false, Zt.get(), b, b, Zq.get(), b);
        gemm(c, K_FINAL, false, n, b, r, 1.0, st.Bt.get(), st.cap, Zq.get(), b, 0.0, Wn.get(), b);
        gemm(c, K_FINAL, true, r, b, n, 1.0, st.Bt.get(), st.cap, Wn.get(), b, 0.0, Z.get(), b);
        gemm(c, K_FINAL, true, b, b, r, 1.0, Zq.get(), b, Z.get(), b, 0.0, H.get(), b);
        sym_eig(c, H.get(), b, Yh.get(), th.get());
        gemm(c, K_FINAL, false, r, b, b, 1.0, Z.get(), b, Yh.get(), b, 0.0, ZY.get(), b);   // G X
        gemm(c, K_FINAL, false, r, b, b, 1.0, Zq.get(), b, Yh.get(), b, 0.0, Xr.get(), b);  // X (Ritz)
        copy2d(c, ZY.get(), b, Zt.get(), b, r, b);
        sub_scaled_cols(c, Zt.get(), Xr.get(), r, b, b, th.get());
        col_sumsq(c, Zt.get(), r, b, b, res2.get());
        th_h.resize(static_cast<size_t>(b));
        res_h.resize(static_cast<size_t>(b));
        read_doubles2(c, th.get(), res2.get(), static_cast<size_t>(b), th_h.data(), res_h.data());
        kk = 0;
        while (kk < b && th_h[static_cast<size_t>(kk)] > tau2 * (1.0 - 1e-6)) ++kk;
        if (kk == b && b < r) {
            // the block does not reach below the threshold: widen it
            const i64 b2 = std::min<i64>(r, 2 * b);
            Zt.ensure(static_cast<size_t>(rc * b2));
            copy2d(c, Zq.get(), b, Zt.get(), b2, r, b);
            gaussian_block_dev(c, r, b2 - b, derive_seed_u(seed, 0x5EEDF1A2ULL + static_cast<u64>(it)), Zt.get() + b,
                               b2);
            b = b2;
            std::swap(Z, Zt);
            grow(b);
            continue;
        }
        const double tol = 1e-12 * std::max(th_h[0], 0.0);
        bool conv = true;
        for (i64 i = 0; i < kk; ++i)
            if (!(std::sqrt(std::max(res_h[static_cast<size_t>(i)], 0.0)) <= tol)) conv = false;
        // first pair below the threshold: either converged to 1e-8 * theta_1,
        // or -- once the kept pairs have converged and the count held over
        // two sweeps -- its residual interval lies clearly below tau^2 (the
        // bulk under the threshold converges slowly but is rarely close to it)
        if (kk < b) {
            const double rk = std::sqrt(std::max(res_h[static_cast<size_t>(kk)], 0.0));
            const double tk = th_h[static_cast<size_t>(kk)];
            const bool settled = it >= 1 && kk == kk_prev && tk + rk < tau2 * (1.0 - 1e-6);
            if (!(rk <= 1e4 * tol || settled)) conv = false;
        }
        kk_prev = kk;
        sweeps = it + 1;
        if (dbg) {
            double mw = 0.0;
            for (i64 i = 0; i < kk; ++i) mw = std::max(mw, std::sqrt(std::max(res_h[static_cast<size_t>(i)], 0.0)));
            const double rb = kk < b ? std::sqrt(std::max(res_h[static_cast<size_t>(kk)], 0.0)) : 0.0;
            std::fprintf(stderr, "  sweep %d b=%lld kk=%lld wanted_res=%.3e bound_res=%.3e th0=%.6e thk=%.6e\n", it,
                         static_cast<long long>(b), static_cast<long long>(kk), mw / th_h[0], rb / th_h[0], th_h[0],
                         kk < b ? th_h[static_cast<size_t>(kk)] / tau2 : 0.0);
        }
        if (conv || b == r) break;
        if (it == maxit - 1) {
            // not converged in maxit sweeps: never hand back unconverged Ritz
            // pairs silently — the dense Gram eigensolve (exact to
            // rounding) where it is affordable, else a warning
            if (r <= 4096) {
                std::fprintf(stderr, "[svt_b200] finalize_kept: %d sweeps without convergence at r = %lld; "
                                     "using the dense Gram eigensolve\n", maxit, static_cast<long long>(r));
                finalize(E, st, FinalizeMode::Kept, tau, out);
                return;
            }
            std::fprintf(stderr, "[svt_b200] finalize_kept: %d sweeps without convergence at r = %lld "
                                 "(kept pairs' residual above 1e-12 theta_1)\n", maxit, static_cast<long long>(r));
            break;
        }
        // Chebyshev-accelerated subspace step (Zhou & Saad's scaled
        // recurrence): damp [0, theta_b] -- everything below the block's
        // smallest Ritz value -- and amplify the block, then rescale column i
        // by 1 / p(theta_i) so the filtered Ritz block stays well
        // conditioned for the Cholesky QR.  The degree keeps
        // p(theta_1) / p(theta_b) <= 1e4.
        const double cut = std::max(th_h[static_cast<size_t>(b - 1)], 0.0);
        const double lmax = th_h[0];
        const double e = 0.5 * cut, cc = 0.5 * cut;
        const double x0 = e > 0.0 ? (lmax - cc) / e : 0.0;
        int degree = 1;
        if (x0 > 1.0 + 1e-9) degree = static_cast<int>(std::clamp(std::floor(std::acosh(1e4) / std::acosh(x0)), 1.0, 12.0));
        if (degree >= 2) {
            const double sigma1 = e / (lmax - cc);
            double sigma = sigma1;
            double* Xp = Xr.get();  // p_{j-1}
            double* Yc = Z.get();   // p_j
            double* GY = ZY.get();  // G p_j (starts as G X)
            cheb_combine(c, Yc, GY, Xp, nullptr, r * b, cc, sigma1 / e, 0.0);  // p_1
            for (int j = 2; j <= degree; ++j) {
                gemm(c, K_FINAL, false, n, b, r, 1.0, st.Bt.get(), st.cap, Yc, b, 0.0, Wn.get(), b);
                gemm(c, K_FINAL, true, r, b, n, 1.0, st.Bt.get(), st.cap, Wn.get(), b, 0.0, GY, b);
                const double sn = 1.0 / (2.0 / sigma1 - sigma);
                cheb_combine(c, Xp, GY, Yc, Xp, r * b, cc, 2.0 * sn / e, sigma * sn);  // p_j -> Xp
                std::swap(Xp, Yc);
                sigma = sn;
            }
            if (Yc != Z.get()) copy2d(c, Yc, b, Z.get(), b, r, b);
            std::vector<double> sc(static_cast<size_t>(b));
            const double tx0 = std::cosh(degree * std::acosh(x0));
            for (i64 i = 0; i < b; ++i) {
                const double xi = std::max((th_h[static_cast<size_t>(i)] - cc) / e, 1.0);
                sc[static_cast<size_t>(i)] = tx0 / std::cosh(degree * std::acosh(xi));
            }
            SVT_CUDA(cudaMemcpyAsync(res2.get(), sc.data(), sizeof(double) * b, cudaMemcpyHostToDevice, c->stream));
            scale_cols(c, Z.get(), r, b, b, res2.get());
            sync_stream(c);  // sc dies with this scope
        } else {
            copy2d(c, ZY.get(), b, Z.get(), b, r, b);  // plain subspace step
        }
    }
    if (std::getenv("SVTB_DEBUG_FINAL"))
        std::fprintf(stderr, "[finalize_kept] r=%lld b=%lld kept=%lld sweeps=%d\n", static_cast<long long>(r),
                     static_cast<long long>(b), static_cast<long long>(kk), sweeps);
    c->stats[K_FINAL].flops += 0.0;
    const i64 kc = std::min(b, kk + 1);
    // V_raw = B^T (Zq Yh) = Wn Yh; sigma = column norms (Rayleigh quotients)
    E.Vraw.ensure(static_cast<size_t>(n * std::max<i64>(kc, factor_cols(m + n, st.min_dim))));
    gemm(c, K_FINAL, false, n, kc, b, 1.0, Wn.get(), b, Yh.get(), b, 0.0, E.Vraw.get(), kc);
    E.lam.ensure(static_cast<size_t>(std::max<i64>(kc, factor_cols(m + n, st.min_dim))));  // kept rank creeps up: no regrow
    col_sumsq(c, E.Vraw.get(), n, kc, kc, E.lam.get());
    std::vector<double> s2(static_cast<size_t>(kc));
    read_doubles(c, E.lam.get(), static_cast<size_t>(kc), s2.data());
    std::vector<double> sig(static_cast<size_t>(kc));
    for (i64 j = 0; j < kc; ++j) sig[static_cast<size_t>(j)] = std::sqrt(s2[static_cast<size_t>(j)]);
    std::vector<int> perm(static_cast<size_t>(kc));
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(),
                     [&](int a, int bb) { return sig[static_cast<size_t>(a)] > sig[static_cast<size_t>(bb)]; });
    i64 k = 0;
    while (k < kc && sig[static_cast<size_t>(perm[static_cast<size_t>(k)])] > tau) ++k;
    out.k = k;
    if (k == 0) return;
    out.sigma.resize(static_cast<size_t>(k));
    std::vector<double> inv(static_cast<size_t>(k));
    for (i64 j = 0; j < k; ++j) {
        out.sigma[static_cast<size_t>(j)] = sig[static_cast<size_t>(perm[static_cast<size_t>(j)])];
        inv[static_cast<size_t>(j)] = 1.0 / out.sigma[static_cast<size_t>(j)];
    }
    E.perm.ensure(static_cast<size_t>(std::max<i64>(k, factor_cols(m + n, st.min_dim))));
    out.d_sigma.ensure(static_cast<size_t>(2 * std::max<i64>(k, factor_cols(m + n, st.min_dim))));
    SVT_CUDA(cudaMemcpyAsync(E.perm.get(), perm.data(), sizeof(int) * k, cudaMemcpyHostToDevice, c->stream));
    SVT_CUDA(cudaMemcpyAsync(out.d_sigma.get(), out.sigma.data(), sizeof(double) * k, cudaMemcpyHostToDevice,
                             c->stream));
    SVT_CUDA(cudaMemcpyAsync(out.d_sigma.get() + k, inv.data(), sizeof(double) * k, cudaMemcpyHostToDevice,
                             c->stream));
    out.V.ensure(static_cast<size_t>(n * std::max<i64>(k, factor_cols(m + n, st.min_dim))));
    permute_cols(c, E.Vraw.get(), n, kc, E.perm.get(), k, out.V.get(), k);
    scale_cols(c, out.V.get(), n, k, k, out.d_sigma.get() + k);
    E.Wk.ensure(static_cast<size_t>(std::max<i64>(r * k, std::max(r, st.cap) * factor_cols(m + n, st.min_dim))));
    permute_cols(c, Xr.get(), r, b, E.perm.get(), k, E.Wk.get(), k);
    out.U.ensure(static_cast<size_t>(std::max<i64>(1, m) * std::max<i64>(k, factor_cols(m + n, st.min_dim))));
    gemm(c, K_FINAL, false, m, k, r, 1.0, st.Q.get(), st.cap, E.Wk.get(), k, 0.0, out.U.get(), k);
    sync_stream(c);
}

static double error_percentage(const QBDev& st) {
    if (!(st.frob_y_sq > 0.0)) throw std::domain_error("error_percentage: target has zero Frobenius norm");
    const double eps = (st.frob_y_sq - st.norm_b_sq) / st.frob_y_sq;
    return std::clamp(eps, 0.0, 1.0);
}

static void check_sketch_params(const svt_sketch_params& p) {
    if (p.t < 1 || p.dt < 1 || p.np < 0) throw std::invalid_argument("SketchParams: need t >= 1, dt >= 1, np >= 0");
    if (!(p.eps_threshold > 0.0 && p.eps_threshold < 1.0))
        throw std::invalid_argument("SketchParams: eps_threshold must lie in (0, 1)");
}

static void finalize_mode(Engine& E, const QBDev& st, FinalizeMode mode, double tau, i64 s_warm, u64 seed,
                          DevFactors& out) {
    const bool dense = std::getenv("SVTB_FINALIZE_DENSE") != nullptr;  // per sketch; test / debug switch
    if (mode == FinalizeMode::Kept && !dense)
        finalize_kept(E, st, tau, s_warm, seed, out);
    else
        finalize(E, st, mode, tau, out);
}

// Speculative batch of K extension rounds.  Round j's sketch
// Y Y^T Y Omega_j does not depend on the basis, so rounds round0..round0+K-1
// are sketched together as one W = K*dt wide panel; the panel is projected
// against Q with classical Gram-Schmidt (second pass when any block needs
// it, the reference's test of sketch.hpp:134 per block) and factored by one
// Cholesky QR of the whole panel — R is upper triangular, so the first j
// blocks of the result span exactly what j sequential rounds would have
// added (same nested spans as qb_extend's block-by-block QR).  The energy of
// each block's coefficient rows then replays the reference's
// `while error_percentage > eps` test round by round; the blocks after the
// stopping round are discarded.  Returns the number of rounds accepted, or
// -1 when the panel is numerically rank deficient (the caller re-runs the
// rounds one by one with the exact fallback semantics).
// Sketch of a batch (Omega for rounds round0 .. round0 + K - 1, then
// Gram-Schmidt coefficients C (r0 x w) = Q[:, :r0]^T X (sketch.hpp:133) on
// the INT8 tensor cores from cached digit slices of the basis (ozaki.cu),
// else the DMMA GEMM.  The slices of a column are built once, the first time
// the column takes part in a product.  Opt-in (SVTB_OZAKI=1, bases of >= 64
// columns): in isolation the INT8 kernel measured slower than cuBLAS DGEMM
// on the config-4 Gram-Schmidt shape (profiles/r01_ozaki_bench.txt), so the
// default is the DMMA kernel.
static bool ozaki_enabled(i64 r0) {  // read per batch (cheap), so tests can toggle it
    const char* e = std::getenv("SVTB_OZAKI");
    (void)r0;
    return e != nullptr && std::atoi(e) != 0;
}

static void basis_tx(Engine& E, QBDev& st, i64 r0, i64 w, const double* X, i64 ldx, double* C) {
    svt_ctx* c = E.ctx;
    const i64 m = st.m_local;
    const double* Q = st.Q.get();
    if (ozaki_enabled(r0) && m >= 4096 && r0 >= 64 && w > 16) {
        const i64 tiles = ozaki_rows_pad(st.cap) / 128;
        const size_t bytes = static_cast<size_t>(8) * tiles * 128 * ozaki_kpad(m);
        if (st.qs_tiles != tiles) {
            st.qs.release();
            st.qe.release();
            st.qs_tiles = 0;
            st.qs_valid = 0;
            size_t free_b = 0, total_b = 0;
            SVT_CUDA(cudaMemGetInfo(&free_b, &total_b));
            if (bytes < free_b / 2) {
                st.qs.alloc(bytes / 8 + 2);
                st.qe.alloc(static_cast<size_t>(tiles * 128));
                st.qs_tiles = tiles;
            }
        }
        if (st.qs_tiles == tiles) {
            int8_t* sl = reinterpret_cast<int8_t*>(st.qs.get());
            if (st.qs_valid < r0) {
                ozaki_slice_basis(c, Q + st.qs_valid, m, r0 - st.qs_valid, st.cap, st.qs_valid, sl, tiles,
                                  st.qe.get());
                st.qs_valid = r0;
            }
            gemm_tn_ozaki_cached(c, r0, w, m, sl, tiles, st.qe.get(), X, ldx, C, w);
            return;
        }
    }
    gemm(c, K_GEMM, true, r0, w, m, 1.0, Q, st.cap, X, ldx, 0.0, C, w);
}

// SVTB_COEFF_VIA_B=0: Gram-Schmidt coefficients of a batch as Q^T X (an
// m-row contraction) instead of B T (read per batch: A/B and test switch)
static bool coeff_via_b() {
    const char* e = std::getenv("SVTB_COEFF_VIA_B");
    return e == nullptr || e[0] != '0';
}

// X = Y (Y^T (Y Omega))) into spec slot `slot`, on `stream` (main or side).
static void batch_sketch(Engine& E, const svt_sketch_params& p, int round0, int K, int slot, bool side) {
    svt_ctx* c = E.ctx;
    svt_mat* A = E.mat;
    auto& sp = E.spec;
    const i64 w = p.dt, W = static_cast<i64>(K) * w, m = A->m_local, n = A->n;
    cudaStream_t s = side ? c->side : c->stream;
    NvtxRange nvtx(side ? "r4svd.batch_sketch (side stream)" : "r4svd.batch_sketch");
    DevBuf<double>* part = side ? &sp.part : nullptr;
    u64 seeds[kMaxOmegaBatch];
    for (int k = 0; k < K; ++k) seeds[k] = derive_seed_u(p.seed, static_cast<u64>(round0 + k));
    // batch panels sized for the widest batch at once (W grows over the first
    // batches; a regrow inside an SVT iteration is a device-wide sync)
    const i64 Wc = std::max<i64>(W, kMaxBatchW);
    sp.om[slot].ensure(static_cast<size_t>(n * Wc));
    sp.x[slot].ensure(static_cast<size_t>(std::max<i64>(1, m) * Wc));
    sp.t[slot].ensure(static_cast<size_t>(n * Wc));
    gaussian_blocks_dev(c, n, w, seeds, K, sp.om[slot].get(), w, W, side);
    sp_mult(E, W, sp.om[slot].get(), W, sp.x[slot].get(), W, s, part);
    for (int j = 0; j < p.np; ++j) {  // np <= 1 on this path
        sp_mult_t(E, W, sp.x[slot].get(), W, sp.t[slot].get(), s, part);
        sp_mult(E, W, sp.t[slot].get(), W, sp.x[slot].get(), W, s, part);
    }
}

static int qb_extend_batch(Engine& E, QBDev& st, const svt_sketch_params& p, int round0, int K,
                           double* last_gain, int K_next) {
    svt_ctx* c = E.ctx;
    svt_mat* A = E.mat;
    auto& sp = E.spec;
    const i64 w = p.dt, m = A->m_local, n = A->n, r0 = st.rank;
    static const bool no_spec = std::getenv("SVTB_NO_SPECULATION") != nullptr;
    const bool use_spec = sp.valid && sp.gen == E.sketch_gen && sp.seed == p.seed && sp.round0 == round0;
    int slot = 0;
    if (sp.valid) {
        // the batch sketched on the side stream during the previous batch
        // (or a stale one from an ended sketch, drained here)
        SVT_CUDA(cudaStreamWaitEvent(c->stream, sp.ready, 0));
        slot = use_spec ? sp.slot : (sp.slot ^ 1);
        if (use_spec) K = sp.K;
    }
    sp.valid = false;
    const i64 W = static_cast<i64>(K) * w;
    ensure_cap(E, st, r0 + W);
    if (!use_spec) batch_sketch(E, p, round0, K, slot, false);
    // speculative sketch of the next batch (rounds round0 + K ..): it only
    // needs Omega and Y, so it runs on the side stream concurrently with this
    // batch's Gram-Schmidt / QR; the replay below decides whether it is used
    const i64 room = (st.min_dim - (r0 + W)) / w;
    const int Kn = static_cast<int>(std::min<i64>(K_next, room));
    // multi-rank: the side stream's Y^T X all-reduces need their own
    // communicator (ncclCommSplit) or the host-staged mode; opt-in there
    // (SVTB_SPEC_MULTI=1) until it has run on NVLink hardware
    const char* sm_env = std::getenv("SVTB_SPEC_MULTI");  // per batch: tests toggle it
    const bool spec_multi = sm_env != nullptr && sm_env[0] == '1';
    const bool spec_ok = !c->comm.dist() || (spec_multi && c->comm.side_capable());
    // enqueued after this batch's first main-stream kernels, so the main
    // stream (the critical path) restarts as early as possible after the
    // previous batch's host synchronization
    bool spec_launched = false;
    auto launch_spec = [&]() {
        if (spec_launched) return;
        spec_launched = true;
        if (c->side && Kn >= 2 && !no_spec && spec_ok && c->speculate) {
            if (!sp.ready) {
                SVT_CUDA(cudaEventCreateWithFlags(&sp.ready, cudaEventDisableTiming));
                SVT_CUDA(cudaEventCreateWithFlags(&sp.freed[0], cudaEventDisableTiming));
                SVT_CUDA(cudaEventCreateWithFlags(&sp.freed[1], cudaEventDisableTiming));
                SVT_CUDA(cudaEventRecord(sp.freed[0], c->stream));
                SVT_CUDA(cudaEventRecord(sp.freed[1], c->stream));
            }
            const int ns = slot ^ 1;
            // buffers of slot ns are free once the main stream is done with the
            // batch that used them; regrowth (cudaFree) synchronizes the device
            SVT_CUDA(cudaStreamWaitEvent(c->side, sp.freed[ns], 0));
            batch_sketch(E, p, round0 + K, Kn, ns, true);
            SVT_CUDA(cudaEventRecord(sp.ready, c->side));
            sp.valid = true;
            sp.gen = E.sketch_gen;
            sp.seed = p.seed;
            sp.round0 = round0 + K;
            sp.K = Kn;
            sp.slot = ns;
        }
    };
    double* XW = sp.x[slot].get();
    const i64 Wc = std::max<i64>(W, kMaxBatchW);
    E.TW.ensure(static_cast<size_t>(n * Wc));
    double* Q = st.Q.get();
    const i64 ldq = st.cap;
    if (r0 > 0) {
        NvtxRange nvtx("r4svd.block_gram_schmidt");
        // block Gram-Schmidt against Q, then the reference's per-round test
        // ||Q^T X_k|| > 1e-8 ||X_k|| for a second pass (sketch.hpp:134).
        // After one pass ||Q^T X_k|| is a rounding residual, at most
        // ~(m + r0) * eps * ||X_k before||; while the projection
        // keeps more than max(1e-3, 1e8 (m + r0) eps) of every block's norm
        // the test is false with that margin, so the check product Q^T X is
        // only formed when some block lost more (near-dependent rounds).
        E.CW.ensure(static_cast<size_t>(std::max(r0, st.cap) * Wc));  // basis capacity: no regrow as r0 grows
        E.eW.ensure(static_cast<size_t>(4 * Wc));
        // Gram-Schmidt coefficients C = Q^T X.  The batch panel is
        // X = Y T with T = Y^T Y Omega (np = 1) or Omega (np = 0), and the
        // coefficient rows B = Q^T Y of the basis are already stored (B^T,
        // n x r0), so C = B T: a contraction over n instead of m rows
        // (6.5x fewer flops at config 4), replicated on every rank (no
        // all-reduce).  In exact arithmetic it is Q^T X.  Measured at
        // config 4 (SVTB_DEBUG_BATCH), the residual max ||Q^T X'_k|| /
        // ||X'_k|| after the pass is the same either way (1e-15 .. 9e-10,
        // set by the basis' own orthogonality level amplified by the
        // cancellation ||X_k|| / ||X'_k||), so the reference's second-pass
        // test below is predicted by the same rule.
        const double* Tp = (p.np == 1) ? sp.t[slot].get() : sp.om[slot].get();
        const bool via_b = coeff_via_b() && p.np <= 1 && n < m;
        col_sumsq(c, XW, m, W, W, E.eW.get() + 2 * W);
        if (via_b) {
            gemm(c, K_GEMM, true, r0, W, n, 1.0, st.Bt.get(), ldq, Tp, W, 0.0, E.CW.get(), W);
        } else {
            basis_tx(E, st, r0, W, XW, W, E.CW.get());
            allreduce(c, E.CW.get(), static_cast<size_t>(r0 * W));
        }
        gemm(c, K_GEMM, false, m, W, r0, -1.0, Q, ldq, E.CW.get(), W, 1.0, XW, W);
        launch_spec();
        col_sumsq(c, XW, m, W, W, E.eW.get());
        allreduce(c, E.eW.get(), static_cast<size_t>(W));
        if (debug_batch()) {
            // SVTB_DEBUG_BATCH: the residual max_k ||Q^T X'_k|| / ||X'_k|| after
            // the first pass (a direct product: diagnostics only)
            E.D.ensure(static_cast<size_t>(std::max(r0, st.cap) * Wc));
            gemm(c, K_OTHER, true, r0, W, m, 1.0, Q, ldq, XW, W, 0.0, E.D.get(), W);
            allreduce(c, E.D.get(), static_cast<size_t>(r0 * W));
            std::vector<double> dn(static_cast<size_t>(W)), xn(static_cast<size_t>(W)), bn(static_cast<size_t>(W));
            E.G.ensure(static_cast<size_t>(3 * Wc));
            col_sumsq(c, E.D.get(), r0, W, W, E.G.get());
            read_doubles(c, E.G.get(), static_cast<size_t>(W), dn.data());
            read_doubles(c, E.eW.get(), static_cast<size_t>(W), xn.data());
            read_doubles(c, E.eW.get() + 2 * W, static_cast<size_t>(W), bn.data());
            double worst = 0.0, kept = 1e300;
            for (int k = 0; k < K; ++k) {
                double d2 = 0, x2 = 0, b2 = 0;
                for (i64 q = 0; q < w; ++q) {
                    d2 += dn[static_cast<size_t>(k * w + q)];
                    x2 += xn[static_cast<size_t>(k * w + q)];
                    b2 += bn[static_cast<size_t>(k * w + q)];
                }
                worst = std::max(worst, std::sqrt(d2 / x2));
                kept = std::min(kept, std::sqrt(x2 / b2));
            }
            std::fprintf(stderr, "[batch] r0=%lld via_b=%d residual max ||Q^T X'_k||/||X'_k|| = %.3e, min kept ratio %.3e\n",
                         static_cast<long long>(r0), via_b ? 1 : 0, worst, kept);
        }
        // the decisions are taken on the device (predicated kernels), so the
        // batch issues no host synchronization here
        // the check product Q^T X' (and with it the reference's test) is only
        // formed when some block kept less than max(1e-3, 1e8 (m + r0) eps)
        // of its norm (near-dependent rounds)
        allreduce(c, E.eW.get() + 2 * W, static_cast<size_t>(W));
        const double thr = std::max(1e-3, 1.1e-8 * static_cast<double>(A->m + r0));
        block_flags(c, E.eW.get(), E.eW.get() + 2 * W, nullptr, K, static_cast<int>(w), thr * thr, 0, nullptr,
                    dfl(c, F_CHECK));
        gemm(c, K_GEMM, true, r0, W, m, 1.0, Q, ldq, XW, W, 0.0, E.CW.get(), W, dfl(c, F_CHECK));
        allreduce(c, E.CW.get(), static_cast<size_t>(r0 * W));
        col_sumsq(c, E.CW.get(), r0, W, W, E.eW.get() + W);
        block_flags(c, E.eW.get(), nullptr, E.eW.get() + W, K, static_cast<int>(w), 0.0, 1, dfl(c, F_CHECK),
                    dfl(c, F_SECOND));
        gemm(c, K_GEMM, false, m, W, r0, -1.0, Q, ldq, E.CW.get(), W, 1.0, XW, W, dfl(c, F_SECOND));
        if (debug_batch())
            std::fprintf(stderr, "[batch] round0=%d K=%d r0=%lld check=%d second_pass=%d\n", round0, K,
                         static_cast<long long>(r0), read_flag(c, F_CHECK), read_flag(c, F_SECOND));
    }
    launch_spec();  // (r0 == 0: no Gram-Schmidt kernels before it)
    NvtxRange nvtx_qr("r4svd.cholqr2 + coefficients");
    // one Cholesky QR (twice) of the whole panel: nested spans per block
    E.GW.ensure(static_cast<size_t>(Wc * Wc));
    E.RW.ensure(static_cast<size_t>(Wc * Wc));
    E.X2.ensure(static_cast<size_t>(std::max<i64>(1, m) * Wc));
    zero_flag(c, F_QRSTAT);
    int* status = dfl(c, F_QRSTAT);
    gemm(c, K_QR, true, W, W, m, 1.0, XW, W, XW, W, 0.0, E.GW.get(), W);
    allreduce(c, E.GW.get(), static_cast<size_t>(W * W));
    chol_rinv(c, E.GW.get(), W, E.RW.get(), status, nullptr);
    gemm(c, K_QR, false, m, W, W, 1.0, XW, W, E.RW.get(), W, 0.0, E.X2.get(), W);
    if (sp.freed[slot]) SVT_CUDA(cudaEventRecord(sp.freed[slot], c->stream));  // XW is dead from here
    gemm(c, K_QR, true, W, W, m, 1.0, E.X2.get(), W, E.X2.get(), W, 0.0, E.GW.get(), W);
    allreduce(c, E.GW.get(), static_cast<size_t>(W * W));
    static const bool debug_g2 = std::getenv("SVTB_DEBUG_G2") != nullptr;
    if (debug_g2) {
        maxabs(c, E.GW.get(), W, W, W, 1.0, dsc(c, S_TMP));
        std::fprintf(stderr, "[g2] W=%lld max|G2-I|=%.3e\n", static_cast<long long>(W), read_scalar(c, S_TMP));
    }
    chol_rinv(c, E.GW.get(), W, E.RW.get(), status, nullptr);
    gemm(c, K_QR, false, m, W, W, 1.0, E.X2.get(), W, E.RW.get(), W, 0.0, Q + r0, ldq);
    // coefficient rows of the whole batch and their per-block energies,
    // enqueued before the QR status is known: status and energies come back
    // with one synchronization (after a failed QR the columns r0.. of Q and
    // B^T are rewritten by the sequential rounds that replace the batch)
    if (!c->comm.dist()) {  // straight into the coefficient rows (no staging copy)
        sp_mult_t(E, W, Q + r0, ldq, st.Bt.get() + r0, nullptr, nullptr, ldq);
        col_sumsq(c, st.Bt.get() + r0, n, W, ldq, E.eW.get());
    } else {
        sp_mult_t(E, W, Q + r0, ldq, E.TW.get());
        copy2d(c, E.TW.get(), W, st.Bt.get() + r0, ldq, n, W);
        col_sumsq(c, E.TW.get(), n, W, W, E.eW.get());
    }
    std::vector<double> e(static_cast<size_t>(W));
    if (read_flag_and_doubles(c, F_QRSTAT, E.eW.get(), static_cast<size_t>(W), e.data()) != 0) {
        if (debug_batch())
            std::fprintf(stderr, "[batch] round0=%d K=%d W=%lld r0=%lld: Cholesky QR failed, sequential rounds\n",
                         round0, K, static_cast<long long>(W), static_cast<long long>(r0));
        return -1;
    }
    // replay the reference's loop test round by round
    int accepted = 0;
    for (int k = 0; k < K; ++k) {
        if (k > 0 && !(error_percentage(st) > p.eps_threshold)) break;
        double ek = 0.0;
        for (i64 q = 0; q < w; ++q) ek += e[static_cast<size_t>(k * w + q)];
        st.norm_b_sq += ek;
        *last_gain = ek / st.frob_y_sq;
        st.rank += w;
        ++accepted;
    }
    st.saturated = (st.rank == st.min_dim);
    return accepted;
}

static SketchOut run_loop(Engine& E, QBDev& st, const svt_sketch_params& p, FinalizeMode mode, double tau,
                          i64 s_warm) {
    SketchOut out;
    out.f = std::move(E.fpool);  // reuse the previous sketch's factor buffers (no per-sketch cudaMalloc / cudaFree)
    int rounds = 0;
    ++E.sketch_gen;  // speculative batches of an earlier sketch can never be used by this one
    // Omega bank: the Gaussian blocks of the next rounds depend only on
    // (seed, round) (sketch.hpp:246-247), so they are generated kMaxOmegaBatch
    // at a time by independent mt19937_64 warps in two launches.
    int bank_first = 1, bank_count = 0;
    double last_gain = -1.0;  // energy fraction added by the latest round
    const i64 n = E.mat->n;
    while (error_percentage(st) > p.eps_threshold) {
        if (st.saturated) {
            finalize_mode(E, st, mode, tau, s_warm, p.seed, out.f);
            out.rank = st.rank;
            out.saturated = true;
            out.rounds = rounds;
            return out;
        }
        // speculative batch: size from the previous sketch's round count
        // (ramp 2, 4, 8, ... without history), bounded by the remaining
        // dimensions and the 128-column Cholesky panel
        if (E.batching && p.np <= 1) {
            const i64 room = (st.min_dim - st.rank) / p.dt;
            const int kmax = static_cast<int>(std::min<i64>(std::min<i64>(kMaxOmegaBatch, 128 / p.dt), room));
            // rounds still needed: the previous sketch's count (round counts
            // grow slowly while the threshold cools) and a linear
            // extrapolation of the last round's energy gain (gains shrink
            // round by round, so this underestimates: no wasted work)
            int est = (E.last_rounds > 0) ? (E.last_rounds - rounds + 1) : std::max(2, 2 * rounds);
            const double ep = error_percentage(st);
            if (last_gain > 0.0) {
                const double need = (ep - p.eps_threshold) / last_gain;
                est = std::max(est, static_cast<int>(std::min(1e6, std::ceil(need))) + 1);
            }
            const int K = std::min(kmax, est);
            // a batch already sketched on the side stream for this round
            // is used whatever the current estimate
            const bool spec_here = E.spec.valid && E.spec.gen == E.sketch_gen && E.spec.seed == p.seed &&
                                   E.spec.round0 == rounds + 1;
            if (K >= 2 || spec_here) {
                // size of the batch after this one if all of this one's
                // rounds are accepted (same estimate, K rounds later)
                const int Kb = spec_here ? E.spec.K : K;
                const int est_next = est - Kb;
                const int K_next = std::min<int>(static_cast<int>(std::min<i64>(kMaxOmegaBatch, 128 / p.dt)), est_next);
                const int acc = qb_extend_batch(E, st, p, rounds + 1, K, &last_gain, K_next);
                if (acc > 0) {
                    rounds += acc;
                    continue;
                }
            }
        }
        ++rounds;
        const double* omega = nullptr;
        if (st.min_dim - st.rank >= p.dt) {
            if (rounds >= bank_first + bank_count) {
                const i64 left = (st.min_dim - st.rank) / p.dt;
                const int K = static_cast<int>(std::max<i64>(1, std::min<i64>(kMaxOmegaBatch, left)));
                u64 seeds[kMaxOmegaBatch];
                for (int k = 0; k < K; ++k) seeds[k] = derive_seed_u(p.seed, static_cast<u64>(rounds + k));
                E.OmBank.ensure(static_cast<size_t>(K * n * p.dt));
                gaussian_blocks_dev(E.ctx, n, p.dt, seeds, K, E.OmBank.get(), n * p.dt, p.dt);
                bank_first = rounds;
                bank_count = K;
            }
            omega = E.OmBank.get() + static_cast<i64>(rounds - bank_first) * n * p.dt;
        }
        const double nb_before = st.norm_b_sq;
        qb_extend(E, st, p.dt, p.np, derive_seed_u(p.seed, static_cast<u64>(rounds)), omega);
        last_gain = (st.norm_b_sq - nb_before) / st.frob_y_sq;
    }
    E.last_rounds = rounds;
    finalize_mode(E, st, mode, tau, s_warm, p.seed, out.f);
    out.rank = st.rank;
    out.saturated = false;
    out.rounds = rounds;
    return out;
}

// sketch.hpp:188-201
SketchOut r3svd(Engine& E, const svt_sketch_params& p, FinalizeMode mode, double tau, double frob_y_sq) {
    check_sketch_params(p);
    prepare_tiles(E);  // Y may have changed since the previous sketch
    QBDev& st = E.qb;
    qb_init(E, st, p.t, p.np, derive_seed_u(p.seed, 0), frob_y_sq);
    return run_loop(E, st, p, mode, tau, 0);
}

// sketch.hpp:207-250
SketchOut r4svd(Engine& E, const double* U_prev, i64 ldu, i64 s, const svt_sketch_params& p, FinalizeMode mode,
                double tau, double frob_y_sq) {
    check_sketch_params(p);
    if (s == 0) {
        svt_sketch_params fresh = p;
        fresh.t = p.dt;
        return r3svd(E, fresh, mode, tau, frob_y_sq);
    }
    svt_ctx* c = E.ctx;
    svt_mat* A = E.mat;
    const i64 min_dim = std::min(A->m, A->n);
    if (s > min_dim) throw std::invalid_argument("r4svd: recycled basis wider than min(m, n)");
    prepare_tiles(E);
    if (frob_y_sq < 0.0) frob_y_sq = frob_sq(E);
    if (!(frob_y_sq > 0.0)) throw std::domain_error("r4svd: target matrix is all zero");
    const i64 m = A->m_local;
    QBDev& st = E.qb;
    reset_qb(st, A);
    st.m_local = m;
    st.n = A->n;
    st.min_dim = min_dim;
    ensure_cap(E, st, s);
    copy2d(c, U_prev, ldu, st.Q.get(), st.cap, m, s);
    // drift test max|U^T U - I| > 1e-8 -> qr_orthonormal (sketch.hpp:229-233)
    E.D.ensure(static_cast<size_t>(s * s));
    gemm(c, K_GEMM, true, s, s, m, 1.0, st.Q.get(), st.cap, st.Q.get(), st.cap, 0.0, E.D.get(), s);
    allreduce(c, E.D.get(), static_cast<size_t>(s * s));
    maxabs(c, E.D.get(), s, s, s, 1.0, dsc(c, S_MAXD));
    set_flag(c, dsc(c, S_MAXD), nullptr, 1e-8, 1, dfl(c, F_DRIFT));
    if (s <= 64) {
        E.X2.ensure(static_cast<size_t>(std::max<i64>(1, m) * s));
        copy2d(c, U_prev, ldu, E.X2.get(), s, m, s, dfl(c, F_DRIFT));
        qr_panel(E, m, true, E.X2.get(), s, s, st.Q.get(), st.cap, dfl(c, F_DRIFT));
    } else if (read_flag(c, F_DRIFT)) {
        E.X2.ensure(static_cast<size_t>(std::max<i64>(1, m) * s));
        copy2d(c, U_prev, ldu, E.X2.get(), s, m, s);
        qr_orthonormal(E, E.X2.get(), s, s, st.Q.get(), st.cap);
    }
    append_coefficients(E, st, 0, s, 0);
    st.norm_b_sq = read_scalar(c, S_NB);
    st.frob_y_sq = frob_y_sq;
    st.rank = s;
    st.saturated = (s == min_dim);
    return run_loop(E, st, p, mode, tau, s);
}

// sketch.hpp:165-182
DevFactors rsvd(Engine& E, i64 k, const svt_sketch_params& p) {
    svt_mat* A = E.mat;
    const i64 min_dim = std::min(A->m, A->n);
    if (k < 1) throw std::invalid_argument("rsvd: k must be >= 1");
    if (p.p < 0 || k + p.p > min_dim) throw std::invalid_argument("rsvd: k + p must not exceed min(m, n)");
    prepare_tiles(E);
    QBDev st;
    // same kernels as qb_init (sketch.hpp:173-176), no zero-norm check
    const i64 t = k + p.p;
    st.m_local = A->m_local;
    st.n = A->n;
    st.min_dim = min_dim;
    ensure_cap(E, st, t);
    const i64 m = A->m_local;
    E.Om.ensure(static_cast<size_t>(A->n * t));
    E.X.ensure(static_cast<size_t>(std::max<i64>(1, m) * t));
    gaussian_block_dev(E.ctx, A->n, t, derive_seed_u(p.seed, 0), E.Om.get(), t);
    sp_mult(E, t, E.Om.get(), t, E.X.get(), t);
    power_iterate(E, t, p.np);
    qr_orthonormal(E, E.X.get(), t, t, st.Q.get(), st.cap);
    append_coefficients(E, st, 0, t, 0);
    st.rank = t;
    DevFactors f;
    finalize(E, st, FinalizeMode::Full, 0.0, f);
    // keep the leading k triplets
    if (f.k > k) {
        DevFactors g;
        g.m_local = f.m_local;
        g.n = f.n;
        g.k = k;
        g.sigma.assign(f.sigma.begin(), f.sigma.begin() + k);
        g.U.ensure(static_cast<size_t>(std::max<i64>(1, f.m_local) * k));
        g.V.ensure(static_cast<size_t>(f.n * k));
        g.d_sigma.ensure(static_cast<size_t>(2 * k));
        copy2d(E.ctx, f.U.get(), f.k, g.U.get(), k, f.m_local, k);
        copy2d(E.ctx, f.V.get(), f.k, g.V.get(), k, f.n, k);
        SVT_CUDA(cudaMemcpyAsync(g.d_sigma.get(), f.d_sigma.get(), sizeof(double) * k, cudaMemcpyDeviceToDevice,
                                 E.ctx->stream));
        sync_stream(E.ctx);
        return g;
    }
    return f;
}

// Full SVD of the densified iterate (solver.hpp:271-274): Q = I (m x m), B = Y.
DevFactors full_svd(Engine& E) {
    svt_ctx* c = E.ctx;
    svt_mat* A = E.mat;
    if (c->comm.world != 1) throw std::invalid_argument("full-svd backend is single-GPU only");
    QBDev st;
    st.m_local = A->m;
    st.n = A->n;
    st.min_dim = std::min(A->m, A->n);
    st.cap = A->m;
    st.rank = A->m;
    st.Q.ensure(static_cast<size_t>(A->m * A->m));
    fill(c, st.Q.get(), A->m * A->m, 0.0);
    std::vector<double> eye(static_cast<size_t>(A->m * A->m), 0.0);
    for (i64 i = 0; i < A->m; ++i) eye[static_cast<size_t>(i * A->m + i)] = 1.0;
    SVT_CUDA(cudaMemcpyAsync(st.Q.get(), eye.data(), sizeof(double) * eye.size(), cudaMemcpyHostToDevice, c->stream));
    DevBuf<double> dense(static_cast<size_t>(A->m * A->n));
    densify_dev(c, A->m, A->n, A->rowptr.get(), A->col.get(), E.Y.csr, dense.get());
    st.Bt.ensure(static_cast<size_t>(A->n * A->m));
    transpose(c, dense.get(), A->m, A->n, A->n, st.Bt.get());
    sync_stream(c);
    DevFactors f;
    finalize(E, st, FinalizeMode::Full, 0.0, f);
    return f;
}

}  // namespace svtb
