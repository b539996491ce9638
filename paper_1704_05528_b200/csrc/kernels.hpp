// Host-side launchers of the sm_100a kernels (rng.cu, sparse.cu, dense.cu).
// All run on ctx->stream; none synchronizes.  Dense "panels" are ROW-MAJOR
// (element (i, j) at p[i * ld + j]) so that a sparse row gather reads one
// contiguous w-wide row; the C ABI converts to/from the reference's
// column-major Eigen layout at the boundary.
#pragma once

#include "common.hpp"

namespace svtb {

// ---- RNG (dense.hpp:52-98) ---------------------------------------------
// out (rows x cols, row-major, leading dim ld) <- the column-major fill of one
// fresh std::mt19937_64(seed) Box-Muller stream: out[i*ld + j] = z[i + j*rows].
void gaussian_block_dev(svt_ctx* ctx, i64 rows, i64 cols, u64 seed, double* out, i64 ld);
// K <= kMaxOmegaBatch independent blocks in two launches (one warp per
// stream): block k from std::mt19937_64(seeds[k]) into out + k * out_stride.
constexpr int kMaxOmegaBatch = 32;
// on_side: run on ctx->side with its own scratch (the caller orders it
// against the main stream with events).
void gaussian_blocks_dev(svt_ctx* ctx, i64 rows, i64 cols, const u64* seeds, int K, double* out, i64 out_stride,
                         i64 ld, bool on_side = false);

// ---- sparse (sampled.hpp) ---------------------------------------------------
// out[i, 0:w] = sum_{k in ptr[i]..ptr[i+1]} val[k] * X[idx[k], 0:w], i < nrows.
// CSR (Y*X, sampled.hpp:113) and CSC (Y^T*X, sampled.hpp:130) use the same
// kernel with the respective arrays.
// nnz and x_rows only feed the algorithmic-bytes accounting (SURVEY §8d:
// 12 B per entry + 8 B per row pointer + panel in + panel out).
// stream / scratch (optional): launch on another stream with its own
// long-row partial buffer (a speculative batch on ctx->side).
void spmm(svt_ctx* ctx, int cls, const SegPlanView& plan, i64 nrows, const int* idx, const double* val, i64 nnz,
          i64 x_rows, i64 w, const double* X, i64 ldx, double* out, i64 ldo, cudaStream_t stream = nullptr,
          DevBuf<double>* scratch = nullptr);

// Shared-memory-tiled variant for wide panels (TilePlanView); returns false
// when the call is outside its limits (the caller then uses spmm).  The
// plan's entries must mirror the current values (tile_values).
bool tile_spmm_enabled();
bool spmm_tiled(svt_ctx* ctx, int cls, const TilePlanView& P, i64 x_rows, i64 w, const double* X, i64 ldx,
                double* out, i64 ldo, cudaStream_t stream = nullptr, DevBuf<double>* scratch = nullptr);
void tile_values(svt_ctx* ctx, const TilePlanView& P, const double* Ycsr);

// Fused SDDMM + Bregman update + reductions (sampled.hpp:148-176,
// solver.hpp:143-168, 321-323).  For each stored (i, j):
//   p = U[i,:] . Vs[j,:]   (Vs = V diag(sigma))
//   d = A - p;  y_old = Y;
//   mode 1: Y = y_old + delta * d (and the Ycsc mirror)   [Bregman update]
//   mode 2: Y = p                                          [project_low_rank]
//   mode 0: no write                                       [held-out metrics]
// sums[0..3] (device) = sum|d|, sum d^2, sum (A - y_old)^2, sum Y_out^2.
void sddmm_update(svt_ctx* ctx, const SegPlanView& plan, i64 m_local, const int* col, const double* A, double* Y,
                  double* Ycsc, const int* csr2csc, i64 nnz, i64 n, const double* U, i64 ldu, const double* Vs,
                  i64 ldv, i64 k, double delta, int mode, double* d_sums4);

// Ycsc[p] = Y[csc2csr[p]]: rebuild the CSC value mirror after an update
void mirror_csc(svt_ctx* ctx, i64 nnz, const int* csc2csr, const double* Y, double* Ycsc);
// vals_out = alpha * vals_in (and the CSC mirror through csr2csc when given)
void scale_values(svt_ctx* ctx, i64 nnz, const double* in, double alpha, double* out, const int* csr2csc,
                  double* out_csc);
// out[k] = a[k] + alpha * b[k]
void axpy_values(svt_ctx* ctx, i64 nnz, const double* a, double alpha, const double* b, double* out);
// dense (m_local x n, row-major) <- scatter of CSR values (FullSvd backend)
void densify_dev(svt_ctx* ctx, i64 m_local, i64 n, const i64* rowptr, const int* col, const double* val,
                 double* out);

// ---- FP64 on the INT8 tensor cores (ozaki.cu) ----------------------------------
// C (M x N) = alpha * A^T B + beta * C; A: K x M, B: K x N, row-major FP64;
// slices = int8 digits per entry (8: FP64-equivalent, 6..8 accepted).
void gemm_tn_ozaki(svt_ctx* ctx, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda, const double* B,
                   i64 ldb, double beta, double* C, i64 ldc, int slices = 8);
// cached-A form (8 slices): the basis slices live in a 128-row tiled int8
// array of ctiles row tiles x ozaki_kpad(K) digits per slice
i64 ozaki_kpad(i64 K);
i64 ozaki_rows_pad(i64 rows);
void ozaki_slice_basis(svt_ctx* ctx, const double* X, i64 K, i64 C, i64 ld, i64 c_off, int8_t* tiles, i64 ctiles,
                       int* e);
void gemm_tn_ozaki_cached(svt_ctx* ctx, i64 M, i64 N, i64 K, const int8_t* tiles, i64 ctiles, const int* e,
                          const double* B, i64 ldb, double* C, i64 ldc);

// ---- dense ------------------------------------------------------------------
// C (M x N) = alpha * op(A) * B + beta * C; op(A) = A^T when transA (A stored
// K x M row-major), else A (M x K row-major).  B is K x N row-major.  Large K
// with a small output is split across CTAs with a deterministic fixed-order
// reduction.  pred (device int, may be null): skip entirely when *pred == 0.
void gemm(svt_ctx* ctx, int cls, bool transA, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
          const double* B, i64 ldb, double beta, double* C, i64 ldc, const int* pred = nullptr);
// Tall row-major C = alpha A B + beta C through the CUTLASS DMMA template
// (cutlass_gemm.cu); false when the shape is outside its limits (the caller
// uses its own kernels).
bool cutlass_gemm_nn(svt_ctx* ctx, cudaStream_t s, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
                     const double* B, i64 ldb, double beta, double* C, i64 ldc);
// C = alpha A^T B + beta C (A stored K x M row-major), CUTLASS DMMA template
// with a deterministic parallel split-K through ws; false when it does not
// apply (shape limits, workspace)
bool cutlass_gemm_tn(svt_ctx* ctx, cudaStream_t s, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
                     const double* B, i64 ldb, double beta, double* C, i64 ldc, DevBuf<double>& ws);
// The same partials through a CUTLASS template with the panel-row gather in
// its operand iterator (returns the split count, 0 = not applicable)
int cutlass_dense_block(svt_ctx* ctx, cudaStream_t s, bool transA, i64 M, i64 N, i64 K, const double* D, i64 ldd,
                        const double* B, i64 ldb, const int* brow, DevBuf<double>& ws);
// Dense corner of a split sparse product: split-K partials of op(D) B[brow, :]
// on the FP64 tensor cores into ws on stream s (returns the split count, 0 =
// operands not 16-byte aligned, nothing launched); dense_block_add adds their
// fixed-order sum into out[orow[i], :].
int dense_block_mm(svt_ctx* ctx, cudaStream_t s, int cls, bool transA, i64 M, i64 N, i64 K, const double* D,
                   i64 ldd, const double* B, i64 ldb, const int* brow, DevBuf<double>& ws, double alg_bytes,
                   double alg_flops);
void dense_block_add(svt_ctx* ctx, cudaStream_t s, int cls, i64 M, i64 N, int S, const DevBuf<double>& ws,
                     const int* orow, double* out, i64 ldo);

// Fused Cholesky-QR pass head for a narrow panel (w <= 16, single rank):
// G = X^T X reduced on the device, then Cholesky and Rinv = L^{-T} in the
// same launch; status[0] = 1 on an unsafe pivot.
void gram_chol(svt_ctx* ctx, const double* X, i64 ldx, i64 m, i64 w, double* G, double* Rinv, int* status,
               const int* pred);

// d_out[0] (op) sum of squares of X (rows x cols, ld).  op: 0 store, 1 add.
void sumsq(svt_ctx* ctx, const double* X, i64 rows, i64 cols, i64 ld, double* d_out, int op,
           const int* pred = nullptr);
// d_out[0] = max |X - I*diag_shift| over the rows x cols block (diag_shift 0 or 1)
void maxabs(svt_ctx* ctx, const double* X, i64 rows, i64 cols, i64 ld, double diag_shift, double* d_out);
// flag[0] = (sqrt(a[0]) > coef * sqrt(b[0]))  (sumsq inputs)  when mode 0
// flag[0] = (a[0] > coef)                                    when mode 1
void set_flag(svt_ctx* ctx, const double* a, const double* b, double coef, int mode, int* flag);

// Round-batch decisions on the device (no host synchronization): mode 0,
// flag = any block with sum(after_k) < thr2 * sum(before_k); mode 1, flag =
// *gate && any block with ||proj_k|| > 1e-8 ||after_k|| (sketch.hpp:134).
void block_flags(svt_ctx* ctx, const double* after, const double* before, const double* proj, int K, int w,
                 double thr2, int mode, const int* gate, int* flag);
// Single-CTA Cholesky of the w x w Gram G (w <= 64): Rinv = L^{-T} (upper,
// row-major, w x w).  status[0] = 1 when a pivot is not safely positive
// (triggers the Householder fallback).  Skipped when *pred == 0.
void chol_rinv(svt_ctx* ctx, const double* G, i64 w, double* Rinv, int* status, const int* pred);
// Householder QR fallback (Eigen convention, all columns kept), single CTA,
// w <= 64: Q (m x w, ldq) from X (m x w, ldx).  Runs only when
// (pred == null || *pred) && (status == null || *status).
void householder_qr(svt_ctx* ctx, const double* X, i64 m, i64 w, i64 ldx, double* Q, i64 ldq, double* work,
                    const int* pred, const int* status);

// Symmetric eigen-decomposition of the r x r Gram (row-major, overwritten):
// W (r x r row-major, column j = eigenvector j), lambda descending.
void sym_eig(svt_ctx* ctx, double* G, i64 r, double* W, double* lambda);

// column norms: out[j] = ||X[:, j]||^2 for j < cols
void col_sumsq(svt_ctx* ctx, const double* X, i64 rows, i64 cols, i64 ld, double* out);
// X[:, j] *= s[j]  (s on device)
void scale_cols(svt_ctx* ctx, double* X, i64 rows, i64 cols, i64 ld, const double* s);
// dst (rows x cols, ldd) <- src (rows x cols, lds), optionally predicated
void copy2d(svt_ctx* ctx, const double* src, i64 lds, double* dst, i64 ldd, i64 rows, i64 cols,
            const int* pred = nullptr);
void fill(svt_ctx* ctx, double* p, i64 n, double v);
// Z[:, 0:s] <- the first s columns of the identity (rows x s, ld)
void set_identity_cols(svt_ctx* ctx, double* Z, i64 rows, i64 ld, i64 s);
// out[i] = alpha * (GY[i] - c * Y[i]) - beta * Xp[i]  (Chebyshev filter step;
// Xp may be null when beta == 0; out may alias Xp)
void cheb_combine(svt_ctx* ctx, double* out, const double* GY, const double* Y, const double* Xp, i64 count,
                  double c, double alpha, double beta);
// Y[:, j] -= theta[j] * X[:, j]  (rows x cols, same ld)
void sub_scaled_cols(svt_ctx* ctx, double* Y, const double* X, i64 rows, i64 cols, i64 ld, const double* theta);
// out (cols x rows) = in^T ; in (rows x cols, ldi) ; out ld = rows
void transpose(svt_ctx* ctx, const double* in, i64 rows, i64 cols, i64 ldi, double* out);
// W2[:, j] = W[:, perm[j]] for j < kcols (perm on device, int)
void permute_cols(svt_ctx* ctx, const double* W, i64 rows, i64 ldw, const int* perm, i64 kcols, double* W2,
                  i64 ldw2);

}  // namespace svtb
