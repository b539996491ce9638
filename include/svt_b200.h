/*
 * svt_b200.h — the C-ABI boundary of the B200-native SVT / R3SVD / R4SVD hot
 * path (arXiv 1704.05528).  Plain pointers and sizes only; no torch, Eigen or
 * CUDA types cross this boundary.
 *
 * Every entry point replaces one function of the reference's header-only C++
 * API (`proj/include/svt/` headers, cited per function).  Dense host buffers use
 * the reference's Eigen::MatrixXd layout (column-major, leading dimension =
 * rows), so a reference-side binding passes `M.data()` straight through (see
 * INTEGRATION.md).  Errors are reported as return codes mapping one-to-one
 * onto the reference's exception types; the message is in svt_last_error().
 *
 * Multi-GPU: one process per GPU.  A distributed context owns a row block
 * [row_begin, row_end) of every sampled matrix; "local" row-indexed arrays
 * (U, X, Q) cover only that block, n-indexed arrays (V, Omega, B^T) are
 * replicated.  Collectives are NCCL all-reduces inside the library.
 */
#ifndef SVT_B200_H
#define SVT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define SVT_OK 0
#define SVT_EINVAL 1   /* std::invalid_argument (shapes, parameters)        */
#define SVT_EDOMAIN 2  /* std::domain_error (all-zero target)               */
#define SVT_ERUNTIME 3 /* std::runtime_error                                */
#define SVT_ECUDA 4    /* CUDA runtime / kernel failure                     */
#define SVT_ENCCL 5    /* NCCL failure                                      */
#define SVT_EOOM 6     /* device allocation failed                          */

/* ---- parameter / record structs (mirror the reference structs) --------- */

/* SketchParams, sketch.hpp:20-27 */
typedef struct svt_sketch_params {
    int64_t t;
    int64_t dt;
    int32_t np;
    int32_t reserved0;
    double eps_threshold;
    uint64_t seed;
    int64_t p;
} svt_sketch_params;

/* SvtConfig, solver.hpp:32-43, plus the two Appendix-B harness extensions
 * (0 = reference behaviour). */
typedef struct svt_config {
    double tau;
    double delta;
    int32_t maxit;
    int32_t np;
    int64_t dt;
    double eps_stop;
    double eps_threshold0;
    double beta;
    int64_t t0;
    uint64_t seed;
    double eps_threshold_min; /* cooling floor: eps <- max(eps*beta, min) */
    double rel_residual_stop; /* stop when ||P(X-A)||/||P A|| < this      */
} svt_config;

/* StopRule, solver.hpp:59-67 */
#define SVT_STOP_TRAIN_MAE 0
#define SVT_STOP_RESIDUAL 1
#define SVT_STOP_NONE 2
typedef struct svt_stop {
    int32_t kind;
    int32_t reserved0;
    double threshold;
} svt_stop;

/* Backend, solver.hpp:69-78 */
#define SVT_BACKEND_R4SVD 0
#define SVT_BACKEND_R3SVD 1
#define SVT_BACKEND_RSVD_FIXED 2
#define SVT_BACKEND_FULL_SVD 3
typedef struct svt_backend {
    int32_t kind;
    int32_t reserved0;
    int64_t fixed_rank;
} svt_backend;

/* IterationRecord, solver.hpp:49-57 (+ extension columns) */
typedef struct svt_record {
    int32_t iter;
    int32_t extension_rounds;
    int64_t rank;
    double residual;
    double eps_threshold;
    double train_mae;
    double sketch_ms;
    double total_ms;
    int64_t kept;          /* rank of the shrunk iterate X             */
    double rel_residual_x; /* ||P_Lambda(X - A)||_F / ||P_Lambda A||_F */
    double test_mae;       /* held-out MAE (0 without a test set)      */
    double test_rmse;      /* held-out RMSE (0 without a test set)     */
} svt_record;

/* IterationObserver, solver.hpp:88.  U is m_local x k, V is n x k
 * (column-major host copies valid during the call).  Return 0 to stop. */
typedef int (*svt_observer_fn)(const svt_record* rec, int64_t m_local, int64_t n, int64_t k,
                               const double* U, const double* sigma, const double* V, void* user);

/* ---- opaque handles ---------------------------------------------------- */
typedef struct svt_ctx svt_ctx;         /* device, stream, comm, workspaces */
typedef struct svt_mat svt_mat;         /* SampledMatrix on the device      */
typedef struct svt_factors svt_factors; /* SketchResult / LowRankFactors    */
typedef struct svt_solver svt_solver;   /* svt_run_backend state            */
typedef struct svt_result svt_result;   /* SvtResult                        */

/* ---- context ----------------------------------------------------------- */
const char* svt_last_error(void);
int svt_version(void);
int svt_ctx_create(int device, svt_ctx** out);
/* One rank of a world: nccl_id is the 128-byte ncclUniqueId of rank 0.
 * world = 1 with an id makes a one-rank communicator: the distributed code
 * path (row-blocked collectives, side communicator) on a single GPU. */
int svt_ctx_create_dist(int device, int rank, int world, const void* nccl_id, svt_ctx** out);
int svt_nccl_get_unique_id(void* out128);
/* Host-staged collectives instead of NCCL: every all-reduce of the library
 * (the n x w partials of Y^T X, the Gram blocks and the norms)
 * is copied to pinned host memory and handed to `fn`, which must sum the
 * `count` doubles element-wise across the `world` ranks in place (e.g.
 * torch.distributed over gloo) and return 0.  All ranks issue the same
 * sequence of calls (every branch is taken on all-reduced values).  Runs the
 * row-sharded path where NVLink / NCCL is not available: several ranks
 * sharing one GPU in tests, or host-coordinated clusters. */
typedef int (*svt_allreduce_fn)(double* buf, int64_t count, void* user);
int svt_ctx_create_hostcomm(int device, int rank, int world, svt_allreduce_fn fn, void* user, svt_ctx** out);
/* all-reduces issued by this context and the doubles they carried */
int svt_ctx_comm_stats(svt_ctx* ctx, int64_t* calls, double* doubles);
int svt_ctx_destroy(svt_ctx* ctx);
int svt_ctx_sync(svt_ctx* ctx);
/* make the context stream wait for all work issued on the library's side
 * stream (speculative batches); asynchronous */
int svt_ctx_join(svt_ctx* ctx);
void* svt_ctx_stream(svt_ctx* ctx); /* the cudaStream_t every kernel runs on */
int svt_ctx_rank(svt_ctx* ctx, int* rank, int* world);
/* instrumentation: per-kernel-class CUDA-event timing (0 = off) */
int svt_ctx_set_profiling(svt_ctx* ctx, int on);
/* speculative side-stream round batches (1 = on, the default).  Off, every
 * batch is sketched on the main stream after the previous one: the same
 * results (the batches are identical), kernels serialised — the bench's
 * per-kernel roofline pass uses it so launch durations are not inflated by
 * SM sharing with the other stream. */
int svt_ctx_set_speculation(svt_ctx* ctx, int on);
int svt_ctx_reset_stats(svt_ctx* ctx);
/* class: 0 SpMM, 1 SpMM^T, 2 SDDMM+update, 3 CGS/GEMM passes, 4 RNG, 5 QR, 6 finalize, 7 other */
int svt_ctx_kernel_stats(svt_ctx* ctx, int cls, int64_t* launches, double* total_ms, double* bytes,
                         double* flops);
int64_t svt_ctx_launch_count(svt_ctx* ctx);
/* host-side accounting: stream synchronizations the library issued and the
 * host time spent blocked in them (timed only while profiling is on) */
int svt_ctx_host_stats(svt_ctx* ctx, int64_t* syncs, double* sync_ms);
/* 1 (default): speculative multi-round batches in the rank-revealing loop
 * (same rounds / ranks; exact-arithmetic equivalent); 0: one round at a time. */
int svt_ctx_set_batching(svt_ctx* ctx, int on);

/* ---- host-side sample-set construction (SampledMatrix ctor, sampled.hpp:27-62) */
/* Validates and sorts triplets into CSR; throws-equivalent SVT_EINVAL on
 * out-of-range, duplicate or non-finite entries. */
int svt_sampled_build(int64_t m, int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                      const double* vals, int64_t* rowptr_out, int64_t* col_out, double* val_out);
/* nnz-balanced row partition for `world` ranks: bounds[world+1]. */
int svt_partition_rows(int64_t m, const int64_t* rowptr, int world, int64_t* bounds);

/* ---- device sample-set matrices --------------------------------------- */
/* rowptr has (row_end-row_begin+1) entries, offsets into col/val (rowptr[0]
 * is subtracted).  col is 0-based global column index. */
int svt_matrix_upload(svt_ctx* ctx, int64_t m, int64_t n, int64_t row_begin, int64_t row_end,
                      const int64_t* rowptr, const int64_t* col, const double* val, svt_mat** out);
/* SampledMatrix(rows, cols, values) (sampled.hpp:27-62) built on the device:
 * unsorted triplets are uploaded, validated (range, finiteness, duplicates;
 * SVT_EINVAL with the reference's messages), radix-sorted by (row, col), and
 * the rows [row_begin, row_end) kept as this rank's block. */
int svt_matrix_from_triplets(svt_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                             const int64_t* cols, const double* vals, int64_t row_begin, int64_t row_end,
                             svt_mat** out);
/* The rank's local CSR back on the host: rowptr (m_local + 1, rebased),
 * col (nnz_local, global column index), val (nnz_local). */
int svt_matrix_csr(svt_mat* mat, int64_t* rowptr, int64_t* col, double* val);
int svt_matrix_free(svt_mat* mat);
int svt_matrix_info(svt_mat* mat, int64_t* m, int64_t* n, int64_t* nnz_local, int64_t* row_begin,
                    int64_t* row_end);
int svt_matrix_set_values(svt_mat* mat, const double* vals);
int svt_matrix_get_values(svt_mat* mat, double* vals);
/* The dense-corner split of the sample pattern used by the wide products
 * (no reference counterpart: a B200 layout of sampled.hpp:113-144's
 * operand).  Builds it if not tried yet (SVTB_HYBRID=0 disables), then
 * reports: on (1 when the cost model kept a block), block rows R / columns C,
 * entries inside the block and outside it. */
int svt_matrix_hybrid_info(svt_mat* mat, int* on, int64_t* rows, int64_t* cols, int64_t* nnz_block,
                           int64_t* nnz_cold);

/* ---- formats (io.hpp): readers / writers either side of the path ------ */
/* Host triplet set: 0-based (row, col, value) in an m x n frame; a ratings
 * file also carries the original user / item ids of the dense indices. */
typedef struct svt_triplets svt_triplets;
int svt_read_matrix_market(const char* path, svt_triplets** out);              /* io.hpp:118-173 */
int svt_read_ratings(const char* path, const char* separator, svt_triplets** out); /* io.hpp:383-470 */
int svt_sample_image(int64_t width, int64_t height, const uint8_t* pixels, double fraction, uint64_t seed,
                     svt_triplets** out);                                         /* io.hpp:329-350 */
int svt_split_ratings(svt_triplets* ds, double train_fraction, uint64_t seed, svt_triplets** train,
                      svt_triplets** test);                                       /* io.hpp:474-497 */
/* a triplet set from host arrays (no validation; SampledMatrix construction validates) */
int svt_triplets_create(int64_t m, int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                        const double* vals, svt_triplets** out);
int svt_triplets_info(svt_triplets* t, int64_t* m, int64_t* n, int64_t* nnz);
int svt_triplets_copy(svt_triplets* t, int64_t* rows, int64_t* cols, double* vals);
/* ratings only: user_ids (m entries), item_ids (n entries); provenance line */
int svt_triplets_ids(svt_triplets* t, int64_t* user_ids, int64_t* item_ids);
const char* svt_triplets_provenance(svt_triplets* t);
int svt_triplets_free(svt_triplets* t);
/* device SampledMatrix of a triplet set (svt_matrix_from_triplets semantics) */
int svt_matrix_from_triplet_set(svt_ctx* ctx, svt_triplets* t, int64_t row_begin, int64_t row_end, svt_mat** out);
/* coordinate writer of a host CSR (1-based, %.17g: exact round trip), io.hpp:176-193 */
int svt_write_matrix_market(const char* path, int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col,
                            const double* val);
/* dense `array real general`, column-major; data == NULL queries the shape */
int svt_read_matrix_market_array(const char* path, int64_t* rows, int64_t* cols, double* data); /* io.hpp:196-231 */
int svt_write_matrix_market_array(const char* path, int64_t rows, int64_t cols, const double* data); /* :233-246 */
/* PGM (P5 / P2, maxval 255); pixels row-major; pixels == NULL queries the shape */
int svt_read_pgm(const char* path, int64_t* width, int64_t* height, uint8_t* pixels); /* io.hpp:272-313 */
int svt_write_pgm(const char* path, int64_t width, int64_t height, const uint8_t* pixels); /* io.hpp:316-327 */
/* round + clamp a column-major rows x cols reconstruction into 8-bit pixels (row-major) */
int svt_quantize_image(int64_t rows, int64_t cols, const double* X, uint8_t* pixels); /* io.hpp:367-381 */

/* trace export, schema "svt-trace v1": json = 0 -> write_trace_csv, 1 ->
 * write_trace_json (solver.hpp:346-386) */
int svt_write_trace(const svt_record* records, int64_t count, const char* path, int json);

/* ---- primitives (host in/out; dense.hpp / sampled.hpp) ---------------- */
int svt_gaussian_block(svt_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, double* out); /* dense.hpp:86 */
int svt_qr_orthonormal(svt_ctx* ctx, int64_t rows, int64_t cols, const double* X, double* Q); /* dense.hpp:103 */
int svt_small_svd(svt_ctx* ctx, int64_t rows, int64_t cols, const double* B, double* U, double* sigma,
                  double* V); /* dense.hpp:114; U rows x k, V cols x k, k = min */
int svt_sp_mult(svt_mat* S, int64_t w, const double* X, double* out);   /* sampled.hpp:113 */
int svt_sp_mult_t(svt_mat* S, int64_t w, const double* X, double* out); /* sampled.hpp:130 */
int svt_project_low_rank(svt_mat* pattern, int64_t k, const double* U, const double* sigma, const double* V,
                         double* out_vals); /* sampled.hpp:148 */
int svt_sp_axpy(svt_mat* Y, double alpha, const double* d_vals, double* out_vals); /* sampled.hpp:166 */
int svt_sp_frob_norm_sq(svt_mat* S, double* out);                                 /* sampled.hpp:178 */
int svt_spectral_norm_est(svt_mat* S, int iters, uint64_t seed, double* out);     /* sampled.hpp:188 */
int svt_kickstart(svt_mat* A, double tau, double delta, uint64_t seed, double* out_vals); /* solver.hpp:125 */

/* Device-pointer FP64 contraction on the context stream, row-major:
 * C (M x N) = alpha * op(A) * B + beta * C, op(A) = A^T (A stored K x M) when
 * transA, else A (M x K).  The kernel family behind every dense product of
 * the sketch (block Gram-Schmidt Q^T X / X - Q C, CholQR Grams, B = Q^T Y
 * updates; sketch.hpp:133-141, dense.hpp:103-110); exposed for tuning and
 * its own parity tests.  Asynchronous. */
int svt_dev_gemm(svt_ctx* ctx, int transA, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                 int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc);

/* Device-pointer symmetric eigensolve on the context stream: G (r x r,
 * row-major, symmetric) = W diag(lambda) W^T, lambda descending, W row-major
 * with the eigenvectors as columns -- the dense step of sketch.hpp:158-162
 * (SVD of B through its Gram), exposed for its own parity tests.  G is not
 * modified.  Synchronous. */
int svt_dev_sym_eig(svt_ctx* ctx, const double* G, int64_t r, double* W, double* lambda);
/* C (M x N, row-major, ld ldc) = A^T B for row-major FP64 device operands A
 * (K x M, ld lda) and B (K x N, ld ldb), computed on the INT8 tensor cores
 * by the Ozaki digit-splitting scheme (slices = int8 digits per entry, 6..8;
 * 8 carries the FP64 GEMM error bound).  The FP64 contraction of the
 * Gram-Schmidt step (sketch.hpp:133-141, Q^T X) in this form. */
/* Process-wide device allocation counters: cudaMalloc calls, cudaFree calls
 * and host milliseconds spent in them (instrumentation). */
int svt_alloc_stats(int64_t* mallocs, int64_t* frees, double* ms);
int svt_dev_gemm_tn_ozaki(svt_ctx* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                          const double* B, int64_t ldb, double* C, int64_t ldc, int slices);

/* Device-pointer sparse products on the context stream (row-major panels):
 * out (m_local x w) = S * X (X: n x w) or, transpose != 0, out (n x w) = S^T * X
 * (X: m_local x w, out packed, all-reduced across ranks) -- sampled.hpp:113 /
 * :130 without the host copies.  Asynchronous. */
int svt_dev_sp_mult(svt_mat* S, int transpose, int64_t w, const double* X, int64_t ldx, double* out,
                    int64_t ldo);
/* Device-pointer fused SDDMM + Bregman update on A's pattern, the SVT loop's
 * last step (solver.hpp:321-323 with project_low_rank / sp_axpy,
 * sampled.hpp:148-176): with P = U Vs^T on Lambda (U: m_local x k, Vs = V
 * diag(sigma - tau): n x k, row-major), d = A - P and Y_csr += delta * d
 * (y_csr: nnz_local values in CSR order, updated in place); y_csc (nullable)
 * receives the CSC-ordered mirror.  sums4 (host, nullable) <- {sum |d|,
 * sum d^2, sum (A - Y_old)^2, sum Y_new^2} (all-reduced).  Asynchronous
 * unless sums4 is given. */
int svt_dev_sddmm_update(svt_mat* A, int64_t k, const double* U, int64_t ldu, const double* Vs, int64_t ldv,
                         double delta, double* y_csr, double* y_csc, double* sums4);

/* ---- sketch engines (sketch.hpp) -------------------------------------- */
int svt_rsvd(svt_mat* Y, int64_t k, const svt_sketch_params* p, svt_factors** out);  /* sketch.hpp:165 */
int svt_r3svd(svt_mat* Y, const svt_sketch_params* p, svt_factors** out);            /* sketch.hpp:188 */
int svt_r4svd(svt_mat* Y, int64_t s, const double* U_prev, int64_t ldu, const svt_sketch_params* p,
              svt_factors** out); /* sketch.hpp:207 */
int svt_factors_info(svt_factors* f, int64_t* m_local, int64_t* n, int64_t* rank, int* saturated,
                     int* extension_rounds);
int svt_factors_copy(svt_factors* f, double* U, double* sigma, double* V);
int svt_factors_free(svt_factors* f);

/* ---- solver (solver.hpp:215-340) -------------------------------------- */
int svt_default_config(svt_mat* A, svt_config* out); /* solver.hpp:95 */
int svt_solver_create(svt_mat* A, const svt_config* cfg, svt_stop stop, svt_backend backend, svt_mat* test,
                      svt_solver** out);
/* one Bregman iteration; *done = 1 when the run stopped (stop rule/observer
 * or maxit) — then svt_solver_result() is final. */
int svt_solver_step(svt_solver* s, svt_observer_fn obs, void* user, svt_record* rec, int* done);
int svt_solver_result(svt_solver* s, svt_result** out);
int svt_solver_free(svt_solver* s);
int svt_run(svt_mat* A, const svt_config* cfg, svt_stop stop, svt_backend backend, svt_mat* test,
            svt_observer_fn obs, void* user, svt_result** out); /* solver.hpp:215 / 333 / 340 */
int svt_result_info(svt_result* r, int64_t* n_records, int64_t* m_local, int64_t* n, int64_t* k, int* converged);
int svt_result_trace(svt_result* r, svt_record* out);
int svt_result_factors(svt_result* r, double* U, double* sigma, double* V);
int svt_result_free(svt_result* r);

/* ---- checkpoint / resume ------------------------------------------------
 * The reference has no solver checkpoint (the manifest re-runs
 * from scratch).  The state below is everything svt_run_backend carries
 * from one iteration to the next (solver.hpp:221-238, 280-284, 299-303,
 * 321-324), so resuming at iteration i reproduces iterations i+1.. of the
 * uninterrupted run bit for bit (same seeds, thresholds, recycled basis).
 * Host buffers: y_vals = the iterate Y on this rank's pattern (nnz_local,
 * CSR order); u_prev = U_prev (m_local x s, column-major); best_U / best_V
 * column-major (m_local x best_k, n x best_k), best_sigma (best_k).  In
 * svt_solver_checkpoint any buffer may be NULL (query the sizes first). */
typedef struct svt_solver_state {
    int32_t iter;        /* iterations completed                              */
    int32_t done;        /* the run already stopped                            */
    int32_t converged;
    int32_t last_rounds; /* previous sketch's round count (batch-size hint)    */
    int64_t s;           /* recycled basis width                               */
    int64_t best_k;      /* rank of the best-so-far factors                    */
    double eps_threshold;
    double eps_min;      /* running minimum of the dual residual (cooling)     */
    double best_metric;
    double frob_y_sq;    /* ||Y||_F^2 of the current iterate (all ranks)       */
    double frob_a;       /* ||P_Lambda A||_F                                   */
} svt_solver_state;
int svt_solver_checkpoint(svt_solver* s, svt_solver_state* st, double* y_vals, double* u_prev, double* best_U,
                          double* best_sigma, double* best_V);
int svt_solver_resume(svt_mat* A, const svt_config* cfg, svt_stop stop, svt_backend backend, svt_mat* test,
                      const svt_solver_state* st, const double* y_vals, const double* u_prev, const double* best_U,
                      const double* best_sigma, const double* best_V, svt_solver** out);

/* ---- synthetic inputs for the five BASELINE configs (host) ------------- */
/* Generates the observed (train) triplets and, for configs 3/4, the held-out
 * test triplets.  Two-phase: call with NULL buffers to get sizes. */
int svt_synth_config(int config, uint64_t seed, int64_t* m, int64_t* n, int64_t* nnz_train, int64_t* nnz_test,
                     int64_t* train_rows, int64_t* train_cols, double* train_vals, int64_t* test_rows,
                     int64_t* test_cols, double* test_vals);
/* CSR directly (configs too large for triplets, e.g. config 5): rowptr m+1. */
int svt_synth_config_csr(int config, uint64_t seed, int64_t* m, int64_t* n, int64_t* nnz, int64_t* rowptr,
                         int64_t* col, double* val);

/* ---- the reference's experiment generators (proj/include/svt/synth.hpp) --
 * Host-side, seeded; the inputs of the CLI's --synthetic / bench modes. */
uint64_t svt_derive_seed(uint64_t seed, uint64_t stream);                                /* dense.hpp:44 */
int svt_make_low_rank(int64_t m, int64_t n, int64_t rank, uint64_t seed, double* out);   /* synth.hpp:21-28; out m x n column-major */
int svt_sample_dense(int64_t m, int64_t n, const double* A, double fraction, uint64_t seed,
                     svt_triplets** out);                                                /* synth.hpp:64-84 */
int svt_synthetic_image(int64_t size, int64_t rank, uint64_t seed, uint8_t* pixels);     /* synth.hpp:89-114; size*size row-major */
int svt_synthetic_ratings(int64_t users, int64_t items, int64_t rank, double fill, double noise, uint64_t seed,
                          svt_triplets** out);                                           /* synth.hpp:119-160 */
/* default_config (solver.hpp:95-106) from the CSR-ordered values on the host. */
int svt_default_config_host(int64_t m, int64_t n, int64_t nnz, const double* csr_vals, svt_config* out);

#ifdef __cplusplus
}
#endif

#endif /* SVT_B200_H */
