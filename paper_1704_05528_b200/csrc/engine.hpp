// The B200 engine behind the C ABI: device sample sets, the QB state, the
// R3SVD / R4SVD rank-revealing loops (host control, device data) and the SVT
// Bregman iteration (solver.hpp:215-328).
#pragma once

#include <limits>
#include <memory>
#include <vector>

#include "../../include/svt_b200.h"
#include "common.hpp"

// Segment plan storage behind svtb::SegPlanView.
struct SegPlan {
    svtb::DevBuf<int> seg_row, seg_slot, long_row, long_first, long_count;
    svtb::DevBuf<long long> seg_beg, seg_end;
    svtb::DevBuf<int> grp_first;
    svtb::DevBuf<long long> chunk_off;
    svtb::SegPlanView v;
};

// Tiled view storage behind svtb::TilePlanView (built lazily, on the first
// wide product).  `src` is the CSR value array the entries currently mirror.
struct TilePlan {
    svtb::DevBuf<long long> tile_e, tile_u;
    svtb::DevBuf<int> ucol, perm, item_t0, item_t1, item_blk, item_part, split_blk, split_first, split_count;
    svtb::DevBuf<unsigned short> roff;
    svtb::DevBuf<svtb::TileEnt> ent;
    svtb::TilePlanView v;
    const double* src = nullptr;
    bool built = false;
};

// Dense-corner split of a power-law sample pattern for the wide products
// (build.cu builds it, engine.cpp uses it).  Power-law users and Zipf items
// concentrate a large share of the entries in the block of the R
// highest-degree local rows x the C highest-degree columns (config 4:
// 4096 x 2048 holds 37 % of the entries at 40 % density).  That block is held
// DENSE (R x C, row-major) and multiplied on the FP64 tensor cores; the other
// ("cold") entries keep the gather kernels through their own CSR / CSC views
// and segment plans.  Y's values are mirrored into the cold arrays and the
// block once per sketch (`src` = the CSR value array mirrored).
struct HybridPlan {
    bool tried = false, on = false;
    svtb::i64 R = 0, C = 0, nnz_cold = 0, nnz_blk = 0;
    svtb::DevBuf<int> hot_rows, hot_cols;  // block row r -> local row, block column c -> column
    svtb::DevBuf<int> blk_map, blk_pos;    // block entries: CSR position, r * C + c
    svtb::DevBuf<svtb::i64> rowptr_c, colptr_c;
    svtb::DevBuf<int> col_c, row_c;        // cold CSR columns / cold CSC local rows
    svtb::DevBuf<int> map_c, mapt_c;       // their CSR positions (value source)
    svtb::DevBuf<double> val_c, valt_c, D;
    SegPlan plan_c, plant_c;
    const double* src = nullptr;
    long long src_version = -1;  // the matrix's own values: their version when mirrored
    svtb::DevBuf<double> ws[2];  // split-K partials of the block product (main / side stream)
};

// Device SampledMatrix (sampled.hpp:25-110): this rank's row block as CSR
// (int64 rowptr, int32 col, fp64 val) plus a CSC view whose value array
// mirrors the CSR values through csr2csc.
struct svt_mat {
    SegPlan plan_csr, plan_csc;
    TilePlan tile_csr, tile_csc;  // shared-memory-tiled views for wide panels
    HybridPlan hyb;               // dense-corner split (wide panels, power-law patterns)
    svt_ctx* ctx = nullptr;
    svtb::i64 m = 0, n = 0, row_begin = 0, row_end = 0, m_local = 0, nnz_local = 0, nnz_global = 0;
    svtb::DevBuf<svtb::i64> rowptr;
    svtb::DevBuf<int> col;
    svtb::DevBuf<double> val;
    svtb::DevBuf<svtb::i64> colptr;
    svtb::DevBuf<int> cscrow;
    svtb::DevBuf<double> val_csc;
    svtb::DevBuf<int> csr2csc;
    svtb::DevBuf<int> csc2csr;  // inverse permutation (CSC position -> CSR entry)
    long long val_version = 0;  // bumped whenever val is rewritten (svt_matrix_set_values)
};

namespace svtb {

// A value array on a matrix's pattern (CSR order + CSC mirror).
struct Vals {
    double* csr;
    double* csc;
};

// Device factors U (m_local x k), sigma (k), V (n x k), row-major.
struct DevFactors {
    i64 m_local = 0, n = 0, k = 0;
    DevBuf<double> U, V;
    std::vector<double> sigma;
    DevBuf<double> d_sigma;
};

// QBState (sketch.hpp:32-39) with capacity-preallocated Q (m_local x cap) and
// B^T (n x cap), both row-major with ld = cap; appending a block is a
// pointer offset (no conservativeResize copy, sketch.hpp:145-152).
struct QBDev {
    i64 m_local = 0, n = 0, min_dim = 0, cap = 0, rank = 0;
    DevBuf<double> Q, Bt;
    // INT8 digit slices of Q's leading columns for the Gram-Schmidt product
    // Q^T X on the tensor cores (ozaki.cu): valid for columns [0, qs_valid)
    // of this sketch; extended lazily, reset with the basis
    DevBuf<double> qs;  // raw int8 tiles
    DevBuf<int> qe;     // per-column exponents
    i64 qs_tiles = 0, qs_valid = 0;
    double norm_b_sq = 0.0;
    double frob_y_sq = 0.0;
    bool saturated = false;
};

enum class FinalizeMode { Full, Kept };

struct SketchOut {
    DevFactors f;
    i64 rank = 0;
    bool saturated = false;
    int rounds = 0;
};

// widest speculative round batch (the 128-column Cholesky panel)
constexpr i64 kMaxBatchW = 128;

// Per-context reusable workspaces of the sketch engines.
struct Engine {
    svt_ctx* ctx;
    svt_mat* mat;  // pattern of the target
    Vals Y;
    DevBuf<double> Om, OmBank, X, X2, P, T, C, D, G, Rinv, hh, tmp, W, lam, Vraw, Wk;
    DevBuf<double> fkZ, fkZq, fkZt, fkWn, fkH, fkYh, fkth, fkZY, fkXr, fkres;  // finalize_kept
    DevBuf<double> TW, CW, GW, RW, eW;  // round batches (the sketch panels live in spec)
    // Speculative sketch of the next round batch (Omega + the power-iteration
    // products, which do not depend on the basis) computed on ctx->side while
    // the current batch's Gram-Schmidt / QR run on the main stream.  Two
    // buffer slots alternate between the batch in flight and the next one.
    struct SpecSketch {
        DevBuf<double> om[2], x[2], t[2];
        DevBuf<double> part;  // long-row partials of the side-stream SpMMs
        bool valid = false;   // a speculative batch is in flight / ready
        u64 seed = 0;
        u64 gen = 0;          // sketch generation it belongs to
        int round0 = 0, K = 0, slot = 0;
        cudaEvent_t ready = nullptr, freed[2] = {nullptr, nullptr};
    } spec;
    DevBuf<int> perm;
    QBDev qb;  // persistent QB storage: capacity survives across SVT iterations
    bool batching = true;  // speculative multi-round batches (exact-arithmetic equivalent)
    int last_rounds = -1;  // rounds of the previous sketch (batch-size predictor)
    u64 sketch_gen = 0;    // incremented per sketch: a speculative batch never outlives its sketch
    DevFactors fpool;          // factor buffers handed back by the solver for the next sketch
    bool tiled = false;        // shared-memory-tiled SpMM for wide panels (opt-in, per sketch)
    bool tiles_fresh = false;  // the tiled views mirror Y (cleared at every sketch entry)
    bool hyb_fresh = false;    // the dense-corner split mirrors Y (cleared at every sketch entry)
    Engine(svt_ctx* c, svt_mat* m, Vals y) : ctx(c), mat(m), Y(y), batching(c->batching != 0) {}
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    Engine(Engine&&) = delete;
    ~Engine() {
        if (spec.ready) {
            if (ctx && ctx->side) cudaStreamSynchronize(ctx->side);
            cudaEventDestroy(spec.ready);
            cudaEventDestroy(spec.freed[0]);
            cudaEventDestroy(spec.freed[1]);
        }
    }
};

// primitives
double frob_sq(Engine& E);  // ||Y||_F^2 (all ranks)
// Y X (local rows) / Y^T X (n x w, ld w, all-reduced); stream / scratch:
// optional launch on another stream with its own long-row partial buffer
void sp_mult(Engine& E, i64 w, const double* X, i64 ldx, double* out, i64 ldo, cudaStream_t stream = nullptr,
             DevBuf<double>* scratch = nullptr);
void sp_mult_t(Engine& E, i64 w, const double* X, i64 ldx, double* out, cudaStream_t stream = nullptr,
               DevBuf<double>* scratch = nullptr, i64 ldo = -1);  // ldo != w: single rank only
void qr_orthonormal(Engine& E, double* X, i64 ldx, i64 w, double* Qout, i64 ldq);            // dense.hpp:103
void qr_orthonormal(Engine& E, i64 rows, bool dist, double* X, i64 ldx, i64 w, double* Qout, i64 ldq);
double spectral_norm_est(Engine& E, int iters, u64 seed);
// mark the tiled views stale and re-gather them from E.Y (sketch entry)
void prepare_tiles(Engine& E);                                   // sampled.hpp:188

// sketch.hpp
void qb_init(Engine& E, QBDev& st, i64 t, int np, u64 seed, double frob_y_sq = -1.0);
void qb_extend(Engine& E, QBDev& st, i64 dt, int np, u64 seed, const double* omega = nullptr);
void finalize(Engine& E, const QBDev& st, FinalizeMode mode, double tau, DevFactors& out);
SketchOut r3svd(Engine& E, const svt_sketch_params& p, FinalizeMode mode, double tau, double frob_y_sq = -1.0);
SketchOut r4svd(Engine& E, const double* U_prev, i64 ldu, i64 s, const svt_sketch_params& p, FinalizeMode mode,
                double tau, double frob_y_sq = -1.0);
DevFactors rsvd(Engine& E, i64 k, const svt_sketch_params& p);
DevFactors full_svd(Engine& E);

u64 derive_seed_u(u64 seed, u64 stream);

// host.cpp: the segment groups of a plan (from its host-side segment bounds)
void build_groups(const std::vector<long long>& beg, const std::vector<long long>& end, cudaStream_t s, SegPlan& P);
// build.cu: device-side CSC view / csr2csc / segment plans of an uploaded CSR
void build_plan_device(svt_ctx* ctx, const long long* ptr, i64 rows, SegPlan& P);
int build_sampled_device(svt_ctx* ctx, svt_mat* M, const long long* col64);
// build.cu: the shared-memory-tiled view of a CSR-like pattern (map: source
// position -> CSR position of its value, or null for the identity)
void build_tile_plan(svt_ctx* ctx, const long long* ptr, const int* idx, i64 rows, i64 nnz, const int* map,
                     TilePlan& P);
void ensure_tile_plans(svt_ctx* ctx, svt_mat* M);
// build.cu: the dense-corner split of M (once; M->hyb.on says whether the
// cost model found a block worth splitting off), and the per-sketch value
// mirror from a CSR value array
void ensure_hybrid(svt_ctx* ctx, svt_mat* M);
void hybrid_refresh(svt_ctx* ctx, svt_mat* M, const double* Ycsr);
void build_from_triplets_device(svt_ctx* ctx, svt_mat* M, i64 nnz, const i64* rows, const i64* cols,
                                const double* vals);

}  // namespace svtb

struct svt_factors {
    svtb::DevFactors f;
    svtb::i64 rank = 0;
    int saturated = 0;
    int rounds = 0;
};

struct svt_result {
    std::vector<svt_record> trace;
    svtb::i64 m_local = 0, n = 0, k = 0;
    std::vector<double> U, sigma, V;  // column-major host copies
    int converged = 0;
};

struct svt_solver {
    svt_ctx* ctx = nullptr;
    svt_mat* A = nullptr;
    svt_mat* test = nullptr;
    svt_config cfg{};
    svt_stop stop{};
    svt_backend backend{};
    svtb::DevBuf<double> Ycsr, Ycsc;
    svtb::DevFactors X;          // current shrunk factors (U, sigma - tau, V)
    svtb::DevFactors best;       // best-so-far
    svtb::DevBuf<double> U_prev;  // recycled basis (m_local x s)
    svtb::i64 s = 0;
    svtb::DevBuf<double> Vs;  // V diag(sigma - tau)
    double eps_threshold = 0.0;
    double eps_min = std::numeric_limits<double>::infinity();
    double best_metric = std::numeric_limits<double>::infinity();
    double frob_a = 0.0;
    double frob_y_sq = -1.0;
    double t_start_ms = 0.0;
    int iter = 0;
    bool done = false;
    bool converged = false;
    bool result_is_current = false;
    int resume_last_rounds = -1;  // batch-size hint carried over by a resume
    std::vector<svt_record> trace;
    std::unique_ptr<svtb::Engine> engine;
};
