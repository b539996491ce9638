// Tall row-major FP64 products C = alpha A B + beta C (M >> N: the block
// Gram-Schmidt update X - Q C and the CholQR products X R^-1) through a CUTLASS
// 2.x device-GEMM template instantiated here (the vendored CuTe/CUTLASS header
// tree; compiled into this library for sm_100a).  Configuration: 64 x 128
// threadblock tiles with 32 x 64 warp tiles and a 3-stage multistage
// mainloop for the batch panels (N > 64), 64 x 64 / 32 x 32 / 4 stages below;
// DMMA 8x8x4 (SASS DMMA.8x8x4 — the FP64 tensor path of sm_100a), 8-byte
// operand alignment (any leading dimension / column offset).  No split-K: the result
// is deterministic.  Measured against our hand-written 64 x 128 kernel on the
// config-4 / config-5 Gram-Schmidt shapes in profiles/r02c_gemm_bench*.txt.
#include <cutlass/gemm/device/gemm.h>
#include <cutlass/gemm/device/gemm_splitk_parallel.h>
#include <cutlass/gemm/device/gemm_universal.h>

#include "common.hpp"
#include "kernels.hpp"

namespace svtb {

namespace {

// SW: threadblock swizzle width (2: the two 64-column tiles of one 64-row
// block run next to each other, so the A tile is read from HBM once)
template <int TM, int TN, int WM, int WN, int STG, int AL, int SW = 1>
using GemmNNT = cutlass::gemm::device::Gemm<
    double, cutlass::layout::RowMajor, double, cutlass::layout::RowMajor, double, cutlass::layout::RowMajor, double,
    cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80, cutlass::gemm::GemmShape<TM, TN, 16>,
    cutlass::gemm::GemmShape<WM, WN, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
    cutlass::epilogue::thread::LinearCombination<double, 1, double, double>,
    cutlass::gemm::threadblock::GemmIdentityThreadblockSwizzle<SW>, STG, AL, AL>;

template <typename G>
bool run(svt_ctx* ctx, cudaStream_t s, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda, const double* B,
         i64 ldb, double beta, double* C, i64 ldc) {
    G op;
    typename G::Arguments args({static_cast<int>(M), static_cast<int>(N), static_cast<int>(K)},
                               {A, static_cast<int>(lda)}, {B, static_cast<int>(ldb)}, {C, static_cast<int>(ldc)},
                               {C, static_cast<int>(ldc)}, {alpha, beta});
    if (op.can_implement(args) != cutlass::Status::kSuccess) return false;
    const cutlass::Status st = op(args, nullptr, s ? s : ctx->stream);
    if (st != cutlass::Status::kSuccess) throw cuda_error("CUTLASS DGEMM launch failed");
    return true;
}

// SVTB_CUTLASS_CFG (tuning A/B; 8-byte operand alignment throughout — the
// FP64 tensor-op iterators take no wider access for row-major operands):
// 1 = 64x32 (warp 32x16, 4 stages), 2 = default: 64x128 (warp 32x64, 3
// stages) for N > 64, 64x64 (warp 32x32, 4 stages) below (config-4 X - QC
// 737 -> 716 us, config-5 X - QC 16.1 -> 14.6 ms = 97 % of the measured
// DGEMM peak), 6 = 64x64 with a 2-wide tile swizzle,
// 3 = 128x64 (warp 64x32, 3 stages), 4 = 128x32 (warp 64x16), 5 = 64x32 with 5 stages
int cfg() {
    static const int v = [] {
        const char* e = std::getenv("SVTB_CUTLASS_CFG");
        return e ? std::atoi(e) : 2;
    }();
    return v;
}

// C = alpha A^T B + beta C with A stored K x M row-major (column-major M x K):
// the Gram-Schmidt coefficients B T and Q^T X, finalize's B W.  Split-K
// "parallel": each K slice writes its partial tile to a workspace and a
// reduction kernel adds the slices in order (deterministic) and applies
// alpha / beta.
using GemmTNSplit = cutlass::gemm::device::GemmSplitKParallel<
    double, cutlass::layout::ColumnMajor, double, cutlass::layout::RowMajor, double, cutlass::layout::RowMajor, double,
    cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80, cutlass::gemm::GemmShape<64, 64, 16>,
    cutlass::gemm::GemmShape<32, 32, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
    cutlass::epilogue::thread::LinearCombination<double, 1, double, double>,
    cutlass::epilogue::thread::Convert<double, 1, double>, cutlass::reduction::thread::ReduceAdd<double, double, 1>,
    cutlass::gemm::threadblock::GemmSplitKHorizontalThreadblockSwizzle, 4, 1, 1>;

// The dense corner of a split SpMM (engine.cpp): op(D) B[brow, :] with the
// panel rows gathered by the operand iterator (GatherB), K split in
// "parallel" mode into [S][M][N] partial tiles that the caller's fixed-order
// scatter-add reduces into the output rows.
template <typename LayoutA>
using GemmCorner = cutlass::gemm::device::GemmUniversal<
    double, LayoutA, double, cutlass::layout::RowMajor, double, cutlass::layout::RowMajor, double,
    cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80, cutlass::gemm::GemmShape<64, 64, 16>,
    cutlass::gemm::GemmShape<32, 32, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
    cutlass::epilogue::thread::LinearCombination<double, 1, double, double>,
    cutlass::gemm::threadblock::GemmIdentityThreadblockSwizzle<>, 4, 1, 1, cutlass::arch::OpMultiplyAdd,
    cutlass::ComplexTransform::kNone, cutlass::ComplexTransform::kNone, false, true, false>;

template <typename G>
int corner(svt_ctx* ctx, cudaStream_t s, i64 M, i64 N, i64 K, const double* D, i64 ldd, const double* B, i64 ldb,
           const int* brow, DevBuf<double>& ws) {
    const i64 tiles = ((M + 63) / 64) * ((N + 63) / 64);
    i64 S = std::max<i64>(1, std::min<i64>((3 * ctx->num_sms) / tiles, K / 256));
    S = std::max<i64>(1, std::min<i64>(S, static_cast<i64>(ws.n / static_cast<size_t>(M * N))));
    if (static_cast<size_t>(M * N) > ws.n) return 0;
    // every slice exactly K / S deep (a multiple of 16), so CUTLASS launches
    // exactly S slices and every partial tile the reduction reads is written
    while (S > 1 && K % (16 * S) != 0) --S;
    typename G::Arguments args(cutlass::gemm::GemmUniversalMode::kGemmSplitKParallel,
                               {static_cast<int>(M), static_cast<int>(N), static_cast<int>(K)}, static_cast<int>(S),
                               {1.0, 0.0}, D, B, ws.get(), ws.get(), 0, 0, 0, M * N, ldd, ldb, N, N, nullptr, brow,
                               nullptr);
    G op;
    if (op.can_implement(args) != cutlass::Status::kSuccess) return 0;
    if (G::get_workspace_size(args) != 0) return 0;
    const cutlass::Status st = op(args, nullptr, s);
    if (st != cutlass::Status::kSuccess) throw cuda_error("CUTLASS dense-corner launch failed");
    return static_cast<int>(S);
}

}  // namespace

int cutlass_dense_block(svt_ctx* ctx, cudaStream_t s, bool transA, i64 M, i64 N, i64 K, const double* D, i64 ldd,
                        const double* B, i64 ldb, const int* brow, DevBuf<double>& ws) {
    const i64 lim = (1LL << 31) - 1;
    if (M > lim || N > lim || K > lim || ldd > lim || ldb > lim) return 0;
    if (transA)
        return corner<GemmCorner<cutlass::layout::ColumnMajor>>(ctx, s, M, N, K, D, ldd, B, ldb, brow, ws);
    return corner<GemmCorner<cutlass::layout::RowMajor>>(ctx, s, M, N, K, D, ldd, B, ldb, brow, ws);
}

bool cutlass_gemm_tn(svt_ctx* ctx, cudaStream_t s, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
                     const double* B, i64 ldb, double beta, double* C, i64 ldc, DevBuf<double>& ws) {
    const i64 lim = (1LL << 31) - 1;
    if (M > lim || N > lim || K > lim || lda > lim || ldb > lim || ldc > lim) return false;
    // K slices: about two waves of 64 x 64 tiles (three resident per SM), at
    // least 256 of K per slice, partials within the workspace
    const i64 tiles = ((M + 63) / 64) * ((N + 63) / 64);
    i64 splits = std::max<i64>(1, std::min<i64>((6 * ctx->num_sms + tiles - 1) / tiles, K / 256));
    splits = std::max<i64>(1, std::min<i64>(splits, static_cast<i64>(ws.n / static_cast<size_t>(M * N))));
    GemmTNSplit op;
    GemmTNSplit::Arguments args({static_cast<int>(M), static_cast<int>(N), static_cast<int>(K)},
                                {A, static_cast<int>(lda)}, {B, static_cast<int>(ldb)}, {C, static_cast<int>(ldc)},
                                {C, static_cast<int>(ldc)}, {alpha, beta}, static_cast<int>(splits));
    if (op.can_implement(args) != cutlass::Status::kSuccess) return false;
    if (GemmTNSplit::get_workspace_size(args) > ws.n * sizeof(double)) return false;
    const cutlass::Status st = op(args, ws.get(), s ? s : ctx->stream);
    if (st != cutlass::Status::kSuccess) throw cuda_error("CUTLASS split-K DGEMM launch failed");
    return true;
}

bool cutlass_gemm_nn(svt_ctx* ctx, cudaStream_t s, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
                     const double* B, i64 ldb, double beta, double* C, i64 ldc) {
    const i64 lim = (1LL << 31) - 1;
    if (M > lim || N > lim || K > lim || lda > lim || ldb > lim || ldc > lim) return false;
    const int c = cfg();
    if (c == 3) return run<GemmNNT<128, 64, 64, 32, 3, 1>>(ctx, s, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    if (c == 4) return run<GemmNNT<128, 32, 64, 16, 4, 1>>(ctx, s, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    if (c == 5) return run<GemmNNT<64, 32, 32, 16, 5, 1>>(ctx, s, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    if (c == 1) return run<GemmNNT<64, 32, 32, 16, 4, 1>>(ctx, s, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    if (c == 6) return run<GemmNNT<64, 64, 32, 32, 4, 1, 2>>(ctx, s, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    // default: one 128-column tile for the batch panels (W = 120 / 128: the
    // A rows are read once), 64-column tiles for narrower products
    if (N > 64) return run<GemmNNT<64, 128, 32, 64, 3, 1>>(ctx, s, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    return run<GemmNNT<64, 64, 32, 32, 4, 1>>(ctx, s, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
}

}  // namespace svtb
