// Dense kernels: tall-skinny FP64 GEMMs for block Gram-Schmidt (sketch.hpp:
// 133-141), CholQR2 with a Householder fallback (dense.hpp:103-110), the Gram
// eigensolver of finalize (sketch.hpp:158-162 / dense.hpp:114-117), and small
// reductions that drive the reference's data-dependent branches on the device
// (no host round trip inside a rank-revealing round).
//
// FP64 note: tcgen05 has no f64 kind on sm_100a, so FP64 contractions run on
// the FP64 pipes.  The dt = 10 passes are HBM-bound (2.5 flop/B on Q), so the
// GEMM is a register-tiled CUDA-core kernel whose job is to stream Q at HBM
// rate; split-K with a fixed-order reduction keeps results deterministic.
#include <math_constants.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"

namespace svtb {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ---------------------------------------------------------------------------
// GEMM
// ---------------------------------------------------------------------------
template <int BM, int BN, int BK, int TM, int TN, bool TA>
__global__ void __launch_bounds__((BM / TM) * (BN / TN)) gemm_kernel(
    long long M, long long N, long long K, double alpha, const double* __restrict__ A, long long lda,
    const double* __restrict__ B, long long ldb, double beta, double* __restrict__ C, long long ldc,
    long long kchunk, double* __restrict__ partial, const int* __restrict__ pred) {
    if (pred != nullptr && *pred == 0) return;
    constexpr int NT = (BM / TM) * (BN / TN);
    constexpr int TX = BN / TN;
    constexpr int TY = BM / TM;
    __shared__ double As[BK][BM + 1];
    __shared__ double Bs[BK][BN];
    const int tid = threadIdx.x;
    const int tx = tid % TX;
    const int ty = tid / TX;
    const long long i0 = static_cast<long long>(blockIdx.x) * BM;
    const long long j0 = static_cast<long long>(blockIdx.y) * BN;
    const long long kbeg = static_cast<long long>(blockIdx.z) * kchunk;
    const long long kend = min(K, kbeg + kchunk);
    double acc[TM][TN];
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) acc[a][b] = 0.0;

    for (long long k0 = kbeg; k0 < kend; k0 += BK) {
        if (TA) {
            for (int e = tid; e < BK * BM; e += NT) {
                const int kk = e / BM, ii = e % BM;
                const long long k = k0 + kk, i = i0 + ii;
                As[kk][ii] = (k < kend && i < M) ? __ldg(A + k * lda + i) : 0.0;
            }
        } else {
            for (int e = tid; e < BK * BM; e += NT) {
                const int ii = e / BK, kk = e % BK;
                const long long k = k0 + kk, i = i0 + ii;
                As[kk][ii] = (k < kend && i < M) ? __ldg(A + i * lda + k) : 0.0;
            }
        }
        for (int e = tid; e < BK * BN; e += NT) {
            const int kk = e / BN, jj = e % BN;
            const long long k = k0 + kk, j = j0 + jj;
            Bs[kk][jj] = (k < kend && j < N) ? __ldg(B + k * ldb + j) : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            double a[TM], b[TN];
#pragma unroll
            for (int t = 0; t < TM; ++t) a[t] = As[kk][ty + t * TY];
#pragma unroll
            for (int t = 0; t < TN; ++t) b[t] = Bs[kk][tx + t * TX];
#pragma unroll
            for (int p = 0; p < TM; ++p)
#pragma unroll
                for (int q = 0; q < TN; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int p = 0; p < TM; ++p) {
        const long long i = i0 + ty + p * TY;
        if (i >= M) continue;
#pragma unroll
        for (int q = 0; q < TN; ++q) {
            const long long j = j0 + tx + q * TX;
            if (j >= N) continue;
            if (gridDim.z == 1) {
                const double c = (beta != 0.0) ? beta * C[i * ldc + j] : 0.0;
                C[i * ldc + j] = fma(alpha, acc[p][q], c);
            } else {
                partial[(static_cast<long long>(blockIdx.z) * M + i) * N + j] = acc[p][q];
            }
        }
    }
}

// Split-K partial sums -> C.  A CTA owns 32 consecutive output elements;
// warp q adds splits q, q + 8, ... (lanes = elements, coalesced), then the 8
// warp sums are added in warp order: fixed order, deterministic.
constexpr int kRedWarps = 8;
__global__ void __launch_bounds__(32 * kRedWarps) gemm_reduce_kernel(long long M, long long N, int splits,
                                                                   const double* __restrict__ partial,
                                                                   double alpha, double beta,
                                                                   double* __restrict__ C, long long ldc,
                                                                   const int* __restrict__ pred) {
    if (pred != nullptr && *pred == 0) return;
    __shared__ double red[kRedWarps][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long e = blockIdx.x * 32LL + lane;
    const long long tot = M * N;
    double s0 = 0.0, s1 = 0.0;
    if (e < tot) {
        int z = warp;
        for (; z + kRedWarps < splits; z += 2 * kRedWarps) {
            s0 += partial[static_cast<long long>(z) * tot + e];
            s1 += partial[static_cast<long long>(z + kRedWarps) * tot + e];
        }
        if (z < splits) s0 += partial[static_cast<long long>(z) * tot + e];
    }
    red[warp][lane] = s0 + s1;
    __syncthreads();
    if (warp == 0 && e < tot) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < kRedWarps; ++q) t += red[q][lane];
        const long long i = e / N, j = e % N;
        const double c = (beta != 0.0) ? beta * C[i * ldc + j] : 0.0;
        C[i * ldc + j] = fma(alpha, t, c);
    }
}

__global__ void scale2d_kernel(double* C, long long M, long long N, long long ldc, double beta, const int* pred) {
    if (pred != nullptr && *pred == 0) return;
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= M * N) return;
    const long long i = e / N, j = e % N;
    C[i * ldc + j] = (beta != 0.0) ? beta * C[i * ldc + j] : 0.0;
}

// ---------------------------------------------------------------------------
// FP64 tensor-core GEMM: mma.sync.aligned.m8n8k4.f64 (SASS DMMA).  tcgen05
// has no f64 kind on sm_100a, so DMMA is the FP64 tensor path.  CTA tile
// 64 x BN, 8 warps as 2 (M) x 4 (N), warp tile 32 x BN/4 = 4 x (BN/32)
// m8n8 accumulators; BK = 16 staged in shared memory with a register
// prefetch of the next stage (double buffer).  Fragment layouts (PTX ISA,
// m8n8k4 .f64): A[g][t], B[t][g], C[g][2t..2t+1] with g = lane / 4,
// t = lane % 4.  Shared rows are padded to a stride of 4 mod 16 doubles so
// the 4 k-rows x 8 m-columns of a fragment load hit distinct bank pairs.
// ---------------------------------------------------------------------------
// Split-K partial buffer: sized once for the largest split the launchers
// allow (32M doubles), so it never regrows (a cudaFree inside an SVT step
// would stall the device mid-iteration).
inline void ensure_partial(svt_ctx* ctx, size_t need) {
    if (need > ctx->ws_partial.n) ctx->ws_partial.ensure(std::max<size_t>(need, size_t(32) << 20));
}

constexpr int kDmmaBM = 64;
constexpr int kDmmaBK = 16;

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int BN, bool TA>
__global__ void __launch_bounds__(256) dmma_gemm_kernel(long long M, long long N, long long K, double alpha,
                                                        const double* __restrict__ A, long long lda,
                                                        const double* __restrict__ B, long long ldb, double beta,
                                                        double* __restrict__ C, long long ldc, long long kchunk,
                                                        double* __restrict__ partial, const int* __restrict__ pred) {
    if (pred != nullptr && *pred == 0) return;
    constexpr int BM = kDmmaBM, BK = (BN == 128) ? 8 : kDmmaBK;  // 128-wide tiles stage 8 k-rows (smem)
    constexpr int SA = BM + 4;          // padded strides (== 4 mod 16 doubles)
    constexpr int SB = BN + ((BN % 16 == 4) ? 0 : (4 + 16 - (BN % 16)) % 16);
    constexpr int NT = BN / 32;         // n8 tiles per warp
    constexpr int A_PER = BK * BM / 256;
    constexpr int B_PER = BK * BN / 256;
    // A tile: k-major [BK][SA] when A^T is streamed (rows of A are k), and
    // row-major [BM][BK + 4] otherwise so the coalesced global rows store
    // without bank conflicts (stride 4 mod 16 doubles for the fragments)
    constexpr int SAR = BK + 4;
    __shared__ double As[2][TA ? BK * SA : BM * SAR];
    __shared__ double Bs[2][BK][SB];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp >> 2) * 32;          // warp's m offset in the tile
    const int wn = (warp & 3) * (BN / 4);     // warp's n offset
    const long long i0 = static_cast<long long>(blockIdx.x) * BM;
    const long long j0 = static_cast<long long>(blockIdx.y) * BN;
    const long long kbeg = static_cast<long long>(blockIdx.z) * kchunk;
    const long long kend = min(K, kbeg + kchunk);
    double acc[4][NT][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    double ra[A_PER], rb[B_PER];
    auto load = [&](long long k0) {
#pragma unroll
        for (int q = 0; q < A_PER; ++q) {
            const int e = tid + q * 256;
            int kk, ii;
            if (TA) {
                kk = e / BM;
                ii = e % BM;
            } else {
                ii = e / BK;
                kk = e % BK;
            }
            const long long k = k0 + kk, i = i0 + ii;
            ra[q] = (k < kend && i < M) ? __ldg(TA ? (A + k * lda + i) : (A + i * lda + k)) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < B_PER; ++q) {
            const int e = tid + q * 256;
            const int kk = e / BN, jj = e % BN;
            const long long k = k0 + kk, j = j0 + jj;
            rb[q] = (k < kend && j < N) ? __ldg(B + k * ldb + j) : 0.0;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int q = 0; q < A_PER; ++q) {
            const int e = tid + q * 256;
            int kk, ii;
            if (TA) {
                kk = e / BM;
                ii = e % BM;
            } else {
                ii = e / BK;
                kk = e % BK;
            }
            if (TA)
                As[buf][kk * SA + ii] = ra[q];
            else
                As[buf][ii * SAR + kk] = ra[q];
        }
#pragma unroll
        for (int q = 0; q < B_PER; ++q) {
            const int e = tid + q * 256;
            Bs[buf][e / BN][e % BN] = rb[q];
        }
    };
    int buf = 0;
    if (kbeg < kend) {
        load(kbeg);
        store(0);
    }
    __syncthreads();
    for (long long k0 = kbeg; k0 < kend; k0 += BK) {
        const bool more = k0 + BK < kend;
        if (more) load(k0 + BK);
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[4], bf[NT];
#pragma unroll
            for (int a = 0; a < 4; ++a)
                af[a] = TA ? As[buf][(kk + t) * SA + wm + a * 8 + g] : As[buf][(wm + a * 8 + g) * SAR + kk + t];
#pragma unroll
            for (int b = 0; b < NT; ++b) bf[b] = Bs[buf][kk + t][wn + b * 8 + g];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < NT; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
        if (more) store(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
    // epilogue: C fragment (g, 2t) and (g, 2t + 1) of each 8x8 tile
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const long long i = i0 + wm + a * 8 + g;
        if (i >= M) continue;
#pragma unroll
        for (int b = 0; b < NT; ++b) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const long long j = j0 + wn + b * 8 + 2 * t + h;
                if (j >= N) continue;
                if (gridDim.z == 1) {
                    const double o = (beta != 0.0) ? beta * C[i * ldc + j] : 0.0;
                    C[i * ldc + j] = fma(alpha, acc[a][b][h], o);
                } else {
                    partial[(static_cast<long long>(blockIdx.z) * M + i) * N + j] = acc[a][b][h];
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Same DMMA tile, fed by a 3-stage cp.async (LDGSTS) pipeline with BK = 16:
// global -> shared copies bypass the registers (no staging registers, so the
// 64 accumulator registers fit two CTAs per SM) and two stages are in flight
// while the warps run 64 DMMA per stage.  Requires 16-byte aligned operands
// with even leading dimensions (checked by the launcher; the register-staged
// kernel above handles the rest).  Out-of-range elements are zero-filled by
// the copy's src-size operand.
// ---------------------------------------------------------------------------
constexpr int kCpStages = 3;
constexpr int kCpBK = 16;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int bytes) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int BN, bool TA, int STG = kCpStages>
struct CpTile {
    static constexpr int BM = kDmmaBM, BK = kCpBK;
    static constexpr int SA = BM + 4;   // TA: [BK][SA]
    static constexpr int SAR = BK + 4;  // !TA: [BM][SAR]
    static constexpr int SB = BN + 4;   // [BK][SB]; BN + 4 == 4 mod 16 for BN in {32, 64, 128}
    static constexpr int A_ELEMS = TA ? BK * SA : BM * SAR;
    static constexpr int B_ELEMS = BK * SB;
    static constexpr size_t SMEM = sizeof(double) * STG * (A_ELEMS + B_ELEMS);
};

// GS (dense corner of a split sparse pattern, engine.cpp): row k of B is row
// brow[k] of the panel (a gather folded into the cp.async B loads) and every
// CTA writes its split-K partial tile (the caller's fixed-order reduction
// scatter-adds the block rows into the sparse product's output).
template <int BN, bool TA, bool GS = false, bool B8 = false, int STG = kCpStages>
__global__ void __launch_bounds__(256, 2) dmma_cp_kernel(long long M, long long N, long long K, double alpha,
                                                         const double* __restrict__ A, long long lda,
                                                         const double* __restrict__ B, long long ldb, double beta,
                                                         double* __restrict__ C, long long ldc, long long kchunk,
                                                         double* __restrict__ partial, const int* __restrict__ pred,
                                                         const int* __restrict__ brow = nullptr) {
    if (pred != nullptr && *pred == 0) return;
    using T = CpTile<BN, TA, STG>;
    constexpr int BM = T::BM, BK = T::BK, SA = T::SA, SAR = T::SAR, SB = T::SB;
    constexpr int NT = BN / 32;
    constexpr int A_CH = BM * BK / 2 / 256;  // 16-byte chunks per thread
    constexpr int B_CH = BK * BN / 2 / 256;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + STG * T::A_ELEMS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp >> 2) * 32;
    const int wn = (warp & 3) * (BN / 4);
    const long long i0 = static_cast<long long>(blockIdx.x) * BM;
    const long long j0 = static_cast<long long>(blockIdx.y) * BN;
    const long long kbeg = static_cast<long long>(blockIdx.z) * kchunk;
    const long long kend = min(K, kbeg + kchunk);
    const long long nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
    auto issue = [&](int stage, long long k0) {
        double* as = As + stage * T::A_ELEMS;
        double* bs = Bs + stage * T::B_ELEMS;
#pragma unroll
        for (int q = 0; q < A_CH; ++q) {
            const int c = tid + q * 256;
            if (TA) {
                const int kk = c / (BM / 2), ii = (c % (BM / 2)) * 2;
                const long long k = k0 + kk, i = i0 + ii;
                const int v = (k < kend) ? static_cast<int>(max(0LL, min(2LL, M - i))) : 0;
                cp_async16(as + kk * SA + ii, v ? A + k * lda + i : A, 8 * v);
            } else {
                const int ii = c / (BK / 2), kk = (c % (BK / 2)) * 2;
                const long long k = k0 + kk, i = i0 + ii;
                const int v = (i < M) ? static_cast<int>(max(0LL, min(2LL, kend - k))) : 0;
                cp_async16(as + ii * SAR + kk, v ? A + i * lda + k : A, 8 * v);
            }
        }
#pragma unroll
        for (int q = 0; q < B_CH; ++q) {
            const int c = tid + q * 256;
            const int kk = c / (BN / 2), jj = (c % (BN / 2)) * 2;
            const long long k = k0 + kk, j = j0 + jj;
            const int v = (k < kend) ? static_cast<int>(max(0LL, min(2LL, N - j))) : 0;
            const long long kr = (GS && v) ? static_cast<long long>(__ldg(brow + k)) : k;
            if (B8) {  // B rows not 16-byte aligned (a panel at an odd column offset)
                cp_async8(bs + kk * SB + jj, v >= 1 ? B + kr * ldb + j : B, v >= 1 ? 8 : 0);
                cp_async8(bs + kk * SB + jj + 1, v >= 2 ? B + kr * ldb + j + 1 : B, v >= 2 ? 8 : 0);
            } else {
                cp_async16(bs + kk * SB + jj, v ? B + kr * ldb + j : B, 8 * v);
            }
        }
    };
    double acc[4][NT][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
    for (int st = 0; st < STG - 1; ++st) {
        if (st < nk) issue(st, kbeg + st * BK);
        cp_async_commit();
    }
    for (long long it = 0; it < nk; ++it) {
        cp_async_wait<STG - 2>();
        __syncthreads();
        const long long nx = it + STG - 1;
        if (nx < nk) issue(static_cast<int>(nx % STG), kbeg + nx * BK);
        cp_async_commit();
        const int stg = static_cast<int>(it % STG);
        const double* as = As + stg * T::A_ELEMS;
        const double* bs = Bs + stg * T::B_ELEMS;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[4], bf[NT];
#pragma unroll
            for (int a = 0; a < 4; ++a)
                af[a] = TA ? as[(kk + t) * SA + wm + a * 8 + g] : as[(wm + a * 8 + g) * SAR + kk + t];
#pragma unroll
            for (int b = 0; b < NT; ++b) bf[b] = bs[(kk + t) * SB + wn + b * 8 + g];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < NT; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const long long i = i0 + wm + a * 8 + g;
        if (i >= M) continue;
#pragma unroll
        for (int b = 0; b < NT; ++b) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const long long j = j0 + wn + b * 8 + 2 * t + h;
                if (j >= N) continue;
                if (gridDim.z == 1 && !GS) {
                    const double o = (beta != 0.0) ? beta * C[i * ldc + j] : 0.0;
                    C[i * ldc + j] = fma(alpha, acc[a][b][h], o);
                } else {
                    partial[(static_cast<long long>(blockIdx.z) * M + i) * N + j] = acc[a][b][h];
                }
            }
        }
    }
}


static bool cutlass_nn_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SVTB_CUTLASS_NN");
        return e == nullptr || e[0] != '0';
    }();
    return on;
}

static bool cutlass_tn_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SVTB_CUTLASS_TN");
        return e == nullptr || e[0] != '0';
    }();
    return on;
}

static i64 cutlass_tn_min_m() {  // SVTB_CUTLASS_TN_MIN_M (A/B): smallest output height routed to CUTLASS
    static const i64 v = [] {
        const char* e = std::getenv("SVTB_CUTLASS_TN_MIN_M");
        return e ? static_cast<i64>(std::atoll(e)) : static_cast<i64>(512);
    }();
    return v;
}

// SVTB_CUTLASS_CORNER=1: the dense corner through the CUTLASS gather-B
// template instead of the hand-written GS kernel (measured equal in the
// step, 9.165 vs 9.171 it/s: the corner hides behind the cold gather)
static bool cutlass_corner_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SVTB_CUTLASS_CORNER");
        return e != nullptr && e[0] == '1';
    }();
    return on;
}

static int dmma_stages() {
    static const int v = [] {
        const char* e = std::getenv("SVTB_DMMA_STAGES");
        return e ? std::atoi(e) : 3;
    }();
    return v;
}

template <int BN>
void dmma_launch(svt_ctx* ctx, bool transA, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
                 const double* B, i64 ldb, double beta, double* C, i64 ldc, const int* pred) {
    const i64 mt = (M + kDmmaBM - 1) / kDmmaBM, nt = (N + BN - 1) / BN;
    const i64 tiles = mt * nt;
    static const bool no_cpasync = std::getenv("SVTB_NO_CPASYNC") != nullptr;
    // the cp.async pipeline needs 16-byte aligned rows
    const bool cp = (lda % 2 == 0) && (ldb % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                    (reinterpret_cast<uintptr_t>(B) % 16 == 0) && !no_cpasync;
    // resident CTAs per wave (occupancy of this instantiation, cached)
    static int per_sm[4] = {0, 0, 0, 0};
    int& ps = per_sm[(transA ? 1 : 0) + (cp ? 2 : 0)];
    if (ps == 0) {
        if (cp) {
            SVT_CUDA(cudaFuncSetAttribute(dmma_cp_kernel<BN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(CpTile<BN, true>::SMEM)));
            SVT_CUDA(cudaFuncSetAttribute(dmma_cp_kernel<BN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(CpTile<BN, false>::SMEM)));
            if (transA)
                SVT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, dmma_cp_kernel<BN, true>, 256,
                                                                       CpTile<BN, true>::SMEM));
            else
                SVT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, dmma_cp_kernel<BN, false>, 256,
                                                                       CpTile<BN, false>::SMEM));
        } else if (transA) {
            SVT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, dmma_gemm_kernel<BN, true>, 256, 0));
        } else {
            SVT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, dmma_gemm_kernel<BN, false>, 256, 0));
        }
        ps = std::max(1, ps);
    }
    const i64 cap = static_cast<i64>(ps) * ctx->num_sms;
    // split-K: minimise waves x k-steps per CTA (+ the partial-sum traffic of
    // the fixed-order reduction), so a grid never ends in a nearly empty wave
    i64 splits = 1;
    if (K > 32 * kDmmaBK) {
        const i64 kmax = std::min<i64>(512, (K + 32 * kDmmaBK - 1) / (32 * kDmmaBK));
        double best = 1e300;
        for (i64 sp = 1; sp <= kmax; ++sp) {
            if (sp > 1 && sp * M * N > (32LL << 20)) break;
            const i64 waves = (tiles * sp + cap - 1) / cap;
            const double ksteps = std::ceil(static_cast<double>(K) / (sp * kDmmaBK));
            // a k-step of one CTA streams (BM + BN) x BK doubles; the reduce
            // reads sp partial tiles once
            const double cost = waves * ksteps * (kDmmaBM + BN) * kDmmaBK +
                                (sp > 1 ? static_cast<double>(sp) * M * N / cap * 4.0 : 0.0);
            if (cost < best * 0.999) {
                best = cost;
                splits = sp;
            }
        }
    }
    i64 kchunk = (K + splits - 1) / splits;
    kchunk = ((kchunk + kDmmaBK - 1) / kDmmaBK) * kDmmaBK;  // multiple of both 16 and 8
    splits = std::max<i64>(1, (K + kchunk - 1) / kchunk);
    if (splits > 1) ensure_partial(ctx, static_cast<size_t>(splits * M * N));
    dim3 grid(static_cast<unsigned>(mt), static_cast<unsigned>(nt), static_cast<unsigned>(splits));
    if (cp && transA)
        dmma_cp_kernel<BN, true><<<grid, 256, CpTile<BN, true>::SMEM, ctx->stream>>>(
            M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, ctx->ws_partial.get(), pred);
    else if (cp && dmma_stages() == 4) {  // A/B switch SVTB_DMMA_STAGES=4 (4-stage cp.async pipeline)
        static bool attr4 = false;
        if (!attr4) {
            SVT_CUDA(cudaFuncSetAttribute(dmma_cp_kernel<BN, false, false, false, 4>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(CpTile<BN, false, 4>::SMEM)));
            attr4 = true;
        }
        dmma_cp_kernel<BN, false, false, false, 4><<<grid, 256, CpTile<BN, false, 4>::SMEM, ctx->stream>>>(
            M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, ctx->ws_partial.get(), pred);
    } else if (cp)
        dmma_cp_kernel<BN, false><<<grid, 256, CpTile<BN, false>::SMEM, ctx->stream>>>(
            M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, ctx->ws_partial.get(), pred);
    else if (transA)
        dmma_gemm_kernel<BN, true><<<grid, 256, 0, ctx->stream>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
                                                                  kchunk, ctx->ws_partial.get(), pred);
    else
        dmma_gemm_kernel<BN, false><<<grid, 256, 0, ctx->stream>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
                                                                   kchunk, ctx->ws_partial.get(), pred);
    if (splits > 1) {
        const i64 tot = M * N;
        gemm_reduce_kernel<<<static_cast<unsigned>((tot + 31) / 32), 32 * kRedWarps, 0, ctx->stream>>>(
            M, N, static_cast<int>(splits), ctx->ws_partial.get(), alpha, beta, C, ldc, pred);
    }
}

// out[orow[i] * ldo + j] += sum_z partial[z][i][j]  (fixed order: deterministic)
__global__ void block_scatter_add_kernel(long long M, long long N, int S, const double* __restrict__ partial,
                                         const int* __restrict__ orow, double* __restrict__ out, long long ldo) {
    const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (t >= M * N) return;
    const long long i = t / N, j = t - i * N;
    double acc = 0.0;
    for (int z = 0; z < S; ++z) acc += partial[(static_cast<long long>(z) * M + i) * N + j];
    out[static_cast<long long>(__ldg(orow + i)) * ldo + j] += acc;
}

template <int BN, bool TA, bool B8>
int dense_block_launch(svt_ctx* ctx, cudaStream_t s, i64 M, i64 N, i64 K, const double* D, i64 ldd,
                       const double* B, i64 ldb, const int* brow, DevBuf<double>& ws) {
    static bool attr = false;
    if (!attr) {
        SVT_CUDA(cudaFuncSetAttribute(dmma_cp_kernel<BN, TA, true, B8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(CpTile<BN, TA>::SMEM)));
        attr = true;
    }
    const i64 mt = (M + kDmmaBM - 1) / kDmmaBM, nt = (N + BN - 1) / BN, tiles = mt * nt;
    // K splits: as many as fill ONE wave of two resident CTAs per SM (a
    // second, nearly empty wave would double the time), at least 16 k-steps
    // per CTA
    i64 S = std::max<i64>(1, std::min<i64>((2 * ctx->num_sms) / tiles, K / (16 * kCpBK)));
    if (ws.n < static_cast<size_t>(M * N)) ws.ensure(static_cast<size_t>(M * N * S));  // one-time growth
    S = std::max<i64>(1, std::min<i64>(S, static_cast<i64>(ws.n / static_cast<size_t>(M * N))));
    i64 kchunk = (K + S - 1) / S;
    kchunk = ((kchunk + kCpBK - 1) / kCpBK) * kCpBK;
    S = (K + kchunk - 1) / kchunk;
    dim3 grid(static_cast<unsigned>(mt), static_cast<unsigned>(nt), static_cast<unsigned>(S));
    dmma_cp_kernel<BN, TA, true, B8><<<grid, 256, CpTile<BN, TA>::SMEM, s>>>(M, N, K, 1.0, D, ldd, B, ldb, 0.0,
                                                                            nullptr, 0, kchunk, ws.get(), nullptr,
                                                                            brow);
    return static_cast<int>(S);
}

template <int BM, int BN, int BK, int TM, int TN>
void gemm_launch(svt_ctx* ctx, bool transA, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
                 const double* B, i64 ldb, double beta, double* C, i64 ldc, const int* pred) {
    const i64 mt = (M + BM - 1) / BM, nt = (N + BN - 1) / BN;
    const i64 tiles = mt * nt;
    i64 splits = 1;
    const i64 target = 2LL * ctx->num_sms;
    if (tiles < target && K > 8 * BK) {
        splits = std::min<i64>((target + tiles - 1) / tiles, (K + 8 * BK - 1) / (8 * BK));
        splits = std::min<i64>(splits, 512);
        // bound the partial workspace to 256 MB
        while (splits > 1 && splits * M * N > (32LL << 20)) splits /= 2;
    }
    i64 kchunk = (K + splits - 1) / splits;
    kchunk = ((kchunk + BK - 1) / BK) * BK;
    splits = (K + kchunk - 1) / kchunk;
    if (splits < 1) splits = 1;
    if (splits > 1) ensure_partial(ctx, static_cast<size_t>(splits * M * N));
    dim3 grid(static_cast<unsigned>(mt), static_cast<unsigned>(nt), static_cast<unsigned>(splits));
    constexpr int NT = (BM / TM) * (BN / TN);
    if (transA)
        gemm_kernel<BM, BN, BK, TM, TN, true><<<grid, NT, 0, ctx->stream>>>(
            M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, ctx->ws_partial.get(), pred);
    else
        gemm_kernel<BM, BN, BK, TM, TN, false><<<grid, NT, 0, ctx->stream>>>(
            M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, ctx->ws_partial.get(), pred);
    if (splits > 1) {
        const i64 tot = M * N;
        gemm_reduce_kernel<<<static_cast<unsigned>((tot + 31) / 32), 32 * kRedWarps, 0, ctx->stream>>>(
            M, N, static_cast<int>(splits), ctx->ws_partial.get(), alpha, beta, C, ldc, pred);
    }
}

// ---------------------------------------------------------------------------
// Skinny GEMMs of the rank-revealing rounds (N = dt <= 16 output columns).
// These stream the basis Q once per pass at HBM rate; the tile GEMM above
// serves the wide cases.
// ---------------------------------------------------------------------------

// C (M x N) = alpha * A^T B + beta * C;  A: K x M row-major (Q), B: K x N (X).
// A CTA owns 32 columns of A (lane = column: one 256-byte row segment per
// load) and a slab of rows split over its 8 warps; each warp stages 32 rows
// of B in its own shared-memory slice (__syncwarp only) and keeps kTnUnroll
// independent loads of A in flight.  The 8 warp partials are folded in
// shared memory; CTAs along the row split write partials and the last CTA
// of each column group reduces them in fixed order (deterministic, no extra
// launch).
constexpr int kTnWarps = 8;
constexpr int kTnRows = 32;
constexpr int kTnUnroll = 16;

template <int N>
__global__ void __launch_bounds__(32 * kTnWarps) skinny_tn_kernel(
    long long M, long long K, const double* __restrict__ A, long long lda, const double* __restrict__ B,
    long long ldb, double alpha, double beta, double* __restrict__ C, long long ldc, long long rows_per_cta,
    double* __restrict__ partial, unsigned* __restrict__ counters, const int* __restrict__ pred) {
    if (pred != nullptr && *pred == 0) return;
    // one buffer per warp: staged B rows during the stream, then the
    // warp's per-column partials (stride N + 1) for the CTA fold
    __shared__ double sm[kTnWarps][32 * (N + 1)];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* Bs = sm[warp];
    const long long c = blockIdx.x * 32LL + lane;
    const bool cok = c < M;
    const long long cta_k0 = blockIdx.y * rows_per_cta;
    const long long cta_k1 = min(K, cta_k0 + rows_per_cta);
    const long long per_warp = (rows_per_cta + kTnWarps - 1) / kTnWarps;
    const long long k0 = min(cta_k1, cta_k0 + warp * per_warp);
    const long long k1 = min(cta_k1, k0 + per_warp);
    double acc[N];
#pragma unroll
    for (int j = 0; j < N; ++j) acc[j] = 0.0;
    const double* ac = A + (cok ? c : 0);
    for (long long kb = k0; kb < k1; kb += kTnRows) {
        const int nr = static_cast<int>(min(static_cast<long long>(kTnRows), k1 - kb));
        __syncwarp();
        for (int e = lane; e < kTnRows * N; e += 32) {
            const int rr = e / N, jj = e - (e / N) * N;
            Bs[rr * N + jj] = (rr < nr) ? __ldg(B + (kb + rr) * ldb + jj) : 0.0;
        }
        __syncwarp();
        const double* ap = ac + kb * lda;
#pragma unroll
        for (int r0 = 0; r0 < kTnRows; r0 += kTnUnroll) {
            double a[kTnUnroll];
#pragma unroll
            for (int u = 0; u < kTnUnroll; ++u) a[u] = (cok && r0 + u < nr) ? __ldg(ap + (r0 + u) * lda) : 0.0;
#pragma unroll
            for (int u = 0; u < kTnUnroll; ++u)
#pragma unroll
                for (int j = 0; j < N; ++j) acc[j] = fma(a[u], Bs[(r0 + u) * N + j], acc[j]);
        }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < N; ++j) Bs[lane * (N + 1) + j] = acc[j];
    __syncthreads();
    // fold the 8 warps: thread t -> (column lane t % 32, output j range)
    for (int e = threadIdx.x; e < 32 * N; e += 32 * kTnWarps) {
        const int cl = e / N, j = e - (e / N) * N;
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kTnWarps; ++w) s += sm[w][cl * (N + 1) + j];
        const long long cc = blockIdx.x * 32LL + cl;
        if (cc >= M) continue;
        if (gridDim.y == 1) {
            const double o = (beta != 0.0) ? beta * C[cc * ldc + j] : 0.0;
            C[cc * ldc + j] = fma(alpha, s, o);
        } else {
            partial[(blockIdx.y * M + cc) * N + j] = s;
        }
    }
    if (gridDim.y == 1) return;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(counters + blockIdx.x, 1u) == gridDim.y - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int e = threadIdx.x; e < 32 * N; e += 32 * kTnWarps) {
        const int cl = e / N, j = e - (e / N) * N;
        const long long cc = blockIdx.x * 32LL + cl;
        if (cc >= M) continue;
        double s = 0.0;
        for (unsigned z = 0; z < gridDim.y; ++z) s += __ldcg(partial + (z * M + cc) * N + j);
        const double o = (beta != 0.0) ? beta * C[cc * ldc + j] : 0.0;
        C[cc * ldc + j] = fma(alpha, s, o);
    }
    if (threadIdx.x == 0) counters[blockIdx.x] = 0u;
}

// C (M x N) = alpha * A B + beta * C;  A: M x K row-major (Q), B: K x N.
// One warp per kNnRows rows, lanes stride K (coalesced row segments of A),
// B staged transposed in shared memory (conflict-free per lane); per-row
// warp-shuffle reduction at the end.
constexpr int kNnWarps = 8, kNnRows = 4, kNnChunk = 256;

template <int N>
__global__ void __launch_bounds__(32 * kNnWarps) skinny_nn_kernel(long long M, long long K, double alpha,
                                                                  const double* __restrict__ A, long long lda,
                                                                  const double* __restrict__ B, long long ldb,
                                                                  double beta, double* __restrict__ C, long long ldc,
                                                                  const int* __restrict__ pred) {
    if (pred != nullptr && *pred == 0) return;
    __shared__ double Bs[N][kNnChunk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long r0 = (static_cast<long long>(blockIdx.x) * kNnWarps + warp) * kNnRows;
    double acc[kNnRows][N];
#pragma unroll
    for (int r = 0; r < kNnRows; ++r)
#pragma unroll
        for (int j = 0; j < N; ++j) acc[r][j] = 0.0;
    const double* ar[kNnRows];
    bool ok[kNnRows];
#pragma unroll
    for (int r = 0; r < kNnRows; ++r) {
        ok[r] = (r0 + r) < M;
        ar[r] = A + (ok[r] ? (r0 + r) : 0) * lda;
    }
    for (long long kb = 0; kb < K; kb += kNnChunk) {
        const int nk = static_cast<int>(min(static_cast<long long>(kNnChunk), K - kb));
        __syncthreads();
        for (int e = threadIdx.x; e < kNnChunk * N; e += 32 * kNnWarps) {
            const int kk = e / N, jj = e % N;
            Bs[jj][kk] = (kk < nk) ? __ldg(B + (kb + kk) * ldb + jj) : 0.0;
        }
        __syncthreads();
#pragma unroll 2
        for (int kk = lane; kk < nk; kk += 32) {
            double b[N];
#pragma unroll
            for (int j = 0; j < N; ++j) b[j] = Bs[j][kk];
#pragma unroll
            for (int r = 0; r < kNnRows; ++r) {
                const double a = ok[r] ? __ldg(ar[r] + kb + kk) : 0.0;
#pragma unroll
                for (int j = 0; j < N; ++j) acc[r][j] = fma(a, b[j], acc[r][j]);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < kNnRows; ++r) {
        double mine = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double s = warp_sum(acc[r][j]);
            if (lane == j) mine = s;
        }
        if (ok[r] && lane < N) {
            double* cp = C + (r0 + r) * ldc + lane;
            const double o = (beta != 0.0) ? beta * (*cp) : 0.0;
            *cp = fma(alpha, mine, o);
        }
    }
}

// Gram-type C = A^T B with M, N <= 16 and long K (a narrow panel's Gram
// matrix): warps stride rows, lanes own (a, b) products; the last CTA
// reduces the per-CTA partials in fixed order and, for a Cholesky QR pass,
// factors the Gram right there (Rinv = L^{-T}, status = 1 on a bad pivot).
constexpr int kTinyThreads = 256;
constexpr int kTinyMaxW = 16;

template <int QN>
__global__ void __launch_bounds__(kTinyThreads) tiny_tn_kernel(long long K, int M, int N,
                                                               const double* __restrict__ A, long long lda,
                                                               const double* __restrict__ B, long long ldb,
                                                               double* __restrict__ C, double* __restrict__ partial,
                                                               unsigned* __restrict__ counter, int do_chol,
                                                               double* __restrict__ Rinv, int* __restrict__ status,
                                                               const int* __restrict__ pred) {
    if (pred != nullptr && *pred == 0) return;
    constexpr int RU = (QN <= 4) ? 8 : 4;  // rows whose loads are in flight together
    __shared__ double red[kTinyThreads / 32][kTinyMaxW * kTinyMaxW];
    __shared__ double L[kTinyMaxW][kTinyMaxW + 1];
    __shared__ double dorig[kTinyMaxW];
    __shared__ bool last;
    __shared__ int fail;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int P = M * N;
    double acc[QN];
#pragma unroll
    for (int q = 0; q < QN; ++q) acc[q] = 0.0;
    const long long gw = blockIdx.x * static_cast<long long>(kTinyThreads / 32) + warp;
    const long long nw = static_cast<long long>(gridDim.x) * (kTinyThreads / 32);
    long long i = gw;
    for (; i + (RU - 1) * nw < K; i += RU * nw) {
        double a[RU][QN], b[RU][QN];
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            const double* ai = A + (i + u * nw) * lda;
            const double* bi = B + (i + u * nw) * ldb;
#pragma unroll
            for (int q = 0; q < QN; ++q) {
                const int p = lane + 32 * q;
                a[u][q] = (p < P) ? __ldg(ai + p / N) : 0.0;
                b[u][q] = (p < P) ? __ldg(bi + p % N) : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < RU; ++u)
#pragma unroll
            for (int q = 0; q < QN; ++q) acc[q] = fma(a[u][q], b[u][q], acc[q]);
    }
    for (; i < K; i += nw) {
        const double* ai = A + i * lda;
        const double* bi = B + i * ldb;
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int p = lane + 32 * q;
            if (p < P) acc[q] = fma(__ldg(ai + p / N), __ldg(bi + p % N), acc[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < QN; ++q) {
        const int p = lane + 32 * q;
        if (p < P) red[warp][p] = acc[q];
    }
    __syncthreads();
    for (int p = threadIdx.x; p < P; p += kTinyThreads) {
        double s = 0.0;
        for (int w = 0; w < kTinyThreads / 32; ++w) s += red[w][p];
        partial[blockIdx.x * static_cast<long long>(kTinyMaxW * kTinyMaxW) + p] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    // fixed-order reduction over the CTA partials: 8 independent loads in
    // flight per thread, combined in block order
    for (int p = threadIdx.x; p < P; p += kTinyThreads) {
        double s = 0.0;
        unsigned b = 0;
        const long long stride = static_cast<long long>(kTinyMaxW * kTinyMaxW);
        for (; b + 8 <= gridDim.x; b += 8) {
            double t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) t[u] = __ldcg(partial + (b + u) * stride + p);
#pragma unroll
            for (int u = 0; u < 8; ++u) s += t[u];
        }
        for (; b < gridDim.x; ++b) s += __ldcg(partial + b * stride + p);
        C[p] = s;
        L[p / N][p % N] = s;
    }
    if (threadIdx.x == 0) {
        *counter = 0u;
        fail = 0;
    }
    __syncthreads();
    if (!do_chol) return;
    const int w = M;
    if (threadIdx.x < w) dorig[threadIdx.x] = L[threadIdx.x][threadIdx.x];
    __syncthreads();
    for (int j = 0; j < w; ++j) {
        const double d = L[j][j];
        const bool bad = !(dorig[j] > 0.0) || !(d > 1e-13 * dorig[j]) || !(d < CUDART_INF);
        const double ljj = sqrt(bad ? 1.0 : d);
        __syncthreads();
        if (threadIdx.x == 0) {
            if (bad) fail = 1;
            L[j][j] = ljj;
        }
        for (int i = j + 1 + threadIdx.x; i < w; i += kTinyThreads) L[i][j] /= ljj;
        __syncthreads();
        const int rem = w - j - 1;
        for (int e = threadIdx.x; e < rem * rem; e += kTinyThreads) {
            const int i = j + 1 + e / rem, k = j + 1 + e % rem;
            if (k <= i) L[i][k] -= L[i][j] * L[k][j];
        }
        __syncthreads();
    }
    if (threadIdx.x < w) {
        const int c = threadIdx.x;
        double x[kTinyMaxW];
        for (int r = 0; r < w; ++r) x[r] = 0.0;
        x[c] = 1.0 / L[c][c];
        for (int r = c - 1; r >= 0; --r) {
            double s = 0.0;
            for (int t = r + 1; t <= c; ++t) s += L[t][r] * x[t];
            x[r] = -s / L[r][r];
        }
        for (int r = 0; r < w; ++r) Rinv[r * w + c] = x[r];
    }
    if (threadIdx.x == 0 && fail) status[0] = 1;
}

// Cholesky of the w x w Gram in shared memory L and Rinv = L^{-T}; all
// threads of the block participate.  fail is block-shared.
__device__ void block_chol_rinv(double (*L)[kTinyMaxW + 1], int w, double* dorig, int* fail, double* Rinv,
                                int* status) {
    if (threadIdx.x == 0) *fail = 0;
    if (threadIdx.x < w) dorig[threadIdx.x] = L[threadIdx.x][threadIdx.x];
    __syncthreads();
    for (int j = 0; j < w; ++j) {
        const double d = L[j][j];
        const bool bad = !(dorig[j] > 0.0) || !(d > 1e-13 * dorig[j]) || !(d < CUDART_INF);
        const double ljj = sqrt(bad ? 1.0 : d);
        __syncthreads();
        if (threadIdx.x == 0) {
            if (bad) *fail = 1;
            L[j][j] = ljj;
        }
        for (int i = j + 1 + threadIdx.x; i < w; i += blockDim.x) L[i][j] /= ljj;
        __syncthreads();
        const int rem = w - j - 1;
        for (int e = threadIdx.x; e < rem * rem; e += blockDim.x) {
            const int i = j + 1 + e / rem, k = j + 1 + e % rem;
            if (k <= i) L[i][k] -= L[i][j] * L[k][j];
        }
        __syncthreads();
    }
    if (threadIdx.x < w) {
        const int c = threadIdx.x;
        double x[kTinyMaxW];
        for (int r = 0; r < w; ++r) x[r] = 0.0;
        x[c] = 1.0 / L[c][c];
        for (int r = c - 1; r >= 0; --r) {
            double s = 0.0;
            for (int t = r + 1; t <= c; ++t) s += L[t][r] * x[t];
            x[r] = -s / L[r][r];
        }
        for (int r = 0; r < w; ++r) Rinv[r * w + c] = x[r];
    }
    __syncthreads();
    if (threadIdx.x == 0 && *fail) status[0] = 1;
}

// Symmetric Gram G = X^T X of a narrow panel (W <= 12): one thread per row
// (one contiguous 8W-byte load), the W(W+1)/2 products in registers, warp
// shuffle + shared-memory fold per CTA, last CTA reduces the CTA partials in
// fixed order and optionally runs the Cholesky (CholQR pass head).
constexpr int kGramThreads = 256;

template <int W>
__global__ void __launch_bounds__(kGramThreads) gram_sym_kernel(long long K, const double* __restrict__ X,
                                                                long long ldx, double* __restrict__ G,
                                                                double* __restrict__ partial,
                                                                unsigned* __restrict__ counter, int do_chol,
                                                                double* __restrict__ Rinv, int* __restrict__ status,
                                                                const int* __restrict__ pred) {
    if (pred != nullptr && *pred == 0) return;
    constexpr int P = W * (W + 1) / 2;
    __shared__ double red[kGramThreads / 32][P];
    __shared__ double L[kTinyMaxW][kTinyMaxW + 1];
    __shared__ double dorig[kTinyMaxW];
    __shared__ bool last;
    __shared__ int fail;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc[P];
#pragma unroll
    for (int p = 0; p < P; ++p) acc[p] = 0.0;
    const long long stride = static_cast<long long>(gridDim.x) * kGramThreads;
    for (long long i = blockIdx.x * static_cast<long long>(kGramThreads) + threadIdx.x; i < K; i += stride) {
        double x[W];
#pragma unroll
        for (int a = 0; a < W; ++a) x[a] = __ldg(X + i * ldx + a);
        int p = 0;
#pragma unroll
        for (int a = 0; a < W; ++a)
#pragma unroll
            for (int b = 0; b <= a; ++b) {
                acc[p] = fma(x[a], x[b], acc[p]);
                ++p;
            }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const double s = warp_sum(acc[p]);
        if (lane == 0) red[warp][p] = s;
    }
    __syncthreads();
    for (int p = threadIdx.x; p < P; p += kGramThreads) {
        double s = 0.0;
        for (int w = 0; w < kGramThreads / 32; ++w) s += red[w][p];
        partial[blockIdx.x * static_cast<long long>(P) + p] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int p = threadIdx.x; p < P; p += kGramThreads) {
        double s = 0.0;
        unsigned b = 0;
        for (; b + 8 <= gridDim.x; b += 8) {
            double t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) t[u] = __ldcg(partial + (b + u) * static_cast<long long>(P) + p);
#pragma unroll
            for (int u = 0; u < 8; ++u) s += t[u];
        }
        for (; b < gridDim.x; ++b) s += __ldcg(partial + b * static_cast<long long>(P) + p);
        // p -> (a, b) with b <= a
        int a = 0;
        while ((a + 1) * (a + 2) / 2 <= p) ++a;
        const int bb = p - a * (a + 1) / 2;
        G[a * W + bb] = s;
        G[bb * W + a] = s;
        L[a][bb] = s;
        L[bb][a] = s;
    }
    if (threadIdx.x == 0) *counter = 0u;
    __syncthreads();
    if (do_chol) block_chol_rinv(L, W, dorig, &fail, Rinv, status);
}

// C (M x N) = alpha * A B + beta * C for a short inner dimension (K <= 16):
// one thread per row of A (contiguous 8K-byte row), B broadcast from shared.
template <int KK>
__global__ void __launch_bounds__(256) smallk_nn_kernel(long long M, int N, double alpha,
                                                        const double* __restrict__ A, long long lda,
                                                        const double* __restrict__ B, long long ldb, double beta,
                                                        double* __restrict__ C, long long ldc,
                                                        const int* __restrict__ pred) {
    if (pred != nullptr && *pred == 0) return;
    __shared__ double Bs[KK * 16];
    for (int e = threadIdx.x; e < KK * N; e += blockDim.x) Bs[e] = B[(e / N) * ldb + e % N];
    __syncthreads();
    const long long row = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (row >= M) return;
    double a[KK];
#pragma unroll
    for (int k = 0; k < KK; ++k) a[k] = __ldg(A + row * lda + k);
    for (int j = 0; j < N; ++j) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < KK; ++k) s = fma(a[k], Bs[k * N + j], s);
        double* cp = C + row * ldc + j;
        const double o = (beta != 0.0) ? beta * (*cp) : 0.0;
        *cp = fma(alpha, s, o);
    }
}

unsigned* counters(svt_ctx* ctx) {
    if (ctx->ws_counters.n < 8192) {
        ctx->ws_counters.alloc(8192);
        SVT_CUDA(cudaMemsetAsync(ctx->ws_counters.get(), 0, 8192 * sizeof(unsigned), ctx->stream));
    }
    return ctx->ws_counters.get();
}

template <int N>
void skinny_tn_launch(svt_ctx* ctx, i64 M, i64 K, double alpha, const double* A, i64 lda, const double* B, i64 ldb,
                      double beta, double* C, i64 ldc, const int* pred) {
    const i64 groups = (M + 31) / 32;
    if (groups > 8000) throw std::invalid_argument("skinny_tn: too many column groups");
    // aim for ~6 CTAs per SM overall; at least 32 rows per warp
    i64 splits = std::max<i64>(1, (6LL * ctx->num_sms + groups - 1) / groups);
    splits = std::min<i64>(splits, std::max<i64>(1, K / (kTnWarps * 32)));
    splits = std::min<i64>(splits, 4096);
    while (splits > 1 && splits * M * N > (32LL << 20)) splits /= 2;
    i64 rpc = (K + splits - 1) / splits;
    rpc = ((rpc + kTnWarps * kTnRows - 1) / (kTnWarps * kTnRows)) * (kTnWarps * kTnRows);
    splits = std::max<i64>(1, (K + rpc - 1) / rpc);
    unsigned* cnt = counters(ctx);
    if (splits > 1) ensure_partial(ctx, static_cast<size_t>(splits * M * N));
    dim3 grid(static_cast<unsigned>(groups), static_cast<unsigned>(splits));
    skinny_tn_kernel<N><<<grid, 32 * kTnWarps, 0, ctx->stream>>>(M, K, A, lda, B, ldb, alpha, beta, C, ldc, rpc,
                                                                 ctx->ws_partial.get(), cnt, pred);
}

template <int N>
void skinny_nn_launch(svt_ctx* ctx, i64 M, i64 K, double alpha, const double* A, i64 lda, const double* B, i64 ldb,
                      double beta, double* C, i64 ldc, const int* pred) {
    const i64 rows_per_block = static_cast<i64>(kNnWarps) * kNnRows;
    const unsigned blocks = static_cast<unsigned>((M + rows_per_block - 1) / rows_per_block);
    skinny_nn_kernel<N><<<blocks, 32 * kNnWarps, 0, ctx->stream>>>(M, K, alpha, A, lda, B, ldb, beta, C, ldc, pred);
}

void gram_sym_launch(svt_ctx* ctx, i64 K, int w, const double* X, i64 ldx, double* G, bool do_chol, double* Rinv,
                     int* status, const int* pred) {
    const i64 blocks = std::max<i64>(1, std::min<i64>(ctx->num_sms, (K + kGramThreads - 1) / kGramThreads));
    unsigned* cnt = counters(ctx) + 8190;
    ctx->ws_partial2.ensure(static_cast<size_t>(blocks * w * (w + 1) / 2));
    const unsigned nb = static_cast<unsigned>(blocks);
    double* part = ctx->ws_partial2.get();
    const int dc = do_chol ? 1 : 0;
    switch (w) {
#define SVT_CASE(WW)                                                                                          \
    case WW:                                                                                                  \
        gram_sym_kernel<WW><<<nb, kGramThreads, 0, ctx->stream>>>(K, X, ldx, G, part, cnt, dc, Rinv, status, pred); \
        break;
        SVT_CASE(1) SVT_CASE(2) SVT_CASE(3) SVT_CASE(4) SVT_CASE(5) SVT_CASE(6) SVT_CASE(7) SVT_CASE(8)
        SVT_CASE(9) SVT_CASE(10) SVT_CASE(11) SVT_CASE(12)
#undef SVT_CASE
        default:
            throw std::invalid_argument("gram_sym: w > 12");
    }
}

void smallk_nn_launch(svt_ctx* ctx, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda, const double* B,
                      i64 ldb, double beta, double* C, i64 ldc, const int* pred) {
    const unsigned blocks = static_cast<unsigned>((M + 255) / 256);
    const int n = static_cast<int>(N);
    switch (K) {
#define SVT_CASE(KK)                                                                                              \
    case KK:                                                                                                      \
        smallk_nn_kernel<KK><<<blocks, 256, 0, ctx->stream>>>(M, n, alpha, A, lda, B, ldb, beta, C, ldc, pred); \
        break;
        SVT_CASE(1) SVT_CASE(2) SVT_CASE(3) SVT_CASE(4) SVT_CASE(5) SVT_CASE(6) SVT_CASE(7) SVT_CASE(8)
        SVT_CASE(9) SVT_CASE(10) SVT_CASE(11) SVT_CASE(12) SVT_CASE(13) SVT_CASE(14) SVT_CASE(15) SVT_CASE(16)
#undef SVT_CASE
        default:
            throw std::invalid_argument("smallk_nn: K > 16");
    }
}

void tiny_tn_launch(svt_ctx* ctx, i64 K, int M, int N, const double* A, i64 lda, const double* B, i64 ldb, double* C,
                    bool do_chol, double* Rinv, int* status, const int* pred) {
    // few CTAs with deep per-warp row unrolling: the fixed-order partial
    // reduction in the last CTA stays short
    const i64 blocks = std::max<i64>(1, std::min<i64>(64, (K + 1023) / 1024));
    unsigned* cnt = counters(ctx) + 8191;
    ctx->ws_partial2.ensure(static_cast<size_t>(blocks * kTinyMaxW * kTinyMaxW));
    const int P = M * N;
    const unsigned nb = static_cast<unsigned>(blocks);
    double* part = ctx->ws_partial2.get();
    const int dc = do_chol ? 1 : 0;
    if (P <= 32)
        tiny_tn_kernel<1><<<nb, kTinyThreads, 0, ctx->stream>>>(K, M, N, A, lda, B, ldb, C, part, cnt, dc, Rinv, status, pred);
    else if (P <= 64)
        tiny_tn_kernel<2><<<nb, kTinyThreads, 0, ctx->stream>>>(K, M, N, A, lda, B, ldb, C, part, cnt, dc, Rinv, status, pred);
    else if (P <= 128)
        tiny_tn_kernel<4><<<nb, kTinyThreads, 0, ctx->stream>>>(K, M, N, A, lda, B, ldb, C, part, cnt, dc, Rinv, status, pred);
    else
        tiny_tn_kernel<8><<<nb, kTinyThreads, 0, ctx->stream>>>(K, M, N, A, lda, B, ldb, C, part, cnt, dc, Rinv, status, pred);
}

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------
constexpr int kRedBlocks = 256;

__global__ void sumsq_partial_kernel(const double* __restrict__ X, long long rows, long long cols, long long ld,
                                     double* __restrict__ partial, const int* __restrict__ pred) {
    if (pred != nullptr && *pred == 0) return;
    __shared__ double red[32];
    double s = 0.0;
    const long long tot = rows * cols;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = e / cols, j = e % cols;
        const double v = X[i * ld + j];
        s = fma(v, v, s);
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = (threadIdx.x < blockDim.x / 32) ? red[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) partial[blockIdx.x] = t;
    }
}

__global__ void maxabs_partial_kernel(const double* __restrict__ X, long long rows, long long cols, long long ld,
                                      double shift, double* __restrict__ partial) {
    __shared__ double red[32];
    double s = 0.0;
    const long long tot = rows * cols;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = e / cols, j = e % cols;
        double v = X[i * ld + j];
        if (i == j) v -= shift;
        s = fmax(s, fabs(v));
        if (v != v) s = CUDART_INF;  // NaN forces the branch
    }
    s = warp_max(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = (threadIdx.x < blockDim.x / 32) ? red[threadIdx.x] : 0.0;
        t = warp_max(t);
        if (threadIdx.x == 0) partial[blockIdx.x] = t;
    }
}

// op: 0 store sum, 1 add sum, 2 store max
__global__ void finish_kernel(const double* __restrict__ partial, int n, double* __restrict__ out, int op,
                              const int* __restrict__ pred) {
    if (pred != nullptr && *pred == 0) return;
    double t = 0.0;
    for (int b = threadIdx.x; b < n; b += 32) t = (op == 2) ? fmax(t, partial[b]) : t + partial[b];
    t = (op == 2) ? warp_max(t) : warp_sum(t);
    if (threadIdx.x == 0) {
        if (op == 1)
            out[0] += t;
        else
            out[0] = t;
    }
}

__global__ void set_flag_kernel(const double* a, const double* b, double coef, int mode, int* flag) {
    if (mode == 0)
        flag[0] = (sqrt(a[0]) > coef * sqrt(b[0])) ? 1 : 0;
    else
        flag[0] = (a[0] > coef) ? 1 : 0;
}

// Per-block decisions of a round batch (K blocks of w columns), one warp:
// mode 0: flag = some block kept less than thr2 of its squared norm
//         (after[k] < thr2 * before[k]): the re-check product is needed;
// mode 1: flag = gate && some block has ||Q^T X_k|| > 1e-8 ||X_k||
//         (sketch.hpp:134): the second Gram-Schmidt pass is needed.
__global__ void block_flags_kernel(const double* __restrict__ after, const double* __restrict__ before,
                                   const double* __restrict__ proj, int K, int w, double thr2, int mode,
                                   const int* __restrict__ gate, int* __restrict__ flag) {
    const int lane = threadIdx.x;
    int hit = 0;
    if (mode == 0 || *gate != 0) {
        for (int k = lane; k < K; k += 32) {
            double a = 0.0, b = 0.0;
            for (int q = 0; q < w; ++q) {
                a += after[k * w + q];
                b += (mode == 0) ? before[k * w + q] : proj[k * w + q];
            }
            if (mode == 0 ? !(a >= thr2 * b) : (sqrt(b) > 1e-8 * sqrt(a))) hit = 1;
        }
    }
    hit = __any_sync(0xffffffffu, hit);
    if (lane == 0) flag[0] = hit;
}

// ---------------------------------------------------------------------------
// CholQR: Cholesky + explicit inverse of R = L^T, one CTA, w <= 64
// ---------------------------------------------------------------------------
constexpr int kCholMax = 128;  // widest Cholesky panel (a batch of rounds)
constexpr int kHhMax = 64;     // widest Householder fallback panel

// L lives in dynamic shared memory, row stride w + 1 (w <= 128: 132 KB), plus
// a w x 8 panel temporary.  Blocked in 8-column panels:
//  * Cholesky (right-looking): warp 0 factors the 8-column panel in registers
//    (lane = row, shuffles broadcast the pivots and the panel rows), then all
//    32 warps apply the rank-8 update to the trailing lower triangle -- two
//    barriers per panel instead of one per column;
//  * inverse of the lower factor, block columns from the last: with
//    L = [[D, 0], [B, E]], L^{-1} = [[D^{-1}, 0], [-E^{-1} B D^{-1}, E^{-1}]],
//    E^{-1} already in place; T = E^{-1} B is one dot product per element
//    (all threads), then the block is T D^{-1} and D is inverted by one warp.
// A pivot that lost more than ~13 digits (kappa(X) beyond ~3e6 in that
// direction) or a zero / non-finite column sets status, which routes the
// panel to the Householder fallback (it keeps all columns like
// qr_orthonormal, dense.hpp:100-102).
constexpr int kCholPanel = 8;

__global__ void __launch_bounds__(512) chol_rinv_kernel(const double* __restrict__ G, int w,
                                                        double* __restrict__ Rinv, int* __restrict__ status,
                                                        const int* __restrict__ pred) {
    if (pred != nullptr && *pred == 0) return;
    constexpr int P = kCholPanel;
    extern __shared__ double dyn[];
    double* L = dyn;                   // w x (w + 1)
    double* dorig = dyn + w * (w + 1);  // w
    double* T = dorig + w;              // w x P (panel temporary)
    __shared__ int fail;
    const int ld = w + 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ double wmax[16];
    if (tid == 0) fail = 0;
    double emax = 0.0;
    for (int e = tid; e < w * w; e += blockDim.x) {
        const double g = G[e];
        L[(e / w) * ld + e % w] = g;
        const double d = fabs(g - ((e / w == e % w) ? 1.0 : 0.0));
        emax = (d > emax || d != d) ? d : emax;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    if (lane == 0) wmax[warp] = emax;
    __syncthreads();
    emax = 0.0;
    for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) emax = fmax(emax, wmax[q]);
    // Second CholQR pass: G = I + E with E at rounding level (measured
    // max|E| ~ 1e-13 at W = 120).  Then R = I + triu(E, 1) + diag(E) / 2 +
    // O(E^2) and R^{-1} = I - triu(E, 1) - diag(E) / 2 + O(E^2): with
    // max|E| <= 1e-8 / w the O(E^2) term is below 1e-16, so the factor is
    // written directly (upper triangular: the nested spans are unchanged).
    if (emax <= 1e-8 / static_cast<double>(w)) {
        for (int e = tid; e < w * w; e += blockDim.x) {
            const int r = e / w, c = e % w;
            const double g = L[r * ld + c];
            Rinv[e] = (r < c) ? -g : (r == c ? 1.0 - 0.5 * (g - 1.0) : 0.0);
        }
        return;
    }
    if (tid < w) dorig[tid] = L[tid * ld + tid];
    __syncthreads();
    // ---- Cholesky --------------------------------------------------------
    for (int c0 = 0; c0 < w; c0 += P) {
        const int pw = min(P, w - c0);
        if (warp == 0) {
            double a[4][P];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int r = c0 + lane + 32 * q;
#pragma unroll
                for (int jj = 0; jj < P; ++jj) a[q][jj] = (r < w && jj < pw) ? L[r * ld + c0 + jj] : 0.0;
            }
            bool bad_any = false;
#pragma unroll
            for (int jj = 0; jj < P; ++jj) {
                if (jj < pw) {
                    const int j = c0 + jj;
                    const double d = __shfl_sync(0xffffffffu, a[0][jj], jj);
                    const bool bad = !(dorig[j] > 0.0) || !(d > 1e-13 * dorig[j]) || !(d < CUDART_INF);
                    bad_any |= bad;
                    const double sq = sqrt(bad ? 1.0 : d);
                    const double inv = 1.0 / sq;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int r = c0 + lane + 32 * q;
                        if (r > j) a[q][jj] *= inv;
                        else if (r == j) a[q][jj] = sq;
                    }
#pragma unroll
                    for (int kk = jj + 1; kk < P; ++kk) {
                        if (kk < pw) {
                            const double lk = __shfl_sync(0xffffffffu, a[0][jj], kk);  // L[c0 + kk][j]
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const int r = c0 + lane + 32 * q;
                                if (r >= c0 + kk) a[q][kk] -= a[q][jj] * lk;
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int r = c0 + lane + 32 * q;
                if (r < w)
#pragma unroll
                    for (int jj = 0; jj < P; ++jj)
                        if (jj < pw && c0 + jj <= r) L[r * ld + c0 + jj] = a[q][jj];
            }
            if (lane == 0 && bad_any) fail = 1;
        }
        __syncthreads();
        // rank-pw update of the trailing lower triangle
        const int t0 = c0 + pw;
        for (int i = t0 + (tid >> 5); i < w; i += (blockDim.x >> 5)) {
            double li[P];
#pragma unroll
            for (int jj = 0; jj < P; ++jj) li[jj] = jj < pw ? L[i * ld + c0 + jj] : 0.0;
            for (int k = t0 + lane; k <= i; k += 32) {
                double s = L[i * ld + k];
#pragma unroll
                for (int jj = 0; jj < P; ++jj) s -= li[jj] * L[k * ld + c0 + jj];
                L[i * ld + k] = s;
            }
        }
        __syncthreads();
    }
    // ---- inverse of the lower factor, block columns from the last ---------
    const int nblk = (w + P - 1) / P;
    for (int bj = nblk - 1; bj >= 0; --bj) {
        const int c0 = bj * P, pw = min(P, w - c0), t0 = c0 + pw;
        // T[i - t0][jj] = sum_{t0 <= k <= i} Einv[i][k] * B[k][jj]  (E^{-1} in place)
        const int nrow = w - t0;
        for (int e = tid; e < nrow * pw; e += blockDim.x) {
            const int i = t0 + e / pw, jj = e % pw;
            double s0 = 0.0, s1 = 0.0;
            int k = t0;
            for (; k + 1 <= i; k += 2) {
                s0 = fma(L[i * ld + k], L[k * ld + c0 + jj], s0);
                s1 = fma(L[i * ld + k + 1], L[(k + 1) * ld + c0 + jj], s1);
            }
            if (k <= i) s0 = fma(L[i * ld + k], L[k * ld + c0 + jj], s0);
            T[(i - t0) * P + jj] = s0 + s1;
        }
        // invert the diagonal block in place (one warp, lane jj = column jj):
        // x_jj = 1 / D_jj, x_i = -(sum_{jj <= k < i} D_ik x_k) / D_ii
        if (warp == 0) {
            double x[P];
#pragma unroll
            for (int i = 0; i < P; ++i) x[i] = 0.0;
            if (lane < pw) {
#pragma unroll
                for (int i = 0; i < P; ++i) {
                    if (i < pw && i >= lane) {
                        double sacc = (i == lane) ? 1.0 : 0.0;
#pragma unroll
                        for (int k = 0; k < P; ++k)
                            if (k >= lane && k < i) sacc -= L[(c0 + i) * ld + c0 + k] * x[k];
                        x[i] = sacc / L[(c0 + i) * ld + c0 + i];
                    }
                }
            }
            __syncwarp();
            if (lane < pw)
#pragma unroll
                for (int i = 0; i < P; ++i)
                    if (i < pw && i >= lane) L[(c0 + i) * ld + c0 + lane] = x[i];
        }
        __syncthreads();
        // block below the diagonal: -T * D^{-1}  (D^{-1} lower, in place now)
        for (int e = tid; e < nrow * pw; e += blockDim.x) {
            const int i = t0 + e / pw, jj = e % pw;
            double sacc = 0.0;
#pragma unroll
            for (int k = 0; k < P; ++k)
                if (k >= jj && k < pw) sacc = fma(T[(i - t0) * P + k], L[(c0 + k) * ld + c0 + jj], sacc);
            L[i * ld + c0 + jj] = -sacc;
        }
        __syncthreads();
    }
    // Rinv = L^{-T} (upper), row-major
    for (int e = tid; e < w * w; e += blockDim.x) {
        const int r = e / w, c = e % w;
        Rinv[e] = (r <= c) ? L[c * ld + r] : 0.0;
    }
    if (tid == 0 && fail) status[0] = 1;
}

// ---------------------------------------------------------------------------
// Householder QR fallback (Eigen's makeHouseholder convention), one CTA
// ---------------------------------------------------------------------------
constexpr int kHhThreads = 512;

__device__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[i];
    return t;
}

__global__ void __launch_bounds__(kHhThreads) householder_kernel(const double* __restrict__ X, long long m, int w,
                                                                 long long ldx, double* __restrict__ Q,
                                                                 long long ldq, double* __restrict__ Wk,
                                                                 const int* __restrict__ pred,
                                                                 const int* __restrict__ status) {
    if (pred != nullptr && *pred == 0) return;
    if (status != nullptr && *status == 0) return;
    __shared__ double red[32];
    __shared__ double tau[kHhMax];
    const int tid = threadIdx.x;
    for (long long e = tid; e < m * w; e += blockDim.x) Wk[e] = X[(e / w) * ldx + e % w];
    __syncthreads();
    for (int j = 0; j < w; ++j) {
        double ts = 0.0;
        for (long long i = j + 1 + tid; i < m; i += blockDim.x) {
            const double v = Wk[i * w + j];
            ts = fma(v, v, ts);
        }
        const double tail_sq = block_sum(ts, red);
        const double c0 = Wk[static_cast<long long>(j) * w + j];
        double t, beta;
        if (tail_sq <= DBL_MIN) {
            t = 0.0;
            beta = c0;
            for (long long i = j + 1 + tid; i < m; i += blockDim.x) Wk[i * w + j] = 0.0;
        } else {
            beta = sqrt(c0 * c0 + tail_sq);
            if (c0 >= 0.0) beta = -beta;
            const double inv = 1.0 / (c0 - beta);
            for (long long i = j + 1 + tid; i < m; i += blockDim.x) Wk[i * w + j] *= inv;
            t = (beta - c0) / beta;
        }
        __syncthreads();
        if (tid == 0) {
            Wk[static_cast<long long>(j) * w + j] = beta;
            tau[j] = t;
        }
        __syncthreads();
        if (t != 0.0) {
            for (int c = j + 1; c < w; ++c) {
                double ds = 0.0;
                for (long long i = j + 1 + tid; i < m; i += blockDim.x) ds = fma(Wk[i * w + j], Wk[i * w + c], ds);
                double dot = block_sum(ds, red) + Wk[static_cast<long long>(j) * w + c];
                dot *= t;
                __syncthreads();
                if (tid == 0) Wk[static_cast<long long>(j) * w + c] -= dot;
                for (long long i = j + 1 + tid; i < m; i += blockDim.x) Wk[i * w + c] -= dot * Wk[i * w + j];
                __syncthreads();
            }
        }
    }
    // Q = H_0 ... H_{w-1} [I_w; 0]
    for (long long e = tid; e < m * w; e += blockDim.x) {
        const long long i = e / w, c = e % w;
        Q[i * ldq + c] = (i == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int j = w - 1; j >= 0; --j) {
        const double t = tau[j];
        if (t == 0.0) continue;
        for (int c = 0; c < w; ++c) {
            double ds = 0.0;
            for (long long i = j + 1 + tid; i < m; i += blockDim.x) ds = fma(Wk[i * w + j], Q[i * ldq + c], ds);
            double dot = block_sum(ds, red) + Q[static_cast<long long>(j) * ldq + c];
            dot *= t;
            __syncthreads();
            if (tid == 0) Q[static_cast<long long>(j) * ldq + c] -= dot;
            for (long long i = j + 1 + tid; i < m; i += blockDim.x) Q[i * ldq + c] -= dot * Wk[i * w + j];
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// single-CTA Jacobi eigensolver for the small symmetric matrices (r <= 112)
// ---------------------------------------------------------------------------

// Two-sided cyclic Jacobi for a symmetric r x r matrix (r <= RP <= 112), one
// CTA, A and V in (dynamic) shared memory: round-robin parallel ordering (the
// step's RP/2 pairs precomputed), the disjoint rotations of a step computed
// from (a_pp, a_qq, a_pq) alone, then applied to the rows and to the columns
// (and V) in barrier-separated phases; a warp per pair (two for RP > 64).  RP
// is a compile-time bucket, the matrix zero-padded to it (padding never
// rotates).  A pair below the absolute floor 1e-17 * max|a_ii| is rounding
// noise of a rank-deficient Gram and is not rotated.  Eigenvalues = diag(A),
// eigenvectors = columns of V, sorted descending (stable).
template <int RP>
struct JacSym {
    static constexpr int NP = RP / 2;
    static constexpr int WARPS = NP < 32 ? NP : 32;
    static constexpr int NT = 32 * WARPS;
    static constexpr size_t SMEM = sizeof(double) * 2 * RP * (RP + 1);  // A and V
};

template <int RP>
__global__ void __launch_bounds__(JacSym<RP>::NT) jacobi_sym_kernel(const double* __restrict__ G, int r,
                                                                    double* __restrict__ W,
                                                                    double* __restrict__ lambda) {
    constexpr int NP = JacSym<RP>::NP, WARPS = JacSym<RP>::WARPS, NT = JacSym<RP>::NT;
    extern __shared__ __align__(16) double jac_smem[];
    double(*A)[RP + 1] = reinterpret_cast<double(*)[RP + 1]>(jac_smem);
    double(*V)[RP + 1] = reinterpret_cast<double(*)[RP + 1]>(jac_smem + RP * (RP + 1));
    __shared__ double cs[NP][2];
    __shared__ unsigned char sched[RP - 1][NP][2];
    __shared__ double dg[RP];
    __shared__ int order[RP];
    __shared__ int rotated;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double tol = 4.0 * 2.220446049250313e-16;
    for (int e = tid; e < RP * RP; e += NT) {
        const int i = e / RP, j = e % RP;
        A[i][j] = (i < r && j < r) ? G[i * r + j] : 0.0;
        V[i][j] = (i == j) ? 1.0 : 0.0;
    }
    for (int e = tid; e < (RP - 1) * NP; e += NT) {
        const int step = e / NP, k = e % NP;
        const int a = k, b = RP - 1 - k;
        int p = (a == 0) ? 0 : 1 + (a - 1 + step) % (RP - 1);
        int q = (b == 0) ? 0 : 1 + (b - 1 + step) % (RP - 1);
        sched[step][k][0] = static_cast<unsigned char>(p < q ? p : q);
        sched[step][k][1] = static_cast<unsigned char>(p < q ? q : p);
    }
    __syncthreads();
    double dmax = 0.0;
    for (int i = 0; i < r; ++i) dmax = fmax(dmax, fabs(A[i][i]));
    const double afloor = 1e-17 * dmax;
    for (int sweep = 0; sweep < 60; ++sweep) {
        if (tid == 0) rotated = 0;
        __syncthreads();
        for (int step = 0; step < RP - 1; ++step) {
            if (lane == 0)
                for (int k = warp; k < NP; k += WARPS) {
                    const int p = sched[step][k][0], q = sched[step][k][1];
                    const double app = A[p][p], aqq = A[q][q], apq = A[p][q];
                    double c = 1.0, sn = 0.0;
                    if (apq != 0.0 && fabs(apq) > tol * sqrt(fabs(app) * fabs(aqq)) && fabs(apq) > afloor) {
                        const double tau = (aqq - app) / (2.0 * apq);
                        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = rsqrt(1.0 + t * t);
                        sn = t * c;
                        rotated = 1;
                    }
                    cs[k][0] = c;
                    cs[k][1] = sn;
                }
            __syncwarp();
            // rows p, q of A (this warp's pairs: disjoint from the others)
            for (int k = warp; k < NP; k += WARPS) {
                const double c = cs[k][0], sn = cs[k][1];
                if (sn == 0.0) continue;
                const int p = sched[step][k][0], q = sched[step][k][1];
                for (int j = lane; j < RP; j += 32) {
                    const double x = A[p][j], y = A[q][j];
                    A[p][j] = c * x - sn * y;
                    A[q][j] = sn * x + c * y;
                }
            }
            __syncthreads();
            // columns p, q of A and V
            for (int k = warp; k < NP; k += WARPS) {
                const double c = cs[k][0], sn = cs[k][1];
                if (sn == 0.0) continue;
                const int p = sched[step][k][0], q = sched[step][k][1];
                for (int i = lane; i < RP; i += 32) {
                    const double x = A[i][p], y = A[i][q];
                    A[i][p] = c * x - sn * y;
                    A[i][q] = sn * x + c * y;
                    const double vx = V[i][p], vy = V[i][q];
                    V[i][p] = c * vx - sn * vy;
                    V[i][q] = sn * vx + c * vy;
                }
            }
            __syncthreads();
        }
        if (!rotated) break;
    }
    if (tid < r) {
        dg[tid] = A[tid][tid];
        order[tid] = tid;
    }
    __syncthreads();
    if (tid == 0) {  // stable insertion sort, descending
        for (int i = 1; i < r; ++i) {
            const int o = order[i];
            int j = i - 1;
            while (j >= 0 && dg[order[j]] < dg[o]) {
                order[j + 1] = order[j];
                --j;
            }
            order[j + 1] = o;
        }
    }
    __syncthreads();
    for (int e = tid; e < r * r; e += NT) {
        const int i = e / r, j = e % r;
        W[i * r + j] = V[i][order[j]];
    }
    if (tid < r) lambda[tid] = dg[order[tid]];
}


// ---------------------------------------------------------------------------
// Cooperative one-sided Jacobi for larger Grams: columns of A (= G) and V live
// column-major in global memory (L2-resident up to r ~ 3000); each round of
// the round-robin tournament rotates rp/2 disjoint column pairs, one warp per
// pair, separated by a grid-wide barrier (all CTAs co-resident through a
// cooperative launch).  L1 is bypassed (__ldcg) so every round reads the
// previous round's columns.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = atomicAdd(gen, 0u);
        if (atomicAdd(count, 1u) == nblocks - 1) {
            atomicExch(count, 0u);
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (atomicAdd(gen, 0u) == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256) jacobi_coop_kernel(double* __restrict__ A, double* __restrict__ V, int rp,
                                                          int max_sweeps, unsigned* __restrict__ sync,
                                                          double* __restrict__ lambda) {
    const int lane = threadIdx.x & 31;
    const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    unsigned* count = sync;
    unsigned* gen = sync + 1;
    unsigned* rot = sync + 2;  // rot[0], rot[1]: rotations of the current / next sweep
    const double jtol = 8.0 * sqrt(static_cast<double>(rp)) * 1.1102230246251565e-16;
    // absolute floor: ||A||_F is invariant under the rotations; a pair whose
    // inner product is below (rounding x ||A||_F)^2 is left alone (columns
    // of negligible norm -- rank-deficient Grams -- never meet the relative
    // test and would burn every sweep)
    __shared__ double fro2_s;
    if (threadIdx.x == 0) fro2_s = 0.0;
    __syncthreads();
    {
        double part = 0.0;
        for (long long e = threadIdx.x; e < static_cast<long long>(rp) * rp; e += blockDim.x) {
            const double x = __ldcg(A + e);
            part = fma(x, x, part);
        }
        part = warp_sum(part);
        if (lane == 0) atomicAdd(&fro2_s, part);
    }
    __syncthreads();
    const double afloor = 1e-30 * fro2_s;
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        if (blockIdx.x == 0 && threadIdx.x == 0) rot[(sweep + 1) & 1] = 0u;
        for (int step = 0; step < rp - 1; ++step) {
            for (int k = gwarp; k < rp / 2; k += nwarps) {
                const int a = k, b = rp - 1 - k;
                int p = (a == 0) ? 0 : 1 + (a - 1 + step) % (rp - 1);
                int q = (b == 0) ? 0 : 1 + (b - 1 + step) % (rp - 1);
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                double* ap = A + static_cast<long long>(p) * rp;
                double* aq = A + static_cast<long long>(q) * rp;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int i = lane; i < rp; i += 32) {
                    const double x = __ldcg(ap + i), y = __ldcg(aq + i);
                    al = fma(x, x, al);
                    be = fma(y, y, be);
                    ga = fma(x, y, ga);
                }
                al = warp_sum(al);
                be = warp_sum(be);
                ga = warp_sum(ga);
                if (ga != 0.0 && fabs(ga) > jtol * sqrt(al * be) && fabs(ga) > afloor) {
                    const double zeta = (be - al) / (2.0 * ga);
                    const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                    double* vp = V + static_cast<long long>(p) * rp;
                    double* vq = V + static_cast<long long>(q) * rp;
                    for (int i = lane; i < rp; i += 32) {
                        const double x = __ldcg(ap + i), y = __ldcg(aq + i);
                        __stcg(ap + i, c * x - s * y);
                        __stcg(aq + i, s * x + c * y);
                        const double vx = __ldcg(vp + i), vy = __ldcg(vq + i);
                        __stcg(vp + i, c * vx - s * vy);
                        __stcg(vq + i, s * vx + c * vy);
                    }
                    if (lane == 0) atomicAdd(rot + (sweep & 1), 1u);
                }
            }
            grid_barrier(count, gen, gridDim.x);
        }
        if (atomicAdd(rot + (sweep & 1), 0u) == 0u) {
            if (blockIdx.x == 0 && threadIdx.x == 0) sync[4] = sweep + 1;
            break;
        }
        grid_barrier(count, gen, gridDim.x);
        if (blockIdx.x == 0 && threadIdx.x == 0) sync[4] = sweep + 1;
    }
    // eigenvalue j = sign(v_j . a_j) ||a_j||
    for (int j = gwarp; j < rp; j += nwarps) {
        const double* aj = A + static_cast<long long>(j) * rp;
        const double* vj = V + static_cast<long long>(j) * rp;
        double s = 0.0, d = 0.0;
        for (int i = lane; i < rp; i += 32) {
            const double x = __ldcg(aj + i);
            s = fma(x, x, s);
            d = fma(__ldcg(vj + i), x, d);
        }
        s = warp_sum(s);
        d = warp_sum(d);
        if (lane == 0) lambda[j] = (d < 0.0 ? -1.0 : 1.0) * sqrt(s);
    }
}

// ---------------------------------------------------------------------------
// Blocked one-sided Jacobi (the mid-size Grams, 112 < r <= ~6000): the
// columns of A (= G) and V are grouped into nb blocks of b columns; each step
// of the round-robin tournament over the blocks gives every CTA one block
// pair, which it stages in shared memory (2b columns of A and of V), sweeps
// with all 2b(2b-1)/2 column rotations (one warp per disjoint pair, a
// __syncthreads between the 2b-1 rounds) and writes back.  One grid barrier
// per step instead of one per column-pair round: nb - 1 = rp/b - 1 barriers
// a sweep rather than rp - 1, and the rotations read shared memory instead
// of L2.  Convergence: a sweep that rotated nothing (same relative test and
// absolute floor as jacobi_coop_kernel).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) jacobi_blk_kernel(double* __restrict__ A, double* __restrict__ V, int rp,
                                                         int b, int max_sweeps, unsigned* __restrict__ sync,
                                                         double* __restrict__ lambda) {
    extern __shared__ double jb_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int nb = rp / b, npair = nb / 2, w2 = 2 * b;
    const long long blk = static_cast<long long>(b) * rp;  // doubles per block
    double* sA = jb_smem;                                  // 2b columns x rp
    double* sV = jb_smem + 2 * blk;
    unsigned* count = sync;
    unsigned* gen = sync + 1;
    unsigned* rot = sync + 2;
    const double jtol = 8.0 * sqrt(static_cast<double>(rp)) * 1.1102230246251565e-16;
    __shared__ double fro2_s;
    __shared__ unsigned nrot_s;
    if (threadIdx.x == 0) fro2_s = 0.0;
    __syncthreads();
    {
        double part = 0.0;
        for (long long e = threadIdx.x; e < static_cast<long long>(rp) * rp; e += blockDim.x) {
            const double x = __ldcg(A + e);
            part = fma(x, x, part);
        }
        part = warp_sum(part);
        if (lane == 0) atomicAdd(&fro2_s, part);
    }
    __syncthreads();
    // absolute test: after rotations every column carries rounding of
    // ~eps ||G||_F, so a pair whose inner product is below
    // 8 eps ||G||_F (||a_p|| + ||a_q||) is left alone -- the rotation would
    // only mix rounding noise (the residual it removes is |ga| / (|l_p| +
    // |l_q|) <= 8 eps ||G||_F, the backward error of any stable eigensolver)
    const double afro = 8.0 * 1.1102230246251565e-16 * sqrt(fro2_s);
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
        if (blockIdx.x == 0 && threadIdx.x == 0) rot[(sweep + 1) & 1] = 0u;
        for (int step = 0; step < nb - 1; ++step) {
            for (int k = blockIdx.x; k < npair; k += gridDim.x) {
                const int a = k, bb = nb - 1 - k;
                const int P = (a == 0) ? 0 : 1 + (a - 1 + step) % (nb - 1);
                const int Q = (bb == 0) ? 0 : 1 + (bb - 1 + step) % (nb - 1);
                const double2* gA0 = reinterpret_cast<const double2*>(A + P * blk);
                const double2* gA1 = reinterpret_cast<const double2*>(A + Q * blk);
                const double2* gV0 = reinterpret_cast<const double2*>(V + P * blk);
                const double2* gV1 = reinterpret_cast<const double2*>(V + Q * blk);
                double2* s2A = reinterpret_cast<double2*>(sA);
                double2* s2V = reinterpret_cast<double2*>(sV);
                const long long h = blk / 2;  // blk is even (rp is)
                for (long long e = threadIdx.x; e < h; e += blockDim.x) {
                    s2A[e] = __ldcg(gA0 + e);
                    s2A[h + e] = __ldcg(gA1 + e);
                    s2V[e] = __ldcg(gV0 + e);
                    s2V[h + e] = __ldcg(gV1 + e);
                }
                if (threadIdx.x == 0) nrot_s = 0u;
                __syncthreads();
                for (int t = 0; t < w2 - 1; ++t) {
                    for (int i = warp; i < b; i += nwarps) {
                        const int x = i, y = w2 - 1 - i;
                        int p = (x == 0) ? 0 : 1 + (x - 1 + t) % (w2 - 1);
                        int q = (y == 0) ? 0 : 1 + (y - 1 + t) % (w2 - 1);
                        if (p > q) {
                            const int tmp = p;
                            p = q;
                            q = tmp;
                        }
                        double* ap = sA + static_cast<long long>(p) * rp;
                        double* aq = sA + static_cast<long long>(q) * rp;
                        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll 4
                        for (int r = lane; r < rp; r += 32) {
                            const double u = ap[r], v = aq[r];
                            al = fma(u, u, al);
                            be = fma(v, v, be);
                            ga = fma(u, v, ga);
                        }
                        al = warp_sum(al);
                        be = warp_sum(be);
                        ga = warp_sum(ga);
                        if (ga != 0.0 && fabs(ga) > jtol * sqrt(al * be) && fabs(ga) > afro * (sqrt(al) + sqrt(be))) {
                            const double zeta = (be - al) / (2.0 * ga);
                            const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                            const double c = 1.0 / sqrt(1.0 + tt * tt), sn = c * tt;
                            double* vp = sV + static_cast<long long>(p) * rp;
                            double* vq = sV + static_cast<long long>(q) * rp;
#pragma unroll 4
                            for (int r = lane; r < rp; r += 32) {
                                const double u = ap[r], v = aq[r];
                                ap[r] = c * u - sn * v;
                                aq[r] = sn * u + c * v;
                                const double vu = vp[r], vv = vq[r];
                                vp[r] = c * vu - sn * vv;
                                vq[r] = sn * vu + c * vv;
                            }
                            if (lane == 0) atomicAdd(&nrot_s, 1u);
                        }
                    }
                    __syncthreads();
                }
                double2* oA0 = reinterpret_cast<double2*>(A + P * blk);
                double2* oA1 = reinterpret_cast<double2*>(A + Q * blk);
                double2* oV0 = reinterpret_cast<double2*>(V + P * blk);
                double2* oV1 = reinterpret_cast<double2*>(V + Q * blk);
                for (long long e = threadIdx.x; e < h; e += blockDim.x) {
                    __stcg(oA0 + e, s2A[e]);
                    __stcg(oA1 + e, s2A[h + e]);
                    __stcg(oV0 + e, s2V[e]);
                    __stcg(oV1 + e, s2V[h + e]);
                }
                if (threadIdx.x == 0 && nrot_s) atomicAdd(rot + (sweep & 1), nrot_s);
                __syncthreads();
            }
            grid_barrier(count, gen, gridDim.x);
        }
        if (atomicAdd(rot + (sweep & 1), 0u) == 0u) break;
        grid_barrier(count, gen, gridDim.x);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) sync[4] = sweep + 1;
    // eigenvalue j = sign(v_j . a_j) ||a_j||
    const int gwarp = blockIdx.x * nwarps + warp, gw = gridDim.x * nwarps;
    for (int j = gwarp; j < rp; j += gw) {
        const double* aj = A + static_cast<long long>(j) * rp;
        const double* vj = V + static_cast<long long>(j) * rp;
        double s = 0.0, d = 0.0;
        for (int i = lane; i < rp; i += 32) {
            const double x = __ldcg(aj + i);
            s = fma(x, x, s);
            d = fma(__ldcg(vj + i), x, d);
        }
        s = warp_sum(s);
        d = warp_sum(d);
        if (lane == 0) lambda[j] = (d < 0.0 ? -1.0 : 1.0) * sqrt(s);
    }
}

// W (r x r row-major) column j <- column perm[j] of the column-major V (ld)
__global__ void gather_eigvecs_kernel(const double* __restrict__ Vcm, long long ldv, const int* __restrict__ perm,
                                      long long r, double* __restrict__ W) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= r * r) return;
    const long long i = e / r, j = e % r;
    W[i * r + j] = Vcm[perm[j] * ldv + i];
}

__global__ void init_jacobi_kernel(const double* __restrict__ G, long long r, long long rp, double* __restrict__ A,
                                   double* __restrict__ V) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= rp * rp) return;
    const long long j = e / rp, i = e % rp;  // column-major (i, j)
    A[e] = (i < r && j < r) ? G[i * r + j] : 0.0;
    V[e] = (i == j) ? 1.0 : 0.0;
}

// ---------------------------------------------------------------------------
// small utilities
// ---------------------------------------------------------------------------
__global__ void col_sumsq_partial_kernel(const double* __restrict__ X, long long rows, long long cols, long long ld,
                                         long long rows_per_block, double* __restrict__ partial) {
    const long long j = blockIdx.x * 32LL + (threadIdx.x & 31);
    const int ty = threadIdx.x >> 5;  // 8 row lanes
    __shared__ double red[8][33];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const long long r0 = blockIdx.y * rows_per_block;
    const long long r1 = min(rows, r0 + rows_per_block);
    if (j < cols) {
        long long i = r0 + ty;
        for (; i + 24 < r1; i += 32) {  // four independent chains
            const double a = X[i * ld + j], b = X[(i + 8) * ld + j];
            const double c = X[(i + 16) * ld + j], d = X[(i + 24) * ld + j];
            s0 = fma(a, a, s0);
            s1 = fma(b, b, s1);
            s2 = fma(c, c, s2);
            s3 = fma(d, d, s3);
        }
        for (; i < r1; i += 8) {
            const double v = X[i * ld + j];
            s0 = fma(v, v, s0);
        }
    }
    red[ty][threadIdx.x & 31] = (s0 + s1) + (s2 + s3);
    __syncthreads();
    if (ty == 0 && j < cols) {
        double t = 0.0;
        for (int q = 0; q < 8; ++q) t += red[q][threadIdx.x & 31];
        partial[blockIdx.y * cols + j] = t;
    }
}

// Single-launch variant: every (column block, row part) CTA writes its
// partial sums; the last CTA to arrive for a column block (arrival counter)
// adds the parts in part order — the same fixed order as the two-kernel
// path, so the result is deterministic — and resets the counter.
__global__ void col_sumsq_fused_kernel(const double* __restrict__ X, long long rows, long long cols, long long ld,
                                       long long rows_per_block, double* __restrict__ partial,
                                       double* __restrict__ out, unsigned* __restrict__ tickets) {
    const long long j = blockIdx.x * 32LL + (threadIdx.x & 31);
    const int ty = threadIdx.x >> 5;  // 8 row lanes
    __shared__ double red[8][33];
    __shared__ bool last;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const long long r0 = blockIdx.y * rows_per_block;
    const long long r1 = min(rows, r0 + rows_per_block);
    if (j < cols) {
        long long i = r0 + ty;
        for (; i + 24 < r1; i += 32) {
            const double a = X[i * ld + j], b = X[(i + 8) * ld + j];
            const double c = X[(i + 16) * ld + j], d = X[(i + 24) * ld + j];
            s0 = fma(a, a, s0);
            s1 = fma(b, b, s1);
            s2 = fma(c, c, s2);
            s3 = fma(d, d, s3);
        }
        for (; i < r1; i += 8) {
            const double v = X[i * ld + j];
            s0 = fma(v, v, s0);
        }
    }
    red[ty][threadIdx.x & 31] = (s0 + s1) + (s2 + s3);
    __syncthreads();
    if (ty == 0 && j < cols) {
        double t = 0.0;
        for (int q = 0; q < 8; ++q) t += red[q][threadIdx.x & 31];
        partial[blockIdx.y * cols + j] = t;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(tickets + blockIdx.x, 1u) == gridDim.y - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (ty == 0 && j < cols) {
        double t = 0.0;
        for (unsigned p = 0; p < gridDim.y; ++p) t += __ldcg(partial + p * cols + j);
        out[j] = t;
    }
    if (threadIdx.x == 0) tickets[blockIdx.x] = 0;
}

__global__ void col_sumsq_finish_kernel(const double* __restrict__ partial, long long cols, int nparts,
                                        double* __restrict__ out) {
    const long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (j >= cols) return;
    double t = 0.0;
    for (int p = 0; p < nparts; ++p) t += partial[p * cols + j];
    out[j] = t;
}

__global__ void scale_cols_kernel(double* X, long long rows, long long cols, long long ld, const double* s) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= rows * cols) return;
    const long long i = e / cols, j = e % cols;
    X[i * ld + j] *= s[j];
}

__global__ void copy2d_kernel(const double* __restrict__ src, long long lds, double* __restrict__ dst, long long ldd,
                              long long rows, long long cols, const int* __restrict__ pred) {
    if (pred != nullptr && *pred == 0) return;
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= rows * cols) return;
    const long long i = e / cols, j = e % cols;
    dst[i * ldd + j] = src[i * lds + j];
}

__global__ void fill_kernel(double* p, long long n, double v) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e < n) p[e] = v;
}

__global__ void transpose_kernel(const double* __restrict__ in, long long rows, long long cols, long long ldi,
                                 double* __restrict__ out) {
    __shared__ double tile[32][33];
    const long long bx = blockIdx.x * 32LL, by = blockIdx.y * 32LL;
    for (int t = threadIdx.y; t < 32; t += blockDim.y) {
        const long long i = by + t, j = bx + threadIdx.x;
        if (i < rows && j < cols) tile[t][threadIdx.x] = in[i * ldi + j];
    }
    __syncthreads();
    for (int t = threadIdx.y; t < 32; t += blockDim.y) {
        const long long j = bx + t, i = by + threadIdx.x;
        if (i < rows && j < cols) out[j * rows + i] = tile[threadIdx.x][t];
    }
}

__global__ void permute_cols_kernel(const double* __restrict__ W, long long rows, long long ldw,
                                    const int* __restrict__ perm, long long kcols, double* __restrict__ W2,
                                    long long ldw2) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= rows * kcols) return;
    const long long i = e / kcols, j = e % kcols;
    W2[i * ldw2 + j] = W[i * ldw + perm[j]];
}

__global__ void set_identity_cols_kernel(double* Z, long long rows, long long ld, long long s) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= rows * s) return;
    const long long i = e / s, j = e % s;
    Z[i * ld + j] = (i == j) ? 1.0 : 0.0;
}

__global__ void sub_scaled_cols_kernel(double* Y, const double* __restrict__ X, long long rows, long long cols,
                                       long long ld, const double* __restrict__ theta) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= rows * cols) return;
    const long long i = e / cols, j = e % cols;
    Y[i * ld + j] -= X[i * ld + j] * theta[j];
}

inline unsigned nblk(i64 n, int bs = 256) { return static_cast<unsigned>(std::max<i64>(1, (n + bs - 1) / bs)); }

}  // namespace

// ---------------------------------------------------------------------------
// Dense corner of a split sparse product (engine.cpp), in two launches so the
// tensor-core part can run on a helper stream while the gather kernel of the
// cold entries runs on the caller's: dense_block_mm computes the split-K
// partials of op(D) B[brow, :] (M x N; D the R x C dense block, op =
// transpose for Y^T X; the B-row gather folded into the cp.async loads) into
// ws on stream s and returns the split count; dense_block_add then adds
// their fixed-order sum into out[orow[i], :] (deterministic).  alg_bytes /
// alg_flops: the algorithmic cost of the sparse entries the block stands for
// (the SpMM roofline's accounting).  Operands must be 16-byte aligned rows
// (returns 0 otherwise, nothing launched).
int dense_block_mm(svt_ctx* ctx, cudaStream_t s, int cls, bool transA, i64 M, i64 N, i64 K, const double* D,
                   i64 ldd, const double* B, i64 ldb, const int* brow, DevBuf<double>& ws, double alg_bytes,
                   double alg_flops) {
    if (M <= 0 || N <= 0 || K <= 0) return 0;
    if ((ldd % 2) != 0 || (reinterpret_cast<uintptr_t>(D) % 16) != 0 || (reinterpret_cast<uintptr_t>(B) % 8) != 0)
        return 0;
    // 8-byte operand copies when the panel rows are not 16-byte aligned
    const bool b8 = (ldb % 2) != 0 || (reinterpret_cast<uintptr_t>(B) % 16) != 0;
    LaunchScope ls(ctx, cls, alg_bytes, alg_flops, s);
    if (cutlass_corner_enabled()) {
        const int S = cutlass_dense_block(ctx, s, transA, M, N, K, D, ldd, B, ldb, brow, ws);
        if (S > 0) return S;
    }
#define SVT_DB(BN_)                                                                                       \
    return transA ? (b8 ? dense_block_launch<BN_, true, true>(ctx, s, M, N, K, D, ldd, B, ldb, brow, ws)   \
                        : dense_block_launch<BN_, true, false>(ctx, s, M, N, K, D, ldd, B, ldb, brow, ws)) \
                  : (b8 ? dense_block_launch<BN_, false, true>(ctx, s, M, N, K, D, ldd, B, ldb, brow, ws)  \
                        : dense_block_launch<BN_, false, false>(ctx, s, M, N, K, D, ldd, B, ldb, brow, ws))
    if (N <= 32) SVT_DB(32);
    if (N <= 64) SVT_DB(64);
    SVT_DB(128);
#undef SVT_DB
}

void dense_block_add(svt_ctx* ctx, cudaStream_t s, int cls, i64 M, i64 N, int S, const DevBuf<double>& ws,
                     const int* orow, double* out, i64 ldo) {
    if (M <= 0 || N <= 0 || S <= 0) return;
    LaunchScope ls(ctx, cls, 0.0, 0.0, s);
    block_scatter_add_kernel<<<static_cast<unsigned>((M * N + 255) / 256), 256, 0, s>>>(M, N, S, ws.get(), orow, out,
                                                                                       ldo);
}

void gemm(svt_ctx* ctx, int cls, bool transA, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
          const double* B, i64 ldb, double beta, double* C, i64 ldc, const int* pred) {
    if (M <= 0 || N <= 0) return;
    // a predicated product (second Gram-Schmidt pass, re-projection check)
    // usually exits at once: it is timed but its bytes / flops are not
    // counted (they are unknown when it is queued)
    LaunchScope ls(ctx, cls, pred ? 0.0 : 8.0 * (M * K + K * N + M * N * (beta != 0.0 ? 2 : 1)),
                   pred ? 0.0 : 2.0 * M * N * K);
    if (K <= 0) {
        scale2d_kernel<<<nblk(M * N), 256, 0, ctx->stream>>>(C, M, N, ldc, beta, pred);
        return;
    }
    if (N <= 16) {
        if (transA && A == B && lda == ldb && M == N && M <= 12 && alpha == 1.0 && beta == 0.0 && ldc == N) {
            gram_sym_launch(ctx, K, static_cast<int>(M), A, lda, C, false, nullptr, nullptr, pred);
            return;
        }
        if (!transA && K <= 16) {
            smallk_nn_launch(ctx, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, pred);
            return;
        }
        if (transA && M <= kTinyMaxW && alpha == 1.0 && beta == 0.0 && ldc == N) {
            tiny_tn_launch(ctx, K, static_cast<int>(M), static_cast<int>(N), A, lda, B, ldb, C, false, nullptr,
                           nullptr, pred);
            return;
        }
        switch (N) {
#define SVT_CASE(NN)                                                                            \
    case NN:                                                                                    \
        if (transA)                                                                             \
            skinny_tn_launch<NN>(ctx, M, K, alpha, A, lda, B, ldb, beta, C, ldc, pred);         \
        else                                                                                    \
            skinny_nn_launch<NN>(ctx, M, K, alpha, A, lda, B, ldb, beta, C, ldc, pred);         \
        return;
            SVT_CASE(1) SVT_CASE(2) SVT_CASE(3) SVT_CASE(4) SVT_CASE(5) SVT_CASE(6) SVT_CASE(7) SVT_CASE(8)
            SVT_CASE(9) SVT_CASE(10) SVT_CASE(11) SVT_CASE(12) SVT_CASE(13) SVT_CASE(14) SVT_CASE(15) SVT_CASE(16)
#undef SVT_CASE
            default:
                break;
        }
    }
    // FP64 tensor cores (DMMA) for everything wider than the skinny paths.
    // Tall unpredicated NN products (Gram-Schmidt X - Q C, CholQR X R^-1):
    // the CUTLASS 64 x 32 multistage template (SVTB_CUTLASS_NN=0: our 64 x 128
    // kernel)
    if (!transA && pred == nullptr && N > 32 && M >= 64LL * ctx->num_sms && cutlass_nn_enabled() &&
        cutlass_gemm_nn(ctx, ctx->stream, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc))
        return;
    // wide TN contractions (Gram-Schmidt coefficients B T / Q^T X, finalize
    // B W): the CUTLASS template with parallel split-K (SVTB_CUTLASS_TN=0:
    // our kernel).  The W x W Gram blocks stay on our split-K kernel.
    if (transA && pred == nullptr && N > 32 && M >= cutlass_tn_min_m() && K >= 2048 && cutlass_tn_enabled()) {
        ensure_partial(ctx, 1);
        if (cutlass_gemm_tn(ctx, ctx->stream, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ctx->ws_partial)) return;
    }
    if (N <= 32)
        dmma_launch<32>(ctx, transA, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, pred);
    else if (N <= 64)
        dmma_launch<64>(ctx, transA, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, pred);
    else
        dmma_launch<128>(ctx, transA, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, pred);
}

void gram_chol(svt_ctx* ctx, const double* X, i64 ldx, i64 m, i64 w, double* G, double* Rinv, int* status,
               const int* pred) {
    if (w > kTinyMaxW) throw std::invalid_argument("gram_chol: panel wider than 16");
    LaunchScope ls(ctx, K_QR, 8.0 * m * w, 1.0 * m * w * w);
    if (w <= 12)
        gram_sym_launch(ctx, m, static_cast<int>(w), X, ldx, G, true, Rinv, status, pred);
    else
        tiny_tn_launch(ctx, m, static_cast<int>(w), static_cast<int>(w), X, ldx, X, ldx, G, true, Rinv, status, pred);
}

void sumsq(svt_ctx* ctx, const double* X, i64 rows, i64 cols, i64 ld, double* d_out, int op, const int* pred) {
    ctx->ws_partial2.ensure(kRedBlocks);
    const i64 tot = rows * cols;
    if (tot <= 0) {
        LaunchScope ls(ctx, K_OTHER, 0.0, 0.0);
        finish_kernel<<<1, 32, 0, ctx->stream>>>(ctx->ws_partial2.get(), 0, d_out, op, pred);
        return;
    }
    const int blocks = static_cast<int>(std::min<i64>(kRedBlocks, (tot + 255) / 256));
    LaunchScope ls(ctx, K_OTHER, 8.0 * tot, 2.0 * tot);
    sumsq_partial_kernel<<<blocks, 256, 0, ctx->stream>>>(X, rows, cols, ld, ctx->ws_partial2.get(), pred);
    finish_kernel<<<1, 32, 0, ctx->stream>>>(ctx->ws_partial2.get(), blocks, d_out, op, pred);
}

void maxabs(svt_ctx* ctx, const double* X, i64 rows, i64 cols, i64 ld, double diag_shift, double* d_out) {
    ctx->ws_partial2.ensure(kRedBlocks);
    const i64 tot = rows * cols;
    const int blocks = static_cast<int>(std::max<i64>(1, std::min<i64>(kRedBlocks, (tot + 255) / 256)));
    LaunchScope ls(ctx, K_OTHER, 8.0 * tot, 0.0);
    maxabs_partial_kernel<<<blocks, 256, 0, ctx->stream>>>(X, rows, cols, ld, diag_shift, ctx->ws_partial2.get());
    finish_kernel<<<1, 32, 0, ctx->stream>>>(ctx->ws_partial2.get(), blocks, d_out, 2, nullptr);
}

void block_flags(svt_ctx* ctx, const double* after, const double* before, const double* proj, int K, int w,
                 double thr2, int mode, const int* gate, int* flag) {
    LaunchScope ls(ctx, K_OTHER, 0.0, 0.0);
    block_flags_kernel<<<1, 32, 0, ctx->stream>>>(after, before, proj, K, w, thr2, mode, gate, flag);
}

void set_flag(svt_ctx* ctx, const double* a, const double* b, double coef, int mode, int* flag) {
    LaunchScope ls(ctx, K_OTHER, 0.0, 0.0);
    set_flag_kernel<<<1, 1, 0, ctx->stream>>>(a, b, coef, mode, flag);
}

void chol_rinv(svt_ctx* ctx, const double* G, i64 w, double* Rinv, int* status, const int* pred) {
    if (w > kCholMax) throw std::invalid_argument("chol_rinv: panel wider than 128");
    const size_t smem = sizeof(double) * static_cast<size_t>(w * (w + 1) + w + w * kCholPanel);
    static bool attr_set = false;
    if (!attr_set) {
        SVT_CUDA(cudaFuncSetAttribute(
            chol_rinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
            static_cast<int>(sizeof(double) * (kCholMax * (kCholMax + 1) + kCholMax + kCholMax * kCholPanel))));
        attr_set = true;
    }
    LaunchScope ls(ctx, K_QR, 16.0 * w * w, w * w * w / 3.0);
    chol_rinv_kernel<<<1, 512, smem, ctx->stream>>>(G, static_cast<int>(w), Rinv, status, pred);
}

void householder_qr(svt_ctx* ctx, const double* X, i64 m, i64 w, i64 ldx, double* Q, i64 ldq, double* work,
                    const int* pred, const int* status) {
    if (w > kHhMax) throw std::invalid_argument("householder_qr: panel wider than 64");
    LaunchScope ls(ctx, K_QR, 0.0, 4.0 * m * w * w);
    householder_kernel<<<1, kHhThreads, 0, ctx->stream>>>(X, m, static_cast<int>(w), ldx, Q, ldq, work, pred,
                                                          status);
}

template <int RP>
void jacobi_sym_launch(svt_ctx* ctx, const double* G, int r, double* W, double* lambda) {
    constexpr size_t smem = JacSym<RP>::SMEM;
    if (smem > 48 * 1024) {
        static bool attr = false;
        if (!attr) {
            SVT_CUDA(cudaFuncSetAttribute(jacobi_sym_kernel<RP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem)));
            attr = true;
        }
    }
    jacobi_sym_kernel<RP><<<1, JacSym<RP>::NT, smem, ctx->stream>>>(G, r, W, lambda);
}

// single-CTA two-sided Jacobi in shared memory for r <= kJacSymMax
constexpr int kJacSymMax = 112;
void launch_jacobi_sym(svt_ctx* ctx, const double* G, int r, double* W, double* lambda) {
    if (r <= 8) jacobi_sym_launch<8>(ctx, G, r, W, lambda);
    else if (r <= 16) jacobi_sym_launch<16>(ctx, G, r, W, lambda);
    else if (r <= 24) jacobi_sym_launch<24>(ctx, G, r, W, lambda);
    else if (r <= 32) jacobi_sym_launch<32>(ctx, G, r, W, lambda);
    else if (r <= 40) jacobi_sym_launch<40>(ctx, G, r, W, lambda);
    else if (r <= 48) jacobi_sym_launch<48>(ctx, G, r, W, lambda);
    else if (r <= 64) jacobi_sym_launch<64>(ctx, G, r, W, lambda);
    else if (r <= 80) jacobi_sym_launch<80>(ctx, G, r, W, lambda);
    else if (r <= 96) jacobi_sym_launch<96>(ctx, G, r, W, lambda);
    else jacobi_sym_launch<112>(ctx, G, r, W, lambda);
}

void sym_eig(svt_ctx* ctx, double* G, i64 r, double* W, double* lambda) {
    if (r <= 0) return;
    if (r <= kJacSymMax) {
        LaunchScope ls(ctx, K_FINAL, 16.0 * r * r, 0.0);
        launch_jacobi_sym(ctx, G, static_cast<int>(r), W, lambda);
        return;
    }
    // Larger Grams: cooperative multi-CTA one-sided Jacobi, blocked with the
    // block pairs staged in shared memory while 2b columns of A and V fit
    // (b chosen for >= 32 block pairs a step), else column pairs in L2.
    constexpr i64 kJbSmem = 200 * 1024;
    i64 bsz = std::min<i64>(16, kJbSmem / (32 * (r + 1)));
    bsz = std::min<i64>(bsz, std::max<i64>(1, r / 64));
    if (const char* e = std::getenv("SVTB_JACOBI_B")) {  // tuning: block width override (must fit shared memory)
        const i64 want = std::atoll(e);
        if (want >= 1 && 32 * want * (r + 2 * want) <= kJbSmem) bsz = want;
    }
    const bool blocked = bsz >= 1 && std::getenv("SVTB_JACOBI_SCALAR") == nullptr;
    const i64 rp = blocked ? (r + 2 * bsz - 1) / (2 * bsz) * (2 * bsz) : (r + 1) & ~1LL;
    // floor at a 1056-wide problem (the dense-Gram finalize range): the
    // basis grows every SVT iteration and each regrow is a device-wide sync
    constexpr i64 kEigFloor = 1056;
    ctx->ws_eig.ensure(static_cast<size_t>(std::max(2 * rp * rp + rp, 2 * kEigFloor * kEigFloor + kEigFloor)));
    ctx->ws_info.ensure(8);
    double* A = ctx->ws_eig.get();
    double* V = A + rp * rp;
    double* lam_u = V + rp * rp;
    SVT_CUDA(cudaMemsetAsync(ctx->ws_info.get(), 0, 8 * sizeof(int), ctx->stream));
    {
        LaunchScope ls(ctx, K_FINAL, 16.0 * rp * rp, 0.0);
        init_jacobi_kernel<<<nblk(rp * rp), 256, 0, ctx->stream>>>(G, r, rp, A, V);
    }
    int per_sm = 0, grid = 1;
    int rpi = static_cast<int>(rp), sweeps = 40;
    unsigned* sync = reinterpret_cast<unsigned*>(ctx->ws_info.get());
    if (blocked) {
        int bi = static_cast<int>(bsz);
        const size_t smem = static_cast<size_t>(4 * bsz * rp) * sizeof(double);
        SVT_CUDA(cudaFuncSetAttribute(jacobi_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        SVT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_blk_kernel, 256, smem));
        const i64 npair = rp / bsz / 2;
        grid = static_cast<int>(std::max<i64>(1, std::min<i64>(npair, std::max(1, per_sm) * ctx->num_sms)));
        void* args[] = {&A, &V, &rpi, &bi, &sweeps, &sync, &lam_u};
        LaunchScope ls(ctx, K_FINAL, 0.0, 6.0 * rp * rp * rp * 8);
        SVT_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(jacobi_blk_kernel), grid, 256, args, smem,
                                             ctx->stream));
    } else {
        SVT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_coop_kernel, 256, 0));
        const int want = static_cast<int>(std::min<i64>(std::max(1, per_sm) * ctx->num_sms, (rp / 2 + 7) / 8));
        grid = std::max(1, std::min(want, std::max(1, per_sm) * ctx->num_sms));
        void* args[] = {&A, &V, &rpi, &sweeps, &sync, &lam_u};
        LaunchScope ls(ctx, K_FINAL, 0.0, 6.0 * rp * rp * rp * 8);
        SVT_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(jacobi_coop_kernel), grid, 256, args, 0,
                                             ctx->stream));
    }
    // sort descending on the host (r values), gather the eigenvectors
    std::vector<double> lh(static_cast<size_t>(rp));
    SVT_CUDA(cudaMemcpyAsync(lh.data(), lam_u, sizeof(double) * rp, cudaMemcpyDeviceToHost, ctx->stream));
    sync_stream(ctx);
    if (std::getenv("SVTB_DEBUG_JACOBI")) {
        unsigned sw = 0;
        SVT_CUDA(cudaMemcpy(&sw, sync + 4, sizeof(unsigned), cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "[jacobi] r=%lld rp=%lld b=%lld grid=%d sweeps=%u\n", static_cast<long long>(r),
                     static_cast<long long>(rp), static_cast<long long>(blocked ? bsz : 0), grid, sw);
    }
    std::vector<int> perm(static_cast<size_t>(r));
    for (i64 j = 0; j < r; ++j) perm[static_cast<size_t>(j)] = static_cast<int>(j);
    // the padded zero columns (if any) are indices >= r and are excluded
    std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return lh[x] > lh[y]; });
    std::vector<double> ls_sorted(static_cast<size_t>(r));
    for (i64 j = 0; j < r; ++j) ls_sorted[static_cast<size_t>(j)] = lh[static_cast<size_t>(perm[static_cast<size_t>(j)])];
    // context workspace: a per-call buffer would cudaFree (a device-wide
    // synchronisation) on every eigensolve
    ctx->ws_perm.ensure(static_cast<size_t>(r));
    int* dperm_p = ctx->ws_perm.get();
    SVT_CUDA(cudaMemcpyAsync(dperm_p, perm.data(), sizeof(int) * r, cudaMemcpyHostToDevice, ctx->stream));
    SVT_CUDA(cudaMemcpyAsync(lambda, ls_sorted.data(), sizeof(double) * r, cudaMemcpyHostToDevice, ctx->stream));
    {
        LaunchScope ls(ctx, K_FINAL, 16.0 * r * r, 0.0);
        gather_eigvecs_kernel<<<nblk(r * r), 256, 0, ctx->stream>>>(V, rp, dperm_p, r, W);
    }
    sync_stream(ctx);
}

void col_sumsq(svt_ctx* ctx, const double* X, i64 rows, i64 cols, i64 ld, double* out) {
    if (cols <= 0) return;
    // ~4 CTAs per SM in total over the column blocks x row parts
    const i64 xblk = (cols + 31) / 32;
    const i64 parts_want = std::max<i64>(1, (4 * ctx->num_sms + xblk - 1) / xblk);
    const i64 rpb = std::max<i64>(64, (rows + parts_want - 1) / parts_want);
    const i64 nparts = std::max<i64>(1, (rows + rpb - 1) / rpb);
    ctx->ws_partial2.ensure(static_cast<size_t>(nparts * cols));
    LaunchScope ls(ctx, K_OTHER, 8.0 * rows * cols, 2.0 * rows * cols);
    dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>(nparts));
    if (ctx->d_tickets.get() != nullptr && static_cast<size_t>(grid.x) <= kTickets) {
        col_sumsq_fused_kernel<<<grid, 256, 0, ctx->stream>>>(X, rows, cols, ld, rpb, ctx->ws_partial2.get(), out,
                                                              ctx->d_tickets.get());
        return;
    }
    col_sumsq_partial_kernel<<<grid, 256, 0, ctx->stream>>>(X, rows, cols, ld, rpb, ctx->ws_partial2.get());
    col_sumsq_finish_kernel<<<nblk(cols), 256, 0, ctx->stream>>>(ctx->ws_partial2.get(), cols,
                                                                 static_cast<int>(nparts), out);
}

void scale_cols(svt_ctx* ctx, double* X, i64 rows, i64 cols, i64 ld, const double* s) {
    if (rows * cols <= 0) return;
    LaunchScope ls(ctx, K_OTHER, 16.0 * rows * cols, 0.0);
    scale_cols_kernel<<<nblk(rows * cols), 256, 0, ctx->stream>>>(X, rows, cols, ld, s);
}

void copy2d(svt_ctx* ctx, const double* src, i64 lds, double* dst, i64 ldd, i64 rows, i64 cols, const int* pred) {
    if (rows * cols <= 0) return;
    LaunchScope ls(ctx, K_OTHER, 16.0 * rows * cols, 0.0);
    copy2d_kernel<<<nblk(rows * cols), 256, 0, ctx->stream>>>(src, lds, dst, ldd, rows, cols, pred);
}

__global__ void cheb_combine_kernel(double* out, const double* __restrict__ GY, const double* __restrict__ Y,
                                    const double* Xp, long long count, double c, double alpha, double beta) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= count) return;
    double v = alpha * (GY[e] - c * Y[e]);
    if (Xp != nullptr) v -= beta * Xp[e];
    out[e] = v;
}

void cheb_combine(svt_ctx* ctx, double* out, const double* GY, const double* Y, const double* Xp, i64 count,
                  double c, double alpha, double beta) {
    if (count <= 0) return;
    LaunchScope ls(ctx, K_FINAL, 32.0 * count, 4.0 * count);
    cheb_combine_kernel<<<nblk(count), 256, 0, ctx->stream>>>(out, GY, Y, beta != 0.0 ? Xp : nullptr, count, c,
                                                              alpha, beta);
}

void set_identity_cols(svt_ctx* ctx, double* Z, i64 rows, i64 ld, i64 s) {
    if (rows * s <= 0) return;
    LaunchScope ls(ctx, K_OTHER, 8.0 * rows * s, 0.0);
    set_identity_cols_kernel<<<nblk(rows * s), 256, 0, ctx->stream>>>(Z, rows, ld, s);
}

void sub_scaled_cols(svt_ctx* ctx, double* Y, const double* X, i64 rows, i64 cols, i64 ld, const double* theta) {
    if (rows * cols <= 0) return;
    LaunchScope ls(ctx, K_OTHER, 24.0 * rows * cols, 2.0 * rows * cols);
    sub_scaled_cols_kernel<<<nblk(rows * cols), 256, 0, ctx->stream>>>(Y, X, rows, cols, ld, theta);
}

void fill(svt_ctx* ctx, double* p, i64 n, double v) {
    if (n <= 0) return;
    LaunchScope ls(ctx, K_OTHER, 8.0 * n, 0.0);
    fill_kernel<<<nblk(n), 256, 0, ctx->stream>>>(p, n, v);
}

void transpose(svt_ctx* ctx, const double* in, i64 rows, i64 cols, i64 ldi, double* out) {
    if (rows * cols <= 0) return;
    LaunchScope ls(ctx, K_OTHER, 16.0 * rows * cols, 0.0);
    dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, ctx->stream>>>(in, rows, cols, ldi, out);
}

void permute_cols(svt_ctx* ctx, const double* W, i64 rows, i64 ldw, const int* perm, i64 kcols, double* W2,
                  i64 ldw2) {
    if (rows * kcols <= 0) return;
    LaunchScope ls(ctx, K_OTHER, 16.0 * rows * kcols, 0.0);
    permute_cols_kernel<<<nblk(rows * kcols), 256, 0, ctx->stream>>>(W, rows, ldw, perm, kcols, W2, ldw2);
}

}  // namespace svtb
