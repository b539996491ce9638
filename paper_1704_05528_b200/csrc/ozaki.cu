// FP64 contractions on the INT8 tensor cores (tcgen05.mma kind::i8), by the
// Ozaki splitting scheme.  B200 runs FP64 matrix math at ~36 TF/s (DMMA) but
// INT8 at ~4.5 POPS: C = A^T B in FP64 is rebuilt exactly from integer
// products of 7-bit digit slices.
//
//   x = 2^e * sum_{p=1..S} d_p 2^{-7p},  d_p in [-127, 127]
//
// with one exponent e per column of A (output row) and per column of B
// (output column), chosen so that |x| 2^{-e} < 1 for every entry of the
// column; the digits are the exact truncated base-2^7 expansion (FP64
// multiply by 128 and subtract the integer part: no rounding).  Then
//
//   (A^T B)_mn = 2^{eA_m + eB_n} sum_{d=2..S+1} 2^{-7d} D_d,
//   D_d = sum_{p+q=d} sum_k dA_p[m,k] dB_q[n,k]        (int32, exact)
//
// keeping the pairs p + q <= S + 1 (the dropped ones are below the digit
// truncation).  With S = 8 the truncation error of an operand column is
// < 2^{-56} of its largest entry — the contraction carries the error bound of
// an FP64 GEMM (FP64 products of entries ~2^{-53} relative), and the
// integer sums are exact, so the result is deterministic and independent of
// the summation order.
//
// Kernel: one CTA per (128-row output tile, 64-column output tile, K chunk).
// Operands are the digit slices, K-major int8 (each output row / column's K
// digits contiguous), staged in shared memory with cp.async in the
// 64-byte-swizzled canonical UMMA layout, two stages.  One thread issues the
// S(S+1)/2 x 2 MMAs (M=128, N=64, K=32) per 64-deep k-block; the S diagonal
// sums D_d live in TMEM (S x 64 columns of 32-bit, all 512 for S = 8).  A K
// chunk is at most 16384 deep so a diagonal's int32 sum cannot overflow
// (S x 16384 x 127^2 < 2^31).  The epilogue reads the diagonals back
// (tcgen05.ld), combines them in FP64 smallest first, applies the exponents
// and writes one FP64 partial tile per K chunk; the chunks are added in
// fixed order afterwards.
#include <cstdint>

#include "common.hpp"
#include "kernels.hpp"

namespace svtb {

namespace {

constexpr int OZ_BM = 128;           // output rows per CTA (UMMA M)
constexpr int OZ_BN = 64;            // output columns per CTA (UMMA N)
constexpr int OZ_BK = 32;            // K bytes (= digits) per stage row: one MMA-K step
constexpr int OZ_NST = 4;            // pipeline stages
constexpr int OZ_KC = 16384;         // K per CTA (int32 diagonal sums cannot overflow)
constexpr int OZ_THREADS = 128;

template <int S>
struct OzTile {
    static constexpr int A_BYTES = OZ_BM * OZ_BK;  // one slice's A tile
    static constexpr int B_BYTES = OZ_BN * OZ_BK;
    static constexpr int STAGE = S * (A_BYTES + B_BYTES);
    static constexpr size_t SMEM = OZ_NST * static_cast<size_t>(STAGE) + 1024;  // + alignment slack
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// K-major, 32-byte swizzle (Swizzle<1,4,3>): 16-byte chunk c of row r lives
// at chunk c ^ ((r >> 2) & 1); 8-row atoms of 256 bytes stacked along M/N.
__device__ __forceinline__ uint64_t umma_desc_sw32(unsigned saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);  // start address
    d |= static_cast<uint64_t>(1) << 16;                 // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(256 >> 4) << 32;          // SBO: next 8-row atom
    d |= static_cast<uint64_t>(1) << 46;                 // descriptor version (sm_100)
    d |= static_cast<uint64_t>(6) << 61;                 // SWIZZLE_32B
    return d;
}

// kind::i8, D s32, A/B signed int8, both K-major, M = 128, N = 64
constexpr uint32_t kOzIdesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(OZ_BN >> 3) << 17) |
                              (static_cast<uint32_t>(OZ_BM >> 4) << 24);

__device__ __forceinline__ void cp16(unsigned dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity));
}

template <int S>
__global__ void __launch_bounds__(OZ_THREADS, 1)
    ozaki_tn_kernel(const int8_t* __restrict__ SA, long long a_tiles, const int8_t* __restrict__ SB,
                    long long b_tiles, const int* __restrict__ eA, const int* __restrict__ eB, long long M,
                    long long N, long long kchunk, long long Kpad, double* __restrict__ partial) {
    using T = OzTile<S>;
    extern __shared__ __align__(1024) unsigned char oz_raw[];
    __shared__ uint64_t mma_done[OZ_NST];
    __shared__ uint32_t tmem_base_sh;
    unsigned char* sm = oz_raw + ((1024 - (smem_u32(oz_raw) & 1023)) & 1023);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long m0 = static_cast<long long>(blockIdx.x) * OZ_BM;
    const long long n0 = static_cast<long long>(blockIdx.y) * OZ_BN;
    const long long k0 = static_cast<long long>(blockIdx.z) * kchunk;
    const long long k1 = min(Kpad, k0 + kchunk);
    const int nkb = static_cast<int>((k1 - k0) / OZ_BK);

    // barriers: full[s] — stage s's bulk copies landed (transaction count);
    // empty[s] (mma_done) — the MMAs reading stage s completed (tcgen05.commit)
    __shared__ uint64_t full_bar[OZ_NST];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            smem_u32(&tmem_base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        for (int q = 0; q < OZ_NST; ++q) {
            mbar_init(&mma_done[q], 1);
            mbar_init(&full_bar[q], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base_sh;

    if (warp == 1) {
        // ---- producer (one thread): per stage one bulk copy per slice tile ----
        if (lane == 0) {
            const long long KT = Kpad / OZ_BK, kt0 = k0 / OZ_BK;
            const long long mt = m0 / OZ_BM, nt = n0 / OZ_BN;
            for (int kb = 0; kb < nkb; ++kb) {
                const int st = kb % OZ_NST;
                if (kb >= OZ_NST) mbar_wait(&mma_done[st], static_cast<unsigned>((kb / OZ_NST - 1) & 1));
                const unsigned fb = smem_u32(&full_bar[st]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fb),
                             "r"(static_cast<unsigned>(T::STAGE)));
                unsigned char* base = sm + static_cast<size_t>(st) * T::STAGE;
                const long long kt = kt0 + kb;
#pragma unroll 1
                for (int p = 0; p < S; ++p) {
                    const int8_t* ga = SA + ((p * a_tiles + mt) * KT + kt) * T::A_BYTES;
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                            smem_u32(base + p * T::A_BYTES)),
                        "l"(ga), "r"(T::A_BYTES), "r"(fb)
                        : "memory");
                    const int8_t* gb = SB + ((p * b_tiles + nt) * KT + kt) * T::B_BYTES;
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                            smem_u32(base + S * T::A_BYTES + p * T::B_BYTES)),
                        "l"(gb), "r"(T::B_BYTES), "r"(fb)
                        : "memory");
                }
            }
        }
        __syncwarp();
    } else if (warp == 0) {
        // ---- MMA issuer (warp 0, one thread) -------------------------------
        if (lane == 0) {
            for (int kb = 0; kb < nkb; ++kb) {
                const int st = kb % OZ_NST;
                mbar_wait(&full_bar[st], static_cast<unsigned>((kb / OZ_NST) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                unsigned char* base = sm + static_cast<size_t>(st) * T::STAGE;
                const uint64_t da0 = umma_desc_sw32(smem_u32(base));
                const uint64_t db0 = umma_desc_sw32(smem_u32(base + S * T::A_BYTES));
                // the p = 1 row of pairs opens every diagonal: it overwrites
                // on the first k-block and accumulates afterwards
                const unsigned first_acc = kb > 0 ? 1u : 0u;
#pragma unroll
                for (int p = 1; p <= S; ++p) {
#pragma unroll
                    for (int q = 1; p + q <= S + 1; ++q) {
                        const uint32_t dt = tmem + static_cast<uint32_t>((p + q - 2) * OZ_BN);
                        const uint64_t da = da0 + static_cast<uint64_t>(((p - 1) * T::A_BYTES) >> 4);
                        const uint64_t db = db0 + static_cast<uint64_t>(((q - 1) * T::B_BYTES) >> 4);
                        asm volatile(
                            "{\n"
                            ".reg .pred pa;\n"
                            "setp.ne.b32 pa, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pa;\n"
                            "}\n" ::"r"(dt),
                            "l"(da), "l"(db), "r"(kOzIdesc), "r"(p == 1 ? first_acc : 1u));
                    }
                }
                asm volatile(
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                        smem_u32(&mma_done[st])));
            }
            // the last commit tracks every MMA issued before it
            if (nkb > 0)
                mbar_wait(&mma_done[(nkb - 1) % OZ_NST], static_cast<unsigned>(((nkb - 1) / OZ_NST) & 1));
        }
        __syncwarp();
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");

    // epilogue: thread (warp, lane) owns output row m0 + 32 warp + lane
    const long long m = m0 + warp * 32 + lane;
    const double sm_row = (m < M) ? ldexp(1.0, eA[m]) : 0.0;
    double* prow = partial + (static_cast<long long>(blockIdx.z) * M + m) * N;
#pragma unroll 1
    for (int cc = 0; cc < OZ_BN / 16; ++cc) {
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.0;
        for (int d = S - 1; d >= 0; --d) {  // smallest weights first
            uint32_t v[16];
            const uint32_t ta = tmem + (static_cast<uint32_t>(warp * 32) << 16) +
                                static_cast<uint32_t>(d * OZ_BN + cc * 16);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];\n"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15])
                : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
            const double w = ldexp(1.0, -7 * (d + 2));
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] = fma(static_cast<double>(static_cast<int>(v[j])), w, acc[j]);
        }
        if (m < M) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const long long n = n0 + cc * 16 + j;
                if (n < N) prow[n] = (nkb > 0) ? acc[j] * sm_row * ldexp(1.0, eB[n]) : 0.0;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// column exponents of a row-major K x C matrix: e_c with max_k |x_kc| < 2^{e_c}
// (grid: column blocks x row parts; the parts combine with atomicMax on the
// exponent, which is order-independent).  e must be preset to INT_MIN.
__global__ void oz_colexp_kernel(const double* __restrict__ X, long long K, long long C, long long ld,
                                 long long rows_per_part, int* __restrict__ e) {
    const long long c = blockIdx.x * 32LL + (threadIdx.x & 31);
    const int ty = threadIdx.x >> 5;
    __shared__ double red[8][33];
    double mx = 0.0;
    const long long r0 = blockIdx.y * rows_per_part, r1 = min(K, r0 + rows_per_part);
    if (c < C)
        for (long long k = r0 + ty; k < r1; k += 8) mx = fmax(mx, fabs(X[k * ld + c]));
    red[ty][threadIdx.x & 31] = mx;
    __syncthreads();
    if (ty == 0 && c < C) {
        for (int q = 1; q < 8; ++q) mx = fmax(mx, red[q][threadIdx.x & 31]);
        int ex = 0;
        if (mx > 0.0) frexp(mx, &ex);
        atomicMax(e + c, mx > 0.0 ? ex : -1074);
    }
}

__global__ void oz_fill_int_kernel(int* p, long long n, int v) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i < n) p[i] = v;
}

// Digit slices in the GEMM's shared-memory image: operand row c (an output
// row / column), K index k -> tile (c / TR, k / 32) of TR x 32 bytes, stored
// contiguously (slice p, row tile, k tile) in the 32-byte-swizzled K-major
// UMMA layout, so a pipeline stage is one contiguous bulk copy per slice.
// Zero outside K x C.  32 x 32 element tiles through shared memory keep the
// FP64 reads coalesced.
template <int S, int TR>
__global__ void __launch_bounds__(256) oz_slice_kernel(const double* __restrict__ X, long long K, long long C,
                                                       long long ld, const int* __restrict__ e, long long Kpad,
                                                       long long Ctiles, long long c_off, int8_t* __restrict__ out) {
    // block: 128 K values x 32 columns; thread: one column, 16 consecutive K
    // values -> one 16-byte store per slice (a swizzle chunk of the tile)
    __shared__ double tile[128][33];
    const long long kb = blockIdx.x * 128LL, cb = blockIdx.y * 32LL;
    const int t = threadIdx.x, tx = t & 31, ty = t >> 5;
    const long long c_rd = cb + tx;
    const int ex = (c_rd < C) ? e[c_rd] : 0;
    for (int r = ty; r < 128; r += 8) {
        const long long k = kb + r;
        double v = 0.0;
        if (k < K && c_rd < C) v = ldexp(X[k * ld + c_rd], -ex);
        tile[r][tx] = v;
    }
    __syncthreads();
    const long long c = cb + tx;            // operand row
    const int kq = ty;                      // 16-wide K group within the block
    const long long k0 = kb + 16 * kq;
    if (c >= C || k0 >= Kpad) return;
    const long long row = c_off + c;
    const long long ct = row / TR, kt = k0 / 32;
    const int rr = static_cast<int>(row - ct * TR);
    const int chunk = static_cast<int>((k0 / 16) & 1);
    const int inner = rr * 32 + ((chunk ^ ((rr >> 2) & 1)) << 4);
    const long long KT = Kpad / 32;
    double v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = tile[16 * kq + j][tx];
#pragma unroll
    for (int p = 0; p < S; ++p) {
        unsigned w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            unsigned packed = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                double x = v[4 * q + b] * 128.0;
                const double dgt = trunc(x);
                v[4 * q + b] = x - dgt;
                packed |= (static_cast<unsigned>(static_cast<int>(dgt)) & 0xFFu) << (8 * b);
            }
            w[q] = packed;
        }
        *reinterpret_cast<uint4*>(out + ((p * Ctiles + ct) * KT + kt) * (TR * 32) + inner) =
            make_uint4(w[0], w[1], w[2], w[3]);
    }
}

__global__ void oz_reduce_kernel(long long M, long long N, int splits, const double* __restrict__ partial,
                                 double alpha, double beta, double* __restrict__ C, long long ldc) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= M * N) return;
    const long long i = e / N, j = e - i * N;
    double s = 0.0;
    for (int q = 0; q < splits; ++q) s += partial[(static_cast<long long>(q) * M + i) * N + j];
    const double o = (beta != 0.0) ? beta * C[i * ldc + j] : 0.0;
    C[i * ldc + j] = fma(alpha, s, o);
}

inline long long rup(long long x, long long a) { return (x + a - 1) / a * a; }

// exponents e[0..C) and digit slices of the C columns of a row-major K x C
// FP64 matrix into rows [c_off, c_off + C) of a TR-row tiled slice array
template <int S, int TR>
void slice_columns(svt_ctx* ctx, const double* X, i64 K, i64 C, i64 ld, i64 Kpad, i64 Ctiles, i64 c_off,
                   int8_t* tiles, int* e) {
    cudaStream_t s = ctx->stream;
    if (C <= 0) return;
    LaunchScope ls(ctx, K_GEMM, 16.0 * K * C + 1.0 * S * C * Kpad, 0.0);  // part of the contraction
    oz_fill_int_kernel<<<static_cast<unsigned>((C + 255) / 256), 256, 0, s>>>(e, C, -2147483647);
    const i64 xb = (C + 31) / 32;
    const i64 parts = std::max<i64>(1, std::min<i64>((4 * ctx->num_sms + xb - 1) / xb, (K + 255) / 256));
    const i64 rpp = (std::max<i64>(K, 1) + parts - 1) / parts;
    oz_colexp_kernel<<<dim3(static_cast<unsigned>(xb), static_cast<unsigned>(parts)), 256, 0, s>>>(X, K, C, ld, rpp,
                                                                                                   e);
    oz_slice_kernel<S, TR><<<dim3(static_cast<unsigned>((Kpad + 127) / 128), static_cast<unsigned>(xb)), 256, 0, s>>>(
        X, K, C, ld, e, Kpad, Ctiles, c_off, tiles);
}

// C (M x N) = alpha * A^T B + beta * C from A's slices (a_tiles 128-row
// tiles, K padded to Kpad) and B (row-major K x N FP64, sliced here)
template <int S>
void ozaki_gemm(svt_ctx* ctx, i64 M, i64 N, i64 K, const int8_t* SA, i64 a_tiles, i64 Kpad, const int* eA,
                double alpha, const double* B, i64 ldb, double beta, double* C, i64 ldc) {
    cudaStream_t s = ctx->stream;
    const i64 Mpad = rup(M, OZ_BM), Npad = rup(N, OZ_BN);
    const size_t b_bytes = static_cast<size_t>(S) * Npad * Kpad;
    ctx->ws_ozakib.ensure((b_bytes + 7) / 8 + 2);
    int8_t* SB = reinterpret_cast<int8_t*>(ctx->ws_ozakib.get());
    ctx->ws_ozexpb.ensure(static_cast<size_t>(N));
    int* eB = ctx->ws_ozexpb.get();
    slice_columns<S, OZ_BN>(ctx, B, K, N, ldb, Kpad, Npad / OZ_BN, 0, SB, eB);
    // K split: the int32 diagonal sums bound a chunk at OZ_KC; among the
    // admissible split counts take the one with the fewest waves x chunk
    // depth (one CTA per SM)
    const i64 tiles = (Mpad / OZ_BM) * (Npad / OZ_BN);
    const i64 smin = (Kpad + OZ_KC - 1) / OZ_KC;
    i64 splits = smin;
    double best = 1e300;
    for (i64 sp = smin; sp <= std::max<i64>(smin, std::min<i64>(Kpad / OZ_BK, 64)); ++sp) {
        const i64 waves = (tiles * sp + ctx->num_sms - 1) / ctx->num_sms;
        const double cost = static_cast<double>(waves) * std::ceil(static_cast<double>(Kpad) / sp);
        if (cost < best * 0.999) {
            best = cost;
            splits = sp;
        }
    }
    const i64 kchunk = rup((Kpad + splits - 1) / splits, OZ_BK);
    splits = (Kpad + kchunk - 1) / kchunk;
    ctx->ws_partial.ensure(static_cast<size_t>(splits * M * N));
    static bool attr = false;
    if (!attr) {
        SVT_CUDA(cudaFuncSetAttribute(ozaki_tn_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(OzTile<S>::SMEM)));
        attr = true;
    }
    {
        LaunchScope ls(ctx, K_GEMM, static_cast<double>(S) * (Mpad + Npad) * Kpad + 8.0 * splits * M * N,
                       2.0 * M * N * K);
        const dim3 grid(static_cast<unsigned>(Mpad / OZ_BM), static_cast<unsigned>(Npad / OZ_BN),
                        static_cast<unsigned>(splits));
        ozaki_tn_kernel<S><<<grid, OZ_THREADS, OzTile<S>::SMEM, s>>>(SA, a_tiles, SB, Npad / OZ_BN, eA, eB, M, N,
                                                                     kchunk, Kpad, ctx->ws_partial.get());
    }
    LaunchScope ls(ctx, K_OTHER, 8.0 * (splits + 2) * M * N, 0.0);
    oz_reduce_kernel<<<static_cast<unsigned>((M * N + 255) / 256), 256, 0, s>>>(
        M, N, static_cast<int>(splits), ctx->ws_partial.get(), alpha, beta, C, ldc);
}

template <int S>
void ozaki_run(svt_ctx* ctx, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda, const double* B,
               i64 ldb, double beta, double* C, i64 ldc) {
    const i64 Kpad = rup(std::max<i64>(K, 1), OZ_BK);
    const i64 Mpad = rup(M, OZ_BM);
    const size_t a_bytes = static_cast<size_t>(S) * Mpad * Kpad;
    ctx->ws_ozaki.ensure((a_bytes + 7) / 8 + 2);
    int8_t* SA = reinterpret_cast<int8_t*>(ctx->ws_ozaki.get());
    ctx->ws_ozexp.ensure(static_cast<size_t>(M));
    slice_columns<S, OZ_BM>(ctx, A, K, M, lda, Kpad, Mpad / OZ_BM, 0, SA, ctx->ws_ozexp.get());
    ozaki_gemm<S>(ctx, M, N, K, SA, Mpad / OZ_BM, Kpad, ctx->ws_ozexp.get(), alpha, B, ldb, beta, C, ldc);
}

}  // namespace

// C (M x N, ld ldc) = alpha * A^T B + beta * C; A: K x M, B: K x N, row-major
// FP64.  slices: digits per operand entry (8: FP64-equivalent; 4..8).
void gemm_tn_ozaki(svt_ctx* ctx, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda, const double* B,
                   i64 ldb, double beta, double* C, i64 ldc, int slices) {
    if (M <= 0 || N <= 0) return;
    switch (slices) {
        case 6:
            ozaki_run<6>(ctx, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
            break;
        case 7:
            ozaki_run<7>(ctx, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
            break;
        default:
            ozaki_run<8>(ctx, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
            break;
    }
}


// Cached A operand (the Gram-Schmidt basis Q, whose columns only ever get
// appended during a sketch): slices of columns [c_off, c_off + C) of a
// row-major K x C block into the 128-row tiled cache, exponents into e.
i64 ozaki_kpad(i64 K) { return rup(std::max<i64>(K, 1), OZ_BK); }
i64 ozaki_rows_pad(i64 rows) { return rup(std::max<i64>(rows, 1), OZ_BM); }
void ozaki_slice_basis(svt_ctx* ctx, const double* X, i64 K, i64 C, i64 ld, i64 c_off, int8_t* tiles, i64 ctiles,
                       int* e) {
    slice_columns<8, OZ_BM>(ctx, X, K, C, ld, ozaki_kpad(K), ctiles, c_off, tiles, e + c_off);
}
void gemm_tn_ozaki_cached(svt_ctx* ctx, i64 M, i64 N, i64 K, const int8_t* tiles, i64 ctiles, const int* e,
                          const double* B, i64 ldb, double* C, i64 ldc) {
    if (M <= 0 || N <= 0) return;
    ozaki_gemm<8>(ctx, M, N, K, tiles, ctiles, ozaki_kpad(K), e, 1.0, B, ldb, 0.0, C, ldc);
}

}  // namespace svtb
