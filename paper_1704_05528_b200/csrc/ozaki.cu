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
constexpr int OZ_BK = 64;            // K bytes (= digits) per stage row
constexpr int OZ_KC = 16384;         // K per CTA (int32 diagonal sums cannot overflow)
constexpr int OZ_THREADS = 128;

template <int S>
struct OzTile {
    static constexpr int A_BYTES = OZ_BM * OZ_BK;  // one slice's A tile
    static constexpr int B_BYTES = OZ_BN * OZ_BK;
    static constexpr int STAGE = S * (A_BYTES + B_BYTES);
    static constexpr size_t SMEM = 2 * static_cast<size_t>(STAGE) + 1024;  // + alignment slack
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// K-major, 64-byte swizzle (Swizzle<2,4,3>): 16-byte chunk c of row r lives
// at chunk c ^ ((r >> 1) & 3); 8-row atoms of 512 bytes stacked along M/N.
__device__ __forceinline__ uint64_t umma_desc_sw64(unsigned saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);  // start address
    d |= static_cast<uint64_t>(1) << 16;                 // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(512 >> 4) << 32;          // SBO: next 8-row atom
    d |= static_cast<uint64_t>(1) << 46;                 // descriptor version (sm_100)
    d |= static_cast<uint64_t>(4) << 61;                 // SWIZZLE_64B
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
    ozaki_tn_kernel(const int8_t* __restrict__ SA, long long a_pitch, long long a_slice,
                    const int8_t* __restrict__ SB, long long b_pitch, long long b_slice,
                    const int* __restrict__ eA, const int* __restrict__ eB, long long M, long long N,
                    long long kchunk, long long Kpad, double* __restrict__ partial) {
    using T = OzTile<S>;
    extern __shared__ __align__(1024) unsigned char oz_raw[];
    __shared__ uint64_t mma_done[2];
    __shared__ uint32_t tmem_base_sh;
    unsigned char* sm = oz_raw + ((1024 - (smem_u32(oz_raw) & 1023)) & 1023);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long m0 = static_cast<long long>(blockIdx.x) * OZ_BM;
    const long long n0 = static_cast<long long>(blockIdx.y) * OZ_BN;
    const long long k0 = static_cast<long long>(blockIdx.z) * kchunk;
    const long long k1 = min(Kpad, k0 + kchunk);
    const int nkb = static_cast<int>((k1 - k0) / OZ_BK);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            smem_u32(&tmem_base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        mbar_init(&mma_done[0], 1);
        mbar_init(&mma_done[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base_sh;

    // stage issue: every thread copies its 16-byte chunks of all S slices
    auto load = [&](int kb, int st) {
        unsigned char* base = sm + static_cast<size_t>(st) * T::STAGE;
        const long long kk = k0 + static_cast<long long>(kb) * OZ_BK;
#pragma unroll 1
        for (int p = 0; p < S; ++p) {
            const int8_t* ga = SA + p * a_slice + m0 * a_pitch + kk;
            const unsigned sa = smem_u32(base + p * T::A_BYTES);
#pragma unroll
            for (int j = 0; j < OZ_BM * 4 / OZ_THREADS; ++j) {
                const int g = tid + j * OZ_THREADS;
                const int r = g >> 2, c = g & 3;
                cp16(sa + r * OZ_BK + ((c ^ ((r >> 1) & 3)) << 4), ga + r * a_pitch + (c << 4));
            }
            const int8_t* gb = SB + p * b_slice + n0 * b_pitch + kk;
            const unsigned sb = smem_u32(base + S * T::A_BYTES + p * T::B_BYTES);
#pragma unroll
            for (int j = 0; j < OZ_BN * 4 / OZ_THREADS; ++j) {
                const int g = tid + j * OZ_THREADS;
                const int r = g >> 2, c = g & 3;
                cp16(sb + r * OZ_BK + ((c ^ ((r >> 1) & 3)) << 4), gb + r * b_pitch + (c << 4));
            }
        }
        asm volatile("cp.async.commit_group;\n");
    };

    unsigned phase[2] = {0u, 0u};
    unsigned started = 0;  // diagonals that already hold a partial sum (issuing thread)
    if (nkb > 0) load(0, 0);
    for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb & 1;
        if (kb + 1 < nkb) {
            // the other stage was last read by the MMAs of k-block kb - 1
            if (kb >= 1) {
                mbar_wait(&mma_done[st ^ 1], phase[st ^ 1]);
                phase[st ^ 1] ^= 1u;
            }
            load(kb + 1, st ^ 1);
            asm volatile("cp.async.wait_group 1;\n");
        } else {
            asm volatile("cp.async.wait_group 0;\n");
        }
        // generic-proxy smem writes -> visible to the tensor core's async proxy
        asm volatile("fence.proxy.async.shared::cta;\n");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            unsigned char* base = sm + static_cast<size_t>(st) * T::STAGE;
            const unsigned sa0 = smem_u32(base), sb0 = smem_u32(base + S * T::A_BYTES);
#pragma unroll 1
            for (int p = 1; p <= S; ++p) {
#pragma unroll 1
                for (int q = 1; p + q <= S + 1; ++q) {
                    const int d = p + q - 2;
                    const uint32_t dt = tmem + static_cast<uint32_t>(d * OZ_BN);
#pragma unroll
                    for (int ks = 0; ks < OZ_BK / 32; ++ks) {
                        const uint64_t da = umma_desc_sw64(sa0 + (p - 1) * T::A_BYTES + ks * 32);
                        const uint64_t db = umma_desc_sw64(sb0 + (q - 1) * T::B_BYTES + ks * 32);
                        const unsigned acc = (started >> d) & 1u;
                        asm volatile(
                            "{\n"
                            ".reg .pred pa;\n"
                            "setp.ne.b32 pa, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pa;\n"
                            "}\n" ::"r"(dt),
                            "l"(da), "l"(db), "r"(kOzIdesc), "r"(acc));
                        started |= 1u << d;
                    }
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                smem_u32(&mma_done[st])));
        }
    }
    // all MMAs done: the last commit covers every earlier MMA
    if (nkb > 0) {
        const int st = (nkb - 1) & 1;
        mbar_wait(&mma_done[st], phase[st]);
    }
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

// digit slices, transposed to K-major: out[p][c][k] (pitch Kpad, slice
// stride Cpad * Kpad), zero outside K x C.  32 x 32 tiles through shared
// memory so both the FP64 reads and the int8 writes are coalesced.
template <int S>
__global__ void oz_slice_kernel(const double* __restrict__ X, long long K, long long C, long long ld,
                                const int* __restrict__ e, long long Kpad, long long Cpad,
                                int8_t* __restrict__ out) {
    __shared__ double tile[32][33];
    const long long kb = blockIdx.x * 32LL, cb = blockIdx.y * 32LL;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
    for (int r = ty; r < 32; r += 8) {
        const long long k = kb + r, c = cb + tx;
        double v = 0.0;
        if (k < K && c < C) v = ldexp(X[k * ld + c], -e[c]);
        tile[r][tx] = v;
    }
    __syncthreads();
    const long long slice = Cpad * Kpad;
    for (int r = ty; r < 32; r += 8) {  // r: column within the tile, tx: k within the tile
        const long long c = cb + r, k = kb + tx;
        if (c >= Cpad || k >= Kpad) continue;
        double v = tile[tx][r];
#pragma unroll
        for (int p = 0; p < S; ++p) {
            v *= 128.0;
            const double dgt = trunc(v);
            v -= dgt;
            out[p * slice + c * Kpad + k] = static_cast<int8_t>(static_cast<int>(dgt));
        }
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

template <int S>
void ozaki_run(svt_ctx* ctx, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda, const double* B,
               i64 ldb, double beta, double* C, i64 ldc) {
    cudaStream_t s = ctx->stream;
    const i64 Kpad = rup(std::max<i64>(K, 1), OZ_BK);
    const i64 Mpad = rup(M, OZ_BM), Npad = rup(N, OZ_BN);
    const size_t a_bytes = static_cast<size_t>(S) * Mpad * Kpad, b_bytes = static_cast<size_t>(S) * Npad * Kpad;
    ctx->ws_ozaki.ensure((a_bytes + b_bytes + 7) / 8 + 2);
    int8_t* SA = reinterpret_cast<int8_t*>(ctx->ws_ozaki.get());
    int8_t* SB = SA + a_bytes;
    ctx->ws_ozexp.ensure(static_cast<size_t>(M + N));
    int* eA = ctx->ws_ozexp.get();
    int* eB = eA + M;
    {
        LaunchScope ls(ctx, K_OTHER, 8.0 * (M * K + N * K) * 2 + S * 1.0 * (Mpad + Npad) * Kpad, 0.0);
        oz_fill_int_kernel<<<static_cast<unsigned>((M + N + 255) / 256), 256, 0, s>>>(eA, M + N, -2147483647);
        for (int q = 0; q < 2; ++q) {
            const i64 cols = q ? N : M;
            const i64 xb = (cols + 31) / 32;
            const i64 parts = std::max<i64>(1, std::min<i64>((4 * ctx->num_sms + xb - 1) / xb, (K + 255) / 256));
            const i64 rpp = (K + parts - 1) / parts;
            oz_colexp_kernel<<<dim3(static_cast<unsigned>(xb), static_cast<unsigned>(parts)), 256, 0, s>>>(
                q ? B : A, K, cols, q ? ldb : lda, rpp, q ? eB : eA);
        }
        oz_slice_kernel<S><<<dim3(static_cast<unsigned>(Kpad / 32), static_cast<unsigned>(Mpad / 32)), 256, 0, s>>>(
            A, K, M, lda, eA, Kpad, Mpad, SA);
        oz_slice_kernel<S><<<dim3(static_cast<unsigned>(Kpad / 32), static_cast<unsigned>(Npad / 32)), 256, 0, s>>>(
            B, K, N, ldb, eB, Kpad, Npad, SB);
    }
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
        LaunchScope ls(ctx, K_GEMM, static_cast<double>(a_bytes + b_bytes) + 8.0 * splits * M * N,
                       2.0 * M * N * K);
        const dim3 grid(static_cast<unsigned>(Mpad / OZ_BM), static_cast<unsigned>(Npad / OZ_BN),
                        static_cast<unsigned>(splits));
        ozaki_tn_kernel<S><<<grid, OZ_THREADS, OzTile<S>::SMEM, s>>>(SA, Kpad, Mpad * Kpad, SB, Kpad, Npad * Kpad,
                                                                     eA, eB, M, N, kchunk, Kpad,
                                                                     ctx->ws_partial.get());
    }
    LaunchScope ls(ctx, K_OTHER, 8.0 * (splits + 2) * M * N, 0.0);
    oz_reduce_kernel<<<static_cast<unsigned>((M * N + 255) / 256), 256, 0, s>>>(
        M, N, static_cast<int>(splits), ctx->ws_partial.get(), alpha, beta, C, ldc);
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

}  // namespace svtb
