// Device Gaussian sketch generator: a bit-exact std::mt19937_64 integer stream
// (the C++ standard fixes every output) followed by the reference's explicit
// Box-Muller transform, dense.hpp:52-98.
//
// Stage 1 (mt_twist_kernel): one 160-thread CTA owns the 312-word state in
// shared memory (ping-pong) and runs each twist as two data-parallel halves
// (words 0..155 read only old words; words 156..311 read the new words
// 0..155), tempering and streaming the raw 64-bit draws to HBM as they form.  The state persists in global memory
// between chunks, so arbitrarily long streams (qb_init at t0 = 5000 needs
// 5e8 draws) are produced in bounded scratch.
// Stage 2 (box_muller_kernel): grid-wide; pair p consumes draws 2p (u1 = 1-u)
// and 2p+1 (u2), emits r*cos (normal 2p) and r*sin (normal 2p+1, the
// reference's "spare"), scattered to the column-major fill position of the
// row-major output panel.  log/sqrt/sin/cos are the CUDA double-precision
// functions (<= 1-2 ulp from glibc; the integer stream is identical).
#include "common.hpp"
#include "kernels.hpp"

namespace svtb {

namespace {

constexpr int MT_N = 312;
constexpr int MT_M = 156;
constexpr unsigned long long MT_A = 0xB5026F5AA96619E9ULL;
constexpr unsigned long long MT_UM = 0xFFFFFFFF80000000ULL;
constexpr unsigned long long MT_LM = 0x7FFFFFFFULL;

__device__ __forceinline__ unsigned long long temper(unsigned long long y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

__device__ __forceinline__ unsigned long long twist_word(unsigned long long cur, unsigned long long nxt,
                                                         unsigned long long far) {
    const unsigned long long x = (cur & MT_UM) | (nxt & MT_LM);
    unsigned long long xa = x >> 1;
    if (x & 1ULL) xa ^= MT_A;
    return far ^ xa;
}

// One CTA of 160 threads (thread i < 156 owns words i and i + 156).  The
// twist x[k + 312] = f(x[k], x[k + 1], x[k + 156]) has dependency distance
// 156, so each half of a twist is one data-parallel step: words 0..155 read
// only the previous state, words 156..311 the previous state and the new
// words 0..155 (word 311 reads the new word 0).  The state is ping-ponged
// between two shared arrays (no read-before-overwrite hazard), so a twist
// costs two barriers; every new word is tempered and written out as soon as
// it is formed.  init != 0: seed the state (std::mt19937_64 seeding
// recurrence, f = 6364136223846793005); else continue from `state`.
// Generates ntwists * 312 draws into out and saves the final state.
constexpr int kMtThreads = 160;
__device__ __forceinline__ void mt_seed(unsigned long long seed, unsigned long long* mt) {
    unsigned long long x = seed;
    mt[0] = x;
    for (int i = 1; i < MT_N; ++i) {
        x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<unsigned long long>(i);
        mt[i] = x;
    }
}

__device__ __forceinline__ void mt_run(unsigned long long (*mt)[MT_N], long long ntwists,
                                       unsigned long long* __restrict__ out, int& cur) {
    const int i = threadIdx.x;
    for (long long t = 0; t < ntwists; ++t) {
        const unsigned long long* o = mt[cur];
        unsigned long long* nw = mt[cur ^ 1];
        unsigned long long* dst = out + t * MT_N;
        if (i < MT_M) {
            const unsigned long long v = twist_word(o[i], o[i + 1], o[i + MT_M]);
            nw[i] = v;
            dst[i] = temper(v);
        }
        __syncthreads();
        if (i < MT_M) {
            const int j = i + MT_M;
            const unsigned long long v = twist_word(o[j], (j + 1 < MT_N) ? o[j + 1] : nw[0], nw[i]);
            nw[j] = v;
            dst[j] = temper(v);
        }
        __syncthreads();
        cur ^= 1;
    }
}

__global__ void __launch_bounds__(kMtThreads) mt_twist_kernel(unsigned long long seed, int init,
                                                              unsigned long long* state, long long ntwists,
                                                              unsigned long long* out) {
    __shared__ unsigned long long mt[2][MT_N];
    if (init) {
        if (threadIdx.x == 0) mt_seed(seed, mt[0]);
    } else {
        for (int i = threadIdx.x; i < MT_N; i += blockDim.x) mt[0][i] = state[i];
    }
    __syncthreads();
    int cur = 0;
    mt_run(mt, ntwists, out, cur);
    for (int i = threadIdx.x; i < MT_N; i += blockDim.x) state[i] = mt[cur][i];
}

// normal q of the block lands at (row q % rows, column q / rows) of the
// row-major panel: one 64-bit division per pair (the second normal is the
// next row, or the top of the next column)
__device__ __forceinline__ void store_pair(double* __restrict__ out, long long ld, long long rows, long long total,
                                           long long q0, double z0, double z1) {
    const long long c0 = q0 / rows;
    const long long r0 = q0 - c0 * rows;
    if (q0 < total) out[r0 * ld + c0] = z0;
    if (q0 + 1 < total) {
        const bool wrap = (r0 + 1 == rows);
        out[(wrap ? 0 : r0 + 1) * ld + (wrap ? c0 + 1 : c0)] = z1;
    }
}

// pairs [0, npairs) of this chunk; global normal index q = 2*(pair0 + p) + {0,1}
__global__ void box_muller_kernel(const unsigned long long* __restrict__ draws, long long npairs, long long pair0,
                                  long long rows, long long total, double* __restrict__ out, long long ld) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= npairs) return;
    const unsigned long long a = draws[2 * p];
    const unsigned long long b = draws[2 * p + 1];
    const double u1 = 1.0 - static_cast<double>(a >> 11) * 0x1.0p-53;
    const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    const long long q0 = 2 * (pair0 + p);
    double sn, cs;
    sincos(angle, &sn, &cs);
    store_pair(out, ld, rows, total, q0, radius * cs, radius * sn);
}

// K independent streams at once: block k seeds std::mt19937_64 with
// seeds[k] and writes ntwists * 312 draws to out + k * stride.
struct SeedPack {
    unsigned long long s[kMaxOmegaBatch];
};

__global__ void __launch_bounds__(kMtThreads) mt_twist_multi_kernel(SeedPack seeds, long long ntwists,
                                                                    unsigned long long* __restrict__ out,
                                                                    long long stride) {
    __shared__ unsigned long long mt[2][MT_N];
    if (threadIdx.x == 0) mt_seed(seeds.s[blockIdx.x], mt[0]);
    __syncthreads();
    int cur = 0;
    mt_run(mt, ntwists, out + blockIdx.x * stride, cur);
}

__global__ void box_muller_multi_kernel(const unsigned long long* __restrict__ draws, long long draw_stride,
                                        long long npairs, long long rows, long long total,
                                        double* __restrict__ out, long long out_stride, long long ld) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= npairs) return;
    const unsigned long long* d = draws + blockIdx.y * draw_stride;
    double* o = out + blockIdx.y * out_stride;
    const unsigned long long a = d[2 * p];
    const unsigned long long b = d[2 * p + 1];
    const double u1 = 1.0 - static_cast<double>(a >> 11) * 0x1.0p-53;
    const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    const long long q0 = 2 * p;
    double sn, cs;
    sincos(angle, &sn, &cs);
    store_pair(o, ld, rows, total, q0, radius * cs, radius * sn);
}

}  // namespace

void gaussian_blocks_dev(svt_ctx* ctx, i64 rows, i64 cols, const u64* seeds, int K, double* out, i64 out_stride,
                         i64 ld, bool on_side) {
    cudaStream_t stream = on_side ? ctx->side : ctx->stream;
    DevBuf<unsigned long long>& scratch = on_side ? ctx->ws_rng_side : ctx->ws_rng;
    if (rows < 1 || cols < 1) throw std::invalid_argument("gaussian_block: dimensions must be >= 1");
    if (K < 1) return;
    if (K > kMaxOmegaBatch) throw std::invalid_argument("gaussian_blocks_dev: too many streams");
    const i64 total = rows * cols;
    const i64 pairs = (total + 1) / 2;
    const i64 twists = (2 * pairs + MT_N - 1) / MT_N;
    const i64 draw_stride = twists * MT_N;
    scratch.ensure(static_cast<size_t>(draw_stride * K));
    SeedPack pack{};
    for (int k = 0; k < K; ++k) pack.s[k] = seeds[k];
    {
        LaunchScope ls(ctx, K_RNG, 8.0 * draw_stride * K, 0.0, stream);
        mt_twist_multi_kernel<<<K, kMtThreads, 0, stream>>>(pack, twists, scratch.get(), draw_stride);
    }
    LaunchScope ls(ctx, K_RNG, 32.0 * pairs * K, 0.0, stream);
    dim3 grid(static_cast<unsigned>((pairs + 255) / 256), static_cast<unsigned>(K));
    box_muller_multi_kernel<<<grid, 256, 0, stream>>>(scratch.get(), draw_stride, pairs, rows, total, out,
                                                           out_stride, ld);
}

void gaussian_block_dev(svt_ctx* ctx, i64 rows, i64 cols, u64 seed, double* out, i64 ld) {
    if (rows < 1 || cols < 1) throw std::invalid_argument("gaussian_block: dimensions must be >= 1");
    const i64 total = rows * cols;
    const i64 pairs_needed = (total + 1) / 2;
    const i64 twists_needed = (2 * pairs_needed + MT_N - 1) / MT_N;
    const i64 max_twists_per_chunk = 16384;  // 5.1M draws, 40 MB scratch
    const i64 chunk_twists = std::min<i64>(twists_needed, max_twists_per_chunk);
    ctx->ws_rng.ensure(static_cast<size_t>(chunk_twists * MT_N));
    ctx->ws_mt.ensure(MT_N);
    i64 done_twists = 0;
    bool first = true;
    while (done_twists < twists_needed) {
        const i64 nt = std::min<i64>(chunk_twists, twists_needed - done_twists);
        {
            LaunchScope ls(ctx, K_RNG, nt * MT_N * 8.0, 0.0);
            mt_twist_kernel<<<1, kMtThreads, 0, ctx->stream>>>(seed, first ? 1 : 0, ctx->ws_mt.get(), nt, ctx->ws_rng.get());
        }
        first = false;
        const i64 pair0 = done_twists * MT_N / 2;
        const i64 npairs = std::min<i64>(nt * MT_N / 2, pairs_needed - pair0);
        if (npairs > 0) {
            LaunchScope ls(ctx, K_RNG, npairs * 2 * 8.0 + npairs * 2 * 8.0, 0.0);
            const int bs = 256;
            box_muller_kernel<<<static_cast<unsigned>((npairs + bs - 1) / bs), bs, 0, ctx->stream>>>(
                ctx->ws_rng.get(), npairs, pair0, rows, total, out, ld);
        }
        done_twists += nt;
    }
}

}  // namespace svtb
