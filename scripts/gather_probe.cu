// Microbenchmark: the L2 -> SM row-gather ceiling behind the wide SpMM.
// Every "entry" gathers one W = 128-double (1 KB) row of a panel and adds it
// into a per-warp accumulator (what spmm_wide_kernel does per stored entry).
// Variants: (a) LDG.64 x4 per lane (the current kernel's access pattern),
// (b) LDG.128 x2 per lane, (c) cp.async.bulk of the whole row into a
// per-warp shared-memory ring with mbarrier completion (TMA unit).
// Indices: uniform, or Zipf(1.1)-like popularity (cfg3/cfg4 items).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_probe gather_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            std::printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                    \
            std::exit(1);                                                                       \
        }                                                                                       \
    } while (0)

constexpr int W = 128;
constexpr int SEG = 512;

template <int U>
__global__ void __launch_bounds__(128) ldg64_kernel(const int* __restrict__ idx, long long nnz,
                                                    const double* __restrict__ X, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long seg = (blockIdx.x * 4LL + (threadIdx.x >> 5));
    const long long beg = seg * SEG, end = min(nnz, beg + SEG);
    if (beg >= nnz) return;
    double acc[4] = {0, 0, 0, 0};
    for (long long k0 = beg; k0 < end; k0 += 32) {
        const long long k = k0 + lane;
        const int cl = k < end ? __ldg(idx + k) : 0;
        const int cnt = static_cast<int>(min(32LL, end - k0));
        for (int e = 0; e < cnt; e += U) {
            double xv[U][4];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = __shfl_sync(0xffffffffu, cl, (e + u) & 31);
                const double* xr = X + static_cast<long long>(c) * W + lane;
#pragma unroll
                for (int q = 0; q < 4; ++q) xv[u][q] = __ldg(xr + 32 * q);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] += xv[u][q];
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) out[seg * W + lane + 32 * q] = acc[q];
}

template <int U>
__global__ void __launch_bounds__(128) ldg128_kernel(const int* __restrict__ idx, long long nnz,
                                                     const double* __restrict__ X, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long seg = (blockIdx.x * 4LL + (threadIdx.x >> 5));
    const long long beg = seg * SEG, end = min(nnz, beg + SEG);
    if (beg >= nnz) return;
    double2 acc[2] = {{0, 0}, {0, 0}};
    for (long long k0 = beg; k0 < end; k0 += 32) {
        const long long k = k0 + lane;
        const int cl = k < end ? __ldg(idx + k) : 0;
        const int cnt = static_cast<int>(min(32LL, end - k0));
        for (int e = 0; e < cnt; e += U) {
            double2 xv[U][2];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = __shfl_sync(0xffffffffu, cl, (e + u) & 31);
                const double2* xr = reinterpret_cast<const double2*>(X + static_cast<long long>(c) * W) + lane;
                xv[u][0] = __ldg(xr);
                xv[u][1] = __ldg(xr + 32);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    acc[q].x += xv[u][q].x;
                    acc[q].y += xv[u][q].y;
                }
        }
    }
    double2* o = reinterpret_cast<double2*>(out + seg * W) + lane;
    o[0] = acc[0];
    o[32] = acc[1];
}

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

// per-warp ring of R rows; lane 0 issues one bulk copy per entry
template <int R, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) bulk_kernel(const int* __restrict__ idx, long long nnz,
                                                          const double* __restrict__ X, double* __restrict__ out,
                                                          long long nseg) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* ring = reinterpret_cast<double*>(smem) + static_cast<size_t>(warp) * R * W;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + static_cast<size_t>(WARPS) * R * W * 8) +
                              warp * R;
    if (lane == 0)
        for (int s = 0; s < R; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncwarp();
    unsigned phase_bits = 0;  // one parity bit per slot (R <= 32)
    for (long long seg = blockIdx.x * static_cast<long long>(WARPS) + warp; seg < nseg;
         seg += static_cast<long long>(gridDim.x) * WARPS) {
        const long long beg = seg * SEG, end = min(nnz, beg + SEG);
        const int cnt = static_cast<int>(end - beg);
        auto issue = [&](int e) {
            const int s = e % R;
            const int c = __ldg(idx + beg + e);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar + s)), "r"(W * 8));
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                    su32(ring + s * W)),
                "l"(X + static_cast<long long>(c) * W), "r"(W * 8), "r"(su32(bar + s))
                : "memory");
        };
        if (lane == 0)
            for (int e = 0; e < min(R, cnt); ++e) issue(e);
        double2 acc[2] = {{0, 0}, {0, 0}};
        for (int e = 0; e < cnt; ++e) {
            const int s = e % R;
            const unsigned par = (phase_bits >> s) & 1u;
            asm volatile(
                "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                    su32(bar + s)),
                "r"(par)
                : "memory");
            phase_bits ^= (1u << s);
            const double2* r = reinterpret_cast<const double2*>(ring + s * W) + lane;
            const double2 a = r[0], b = r[32];
            acc[0].x += a.x;
            acc[0].y += a.y;
            acc[1].x += b.x;
            acc[1].y += b.y;
            __syncwarp();
            if (lane == 0 && e + R < cnt) issue(e + R);
        }
        double2* o = reinterpret_cast<double2*>(out + seg * W) + lane;
        o[0] = acc[0];
        o[32] = acc[1];
    }
}

int main(int argc, char** argv) {
    const long long nnz = 9000000;
    int dev_sms = 0;
    CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, 0));
    const long long nseg = (nnz + SEG - 1) / SEG;
    double* out;
    CK(cudaMalloc(&out, nseg * W * 8));
    for (int rows : {10677, 69878}) {
        for (int dist = 0; dist < 2; ++dist) {
            // indices: CSR-like (sorted within each 129-entry "row"), uniform or Zipf(1.1) popularity
            std::mt19937_64 g(7);
            std::vector<double> cdf(rows);
            double z = 0;
            for (int i = 0; i < rows; ++i) cdf[i] = (z += (dist ? std::pow(i + 1.0, -1.1) : 1.0));
            for (auto& v : cdf) v /= z;
            std::vector<int> h(nnz);
            std::uniform_real_distribution<double> U01(0, 1);
            for (long long k = 0; k < nnz; ++k)
                h[k] = static_cast<int>(std::lower_bound(cdf.begin(), cdf.end(), U01(g)) - cdf.begin());
            for (long long k = 0; k < nnz; k += 129) std::sort(h.begin() + k, h.begin() + std::min(nnz, k + 129));
            int* idx;
            double* X;
            CK(cudaMalloc(&idx, nnz * 4));
            CK(cudaMalloc(&X, static_cast<size_t>(rows) * W * 8));
            CK(cudaMemcpy(idx, h.data(), nnz * 4, cudaMemcpyHostToDevice));
            CK(cudaMemset(X, 0, static_cast<size_t>(rows) * W * 8));
            cudaEvent_t a, b;
            CK(cudaEventCreate(&a));
            CK(cudaEventCreate(&b));
            auto timeit = [&](const char* name, auto launch) {
                for (int i = 0; i < 3; ++i) launch();
                CK(cudaDeviceSynchronize());
                CK(cudaEventRecord(a));
                const int reps = 10;
                for (int i = 0; i < reps; ++i) launch();
                CK(cudaEventRecord(b));
                CK(cudaEventSynchronize(b));
                float ms;
                CK(cudaEventElapsedTime(&ms, a, b));
                ms /= reps;
                std::printf("rows %6d %-8s %-28s %8.1f us  gather %6.2f TB/s\n", rows, dist ? "zipf1.1" : "uniform",
                            name, ms * 1e3, nnz * W * 8.0 / (ms * 1e-3) / 1e12);
            };
            const unsigned nb = static_cast<unsigned>((nseg + 3) / 4);
            timeit("ldg64 U=4", [&] { ldg64_kernel<4><<<nb, 128>>>(idx, nnz, X, out); });
            timeit("ldg64 U=8", [&] { ldg64_kernel<8><<<nb, 128>>>(idx, nnz, X, out); });
            timeit("ldg128 U=4", [&] { ldg128_kernel<4><<<nb, 128>>>(idx, nnz, X, out); });
            timeit("ldg128 U=8", [&] { ldg128_kernel<8><<<nb, 128>>>(idx, nnz, X, out); });
            {
                constexpr int R = 8, WP = 4;
                const size_t sm = static_cast<size_t>(WP) * R * (W * 8 + 8);
                CK(cudaFuncSetAttribute(bulk_kernel<R, WP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                int occ = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bulk_kernel<R, WP>, 32 * WP, sm));
                const unsigned g2 = static_cast<unsigned>(occ * dev_sms);
                timeit("bulk R=8 4w (persistent)", [&] { bulk_kernel<R, WP><<<g2, 32 * WP, sm>>>(idx, nnz, X, out, nseg); });
            }
            {
                constexpr int R = 12, WP = 4;
                const size_t sm = static_cast<size_t>(WP) * R * (W * 8 + 8);
                CK(cudaFuncSetAttribute(bulk_kernel<R, WP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                int occ = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bulk_kernel<R, WP>, 32 * WP, sm));
                const unsigned g2 = static_cast<unsigned>(occ * dev_sms);
                timeit("bulk R=12 4w (persistent)", [&] { bulk_kernel<R, WP><<<g2, 32 * WP, sm>>>(idx, nnz, X, out, nseg); });
            }
            {
                constexpr int R = 16, WP = 2;
                const size_t sm = static_cast<size_t>(WP) * R * (W * 8 + 8);
                CK(cudaFuncSetAttribute(bulk_kernel<R, WP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                int occ = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bulk_kernel<R, WP>, 32 * WP, sm));
                const unsigned g2 = static_cast<unsigned>(occ * dev_sms);
                timeit("bulk R=16 2w (persistent)", [&] { bulk_kernel<R, WP><<<g2, 32 * WP, sm>>>(idx, nnz, X, out, nseg); });
            }
            CK(cudaFree(idx));
            CK(cudaFree(X));
        }
    }
    return 0;
}
