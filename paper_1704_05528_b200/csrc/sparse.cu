// Sparse kernels on the sample set Lambda (sampled.hpp).
//
// Storage (per rank, its row block): CSR rowptr int64 / col int32 / val fp64,
// plus a CSC view (colptr int64 / local row int32) whose value array is a
// mirror of the CSR values kept in sync through csr2csc.  Y*X runs over CSR
// and Y^T*X over CSC with the SAME gather kernel, so both are deterministic
// (no atomics) — the reference's single-threaded results are reproducible
// run-to-run (SPEC: bit-reproducible single-thread runs).
//
// Narrow panels (w <= 16, the dt = 10 rank-revealing rounds): one warp per
// output row, one stored entry per lane, w register accumulators, warp-shuffle
// tree reduction.  The w-wide dense row of an entry is one contiguous 8w-byte
// gather (row-major panel), read through the read-only path; the panel is
// L2-resident (n x 10 doubles = 8 MB at n = 1e5).
// Wide panels (qb_init at t0 up to 5000): one warp per (row, 128-column
// chunk); entries are broadcast 32 at a time by shuffle, lanes stride the
// contiguous panel row (1 KB coalesced per entry).
#include <cstdlib>

#include "common.hpp"
#include "kernels.hpp"

namespace svtb {

namespace {

constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One warp per SEGMENT of at most kSegLen stored entries (host.cpp builds
// the plan): short rows are one segment and write their output row
// directly; long rows (power-law users, Zipf-popular items) are split across
// warps that write partial rows, summed afterwards in segment order
// (deterministic).
//
// Lane mapping (column-cooperative): the warp is G = 32 / W groups of W
// lanes; group g handles every G-th stored entry and lane j of the group its
// column j, so one load instruction gathers G whole W-wide panel rows
// (contiguous 8W-byte segments) instead of 32 scattered 8-byte words — the
// L1/L2 request count per entry drops ~W-fold.  Indices and values are read
// 32 at a time, coalesced, and broadcast by shuffle.
template <int W>
__global__ void __launch_bounds__(32 * kWarpsPerBlock) spmm_narrow_kernel(
    SegPlanView plan, const int* __restrict__ idx, const double* __restrict__ val, const double* __restrict__ X,
    long long ldx, double* __restrict__ out, long long ldo, double* __restrict__ partial) {
    constexpr int G = 32 / W;
    const int lane = threadIdx.x & 31;
    const int g = lane / W, j = lane - (lane / W) * W;
    const bool active = lane < G * W;
    const long long sg = static_cast<long long>(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
    if (sg >= plan.nseg) return;
    double acc = 0.0;
    const long long beg = plan.seg_beg[sg], end = plan.seg_end[sg];
    constexpr int STEPS = (32 + G - 1) / G;
    // software pipeline: the next 32 indices / values are in flight while
    // the current chunk's gathers issue (all STEPS gathers independent)
    int cl_n = 0;
    double vl_n = 0.0;
    if (beg + lane < end) {
        cl_n = __ldg(idx + beg + lane);
        vl_n = __ldg(val + beg + lane);
    }
    for (long long base = beg; base < end; base += 32) {
        const int cl = cl_n;
        const double vl = vl_n;
        const long long kn = base + 32 + lane;
        cl_n = 0;
        vl_n = 0.0;
        if (kn < end) {
            cl_n = __ldg(idx + kn);
            vl_n = __ldg(val + kn);
        }
#pragma unroll
        for (int s = 0; s < STEPS; ++s) {
            const int e = s * G + g;
            const int src = e < 32 ? e : 31;
            const int c = __shfl_sync(0xffffffffu, cl, src);
            double v = __shfl_sync(0xffffffffu, vl, src);
            if (e >= 32) v = 0.0;  // lanes past the row end already carry v = 0
            const double x = active ? __ldg(X + static_cast<long long>(c) * ldx + j) : 0.0;
            acc = fma(v, x, acc);
        }
    }
    // fold the G groups onto lanes 0..W-1 (fixed order)
    double tot = acc;
#pragma unroll
    for (int q = 1; q < G; ++q) {
        const int src = lane + q * W;
        const double o = __shfl_sync(0xffffffffu, acc, src < 32 ? src : 31);
        if (src < 32) tot += o;
    }
    if (lane < W) {
        const int slot = plan.seg_slot[sg];
        if (slot < 0)
            out[static_cast<long long>(plan.seg_row[sg]) * ldo + lane] = tot;
        else
            partial[static_cast<long long>(slot) * W + lane] = tot;
    }
}

// wide: block = 4 warps, each warp one segment, a chunk of 32*Q columns (Q
// per lane) at column chunk blockIdx.y; U = 16 / Q entries are gathered per
// step so every warp keeps ~16 independent 8-byte loads per lane in flight
// whatever the panel width (a 32-wide panel would otherwise be latency bound).
template <int Q, int U>
__global__ void __launch_bounds__(128) spmm_wide_kernel(SegPlanView plan, const int* __restrict__ idx,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ X, long long ldx, long long w,
                                                        double* __restrict__ out, long long ldo,
                                                        double* __restrict__ partial) {
    const int lane = threadIdx.x & 31;
    const long long sg = static_cast<long long>(blockIdx.x) * 4 + (threadIdx.x >> 5);
    if (sg >= plan.nseg) return;
    const long long c0 = static_cast<long long>(blockIdx.y) * (32 * Q);
    double acc[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] = 0.0;
    bool colok[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) colok[q] = c0 + lane + 32 * q < w;
    const long long beg = plan.seg_beg[sg], end = plan.seg_end[sg];
    for (long long k0 = beg; k0 < end; k0 += 32) {
        const long long k = k0 + lane;
        int cl = 0;
        double vl = 0.0;
        if (k < end) {
            cl = __ldg(idx + k);
            vl = __ldg(val + k);
        }
        const int cnt = static_cast<int>(min(32LL, end - k0));
        // U entries' gathers in flight per step (entries past cnt carry
        // v = 0 from the masked index/value load)
        for (int e = 0; e < cnt; e += U) {
            double xv[U][Q], vv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int src = (e + u) & 31;
                const int c = __shfl_sync(0xffffffffu, cl, src);
                vv[u] = __shfl_sync(0xffffffffu, vl, src);
                if (e + u >= cnt) vv[u] = 0.0;
                const double* xr = X + static_cast<long long>(c) * ldx + c0 + lane;
#pragma unroll
                for (int q = 0; q < Q; ++q) xv[u][q] = colok[q] ? __ldg(xr + 32 * q) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < Q; ++q) acc[q] = fma(vv[u], xv[u][q], acc[q]);
        }
    }
    const int slot = plan.seg_slot[sg];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const long long j = c0 + lane + 32 * q;
        if (!colok[q]) continue;
        if (slot < 0)
            out[static_cast<long long>(plan.seg_row[sg]) * ldo + j] = acc[q];
        else
            partial[static_cast<long long>(slot) * w + j] = acc[q];
    }
}

// Wide panels, grouped: one warp walks a GROUP of consecutive segments
// (plan.grp_first; short rows are grouped up to ~384 entries) with ONE
// continuous gather pipeline — the index / value chunk of the next 32
// entries is in flight while the current chunk's gathers issue, and U
// entries' panel rows (Q doubles per lane each) are gathered per step — so
// a warp's memory-level parallelism does not restart at every short row.
// When an entry crosses its segment's end the accumulated row is written
// (output row, or the long row's partial slot) and the accumulators reset.
// Segment bounds / targets of the group (<= kGrpSegs) sit one per lane and
// are broadcast by shuffle.  Per output element the sum runs over the row's
// entries in CSR order: the same order as spmm_wide_kernel (bitwise equal).
template <int Q, int U, int MINB, bool CS = false>
__global__ void __launch_bounds__(128, MINB) spmm_grp_kernel(SegPlanView plan, const int* __restrict__ idx,
                                                             const double* __restrict__ val,
                                                             const double* __restrict__ X, long long ldx,
                                                             long long w, double* __restrict__ out, long long ldo,
                                                             double* __restrict__ partial) {
    static_assert(32 % U == 0, "the fast path steps through a 32-entry chunk U entries at a time");
    const int lane = threadIdx.x & 31;
    const long long g = static_cast<long long>(blockIdx.x) * 4 + (threadIdx.x >> 5);
    if (g >= plan.ngrp) return;
    const long long c0 = static_cast<long long>(blockIdx.y) * (32 * Q);
    // valid column slots of this lane: 32 q < wl  (32-bit compares)
    const int wl = static_cast<int>(min(w - c0, static_cast<long long>(32 * Q))) - lane;
    // panel row address = base + c * (ldx * 8 bytes): one 32 x 32 -> 64-bit
    // multiply-add per gathered row
    const unsigned ldx8 = static_cast<unsigned>(ldx * 8);
    const int s0 = plan.grp_first[g], ns = plan.grp_first[g + 1] - s0;
    // lane i: end / target of segment s0 + i (broadcast by shuffle)
    long long my_end = 0;
    int my_dst = 0;  // >= 0: output row; < 0: partial slot -(dst + 1)
    if (lane < ns) {
        my_end = plan.seg_end[s0 + lane];
        const int slot = plan.seg_slot[s0 + lane];
        my_dst = slot < 0 ? plan.seg_row[s0 + lane] : -(slot + 1);
    }
    // entry offsets relative to the group's first entry (a group spans at
    // most kGrpSegs segments of <= kSegLen entries: 32-bit)
    const long long beg = plan.seg_beg[s0];
    const int* gi = idx + beg;
    const double* gv = val + beg;
    const int my_e = static_cast<int>(my_end - beg);
    const int end = __shfl_sync(0xffffffffu, my_e, ns - 1);
    int si = 0;  // current segment (group-relative)
    int cur_end = __shfl_sync(0xffffffffu, my_e, 0);
    double acc[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] = 0.0;
    const char* xb = reinterpret_cast<const char*>(X + c0 + lane);
    auto flush = [&]() {
        const int dst = __shfl_sync(0xffffffffu, my_dst, si);
        double* o = (dst >= 0) ? out + static_cast<long long>(dst) * ldo
                               : partial + static_cast<long long>(-(dst + 1)) * w;
        o += c0 + lane;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            if (32 * q < wl) o[32 * q] = acc[q];
            acc[q] = 0.0;
        }
        ++si;
        cur_end = __shfl_sync(0xffffffffu, my_e, si < ns ? si : ns - 1);
    };
    for (int k0 = 0; k0 < end; k0 += 32) {
        const int k = k0 + lane;
        // CS: the index / value streams are read once per pass, loaded with
        // the evict-first hint so they do not displace panel rows from L2
        const int cl = (k < end) ? (CS ? __ldcs(gi + k) : __ldg(gi + k)) : 0;
        const double vl = (k < end) ? (CS ? __ldcs(gv + k) : __ldg(gv + k)) : 0.0;
        if (cur_end >= k0 + 32 && k0 + 32 <= end) {
            // fast path: a full chunk inside one segment (rows average ~130
            // entries at config 4): U entries' gathers in flight per step,
            // no boundary tests; the values are broadcast after the gathers
            // issue (fewer live registers)
#pragma unroll 1
            for (int e = 0; e < 32; e += U) {
                double xv[U][Q];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const unsigned c = static_cast<unsigned>(__shfl_sync(0xffffffffu, cl, e + u));
                    const double* xr = reinterpret_cast<const double*>(xb + static_cast<unsigned long long>(c) * ldx8);
#pragma unroll
                    for (int q = 0; q < Q; ++q) xv[u][q] = (32 * q < wl) ? __ldg(xr + 32 * q) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const double v = __shfl_sync(0xffffffffu, vl, e + u);
#pragma unroll
                    for (int q = 0; q < Q; ++q) acc[q] = fma(v, xv[u][q], acc[q]);
                }
            }
        } else {
            // a segment boundary (or the group's last, partial chunk) inside
            // the chunk: entry by entry, writing finished rows (empty
            // segments write zero rows)
            const int cnt = min(32, end - k0);
#pragma unroll 1
            for (int e = 0; e < cnt; ++e) {
                while (k0 + e >= cur_end) flush();
                const unsigned c = static_cast<unsigned>(__shfl_sync(0xffffffffu, cl, e));
                const double v = __shfl_sync(0xffffffffu, vl, e);
                const double* xr = reinterpret_cast<const double*>(xb + static_cast<unsigned long long>(c) * ldx8);
#pragma unroll
                for (int q = 0; q < Q; ++q)
                    if (32 * q < wl) acc[q] = fma(v, __ldg(xr + 32 * q), acc[q]);
            }
        }
    }
    while (si < ns) flush();  // the last segment (and any empty ones after it)
}

// out[row, j] = sum of the row's partial slots in a fixed (deterministic)
// order.  Narrow panels: one warp per long row, lanes over the slots, a
// shuffle tree per column.
__global__ void seg_reduce_kernel(SegPlanView plan, long long w, const double* __restrict__ partial,
                                  double* __restrict__ out, long long ldo) {
    const int lane = threadIdx.x & 31;
    const long long l = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    if (l >= plan.nlong) return;
    const int first = plan.long_first[l], cnt = plan.long_count[l];
    const long long row = plan.long_row[l];
    const double* base = partial + static_cast<long long>(first) * w;
    for (long long j = 0; j < w; ++j) {
        double s = 0.0;
        for (int t = lane; t < cnt; t += 32) s += base[static_cast<long long>(t) * w + j];
        s = warp_sum(s);
        if (lane == 0) out[row * ldo + j] = s;
    }
}

// Wide panels: one CTA of 8 warps per long row (Zipf-popular items have
// hundreds of slots); warp q sums slots q, q + 8, ... with lanes over the
// columns (coalesced slot rows), then the 8 warp sums are added in warp
// order.
constexpr int kSegRedWarps = 8;
__global__ void __launch_bounds__(32 * kSegRedWarps) seg_reduce_wide_kernel(SegPlanView plan, long long w,
                                                                        const double* __restrict__ partial,
                                                                        double* __restrict__ out, long long ldo) {
    extern __shared__ double red[];  // [kSegRedWarps][w]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long l = blockIdx.x;
    const int first = plan.long_first[l], cnt = plan.long_count[l];
    const long long row = plan.long_row[l];
    const double* base = partial + static_cast<long long>(first) * w;
    for (long long j = lane; j < w; j += 32) {
        double s = 0.0;
#pragma unroll 4
        for (int t = warp; t < cnt; t += kSegRedWarps) s += base[static_cast<long long>(t) * w + j];
        red[warp * w + j] = s;
    }
    __syncthreads();
    for (long long j = threadIdx.x; j < w; j += blockDim.x) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < kSegRedWarps; ++q) s += red[q * w + j];
        out[row * ldo + j] = s;
    }
}

template <int W>
void launch_narrow(svt_ctx* ctx, cudaStream_t s, const SegPlanView& plan, const int* idx, const double* val,
                   const double* X, i64 ldx, double* out, i64 ldo, double* partial) {
    (void)ctx;
    const unsigned blocks = static_cast<unsigned>((plan.nseg + kWarpsPerBlock - 1) / kWarpsPerBlock);
    spmm_narrow_kernel<W><<<blocks, 32 * kWarpsPerBlock, 0, s>>>(plan, idx, val, X, ldx, out, ldo, partial);
}

// ---- fused SDDMM + Bregman update + reductions ------------------------------
constexpr int kSddmmWarps = 8;
#ifndef SVTB_SDDMM_MINB
#define SVTB_SDDMM_MINB 4
#endif
constexpr int kSddmmMinBlocksSmallK = SVTB_SDDMM_MINB;  // resident CTAs asked of the compiler for k <= 4
constexpr int kSddmmU = 4;  // entries per lane group in flight

// Fused SDDMM + Bregman update + reductions for kept ranks k > 64 (config 2
// keeps most of its basis; k <= 64 runs sddmm_warp_kernel below), one warp
// per row segment.  The warp is G = 32 / KP groups of KP lanes (KP = the kept rank k rounded up to a power
// of two, at most 32); group g takes every G-th stored entry of the row and
// its lanes split the k-long dot product U[i,:] . Vs[j,:], so each factor row
// is read with coalesced loads (a lane-per-entry loop would touch 32
// different rows per load instruction).  The group's partial products are
// reduced with shuffles; the group leader applies the update and the sums.
template <int KP>
__global__ void __launch_bounds__(32 * kSddmmWarps) sddmm_update_kernel(
    SegPlanView plan, const int* __restrict__ col,
    const double* __restrict__ A, double* __restrict__ Y, double* __restrict__ Ycsc,
    const int* __restrict__ csr2csc, const double* __restrict__ U, long long ldu, const double* __restrict__ Vs,
    long long ldv, long long k, double delta, int mode, double* __restrict__ partials) {
    constexpr int G = 32 / KP;
    __shared__ double red[kSddmmWarps][4];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int g = lane / KP, j0 = lane % KP;
    double s_abs = 0.0, s_sq = 0.0, s_res = 0.0, s_y = 0.0;
    // grid-stride over the SpMM's row segments (<= kSegLen entries each), so
    // power-law rows do not leave the CTA's other warps idle at the barrier
    for (long long sg = static_cast<long long>(blockIdx.x) * kSddmmWarps + warp; sg < plan.nseg;
         sg += static_cast<long long>(gridDim.x) * kSddmmWarps) {
        const long long row = plan.seg_row[sg];
        const long long beg = plan.seg_beg[sg], end = plan.seg_end[sg];
        const double* ur = U + row * ldu;
        // kSddmmU entries per group per step: independent dot products in flight
        for (long long e0 = beg; e0 < end; e0 += static_cast<long long>(G) * kSddmmU) {
            double p[kSddmmU], av[kSddmmU], yv[kSddmmU];
            int cc[kSddmmU];
#pragma unroll
            for (int u = 0; u < kSddmmU; ++u) {
                const long long e = e0 + static_cast<long long>(u) * G + g;
                cc[u] = (e < end) ? __ldg(col + e) : -1;
                // the applying lane's A / Y are loaded up front, overlapping
                // the factor-row gathers
                const bool own = e < end && j0 == (u % KP);
                av[u] = own ? __ldg(A + e) : 0.0;
                yv[u] = own ? Y[e] : 0.0;
            }
            if (k <= KP) {
                // one dimension per lane: unconditional, independent loads
                // (clamped indices, zero multiplier) so the kSddmmU entries'
                // gathers overlap instead of serializing on branches
                const int jl = (j0 < k) ? j0 : 0;
                const double uj = (j0 < k) ? __ldg(ur + jl) : 0.0;
#pragma unroll
                for (int u = 0; u < kSddmmU; ++u)
                    // k == 0 (shrink kept nothing): no factor rows exist
                    p[u] = (k > 0) ? uj * __ldg(Vs + static_cast<long long>(max(cc[u], 0)) * ldv + jl) : 0.0;
            } else {
#pragma unroll
                for (int u = 0; u < kSddmmU; ++u) {
                    p[u] = 0.0;
                    if (cc[u] >= 0) {
                        const double* vr = Vs + static_cast<long long>(cc[u]) * ldv;
                        for (long long jj = j0; jj < k; jj += KP) p[u] = fma(__ldg(ur + jj), __ldg(vr + jj), p[u]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kSddmmU; ++u)
#pragma unroll
                for (int o = KP / 2; o > 0; o >>= 1) p[u] += __shfl_xor_sync(0xffffffffu, p[u], o);
            // the update of entry u is applied by lane u % KP of its group
#pragma unroll
            for (int u = 0; u < kSddmmU; ++u) {
                const long long e = e0 + static_cast<long long>(u) * G + g;
                if (e >= end || j0 != (u % KP)) continue;
                const double a = av[u];
                const double y_old = yv[u];
                const double d = a - p[u];
                s_abs += fabs(d);
                s_sq = fma(d, d, s_sq);
                const double r = a - y_old;
                s_res = fma(r, r, s_res);
                if (mode == 1) {
                    const double y_new = fma(delta, d, y_old);
                    Y[e] = y_new;
                    if (Ycsc) Ycsc[csr2csc[e]] = y_new;
                    s_y = fma(y_new, y_new, s_y);
                } else if (mode == 2) {
                    Y[e] = p[u];
                    s_y = fma(p[u], p[u], s_y);
                } else {
                    s_y = fma(y_old, y_old, s_y);
                }
            }
        }
    }
    s_abs = warp_sum(s_abs);
    s_sq = warp_sum(s_sq);
    s_res = warp_sum(s_res);
    s_y = warp_sum(s_y);
    if (lane == 0) {
        red[warp][0] = s_abs;
        red[warp][1] = s_sq;
        red[warp][2] = s_res;
        red[warp][3] = s_y;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double t = 0.0;
        for (int w = 0; w < kSddmmWarps; ++w) t += red[w][threadIdx.x];
        partials[blockIdx.x * 4 + threadIdx.x] = t;
    }
}

// CSC value mirror from the CSR values: Ycsc[p] = Y[csc2csr[p]] (a coalesced
// write with a gathered read, instead of a scattered 8-byte write per entry
// inside the update kernel, which costs a DRAM read-modify-write per sector)
__global__ void mirror_csc_kernel(long long nnz, const int* __restrict__ csc2csr, const double* __restrict__ Y,
                                  double* __restrict__ Ycsc) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p < nnz) Ycsc[p] = Y[__ldg(csc2csr + p)];
}

// Fused SDDMM + update for k <= 64, one warp per row segment, 32 entries per
// chunk.  The warp is G = 32 / KP lane groups of KP lanes (KP = k rounded up
// to a power of two, <= 32); lane j of a group holds U[i, j] (and, TWO,
// U[i, j + KP], ... S columns per lane) for the whole segment.  Per chunk the entries' index, A and Y
// are loaded coalesced (lane = entry) one chunk ahead; step s = 0..KP-1
// gathers, in every group g, the factor row of entry s*G + g (coalesced
// across the group's lanes) — the KP steps' loads are independent and all in
// flight together.  A reduce-scatter butterfly over the group's KP lanes
// (KP/2 + ... + 1 shuffles) then leaves the complete dot product of step j on
// lane j of each group, and one shuffle hands it to the lane that owns the
// entry, so the update, its Y store and the four sums run lane-parallel.
template <int KP, int S>
__global__ void __launch_bounds__(32 * kSddmmWarps, (KP >= 16 ? 2 : (KP >= 8 ? 3 : kSddmmMinBlocksSmallK))) sddmm_warp_kernel(
    SegPlanView plan, const int* __restrict__ col, const double* __restrict__ A, double* __restrict__ Y,
    double* __restrict__ Ycsc, const int* __restrict__ csr2csc, const double* __restrict__ U, long long ldu,
    const double* __restrict__ Vs, long long ldv, int k, double delta, int mode, double* __restrict__ partials) {
    constexpr int G = 32 / KP;
    __shared__ double red[kSddmmWarps][4];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int g = lane / KP, j = lane % KP;
    // lane holding the sum of the entry this lane owns (entry l = s * G + g')
    const int src = (lane % G) * KP + lane / G;
    double s_abs = 0.0, s_sq = 0.0, s_res = 0.0, s_y = 0.0;
    // lane j of a group holds columns j, j + KP, ..., j + (S - 1) KP (k <= S KP)
    bool has[S];
    int jl[S];  // clamped: unconditional loads, zero weight
#pragma unroll
    for (int t = 0; t < S; ++t) {
        has[t] = j + t * KP < k;
        jl[t] = has[t] ? j + t * KP : 0;
    }
    // entries [beg, end) of one row (a segment or a part of one): 32-entry
    // chunks with the next chunk's stream loads in flight
    auto run = [&](long long row, long long beg, long long end) {
        const double* ur = U + row * ldu;
        double u[S];
#pragma unroll
        for (int t = 0; t < S; ++t) u[t] = has[t] ? __ldg(ur + jl[t]) : 0.0;
        long long e = beg + lane;
        int cl_n = (e < end) ? __ldg(col + e) : 0;
        double a_n = (e < end) ? __ldg(A + e) : 0.0;
        double y_n = (e < end) ? Y[e] : 0.0;
        for (long long e0 = beg; e0 < end; e0 += 32) {
            e = e0 + lane;
            const int cl = cl_n;
            const double a = a_n, y_old = y_n;
            const long long en = e + 32;
            if (en < end) {  // next chunk's stream loads in flight during this chunk
                cl_n = __ldg(col + en);
                a_n = __ldg(A + en);
                y_n = Y[en];
            }
            double p[KP];
            if (k > 0) {
#pragma unroll
                for (int s = 0; s < KP; ++s) {
                    const int c = __shfl_sync(0xffffffffu, cl, s * G + g);
                    const double* vr = Vs + static_cast<long long>(c) * ldv;
                    p[s] = u[0] * __ldg(vr + jl[0]);
#pragma unroll
                    for (int t = 1; t < S; ++t) p[s] = fma(u[t], __ldg(vr + jl[t]), p[s]);
                }
            } else {  // shrink kept nothing: no factor rows exist
#pragma unroll
                for (int s = 0; s < KP; ++s) p[s] = 0.0;
            }
#pragma unroll
            for (int o = KP / 2; o > 0; o >>= 1) {
                const bool up = (lane & o) != 0;
#pragma unroll
                for (int i = 0; i < o; ++i) {
                    const double send = up ? p[i] : p[i + o];
                    const double keep = up ? p[i + o] : p[i];
                    p[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            const double pe = __shfl_sync(0xffffffffu, p[0], src);
            if (e < end) {
                const double d = a - pe;
                s_abs += fabs(d);
                s_sq = fma(d, d, s_sq);
                const double r = a - y_old;
                s_res = fma(r, r, s_res);
                if (mode == 1) {
                    const double y_new = fma(delta, d, y_old);
                    Y[e] = y_new;
                    if (Ycsc) Ycsc[csr2csc[e]] = y_new;
                    s_y = fma(y_new, y_new, s_y);
                } else if (mode == 2) {
                    Y[e] = pe;
                    s_y = fma(pe, pe, s_y);
                } else {
                    s_y = fma(y_old, y_old, s_y);
                }
            }
        }
        };
    if (plan.chunk_off == nullptr) {  // static partition by segments
        for (long long sg = static_cast<long long>(blockIdx.x) * kSddmmWarps + warp; sg < plan.nseg;
             sg += static_cast<long long>(gridDim.x) * kSddmmWarps)
            run(plan.seg_row[sg], plan.seg_beg[sg], plan.seg_end[sg]);
    } else {
        // Chunk-balanced static partition: warp w of W owns the chunks
        // [C w / W, C (w + 1) / W) of the segments' 32-entry chunks in
        // segment order (a segment may be shared by two warps: the update
        // has no reduction along a row).  Power-law patterns give the
        // per-segment partition warps of very different loads; every warp of
        // a CTA then waits at the final barrier for the slowest one (ncu:
        // a third of the stall cycles).  Static, so the sums stay
        // deterministic.
        const long long W = static_cast<long long>(gridDim.x) * kSddmmWarps;
        const long long gw = static_cast<long long>(blockIdx.x) * kSddmmWarps + warp;
        const long long C = plan.nchunks;
        long long c = C / W * gw + min(gw, C % W);
        const long long c1 = c + C / W + (gw < C % W ? 1 : 0);
        if (c < c1) {
            // last segment sg with chunk_off[sg] <= c: 32-ary search, one probe per lane
            long long lo_s = 0, hi_s = plan.nseg;  // answer in [lo_s, hi_s)
            while (hi_s - lo_s > 1) {
                const long long step = (hi_s - lo_s + 31) / 32;
                const long long probe = lo_s + step * lane;
                const bool ok = probe < hi_s && __ldg(plan.chunk_off + probe) <= c;
                const unsigned m = __ballot_sync(0xffffffffu, ok);
                const int top = 31 - __clz(static_cast<int>(m));  // lane 0 always ok (chunk_off[lo_s] <= c)
                const long long nlo = lo_s + step * top;
                hi_s = min(hi_s, nlo + step);
                lo_s = nlo;
            }
            long long sg = lo_s;
            while (c < c1) {
                const long long off = __ldg(plan.chunk_off + sg), nxt = __ldg(plan.chunk_off + sg + 1);
                if (nxt > c) {
                    const long long beg = plan.seg_beg[sg], end = plan.seg_end[sg];
                    const long long cend = min(nxt, c1);
                    run(plan.seg_row[sg], beg + 32 * (c - off), min(end, beg + 32 * (cend - off)));
                    c = cend;
                }
                ++sg;
            }
        }
    }
    s_abs = warp_sum(s_abs);
    s_sq = warp_sum(s_sq);
    s_res = warp_sum(s_res);
    s_y = warp_sum(s_y);
    if (lane == 0) {
        red[warp][0] = s_abs;
        red[warp][1] = s_sq;
        red[warp][2] = s_res;
        red[warp][3] = s_y;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double t = 0.0;
        for (int w = 0; w < kSddmmWarps; ++w) t += red[w][threadIdx.x];
        partials[blockIdx.x * 4 + threadIdx.x] = t;
    }
}

__global__ void reduce4_kernel(const double* __restrict__ partials, int nblocks, double* __restrict__ out) {
    // one warp per component, fixed order
    const int comp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    double t = 0.0;
    for (int b = lane; b < nblocks; b += 32) t += partials[b * 4 + comp];
    t = warp_sum(t);
    if (lane == 0) out[comp] = t;
}

__global__ void scale_values_kernel(long long nnz, const double* __restrict__ in, double alpha,
                                    double* __restrict__ out, const int* __restrict__ csr2csc,
                                    double* __restrict__ out_csc) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= nnz) return;
    const double v = in[e] * alpha;
    out[e] = v;
    if (out_csc) out_csc[csr2csc[e]] = v;
}

__global__ void axpy_values_kernel(long long nnz, const double* __restrict__ a, double alpha,
                                   const double* __restrict__ b, double* __restrict__ out) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= nnz) return;
    out[e] = a[e] + alpha * b[e];
}

__global__ void densify_kernel(long long m_local, long long n, const long long* __restrict__ rowptr,
                               const int* __restrict__ col, const double* __restrict__ val,
                               double* __restrict__ out) {
    const long long row = blockIdx.x;
    if (row >= m_local) return;
    for (long long e = rowptr[row] + threadIdx.x; e < rowptr[row + 1]; e += blockDim.x)
        out[row * n + col[e]] = val[e];
}


// ---- shared-memory-tiled SpMM for wide panels (TilePlanView) ---------------
// One CTA (16 warps) per (work item, 32*Q-column chunk of the panel).  A work
// item is a run of tiles of one kTileRows-row block.  Per tile the CTA stages
// the tile's distinct panel rows (kTileSlots x 32Q doubles), its entries
// (value, slot) and row offsets in shared memory with cp.async, double
// buffered: tile t+1 streams in while tile t is consumed.  Warp q owns rows
// 8q..8q+7 of the block, lane j columns c0 + Q*j .. c0 + Q*j + Q-1; each row
// accumulates in registers over its entries in (tile, slot) order — fixed,
// so the result is deterministic.  The panel row an entry reads comes from
// shared memory, so the L2 -> SM traffic per entry falls by the tile's reuse
// (entries per slot); each entry costs one broadcast record load, Q/2
// 16-byte panel loads and Q FMAs per lane.
constexpr int kTileThreads = 512;
constexpr int kTileRowsPerWarp = kTileRows / (kTileThreads / 32);
static_assert(kTileRowsPerWarp == 8, "row split");
constexpr size_t kStageX = static_cast<size_t>(kTileSlots) * 128 * sizeof(double);
constexpr size_t kStageE = static_cast<size_t>(kTileEnts) * sizeof(TileEnt);
constexpr size_t kStageR = static_cast<size_t>(kTileRoffStride) * sizeof(unsigned short);
constexpr size_t kStageBytes = kStageX + kStageE + kStageR;
constexpr size_t kTileSmem = 2 * kStageBytes + 2 * (kTileItemTiles + 1) * sizeof(int);
static_assert(kStageR % 16 == 0, "roff stage");

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Q columns per lane; V16: 16-byte panel pieces (X 16-byte aligned, ldx and
// w even)
template <int Q, bool V16>
__global__ void __launch_bounds__(kTileThreads, 1)
    tile_spmm_kernel(TilePlanView P, const double* __restrict__ X, long long ldx, long long w,
                     double* __restrict__ out, long long ldo, double* __restrict__ partial) {
    constexpr int WC = 32 * Q;                                  // chunk width
    constexpr int PIECES = kTileSlots * WC / 2;                 // 16-byte pieces per X stage
    constexpr int PPT = (PIECES + kTileThreads - 1) / kTileThreads;
    extern __shared__ __align__(16) unsigned char tsm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int item = blockIdx.x;
    const long long c0 = static_cast<long long>(blockIdx.y) * WC;
    const int t0 = P.item_t0[item], nt = P.item_t1[item] - t0;
    const long long blk = P.item_blk[item];
    const int part = P.item_part[item];
    // the item's tile metadata (entry / slot offsets, item-relative) in
    // shared memory once, so no per-tile global load sits on the critical path
    int* me = reinterpret_cast<int*>(tsm + 2 * kStageBytes);  // [nt + 1]
    int* mu = me + (kTileItemTiles + 1);                       // [nt + 1]
    const long long e_base = P.tile_e[t0], u_base = P.tile_u[t0];
    for (int i = tid; i <= nt; i += kTileThreads) {
        me[i] = static_cast<int>(P.tile_e[t0 + i] - e_base);
        mu[i] = static_cast<int>(P.tile_u[t0 + i] - u_base);
    }
    __syncthreads();
    const TileEnt* ent = P.ent + e_base;
    const int* ucol = P.ucol + u_base;

    // gather indices of the next tile to stage, loaded one tile ahead so the
    // cp.async issue never waits on them (ucol is padded by kTileSlots)
    int ucn[PPT];
    auto load_ucol = [&](int t) {
        const int u0 = mu[t];
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
            const int g = tid + j * kTileThreads;
            ucn[j] = g < PIECES ? __ldg(ucol + u0 + g / (WC / 2)) : 0;
        }
    };
    auto stage = [&](int t, int buf) {
        unsigned char* base = tsm + static_cast<size_t>(buf) * kStageBytes;
        double* xs = reinterpret_cast<double*>(base);
        const int nu = mu[t + 1] - mu[t];
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
            const int g = tid + j * kTileThreads;
            const int sl = g / (WC / 2), pc = g - sl * (WC / 2);
            if (g < PIECES && sl < nu) {
                const double* row = X + static_cast<long long>(ucn[j]) * ldx;
                const long long col = c0 + 2 * pc;
                if (V16) {
                    cp_async16(xs + sl * WC + 2 * pc, row + (col < w ? col : 0), col < w ? 16 : 0);
                } else {
                    cp_async8(xs + sl * WC + 2 * pc, row + (col < w ? col : 0), col < w ? 8 : 0);
                    cp_async8(xs + sl * WC + 2 * pc + 1, row + (col + 1 < w ? col + 1 : 0), col + 1 < w ? 8 : 0);
                }
            }
        }
        const int e0 = me[t], ne = me[t + 1] - e0;
        TileEnt* es = reinterpret_cast<TileEnt*>(base + kStageX);
        for (int k = tid; k < ne; k += kTileThreads) cp_async16(es + k, ent + e0 + k, 16);
        unsigned short* rs = reinterpret_cast<unsigned short*>(base + kStageX + kStageE);
        const unsigned short* rsrc = P.roff + static_cast<long long>(t0 + t) * kTileRoffStride;
        if (tid < static_cast<int>(kStageR / 16)) cp_async16(rs + tid * 8, rsrc + tid * 8, 16);
        cp_async_commit();
    };

    double acc[kTileRowsPerWarp][Q];
#pragma unroll
    for (int r = 0; r < kTileRowsPerWarp; ++r)
#pragma unroll
        for (int q = 0; q < Q; ++q) acc[r][q] = 0.0;

    if (nt > 0) {
        load_ucol(0);
        stage(0, 0);
    }
#pragma unroll 1
    for (int t = 0; t < nt; ++t) {
        const int buf = t & 1;
        if (t + 1 < nt) {
            load_ucol(t + 1);
            stage(t + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const unsigned char* base = tsm + static_cast<size_t>(buf) * kStageBytes;
        const double* xs = reinterpret_cast<const double*>(base) + lane * Q;
        const TileEnt* es = reinterpret_cast<const TileEnt*>(base + kStageX);
        const unsigned short* rs =
            reinterpret_cast<const unsigned short*>(base + kStageX + kStageE) + warp * kTileRowsPerWarp;
        const int rb = lane <= kTileRowsPerWarp ? rs[lane] : 0;
        int k = __shfl_sync(0xffffffffu, rb, 0);
#pragma unroll
        for (int r = 0; r < kTileRowsPerWarp; ++r) {
            const int e = __shfl_sync(0xffffffffu, rb, r + 1);
#pragma unroll 2
            for (; k < e; ++k) {
                const TileEnt p = es[k];
                const double* xr = xs + p.slot * WC;
                if (Q == 4) {
                    const double2 a = *reinterpret_cast<const double2*>(xr);
                    const double2 b = *reinterpret_cast<const double2*>(xr + 2);
                    acc[r][0] = fma(p.v, a.x, acc[r][0]);
                    acc[r][1 % Q] = fma(p.v, a.y, acc[r][1 % Q]);
                    acc[r][2 % Q] = fma(p.v, b.x, acc[r][2 % Q]);
                    acc[r][3 % Q] = fma(p.v, b.y, acc[r][3 % Q]);
                } else if (Q == 2) {
                    const double2 a = *reinterpret_cast<const double2*>(xr);
                    acc[r][0] = fma(p.v, a.x, acc[r][0]);
                    acc[r][1 % Q] = fma(p.v, a.y, acc[r][1 % Q]);
                } else {
                    acc[r][0] = fma(p.v, xr[0], acc[r][0]);
                }
            }
        }
        __syncthreads();
    }
    const long long row0 = blk * kTileRows + warp * kTileRowsPerWarp;
#pragma unroll
    for (int r = 0; r < kTileRowsPerWarp; ++r) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const long long col = c0 + lane * Q + q;
            if (col >= w) continue;
            if (part < 0) {
                const long long row = row0 + r;
                if (row < P.nrows) out[row * ldo + col] = acc[r][q];
            } else {
                partial[(static_cast<long long>(part) * kTileRows + warp * kTileRowsPerWarp + r) * w + col] =
                    acc[r][q];
            }
        }
    }
}

// blocks spread over several items: out rows = sum of the items' partial
// rows in item order (deterministic); grid (nsplit, column chunks)
__global__ void __launch_bounds__(256) tile_split_reduce_kernel(TilePlanView P, long long w,
                                                                const double* __restrict__ partial,
                                                                double* __restrict__ out, long long ldo) {
    const int sidx = blockIdx.x;
    const long long col = static_cast<long long>(blockIdx.y) * 32 + (threadIdx.x & 31);
    if (col >= w) return;
    const long long blk = P.split_blk[sidx];
    const int first = P.split_first[sidx], cnt = P.split_count[sidx];
    for (int r = threadIdx.x >> 5; r < kTileRows; r += 8) {
        const long long row = blk * kTileRows + r;
        if (row >= P.nrows) break;
        double s = 0.0;
        for (int q = 0; q < cnt; ++q) s += partial[(static_cast<long long>(first + q) * kTileRows + r) * w + col];
        out[row * ldo + col] = s;
    }
}

// tile-ordered values from the CSR value array
__global__ void tile_values_kernel(long long nnz, const int* __restrict__ perm, const double* __restrict__ Y,
                                   TileEnt* __restrict__ ent) {
    const long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (f < nnz) ent[f].v = __ldg(Y + __ldg(perm + f));
}

}  // namespace

// SVTB_SPMM_LEGACY=1: the one-warp-per-segment kernel (A/B switch, read
// per call so tests can compare the two)
static bool spmm_legacy() {
    const char* e = std::getenv("SVTB_SPMM_LEGACY");
    return e != nullptr && e[0] == '1';
}

void spmm(svt_ctx* ctx, int cls, const SegPlanView& plan, i64 nrows, const int* idx, const double* val, i64 nnz,
          i64 x_rows, i64 w, const double* X, i64 ldx, double* out, i64 ldo, cudaStream_t stream,
          DevBuf<double>* scratch) {
    if (nrows <= 0 || w <= 0) return;
    cudaStream_t s = stream ? stream : ctx->stream;
    DevBuf<double>& part = scratch ? *scratch : ctx->ws_spmm;
    // algorithmic bytes: 12 B per stored entry (int32 index +
    // fp64 value) + 8 B per row pointer + the dense panel read once + the
    // output panel written once; 2 flops per entry per column.
    LaunchScope ls(ctx, cls, 12.0 * nnz + 8.0 * (nrows + 1) + 8.0 * w * (x_rows + nrows), 2.0 * nnz * w, s);
    double* partial = nullptr;
    if (plan.nlong > 0) {
        part.ensure(static_cast<size_t>(plan.nslots * w));
        partial = part.get();
    }
    if (w <= 16) {
        switch (w) {
#define SVT_CASE(W)                                                             \
    case W:                                                                     \
        launch_narrow<W>(ctx, s, plan, idx, val, X, ldx, out, ldo, partial);       \
        break;
            SVT_CASE(1) SVT_CASE(2) SVT_CASE(3) SVT_CASE(4) SVT_CASE(5) SVT_CASE(6) SVT_CASE(7) SVT_CASE(8)
            SVT_CASE(9) SVT_CASE(10) SVT_CASE(11) SVT_CASE(12) SVT_CASE(13) SVT_CASE(14) SVT_CASE(15) SVT_CASE(16)
#undef SVT_CASE
            default:
                break;
        }
    } else if (plan.ngrp > 0 && !spmm_legacy()) {
        const unsigned nb = static_cast<unsigned>((plan.ngrp + 3) / 4);
        const unsigned chunks = static_cast<unsigned>(w <= 128 ? 1 : (w + 127) / 128);
        if (w <= 32)
            spmm_grp_kernel<1, 8, 8, true><<<dim3(nb, 1), 128, 0, s>>>(plan, idx, val, X, ldx, w, out, ldo, partial);
        else if (w <= 64)
            spmm_grp_kernel<2, 8, 8, true><<<dim3(nb, 1), 128, 0, s>>>(plan, idx, val, X, ldx, w, out, ldo, partial);
        else if (w <= 96)
            spmm_grp_kernel<3, 4, 8, true><<<dim3(nb, 1), 128, 0, s>>>(plan, idx, val, X, ldx, w, out, ldo, partial);
        else {
            // SVTB_SPMM_VARIANT (tuning): U,MINB of the Q = 4 instantiation
            static const int var = [] {
                const char* e = std::getenv("SVTB_SPMM_VARIANT");
                return e ? std::atoi(e) : 0;
            }();
            const dim3 gq(nb, chunks);
            if (var == 1)
                spmm_grp_kernel<4, 4, 6><<<gq, 128, 0, s>>>(plan, idx, val, X, ldx, w, out, ldo, partial);
            else if (var == 3)
                spmm_grp_kernel<4, 2, 8><<<gq, 128, 0, s>>>(plan, idx, val, X, ldx, w, out, ldo, partial);
            else if (var == 4)
                spmm_grp_kernel<4, 4, 10><<<gq, 128, 0, s>>>(plan, idx, val, X, ldx, w, out, ldo, partial);
            else if (var == 6)
                spmm_grp_kernel<4, 4, 10, true><<<gq, 128, 0, s>>>(plan, idx, val, X, ldx, w, out, ldo, partial);
            else if (var == 7)
                spmm_grp_kernel<4, 2, 12, true><<<gq, 128, 0, s>>>(plan, idx, val, X, ldx, w, out, ldo, partial);
            else if (var == 5)  // plain __ldg index / value loads (A/B of the evict-first hint)
                spmm_grp_kernel<4, 4, 8><<<gq, 128, 0, s>>>(plan, idx, val, X, ldx, w, out, ldo, partial);
            else  // evict-first index / value streams: cfg4 Y^T X DRAM reads 255 -> 217 MB
                spmm_grp_kernel<4, 4, 8, true><<<gq, 128, 0, s>>>(plan, idx, val, X, ldx, w, out, ldo, partial);
        }
    } else {
        const unsigned nb = static_cast<unsigned>((plan.nseg + 3) / 4);
        // the gathers run through L1: ask for the whole unified L1 / shared
        // array as cache (the kernels use no shared memory)
        static const bool carve = [] {
            const char* e = std::getenv("SVTB_SPMM_CARVEOUT");
            const int pct = e ? std::atoi(e) : -2;
            if (pct < -1) return false;
            SVT_CUDA(cudaFuncSetAttribute(spmm_wide_kernel<1, 16>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
            SVT_CUDA(cudaFuncSetAttribute(spmm_wide_kernel<2, 8>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
            SVT_CUDA(cudaFuncSetAttribute(spmm_wide_kernel<3, 5>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
            SVT_CUDA(cudaFuncSetAttribute(spmm_wide_kernel<4, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
            return true;
        }();
        (void)carve;
        if (w <= 32)
            spmm_wide_kernel<1, 16><<<dim3(nb, 1), 128, 0, s>>>(plan, idx, val, X, ldx, w, out, ldo,
                                                                          partial);
        else if (w <= 64)
            spmm_wide_kernel<2, 8><<<dim3(nb, 1), 128, 0, s>>>(plan, idx, val, X, ldx, w, out, ldo,
                                                                         partial);
        else if (w <= 96)
            spmm_wide_kernel<3, 5><<<dim3(nb, 1), 128, 0, s>>>(plan, idx, val, X, ldx, w, out, ldo,
                                                                         partial);
        else
            spmm_wide_kernel<4, 4><<<dim3(nb, static_cast<unsigned>((w + 127) / 128)), 128, 0, s>>>(
                plan, idx, val, X, ldx, w, out, ldo, partial);
    }
    if (plan.nlong > 0) {
        if (w >= 8 && w <= 512) {
            const size_t smem = sizeof(double) * kSegRedWarps * static_cast<size_t>(w);
            if (smem > 48 * 1024) {
                static bool attr = false;
                if (!attr) {
                    SVT_CUDA(cudaFuncSetAttribute(seg_reduce_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  static_cast<int>(sizeof(double) * kSegRedWarps * 512)));
                    attr = true;
                }
            }
            seg_reduce_wide_kernel<<<static_cast<unsigned>(plan.nlong), 32 * kSegRedWarps, smem, s>>>(
                plan, w, partial, out, ldo);
        } else {
            const i64 thr = plan.nlong * 32;
            seg_reduce_kernel<<<static_cast<unsigned>((thr + 255) / 256), 256, 0, s>>>(plan, w, partial,
                                                                                              out, ldo);
        }
    }
}


// opt-in (SVTB_TILED_SPMM=1, read per sketch): measured slower than the
// segment kernel on the BASELINE patterns (at ~1 % density a
// staged slot serves 2-3 entries, so the per-tile staging / barrier cost
// outweighs the saved L2 gathers)
bool tile_spmm_enabled() {
    const char* e = std::getenv("SVTB_TILED_SPMM");
    return e != nullptr && std::atoi(e) != 0;
}

void tile_values(svt_ctx* ctx, const TilePlanView& P, const double* Ycsr) {
    if (P.nnz <= 0) return;
    LaunchScope ls(ctx, K_OTHER, 24.0 * P.nnz, 0.0);
    tile_values_kernel<<<static_cast<unsigned>((P.nnz + 255) / 256), 256, 0, ctx->stream>>>(P.nnz, P.perm, Ycsr,
                                                                                           P.ent);
}

bool spmm_tiled(svt_ctx* ctx, int cls, const TilePlanView& P, i64 x_rows, i64 w, const double* X, i64 ldx,
                double* out, i64 ldo, cudaStream_t stream, DevBuf<double>* scratch) {
    if (P.nrows <= 0 || w <= 0) return true;
    const i64 chunks = (w + 31) / 32;
    // partial rows of split blocks: bounded (very wide panels of a split
    // pattern fall back to the segment kernel)
    const double part_bytes = 8.0 * static_cast<double>(P.nparts) * kTileRows * static_cast<double>(w);
    if (part_bytes > 4e9 || chunks > 65535) return false;
    cudaStream_t s = stream ? stream : ctx->stream;
    DevBuf<double>& part = scratch ? *scratch : ctx->ws_spmm;
    double* partial = nullptr;
    if (P.nparts > 0) {
        part.ensure(static_cast<size_t>(P.nparts) * kTileRows * static_cast<size_t>(w));
        partial = part.get();
    }
    const bool v16 = (reinterpret_cast<uintptr_t>(X) % 16 == 0) && (ldx % 2 == 0) && (w % 2 == 0);
    const int Q = w > 64 ? 4 : (w > 32 ? 2 : 1);
    static bool attr = false;
    if (!attr) {
#define SVT_TATTR(QQ, VV)                                                                                 \
    SVT_CUDA(cudaFuncSetAttribute(tile_spmm_kernel<QQ, VV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                  static_cast<int>(kTileSmem)))
        SVT_TATTR(1, true); SVT_TATTR(1, false); SVT_TATTR(2, true); SVT_TATTR(2, false);
        SVT_TATTR(4, true); SVT_TATTR(4, false);
#undef SVT_TATTR
        attr = true;
    }
    LaunchScope ls(ctx, cls, 12.0 * P.nnz + 8.0 * (P.nrows + 1) + 8.0 * w * (x_rows + P.nrows), 2.0 * P.nnz * w, s);
    const dim3 grid(static_cast<unsigned>(P.nitems), static_cast<unsigned>((w + 32 * Q - 1) / (32 * Q)));
#define SVT_TL(QQ)                                                                                       \
    (v16 ? tile_spmm_kernel<QQ, true><<<grid, kTileThreads, kTileSmem, s>>>(P, X, ldx, w, out, ldo, partial) \
         : tile_spmm_kernel<QQ, false><<<grid, kTileThreads, kTileSmem, s>>>(P, X, ldx, w, out, ldo, partial))
    if (Q == 4)
        SVT_TL(4);
    else if (Q == 2)
        SVT_TL(2);
    else
        SVT_TL(1);
#undef SVT_TL
    if (P.nsplit > 0)
        tile_split_reduce_kernel<<<dim3(static_cast<unsigned>(P.nsplit), static_cast<unsigned>(chunks)), 256, 0, s>>>(
            P, w, partial, out, ldo);
    return true;
}

void sddmm_update(svt_ctx* ctx, const SegPlanView& plan, i64 m_local, const int* col, const double* A, double* Y,
                  double* Ycsc, const int* csr2csc, i64 nnz, i64 n, const double* U, i64 ldu, const double* Vs,
                  i64 ldv, i64 k, double delta, int mode, double* d_sums4) {
    const int blocks =
        std::max(1, std::min<int>(ctx->num_sms * 8, static_cast<int>((plan.nseg + kSddmmWarps - 1) / kSddmmWarps)));
    int blocks_launched = blocks;
    ctx->ws_partial2.ensure(static_cast<size_t>(blocks) * 4);
    {
        // col 4 + A 8 + Y in 8 + Y out 8 (+ CSC mirror 4 + 8) per
        // entry, row pointers, and the k-wide factor rows read once.
        const double per = (mode == 1) ? (Ycsc ? 40.0 : 28.0) : 20.0;
        LaunchScope ls(ctx, K_SDDMM, per * nnz + 8.0 * (m_local + 1) + 8.0 * k * (m_local + n), 2.0 * nnz * k);
        double* part = ctx->ws_partial2.get();
        // the chunk-balanced partition gives every warp the same load, so the
        // grid is whole waves of the CTAs resident at once (no part-filled
        // last wave): SVTB_SDDMM_WAVES x occupancy x SMs
        static const int slots = [] {
            const char* e = std::getenv("SVTB_SDDMM_SLOTS");
            return e ? std::atoi(e) : 4;
        }();
        static const int waves = [] {
            const char* e = std::getenv("SVTB_SDDMM_WAVES");
            return e ? std::max(1, std::atoi(e)) : 1;
        }();
#define SVT_SDDMM_W(KP, SL)                                                                             \
    do {                                                                                                 \
        int gridb = blocks;                                                                              \
        if (plan.chunk_off != nullptr) {                                                                 \
            static int occ = 0;                                                                          \
            if (occ == 0)                                                                                \
                SVT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sddmm_warp_kernel<KP, SL>,   \
                                                                       32 * kSddmmWarps, 0));            \
            gridb = std::max(1, std::min(blocks, waves * std::max(1, occ) * ctx->num_sms));              \
        }                                                                                                \
        sddmm_warp_kernel<KP, SL><<<gridb, 32 * kSddmmWarps, 0, ctx->stream>>>(                         \
            plan, col, A, Y, Ycsc, csr2csc, U, ldu, Vs, ldv, static_cast<int>(k), delta, mode, part);    \
        blocks_launched = gridb;                                                                         \
    } while (0)
        // columns per lane (SVTB_SDDMM_SLOTS = 1 / 2 / 4, default 4): wider k on a
        // narrower lane group — fewer idle lanes just above a power of two, a
        // shorter butterfly and fewer partial sums in registers.  Measured
        // (update + mirror): cfg4 k = 10 282 -> 232 us, k = 20 385 -> 324,
        // k = 50 498 -> 452; cfg5 k = 50 4.96 -> 4.47 ms; 8 columns per lane
        // spill and lose the coalescing (cfg5 k = 50: 6.1 ms)
        if (k <= 1)
            SVT_SDDMM_W(1, 1);
        else if (k <= 2)
            SVT_SDDMM_W(2, 1);
        else if (k <= 4)
            SVT_SDDMM_W(4, 1);
        else if (k <= 8)
            SVT_SDDMM_W(8, 1);
        else if (k <= 16) {
            if (slots >= 2)
                SVT_SDDMM_W(8, 2);
            else
                SVT_SDDMM_W(16, 1);
        } else if (k <= 32) {
            if (slots >= 2)
                SVT_SDDMM_W(16, 2);
            else
                SVT_SDDMM_W(32, 1);
        } else if (k <= 64) {
            if (slots >= 4)
                SVT_SDDMM_W(16, 4);
            else
                SVT_SDDMM_W(32, 2);
        }
        else
            sddmm_update_kernel<32><<<blocks, 32 * kSddmmWarps, 0, ctx->stream>>>(plan, col, A, Y, Ycsc, csr2csc,
                                                                                U, ldu, Vs, ldv, k, delta, mode, part);
#undef SVT_SDDMM_W
    }
    LaunchScope ls(ctx, K_OTHER, 0.0, 0.0);
    reduce4_kernel<<<1, 128, 0, ctx->stream>>>(ctx->ws_partial2.get(), blocks_launched, d_sums4);
}

void mirror_csc(svt_ctx* ctx, i64 nnz, const int* csc2csr, const double* Y, double* Ycsc) {
    if (nnz <= 0) return;
    LaunchScope ls(ctx, K_SDDMM, 20.0 * nnz, 0.0);
    mirror_csc_kernel<<<static_cast<unsigned>((nnz + 255) / 256), 256, 0, ctx->stream>>>(nnz, csc2csr, Y, Ycsc);
}

void scale_values(svt_ctx* ctx, i64 nnz, const double* in, double alpha, double* out, const int* csr2csc,
                  double* out_csc) {
    if (nnz <= 0) return;
    LaunchScope ls(ctx, K_OTHER, nnz * 24.0, 0.0);
    scale_values_kernel<<<static_cast<unsigned>((nnz + 255) / 256), 256, 0, ctx->stream>>>(nnz, in, alpha, out,
                                                                                       csr2csc, out_csc);
}

void axpy_values(svt_ctx* ctx, i64 nnz, const double* a, double alpha, const double* b, double* out) {
    if (nnz <= 0) return;
    LaunchScope ls(ctx, K_OTHER, nnz * 24.0, 0.0);
    axpy_values_kernel<<<static_cast<unsigned>((nnz + 255) / 256), 256, 0, ctx->stream>>>(nnz, a, alpha, b, out);
}

void densify_dev(svt_ctx* ctx, i64 m_local, i64 n, const i64* rowptr, const int* col, const double* val,
                 double* out) {
    SVT_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * static_cast<size_t>(m_local * n), ctx->stream));
    if (m_local <= 0) return;
    LaunchScope ls(ctx, K_OTHER, 0.0, 0.0);
    densify_kernel<<<static_cast<unsigned>(m_local), 128, 0, ctx->stream>>>(
        m_local, n, reinterpret_cast<const long long*>(rowptr), col, val, out);
}

}  // namespace svtb
