// Device-side construction of a rank's sample set (SampledMatrix storage,
// sampled.hpp:25-110): validation of the uploaded CSR, the CSC view by a
// stable radix sort of the column indices (rows stay ascending inside every
// column, exactly the order of the host counting sort it replaces), the
// csr2csc permutation, the CSC value mirror, and both segment plans of the
// load-balanced SpMM.  Only the CSR arrays cross PCIe; everything derived
// from them is built in HBM.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cub/cub.cuh>

#include "common.hpp"
#include "engine.hpp"

namespace svtb {

namespace {

// col int64 -> int32 with range check, value finiteness check.
__global__ void convert_validate_kernel(long long nnz, long long n, const long long* __restrict__ col64,
                                        const double* __restrict__ val, int* __restrict__ col32,
                                        int* __restrict__ iota, int* __restrict__ bad) {
    const long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (k >= nnz) return;
    const long long c = col64[k];
    if (c < 0 || c >= n) atomicOr(bad, 1);
    if (!isfinite(val[k])) atomicOr(bad, 2);
    col32[k] = static_cast<int>(c < 0 ? 0 : (c >= n ? n - 1 : c));
    iota[k] = static_cast<int>(k);
}

// row index of every CSR entry (one warp per row)
__global__ void row_ids_kernel(long long rows, const long long* __restrict__ ptr, int* __restrict__ rid) {
    const long long r = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    for (long long k = ptr[r] + lane; k < ptr[r + 1]; k += 32) rid[k] = static_cast<int>(r);
}

// column counts from the sorted column keys: colptr[j] = first position of
// column j (lower bound), colptr[n] = nnz
__global__ void colptr_kernel(long long nnz, long long n, const int* __restrict__ sorted_col,
                              long long* __restrict__ colptr) {
    const long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (j > n) return;
    long long lo = 0, hi = nnz;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (sorted_col[mid] < j)
            lo = mid + 1;
        else
            hi = mid;
    }
    colptr[j] = lo;
}

__global__ void csc_fill_kernel(long long nnz, const int* __restrict__ perm, const int* __restrict__ rid,
                                const double* __restrict__ val, int* __restrict__ cscrow,
                                double* __restrict__ val_csc, int* __restrict__ csr2csc) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= nnz) return;
    const int k = perm[p];
    cscrow[p] = rid[k];
    val_csc[p] = val[k];
    csr2csc[k] = static_cast<int>(p);
}

// plan pass 1: per row the number of segments (>= 1), long flag, slot count
__global__ void plan_count_kernel(long long rows, const long long* __restrict__ ptr, int* __restrict__ nseg,
                                  int* __restrict__ islong, int* __restrict__ nslot) {
    const long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (r >= rows) return;
    const long long len = ptr[r + 1] - ptr[r];
    const bool lg = len > kSegLen;
    const int ns = lg ? static_cast<int>((len + kSegLen - 1) / kSegLen) : 1;
    nseg[r] = ns;
    islong[r] = lg ? 1 : 0;
    nslot[r] = lg ? ns : 0;
}

// plan pass 2: fill the segment and long-row arrays (same order as the host
// builder: rows ascending, a long row's segments consecutive)
__global__ void plan_fill_kernel(long long rows, const long long* __restrict__ ptr, const int* __restrict__ nseg,
                                 const int* __restrict__ segoff, const int* __restrict__ islong,
                                 const int* __restrict__ longoff, const int* __restrict__ slotoff,
                                 int* __restrict__ seg_row, long long* __restrict__ seg_beg,
                                 long long* __restrict__ seg_end, int* __restrict__ seg_slot,
                                 int* __restrict__ long_row, int* __restrict__ long_first,
                                 int* __restrict__ long_count) {
    const long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (r >= rows) return;
    const long long b = ptr[r], e = ptr[r + 1];
    const int ns = nseg[r], s0 = segoff[r];
    const bool lg = islong[r] != 0;
    for (int q = 0; q < ns; ++q) {
        seg_row[s0 + q] = static_cast<int>(r);
        const long long sb = lg ? b + static_cast<long long>(q) * kSegLen : b;
        seg_beg[s0 + q] = sb;
        seg_end[s0 + q] = lg ? min(e, sb + kSegLen) : e;
        seg_slot[s0 + q] = lg ? slotoff[r] + q : -1;
    }
    if (lg) {
        const int l = longoff[r];
        long_row[l] = static_cast<int>(r);
        long_first[l] = slotoff[r];
        long_count[l] = ns;
    }
}

// ---- SampledMatrix from triplets (sampled.hpp:27-62) -------------------
// keys = row * n + col; the first offending input index of each error kind
// is recorded (atomicMin) so the host can name the entry like the reference.
__global__ void triplet_keys_kernel(long long nnz, long long m, long long n, const long long* __restrict__ rows,
                                    const long long* __restrict__ cols, const double* __restrict__ vals,
                                    unsigned long long* __restrict__ keys, int* __restrict__ idx,
                                    unsigned long long* __restrict__ first_bad) {
    const long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (k >= nnz) return;
    const long long r = rows[k], c = cols[k];
    const bool ok = r >= 0 && r < m && c >= 0 && c < n;
    if (!ok) atomicMin(first_bad, static_cast<unsigned long long>(k));
    if (!isfinite(vals[k])) atomicMin(first_bad + 1, static_cast<unsigned long long>(k));
    keys[k] = ok ? static_cast<unsigned long long>(r) * static_cast<unsigned long long>(n) +
                       static_cast<unsigned long long>(c)
                 : 0ULL;
    idx[k] = static_cast<int>(k);
}

// adjacent equal sorted keys: the later entry (in sorted order) is a duplicate
__global__ void duplicate_kernel(long long nnz, const unsigned long long* __restrict__ keys,
                                 const int* __restrict__ perm, unsigned long long* __restrict__ first_dup) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p < 1 || p >= nnz) return;
    if (keys[p] == keys[p - 1]) atomicMin(first_dup, static_cast<unsigned long long>(perm[p]));
}

__device__ __forceinline__ long long lower_bound_key(const unsigned long long* keys, long long nnz,
                                                     unsigned long long v) {
    long long lo = 0, hi = nnz;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (keys[mid] < v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// local CSR of rows [rb, rb + ml): rowptr (rebased), int64 columns, values
__global__ void triplet_rowptr_kernel(long long ml, long long rb, long long n, long long nnz,
                                      const unsigned long long* __restrict__ keys, long long* __restrict__ rowptr) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i > ml) return;
    const long long lo = lower_bound_key(keys, nnz, static_cast<unsigned long long>(rb) * n);
    rowptr[i] = lower_bound_key(keys, nnz, static_cast<unsigned long long>(rb + i) * n) - lo;
}

__global__ void lower_bound_one_kernel(const unsigned long long* __restrict__ keys, long long nnz,
                                       unsigned long long v, long long* __restrict__ out) {
    out[0] = lower_bound_key(keys, nnz, v);
}

__global__ void triplet_fill_kernel(long long cnt, long long lo, long long n, const unsigned long long* __restrict__ keys,
                                    const int* __restrict__ perm, const double* __restrict__ vals,
                                    long long* __restrict__ col64, double* __restrict__ val) {
    const long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (k >= cnt) return;
    col64[k] = static_cast<long long>(keys[lo + k] % static_cast<unsigned long long>(n));
    val[k] = vals[perm[lo + k]];
}


// ---- shared-memory-tiled view (TilePlanView, common.hpp) -----------------
// keys[k] = (block of k's row) << 32 | gather index; rid[k] = row (one warp
// per row)
__global__ void tile_keys_kernel(long long rows, const long long* __restrict__ ptr, const int* __restrict__ idx,
                                 unsigned long long* __restrict__ keys, int* __restrict__ iota,
                                 int* __restrict__ rid) {
    const long long r = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const unsigned long long hi = static_cast<unsigned long long>(r / kTileRows) << 32;
    for (long long k = ptr[r] + lane; k < ptr[r + 1]; k += 32) {
        keys[k] = hi | static_cast<unsigned int>(idx[k]);
        iota[k] = static_cast<int>(k);
        rid[k] = static_cast<int>(r);
    }
}

__global__ void tile_newcol_kernel(long long nnz, const unsigned long long* __restrict__ skeys,
                                   int* __restrict__ newcol) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= nnz) return;
    newcol[p] = (p == 0 || skeys[p] != skeys[p - 1]) ? 1 : 0;
}

// coarse tile starts: the block's first entry, or where dix / kTileSlots
// changes (dix = distinct gather index within the block)
__global__ void tile_start_kernel(long long nnz, long long rows, const unsigned long long* __restrict__ skeys,
                                  const long long* __restrict__ ptr, const int* __restrict__ G,
                                  int* __restrict__ ts) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= nnz) return;
    const long long blk = static_cast<long long>(skeys[p] >> 32);
    const long long bstart = ptr[blk * kTileRows];
    const int ct = (G[p] - G[bstart]) / kTileSlots;
    const bool st = (p == bstart) || ct != (G[p - 1] - G[bstart]) / kTileSlots;
    ts[p] = st ? 1 : 0;
}

__global__ void tile_coarse_start_kernel(long long nnz, const int* __restrict__ ts, const int* __restrict__ TI,
                                         long long* __restrict__ cstart) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= nnz) return;
    if (ts[p]) cstart[TI[p] - 1] = p;
}

__global__ void tile_nsub_kernel(long long nc, const long long* __restrict__ cstart, int* __restrict__ nsub) {
    const long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (c >= nc) return;
    nsub[c] = static_cast<int>((cstart[c + 1] - cstart[c] + kTileEnts - 1) / kTileEnts);
}

// per entry: its (sub-)tile, slot and the (tile, local row) sort key; tile
// starts, blocks and the slots' gather indices (duplicates write equal values)
__global__ void tile_assign_kernel(long long nnz, const int* __restrict__ TI, const long long* __restrict__ cstart,
                                   const int* __restrict__ sub_base, const int* __restrict__ G,
                                   const int* __restrict__ sp, const int* __restrict__ rid,
                                   const unsigned long long* __restrict__ skeys, int* __restrict__ slot_of,
                                   unsigned long long* __restrict__ key2, long long* __restrict__ tile_e,
                                   int* __restrict__ tile_blk) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= nnz) return;
    const int c = TI[p] - 1;
    const long long q = p - cstart[c];
    const long long sub = sub_base[c] + q / kTileEnts;
    const long long substart = cstart[c] + (q / kTileEnts) * kTileEnts;
    slot_of[p] = G[p] - G[substart];
    key2[p] = (static_cast<unsigned long long>(sub) << 9) | static_cast<unsigned long long>(rid[sp[p]] % kTileRows);
    if (p == substart) {
        tile_e[sub] = p;
        tile_blk[sub] = static_cast<int>(skeys[p] >> 32);
    }
}

__global__ void tile_nslot_kernel(long long nt, const long long* __restrict__ tile_e, const int* __restrict__ G,
                                  int* __restrict__ nslot) {
    const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (t >= nt) return;
    nslot[t] = G[tile_e[t + 1] - 1] - G[tile_e[t]] + 1;
}

__global__ void tile_ucol_kernel(long long nnz, const long long* __restrict__ cstart, const int* __restrict__ TI, const int* __restrict__ sub_base,
                                 const int* __restrict__ slot_of, const int* __restrict__ sp,
                                 const int* __restrict__ idx, const int* __restrict__ tile_u, int* __restrict__ ucol) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= nnz) return;
    const int c = TI[p] - 1;
    const long long sub = sub_base[c] + (p - cstart[c]) / kTileEnts;
    ucol[tile_u[sub] + slot_of[p]] = idx[sp[p]];
}

// final (tile, row)-ordered entries: slot, and the CSR position of the value
__global__ void tile_fill_kernel(long long nnz, const int* __restrict__ o, const int* __restrict__ slot_of,
                                 const int* __restrict__ sp, const int* __restrict__ map, TileEnt* __restrict__ ent,
                                 int* __restrict__ perm) {
    const long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (f >= nnz) return;
    const int p = o[f];
    TileEnt t;
    t.v = 0.0;
    t.slot = slot_of[p];
    t.pad = 0;
    ent[f] = t;
    const int srcpos = sp[p];
    perm[f] = map ? map[srcpos] : srcpos;
}

// roff[t * stride + r] = first entry of local row r in tile t (relative)
__global__ void tile_roff_kernel(long long nt, const long long* __restrict__ tile_e,
                                 const unsigned long long* __restrict__ skey2, unsigned short* __restrict__ roff) {
    const long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (g >= nt * kTileRoffStride) return;
    const long long t = g / kTileRoffStride;
    const int r = static_cast<int>(g - t * kTileRoffStride);
    const long long b = tile_e[t], e = tile_e[t + 1];
    if (r > kTileRows) {
        roff[g] = static_cast<unsigned short>(e - b);
        return;
    }
    const unsigned long long key = (static_cast<unsigned long long>(t) << 9) + static_cast<unsigned long long>(r);
    long long lo = b, hi = e;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (skey2[mid] < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    roff[g] = static_cast<unsigned short>(lo - b);
}

__global__ void invert_perm_kernel(long long n, const int* __restrict__ fwd, int* __restrict__ inv) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p < n) inv[fwd[p]] = static_cast<int>(p);
}

__global__ void iota_kernel(long long n, int* __restrict__ out) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p < n) out[p] = static_cast<int>(p);
}


// ---- dense-corner split (HybridPlan) ----------------------------------------
__global__ void ptr_degree_kernel(long long rows, const long long* __restrict__ ptr, int* __restrict__ deg) {
    const long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (r < rows) deg[r] = static_cast<int>(ptr[r + 1] - ptr[r]);
}

__global__ void scatter_rank_kernel(long long n, const int* __restrict__ order, int* __restrict__ rank) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i < n) rank[order[i]] = static_cast<int>(i);
}

// rank buckets of the cost model: bucket b < kHybB - 1 holds ranks below
// 256 << b (beyond the previous bucket), the last one the rest
constexpr int kHybB = 8;
__device__ __forceinline__ int hyb_bucket(int rank) {
    int b = 0;
    while (b < kHybB - 1 && rank >= (256 << b)) ++b;
    return b;
}

// entries by (row-rank bucket, column-rank bucket)
__global__ void hyb_hist_kernel(long long nnz, const int* __restrict__ rid, const int* __restrict__ col,
                                const int* __restrict__ rrank, const int* __restrict__ crank,
                                unsigned long long* __restrict__ hist) {
    __shared__ unsigned int h[kHybB * kHybB];
    for (int i = threadIdx.x; i < kHybB * kHybB; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < nnz;
         e += static_cast<long long>(gridDim.x) * blockDim.x)
        atomicAdd(&h[hyb_bucket(rrank[rid[e]]) * kHybB + hyb_bucket(crank[col[e]])], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < kHybB * kHybB; i += blockDim.x)
        if (h[i]) atomicAdd(hist + i, static_cast<unsigned long long>(h[i]));
}

__global__ void hyb_flag_kernel(long long nnz, const int* __restrict__ rid, const int* __restrict__ col,
                                const int* __restrict__ rrank, const int* __restrict__ crank, int R, int C,
                                int* __restrict__ fl, int* __restrict__ nfl) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= nnz) return;
    const int f = (rrank[rid[e]] < R && crank[col[e]] < C) ? 1 : 0;
    fl[e] = f;
    nfl[e] = 1 - f;
}

// order-preserving compaction of the CSR entries into block / cold lists
__global__ void hyb_compact_kernel(long long nnz, const int* __restrict__ fl, const int* __restrict__ bpos,
                                   const int* __restrict__ cpos, const int* __restrict__ rid,
                                   const int* __restrict__ col, const int* __restrict__ rrank,
                                   const int* __restrict__ crank, int C, int* __restrict__ col_c,
                                   int* __restrict__ map_c, int* __restrict__ blk_map, int* __restrict__ blk_pos) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= nnz) return;
    if (fl[e]) {
        const int q = bpos[e];
        blk_map[q] = static_cast<int>(e);
        blk_pos[q] = rrank[rid[e]] * C + crank[col[e]];
    } else {
        const int p = cpos[e];
        col_c[p] = col[e];
        map_c[p] = static_cast<int>(e);
    }
}

// pointer array of the compacted pattern: out[i] = pos[ptr[i]] (i <= rows)
__global__ void hyb_ptr_kernel(long long rows, const long long* __restrict__ ptr, const int* __restrict__ pos,
                               long long* __restrict__ out) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i <= rows) out[i] = pos[ptr[i]];
}

__global__ void hyb_flag_csc_kernel(long long nnz, const int* __restrict__ csc2csr, const int* __restrict__ fl,
                                    int* __restrict__ nflt) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p < nnz) nflt[p] = 1 - fl[csc2csr[p]];
}

__global__ void hyb_compact_csc_kernel(long long nnz, const int* __restrict__ csc2csr, const int* __restrict__ nflt,
                                       const int* __restrict__ cpt, const int* __restrict__ cscrow,
                                       int* __restrict__ row_c, int* __restrict__ mapt_c) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= nnz || !nflt[p]) return;
    const int q = cpt[p];
    row_c[q] = cscrow[p];
    mapt_c[q] = csc2csr[p];
}

__global__ void hyb_gather_vals_kernel(long long n, const int* __restrict__ map, const double* __restrict__ Y,
                                       double* __restrict__ out) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p < n) out[p] = Y[__ldg(map + p)];
}

__global__ void hyb_scatter_blk_kernel(long long nb, const int* __restrict__ blk_map, const int* __restrict__ blk_pos,
                                       const double* __restrict__ Y, double* __restrict__ D) {
    const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (q < nb) D[__ldg(blk_pos + q)] = Y[__ldg(blk_map + q)];
}

inline unsigned nb(long long n, int t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

// exclusive scan of n ints into out (n + 1 entries; out[n] = total)
void exclusive_scan(svt_ctx* ctx, const int* in, int* out, long long n, DevBuf<unsigned char>& tmp) {
    size_t bytes = 0;
    SVT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, static_cast<int>(n + 1), ctx->stream));
    tmp.ensure(bytes);
    SVT_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, in, out, static_cast<int>(n + 1), ctx->stream));
}

}  // namespace

// Segment plan of a device row-pointer array (ptr: rows + 1 entries).
void build_plan_device(svt_ctx* ctx, const long long* ptr, i64 rows, SegPlan& P) {
    cudaStream_t s = ctx->stream;
    DevBuf<int> cnt(static_cast<size_t>(3 * (rows + 1)));
    DevBuf<int> off(static_cast<size_t>(3 * (rows + 1)));
    DevBuf<unsigned char> tmp;
    int* nseg = cnt.get();
    int* isl = cnt.get() + (rows + 1);
    int* nsl = cnt.get() + 2 * (rows + 1);
    SVT_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int) * 3 * (rows + 1), s));
    {
        LaunchScope ls(ctx, K_OTHER, 24.0 * rows, 0.0);
        plan_count_kernel<<<nb(rows), 256, 0, s>>>(rows, ptr, nseg, isl, nsl);
    }
    exclusive_scan(ctx, nseg, off.get(), rows, tmp);
    exclusive_scan(ctx, isl, off.get() + (rows + 1), rows, tmp);
    exclusive_scan(ctx, nsl, off.get() + 2 * (rows + 1), rows, tmp);
    int tot[3];
    for (int q = 0; q < 3; ++q)
        SVT_CUDA(cudaMemcpyAsync(&tot[q], off.get() + q * (rows + 1) + rows, sizeof(int), cudaMemcpyDeviceToHost, s));
    sync_stream(ctx);
    const i64 nsegs = tot[0], nlong = tot[1], nslots = tot[2];
    P.seg_row.alloc(static_cast<size_t>(std::max<i64>(1, nsegs)));
    P.seg_slot.alloc(static_cast<size_t>(std::max<i64>(1, nsegs)));
    P.seg_beg.alloc(static_cast<size_t>(std::max<i64>(1, nsegs)));
    P.seg_end.alloc(static_cast<size_t>(std::max<i64>(1, nsegs)));
    P.long_row.alloc(static_cast<size_t>(std::max<i64>(1, nlong)));
    P.long_first.alloc(static_cast<size_t>(std::max<i64>(1, nlong)));
    P.long_count.alloc(static_cast<size_t>(std::max<i64>(1, nlong)));
    if (rows > 0) {
        LaunchScope ls(ctx, K_OTHER, 40.0 * rows + 28.0 * nsegs, 0.0);
        plan_fill_kernel<<<nb(rows), 256, 0, s>>>(rows, ptr, nseg, off.get(), isl, off.get() + (rows + 1),
                                                  off.get() + 2 * (rows + 1), P.seg_row.get(), P.seg_beg.get(),
                                                  P.seg_end.get(), P.seg_slot.get(), P.long_row.get(),
                                                  P.long_first.get(), P.long_count.get());
    }
    sync_stream(ctx);  // cnt / off die here
    {
        std::vector<long long> hb(static_cast<size_t>(nsegs)), he(static_cast<size_t>(nsegs));
        if (nsegs > 0) {
            SVT_CUDA(cudaMemcpyAsync(hb.data(), P.seg_beg.get(), sizeof(long long) * nsegs, cudaMemcpyDeviceToHost, s));
            SVT_CUDA(cudaMemcpyAsync(he.data(), P.seg_end.get(), sizeof(long long) * nsegs, cudaMemcpyDeviceToHost, s));
            sync_stream(ctx);
        }
        build_groups(hb, he, s, P);
    }
    P.v.nseg = nsegs;
    P.v.seg_row = P.seg_row.get();
    P.v.seg_beg = P.seg_beg.get();
    P.v.seg_end = P.seg_end.get();
    P.v.seg_slot = P.seg_slot.get();
    P.v.nlong = nlong;
    P.v.nslots = nslots;
    P.v.long_row = P.long_row.get();
    P.v.long_first = P.long_first.get();
    P.v.long_count = P.long_count.get();
}

// M->rowptr (rebased, device), M->val filled; col64 = the uploaded int64
// column indices.  Builds col (int32), the CSC view, csr2csc and the plans.
// Returns a validation code: 0 ok, 1 column out of range, 2 non-finite value.
int build_sampled_device(svt_ctx* ctx, svt_mat* M, const long long* col64) {
    cudaStream_t s = ctx->stream;
    const i64 nnz = M->nnz_local, n = M->n, ml = M->m_local;
    DevBuf<int> iota(static_cast<size_t>(std::max<i64>(1, nnz)));
    DevBuf<int> sorted_col(static_cast<size_t>(std::max<i64>(1, nnz)));
    DevBuf<int> perm(static_cast<size_t>(std::max<i64>(1, nnz)));
    DevBuf<int> rid(static_cast<size_t>(std::max<i64>(1, nnz)));
    DevBuf<unsigned char> tmp;
    int* bad = ctx->d_flags + 60;
    SVT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    if (nnz > 0) {
        LaunchScope ls(ctx, K_OTHER, 28.0 * nnz, 0.0);
        convert_validate_kernel<<<nb(nnz), 256, 0, s>>>(nnz, n, reinterpret_cast<const long long*>(col64),
                                                        M->val.get(), M->col.get(), iota.get(), bad);
    }
    SVT_CUDA(cudaMemcpyAsync(ctx->h_flags + 60, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    sync_stream(ctx);
    const int code = ctx->h_flags[60];
    if (code != 0) return code;
    if (nnz > 0) {
        int end_bit = 1;
        while ((1LL << end_bit) < n) ++end_bit;
        size_t bytes = 0;
        SVT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, M->col.get(), sorted_col.get(), iota.get(),
                                                 perm.get(), static_cast<int>(nnz), 0, end_bit, s));
        tmp.ensure(bytes);
        SVT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, M->col.get(), sorted_col.get(), iota.get(),
                                                 perm.get(), static_cast<int>(nnz), 0, end_bit, s));
        {
            LaunchScope ls(ctx, K_OTHER, 8.0 * nnz, 0.0);
            row_ids_kernel<<<nb(ml * 32), 256, 0, s>>>(ml, reinterpret_cast<const long long*>(M->rowptr.get()),
                                                       rid.get());
        }
        LaunchScope ls(ctx, K_OTHER, 36.0 * nnz, 0.0);
        csc_fill_kernel<<<nb(nnz), 256, 0, s>>>(nnz, perm.get(), rid.get(), M->val.get(), M->cscrow.get(),
                                                M->val_csc.get(), M->csr2csc.get());
    }
    M->csc2csr = std::move(perm);  // the stable sort's permutation is the CSC -> CSR map
    {
        LaunchScope ls(ctx, K_OTHER, 8.0 * (n + 1), 0.0);
        colptr_kernel<<<nb(n + 1), 256, 0, s>>>(nnz, n, sorted_col.get(),
                                                reinterpret_cast<long long*>(M->colptr.get()));
    }
    build_plan_device(ctx, reinterpret_cast<const long long*>(M->rowptr.get()), ml, M->plan_csr);
    build_plan_device(ctx, reinterpret_cast<const long long*>(M->colptr.get()), n, M->plan_csc);
    sync_stream(ctx);  // temporaries die here
    return 0;
}

// SampledMatrix from unsorted triplets, sorted and validated on the device
// (radix sort of row * n + col; duplicates are adjacent keys).  Fills M's
// local CSR for rows [row_begin, row_end) and the rest of the structure.
// Throws std::invalid_argument with the reference's messages.
void build_from_triplets_device(svt_ctx* ctx, svt_mat* M, i64 nnz, const i64* rows, const i64* cols,
                                const double* vals) {
    cudaStream_t s = ctx->stream;
    const i64 m = M->m, n = M->n, rb = M->row_begin, ml = M->m_local;
    DevBuf<long long> drow(static_cast<size_t>(nnz)), dcol(static_cast<size_t>(nnz));
    DevBuf<double> dval(static_cast<size_t>(nnz));
    DevBuf<unsigned long long> keys(static_cast<size_t>(nnz)), skeys(static_cast<size_t>(nnz));
    DevBuf<int> idx(static_cast<size_t>(nnz)), perm(static_cast<size_t>(nnz));
    DevBuf<unsigned long long> flags(4);
    DevBuf<unsigned char> tmp;
    SVT_CUDA(cudaMemcpyAsync(drow.get(), rows, sizeof(i64) * nnz, cudaMemcpyHostToDevice, s));
    SVT_CUDA(cudaMemcpyAsync(dcol.get(), cols, sizeof(i64) * nnz, cudaMemcpyHostToDevice, s));
    SVT_CUDA(cudaMemcpyAsync(dval.get(), vals, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
    SVT_CUDA(cudaMemsetAsync(flags.get(), 0xff, sizeof(unsigned long long) * 4, s));
    {
        LaunchScope ls(ctx, K_OTHER, 36.0 * nnz, 0.0);
        triplet_keys_kernel<<<nb(nnz), 256, 0, s>>>(nnz, m, n, drow.get(), dcol.get(), dval.get(), keys.get(),
                                                    idx.get(), flags.get());
    }
    unsigned long long hf[4];
    SVT_CUDA(cudaMemcpyAsync(hf, flags.get(), sizeof(hf), cudaMemcpyDeviceToHost, s));
    sync_stream(ctx);
    auto entry = [&](unsigned long long k) {
        return "(" + std::to_string(rows[k]) + ", " + std::to_string(cols[k]) + ")";
    };
    if (hf[0] != ~0ULL) throw std::invalid_argument("SampledMatrix: entry " + entry(hf[0]) + " out of range");
    int end_bit = 1;
    while (end_bit < 64 && (1ULL << end_bit) < static_cast<unsigned long long>(m) * static_cast<unsigned long long>(n))
        ++end_bit;
    size_t bytes = 0;
    SVT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.get(), skeys.get(), idx.get(), perm.get(),
                                             static_cast<int>(nnz), 0, end_bit, s));
    tmp.ensure(bytes);
    SVT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, keys.get(), skeys.get(), idx.get(), perm.get(),
                                             static_cast<int>(nnz), 0, end_bit, s));
    {
        LaunchScope ls(ctx, K_OTHER, 20.0 * nnz, 0.0);
        duplicate_kernel<<<nb(nnz), 256, 0, s>>>(nnz, skeys.get(), perm.get(), flags.get() + 2);
    }
    SVT_CUDA(cudaMemcpyAsync(hf, flags.get(), sizeof(hf), cudaMemcpyDeviceToHost, s));
    sync_stream(ctx);
    if (hf[1] != ~0ULL) throw std::invalid_argument("SampledMatrix: non-finite value at " + entry(hf[1]));
    if (hf[2] != ~0ULL) throw std::invalid_argument("SampledMatrix: duplicate entry " + entry(hf[2]));
    // this rank's rows
    {
        LaunchScope ls(ctx, K_OTHER, 8.0 * (ml + 1), 0.0);
        triplet_rowptr_kernel<<<nb(ml + 1), 256, 0, s>>>(ml, rb, n, nnz, skeys.get(),
                                                         reinterpret_cast<long long*>(M->rowptr.get()));
    }
    // global position of the block's first entry and the block's entry count
    long long lo_hi[2] = {0, 0};
    DevBuf<long long> lo_dev(1);
    lower_bound_one_kernel<<<1, 1, 0, s>>>(skeys.get(), nnz, static_cast<unsigned long long>(rb) * n, lo_dev.get());
    SVT_CUDA(cudaMemcpyAsync(&lo_hi[0], lo_dev.get(), sizeof(long long), cudaMemcpyDeviceToHost, s));
    SVT_CUDA(cudaMemcpyAsync(&lo_hi[1], reinterpret_cast<long long*>(M->rowptr.get()) + ml, sizeof(long long),
                             cudaMemcpyDeviceToHost, s));
    sync_stream(ctx);
    const i64 lo = lo_hi[0], cnt = lo_hi[1];
    if (cnt > 2147483647LL) throw std::invalid_argument("svt_matrix_upload: > 2^31 entries per rank");
    M->nnz_local = cnt;
    M->col.alloc(static_cast<size_t>(std::max<i64>(1, cnt)));
    M->val.alloc(static_cast<size_t>(std::max<i64>(1, cnt)));
    M->cscrow.alloc(static_cast<size_t>(std::max<i64>(1, cnt)));
    M->val_csc.alloc(static_cast<size_t>(std::max<i64>(1, cnt)));
    M->csr2csc.alloc(static_cast<size_t>(std::max<i64>(1, cnt)));
    DevBuf<long long> col64(static_cast<size_t>(std::max<i64>(1, cnt)));
    if (cnt > 0) {
        LaunchScope ls(ctx, K_OTHER, 28.0 * cnt, 0.0);
        triplet_fill_kernel<<<nb(cnt), 256, 0, s>>>(cnt, lo, n, skeys.get(), perm.get(), dval.get(), col64.get(),
                                                    M->val.get());
    }
    const int code = build_sampled_device(ctx, M, col64.get());
    if (code != 0) throw std::invalid_argument("SampledMatrix: invalid entry");
}


// Tiled view of a CSR-like pattern (ptr: rows + 1, idx: gather index per
// entry, sorted within each row).  map (optional) sends a source position to
// the CSR position holding its value (the CSC view passes csc2csr).
void build_tile_plan(svt_ctx* ctx, const long long* ptr, const int* idx, i64 rows, i64 nnz, const int* map,
                     TilePlan& P) {
    cudaStream_t s = ctx->stream;
    const i64 nblocks = (rows + kTileRows - 1) / kTileRows;
    P.v = TilePlanView{};
    P.v.nrows = rows;
    P.v.nnz = nnz;
    P.src = nullptr;
    std::vector<long long> h_te(1, 0);
    std::vector<int> h_tb;
    i64 nt = 0;
    if (nnz > 0) {
        const size_t N = static_cast<size_t>(nnz);
        DevBuf<unsigned long long> keys(N), skeys(N);
        DevBuf<int> iota(N), sp(N), rid(N), A1(N), G(N), TI(N);
        DevBuf<unsigned char> tmp;
        {
            LaunchScope ls(ctx, K_OTHER, 16.0 * nnz, 0.0);
            tile_keys_kernel<<<nb(rows * 32), 256, 0, s>>>(rows, ptr, idx, keys.get(), iota.get(), rid.get());
        }
        int end_bit = 33;
        while ((1LL << (end_bit - 32)) < nblocks + 1) ++end_bit;
        size_t bytes = 0;
        SVT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.get(), skeys.get(), iota.get(), sp.get(),
                                                 static_cast<int>(nnz), 0, end_bit, s));
        tmp.ensure(bytes);
        SVT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, keys.get(), skeys.get(), iota.get(), sp.get(),
                                                 static_cast<int>(nnz), 0, end_bit, s));
        tile_newcol_kernel<<<nb(nnz), 256, 0, s>>>(nnz, skeys.get(), A1.get());
        SVT_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, A1.get(), G.get(), static_cast<int>(nnz), s));
        tmp.ensure(bytes);
        SVT_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), bytes, A1.get(), G.get(), static_cast<int>(nnz), s));
        tile_start_kernel<<<nb(nnz), 256, 0, s>>>(nnz, rows, skeys.get(), ptr, G.get(), A1.get());
        SVT_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, A1.get(), TI.get(), static_cast<int>(nnz), s));
        tmp.ensure(bytes);
        SVT_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), bytes, A1.get(), TI.get(), static_cast<int>(nnz), s));
        int nc = 0;
        SVT_CUDA(cudaMemcpyAsync(&nc, TI.get() + nnz - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
        sync_stream(ctx);
        DevBuf<long long> cstart(static_cast<size_t>(nc) + 1);
        tile_coarse_start_kernel<<<nb(nnz), 256, 0, s>>>(nnz, A1.get(), TI.get(), cstart.get());
        const long long nn = nnz;
        SVT_CUDA(cudaMemcpyAsync(cstart.get() + nc, &nn, sizeof(long long), cudaMemcpyHostToDevice, s));
        DevBuf<int> nsub(static_cast<size_t>(nc) + 1), sub_base(static_cast<size_t>(nc) + 1);
        tile_nsub_kernel<<<nb(nc), 256, 0, s>>>(nc, cstart.get(), nsub.get());
        exclusive_scan(ctx, nsub.get(), sub_base.get(), nc, tmp);
        int ntot = 0;
        SVT_CUDA(cudaMemcpyAsync(&ntot, sub_base.get() + nc, sizeof(int), cudaMemcpyDeviceToHost, s));
        sync_stream(ctx);
        nt = ntot;
        P.tile_e.alloc(static_cast<size_t>(nt) + 1);
        P.tile_u.alloc(static_cast<size_t>(nt) + 1);
        DevBuf<int> tile_blk(static_cast<size_t>(nt)), nslot(static_cast<size_t>(nt) + 1), tu32(static_cast<size_t>(nt) + 1);
        DevBuf<unsigned long long>& key2 = keys;  // keys are dead after the first sort
        DevBuf<int>& slot_of = iota;
        {
            LaunchScope ls(ctx, K_OTHER, 40.0 * nnz, 0.0);
            tile_assign_kernel<<<nb(nnz), 256, 0, s>>>(nnz, TI.get(), cstart.get(), sub_base.get(), G.get(),
                                                       sp.get(), rid.get(), skeys.get(), slot_of.get(), key2.get(),
                                                       P.tile_e.get(), tile_blk.get());
        }
        SVT_CUDA(cudaMemcpyAsync(P.tile_e.get() + nt, &nn, sizeof(long long), cudaMemcpyHostToDevice, s));
        tile_nslot_kernel<<<nb(nt), 256, 0, s>>>(nt, P.tile_e.get(), G.get(), nslot.get());
        exclusive_scan(ctx, nslot.get(), tu32.get(), nt, tmp);
        int nuc = 0;
        SVT_CUDA(cudaMemcpyAsync(&nuc, tu32.get() + nt, sizeof(int), cudaMemcpyDeviceToHost, s));
        sync_stream(ctx);
        P.ucol.alloc(static_cast<size_t>(nuc) + kTileSlots);  // padded: slot loads run past a tile's end
        SVT_CUDA(cudaMemsetAsync(P.ucol.get(), 0, sizeof(int) * (static_cast<size_t>(nuc) + kTileSlots), s));
        tile_ucol_kernel<<<nb(nnz), 256, 0, s>>>(nnz, cstart.get(), TI.get(), sub_base.get(), slot_of.get(),
                                                 sp.get(), idx, tu32.get(), P.ucol.get());
        {
            std::vector<int> h(static_cast<size_t>(nt) + 1);
            std::vector<long long> h64(static_cast<size_t>(nt) + 1);
            SVT_CUDA(cudaMemcpyAsync(h.data(), tu32.get(), sizeof(int) * (nt + 1), cudaMemcpyDeviceToHost, s));
            sync_stream(ctx);
            for (size_t i = 0; i < h.size(); ++i) h64[i] = h[i];
            SVT_CUDA(cudaMemcpyAsync(P.tile_u.get(), h64.data(), sizeof(long long) * (nt + 1), cudaMemcpyHostToDevice,
                                     s));
            sync_stream(ctx);
        }
        // (tile, local row) order; slots ascend inside a row (stable sort)
        int end2 = 10;
        while ((1LL << (end2 - 9)) < nt + 1) ++end2;
        DevBuf<unsigned long long>& skey2 = skeys;
        DevBuf<int>& o = rid;  // rid is dead after tile_assign
        DevBuf<int>& pos = A1;
        {
            LaunchScope ls(ctx, K_OTHER, 0.0, 0.0);
            // pos = iota (reuse tile_keys-free pass: positions 0..nnz-1)
            iota_kernel<<<nb(nnz), 256, 0, s>>>(nnz, pos.get());
        }
        SVT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key2.get(), skey2.get(), pos.get(), o.get(),
                                                 static_cast<int>(nnz), 0, end2, s));
        tmp.ensure(bytes);
        SVT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, key2.get(), skey2.get(), pos.get(), o.get(),
                                                 static_cast<int>(nnz), 0, end2, s));
        P.ent.alloc(N);
        P.perm.alloc(N);
        {
            LaunchScope ls(ctx, K_OTHER, 32.0 * nnz, 0.0);
            tile_fill_kernel<<<nb(nnz), 256, 0, s>>>(nnz, o.get(), slot_of.get(), sp.get(), map, P.ent.get(),
                                                     P.perm.get());
        }
        P.roff.alloc(static_cast<size_t>(nt) * kTileRoffStride);
        tile_roff_kernel<<<nb(nt * kTileRoffStride), 256, 0, s>>>(nt, P.tile_e.get(), skey2.get(), P.roff.get());
        h_te.resize(static_cast<size_t>(nt) + 1);
        h_tb.resize(static_cast<size_t>(nt));
        SVT_CUDA(cudaMemcpyAsync(h_te.data(), P.tile_e.get(), sizeof(long long) * (nt + 1), cudaMemcpyDeviceToHost, s));
        SVT_CUDA(cudaMemcpyAsync(h_tb.data(), tile_blk.get(), sizeof(int) * nt, cudaMemcpyDeviceToHost, s));
        sync_stream(ctx);  // temporaries die here
        SVT_CHECK_LAUNCH();
    }
    // work items: each block's tiles in runs of >= target entries; a block
    // spread over several items writes partial rows, summed in item order
    const i64 target = std::max<i64>(4LL * kTileEnts, nnz / std::max(1, ctx->num_sms));
    std::vector<int> it0, it1, iblk, ipart, sblk, sfirst, scount;
    i64 t = 0, nparts = 0;
    for (i64 b = 0; b < nblocks; ++b) {
        const i64 tb0 = t;
        while (t < nt && h_tb[static_cast<size_t>(t)] == b) ++t;
        const size_t first_item = it0.size();
        i64 a = tb0;
        if (a == t) {  // empty block: one item writes its zero rows
            it0.push_back(static_cast<int>(a));
            it1.push_back(static_cast<int>(a));
            iblk.push_back(static_cast<int>(b));
        }
        while (a < t) {
            i64 e = a;
            long long ents = 0;
            while (e < t && (ents < target || e == a) && e - a < kTileItemTiles) {
                ents += h_te[static_cast<size_t>(e + 1)] - h_te[static_cast<size_t>(e)];
                ++e;
            }
            // do not leave a small remainder behind
            if (t - e > 0 && t - a <= kTileItemTiles) {
                long long rest = h_te[static_cast<size_t>(t)] - h_te[static_cast<size_t>(e)];
                if (rest < target / 2) e = t;
            }
            it0.push_back(static_cast<int>(a));
            it1.push_back(static_cast<int>(e));
            iblk.push_back(static_cast<int>(b));
            a = e;
        }
        const size_t cnt = it0.size() - first_item;
        if (cnt == 1) {
            ipart.push_back(-1);
        } else {
            sblk.push_back(static_cast<int>(b));
            sfirst.push_back(static_cast<int>(nparts));
            scount.push_back(static_cast<int>(cnt));
            for (size_t q = 0; q < cnt; ++q) ipart.push_back(static_cast<int>(nparts++));
        }
    }
    auto up = [&](DevBuf<int>& d, const std::vector<int>& h) {
        d.alloc(std::max<size_t>(1, h.size()));
        if (!h.empty()) SVT_CUDA(cudaMemcpyAsync(d.get(), h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice, s));
    };
    up(P.item_t0, it0);
    up(P.item_t1, it1);
    up(P.item_blk, iblk);
    up(P.item_part, ipart);
    up(P.split_blk, sblk);
    up(P.split_first, sfirst);
    up(P.split_count, scount);
    sync_stream(ctx);
    P.v.ntiles = nt;
    P.v.nitems = static_cast<long long>(it0.size());
    P.v.nsplit = static_cast<long long>(sblk.size());
    P.v.nparts = nparts;
    P.v.tile_e = P.tile_e.get();
    P.v.tile_u = P.tile_u.get();
    P.v.ucol = P.ucol.get();
    P.v.roff = P.roff.get();
    P.v.ent = P.ent.get();
    P.v.perm = P.perm.get();
    P.v.item_t0 = P.item_t0.get();
    P.v.item_t1 = P.item_t1.get();
    P.v.item_blk = P.item_blk.get();
    P.v.item_part = P.item_part.get();
    P.v.split_blk = P.split_blk.get();
    P.v.split_first = P.split_first.get();
    P.v.split_count = P.split_count.get();
    P.built = true;
}


// Both tiled views of M (lazily, on the first wide product).  The CSC view's
// values come from the CSR array through csc2csr (built here if the upload
// path did not keep it).
void ensure_tile_plans(svt_ctx* ctx, svt_mat* M) {
    const i64 nnz = M->nnz_local;
    if (!M->tile_csr.built)
        build_tile_plan(ctx, reinterpret_cast<const long long*>(M->rowptr.get()), M->col.get(), M->m_local, nnz,
                        nullptr, M->tile_csr);
    if (!M->tile_csc.built) {
        if (M->csc2csr.n < static_cast<size_t>(nnz)) {
            M->csc2csr.alloc(static_cast<size_t>(std::max<i64>(1, nnz)));
            if (nnz > 0)
                invert_perm_kernel<<<nb(nnz), 256, 0, ctx->stream>>>(nnz, M->csr2csc.get(), M->csc2csr.get());
        }
        build_tile_plan(ctx, reinterpret_cast<const long long*>(M->colptr.get()), M->cscrow.get(), M->n, nnz,
                        M->csc2csr.get(), M->tile_csc);
    }
}


// Dense-corner split (HybridPlan, engine.hpp).  Cost model: a cold entry of
// a w-wide product costs the gather kernel ~w 8-byte panel loads through the
// L1 data pipe (its bound, profiles/r02a_ncu_full_spmm_cfg4_w120.txt); a
// dense block cell costs ~rho of that on the FP64 tensor cores (measured
// 57.6 ps / entry vs ~8.4 ps / cell at w = 120: rho ~ 0.15), both linear in
// w, so the block (R, C) that maximises  entries(R, C) - rho R C  is the same
// at every width.  R and C run over 256, 512, ..., 16384 (rank buckets of
// the degree orders: rows by local degree, columns by count); the split is
// kept when it saves at least 5 % of the entries' cost.
void ensure_hybrid(svt_ctx* ctx, svt_mat* M) {
    HybridPlan& H = M->hyb;
    if (H.tried) return;
    H.tried = true;
    const char* env = std::getenv("SVTB_HYBRID");
    if (env != nullptr && env[0] == '0') return;
    const i64 nnz = M->nnz_local, ml = M->m_local, n = M->n;
    if (nnz < (1 << 20) || ml < 512 || n < 512 || nnz >= (1LL << 31)) return;
    const char* rh = std::getenv("SVTB_HYBRID_RHO");
    const double rho = rh ? std::atof(rh) : 0.15;
    const bool dbg = std::getenv("SVTB_DEBUG_HYBRID") != nullptr;
    cudaStream_t s = ctx->stream;
    DevBuf<unsigned char> tmp;
    const i64 mx = std::max(ml, n);
    DevBuf<int> deg(static_cast<size_t>(mx)), sdeg(static_cast<size_t>(mx)), iota(static_cast<size_t>(mx));
    DevBuf<int> rorder(static_cast<size_t>(ml)), corder(static_cast<size_t>(n));
    DevBuf<int> rrank(static_cast<size_t>(ml)), crank(static_cast<size_t>(n));
    auto order_of = [&](const long long* ptr, i64 rows, int* order, int* rank) {
        ptr_degree_kernel<<<nb(rows), 256, 0, s>>>(rows, ptr, deg.get());
        iota_kernel<<<nb(rows), 256, 0, s>>>(rows, iota.get());
        size_t bytes = 0;
        SVT_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, deg.get(), sdeg.get(), iota.get(), order,
                                                           static_cast<int>(rows), 0, 32, s));
        tmp.ensure(bytes);
        SVT_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.get(), bytes, deg.get(), sdeg.get(), iota.get(), order,
                                                           static_cast<int>(rows), 0, 32, s));
        scatter_rank_kernel<<<nb(rows), 256, 0, s>>>(rows, order, rank);
    };
    const long long* rp = reinterpret_cast<const long long*>(M->rowptr.get());
    const long long* cp = reinterpret_cast<const long long*>(M->colptr.get());
    {
        LaunchScope ls(ctx, K_OTHER, 0.0, 0.0);
        order_of(rp, ml, rorder.get(), rrank.get());
        order_of(cp, n, corder.get(), crank.get());
    }
    DevBuf<int> rid(static_cast<size_t>(nnz));
    DevBuf<unsigned long long> hist(kHybB * kHybB);
    SVT_CUDA(cudaMemsetAsync(hist.get(), 0, sizeof(unsigned long long) * kHybB * kHybB, s));
    {
        LaunchScope ls(ctx, K_OTHER, 0.0, 0.0);
        row_ids_kernel<<<nb(ml * 32), 256, 0, s>>>(ml, rp, rid.get());
        hyb_hist_kernel<<<ctx->num_sms * 4, 256, 0, s>>>(nnz, rid.get(), M->col.get(), rrank.get(), crank.get(),
                                                         hist.get());
    }
    unsigned long long h[kHybB * kHybB];
    SVT_CUDA(cudaMemcpyAsync(h, hist.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    sync_stream(ctx);
    double best = 0.0;
    i64 R = 0, C = 0, E = 0;
    for (int a = 0; a < kHybB - 1; ++a) {
        for (int b = 0; b < kHybB - 1; ++b) {
            // C even: the dense block's rows are cp.async operands (16-byte rows)
            const i64 r = std::min<i64>(256LL << a, ml), c = std::min<i64>(256LL << b, n) & ~1LL;
            if (8.0 * static_cast<double>(r) * static_cast<double>(c) > 512e6) continue;
            i64 e = 0;
            for (int i = 0; i <= a; ++i)
                for (int j = 0; j <= b; ++j) e += static_cast<i64>(h[i * kHybB + j]);
            const double saved = static_cast<double>(e) - rho * static_cast<double>(r) * static_cast<double>(c);
            if (saved > best) {
                best = saved;
                R = r;
                C = c;
                E = e;
            }
        }
    }
    if (dbg)
        std::fprintf(stderr, "[hybrid] nnz=%lld best R=%lld C=%lld block entries=%lld (%.1f%%, density %.3f) saved %.1f%%\n",
                     static_cast<long long>(nnz), static_cast<long long>(R), static_cast<long long>(C),
                     static_cast<long long>(E), 100.0 * E / nnz, R * C > 0 ? static_cast<double>(E) / (R * C) : 0.0,
                     100.0 * best / nnz);
    if (best < 0.05 * static_cast<double>(nnz)) return;
    H.R = R;
    H.C = C;
    // flags and the two order-preserving compactions of the CSR entries
    DevBuf<int> fl(static_cast<size_t>(nnz) + 1), nfl(static_cast<size_t>(nnz) + 1);
    DevBuf<int> bpos(static_cast<size_t>(nnz) + 1), cpos(static_cast<size_t>(nnz) + 1);
    {
        LaunchScope ls(ctx, K_OTHER, 0.0, 0.0);
        hyb_flag_kernel<<<nb(nnz), 256, 0, s>>>(nnz, rid.get(), M->col.get(), rrank.get(), crank.get(),
                                               static_cast<int>(R), static_cast<int>(C), fl.get(), nfl.get());
    }
    exclusive_scan(ctx, fl.get(), bpos.get(), nnz, tmp);
    exclusive_scan(ctx, nfl.get(), cpos.get(), nnz, tmp);
    int tots[2];
    SVT_CUDA(cudaMemcpyAsync(&tots[0], bpos.get() + nnz, sizeof(int), cudaMemcpyDeviceToHost, s));
    SVT_CUDA(cudaMemcpyAsync(&tots[1], cpos.get() + nnz, sizeof(int), cudaMemcpyDeviceToHost, s));
    sync_stream(ctx);
    H.nnz_blk = tots[0];
    H.nnz_cold = tots[1];
    const size_t ncold = static_cast<size_t>(std::max<i64>(1, H.nnz_cold));
    const size_t nblk = static_cast<size_t>(std::max<i64>(1, H.nnz_blk));
    H.col_c.alloc(ncold);
    H.map_c.alloc(ncold);
    H.val_c.alloc(ncold);
    H.row_c.alloc(ncold);
    H.mapt_c.alloc(ncold);
    H.valt_c.alloc(ncold);
    H.blk_map.alloc(nblk);
    H.blk_pos.alloc(nblk);
    H.rowptr_c.alloc(static_cast<size_t>(ml + 1));
    H.colptr_c.alloc(static_cast<size_t>(n + 1));
    H.hot_rows.alloc(static_cast<size_t>(R));
    H.hot_cols.alloc(static_cast<size_t>(C));
    H.D.alloc(static_cast<size_t>(R * C));
    SVT_CUDA(cudaMemsetAsync(H.D.get(), 0, sizeof(double) * static_cast<size_t>(R * C), s));
    SVT_CUDA(cudaMemcpyAsync(H.hot_rows.get(), rorder.get(), sizeof(int) * R, cudaMemcpyDeviceToDevice, s));
    SVT_CUDA(cudaMemcpyAsync(H.hot_cols.get(), corder.get(), sizeof(int) * C, cudaMemcpyDeviceToDevice, s));
    {
        LaunchScope ls(ctx, K_OTHER, 0.0, 0.0);
        hyb_compact_kernel<<<nb(nnz), 256, 0, s>>>(nnz, fl.get(), bpos.get(), cpos.get(), rid.get(), M->col.get(),
                                                  rrank.get(), crank.get(), static_cast<int>(C), H.col_c.get(),
                                                  H.map_c.get(), H.blk_map.get(), H.blk_pos.get());
        hyb_ptr_kernel<<<nb(ml + 1), 256, 0, s>>>(ml, rp, cpos.get(),
                                                 reinterpret_cast<long long*>(H.rowptr_c.get()));
    }
    // the cold CSC view: CSC positions whose CSR entry is cold, in CSC order
    if (M->csc2csr.n < static_cast<size_t>(nnz)) {
        M->csc2csr.alloc(static_cast<size_t>(nnz));
        invert_perm_kernel<<<nb(nnz), 256, 0, s>>>(nnz, M->csr2csc.get(), M->csc2csr.get());
    }
    {
        LaunchScope ls(ctx, K_OTHER, 0.0, 0.0);
        hyb_flag_csc_kernel<<<nb(nnz), 256, 0, s>>>(nnz, M->csc2csr.get(), fl.get(), nfl.get());
    }
    exclusive_scan(ctx, nfl.get(), cpos.get(), nnz, tmp);
    {
        LaunchScope ls(ctx, K_OTHER, 0.0, 0.0);
        hyb_compact_csc_kernel<<<nb(nnz), 256, 0, s>>>(nnz, M->csc2csr.get(), nfl.get(), cpos.get(), M->cscrow.get(),
                                                      H.row_c.get(), H.mapt_c.get());
        hyb_ptr_kernel<<<nb(n + 1), 256, 0, s>>>(n, cp, cpos.get(), reinterpret_cast<long long*>(H.colptr_c.get()));
    }
    build_plan_device(ctx, reinterpret_cast<const long long*>(H.rowptr_c.get()), ml, H.plan_c);
    build_plan_device(ctx, reinterpret_cast<const long long*>(H.colptr_c.get()), n, H.plant_c);
    // split-K partials of the block product, per stream: sized for panels up
    // to 128 wide and 8 K-splits (wider calls grow them once)
    const size_t wsn = static_cast<size_t>(8 * std::max(R, C) * 128);
    H.ws[0].alloc(wsn);
    H.ws[1].alloc(wsn);
    sync_stream(ctx);  // the temporaries die here
    H.src = nullptr;
    H.on = true;
}

// Mirror a CSR value array into the cold CSR / CSC values and the dense block
// (12 + 12 B per cold entry, 16 B per block entry).
void hybrid_refresh(svt_ctx* ctx, svt_mat* M, const double* Ycsr) {
    HybridPlan& H = M->hyb;
    if (!H.on) return;
    cudaStream_t s = ctx->stream;
    LaunchScope ls(ctx, K_OTHER, 24.0 * H.nnz_cold + 16.0 * H.nnz_blk, 0.0);
    if (H.nnz_cold > 0) {
        hyb_gather_vals_kernel<<<nb(H.nnz_cold), 256, 0, s>>>(H.nnz_cold, H.map_c.get(), Ycsr, H.val_c.get());
        hyb_gather_vals_kernel<<<nb(H.nnz_cold), 256, 0, s>>>(H.nnz_cold, H.mapt_c.get(), Ycsr, H.valt_c.get());
    }
    if (H.nnz_blk > 0)
        hyb_scatter_blk_kernel<<<nb(H.nnz_blk), 256, 0, s>>>(H.nnz_blk, H.blk_map.get(), H.blk_pos.get(), Ycsr,
                                                             H.D.get());
    H.src = Ycsr;
}

}  // namespace svtb
