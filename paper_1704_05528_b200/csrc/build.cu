// Device-side construction of a rank's sample set (SampledMatrix storage,
// sampled.hpp:25-110): validation of the uploaded CSR, the CSC view by a
// stable radix sort of the column indices (rows stay ascending inside every
// column, exactly the order of the host counting sort it replaces), the
// csr2csc permutation, the CSC value mirror, and both segment plans of the
// load-balanced SpMM.  Only the CSR arrays cross PCIe; everything derived
// from them is built in HBM.
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

}  // namespace svtb
