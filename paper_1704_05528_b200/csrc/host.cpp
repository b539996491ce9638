// Host-side sample-set construction and device upload.
//
// svt_sampled_build restates the SampledMatrix constructor (sampled.hpp:27-62:
// row-major sort, range / finiteness / duplicate validation, CSR offsets).
// upload builds this rank's CSR block plus the CSC view and the CSR->CSC
// permutation that keeps the CSC value mirror in sync (counting sort by
// column; rows within a column stay increasing, so Y^T*X accumulates in the
// reference's row order).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <string>

#include "engine.hpp"

namespace svtb {

void sampled_build(i64 m, i64 n, i64 nnz, const i64* rows, const i64* cols, const double* vals, i64* rowptr_out,
                   i64* col_out, double* val_out) {
    if (m < 1 || n < 1) throw std::invalid_argument("SampledMatrix: dimensions must be >= 1");
    if (nnz < 1) throw std::invalid_argument("SampledMatrix: at least one entry required");
    std::vector<i64> order(static_cast<size_t>(nnz));
    std::iota(order.begin(), order.end(), 0);
    for (i64 k = 0; k < nnz; ++k) {
        if (rows[k] < 0 || rows[k] >= m || cols[k] < 0 || cols[k] >= n)
            throw std::invalid_argument("SampledMatrix: entry (" + std::to_string(rows[k]) + ", " +
                                        std::to_string(cols[k]) + ") out of range");
    }
    std::sort(order.begin(), order.end(), [&](i64 a, i64 b) {
        return rows[a] != rows[b] ? rows[a] < rows[b] : cols[a] < cols[b];
    });
    std::fill(rowptr_out, rowptr_out + m + 1, 0);
    for (i64 k = 0; k < nnz; ++k) {
        const i64 o = order[static_cast<size_t>(k)];
        if (!std::isfinite(vals[o]))
            throw std::invalid_argument("SampledMatrix: non-finite value at (" + std::to_string(rows[o]) + ", " +
                                        std::to_string(cols[o]) + ")");
        if (k > 0) {
            const i64 p = order[static_cast<size_t>(k - 1)];
            if (rows[p] == rows[o] && cols[p] == cols[o])
                throw std::invalid_argument("SampledMatrix: duplicate entry (" + std::to_string(rows[o]) + ", " +
                                            std::to_string(cols[o]) + ")");
        }
        col_out[k] = cols[o];
        val_out[k] = vals[o];
        ++rowptr_out[rows[o] + 1];
    }
    for (i64 i = 1; i <= m; ++i) rowptr_out[i] += rowptr_out[i - 1];
}

void partition_rows(i64 m, const i64* rowptr, int world, i64* bounds) {
    if (world < 1) throw std::invalid_argument("partition_rows: world must be >= 1");
    const i64 nnz = rowptr[m] - rowptr[0];
    bounds[0] = 0;
    for (int r = 1; r < world; ++r) {
        const i64 target = rowptr[0] + (nnz * r + world - 1) / world;
        const i64* it = std::lower_bound(rowptr, rowptr + m + 1, target);
        i64 b = static_cast<i64>(it - rowptr);
        b = std::clamp(b, bounds[r - 1], m);
        bounds[r] = b;
    }
    bounds[world] = m;
}

// Segment groups for the wide gather kernel (sparse.cu spmm_grp_kernel):
// consecutive segments, at most kGrpSegs of them and ~SVTB_SPMM_GROUP
// (default 384) entries, a segment never split — one warp streams several
// short rows through one continuous gather pipeline.
void build_groups(const std::vector<long long>& beg, const std::vector<long long>& end, cudaStream_t s, SegPlan& P) {
    static const long long ge = [] {
        const char* e = std::getenv("SVTB_SPMM_GROUP");
        return e ? std::max(1LL, std::atoll(e)) : 384LL;
    }();
    const i64 nsegs = static_cast<i64>(beg.size());
    std::vector<int> gf;
    gf.reserve(static_cast<size_t>(nsegs / 4 + 2));
    i64 q = 0;
    while (q < nsegs) {
        gf.push_back(static_cast<int>(q));
        long long tot = end[q] - beg[q];
        i64 r = q + 1;
        while (r < nsegs && r - q < kGrpSegs && tot + (end[r] - beg[r]) <= ge) {
            tot += end[r] - beg[r];
            ++r;
        }
        q = r;
    }
    gf.push_back(static_cast<int>(nsegs));
    P.grp_first.alloc(gf.size());
    SVT_CUDA(cudaMemcpyAsync(P.grp_first.get(), gf.data(), sizeof(int) * gf.size(), cudaMemcpyHostToDevice, s));
    // 32-entry chunks per segment, exclusive prefix (sddmm_warp_kernel's partition)
    std::vector<long long> co(static_cast<size_t>(nsegs) + 1);
    co[0] = 0;
    for (i64 k = 0; k < nsegs; ++k)
        co[static_cast<size_t>(k) + 1] = co[static_cast<size_t>(k)] + (end[static_cast<size_t>(k)] - beg[static_cast<size_t>(k)] + 31) / 32;
    P.chunk_off.alloc(co.size());
    SVT_CUDA(cudaMemcpyAsync(P.chunk_off.get(), co.data(), sizeof(long long) * co.size(), cudaMemcpyHostToDevice, s));
    SVT_CUDA(cudaStreamSynchronize(s));  // gf / co die here
    P.v.ngrp = static_cast<long long>(gf.size()) - 1;
    P.v.grp_first = P.grp_first.get();
    P.v.nchunks = co.back();
    P.v.chunk_off = P.chunk_off.get();
}

// Row segmentation for the load-balanced SpMM (sparse.cu): rows longer than
// kSegLen entries are cut into kSegLen chunks that write partial rows.
void build_plan(const std::vector<i64>& ptr, i64 nrows, cudaStream_t s, SegPlan& P) {
    std::vector<int> row, slot, lrow, lfirst, lcount;
    std::vector<long long> beg, end;
    int nslots = 0;
    for (i64 r = 0; r < nrows; ++r) {
        const i64 b = ptr[static_cast<size_t>(r)], e = ptr[static_cast<size_t>(r + 1)];
        const i64 len = e - b;
        if (len <= kSegLen) {
            row.push_back(static_cast<int>(r));
            beg.push_back(b);
            end.push_back(e);
            slot.push_back(-1);
            continue;
        }
        const i64 nseg = (len + kSegLen - 1) / kSegLen;
        lrow.push_back(static_cast<int>(r));
        lfirst.push_back(nslots);
        lcount.push_back(static_cast<int>(nseg));
        for (i64 q = 0; q < nseg; ++q) {
            row.push_back(static_cast<int>(r));
            beg.push_back(b + q * kSegLen);
            end.push_back(std::min<long long>(e, b + (q + 1) * kSegLen));
            slot.push_back(nslots++);
        }
    }
    auto up_i = [&](DevBuf<int>& d, const std::vector<int>& h) {
        d.alloc(std::max<size_t>(1, h.size()));
        if (!h.empty()) SVT_CUDA(cudaMemcpyAsync(d.get(), h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice, s));
    };
    auto up_l = [&](DevBuf<long long>& d, const std::vector<long long>& h) {
        d.alloc(std::max<size_t>(1, h.size()));
        if (!h.empty())
            SVT_CUDA(cudaMemcpyAsync(d.get(), h.data(), sizeof(long long) * h.size(), cudaMemcpyHostToDevice, s));
    };
    up_i(P.seg_row, row);
    up_i(P.seg_slot, slot);
    up_l(P.seg_beg, beg);
    up_l(P.seg_end, end);
    up_i(P.long_row, lrow);
    up_i(P.long_first, lfirst);
    up_i(P.long_count, lcount);
    SVT_CUDA(cudaStreamSynchronize(s));  // host vectors die here
    build_groups(beg, end, s, P);
    P.v.nseg = static_cast<long long>(row.size());
    P.v.seg_row = P.seg_row.get();
    P.v.seg_beg = P.seg_beg.get();
    P.v.seg_end = P.seg_end.get();
    P.v.seg_slot = P.seg_slot.get();
    P.v.nlong = static_cast<long long>(lrow.size());
    P.v.nslots = nslots;
    P.v.long_row = P.long_row.get();
    P.v.long_first = P.long_first.get();
    P.v.long_count = P.long_count.get();
}

}  // namespace svtb

using svtb::i64;

// Upload only the CSR arrays; validation, the CSC view, csr2csc and the
// segment plans are built on the device (build.cu).
static svt_mat* upload_device_build(svt_ctx* ctx, i64 m, i64 n, i64 row_begin, i64 row_end,
                                    const std::vector<i64>& rp, const i64* col, const double* val, i64 nnz) {
    const i64 ml = row_end - row_begin;
    auto* M = new svt_mat();
    try {
        M->ctx = ctx;
        M->m = m;
        M->n = n;
        M->row_begin = row_begin;
        M->row_end = row_end;
        M->m_local = ml;
        M->nnz_local = nnz;
        M->rowptr.alloc(static_cast<size_t>(ml + 1));
        M->col.alloc(static_cast<size_t>(std::max<i64>(1, nnz)));
        M->val.alloc(static_cast<size_t>(std::max<i64>(1, nnz)));
        M->colptr.alloc(static_cast<size_t>(n + 1));
        M->cscrow.alloc(static_cast<size_t>(std::max<i64>(1, nnz)));
        M->val_csc.alloc(static_cast<size_t>(std::max<i64>(1, nnz)));
        M->csr2csc.alloc(static_cast<size_t>(std::max<i64>(1, nnz)));
        svtb::DevBuf<i64> col64(static_cast<size_t>(std::max<i64>(1, nnz)));
        cudaStream_t s = ctx->stream;
        SVT_CUDA(cudaMemcpyAsync(M->rowptr.get(), rp.data(), sizeof(i64) * (ml + 1), cudaMemcpyHostToDevice, s));
        if (nnz > 0) {
            SVT_CUDA(cudaMemcpyAsync(col64.get(), col, sizeof(i64) * nnz, cudaMemcpyHostToDevice, s));
            SVT_CUDA(cudaMemcpyAsync(M->val.get(), val, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
        }
        const int code = svtb::build_sampled_device(ctx, M, reinterpret_cast<const long long*>(col64.get()));
        if (code & 1) throw std::invalid_argument("svt_matrix_upload: column out of range");
        if (code & 2) throw std::invalid_argument("svt_matrix_upload: non-finite value");
        double g = static_cast<double>(nnz);
        SVT_CUDA(cudaMemcpyAsync(ctx->d_scalars + 63, &g, sizeof(double), cudaMemcpyHostToDevice, s));
        ctx->comm.allreduce_sum(ctx->d_scalars + 63, 1, s);
        SVT_CUDA(cudaMemcpyAsync(&g, ctx->d_scalars + 63, sizeof(double), cudaMemcpyDeviceToHost, s));
        svtb::sync_stream(ctx);
        M->nnz_global = static_cast<i64>(g + 0.5);
    } catch (...) {
        delete M;
        throw;
    }
    return M;
}

svt_mat* svtb_matrix_upload(svt_ctx* ctx, i64 m, i64 n, i64 row_begin, i64 row_end, const i64* rowptr,
                            const i64* col, const double* val) {
    if (m < 1 || n < 1) throw std::invalid_argument("svt_matrix_upload: dimensions must be >= 1");
    if (row_begin < 0 || row_end < row_begin || row_end > m)
        throw std::invalid_argument("svt_matrix_upload: bad row block");
    const i64 ml = row_end - row_begin;
    const i64 base = rowptr[0];
    const i64 nnz = rowptr[ml] - base;
    if (nnz < 0) throw std::invalid_argument("svt_matrix_upload: bad rowptr");
    if (nnz > 2147483647LL) throw std::invalid_argument("svt_matrix_upload: > 2^31 entries per rank");
    std::vector<i64> rp(static_cast<size_t>(ml + 1));
    for (i64 i = 0; i <= ml; ++i) {
        rp[static_cast<size_t>(i)] = rowptr[i] - base;
        if (i > 0 && rp[static_cast<size_t>(i)] < rp[static_cast<size_t>(i - 1)])
            throw std::invalid_argument("svt_matrix_upload: rowptr not monotone");
    }
    if (!std::getenv("SVTB_HOST_BUILD")) return upload_device_build(ctx, m, n, row_begin, row_end, rp, col + base,
                                                                    val + base, nnz);
    std::vector<int> ci(static_cast<size_t>(nnz));
    for (i64 k = 0; k < nnz; ++k) {
        const i64 c = col[base + k];
        if (c < 0 || c >= n) throw std::invalid_argument("svt_matrix_upload: column out of range");
        if (!std::isfinite(val[base + k])) throw std::invalid_argument("svt_matrix_upload: non-finite value");
        ci[static_cast<size_t>(k)] = static_cast<int>(c);
    }
    // CSC view by counting sort (stable in row order)
    std::vector<i64> cp(static_cast<size_t>(n + 1), 0);
    for (i64 k = 0; k < nnz; ++k) ++cp[static_cast<size_t>(ci[static_cast<size_t>(k)]) + 1];
    for (i64 j = 1; j <= n; ++j) cp[static_cast<size_t>(j)] += cp[static_cast<size_t>(j - 1)];
    std::vector<i64> fillp(cp.begin(), cp.end() - 1);
    std::vector<int> crow(static_cast<size_t>(nnz)), c2c(static_cast<size_t>(nnz));
    std::vector<double> vcsc(static_cast<size_t>(nnz));
    for (i64 i = 0; i < ml; ++i)
        for (i64 k = rp[static_cast<size_t>(i)]; k < rp[static_cast<size_t>(i + 1)]; ++k) {
            const i64 pos = fillp[static_cast<size_t>(ci[static_cast<size_t>(k)])]++;
            crow[static_cast<size_t>(pos)] = static_cast<int>(i);
            c2c[static_cast<size_t>(k)] = static_cast<int>(pos);
            vcsc[static_cast<size_t>(pos)] = val[base + k];
        }
    auto* M = new svt_mat();
    try {
        M->ctx = ctx;
        M->m = m;
        M->n = n;
        M->row_begin = row_begin;
        M->row_end = row_end;
        M->m_local = ml;
        M->nnz_local = nnz;
        M->rowptr.alloc(static_cast<size_t>(ml + 1));
        M->col.alloc(static_cast<size_t>(std::max<i64>(1, nnz)));
        M->val.alloc(static_cast<size_t>(std::max<i64>(1, nnz)));
        M->colptr.alloc(static_cast<size_t>(n + 1));
        M->cscrow.alloc(static_cast<size_t>(std::max<i64>(1, nnz)));
        M->val_csc.alloc(static_cast<size_t>(std::max<i64>(1, nnz)));
        M->csr2csc.alloc(static_cast<size_t>(std::max<i64>(1, nnz)));
        cudaStream_t s = ctx->stream;
        SVT_CUDA(cudaMemcpyAsync(M->rowptr.get(), rp.data(), sizeof(i64) * (ml + 1), cudaMemcpyHostToDevice, s));
        SVT_CUDA(cudaMemcpyAsync(M->colptr.get(), cp.data(), sizeof(i64) * (n + 1), cudaMemcpyHostToDevice, s));
        if (nnz > 0) {
            SVT_CUDA(cudaMemcpyAsync(M->col.get(), ci.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice, s));
            SVT_CUDA(cudaMemcpyAsync(M->val.get(), val + base, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
            SVT_CUDA(cudaMemcpyAsync(M->cscrow.get(), crow.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice, s));
            SVT_CUDA(cudaMemcpyAsync(M->val_csc.get(), vcsc.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
            SVT_CUDA(cudaMemcpyAsync(M->csr2csc.get(), c2c.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice, s));
        }
        svtb::build_plan(rp, ml, s, M->plan_csr);
        svtb::build_plan(cp, n, s, M->plan_csc);
        // global nnz (all ranks)
        double g = static_cast<double>(nnz);
        SVT_CUDA(cudaMemcpyAsync(ctx->d_scalars + 63, &g, sizeof(double), cudaMemcpyHostToDevice, s));
        ctx->comm.allreduce_sum(ctx->d_scalars + 63, 1, s);
        SVT_CUDA(cudaMemcpyAsync(&g, ctx->d_scalars + 63, sizeof(double), cudaMemcpyDeviceToHost, s));
        SVT_CUDA(cudaStreamSynchronize(s));
        M->nnz_global = static_cast<i64>(g + 0.5);
    } catch (...) {
        delete M;
        throw;
    }
    return M;
}
