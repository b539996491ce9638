// The C ABI (include/svt_b200.h).  Every entry point catches and maps the
// engine's exceptions to the status codes that correspond to the reference's
// exception types; messages are kept per thread for svt_last_error().
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "engine.hpp"
#include "io.hpp"
#include "kernels.hpp"

namespace svtb {
void sampled_build(i64 m, i64 n, i64 nnz, const i64* rows, const i64* cols, const double* vals, i64* rowptr_out,
                   i64* col_out, double* val_out);
void partition_rows(i64 m, const i64* rowptr, int world, i64* bounds);
svt_solver* solver_create(svt_mat* A, const svt_config& cfg, svt_stop stop, svt_backend backend, svt_mat* test);
void solver_step(svt_solver* S, svt_observer_fn obs, void* user, svt_record* rec_out, int* done);
svt_result* solver_result(svt_solver* S);
void solver_checkpoint(svt_solver* S, svt_solver_state* st, double* y_vals, double* u_prev, double* best_U,
                       double* best_sigma, double* best_V);
svt_solver* solver_resume(svt_mat* A, const svt_config& cfg, svt_stop stop, svt_backend backend, svt_mat* test,
                          const svt_solver_state& st, const double* y_vals, const double* u_prev,
                          const double* best_U, const double* best_sigma, const double* best_V);
void kickstart_dev(svt_ctx* c, svt_mat* A, double tau, double delta, u64 seed, double* out_csr, double* out_csc);
void synth_config(int config, u64 seed, i64* m, i64* n, i64* nnz_train, i64* nnz_test, i64* train_rows,
                  i64* train_cols, double* train_vals, i64* test_rows, i64* test_cols, double* test_vals);
void synth_config_csr(int config, u64 seed, i64* m, i64* n, i64* nnz, i64* rowptr, i64* col, double* val);
std::vector<double> make_low_rank_cm(i64 m, i64 n, i64 rank, u64 seed);
void sample_dense(i64 m, i64 n, const double* A_cm, double fraction, u64 seed, std::vector<i64>& r,
                  std::vector<i64>& c, std::vector<double>& v);
std::vector<unsigned char> synthetic_image(i64 size, i64 rank, u64 seed);
void synthetic_ratings(i64 users, i64 items, i64 rank, double fill, double noise, u64 seed, std::vector<i64>& r,
                       std::vector<i64>& c, std::vector<double>& v);
u64 derive_seed_u(u64 seed, u64 stream);
}  // namespace svtb

svt_mat* svtb_matrix_upload(svt_ctx* ctx, svtb::i64 m, svtb::i64 n, svtb::i64 row_begin, svtb::i64 row_end,
                            const svtb::i64* rowptr, const svtb::i64* col, const double* val);

using namespace svtb;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return SVT_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SVT_EINVAL;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return SVT_EDOMAIN;
    } catch (const cuda_error& e) {
        g_err = e.what();
        return SVT_ECUDA;
    } catch (const nccl_error& e) {
        g_err = e.what();
        return SVT_ENCCL;
    } catch (const oom_error& e) {
        g_err = e.what();
        return SVT_EOOM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SVT_ERUNTIME;
    } catch (...) {
        g_err = "unknown error";
        return SVT_ERUNTIME;
    }
}

void need(const void* p, const char* what) {
    if (p == nullptr) throw std::invalid_argument(std::string(what) + ": null argument");
}

// column-major host (rows x cols) -> row-major device (rows x cols, ld cols)
DevBuf<double> upload_cm(svt_ctx* c, const double* h, i64 rows, i64 cols) {
    DevBuf<double> d(static_cast<size_t>(std::max<i64>(1, rows * cols)));
    if (rows * cols == 0) return d;
    std::vector<double> rm(static_cast<size_t>(rows * cols));
    for (i64 i = 0; i < rows; ++i)
        for (i64 j = 0; j < cols; ++j) rm[static_cast<size_t>(i * cols + j)] = h[i + j * rows];
    SVT_CUDA(cudaMemcpyAsync(d.get(), rm.data(), sizeof(double) * rm.size(), cudaMemcpyHostToDevice, c->stream));
    sync_stream(c);
    return d;
}

void download_cm(svt_ctx* c, const double* d, i64 rows, i64 cols, i64 ld, double* h) {
    if (rows * cols == 0) return;
    std::vector<double> rm(static_cast<size_t>(rows * ld));
    SVT_CUDA(cudaMemcpyAsync(rm.data(), d, sizeof(double) * rows * ld, cudaMemcpyDeviceToHost, c->stream));
    sync_stream(c);
    for (i64 i = 0; i < rows; ++i)
        for (i64 j = 0; j < cols; ++j) h[i + j * rows] = rm[static_cast<size_t>(i * ld + j)];
}

Engine engine_for(svt_mat* S) { return Engine(S->ctx, S, Vals{S->val.get(), S->val_csc.get()}); }

}  // namespace

extern "C" {

const char* svt_last_error(void) { return g_err.c_str(); }

int svt_version(void) { return 1; }

static void ctx_create(int device, int rank, int world, const void* nccl_id, svt_allreduce_fn host_fn,
                       void* host_user, svt_ctx** out) {
        need(out, "svt_ctx_create");
        if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("svt_ctx_create: bad rank/world");
        if (world > 1 && host_fn == nullptr) need(nccl_id, "svt_ctx_create_dist: nccl_id");
        int ndev = 0;
        SVT_CUDA(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) throw std::invalid_argument("svt_ctx_create: no such CUDA device");
        SVT_CUDA(cudaSetDevice(device));
        auto c = std::make_unique<svt_ctx>();
        c->device = device;
        // the main stream carries the critical path (Gram-Schmidt / QR of the
        // batch in flight); the side stream's speculative sketch fills the
        // SMs it leaves idle: give the main stream the higher priority
        int prio_lo = 0, prio_hi = 0;
        SVT_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        // SVTB_FLAT_PRIORITY / SVTB_SIDE_PRIORITY (A/B switches): equal
        // priorities / the side stream above the main stream
        static const bool flat = std::getenv("SVTB_FLAT_PRIORITY") != nullptr;
        static const bool side_first = std::getenv("SVTB_SIDE_PRIORITY") != nullptr;
        SVT_CUDA(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking,
                                              (flat || side_first) ? prio_lo : prio_hi));
        SVT_CUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, side_first ? prio_hi : prio_lo));
        SVT_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
        SVT_CUDA(cudaMallocHost(&c->h_scalars, 64 * sizeof(double)));
        SVT_CUDA(cudaMallocHost(&c->h_flags, 64 * sizeof(int)));
        c->h_stage_n = 1 << 16;
        SVT_CUDA(cudaMallocHost(&c->h_stage, c->h_stage_n * sizeof(double)));
        SVT_CUDA(cudaMalloc(&c->d_scalars, 64 * sizeof(double)));
        SVT_CUDA(cudaMalloc(&c->d_flags, 64 * sizeof(int)));
        SVT_CUDA(cudaMemsetAsync(c->d_scalars, 0, 64 * sizeof(double), c->stream));
        SVT_CUDA(cudaMemsetAsync(c->d_flags, 0, 64 * sizeof(int), c->stream));
        // reduction / permutation scratch sized once (regrowing inside an SVT
        // iteration would cudaFree: a device-wide sync)
        c->ws_partial2.alloc(size_t(4) << 20);
        c->ws_perm.alloc(4096);
        c->ws_eig.alloc(static_cast<size_t>(2 * 1056 * 1056 + 1056));  // dense Gram eigensolve up to r = 1056
        c->ws_info.alloc(8);
        c->d_tickets.alloc(kTickets);
        SVT_CUDA(cudaMemsetAsync(c->d_tickets.get(), 0, kTickets * sizeof(unsigned), c->stream));
        if (host_fn != nullptr) {
            c->comm.rank = rank;
            c->comm.world = world;
            c->comm.host_fn = host_fn;
            c->comm.host_user = host_user;
        } else {
            nccl_init(c->comm, rank, world, nccl_id);
        }
        sync_stream(c.get());
        *out = c.release();
}

int svt_ctx_create_dist(int device, int rank, int world, const void* nccl_id, svt_ctx** out) {
    return guard([&] { ctx_create(device, rank, world, nccl_id, nullptr, nullptr, out); });
}

int svt_ctx_create_hostcomm(int device, int rank, int world, svt_allreduce_fn fn, void* user, svt_ctx** out) {
    return guard([&] {
        need(reinterpret_cast<const void*>(fn), "svt_ctx_create_hostcomm: fn");
        ctx_create(device, rank, world, nullptr, fn, user, out);
    });
}

int svt_ctx_comm_stats(svt_ctx* ctx, int64_t* calls, double* doubles) {
    return guard([&] {
        need(ctx, "svt_ctx_comm_stats");
        if (calls) *calls = ctx->comm.calls;
        if (doubles) *doubles = ctx->comm.doubles;
    });
}

int svt_ctx_create(int device, svt_ctx** out) { return svt_ctx_create_dist(device, 0, 1, nullptr, out); }

int svt_nccl_get_unique_id(void* out128) {
    return guard([&] {
        need(out128, "svt_nccl_get_unique_id");
        nccl_unique_id(out128);
    });
}

int svt_ctx_destroy(svt_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        if (ctx->side) cudaStreamSynchronize(ctx->side);
        for (auto& p : ctx->pending) {
            cudaEventDestroy(p.a);
            cudaEventDestroy(p.b);
        }
        for (auto e : ctx->event_pool) cudaEventDestroy(e);
        ctx->comm.destroy();
        ctx->ws_partial.release();
        ctx->ws_partial2.release();
        ctx->ws_rng.release();
        ctx->ws_rng_side.release();
        ctx->ws_mt.release();
        ctx->ws_eig.release();
        ctx->ws_info.release();
        cudaFree(ctx->d_scalars);
        cudaFree(ctx->d_flags);
        cudaFreeHost(ctx->h_scalars);
        cudaFreeHost(ctx->h_flags);
        if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
        cudaStreamDestroy(ctx->stream);
        if (ctx->side) cudaStreamDestroy(ctx->side);
        for (int k = 0; k < 2; ++k) {
            if (ctx->aux[k]) cudaStreamDestroy(ctx->aux[k]);
            if (ctx->aux_fork[k]) cudaEventDestroy(ctx->aux_fork[k]);
            if (ctx->aux_join[k]) cudaEventDestroy(ctx->aux_join[k]);
        }
        delete ctx;
    });
}

int svt_ctx_sync(svt_ctx* ctx) {
    return guard([&] {
        need(ctx, "svt_ctx_sync");
        sync_stream(ctx);
    });
}

int svt_ctx_join(svt_ctx* ctx) {
    return guard([&] {
        need(ctx, "svt_ctx_join");
        if (!ctx->side) return;
        cudaEvent_t ev;
        SVT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        SVT_CUDA(cudaEventRecord(ev, ctx->side));
        SVT_CUDA(cudaStreamWaitEvent(ctx->stream, ev, 0));
        SVT_CUDA(cudaEventDestroy(ev));
    });
}

void* svt_ctx_stream(svt_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int svt_ctx_rank(svt_ctx* ctx, int* rank, int* world) {
    return guard([&] {
        need(ctx, "svt_ctx_rank");
        if (rank) *rank = ctx->comm.rank;
        if (world) *world = ctx->comm.world;
    });
}

int svt_ctx_set_profiling(svt_ctx* ctx, int on) {
    return guard([&] {
        need(ctx, "svt_ctx_set_profiling");
        flush_stats(ctx);
        ctx->profiling = on != 0;
        ctx->gap_debug = ctx->profiling && std::getenv("SVTB_DEBUG_GAPS") != nullptr;
    });
}

int svt_ctx_set_speculation(svt_ctx* ctx, int on) {
    return guard([&] {
        need(ctx, "svt_ctx_set_speculation");
        ctx->speculate = on != 0;
    });
}

int svt_ctx_reset_stats(svt_ctx* ctx) {
    return guard([&] {
        need(ctx, "svt_ctx_reset_stats");
        flush_stats(ctx);
        for (auto& s : ctx->stats) s = KStats{};
        ctx->launch_count = 0;
        ctx->host_syncs = 0;
        ctx->host_sync_ms = 0.0;
    });
}

int svt_ctx_kernel_stats(svt_ctx* ctx, int cls, int64_t* launches, double* total_ms, double* bytes, double* flops) {
    return guard([&] {
        need(ctx, "svt_ctx_kernel_stats");
        if (cls < 0 || cls >= K_NCLASS) throw std::invalid_argument("svt_ctx_kernel_stats: bad class");
        flush_stats(ctx);
        const KStats& s = ctx->stats[cls];
        if (launches) *launches = s.launches;
        if (total_ms) *total_ms = s.total_ms;
        if (bytes) *bytes = s.bytes;
        if (flops) *flops = s.flops;
    });
}

int64_t svt_ctx_launch_count(svt_ctx* ctx) { return ctx ? ctx->launch_count : -1; }

int svt_ctx_host_stats(svt_ctx* ctx, int64_t* syncs, double* sync_ms) {
    return guard([&] {
        need(ctx, "svt_ctx_host_stats");
        if (ctx->gap_debug) print_gap_stats(ctx);
        if (syncs) *syncs = ctx->host_syncs;
        if (sync_ms) *sync_ms = ctx->host_sync_ms;
    });
}

int svt_ctx_set_batching(svt_ctx* ctx, int on) {
    return guard([&] {
        need(ctx, "svt_ctx_set_batching");
        ctx->batching = on ? 1 : 0;
    });
}

int svt_sampled_build(int64_t m, int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols, const double* vals,
                      int64_t* rowptr_out, int64_t* col_out, double* val_out) {
    return guard([&] {
        if (nnz > 0) {
            need(rows, "svt_sampled_build");
            need(cols, "svt_sampled_build");
            need(vals, "svt_sampled_build");
        }
        need(rowptr_out, "svt_sampled_build");
        sampled_build(m, n, nnz, rows, cols, vals, rowptr_out, col_out, val_out);
    });
}

int svt_partition_rows(int64_t m, const int64_t* rowptr, int world, int64_t* bounds) {
    return guard([&] {
        need(rowptr, "svt_partition_rows");
        need(bounds, "svt_partition_rows");
        partition_rows(m, rowptr, world, bounds);
    });
}

int svt_matrix_upload(svt_ctx* ctx, int64_t m, int64_t n, int64_t row_begin, int64_t row_end, const int64_t* rowptr,
                      const int64_t* col, const double* val, svt_mat** out) {
    return guard([&] {
        need(ctx, "svt_matrix_upload");
        need(rowptr, "svt_matrix_upload");
        need(out, "svt_matrix_upload");
        SVT_CUDA(cudaSetDevice(ctx->device));
        *out = svtb_matrix_upload(ctx, m, n, row_begin, row_end, rowptr, col, val);
    });
}

int svt_matrix_from_triplets(svt_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                             const int64_t* cols, const double* vals, int64_t row_begin, int64_t row_end,
                             svt_mat** out) {
    return guard([&] {
        need(ctx, "svt_matrix_from_triplets");
        need(out, "svt_matrix_from_triplets");
        if (m < 1 || n < 1) throw std::invalid_argument("SampledMatrix: dimensions must be >= 1");
        if (nnz < 1) throw std::invalid_argument("SampledMatrix: at least one entry required");
        if (nnz > 2147483647LL) throw std::invalid_argument("SampledMatrix: more than 2^31 entries");
        if (!rows || !cols || !vals) throw std::invalid_argument("SampledMatrix: null triplet array");
        if (row_begin < 0 || row_end < row_begin || row_end > m)
            throw std::invalid_argument("svt_matrix_upload: bad row block");
        SVT_CUDA(cudaSetDevice(ctx->device));
        auto M = std::make_unique<svt_mat>();
        M->ctx = ctx;
        M->m = m;
        M->n = n;
        M->row_begin = row_begin;
        M->row_end = row_end;
        M->m_local = row_end - row_begin;
        M->rowptr.alloc(static_cast<size_t>(M->m_local + 1));
        M->colptr.alloc(static_cast<size_t>(n + 1));
        build_from_triplets_device(ctx, M.get(), nnz, rows, cols, vals);
        double g = static_cast<double>(M->nnz_local);
        SVT_CUDA(cudaMemcpyAsync(ctx->d_scalars + 63, &g, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        ctx->comm.allreduce_sum(ctx->d_scalars + 63, 1, ctx->stream);
        SVT_CUDA(cudaMemcpyAsync(&g, ctx->d_scalars + 63, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        sync_stream(ctx);
        M->nnz_global = static_cast<i64>(g + 0.5);
        *out = M.release();
    });
}

int svt_matrix_csr(svt_mat* mat, int64_t* rowptr, int64_t* col, double* val) {
    return guard([&] {
        need(mat, "svt_matrix_csr");
        svt_ctx* c = mat->ctx;
        const i64 nnz = mat->nnz_local, ml = mat->m_local;
        if (rowptr)
            SVT_CUDA(cudaMemcpyAsync(rowptr, mat->rowptr.get(), sizeof(int64_t) * (ml + 1), cudaMemcpyDeviceToHost,
                                     c->stream));
        std::vector<int> ci;
        if (col && nnz > 0) {
            ci.resize(static_cast<size_t>(nnz));
            SVT_CUDA(cudaMemcpyAsync(ci.data(), mat->col.get(), sizeof(int) * nnz, cudaMemcpyDeviceToHost, c->stream));
        }
        if (val && nnz > 0)
            SVT_CUDA(cudaMemcpyAsync(val, mat->val.get(), sizeof(double) * nnz, cudaMemcpyDeviceToHost, c->stream));
        sync_stream(c);
        for (i64 k = 0; k < static_cast<i64>(ci.size()); ++k) col[k] = ci[static_cast<size_t>(k)];
    });
}

// ---- formats ---------------------------------------------------------------
struct svt_triplets {
    svtb::Triplets t;
};

int svt_read_matrix_market(const char* path, svt_triplets** out) {
    return guard([&] {
        need(path, "svt_read_matrix_market");
        need(out, "svt_read_matrix_market");
        auto T = std::make_unique<svt_triplets>();
        T->t = svtb::read_matrix_market(path);
        *out = T.release();
    });
}

int svt_read_ratings(const char* path, const char* separator, svt_triplets** out) {
    return guard([&] {
        need(path, "svt_read_ratings");
        need(out, "svt_read_ratings");
        auto T = std::make_unique<svt_triplets>();
        T->t = svtb::read_ratings(path, separator ? separator : "::");
        *out = T.release();
    });
}

int svt_sample_image(int64_t width, int64_t height, const uint8_t* pixels, double fraction, uint64_t seed,
                     svt_triplets** out) {
    return guard([&] {
        need(pixels, "svt_sample_image");
        need(out, "svt_sample_image");
        if (width < 1 || height < 1) throw std::invalid_argument("sample_image: bad dimensions");
        auto T = std::make_unique<svt_triplets>();
        T->t = svtb::sample_image(width, height, pixels, fraction, seed);
        *out = T.release();
    });
}

int svt_split_ratings(svt_triplets* ds, double train_fraction, uint64_t seed, svt_triplets** train,
                      svt_triplets** test) {
    return guard([&] {
        need(ds, "svt_split_ratings");
        need(train, "svt_split_ratings");
        need(test, "svt_split_ratings");
        auto A = std::make_unique<svt_triplets>(), B = std::make_unique<svt_triplets>();
        svtb::split_ratings(ds->t, train_fraction, seed, A->t, B->t);
        *train = A.release();
        *test = B.release();
    });
}

int svt_triplets_create(int64_t m, int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                        const double* vals, svt_triplets** out) {
    return guard([&] {
        need(out, "svt_triplets_create");
        if (m < 0 || n < 0 || nnz < 0 || (nnz > 0 && (!rows || !cols || !vals)))
            throw std::invalid_argument("svt_triplets_create: bad arguments");
        auto T = std::make_unique<svt_triplets>();
        T->t.m = m;
        T->t.n = n;
        T->t.r.assign(rows, rows + nnz);
        T->t.c.assign(cols, cols + nnz);
        T->t.v.assign(vals, vals + nnz);
        *out = T.release();
    });
}

int svt_triplets_info(svt_triplets* t, int64_t* m, int64_t* n, int64_t* nnz) {
    return guard([&] {
        need(t, "svt_triplets_info");
        if (m) *m = t->t.m;
        if (n) *n = t->t.n;
        if (nnz) *nnz = static_cast<int64_t>(t->t.r.size());
    });
}

int svt_triplets_copy(svt_triplets* t, int64_t* rows, int64_t* cols, double* vals) {
    return guard([&] {
        need(t, "svt_triplets_copy");
        const size_t k = t->t.r.size();
        if (rows) std::memcpy(rows, t->t.r.data(), sizeof(int64_t) * k);
        if (cols) std::memcpy(cols, t->t.c.data(), sizeof(int64_t) * k);
        if (vals) std::memcpy(vals, t->t.v.data(), sizeof(double) * k);
    });
}

int svt_triplets_ids(svt_triplets* t, int64_t* user_ids, int64_t* item_ids) {
    return guard([&] {
        need(t, "svt_triplets_ids");
        if (t->t.user_ids.empty()) throw std::invalid_argument("svt_triplets_ids: not a ratings set");
        if (user_ids) std::memcpy(user_ids, t->t.user_ids.data(), sizeof(int64_t) * t->t.user_ids.size());
        if (item_ids) std::memcpy(item_ids, t->t.item_ids.data(), sizeof(int64_t) * t->t.item_ids.size());
    });
}

const char* svt_triplets_provenance(svt_triplets* t) { return t ? t->t.provenance.c_str() : ""; }

int svt_triplets_free(svt_triplets* t) {
    return guard([&] { delete t; });
}

int svt_matrix_from_triplet_set(svt_ctx* ctx, svt_triplets* t, int64_t row_begin, int64_t row_end, svt_mat** out) {
    const int g = guard([&] { need(t, "svt_matrix_from_triplet_set"); });
    if (g != SVT_OK) return g;
    const int64_t one = 0;
    const double zero = 0.0;
    const bool e = t->t.r.empty();
    return svt_matrix_from_triplets(ctx, t->t.m, t->t.n, static_cast<int64_t>(t->t.r.size()),
                                    e ? &one : t->t.r.data(), e ? &one : t->t.c.data(), e ? &zero : t->t.v.data(),
                                    row_begin, row_end, out);
}

int svt_write_matrix_market(const char* path, int64_t m, int64_t n, const int64_t* rowptr, const int64_t* col,
                            const double* val) {
    return guard([&] {
        need(path, "svt_write_matrix_market");
        need(rowptr, "svt_write_matrix_market");
        if (m < 1 || n < 1) throw std::invalid_argument("write_matrix_market: bad dimensions");
        svtb::write_matrix_market(path, m, n, rowptr, col, val);
    });
}

int svt_read_matrix_market_array(const char* path, int64_t* rows, int64_t* cols, double* data) {
    return guard([&] {
        need(path, "svt_read_matrix_market_array");
        i64 r = 0, c = 0;
        const auto X = svtb::read_matrix_market_array(path, r, c);
        if (rows) *rows = r;
        if (cols) *cols = c;
        if (data) std::memcpy(data, X.data(), sizeof(double) * X.size());
    });
}

int svt_write_matrix_market_array(const char* path, int64_t rows, int64_t cols, const double* data) {
    return guard([&] {
        need(path, "svt_write_matrix_market_array");
        if (rows < 0 || cols < 0 || (rows * cols > 0 && !data))
            throw std::invalid_argument("write_matrix_market_array: bad arguments");
        svtb::write_matrix_market_array(path, rows, cols, data);
    });
}

int svt_read_pgm(const char* path, int64_t* width, int64_t* height, uint8_t* pixels) {
    return guard([&] {
        need(path, "svt_read_pgm");
        i64 w = 0, h = 0;
        const auto px = svtb::read_pgm(path, w, h);
        if (width) *width = w;
        if (height) *height = h;
        if (pixels) std::memcpy(pixels, px.data(), px.size());
    });
}

int svt_write_pgm(const char* path, int64_t width, int64_t height, const uint8_t* pixels) {
    return guard([&] {
        need(path, "svt_write_pgm");
        svtb::write_pgm(path, width, height, pixels);
    });
}

int svt_quantize_image(int64_t rows, int64_t cols, const double* X, uint8_t* pixels) {
    return guard([&] {
        need(X, "svt_quantize_image");
        need(pixels, "svt_quantize_image");
        if (rows < 0 || cols < 0) throw std::invalid_argument("quantize_image: bad dimensions");
        svtb::quantize_image(rows, cols, X, pixels);
    });
}

int svt_write_trace(const svt_record* records, int64_t count, const char* path, int json) {
    return guard([&] {
        need(path, "svt_write_trace");
        if (count < 0 || (count > 0 && !records)) throw std::invalid_argument("svt_write_trace: bad records");
        svtb::write_trace(records, count, path, json != 0);
    });
}

int svt_matrix_free(svt_mat* mat) {
    return guard([&] { delete mat; });
}

int svt_matrix_info(svt_mat* M, int64_t* m, int64_t* n, int64_t* nnz_local, int64_t* row_begin, int64_t* row_end) {
    return guard([&] {
        need(M, "svt_matrix_info");
        if (m) *m = M->m;
        if (n) *n = M->n;
        if (nnz_local) *nnz_local = M->nnz_local;
        if (row_begin) *row_begin = M->row_begin;
        if (row_end) *row_end = M->row_end;
    });
}

int svt_matrix_hybrid_info(svt_mat* M, int* on, int64_t* rows, int64_t* cols, int64_t* nnz_block,
                           int64_t* nnz_cold) {
    return guard([&] {
        need(M, "svt_matrix_hybrid_info");
        ensure_hybrid(M->ctx, M);
        const HybridPlan& H = M->hyb;
        if (on) *on = H.on ? 1 : 0;
        if (rows) *rows = H.R;
        if (cols) *cols = H.C;
        if (nnz_block) *nnz_block = H.nnz_blk;
        if (nnz_cold) *nnz_cold = H.nnz_cold;
    });
}

int svt_matrix_set_values(svt_mat* M, const double* vals) {
    return guard([&] {
        need(M, "svt_matrix_set_values");
        if (M->nnz_local == 0) return;
        need(vals, "svt_matrix_set_values");
        for (i64 k = 0; k < M->nnz_local; ++k)
            if (!std::isfinite(vals[k])) throw std::invalid_argument("with_values: non-finite value");
        svt_ctx* c = M->ctx;
        SVT_CUDA(cudaMemcpyAsync(M->val.get(), vals, sizeof(double) * M->nnz_local, cudaMemcpyHostToDevice, c->stream));
        scale_values(c, M->nnz_local, M->val.get(), 1.0, M->val.get(), M->csr2csc.get(), M->val_csc.get());
        M->val_version++;
        sync_stream(c);
    });
}

int svt_matrix_get_values(svt_mat* M, double* vals) {
    return guard([&] {
        need(M, "svt_matrix_get_values");
        if (M->nnz_local == 0) return;
        need(vals, "svt_matrix_get_values");
        svt_ctx* c = M->ctx;
        SVT_CUDA(cudaMemcpyAsync(vals, M->val.get(), sizeof(double) * M->nnz_local, cudaMemcpyDeviceToHost, c->stream));
        sync_stream(c);
    });
}

// ---- primitives ----------------------------------------------------------
int svt_gaussian_block(svt_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, double* out) {
    return guard([&] {
        need(ctx, "svt_gaussian_block");
        if (rows < 1 || cols < 1) throw std::invalid_argument("gaussian_block: dimensions must be >= 1");
        need(out, "svt_gaussian_block");
        DevBuf<double> d(static_cast<size_t>(rows * cols));
        gaussian_block_dev(ctx, rows, cols, seed, d.get(), cols);
        download_cm(ctx, d.get(), rows, cols, cols, out);
    });
}

int svt_qr_orthonormal(svt_ctx* ctx, int64_t rows, int64_t cols, const double* X, double* Q) {
    return guard([&] {
        need(ctx, "svt_qr_orthonormal");
        if (cols > rows)
            throw std::invalid_argument("qr_orthonormal: need cols <= rows, got " + std::to_string(rows) + "x" +
                                        std::to_string(cols));
        if (rows * cols == 0) return;
        // a row-block-free helper matrix: Engine needs m_local for the panel height
        svt_mat fake;
        fake.ctx = ctx;
        fake.m = rows;
        fake.m_local = rows;
        fake.n = rows;
        fake.row_end = rows;
        Engine E(ctx, &fake, Vals{nullptr, nullptr});
        if (ctx->comm.world != 1) throw std::invalid_argument("svt_qr_orthonormal: single-rank helper");
        DevBuf<double> dX = upload_cm(ctx, X, rows, cols);
        DevBuf<double> dQ(static_cast<size_t>(rows * cols));
        qr_orthonormal(E, dX.get(), cols, cols, dQ.get(), cols);
        download_cm(ctx, dQ.get(), rows, cols, cols, Q);
    });
}

int svt_small_svd(svt_ctx* ctx, int64_t rows, int64_t cols, const double* B, double* U, double* sigma, double* V) {
    return guard([&] {
        need(ctx, "svt_small_svd");
        if (rows < 1 || cols < 1) throw std::invalid_argument("small_svd: empty block");
        // finalize with Q = I: B = I * B, Gram of the shorter side
        const bool tr = rows > cols;
        const i64 r = tr ? cols : rows, n = tr ? rows : cols;
        svt_mat fake;
        fake.ctx = ctx;
        fake.m = r;
        fake.m_local = r;
        fake.n = n;
        fake.row_end = r;
        Engine E(ctx, &fake, Vals{nullptr, nullptr});
        QBDev st;
        st.m_local = r;
        st.n = n;
        st.min_dim = r;
        st.cap = r;
        st.rank = r;
        std::vector<double> eye(static_cast<size_t>(r * r), 0.0);
        for (i64 i = 0; i < r; ++i) eye[static_cast<size_t>(i * r + i)] = 1.0;
        st.Q.alloc(static_cast<size_t>(r * r));
        SVT_CUDA(cudaMemcpyAsync(st.Q.get(), eye.data(), sizeof(double) * r * r, cudaMemcpyHostToDevice, ctx->stream));
        // B^T (n x r) row-major == B (r x n) column-major; for tr, B^T == B^T
        std::vector<double> bt(static_cast<size_t>(n * r));
        for (i64 i = 0; i < r; ++i)
            for (i64 j = 0; j < n; ++j) {
                const double v = tr ? B[j + i * rows] : B[i + j * rows];  // (i, j) of the short-side matrix
                bt[static_cast<size_t>(j * r + i)] = v;
            }
        st.Bt.alloc(static_cast<size_t>(n * r));
        SVT_CUDA(cudaMemcpyAsync(st.Bt.get(), bt.data(), sizeof(double) * n * r, cudaMemcpyHostToDevice, ctx->stream));
        DevFactors f;
        finalize(E, st, FinalizeMode::Full, 0.0, f);
        const i64 k = f.k;
        std::vector<double> Ur, Vr;
        std::vector<double> hU(static_cast<size_t>(r * k)), hV(static_cast<size_t>(n * k));
        download_cm(ctx, f.U.get(), r, k, k, hU.data());
        download_cm(ctx, f.V.get(), n, k, k, hV.data());
        if (!tr) {
            std::memcpy(U, hU.data(), sizeof(double) * r * k);
            std::memcpy(V, hV.data(), sizeof(double) * n * k);
        } else {
            std::memcpy(U, hV.data(), sizeof(double) * n * k);
            std::memcpy(V, hU.data(), sizeof(double) * r * k);
        }
        std::memcpy(sigma, f.sigma.data(), sizeof(double) * k);
    });
}

int svt_dev_gemm(svt_ctx* ctx, int transA, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                 int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
    return guard([&] {
        need(ctx, "svt_dev_gemm");
        if (M < 0 || N < 0 || K < 0) throw std::invalid_argument("dev_gemm: negative dimension");
        if (!A || !B || !C) throw std::invalid_argument("dev_gemm: null operand");
        if (ldb < N || ldc < N || lda < (transA ? M : K)) throw std::invalid_argument("dev_gemm: leading dimension");
        gemm(ctx, K_GEMM, transA != 0, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    });
}

int svt_dev_sym_eig(svt_ctx* ctx, const double* G, int64_t r, double* W, double* lambda) {
    return guard([&] {
        need(ctx, "svt_dev_sym_eig");
        if (r < 0) throw std::invalid_argument("dev_sym_eig: negative order");
        if (r == 0) return;
        if (!G || !W || !lambda) throw std::invalid_argument("dev_sym_eig: null operand");
        // sym_eig may overwrite its input: work on a copy
        DevBuf<double> Gc(static_cast<size_t>(r * r));
        SVT_CUDA(cudaMemcpyAsync(Gc.get(), G, sizeof(double) * r * r, cudaMemcpyDeviceToDevice, ctx->stream));
        sym_eig(ctx, Gc.get(), r, W, lambda);
        sync_stream(ctx);
    });
}

int svt_alloc_stats(int64_t* mallocs, int64_t* frees, double* ms) {
    return guard([&] {
        if (mallocs) *mallocs = alloc_stats().count;
        if (frees) *frees = alloc_stats().frees;
        if (ms) *ms = alloc_stats().ms;
    });
}

int svt_dev_gemm_tn_ozaki(svt_ctx* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                          const double* B, int64_t ldb, double* C, int64_t ldc, int slices) {
    return guard([&] {
        need(ctx, "svt_dev_gemm_tn_ozaki");
        if (M < 0 || N < 0 || K < 0 || lda < M || ldb < N || ldc < N || slices < 6 || slices > 8)
            throw std::invalid_argument("dev_gemm_tn_ozaki: bad shape or slice count");
        if (M == 0 || N == 0) return;
        if (!A || !B || !C) throw std::invalid_argument("dev_gemm_tn_ozaki: null operand");
        gemm_tn_ozaki(ctx, M, N, K, 1.0, A, lda, B, ldb, 0.0, C, ldc, slices);
        sync_stream(ctx);
    });
}

int svt_sp_mult(svt_mat* S, int64_t w, const double* X, double* out) {
    return guard([&] {
        need(S, "svt_sp_mult");
        if (w < 0) throw std::invalid_argument("sp_mult: bad width");
        if (w == 0) return;
        svt_ctx* c = S->ctx;
        Engine E = engine_for(S);
        DevBuf<double> dX = upload_cm(c, X, S->n, w);
        DevBuf<double> dO(static_cast<size_t>(std::max<i64>(1, S->m_local * w)));
        sp_mult(E, w, dX.get(), w, dO.get(), w);
        download_cm(c, dO.get(), S->m_local, w, w, out);
    });
}

int svt_dev_sp_mult(svt_mat* S, int transpose, int64_t w, const double* X, int64_t ldx, double* out, int64_t ldo) {
    return guard([&] {
        need(S, "svt_dev_sp_mult");
        if (w < 0 || ldx < w || ldo < w) throw std::invalid_argument("dev_sp_mult: bad width / leading dimension");
        if (w == 0) return;
        if (!X || !out) throw std::invalid_argument("dev_sp_mult: null panel");
        Engine E = engine_for(S);
        if (transpose) {
            if (ldo != w) throw std::invalid_argument("dev_sp_mult: transposed output must be packed (ldo == w)");
            sp_mult_t(E, w, X, ldx, out);
        } else {
            sp_mult(E, w, X, ldx, out, ldo);
        }
    });
}

int svt_dev_sddmm_update(svt_mat* A, int64_t k, const double* U, int64_t ldu, const double* Vs, int64_t ldv,
                         double delta, double* y_csr, double* y_csc, double* sums4) {
    return guard([&] {
        need(A, "svt_dev_sddmm_update");
        need(y_csr, "svt_dev_sddmm_update: y_csr");
        if (k < 0 || (k > 0 && (!U || !Vs || ldu < k || ldv < k)))
            throw std::invalid_argument("dev_sddmm_update: bad factors");
        svt_ctx* c = A->ctx;
        const bool gather = y_csc != nullptr && A->csc2csr.n > 0 && A->nnz_local > 0;
        sddmm_update(c, A->plan_csr.v, A->m_local, A->col.get(), A->val.get(), y_csr, gather ? nullptr : y_csc,
                     A->csr2csc.get(), A->nnz_local, A->n, U, ldu, Vs, ldv, k, delta, 1, c->d_scalars + 40);
        if (gather) mirror_csc(c, A->nnz_local, A->csc2csr.get(), y_csr, y_csc);
        c->comm.allreduce_sum(c->d_scalars + 40, 4, c->stream);
        if (sums4) {
            SVT_CUDA(cudaMemcpyAsync(sums4, c->d_scalars + 40, sizeof(double) * 4, cudaMemcpyDeviceToHost, c->stream));
            sync_stream(c);
        }
    });
}

int svt_sp_mult_t(svt_mat* S, int64_t w, const double* X, double* out) {
    return guard([&] {
        need(S, "svt_sp_mult_t");
        if (w < 0) throw std::invalid_argument("sp_mult_t: bad width");
        if (w == 0) return;
        svt_ctx* c = S->ctx;
        Engine E = engine_for(S);
        DevBuf<double> dX = upload_cm(c, X, S->m_local, w);
        DevBuf<double> dO(static_cast<size_t>(S->n * w));
        sp_mult_t(E, w, dX.get(), w, dO.get());
        download_cm(c, dO.get(), S->n, w, w, out);
    });
}

int svt_project_low_rank(svt_mat* P, int64_t k, const double* U, const double* sigma, const double* V,
                         double* out_vals) {
    return guard([&] {
        need(P, "svt_project_low_rank");
        if (k < 0) throw std::invalid_argument("project_low_rank: bad rank");
        svt_ctx* c = P->ctx;
        DevBuf<double> dU = upload_cm(c, U, P->m_local, k);
        std::vector<double> vs(static_cast<size_t>(P->n * k));
        for (i64 j = 0; j < k; ++j)
            for (i64 i = 0; i < P->n; ++i) vs[static_cast<size_t>(i + j * P->n)] = V[i + j * P->n] * sigma[j];
        DevBuf<double> dV = upload_cm(c, vs.data(), P->n, k);
        DevBuf<double> out(static_cast<size_t>(std::max<i64>(1, P->nnz_local)));
        sddmm_update(c, P->plan_csr.v, P->m_local, P->col.get(), P->val.get(), out.get(), nullptr, nullptr,
                     P->nnz_local, P->n, dU.get(), k, dV.get(), k, k, 0.0, 2, c->d_scalars + 40);
        SVT_CUDA(cudaMemcpyAsync(out_vals, out.get(), sizeof(double) * P->nnz_local, cudaMemcpyDeviceToHost, c->stream));
        sync_stream(c);
    });
}

int svt_sp_axpy(svt_mat* Y, double alpha, const double* d_vals, double* out_vals) {
    return guard([&] {
        need(Y, "svt_sp_axpy");
        svt_ctx* c = Y->ctx;
        const i64 nnz = Y->nnz_local;
        if (nnz == 0) return;
        DevBuf<double> d(static_cast<size_t>(nnz)), o(static_cast<size_t>(nnz));
        SVT_CUDA(cudaMemcpyAsync(d.get(), d_vals, sizeof(double) * nnz, cudaMemcpyHostToDevice, c->stream));
        axpy_values(c, nnz, Y->val.get(), alpha, d.get(), o.get());
        SVT_CUDA(cudaMemcpyAsync(out_vals, o.get(), sizeof(double) * nnz, cudaMemcpyDeviceToHost, c->stream));
        sync_stream(c);
    });
}

int svt_sp_frob_norm_sq(svt_mat* S, double* out) {
    return guard([&] {
        need(S, "svt_sp_frob_norm_sq");
        need(out, "svt_sp_frob_norm_sq");
        Engine E = engine_for(S);
        *out = frob_sq(E);
    });
}

int svt_spectral_norm_est(svt_mat* S, int iters, uint64_t seed, double* out) {
    return guard([&] {
        need(S, "svt_spectral_norm_est");
        need(out, "svt_spectral_norm_est");
        Engine E = engine_for(S);
        *out = spectral_norm_est(E, iters, seed);
    });
}

int svt_kickstart(svt_mat* A, double tau, double delta, uint64_t seed, double* out_vals) {
    return guard([&] {
        need(A, "svt_kickstart");
        svt_ctx* c = A->ctx;
        const i64 nnz = std::max<i64>(1, A->nnz_local);
        DevBuf<double> y(static_cast<size_t>(nnz)), yc(static_cast<size_t>(nnz));
        kickstart_dev(c, A, tau, delta, seed, y.get(), yc.get());
        if (A->nnz_local > 0)
            SVT_CUDA(cudaMemcpyAsync(out_vals, y.get(), sizeof(double) * A->nnz_local, cudaMemcpyDeviceToHost,
                                     c->stream));
        sync_stream(c);
    });
}

// ---- engines ---------------------------------------------------------------
static int wrap_factors(svt_factors** out, DevFactors&& f, i64 rank, bool sat, int rounds) {
    auto h = std::make_unique<svt_factors>();
    h->f = std::move(f);
    h->rank = rank;
    h->saturated = sat ? 1 : 0;
    h->rounds = rounds;
    *out = h.release();
    return 0;
}

int svt_rsvd(svt_mat* Y, int64_t k, const svt_sketch_params* p, svt_factors** out) {
    return guard([&] {
        need(Y, "svt_rsvd");
        need(p, "svt_rsvd");
        need(out, "svt_rsvd");
        Engine E = engine_for(Y);
        DevFactors f = rsvd(E, k, *p);
        wrap_factors(out, std::move(f), k, false, 0);
    });
}

int svt_r3svd(svt_mat* Y, const svt_sketch_params* p, svt_factors** out) {
    return guard([&] {
        need(Y, "svt_r3svd");
        need(p, "svt_r3svd");
        need(out, "svt_r3svd");
        Engine E = engine_for(Y);
        SketchOut so = r3svd(E, *p, FinalizeMode::Full, 0.0);
        wrap_factors(out, std::move(so.f), so.rank, so.saturated, so.rounds);
    });
}

int svt_r4svd(svt_mat* Y, int64_t s, const double* U_prev, int64_t ldu, const svt_sketch_params* p,
              svt_factors** out) {
    return guard([&] {
        need(Y, "svt_r4svd");
        need(p, "svt_r4svd");
        need(out, "svt_r4svd");
        if (s < 0) throw std::invalid_argument("r4svd: negative basis width");
        if (s > 0) {
            need(U_prev, "svt_r4svd");
            if (ldu < Y->m_local) throw std::invalid_argument("r4svd: U_prev row count does not match Y");
        }
        svt_ctx* c = Y->ctx;
        Engine E = engine_for(Y);
        // column-major host (ldu) -> row-major device
        DevBuf<double> dU(static_cast<size_t>(std::max<i64>(1, Y->m_local * s)));
        if (s > 0) {
            std::vector<double> rm(static_cast<size_t>(Y->m_local * s));
            for (i64 i = 0; i < Y->m_local; ++i)
                for (i64 j = 0; j < s; ++j) rm[static_cast<size_t>(i * s + j)] = U_prev[i + j * ldu];
            SVT_CUDA(cudaMemcpyAsync(dU.get(), rm.data(), sizeof(double) * rm.size(), cudaMemcpyHostToDevice,
                                     c->stream));
            sync_stream(c);
        }
        SketchOut so = r4svd(E, dU.get(), s, s, *p, FinalizeMode::Full, 0.0);
        wrap_factors(out, std::move(so.f), so.rank, so.saturated, so.rounds);
    });
}

int svt_factors_info(svt_factors* f, int64_t* m_local, int64_t* n, int64_t* rank, int* saturated, int* rounds) {
    return guard([&] {
        need(f, "svt_factors_info");
        if (m_local) *m_local = f->f.m_local;
        if (n) *n = f->f.n;
        if (rank) *rank = f->f.k;
        if (saturated) *saturated = f->saturated;
        if (rounds) *rounds = f->rounds;
    });
}

int svt_factors_copy(svt_factors* f, double* U, double* sigma, double* V) {
    return guard([&] {
        need(f, "svt_factors_copy");
        svt_ctx* c = nullptr;
        (void)c;
        const i64 k = f->f.k;
        if (k == 0) return;
        // the factors' context is the one that produced them; copy via the default stream
        std::vector<double> hu(static_cast<size_t>(f->f.m_local * k)), hv(static_cast<size_t>(f->f.n * k));
        SVT_CUDA(cudaMemcpy(hu.data(), f->f.U.get(), sizeof(double) * hu.size(), cudaMemcpyDeviceToHost));
        SVT_CUDA(cudaMemcpy(hv.data(), f->f.V.get(), sizeof(double) * hv.size(), cudaMemcpyDeviceToHost));
        for (i64 i = 0; i < f->f.m_local; ++i)
            for (i64 j = 0; j < k; ++j) U[i + j * f->f.m_local] = hu[static_cast<size_t>(i * k + j)];
        for (i64 i = 0; i < f->f.n; ++i)
            for (i64 j = 0; j < k; ++j) V[i + j * f->f.n] = hv[static_cast<size_t>(i * k + j)];
        std::memcpy(sigma, f->f.sigma.data(), sizeof(double) * k);
    });
}

int svt_factors_free(svt_factors* f) {
    return guard([&] { delete f; });
}

// ---- solver ----------------------------------------------------------------
int svt_default_config(svt_mat* A, svt_config* out) {  // solver.hpp:95-106
    return guard([&] {
        need(A, "svt_default_config");
        need(out, "svt_default_config");
        Engine E = engine_for(A);
        svt_config c{};
        c.maxit = 500;
        c.np = 1;
        c.eps_stop = 1e-3;
        c.eps_threshold0 = 0.5;
        c.seed = 1;
        c.tau = std::sqrt(frob_sq(E));
        c.delta = std::sqrt(static_cast<double>(A->m) * static_cast<double>(A->n) / static_cast<double>(A->nnz_global));
        const i64 min_dim = std::min(A->m, A->n);
        c.t0 = std::max<i64>(1, static_cast<i64>(0.05 * static_cast<double>(min_dim)));
        c.dt = 10;
        c.beta = 0.95;
        *out = c;
    });
}

int svt_solver_create(svt_mat* A, const svt_config* cfg, svt_stop stop, svt_backend backend, svt_mat* test,
                      svt_solver** out) {
    return guard([&] {
        need(A, "svt_solver_create");
        need(cfg, "svt_solver_create");
        need(out, "svt_solver_create");
        *out = solver_create(A, *cfg, stop, backend, test);
    });
}

int svt_solver_step(svt_solver* s, svt_observer_fn obs, void* user, svt_record* rec, int* done) {
    return guard([&] {
        need(s, "svt_solver_step");
        solver_step(s, obs, user, rec, done);
    });
}

int svt_solver_result(svt_solver* s, svt_result** out) {
    return guard([&] {
        need(s, "svt_solver_result");
        need(out, "svt_solver_result");
        *out = solver_result(s);
    });
}

int svt_solver_checkpoint(svt_solver* s, svt_solver_state* st, double* y_vals, double* u_prev, double* best_U,
                          double* best_sigma, double* best_V) {
    return guard([&] {
        need(s, "svt_solver_checkpoint");
        need(st, "svt_solver_checkpoint");
        solver_checkpoint(s, st, y_vals, u_prev, best_U, best_sigma, best_V);
    });
}

int svt_solver_resume(svt_mat* A, const svt_config* cfg, svt_stop stop, svt_backend backend, svt_mat* test,
                      const svt_solver_state* st, const double* y_vals, const double* u_prev, const double* best_U,
                      const double* best_sigma, const double* best_V, svt_solver** out) {
    return guard([&] {
        need(A, "svt_solver_resume");
        need(cfg, "svt_solver_resume");
        need(st, "svt_solver_resume");
        need(out, "svt_solver_resume");
        *out = solver_resume(A, *cfg, stop, backend, test, *st, y_vals, u_prev, best_U, best_sigma, best_V);
    });
}

int svt_solver_free(svt_solver* s) {
    return guard([&] { delete s; });
}

int svt_run(svt_mat* A, const svt_config* cfg, svt_stop stop, svt_backend backend, svt_mat* test,
            svt_observer_fn obs, void* user, svt_result** out) {
    return guard([&] {
        need(A, "svt_run");
        need(cfg, "svt_run");
        need(out, "svt_run");
        std::unique_ptr<svt_solver> s(solver_create(A, *cfg, stop, backend, test));
        int done = 0;
        while (!done) solver_step(s.get(), obs, user, nullptr, &done);
        *out = solver_result(s.get());
    });
}

int svt_result_info(svt_result* r, int64_t* n_records, int64_t* m_local, int64_t* n, int64_t* k, int* converged) {
    return guard([&] {
        need(r, "svt_result_info");
        if (n_records) *n_records = static_cast<int64_t>(r->trace.size());
        if (m_local) *m_local = r->m_local;
        if (n) *n = r->n;
        if (k) *k = r->k;
        if (converged) *converged = r->converged;
    });
}

int svt_result_trace(svt_result* r, svt_record* out) {
    return guard([&] {
        need(r, "svt_result_trace");
        if (!r->trace.empty()) std::memcpy(out, r->trace.data(), sizeof(svt_record) * r->trace.size());
    });
}

int svt_result_factors(svt_result* r, double* U, double* sigma, double* V) {
    return guard([&] {
        need(r, "svt_result_factors");
        if (r->k == 0) return;
        std::memcpy(U, r->U.data(), sizeof(double) * r->U.size());
        std::memcpy(sigma, r->sigma.data(), sizeof(double) * r->sigma.size());
        std::memcpy(V, r->V.data(), sizeof(double) * r->V.size());
    });
}

int svt_result_free(svt_result* r) {
    return guard([&] { delete r; });
}

int svt_synth_config(int config, uint64_t seed, int64_t* m, int64_t* n, int64_t* nnz_train, int64_t* nnz_test,
                     int64_t* train_rows, int64_t* train_cols, double* train_vals, int64_t* test_rows,
                     int64_t* test_cols, double* test_vals) {
    return guard([&] {
        synth_config(config, seed, m, n, nnz_train, nnz_test, train_rows, train_cols, train_vals, test_rows,
                     test_cols, test_vals);
    });
}

int svt_synth_config_csr(int config, uint64_t seed, int64_t* m, int64_t* n, int64_t* nnz, int64_t* rowptr,
                         int64_t* col, double* val) {
    return guard([&] { synth_config_csr(config, seed, m, n, nnz, rowptr, col, val); });
}

// ---- the reference's experiment generators (synth.hpp; the CLI's inputs) ----
uint64_t svt_derive_seed(uint64_t seed, uint64_t stream) { return derive_seed_u(seed, stream); }  // dense.hpp:44

int svt_make_low_rank(int64_t m, int64_t n, int64_t rank, uint64_t seed, double* out) {  // synth.hpp:21-28
    return guard([&] {
        need(out, "svt_make_low_rank");
        const std::vector<double> A = make_low_rank_cm(m, n, rank, seed);
        std::memcpy(out, A.data(), sizeof(double) * A.size());
    });
}

int svt_sample_dense(int64_t m, int64_t n, const double* A, double fraction, uint64_t seed, svt_triplets** out) {
    return guard([&] {  // synth.hpp:64-84
        need(A, "svt_sample_dense");
        need(out, "svt_sample_dense");
        if (m < 1 || n < 1) throw std::invalid_argument("sample_dense: bad dimensions");
        auto T = std::make_unique<svt_triplets>();
        T->t.m = m;
        T->t.n = n;
        sample_dense(m, n, A, fraction, seed, T->t.r, T->t.c, T->t.v);
        *out = T.release();
    });
}

int svt_synthetic_image(int64_t size, int64_t rank, uint64_t seed, uint8_t* pixels) {  // synth.hpp:89-114
    return guard([&] {
        need(pixels, "svt_synthetic_image");
        const std::vector<unsigned char> px = synthetic_image(size, rank, seed);
        std::memcpy(pixels, px.data(), px.size());
    });
}

int svt_synthetic_ratings(int64_t users, int64_t items, int64_t rank, double fill, double noise, uint64_t seed,
                          svt_triplets** out) {  // synth.hpp:119-160
    return guard([&] {
        need(out, "svt_synthetic_ratings");
        auto T = std::make_unique<svt_triplets>();
        synthetic_ratings(users, items, rank, fill, noise, seed, T->t.r, T->t.c, T->t.v);
        T->t.m = users;
        T->t.n = items;
        T->t.user_ids.resize(static_cast<size_t>(users));
        T->t.item_ids.resize(static_cast<size_t>(items));
        for (int64_t u = 0; u < users; ++u) T->t.user_ids[static_cast<size_t>(u)] = u;
        for (int64_t i = 0; i < items; ++i) T->t.item_ids[static_cast<size_t>(i)] = i;
        T->t.provenance = "synthetic";
        *out = T.release();
    });
}

// solver.hpp:95-106 on the host: tau from the serial sum in CSR order (the
// reference's summation order), so a front end can resolve its defaults and
// reject bad input before a device context exists
int svt_default_config_host(int64_t m, int64_t n, int64_t nnz, const double* csr_vals, svt_config* out) {
    return guard([&] {
        need(out, "svt_default_config_host");
        if (m < 1 || n < 1 || nnz < 1 || !csr_vals) throw std::invalid_argument("default_config: empty sample set");
        svt_config c{};
        c.maxit = 500;
        c.np = 1;
        c.eps_stop = 1e-3;
        c.eps_threshold0 = 0.5;
        c.seed = 1;
        double ss = 0.0;
        for (int64_t k = 0; k < nnz; ++k) ss += csr_vals[k] * csr_vals[k];
        c.tau = std::sqrt(ss);
        c.delta = std::sqrt(static_cast<double>(m) * static_cast<double>(n) / static_cast<double>(nnz));
        c.t0 = std::max<i64>(1, static_cast<i64>(0.05 * static_cast<double>(std::min(m, n))));
        c.dt = 10;
        c.beta = 0.95;
        *out = c;
    });
}

}  // extern "C"
