// Context runtime: launch accounting / CUDA-event instrumentation and the
// NCCL communicator (resolved with dlopen so single-GPU use never needs it).
#include <nvtx3/nvToolsExt.h>
#include <dlfcn.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.hpp"

namespace svtb {

LaunchScope::LaunchScope(svt_ctx* c, int k, double bytes, double flops, cudaStream_t stream, const char* f, int l)
    : ctx(c), cls(k), st(stream ? stream : c->stream), file(f), line(l) {
    ctx->launch_count++;
    if (k < 0) return;  // a kernel inside an operation timed as a whole by an enclosing scope
    if (ctx->gap_open) {
        auto& g = ctx->gap_stats[ctx->gap_site];
        g.first++;
        g.second += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ctx->gap_t0).count();
        ctx->gap_open = false;
    }
    KStats& s = ctx->stats[k];
    s.launches++;
    s.bytes += bytes;
    s.flops += flops;
    if (ctx->profiling) {
        if (ctx->event_pool.size() < 2) {
            for (int i = 0; i < 64; ++i) {
                cudaEvent_t e;
                SVT_CUDA(cudaEventCreate(&e));
                ctx->event_pool.push_back(e);
            }
        }
        a = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        b = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        SVT_CUDA(cudaEventRecord(a, st));
    }
}

LaunchScope::~LaunchScope() noexcept(false) {
    cudaError_t e = cudaGetLastError();
    if (a != nullptr) {
        cudaEventRecord(b, st);
        ctx->pending.push_back({a, b, cls, st != ctx->stream});
        if (ctx->pending.size() > 4096) flush_stats(ctx);
    }
    if (e != cudaSuccess && std::uncaught_exceptions() == 0)
        throw cuda_error(std::string("kernel launch failed: ") + cudaGetErrorString(e) + " (launched at " + file +
                         ":" + std::to_string(line) + ")");
    // SVTB_SYNC_CHECK=1 (debug): wait for every launch, so a device fault is
    // reported with the launch site that caused it
    static const bool sync_check = std::getenv("SVTB_SYNC_CHECK") != nullptr;
    if (sync_check && std::uncaught_exceptions() == 0) {
        const cudaError_t se = cudaStreamSynchronize(st);
        if (se != cudaSuccess)
            throw cuda_error(std::string("kernel failed: ") + cudaGetErrorString(se) + " (launched at " + file + ":" +
                             std::to_string(line) + ", class " + std::to_string(cls) + ")");
    }
}

// Host wait for the context stream.  SVTB_SYNC_SPIN=1 polls cudaStreamQuery
// instead of blocking in cudaStreamSynchronize (whose wake-up latency is a
// device-idle gap on the critical path of the round-batch loop: one such
// wait per batch).
static void wait_stream(cudaStream_t s) {
    static const bool spin = [] {
        const char* e = std::getenv("SVTB_SYNC_SPIN");
        return e != nullptr && e[0] == '1';
    }();
    if (!spin) {
        SVT_CUDA(cudaStreamSynchronize(s));
        return;
    }
    for (;;) {
        const cudaError_t e = cudaStreamQuery(s);
        if (e == cudaSuccess) return;
        if (e != cudaErrorNotReady) SVT_CUDA(e);
    }
}

void sync_stream(svt_ctx* c, int site, const char* file) {
    c->host_syncs++;
    if (!c->profiling) {
        wait_stream(c->stream);
        return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    wait_stream(c->stream);
    const auto t1 = std::chrono::steady_clock::now();
    c->host_sync_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
    if (c->gap_debug) {
        c->gap_open = true;
        c->gap_site = site + (file && std::strstr(file, "engine") ? 100000 : file && std::strstr(file, "solver") ? 200000 : 300000);
        c->gap_t0 = t1;
    }
}

void print_gap_stats(svt_ctx* c) {
    std::fprintf(stderr, "[alloc] %lld mallocs, %lld frees, %.1f MB, %.3f ms\n", alloc_stats().count,
                 alloc_stats().frees, alloc_stats().bytes / 1e6, alloc_stats().ms);
    for (auto& kv : c->gap_stats)
        std::fprintf(stderr, "[gaps] site %d: %lld gaps, %.3f ms total, %.1f us mean\n", kv.first, kv.second.first,
                     kv.second.second, 1000.0 * kv.second.second / std::max(1LL, kv.second.first));
    c->gap_stats.clear();
}

void flush_stats(svt_ctx* ctx) {
    if (ctx->pending.empty()) return;
    SVT_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->side) SVT_CUDA(cudaStreamSynchronize(ctx->side));
    for (auto& p : ctx->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) ctx->stats[p.cls].total_ms += ms;
        ctx->event_pool.push_back(p.a);
        ctx->event_pool.push_back(p.b);
    }
    ctx->pending.clear();
}

// ---------------------------------------------------------------------------
// NCCL through dlopen
// ---------------------------------------------------------------------------
namespace {

typedef int ncclResult_t_;
typedef void* ncclComm_t_;
struct NcclApi {
    void* h = nullptr;
    ncclResult_t_ (*GetUniqueId)(void*) = nullptr;
    ncclResult_t_ (*CommInitRank)(ncclComm_t_*, int, /*ncclUniqueId by value*/ ...) = nullptr;
    ncclResult_t_ (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t_, cudaStream_t) = nullptr;
    ncclResult_t_ (*CommDestroy)(ncclComm_t_) = nullptr;
    const char* (*GetErrorString)(ncclResult_t_) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (api.h == nullptr) {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (api.h == nullptr) throw nccl_error("libnccl.so.2 not loadable (multi-GPU needs NCCL)");
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.h, "ncclGetUniqueId"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(api.h, "ncclAllReduce"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.h, "ncclCommDestroy"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.h, "ncclGetErrorString"));
        if (!api.GetUniqueId || !api.AllReduce || !api.CommDestroy)
            throw nccl_error("libnccl.so.2 is missing required symbols");
    }
    return api;
}

struct UniqueId {
    char internal[128];
};

constexpr int kNcclFloat64 = 8;  // ncclDouble
constexpr int kNcclSum = 0;

void check(ncclResult_t_ r, const char* what) {
    if (r != 0) {
        const char* msg = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
        throw nccl_error(std::string(what) + ": " + msg);
    }
}

}  // namespace

void nccl_unique_id(void* out128) { check(nccl().GetUniqueId(out128), "ncclGetUniqueId"); }

void nccl_init(Comm& c, int rank, int world, const void* id128) {
    c.rank = rank;
    c.world = world;
    if (world <= 1 && id128 == nullptr) return;  // world 1 with an id: a one-rank communicator
    auto fn = reinterpret_cast<ncclResult_t_ (*)(ncclComm_t_*, int, UniqueId, int)>(
        dlsym(nccl().h, "ncclCommInitRank"));
    if (!fn) throw nccl_error("ncclCommInitRank missing");
    UniqueId id;
    std::memcpy(id.internal, id128, 128);
    ncclComm_t_ comm = nullptr;
    check(fn(&comm, world, id, rank), "ncclCommInitRank");
    c.handle = comm;
    // a second communicator over the same ranks for the side stream's
    // collectives (speculative batches run Y^T X all-reduces concurrently
    // with the main stream's; one communicator must not be used from two
    // streams at once).  ncclCommSplit(comm, color 0, key rank, &out, NULL).
    auto split = reinterpret_cast<ncclResult_t_ (*)(ncclComm_t_, int, int, ncclComm_t_*, void*)>(
        dlsym(nccl().h, "ncclCommSplit"));
    if (split != nullptr) {
        ncclComm_t_ side = nullptr;
        if (split(comm, 0, rank, &side, nullptr) == 0) c.handle_side = side;
    }
}

void Comm::allreduce_sum(double* buf, size_t count, cudaStream_t s, bool side) {
    if (!dist() || count == 0) return;
    calls++;
    doubles += static_cast<double>(count);
    if (host_fn != nullptr) {
        if (count > h_cap) {
            if (h_buf) cudaFreeHost(h_buf);
            h_buf = nullptr;
            h_cap = std::max(count, 2 * h_cap);
            SVT_CUDA(cudaMallocHost(&h_buf, h_cap * sizeof(double)));
        }
        SVT_CUDA(cudaMemcpyAsync(h_buf, buf, count * sizeof(double), cudaMemcpyDeviceToHost, s));
        SVT_CUDA(cudaStreamSynchronize(s));
        if (host_fn(h_buf, static_cast<std::int64_t>(count), host_user) != 0)
            throw nccl_error("host all-reduce callback failed");
        SVT_CUDA(cudaMemcpyAsync(buf, h_buf, count * sizeof(double), cudaMemcpyHostToDevice, s));
        SVT_CUDA(cudaStreamSynchronize(s));  // the staging buffer is reused by the next call
        return;
    }
    if (side && handle_side == nullptr) throw nccl_error("side-stream all-reduce without a side communicator");
    check(svtb::nccl().AllReduce(buf, buf, count, kNcclFloat64, kNcclSum, side ? handle_side : handle, s),
          "ncclAllReduce");
}

void Comm::destroy() {
    if (h_buf != nullptr) {
        cudaFreeHost(h_buf);
        h_buf = nullptr;
        h_cap = 0;
    }
    if (handle_side != nullptr) {
        svtb::nccl().CommDestroy(handle_side);
        handle_side = nullptr;
    }
    if (handle != nullptr) {
        svtb::nccl().CommDestroy(handle);
        handle = nullptr;
    }
}

NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }

}  // namespace svtb
