// Shared host-side plumbing of libsvt_b200: error handling, device buffers,
// the per-context stream / communicator / instrumentation state.
#pragma once

#include <algorithm>

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace svtb {

using i64 = std::int64_t;
using u64 = std::uint64_t;

// Error types map one-to-one to the reference's exceptions (sketch.hpp /
// sampled.hpp / solver.hpp throw std::invalid_argument, std::domain_error,
// std::runtime_error) plus device-side failures.
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct nccl_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct oom_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define SVT_CUDA(call)                                                                               \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess) {                                                                     \
            if (e_ == cudaErrorMemoryAllocation)                                                     \
                throw ::svtb::oom_error(std::string("CUDA OOM at " __FILE__ ":") +                  \
                                        std::to_string(__LINE__));                                   \
            throw ::svtb::cuda_error(std::string(cudaGetErrorString(e_)) + " at " __FILE__ ":" +    \
                                     std::to_string(__LINE__));                                      \
        }                                                                                            \
    } while (0)

#define SVT_CHECK_LAUNCH() SVT_CUDA(cudaGetLastError())

// Process-wide device allocation counters (host time in cudaMalloc/cudaFree).
struct AllocStats {
    long long count = 0, frees = 0;
    double bytes = 0.0, ms = 0.0;
    bool verbose = std::getenv("SVTB_DEBUG_ALLOC") != nullptr;
};
inline AllocStats& alloc_stats() {
    static AllocStats s;
    return s;
}

// RAII device allocation.
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
        o.p = nullptr;
        o.n = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count == 0) return;
        const auto t0 = std::chrono::steady_clock::now();
        SVT_CUDA(cudaMalloc(&p, count * sizeof(T)));
        alloc_stats().count++;
        alloc_stats().bytes += static_cast<double>(count * sizeof(T));
        alloc_stats().ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (alloc_stats().verbose)
            std::fprintf(stderr, "[alloc] #%lld %.3f MB (%zu x %zu B)\n", alloc_stats().count,
                         count * sizeof(T) / 1e6, count, sizeof(T));
        n = count;
    }
    // grow-only, doubling once allocated (workspaces sized by the basis rank
    // grow a little every SVT iteration, and cudaFree stalls the device, so
    // regrowth must stay logarithmic); contents are not preserved
    void ensure(size_t count) {
        if (count > n) alloc(n ? std::max(count, 2 * n) : count);
    }
    void release() {
        if (p) {
            const auto t0 = std::chrono::steady_clock::now();
            cudaFree(p);
            alloc_stats().frees++;
            alloc_stats().ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        }
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
};

// factor buffers (U, V, sigma of a few dozen kept triplets) are sized for at
// least this many columns, so the kept rank creeping up over SVT iterations
// does not regrow them (each regrow is a cudaFree: a device-wide sync)
constexpr long long kFactorCols = 32;
// ... and, within a 64 MB budget for (rows + n) x columns, for the whole
// possible kept rank (small problems keep most of their basis: config 2)
inline long long factor_cols(long long rows_plus_n, long long max_rank) {
    const long long budget = (64LL << 20) / (8 * std::max<long long>(1, rows_plus_n));
    return std::max<long long>(kFactorCols, std::min<long long>(max_rank, budget));
}

// arrival counters of the single-launch column reductions (one per 32-column block)
constexpr size_t kTickets = 4096;

// Kernel classes for instrumentation (svt_ctx_kernel_stats).
// K_SUB (-1): counted as a launch, timed by the enclosing operation's scope
enum KClass : int { K_SUB = -1, K_SPMM = 0, K_SPMMT = 1, K_SDDMM = 2, K_GEMM = 3, K_RNG = 4, K_QR = 5, K_FINAL = 6, K_OTHER = 7, K_NCLASS = 8 };

struct KStats {
    i64 launches = 0;
    double total_ms = 0.0;
    double bytes = 0.0;
    double flops = 0.0;
};

// NCCL entry points, resolved with dlopen so a single-GPU run never needs
// libnccl (comm.cpp).
// Host-staged mode (svt_ctx_create_hostcomm): every all-reduce goes D2H into
// pinned staging, through the caller's callback (which sums across ranks,
// e.g. gloo), and back H2D — the same collective sequence as NCCL mode.
typedef int (*HostAllreduceFn)(double* buf, std::int64_t count, void* user);
struct Comm {
    int rank = 0;
    int world = 1;
    void* handle = nullptr;       // ncclComm_t
    void* handle_side = nullptr;  // second communicator for the side stream (ncclCommSplit)
    HostAllreduceFn host_fn = nullptr;
    void* host_user = nullptr;
    double* h_buf = nullptr;  // pinned staging (host mode)
    size_t h_cap = 0;
    long long calls = 0;    // all-reduces issued (instrumentation)
    double doubles = 0.0;   // doubles all-reduced
    void allreduce_sum(double* buf, size_t count, cudaStream_t s, bool side = false);
    // collectives may also run on the side stream (speculative batches):
    // host-staged mode, or NCCL with a second communicator
    bool side_capable() const { return dist() && (host_fn != nullptr || handle_side != nullptr); }
    // the distributed code path (row-blocked collectives) runs whenever a
    // communicator exists, also for a one-rank NCCL world (svt_ctx_create_dist
    // with world = 1 and an id: the collective sequence on one GPU)
    bool dist() const { return world > 1 || handle != nullptr || host_fn != nullptr; }
    void destroy();
};
void nccl_unique_id(void* out128);

// Load-balanced row segmentation of a CSR / CSC view (host.cpp builds it at
// upload): every row is one or more segments of <= kSegLen entries.
constexpr long long kSegLen = 512;
struct SegPlanView {
    long long nseg = 0;
    const int* seg_row = nullptr;
    const long long* seg_beg = nullptr;
    const long long* seg_end = nullptr;
    const int* seg_slot = nullptr;  // -1: writes its row directly; else partial slot
    long long nlong = 0;            // rows split over several segments
    long long nslots = 0;
    const int* long_row = nullptr;
    const int* long_first = nullptr;
    const int* long_count = nullptr;
    // groups of consecutive segments (<= kGrpSegs segments, ~kGrpEntries
    // entries) walked by one warp with one continuous gather pipeline
    long long ngrp = 0;
    const int* grp_first = nullptr;  // ngrp + 1 segment offsets
    // 32-entry chunks of the segments, as an exclusive prefix over the
    // segments (nseg + 1 values): the chunk-balanced static partition of the
    // fused SDDMM update
    long long nchunks = 0;
    const long long* chunk_off = nullptr;
};
constexpr int kGrpSegs = 32;
// Shared-memory-tiled view of the same CSR / CSC pattern for wide panels
// (build.cu builds it, sparse.cu consumes it).  Output rows are grouped in
// blocks of kTileRows; a block's entries, ordered by gather index, are cut
// into tiles of at most kTileSlots distinct gather indices ("slots") and
// kTileEnts entries.  A tile stages its slots' panel rows in shared memory
// once and every entry reads them from there, so the L2 -> SM traffic per
// entry drops by the tile's reuse factor (entries / slots).  Inside a tile
// the entries are ordered by (row, slot) with per-row offsets, so each
// output row accumulates in a fixed order (deterministic, no atomics).
constexpr int kTileRows = 128;
constexpr int kTileSlots = 80;
constexpr int kTileEnts = 1024;
constexpr int kTileRoffStride = 136;  // kTileRows + 1 rounded up to 16 B
constexpr int kTileItemTiles = 512;   // tiles per work item (metadata staged in shared memory)
struct TileEnt {
    double v;  // value (refreshed from the CSR values at each sketch)
    int slot;  // slot of the entry's gather index in its tile
    int pad;
};
struct TilePlanView {
    long long nrows = 0, ntiles = 0, nitems = 0, nsplit = 0, nparts = 0, nnz = 0;
    const long long* tile_e = nullptr;     // ntiles + 1 entry offsets
    const long long* tile_u = nullptr;     // ntiles + 1 slot offsets into ucol
    const int* ucol = nullptr;             // gather index of every slot
    const unsigned short* roff = nullptr;  // ntiles x kTileRoffStride row offsets (tile-relative)
    TileEnt* ent = nullptr;                // entries in tile order
    const int* perm = nullptr;             // tile position -> CSR position (value source)
    const int* item_t0 = nullptr;          // work item = (block, tile range)
    const int* item_t1 = nullptr;
    const int* item_blk = nullptr;
    const int* item_part = nullptr;        // -1: writes its block directly; else partial slot
    const int* split_blk = nullptr;        // blocks spread over several items
    const int* split_first = nullptr;
    const int* split_count = nullptr;
};
void nccl_init(Comm& c, int rank, int world, const void* id128);

}  // namespace svtb

// The opaque context behind svt_ctx*.
struct svt_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // side stream: Omega prefetch for the next round batch
    // helper streams of the main / side stream: the dense corner of a split
    // SpMM runs on the tensor cores concurrently with the gather kernel of the
    // cold entries (forked and joined inside the product)
    cudaStream_t aux[2] = {nullptr, nullptr};
    cudaEvent_t aux_fork[2] = {nullptr, nullptr}, aux_join[2] = {nullptr, nullptr};
    int num_sms = 148;
    svtb::Comm comm;
    void* cusolver = nullptr;  // cusolverDnHandle_t
    // instrumentation
    bool profiling = false;
    int batching = 1;  // speculative multi-round batches in the rank-revealing loop
    bool speculate = true;  // next batch sketched on the side stream (svt_ctx_set_speculation)
    svtb::i64 launch_count = 0;
    svtb::KStats stats[svtb::K_NCLASS];
    svtb::i64 host_syncs = 0;     // stream synchronizations issued by the library
    double host_sync_ms = 0.0;    // host time spent blocked in them (profiling only)
    // debug (SVTB_DEBUG_GAPS): host latency from a sync's return to the next
    // launch, per sync site -- the device idles for that long
    bool gap_debug = false;
    bool gap_open = false;
    int gap_site = 0;
    std::chrono::steady_clock::time_point gap_t0;
    std::map<int, std::pair<long long, double>> gap_stats;
    struct Pending {
        cudaEvent_t a, b;
        int cls;
        bool side;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    // device scratch scalars (pinned host mirror for one-shot reads)
    double* h_scalars = nullptr;  // pinned, 64 doubles
    double* d_scalars = nullptr;  // device, 64 doubles
    int* d_flags = nullptr;       // device, 64 ints
    int* h_flags = nullptr;       // pinned, 64 ints
    double* h_stage = nullptr;    // pinned staging for small device -> host reads
    size_t h_stage_n = 0;
    svtb::DevBuf<double> ws_partial;   // split-K / reduction partials
    svtb::DevBuf<double> ws_ozaki;     // int8 digit slices of the Ozaki-scheme GEMM (raw bytes)
    svtb::DevBuf<int> ws_ozexp;        // their per-column exponents
    svtb::DevBuf<double> ws_ozakib;    // B-operand slices
    svtb::DevBuf<int> ws_ozexpb;
    svtb::DevBuf<double> ws_partial2;  // second partial buffer (reductions)
    svtb::DevBuf<int> ws_perm;         // eigenvector permutation (sym_eig)
    svtb::DevBuf<unsigned> d_tickets;  // self-resetting arrival counters (single-launch reductions)
    svtb::DevBuf<double> ws_spmm;      // long-row partials of the segmented SpMM
    svtb::DevBuf<unsigned> ws_counters;  // last-CTA-reduces counters (self-resetting)
    svtb::DevBuf<unsigned long long> ws_rng;  // raw mt19937_64 draws
    svtb::DevBuf<unsigned long long> ws_rng_side;  // raw draws of the side-stream prefetch
    svtb::DevBuf<unsigned long long> ws_mt;   // persistent mt state (312 words + index)
    svtb::DevBuf<double> ws_eig;              // Jacobi eigensolver workspace
    svtb::DevBuf<int> ws_info;
};

namespace svtb {

// Launch bookkeeping: counts every kernel of ours and, when profiling, brackets
// it with CUDA events on the context stream.
struct LaunchScope {
    svt_ctx* ctx;
    int cls;
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t st = nullptr;
    const char* file;
    int line;
    LaunchScope(svt_ctx* c, int k, double bytes, double flops, cudaStream_t stream = nullptr,
                const char* file = __builtin_FILE(), int line = __builtin_LINE());
    ~LaunchScope() noexcept(false);
};
// NVTX range around a host-side phase of the path (iteration, sketch batch,
// Gram-Schmidt, CholQR, finalize, update): visible in Nsight Systems /
// Compute timelines; a no-op unless a tool is attached (header-only NVTX3).
struct NvtxRange {
    explicit NvtxRange(const char* name);
    ~NvtxRange();
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
// Blocking wait for the context stream (counted; timed when profiling).
void print_gap_stats(svt_ctx* c);
void sync_stream(svt_ctx* c, int site = __builtin_LINE(), const char* file = __builtin_FILE());

void flush_stats(svt_ctx* ctx);  // resolve pending event pairs (syncs)

}  // namespace svtb
