// Reference-side binding of libsvt_b200 (what a maintainer of the reference
// adds next to proj/include/svt/): the reference's public R3SVD / R4SVD /
// SVT entry points on the B200 path through the C ABI in include/svt_b200.h.
//
//   #include "svt/svt.hpp"     // the reference (or integration/stub here)
//   #include "svt/b200.hpp"    // this file
//
// Compiled and run against the stand-in types of integration/stub by
// integration/test_shim.cpp (tests/test_capi_cpu.py builds it, the GPU suite
// runs it): the reference itself needs Eigen3, absent from this image.
//
// Errors map back to the reference's exception types (SVT_EINVAL ->
// std::invalid_argument, SVT_EDOMAIN -> std::domain_error, else
// std::runtime_error).  Dense host blocks are column-major (Eigen's layout)
// on both sides, so data() pointers pass straight through.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "svt_b200.h"

namespace svt::b200 {

inline void check(int rc) {
    if (rc == SVT_OK) return;
    const std::string msg = svt_last_error();
    if (rc == SVT_EINVAL) throw std::invalid_argument(msg);
    if (rc == SVT_EDOMAIN) throw std::domain_error(msg);
    throw std::runtime_error(msg);
}

// One device (svt_ctx: stream, workspaces, instrumentation).
class Device {
public:
    explicit Device(int device = 0) { check(svt_ctx_create(device, &ctx_)); }
    ~Device() { svt_ctx_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    svt_ctx* get() const { return ctx_; }

private:
    svt_ctx* ctx_ = nullptr;
};

// A SampledMatrix resident in HBM (CSR + CSC view + segment plans).  The
// pattern is uploaded once; the iterate's values change every SVT iteration
// and are refreshed with set_values (8 bytes per stored entry), so the
// per-iteration r4svd call of svt_run_backend (solver.hpp:251-276) does not
// re-upload the pattern.
class DeviceMatrix {
public:
    DeviceMatrix(Device& dev, const SampledMatrix& S) {
        static_assert(sizeof(Index) == sizeof(int64_t), "Index must be 64-bit");
        check(svt_matrix_upload(dev.get(), S.rows(), S.cols(), 0, S.rows(),
                                reinterpret_cast<const int64_t*>(S.row_offsets().data()),
                                reinterpret_cast<const int64_t*>(S.col_index().data()), S.values().data(), &h_));
    }
    ~DeviceMatrix() { svt_matrix_free(h_); }
    DeviceMatrix(const DeviceMatrix&) = delete;
    DeviceMatrix& operator=(const DeviceMatrix&) = delete;
    // SampledMatrix::with_values (sampled.hpp:79-91) on the resident pattern
    void set_values(const std::vector<double>& v) { check(svt_matrix_set_values(h_, v.data())); }
    svt_mat* get() const { return h_; }

private:
    svt_mat* h_ = nullptr;
};

inline svt_sketch_params to_c(const SketchParams& p) {
    return svt_sketch_params{p.t, p.dt, p.np, 0, p.eps_threshold, p.seed, p.p};
}

inline SketchResult take(svt_factors* f) {
    int64_t ml = 0, n = 0, r = 0;
    int sat = 0, rounds = 0;
    check(svt_factors_info(f, &ml, &n, &r, &sat, &rounds));
    SketchResult out;
    out.factors.U.resize(ml, r);
    out.factors.sigma.resize(r);
    out.factors.V.resize(n, r);
    const int rc = svt_factors_copy(f, out.factors.U.data(), out.factors.sigma.data(), out.factors.V.data());
    svt_factors_free(f);
    check(rc);
    out.rank = r;
    out.saturated = sat != 0;
    out.extension_rounds = rounds;
    return out;
}

// sketch.hpp:188-201
inline SketchResult r3svd(DeviceMatrix& Y, const SketchParams& p) {
    const svt_sketch_params sp = to_c(p);
    svt_factors* f = nullptr;
    check(svt_r3svd(Y.get(), &sp, &f));
    return take(f);
}

// sketch.hpp:207-250
inline SketchResult r4svd(DeviceMatrix& Y, const DenseBlock& U_prev, const SketchParams& p) {
    const svt_sketch_params sp = to_c(p);
    svt_factors* f = nullptr;
    check(svt_r4svd(Y.get(), U_prev.cols(), U_prev.data(), U_prev.rows() > 0 ? U_prev.rows() : 1, &sp, &f));
    return take(f);
}

// sketch.hpp:165-182
inline SketchResult rsvd(DeviceMatrix& Y, Index k, const SketchParams& p) {
    const svt_sketch_params sp = to_c(p);
    svt_factors* f = nullptr;
    check(svt_rsvd(Y.get(), k, &sp, &f));
    return take(f);
}

namespace detail {
struct ObsCtx {
    const IterationObserver* obs;
};
inline int observer_thunk(const svt_record* rec, int64_t m_local, int64_t n, int64_t k, const double* U,
                          const double* sigma, const double* V, void* user) {
    auto* o = static_cast<ObsCtx*>(user);
    IterationRecord r{rec->iter, rec->rank, rec->residual, rec->eps_threshold, rec->train_mae, rec->sketch_ms,
                      rec->total_ms};
    LowRankFactors X;
    X.U.resize(m_local, k);
    X.sigma.resize(k);
    X.V.resize(n, k);
    std::copy(U, U + m_local * k, X.U.data());
    std::copy(sigma, sigma + k, X.sigma.data());
    std::copy(V, V + n * k, X.V.data());
    try {
        return (*o->obs)(r, X) ? 1 : 0;
    } catch (...) {
        return 0;  // an observer that throws stops the run
    }
}
}  // namespace detail

// svt_run_backend (solver.hpp:215-328): the whole Bregman loop on the device;
// the observer gets the reference's IterationRecord and the shrunk factors.
inline SvtResult svt_run_backend(Device& dev, const SampledMatrix& A, const SvtConfig& c, StopRule stop,
                                 Backend backend, const IterationObserver& observer = {}) {
    DeviceMatrix a(dev, A);
    const svt_config cfg{c.tau, c.delta, c.maxit, c.np, c.dt, c.eps_stop, c.eps_threshold0, c.beta, c.t0, c.seed,
                         0.0, 0.0};
    const svt_stop st{static_cast<int32_t>(stop.kind), 0, stop.threshold};
    const svt_backend be{static_cast<int32_t>(backend.kind), 0, backend.fixed_rank};
    detail::ObsCtx oc{&observer};
    svt_result* r = nullptr;
    check(svt_run(a.get(), &cfg, st, be, nullptr, observer ? detail::observer_thunk : nullptr,
                  observer ? &oc : nullptr, &r));
    int64_t nrec = 0, ml = 0, n = 0, k = 0;
    int conv = 0;
    SvtResult out;
    try {
        check(svt_result_info(r, &nrec, &ml, &n, &k, &conv));
        std::vector<svt_record> recs(static_cast<std::size_t>(nrec));
        check(svt_result_trace(r, recs.data()));
        for (const auto& x : recs)
            out.trace.push_back({x.iter, x.rank, x.residual, x.eps_threshold, x.train_mae, x.sketch_ms, x.total_ms});
        out.factors.U.resize(ml, k);
        out.factors.sigma.resize(k);
        out.factors.V.resize(n, k);
        check(svt_result_factors(r, out.factors.U.data(), out.factors.sigma.data(), out.factors.V.data()));
    } catch (...) {
        svt_result_free(r);
        throw;
    }
    svt_result_free(r);
    out.converged = conv != 0;
    return out;
}

inline SvtResult svt_run(Device& dev, const SampledMatrix& A, const SvtConfig& c, StopRule stop,
                         const IterationObserver& observer = {}) {  // solver.hpp:333-336
    return svt_run_backend(dev, A, c, stop, Backend::r4svd(), observer);
}

// default_config (solver.hpp:95-106) computed by the library
inline SvtConfig default_config(DeviceMatrix& A) {
    svt_config c{};
    check(svt_default_config(A.get(), &c));
    SvtConfig out;
    out.tau = c.tau;
    out.delta = c.delta;
    out.maxit = c.maxit;
    out.np = c.np;
    out.dt = c.dt;
    out.eps_stop = c.eps_stop;
    out.eps_threshold0 = c.eps_threshold0;
    out.beta = c.beta;
    out.t0 = c.t0;
    out.seed = c.seed;
    return out;
}

}  // namespace svt::b200
