// Exercises the reference-side binding (integration/svt/b200.hpp) as a C++
// caller of libsvt_b200 would: the reference's types (here the stand-ins of
// integration/stub), a resident device matrix, r3svd / r4svd / rsvd, the SVT
// loop with an IterationObserver, set_values, and the exception mapping.
// Writes the input triplets and every result to argv[1] (one "key values..."
// line each) for tests/test_gpu_cpp_shim.py, which checks them against the
// CPU oracle.  Exit code 0 when the run's own invariants hold.
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <fstream>
#include <iostream>
#include <vector>

#include "svt/svt.hpp"
#include "svt/b200.hpp"

using namespace svt;

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "usage: test_shim <out.txt>\n";
        return 2;
    }
    std::ofstream out(argv[1]);
    out.precision(17);
    // a 150 x 120 rank-4 matrix, 35 % of the cells observed (own LCG)
    const Index m = 150, n = 120, k = 4;
    std::uint64_t s = 88172645463325252ULL;
    auto next = [&]() {
        s = s * 6364136223846793005ULL + 1442695040888963407ULL;
        return static_cast<double>(s >> 11) * 0x1.0p-53;
    };
    std::vector<double> L(m * k), R(n * k);
    for (double& v : L) v = next() - 0.5;
    for (double& v : R) v = next() - 0.5;
    std::vector<Triplet> t;
    for (Index i = 0; i < m; ++i)
        for (Index j = 0; j < n; ++j)
            if (next() < 0.35) {
                double v = 0.0;
                for (Index q = 0; q < k; ++q) v += L[i * k + q] * R[j * k + q];
                t.push_back({i, j, v});
            }
    for (const Triplet& e : t) out << "triplet " << e.row << " " << e.col << " " << e.value << "\n";
    const SampledMatrix A(m, n, t);
    int bad = 0;
    try {
        b200::Device dev(0);
        b200::DeviceMatrix Ad(dev, A);
        // the SVT loop with an observer (solver.hpp:215-328, :311-319)
        SvtConfig cfg = b200::default_config(Ad);
        cfg.maxit = 6;
        cfg.seed = 5;
        out << "config " << cfg.tau << " " << cfg.delta << " " << cfg.t0 << "\n";
        int seen = 0;
        const SvtResult r = b200::svt_run(dev, A, cfg, StopRule::none(), [&](const IterationRecord& rec,
                                                                              const LowRankFactors& X) {
            ++seen;
            out << "observed " << rec.iter << " " << X.rank() << "\n";
            return true;
        });
        for (const IterationRecord& x : r.trace)
            out << "record " << x.iter << " " << x.rank << " " << x.residual << " " << x.eps_threshold << " "
                << x.train_mae << "\n";
        if (seen != 6 || static_cast<int>(r.trace.size()) != 6) bad |= 1;
        // the sketch engines on the resident matrix
        SketchParams p;
        p.t = 5;
        p.dt = 10;
        p.eps_threshold = 0.05;
        p.seed = 11;
        const SketchResult r3 = b200::r3svd(Ad, p);
        out << "r3svd " << r3.rank << " " << r3.extension_rounds << " " << r3.saturated;
        for (Index q = 0; q < std::min<Index>(r3.factors.rank(), 6); ++q) out << " " << r3.factors.sigma(q);
        out << "\n";
        DenseBlock U3(m, 3);
        for (Index j = 0; j < 3; ++j)
            for (Index i = 0; i < m; ++i) U3(i, j) = r3.factors.U(i, j);
        const SketchResult r4 = b200::r4svd(Ad, U3, p);
        out << "r4svd " << r4.rank << " " << r4.extension_rounds << " " << r4.saturated;
        for (Index q = 0; q < std::min<Index>(r4.factors.rank(), 6); ++q) out << " " << r4.factors.sigma(q);
        out << "\n";
        const SketchResult rf = b200::rsvd(Ad, 4, p);
        out << "rsvd " << rf.rank;
        for (Index q = 0; q < rf.factors.rank(); ++q) out << " " << rf.factors.sigma(q);
        out << "\n";
        // U of r3svd orthonormal
        double orth = 0.0;
        for (Index a = 0; a < r3.factors.rank(); ++a)
            for (Index b = 0; b < r3.factors.rank(); ++b) {
                double d = 0.0;
                for (Index i = 0; i < m; ++i) d += r3.factors.U(i, a) * r3.factors.U(i, b);
                orth = std::max(orth, std::abs(d - (a == b ? 1.0 : 0.0)));
            }
        out << "orthonormality " << orth << "\n";
        if (orth > 1e-10) bad |= 2;
        // with_values on the resident pattern: 2 Y has twice the singular values
        std::vector<double> v2(A.values());
        for (double& v : v2) v *= 2.0;
        Ad.set_values(v2);
        const SketchResult r3b = b200::r3svd(Ad, p);
        const double ratio = r3b.factors.sigma(0) / r3.factors.sigma(0);
        out << "scaled " << ratio << "\n";
        if (std::abs(ratio - 2.0) > 1e-10) bad |= 4;
        // exception mapping: eps_threshold outside (0, 1) -> std::invalid_argument
        SketchParams badp = p;
        badp.eps_threshold = 1.5;
        try {
            b200::r3svd(Ad, badp);
            bad |= 8;
        } catch (const std::invalid_argument& e) {
            out << "invalid_argument " << e.what() << "\n";
        }
    } catch (const std::exception& e) {
        std::cerr << "exception: " << e.what() << "\n";
        return 3;
    }
    out << "status " << bad << "\n";
    std::cout << (bad ? "FAILED " : "OK ") << bad << "\n";
    return bad ? 1 : 0;
}
