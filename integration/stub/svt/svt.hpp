// Minimal stand-in for the reference's public types (proj/include/svt/*.hpp),
// written for this repository so the reference-side binding
// (integration/svt/b200.hpp) can be compiled and exercised here: the
// reference needs Eigen3, which this image does not have.  Only the API
// surface the binding touches is provided, with the reference's names and
// field order (dense.hpp:14-27, sampled.hpp:25-110, sketch.hpp:20-46,
// solver.hpp:32-88); DenseBlock / RealVector mimic the subset of
// Eigen::MatrixXd / VectorXd they use (column-major storage, data(), rows(),
// cols(), resize()).  Not a restatement of any algorithm.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace svt {

using Index = std::ptrdiff_t;  // Eigen::Index

class DenseBlock {  // Eigen::MatrixXd subset (column-major)
public:
    DenseBlock() = default;
    DenseBlock(Index r, Index c) { resize(r, c); }
    void resize(Index r, Index c) {
        r_ = r;
        c_ = c;
        a_.assign(static_cast<std::size_t>(r * c), 0.0);
    }
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    double* data() { return a_.data(); }
    const double* data() const { return a_.data(); }
    double& operator()(Index i, Index j) { return a_[static_cast<std::size_t>(i + j * r_)]; }
    double operator()(Index i, Index j) const { return a_[static_cast<std::size_t>(i + j * r_)]; }

private:
    Index r_ = 0, c_ = 0;
    std::vector<double> a_;
};

class RealVector {  // Eigen::VectorXd subset
public:
    void resize(Index n) { a_.assign(static_cast<std::size_t>(n), 0.0); }
    Index size() const { return static_cast<Index>(a_.size()); }
    double* data() { return a_.data(); }
    const double* data() const { return a_.data(); }
    double& operator()(Index i) { return a_[static_cast<std::size_t>(i)]; }
    double operator()(Index i) const { return a_[static_cast<std::size_t>(i)]; }

private:
    std::vector<double> a_;
};

struct LowRankFactors {
    DenseBlock U;
    RealVector sigma;
    DenseBlock V;
    Index rank() const { return sigma.size(); }
};

struct Triplet {
    Index row;
    Index col;
    double value;
};

// Sorted row-major CSR over validated triplets (the reference's storage).
class SampledMatrix {
public:
    SampledMatrix(Index rows, Index cols, std::vector<Triplet> t) : rows_(rows), cols_(cols) {
        if (rows < 1 || cols < 1 || t.empty()) throw std::invalid_argument("SampledMatrix: bad shape");
        std::sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
            return a.row != b.row ? a.row < b.row : a.col < b.col;
        });
        off_.assign(static_cast<std::size_t>(rows) + 1, 0);
        for (const Triplet& e : t) {
            col_.push_back(e.col);
            val_.push_back(e.value);
            ++off_[static_cast<std::size_t>(e.row) + 1];
        }
        for (std::size_t i = 1; i < off_.size(); ++i) off_[i] += off_[i - 1];
    }
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index nnz() const { return static_cast<Index>(val_.size()); }
    const std::vector<Index>& row_offsets() const { return off_; }
    const std::vector<Index>& col_index() const { return col_; }
    const std::vector<double>& values() const { return val_; }

private:
    Index rows_, cols_;
    std::vector<Index> off_, col_;
    std::vector<double> val_;
};

struct SketchParams {
    Index t = 10;
    Index dt = 10;
    int np = 1;
    double eps_threshold = 0.5;
    std::uint64_t seed = 1;
    Index p = 5;
};

struct SketchResult {
    LowRankFactors factors;
    Index rank = 0;
    bool saturated = false;
    int extension_rounds = 0;
};

struct SvtConfig {
    double tau = 0.0;
    double delta = 0.0;
    int maxit = 500;
    Index dt = 10;
    int np = 1;
    double eps_stop = 1e-3;
    double eps_threshold0 = 0.5;
    double beta = 0.95;
    Index t0 = 10;
    std::uint64_t seed = 1;
};

struct IterationRecord {
    int iter = 0;
    Index rank = 0;
    double residual = 0.0;
    double eps_threshold = 0.0;
    double train_mae = 0.0;
    double sketch_ms = 0.0;
    double total_ms = 0.0;
};

struct StopRule {
    enum class Kind { TrainMae, Residual, None };
    Kind kind = Kind::TrainMae;
    double threshold = 0.1;
    static StopRule train_mae(double t) { return {Kind::TrainMae, t}; }
    static StopRule residual(double t) { return {Kind::Residual, t}; }
    static StopRule none() { return {Kind::None, 0.0}; }
};

struct Backend {
    enum class Kind { R4Svd, R3Svd, RsvdFixed, FullSvd };
    Kind kind = Kind::R4Svd;
    Index fixed_rank = 0;
    static Backend r4svd() { return {Kind::R4Svd, 0}; }
    static Backend r3svd() { return {Kind::R3Svd, 0}; }
    static Backend rsvd_fixed(Index rank) { return {Kind::RsvdFixed, rank}; }
    static Backend full_svd() { return {Kind::FullSvd, 0}; }
};

struct SvtResult {
    LowRankFactors factors;
    std::vector<IterationRecord> trace;
    bool converged = false;
};

using IterationObserver = std::function<bool(const IterationRecord&, const LowRankFactors&)>;

}  // namespace svt
