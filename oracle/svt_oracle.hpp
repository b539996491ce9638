// TEST INFRASTRUCTURE ONLY — the CPU parity oracle.
//
// A from-scratch C++20 restatement (no Eigen) of the reference's hot-path
// headers `proj/include/svt/{dense,sampled,sketch,solver}.hpp`.  It is used
// only by tests/, by __graft_entry__.smoke() and by bench.py's cpu_baseline /
// `--impl reference` legs, always as the checker or the CPU baseline — never
// as part of the product path (paper_1704_05528_b200/ never links it).
//
// The reference itself cannot be compiled in this image (Eigen3, Catch2,
// CLI11 and nlohmann/json are absent), so parity is
// pinned by (a) the C++-standard known-answer value of std::mt19937_64,
// (b) the reference's own property / known-answer tests restated in
// tests/test_oracle_*.py, and (c) numpy/LAPACK cross-checks of the dense
// factorizations.  The Eigen boundary (HouseholderQR, BDCSVD) is restated
// with a Householder QR that follows Eigen's makeHouseholder convention and a
// one-sided Jacobi SVD (tolerance parity, as the reference tests require).
//
// Every function cites the reference file:line it restates.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>
#include <chrono>

namespace svt_oracle {

using Index = std::int64_t;

// Column-major dense block (Eigen::MatrixXd layout; dense.hpp:16).
struct Mat {
    Index rows = 0, cols = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(Index r, Index c) : rows(r), cols(c), a(static_cast<size_t>(r * c), 0.0) {}
    double& operator()(Index i, Index j) { return a[static_cast<size_t>(i + j * rows)]; }
    double operator()(Index i, Index j) const { return a[static_cast<size_t>(i + j * rows)]; }
    double* col(Index j) { return a.data() + j * rows; }
    const double* col(Index j) const { return a.data() + j * rows; }
    static Mat identity(Index r, Index c) {
        Mat m(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
        return m;
    }
    double squared_norm() const {
        double s = 0.0;
        for (double v : a) s += v * v;
        return s;
    }
    Mat left_cols(Index k) const {
        Mat m(rows, k);
        std::copy(a.begin(), a.begin() + rows * k, m.a.begin());
        return m;
    }
};

// (U, sigma, V) triple (dense.hpp:21-27).
struct LowRankFactors {
    Mat U;
    std::vector<double> sigma;
    Mat V;
    Index rank() const { return static_cast<Index>(sigma.size()); }
};

// Host parallelism (OpenMP, -fopenmp): every parallel loop below writes
// disjoint outputs and every reduction runs in a fixed order inside one
// thread, so the oracle's results are bitwise identical for any thread count.

// sum_k a[k] * b[k] in a fixed blocked order (8 interleaved partial sums,
// then combined pairwise): vectorizable without reassociation flags.
inline double dot(const double* a, const double* b, Index n) {
    double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    Index k = 0;
    for (; k + 8 <= n; k += 8)
        for (int l = 0; l < 8; ++l) p[l] += a[k + l] * b[k + l];
    for (int l = 0; k < n; ++k, ++l) p[l] += a[k] * b[k];
    return ((p[0] + p[4]) + (p[1] + p[5])) + ((p[2] + p[6]) + (p[3] + p[7]));
}

// C = A^T * B
inline Mat mul_tn(const Mat& A, const Mat& B) {
    Mat C(A.cols, B.cols);
#pragma omp parallel for collapse(2) schedule(static) if (A.rows * A.cols * B.cols > 100000)
    for (Index j = 0; j < B.cols; ++j)
        for (Index i = 0; i < A.cols; ++i) C(i, j) = dot(A.col(i), B.col(j), A.rows);
    return C;
}

// C = A * B
inline Mat mul_nn(const Mat& A, const Mat& B) {
    Mat C(A.rows, B.cols);
#pragma omp parallel for schedule(static) if (A.rows * A.cols * B.cols > 100000)
    for (Index j = 0; j < B.cols; ++j) {
        double* c = C.col(j);
        for (Index k = 0; k < A.cols; ++k) {
            const double bkj = B(k, j);
            if (bkj == 0.0) continue;
            const double* a = A.col(k);
            for (Index i = 0; i < A.rows; ++i) c[i] += a[i] * bkj;
        }
    }
    return C;
}

// X -= Q * C
inline void sub_mul(Mat& X, const Mat& Q, const Mat& C) {
    Mat P = mul_nn(Q, C);
    const Index n = static_cast<Index>(X.a.size());
#pragma omp parallel for schedule(static) if (n > 100000)
    for (Index i = 0; i < n; ++i) X.a[static_cast<size_t>(i)] -= P.a[static_cast<size_t>(i)];
}

inline Mat transpose(const Mat& A) {
    Mat T(A.cols, A.rows);
#pragma omp parallel for schedule(static) if (A.rows * A.cols > 100000)
    for (Index j = 0; j < A.cols; ++j)
        for (Index i = 0; i < A.rows; ++i) T(j, i) = A(i, j);
    return T;
}

// ---------------------------------------------------------------------------
// dense.hpp
// ---------------------------------------------------------------------------

// dense.hpp:32-37
inline std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

// dense.hpp:43-45
inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t stream) {
    return splitmix64(seed ^ splitmix64(stream));
}

// dense.hpp:52-80 — std::mt19937_64 + explicit Box-Muller, cosine first,
// sine kept as the spare.
class GaussianStream {
public:
    explicit GaussianStream(std::uint64_t seed) : state_(seed) {}
    double next() {
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        const double u1 = 1.0 - uniform01();
        const double u2 = uniform01();
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = 2.0 * 3.14159265358979323846 * u2;
        spare_ = radius * std::sin(angle);
        have_spare_ = true;
        return radius * std::cos(angle);
    }

private:
    double uniform01() { return static_cast<double>(state_() >> 11) * 0x1.0p-53; }
    std::mt19937_64 state_;
    double spare_ = 0.0;
    bool have_spare_ = false;
};

// dense.hpp:86-98 — column-major fill from one fresh stream.
inline Mat gaussian_block(Index rows, Index cols, std::uint64_t seed) {
    if (rows < 1 || cols < 1) throw std::invalid_argument("gaussian_block: dimensions must be >= 1");
    GaussianStream stream(seed);
    Mat b(rows, cols);
    for (Index j = 0; j < cols; ++j)
        for (Index i = 0; i < rows; ++i) b(i, j) = stream.next();
    return b;
}

// dense.hpp:103-110 — thin Householder QR keeping all k columns.  The
// reflector convention restates Eigen's makeHouseholder (beta = -sign(c0)
// ||x||, tau = (beta - c0) / beta, v = [1; tail / (c0 - beta)], tau = 0 when
// the tail vanishes), and Q = H_0 H_1 ... H_{k-1} [I_k; 0].
inline Mat qr_orthonormal(const Mat& X) {
    if (X.cols > X.rows) {
        throw std::invalid_argument("qr_orthonormal: need cols <= rows, got " +
                                    std::to_string(X.rows) + "x" + std::to_string(X.cols));
    }
    const Index m = X.rows, k = X.cols;
    Mat R = X;                     // overwritten with essential parts below the diagonal
    std::vector<double> tau(static_cast<size_t>(k), 0.0);
    for (Index j = 0; j < k; ++j) {
        double* x = R.col(j) + j;  // length m - j
        const Index len = m - j;
        const double tail_sq = dot(x + 1, x + 1, len - 1);
        const double c0 = x[0];
        double beta, t;
        if (tail_sq <= std::numeric_limits<double>::min()) {
            t = 0.0;
            beta = c0;
            for (Index i = 1; i < len; ++i) x[i] = 0.0;
        } else {
            beta = std::sqrt(c0 * c0 + tail_sq);
            if (c0 >= 0.0) beta = -beta;
            const double inv = 1.0 / (c0 - beta);
            for (Index i = 1; i < len; ++i) x[i] *= inv;
            t = (beta - c0) / beta;
        }
        x[0] = beta;
        tau[static_cast<size_t>(j)] = t;
        // apply H_j = I - t v v^T to the trailing columns
        if (t != 0.0) {
#pragma omp parallel for schedule(static) if (len * (k - j) > 100000)
            for (Index c = j + 1; c < k; ++c) {
                double* y = R.col(c) + j;
                const double d = t * (y[0] + dot(x + 1, y + 1, len - 1));
                y[0] -= d;
                for (Index i = 1; i < len; ++i) y[i] -= d * x[i];
            }
        }
    }
    Mat Q = Mat::identity(m, k);
    for (Index j = k - 1; j >= 0; --j) {
        const double t = tau[static_cast<size_t>(j)];
        if (t == 0.0) continue;
        const double* v = R.col(j) + j;
        const Index len = m - j;
#pragma omp parallel for schedule(static) if (len * k > 100000)
        for (Index c = 0; c < k; ++c) {
            double* y = Q.col(c) + j;
            const double d = t * (y[0] + dot(v + 1, y + 1, len - 1));
            y[0] -= d;
            for (Index i = 1; i < len; ++i) y[i] -= d * v[i];
        }
    }
    return Q;
}

namespace detail {

// One-sided (Hestenes) Jacobi on the columns of A (len x k): returns the
// column norms as sigma, normalizes A's columns in place and accumulates the
// right rotations in V (k x k).
inline void one_sided_jacobi(Mat& A, Mat& V, std::vector<double>& sigma) {
    const Index len = A.rows, k = A.cols;
    V = Mat::identity(k, k);
    const double eps = 2.220446049250313e-16;
    // Sweeps in round-robin (tournament) order: each of the P - 1 steps of a
    // sweep rotates P / 2 disjoint column pairs, so the pairs of a step run
    // in parallel and the result does not depend on the thread count.
    const Index P = k + (k & 1);  // even number of players (k odd: one bye)
    std::vector<Index> ring(static_cast<size_t>(P));
    for (int sweep = 0; sweep < 80; ++sweep) {
        int rotated = 0;
        for (Index q = 0; q < P; ++q) ring[static_cast<size_t>(q)] = q;
        for (Index step = 0; step + 1 < P; ++step) {
#pragma omp parallel for schedule(dynamic, 1) reduction(| : rotated) if (len * k > 20000)
            for (Index h = 0; h < P / 2; ++h) {
                Index i = ring[static_cast<size_t>(h)], j = ring[static_cast<size_t>(P - 1 - h)];
                if (i > j) std::swap(i, j);
                if (j >= k) continue;  // the bye
                double* ai = A.col(i);
                double* aj = A.col(j);
                const double alpha = dot(ai, ai, len), beta = dot(aj, aj, len), gamma = dot(ai, aj, len);
                if (gamma == 0.0 || !(std::abs(gamma) > eps * std::sqrt(alpha * beta))) continue;
                rotated = 1;
                const double zeta = (beta - alpha) / (2.0 * gamma);
                const double tt = (zeta >= 0.0 ? 1.0 : -1.0) /
                                  (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + tt * tt);
                const double s = c * tt;
                for (Index t = 0; t < len; ++t) {
                    const double x = ai[t], y = aj[t];
                    ai[t] = c * x - s * y;
                    aj[t] = s * x + c * y;
                }
                double* vi = V.col(i);
                double* vj = V.col(j);
                for (Index t = 0; t < k; ++t) {
                    const double x = vi[t], y = vj[t];
                    vi[t] = c * x - s * y;
                    vj[t] = s * x + c * y;
                }
            }
            // rotate every player but the first one place around the ring
            const Index last = ring[static_cast<size_t>(P - 1)];
            for (Index q = P - 1; q > 1; --q) ring[static_cast<size_t>(q)] = ring[static_cast<size_t>(q - 1)];
            if (P > 1) ring[1] = last;
        }
        if (!rotated) break;
    }
    sigma.assign(static_cast<size_t>(k), 0.0);
    for (Index j = 0; j < k; ++j) sigma[static_cast<size_t>(j)] = std::sqrt(dot(A.col(j), A.col(j), len));
    // sort descending (stable: ties keep column order)
    std::vector<Index> order(static_cast<size_t>(k));
    for (Index j = 0; j < k; ++j) order[static_cast<size_t>(j)] = j;
    std::stable_sort(order.begin(), order.end(), [&](Index x, Index y) {
        return sigma[static_cast<size_t>(x)] > sigma[static_cast<size_t>(y)];
    });
    Mat A2(len, k), V2(k, k);
    std::vector<double> s2(static_cast<size_t>(k));
    for (Index j = 0; j < k; ++j) {
        const Index o = order[static_cast<size_t>(j)];
        std::copy(A.col(o), A.col(o) + len, A2.col(j));
        std::copy(V.col(o), V.col(o) + k, V2.col(j));
        s2[static_cast<size_t>(j)] = sigma[static_cast<size_t>(o)];
    }
    A = std::move(A2);
    V = std::move(V2);
    sigma = std::move(s2);
    // normalize; complete null columns to an orthonormal set
    const double smax = k > 0 ? sigma[0] : 0.0;
    const double tiny = std::max(smax * 1e-300, std::numeric_limits<double>::min());
    for (Index j = 0; j < k; ++j) {
        double* a = A.col(j);
        const double s = sigma[static_cast<size_t>(j)];
        if (s > tiny && s > smax * 1e-15 * static_cast<double>(len)) {
            for (Index t = 0; t < len; ++t) a[t] /= s;
            continue;
        }
        // null direction: Gram-Schmidt a unit vector against previous columns
        for (Index e = 0; e < len; ++e) {
            std::fill(a, a + len, 0.0);
            a[e] = 1.0;
            for (int pass = 0; pass < 2; ++pass)
                for (Index p = 0; p < j; ++p) {
                    const double* q = A.col(p);
                    double d = 0.0;
                    for (Index t = 0; t < len; ++t) d += q[t] * a[t];
                    for (Index t = 0; t < len; ++t) a[t] -= d * q[t];
                }
            double nrm = 0.0;
            for (Index t = 0; t < len; ++t) nrm += a[t] * a[t];
            nrm = std::sqrt(nrm);
            if (nrm > 0.5) {
                for (Index t = 0; t < len; ++t) a[t] /= nrm;
                break;
            }
        }
    }
}

}  // namespace detail

// dense.hpp:114-117 — thin SVD, sigma non-increasing.  BDCSVD is restated
// by a one-sided Jacobi SVD (high relative accuracy; tests pin tolerance).
inline LowRankFactors small_svd(const Mat& B) {
    LowRankFactors f;
    // Strongly rectangular blocks (the r x n coefficient block of a sketch):
    // QR-precondition so Jacobi rotates r-length columns instead of n-length
    // ones.  B^T = Qb R  =>  B = R^T Qb^T,  svd(R^T) = Ur S Vr^T,  B = Ur S (Qb Vr)^T.
    if (B.cols > 2 * B.rows && B.rows >= 16) {
        const Mat Bt = transpose(B);          // n x r
        const Mat Qb = qr_orthonormal(Bt);    // n x r
        const Mat Rt = mul_tn(Bt, Qb);        // (Qb^T Bt)^T = R^T, r x r
        LowRankFactors g = small_svd(Rt);
        f.U = std::move(g.U);
        f.sigma = std::move(g.sigma);
        f.V = mul_nn(Qb, g.V);
        return f;
    }
    if (B.rows > 2 * B.cols && B.cols >= 16) {
        const Mat Qb = qr_orthonormal(B);     // m x c
        const Mat R = mul_tn(Qb, B);          // c x c
        LowRankFactors g = small_svd(R);
        f.U = mul_nn(Qb, g.U);
        f.sigma = std::move(g.sigma);
        f.V = std::move(g.V);
        return f;
    }
    if (B.rows >= B.cols) {
        Mat A = B;
        Mat V;
        detail::one_sided_jacobi(A, V, f.sigma);
        f.U = std::move(A);
        f.V = std::move(V);
    } else {
        Mat A = transpose(B);
        Mat V;
        detail::one_sided_jacobi(A, V, f.sigma);
        f.U = std::move(V);
        f.V = std::move(A);
    }
    return f;
}

// dense.hpp:119
inline double frob_norm_sq(const Mat& X) { return X.squared_norm(); }

// ---------------------------------------------------------------------------
// sampled.hpp
// ---------------------------------------------------------------------------

struct Triplet {
    Index row;
    Index col;
    double value;
};

// sampled.hpp:25-110 — CSR over sorted row-major triplets.
class SampledMatrix {
public:
    SampledMatrix(Index rows, Index cols, std::vector<Triplet> entries) : rows_(rows), cols_(cols) {
        if (rows < 1 || cols < 1) throw std::invalid_argument("SampledMatrix: dimensions must be >= 1");
        if (entries.empty()) throw std::invalid_argument("SampledMatrix: at least one entry required");
        std::sort(entries.begin(), entries.end(), [](const Triplet& a, const Triplet& b) {
            return a.row != b.row ? a.row < b.row : a.col < b.col;
        });
        col_index_.resize(entries.size());
        values_.resize(entries.size());
        row_offsets_.assign(static_cast<size_t>(rows) + 1, 0);
        for (size_t k = 0; k < entries.size(); ++k) {
            const Triplet& t = entries[k];
            if (t.row < 0 || t.row >= rows || t.col < 0 || t.col >= cols)
                throw std::invalid_argument("SampledMatrix: entry (" + std::to_string(t.row) + ", " +
                                            std::to_string(t.col) + ") out of range");
            if (!std::isfinite(t.value))
                throw std::invalid_argument("SampledMatrix: non-finite value");
            if (k > 0 && entries[k - 1].row == t.row && entries[k - 1].col == t.col)
                throw std::invalid_argument("SampledMatrix: duplicate entry (" + std::to_string(t.row) +
                                            ", " + std::to_string(t.col) + ")");
            col_index_[k] = t.col;
            values_[k] = t.value;
            ++row_offsets_[static_cast<size_t>(t.row) + 1];
        }
        for (size_t i = 1; i < row_offsets_.size(); ++i) row_offsets_[i] += row_offsets_[i - 1];
    }
    // Direct CSR construction (already validated / sorted), used by the C API.
    SampledMatrix(Index rows, Index cols, std::vector<Index> rowptr, std::vector<Index> col,
                  std::vector<double> val)
        : rows_(rows), cols_(cols), row_offsets_(std::move(rowptr)), col_index_(std::move(col)),
          values_(std::move(val)) {}

    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index nnz() const { return static_cast<Index>(values_.size()); }
    const std::vector<Index>& row_offsets() const { return row_offsets_; }
    const std::vector<Index>& col_index() const { return col_index_; }
    const std::vector<double>& values() const { return values_; }

    bool same_pattern(const SampledMatrix& o) const {
        return rows_ == o.rows_ && cols_ == o.cols_ && row_offsets_ == o.row_offsets_ &&
               col_index_ == o.col_index_;
    }
    // sampled.hpp:79-91
    SampledMatrix with_values(std::vector<double> vals) const {
        if (vals.size() != values_.size()) throw std::invalid_argument("with_values: size mismatch");
        for (double v : vals)
            if (!std::isfinite(v)) throw std::invalid_argument("with_values: non-finite value");
        SampledMatrix out(*this);
        out.values_ = std::move(vals);
        return out;
    }

private:
    Index rows_, cols_;
    std::vector<Index> row_offsets_, col_index_;
    std::vector<double> values_;
};

// sampled.hpp:113-127 — row-gather accumulation, same order.
inline Mat sp_mult(const SampledMatrix& S, const Mat& X) {
    if (X.rows != S.cols()) throw std::invalid_argument("sp_mult: inner dimensions disagree");
    Mat out(S.rows(), X.cols);
    const auto& off = S.row_offsets();
    const auto& cols = S.col_index();
    const auto& vals = S.values();
#pragma omp parallel for schedule(dynamic, 256) if (S.nnz() * X.cols > 200000)
    for (Index i = 0; i < S.rows(); ++i)
        for (Index k = off[static_cast<size_t>(i)]; k < off[static_cast<size_t>(i) + 1]; ++k) {
            const double v = vals[static_cast<size_t>(k)];
            const Index c = cols[static_cast<size_t>(k)];
            for (Index j = 0; j < X.cols; ++j) out(i, j) += v * X(c, j);
        }
    return out;
}

// sampled.hpp:130-144 — scatter in CSR order.
inline Mat sp_mult_t(const SampledMatrix& S, const Mat& X) {
    if (X.rows != S.rows()) throw std::invalid_argument("sp_mult_t: inner dimensions disagree");
    Mat out(S.cols(), X.cols);
    const auto& off = S.row_offsets();
    const auto& cols = S.col_index();
    const auto& vals = S.values();
    // columns of the output are independent: one column per task, each in
    // the reference's CSR scatter order
#pragma omp parallel for schedule(dynamic, 1) if (S.nnz() * X.cols > 200000 && X.cols > 1)
    for (Index j = 0; j < X.cols; ++j) {
        double* oj = out.col(j);
        const double* xj = X.col(j);
        for (Index i = 0; i < S.rows(); ++i)
            for (Index k = off[static_cast<size_t>(i)]; k < off[static_cast<size_t>(i) + 1]; ++k)
                oj[cols[static_cast<size_t>(k)]] += vals[static_cast<size_t>(k)] * xj[i];
    }
    return out;
}

// sampled.hpp:148-163 — SDDMM on the pattern.
inline SampledMatrix project_low_rank(const SampledMatrix& pattern, const LowRankFactors& F) {
    if (F.U.rows != pattern.rows() || F.V.rows != pattern.cols())
        throw std::invalid_argument("project_low_rank: factor dimensions disagree with pattern");
    const Index r = F.rank();
    Mat W = F.V;  // n x r, V * diag(sigma)
    for (Index j = 0; j < r; ++j)
        for (Index i = 0; i < W.rows; ++i) W(i, j) *= F.sigma[static_cast<size_t>(j)];
    const auto& off = pattern.row_offsets();
    const auto& cols = pattern.col_index();
    std::vector<double> vals(static_cast<size_t>(pattern.nnz()));
#pragma omp parallel for schedule(dynamic, 256) if (pattern.nnz() * r > 200000)
    for (Index i = 0; i < pattern.rows(); ++i)
        for (Index p = off[static_cast<size_t>(i)]; p < off[static_cast<size_t>(i) + 1]; ++p) {
            const Index c = cols[static_cast<size_t>(p)];
            double s = 0.0;
            for (Index j = 0; j < r; ++j) s += F.U(i, j) * W(c, j);
            vals[static_cast<size_t>(p - off[0])] = s;
        }
    return pattern.with_values(std::move(vals));
}

// sampled.hpp:166-176
inline SampledMatrix sp_axpy(const SampledMatrix& Yc, double alpha, const SampledMatrix& D) {
    if (!Yc.same_pattern(D)) throw std::invalid_argument("sp_axpy: operands must share the identical pattern");
    std::vector<double> vals(Yc.values());
    const auto& dv = D.values();
    for (size_t k = 0; k < vals.size(); ++k) vals[k] += alpha * dv[k];
    return Yc.with_values(std::move(vals));
}

// sampled.hpp:178-184
inline double sp_frob_norm_sq(const SampledMatrix& S) {
    double acc = 0.0;
    for (double v : S.values()) acc += v * v;
    return acc;
}

inline double norm_of(const Mat& X) { return std::sqrt(X.squared_norm()); }

// sampled.hpp:188-213
inline double spectral_norm_est(const SampledMatrix& S, int iters, std::uint64_t seed) {
    if (iters < 1) throw std::invalid_argument("spectral_norm_est: iters must be >= 1");
    Mat x = gaussian_block(S.cols(), 1, seed);
    double xn = norm_of(x);
    if (xn == 0.0) return 0.0;
    for (double& v : x.a) v /= xn;
    double estimate = 0.0;
    for (int it = 0; it < iters; ++it) {
        Mat y = sp_mult(S, x);
        estimate = norm_of(y);
        if (estimate == 0.0) return 0.0;
        x = sp_mult_t(S, y);
        xn = norm_of(x);
        if (xn == 0.0) return estimate;
        for (double& v : x.a) v /= xn;
    }
    return estimate;
}

// sampled.hpp:217-228
inline Mat densify(const SampledMatrix& S) {
    Mat out(S.rows(), S.cols());
    const auto& off = S.row_offsets();
    for (Index i = 0; i < S.rows(); ++i)
        for (Index k = off[static_cast<size_t>(i)]; k < off[static_cast<size_t>(i) + 1]; ++k)
            out(i, S.col_index()[static_cast<size_t>(k)]) = S.values()[static_cast<size_t>(k)];
    return out;
}

// ---------------------------------------------------------------------------
// sketch.hpp
// ---------------------------------------------------------------------------

// sketch.hpp:20-27
struct SketchParams {
    Index t = 10;
    Index dt = 10;
    int np = 1;
    double eps_threshold = 0.5;
    std::uint64_t seed = 1;
    Index p = 5;
};

// sketch.hpp:32-39
struct QBState {
    Mat Q;   // m x r
    Mat Bt;  // n x r: B^T (columns append without the reference's O(r n)
             // conservativeResize copy of a column-major B; same values)
    double norm_b_sq = 0.0;
    double frob_y_sq = 0.0;
    Index rank = 0;
    bool saturated = false;
};

// sketch.hpp:41-46
struct SketchResult {
    LowRankFactors factors;
    Index rank = 0;
    bool saturated = false;
    int extension_rounds = 0;
};

// sketch.hpp:50-56
inline double error_percentage(const QBState& st) {
    if (!(st.frob_y_sq > 0.0)) throw std::domain_error("error_percentage: target has zero Frobenius norm");
    const double eps = (st.frob_y_sq - st.norm_b_sq) / st.frob_y_sq;
    return std::clamp(eps, 0.0, 1.0);
}

namespace detail {

// sketch.hpp:60-67
inline void check_sketch_params(const SketchParams& p) {
    if (p.t < 1 || p.dt < 1 || p.np < 0) throw std::invalid_argument("SketchParams: need t >= 1, dt >= 1, np >= 0");
    if (!(p.eps_threshold > 0.0 && p.eps_threshold < 1.0))
        throw std::invalid_argument("SketchParams: eps_threshold must lie in (0, 1)");
}

// sketch.hpp:71-79
inline Mat power_iterate(const SampledMatrix& Y, Mat X, int np) {
    for (int j = 0; j < np; ++j) {
        if (j > 0) X = qr_orthonormal(X);
        X = sp_mult(Y, sp_mult_t(Y, X));
    }
    return X;
}

// sketch.hpp:82-84
inline Mat coefficient_block(const SampledMatrix& Y, const Mat& Q) { return transpose(sp_mult_t(Y, Q)); }

inline double max_abs(const Mat& X) {
    double m = 0.0;
    for (double v : X.a) m = std::max(m, std::abs(v));
    return m;
}

}  // namespace detail

// sketch.hpp:89-108
inline QBState qb_init(const SampledMatrix& Y, Index t, int np, std::uint64_t seed) {
    const Index min_dim = std::min(Y.rows(), Y.cols());
    if (t < 1 || t > min_dim) throw std::invalid_argument("qb_init: t must satisfy 1 <= t <= min(m, n)");
    const double frob_y_sq = sp_frob_norm_sq(Y);
    if (!(frob_y_sq > 0.0)) throw std::domain_error("qb_init: target matrix is all zero");
    Mat X = sp_mult(Y, gaussian_block(Y.cols(), t, seed));
    X = detail::power_iterate(Y, std::move(X), np);
    QBState st;
    st.Q = qr_orthonormal(X);
    st.Bt = sp_mult_t(Y, st.Q);  // coefficient_block, transposed
    st.norm_b_sq = frob_norm_sq(st.Bt);
    st.frob_y_sq = frob_y_sq;
    st.rank = t;
    st.saturated = (t == min_dim);
    return st;
}

// sketch.hpp:114-154
inline QBState qb_extend(QBState st, const SampledMatrix& Y, Index dt, int np, std::uint64_t seed) {
    if (dt < 1) throw std::invalid_argument("qb_extend: dt must be >= 1");
    if (st.Q.rows != Y.rows() || st.Bt.rows != Y.cols())
        throw std::invalid_argument("qb_extend: state does not match target dimensions");
    const Index min_dim = std::min(Y.rows(), Y.cols());
    const Index width = std::min(dt, min_dim - st.rank);
    if (width < 1) {
        st.saturated = true;
        return st;
    }
    Mat X = sp_mult(Y, gaussian_block(Y.cols(), width, seed));
    X = detail::power_iterate(Y, std::move(X), np);
    // sketch.hpp:133-141 — CGS, conditional second CGS, QR, conditional re-projection
    sub_mul(X, st.Q, mul_tn(st.Q, X));
    {
        const Mat C = mul_tn(st.Q, X);
        if (norm_of(C) > 1e-8 * norm_of(X)) sub_mul(X, st.Q, C);
    }
    Mat Qp = qr_orthonormal(X);
    {
        const Mat D = mul_tn(st.Q, Qp);
        if (detail::max_abs(D) > 1e-8) {
            sub_mul(Qp, st.Q, D);
            Qp = qr_orthonormal(Qp);
        }
    }
    const Mat Bpt = sp_mult_t(Y, Qp);  // coefficient_block, transposed
    const Index r0 = st.rank;
    // append (sketch.hpp:145-152): column blocks of Q and B^T
    st.Q.a.insert(st.Q.a.end(), Qp.a.begin(), Qp.a.end());
    st.Q.cols += width;
    st.Bt.a.insert(st.Bt.a.end(), Bpt.a.begin(), Bpt.a.end());
    st.Bt.cols += width;
    st.norm_b_sq += frob_norm_sq(Bpt);
    st.rank = r0 + width;
    st.saturated = (st.rank == min_dim);
    return st;
}

// sketch.hpp:158-162
inline LowRankFactors finalize(const QBState& st) {
    LowRankFactors f = small_svd(transpose(st.Bt));
    f.U = mul_nn(st.Q, f.U);
    return f;
}

// sketch.hpp:165-182
inline LowRankFactors rsvd(const SampledMatrix& Y, Index k, const SketchParams& p) {
    const Index min_dim = std::min(Y.rows(), Y.cols());
    if (k < 1) throw std::invalid_argument("rsvd: k must be >= 1");
    if (p.p < 0 || k + p.p > min_dim) throw std::invalid_argument("rsvd: k + p must not exceed min(m, n)");
    Mat X = sp_mult(Y, gaussian_block(Y.cols(), k + p.p, derive_seed(p.seed, 0)));
    X = detail::power_iterate(Y, std::move(X), p.np);
    const Mat Q = qr_orthonormal(X);
    LowRankFactors f = small_svd(detail::coefficient_block(Y, Q));
    f.U = mul_nn(Q, f.U).left_cols(k);
    f.sigma.resize(static_cast<size_t>(k));
    f.V = f.V.left_cols(k);
    return f;
}

// sketch.hpp:188-201
inline SketchResult r3svd(const SampledMatrix& Y, const SketchParams& p) {
    detail::check_sketch_params(p);
    QBState st = qb_init(Y, p.t, p.np, derive_seed(p.seed, 0));
    int rounds = 0;
    while (error_percentage(st) > p.eps_threshold) {
        if (st.saturated) return SketchResult{finalize(st), st.rank, true, rounds};
        ++rounds;
        st = qb_extend(std::move(st), Y, p.dt, p.np, derive_seed(p.seed, static_cast<std::uint64_t>(rounds)));
    }
    return SketchResult{finalize(st), st.rank, false, rounds};
}

// sketch.hpp:207-250
inline SketchResult r4svd(const SampledMatrix& Y, const Mat& U_prev, const SketchParams& p) {
    detail::check_sketch_params(p);
    const Index s = U_prev.cols;
    if (s == 0) {
        SketchParams fresh = p;
        fresh.t = p.dt;
        return r3svd(Y, fresh);
    }
    if (U_prev.rows != Y.rows()) throw std::invalid_argument("r4svd: U_prev row count does not match Y");
    const Index min_dim = std::min(Y.rows(), Y.cols());
    if (s > min_dim) throw std::invalid_argument("r4svd: recycled basis wider than min(m, n)");
    const double frob_y_sq = sp_frob_norm_sq(Y);
    if (!(frob_y_sq > 0.0)) throw std::domain_error("r4svd: target matrix is all zero");
    QBState st;
    st.Q = U_prev;
    Mat gram = mul_tn(st.Q, st.Q);
    for (Index i = 0; i < s; ++i) gram(i, i) -= 1.0;
    if (detail::max_abs(gram) > 1e-8) st.Q = qr_orthonormal(st.Q);
    st.Bt = sp_mult_t(Y, st.Q);  // coefficient_block, transposed
    st.norm_b_sq = frob_norm_sq(st.Bt);
    st.frob_y_sq = frob_y_sq;
    st.rank = s;
    st.saturated = (s == min_dim);
    int rounds = 0;
    while (error_percentage(st) > p.eps_threshold) {
        if (st.saturated) return SketchResult{finalize(st), st.rank, true, rounds};
        ++rounds;
        st = qb_extend(std::move(st), Y, p.dt, p.np, derive_seed(p.seed, static_cast<std::uint64_t>(rounds)));
    }
    return SketchResult{finalize(st), st.rank, false, rounds};
}

// ---------------------------------------------------------------------------
// solver.hpp
// ---------------------------------------------------------------------------

// solver.hpp:32-43 (+ the Appendix-B harness extension eps_threshold_min,
// default 0 == reference behaviour, and rel_residual_stop, default 0 ==
// disabled; both applied identically on the GPU path).
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
    double eps_threshold_min = 0.0;  // extension (cooling floor)
    double rel_residual_stop = 0.0;  // extension (observer-level stop on ||P(X-A)||/||P A||)
};

// solver.hpp:49-57 (+ extension columns computed from the same projection)
struct IterationRecord {
    int iter = 0;
    Index rank = 0;
    double residual = 0.0;
    double eps_threshold = 0.0;
    double train_mae = 0.0;
    double sketch_ms = 0.0;
    double total_ms = 0.0;
    // extensions
    Index kept = 0;                // rank of the shrunk X
    double rel_residual_x = 0.0;   // ||P_Lambda(X - A)||_F / ||P_Lambda A||_F
    double test_mae = 0.0;         // held-out MAE (if a test set is supplied)
    double test_rmse = 0.0;        // held-out RMSE
    int extension_rounds = 0;
};

// solver.hpp:59-67
struct StopRule {
    enum class Kind { TrainMae = 0, Residual = 1, None = 2 };
    Kind kind = Kind::TrainMae;
    double threshold = 0.1;
};

// solver.hpp:69-78
struct Backend {
    enum class Kind { R4Svd = 0, R3Svd = 1, RsvdFixed = 2, FullSvd = 3 };
    Kind kind = Kind::R4Svd;
    Index fixed_rank = 0;
};

// solver.hpp:80-84
struct SvtResult {
    LowRankFactors factors;
    std::vector<IterationRecord> trace;
    bool converged = false;
};

// solver.hpp:88
using IterationObserver = std::function<bool(const IterationRecord&, const LowRankFactors&)>;

inline constexpr int kSpectralNormIters = 20;  // solver.hpp:90

// solver.hpp:95-106
inline SvtConfig default_config(const SampledMatrix& A) {
    SvtConfig cfg;
    cfg.tau = std::sqrt(sp_frob_norm_sq(A));
    cfg.delta = std::sqrt(static_cast<double>(A.rows()) * static_cast<double>(A.cols()) /
                          static_cast<double>(A.nnz()));
    const Index min_dim = std::min(A.rows(), A.cols());
    cfg.t0 = std::max<Index>(1, static_cast<Index>(0.05 * static_cast<double>(min_dim)));
    cfg.dt = 10;
    cfg.beta = 0.95;
    return cfg;
}

// solver.hpp:110-120
inline LowRankFactors shrink(const LowRankFactors& F, double tau) {
    Index keep = 0;
    while (keep < F.rank() && F.sigma[static_cast<size_t>(keep)] > tau) ++keep;
    LowRankFactors out;
    out.U = F.U.left_cols(keep);
    out.sigma.resize(static_cast<size_t>(keep));
    for (Index j = 0; j < keep; ++j) out.sigma[static_cast<size_t>(j)] = F.sigma[static_cast<size_t>(j)] - tau;
    out.V = F.V.left_cols(keep);
    return out;
}

// solver.hpp:125-140
inline SampledMatrix kickstart(const SampledMatrix& A, double tau, double delta, std::uint64_t seed) {
    if (!(tau > 0.0) || !(delta > 0.0)) throw std::invalid_argument("kickstart: tau and delta must be positive");
    const double sigma1 = spectral_norm_est(A, kSpectralNormIters, seed);
    double k0 = 1.0;
    if (sigma1 > 0.0) k0 = std::max(1.0, std::ceil(tau / (delta * sigma1)));
    std::vector<double> vals(A.values());
    for (double& v : vals) v *= k0 * delta;
    return A.with_values(std::move(vals));
}

// solver.hpp:143-155
inline double residual(const SampledMatrix& A, const SampledMatrix& Y) {
    if (!A.same_pattern(Y)) throw std::invalid_argument("residual: operands must share the identical pattern");
    double acc = 0.0;
    for (size_t k = 0; k < A.values().size(); ++k) {
        const double d = A.values()[k] - Y.values()[k];
        acc += d * d;
    }
    return std::sqrt(acc);
}

// solver.hpp:159-168
inline double train_mae(const SampledMatrix& A, const LowRankFactors& F) {
    const SampledMatrix P = project_low_rank(A, F);
    double acc = 0.0;
    for (size_t k = 0; k < A.values().size(); ++k) acc += std::abs(A.values()[k] - P.values()[k]);
    return acc / static_cast<double>(A.values().size());
}

namespace detail {

inline double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

// solver.hpp:186-205
inline void check_config(const SvtConfig& cfg) {
    if (!(cfg.tau > 0.0)) throw std::invalid_argument("SvtConfig: tau must be positive");
    if (!(cfg.delta > 0.0)) throw std::invalid_argument("SvtConfig: delta must be positive");
    if (!(cfg.beta > 0.0 && cfg.beta < 1.0)) throw std::invalid_argument("SvtConfig: beta must lie in (0, 1)");
    if (!(cfg.eps_threshold0 > 0.0 && cfg.eps_threshold0 < 1.0))
        throw std::invalid_argument("SvtConfig: eps_threshold0 must lie in (0, 1)");
    if (cfg.maxit < 1) throw std::invalid_argument("SvtConfig: maxit must be >= 1");
    if (cfg.t0 < 1 || cfg.dt < 1 || cfg.np < 0) throw std::invalid_argument("SvtConfig: need t0 >= 1, dt >= 1, np >= 0");
}

}  // namespace detail

// solver.hpp:215-328 — the Bregman loop.  `test` (optional) is the held-out
// pattern for the Appendix-B RMSE/MAE extension (reference: the ratings
// observer, svt_main.cpp:355-369).
// Test-harness extension (no reference counterpart): the loop-carried state
// after `iter` completed iterations (Y, U_prev, the cooling threshold and
// the running residual minimum), so one iteration of a long run can be
// checked against the device path from a common state.
struct SvtStart {
    int iter = 0;
    std::vector<double> y;  // Y on A's pattern (CSR order)
    Mat U_prev;             // m x s
    double eps_threshold = 0.0;
    double eps_min = 0.0;
};

inline SvtResult svt_run_backend(const SampledMatrix& A, const SvtConfig& cfg, StopRule stop, Backend backend,
                                 const IterationObserver& observer = {}, const SampledMatrix* test = nullptr,
                                 const SvtStart* start = nullptr) {
    detail::check_config(cfg);
    const Index min_dim = std::min(A.rows(), A.cols());
    if (backend.kind == Backend::Kind::RsvdFixed && (backend.fixed_rank < 1 || backend.fixed_rank > min_dim))
        throw std::invalid_argument("svt_run_backend: fixed rank out of range");
    if (cfg.t0 > min_dim) throw std::invalid_argument("SvtConfig: t0 exceeds min(m, n)");

    SampledMatrix Y = start ? A.with_values(start->y) : kickstart(A, cfg.tau, cfg.delta, derive_seed(cfg.seed, 0));
    Mat U_prev = start ? start->U_prev : Mat(A.rows(), 0);
    double eps_threshold = start ? start->eps_threshold : cfg.eps_threshold0;
    double eps_min = start ? start->eps_min : std::numeric_limits<double>::infinity();
    const double frob_a = std::sqrt(sp_frob_norm_sq(A));

    SvtResult result;
    result.factors = LowRankFactors{Mat(A.rows(), 0), {}, Mat(A.cols(), 0)};
    double best_metric = std::numeric_limits<double>::infinity();
    const double t_start = detail::now_ms();
    for (int iter = (start ? start->iter : 0) + 1; iter <= cfg.maxit; ++iter) {
        const std::uint64_t iter_seed = derive_seed(cfg.seed, static_cast<std::uint64_t>(iter));
        SketchParams sp;
        sp.t = cfg.t0;
        sp.dt = cfg.dt;
        sp.np = cfg.np;
        sp.eps_threshold = eps_threshold;
        sp.seed = iter_seed;

        const double t_sketch = detail::now_ms();
        LowRankFactors full;
        Index revealed = 0;
        int rounds = 0;
        switch (backend.kind) {
            case Backend::Kind::R4Svd: {
                SketchResult sr = (iter == 1) ? r3svd(Y, sp) : r4svd(Y, U_prev, sp);
                full = std::move(sr.factors);
                revealed = sr.rank;
                rounds = sr.extension_rounds;
                break;
            }
            case Backend::Kind::R3Svd: {
                SketchResult sr = r3svd(Y, sp);
                full = std::move(sr.factors);
                revealed = sr.rank;
                rounds = sr.extension_rounds;
                break;
            }
            case Backend::Kind::RsvdFixed: {
                SketchParams fixed = sp;
                fixed.p = std::min<Index>(sp.p, min_dim - backend.fixed_rank);
                full = rsvd(Y, backend.fixed_rank, fixed);
                revealed = backend.fixed_rank;
                break;
            }
            case Backend::Kind::FullSvd: {
                full = small_svd(densify(Y));
                revealed = min_dim;
                break;
            }
        }
        const double sketch_ms = detail::now_ms() - t_sketch;

        const double eps_i = residual(A, Y);
        if (eps_i < eps_min) {
            eps_min = eps_i;
        } else {
            eps_threshold = std::max(eps_threshold * cfg.beta, cfg.eps_threshold_min);
        }

        LowRankFactors X = shrink(full, cfg.tau);
        // train_mae (solver.hpp:159-168) and the relative residual share one projection
        const SampledMatrix P = project_low_rank(A, X);
        double mae_acc = 0.0, sq_acc = 0.0;
        for (size_t k = 0; k < A.values().size(); ++k) {
            const double d = A.values()[k] - P.values()[k];
            mae_acc += std::abs(d);
            sq_acc += d * d;
        }
        const double mae = mae_acc / static_cast<double>(A.values().size());

        IterationRecord rec;
        rec.iter = iter;
        rec.rank = revealed;
        rec.residual = eps_i;
        rec.eps_threshold = eps_threshold;
        rec.train_mae = mae;
        rec.sketch_ms = sketch_ms;
        rec.total_ms = detail::now_ms() - t_start;
        rec.kept = X.rank();
        rec.rel_residual_x = std::sqrt(sq_acc) / frob_a;
        rec.extension_rounds = rounds;
        if (test != nullptr) {
            const SampledMatrix Pt = project_low_rank(*test, X);
            double ta = 0.0, ts = 0.0;
            for (size_t k = 0; k < test->values().size(); ++k) {
                const double d = test->values()[k] - Pt.values()[k];
                ta += std::abs(d);
                ts += d * d;
            }
            rec.test_mae = ta / static_cast<double>(test->values().size());
            rec.test_rmse = std::sqrt(ts / static_cast<double>(test->values().size()));
        }
        result.trace.push_back(rec);

        const double metric = (stop.kind == StopRule::Kind::Residual) ? eps_i : mae;
        if (metric < best_metric) {
            best_metric = metric;
            result.factors = X;
        }
        bool stop_hit = false;
        if (stop.kind == StopRule::Kind::TrainMae && mae < stop.threshold) stop_hit = true;
        else if (stop.kind == StopRule::Kind::Residual && eps_i < stop.threshold) stop_hit = true;
        bool keep_going = true;
        if (cfg.rel_residual_stop > 0.0 && rec.rel_residual_x < cfg.rel_residual_stop) keep_going = false;
        if (keep_going && observer) keep_going = observer(rec, X);
        if (stop_hit || !keep_going) {
            result.factors = std::move(X);
            result.converged = true;
            return result;
        }
        // solver.hpp:321-324 — Y <- Y + delta * (A - P_Lambda(X))
        const SampledMatrix D = sp_axpy(A, -1.0, P);
        Y = sp_axpy(Y, cfg.delta, D);
        U_prev = X.U;
    }
    result.converged = false;
    return result;
}

}  // namespace svt_oracle
