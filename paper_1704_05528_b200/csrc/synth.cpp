// Seeded synthetic inputs for the five BASELINE.json configurations (host).
//
// These stand in for the paper's photographs and MovieLens sets, which are not
// in this container.  The reference's own generators do not match
// the BASELINE configs, so these are new; their
// building blocks restate the reference's: the mt19937_64 Box-Muller stream
// and derive_seed (dense.hpp:43-98), the multiply-shift bounded draw and
// partial Fisher-Yates sampler (io.hpp:93-113) and split_ratings
// (io.hpp:474-495).  Every per-row / per-user stream is derived from the
// master seed, so the output is identical for any host thread count.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <random>
#include <stdexcept>
#include <thread>
#include <unordered_set>
#include <vector>

#include "common.hpp"

namespace svtb {

u64 derive_seed_u(u64 seed, u64 stream);

namespace {

struct Gauss {  // dense.hpp:52-80
    std::mt19937_64 g;
    double spare = 0.0;
    bool have = false;
    explicit Gauss(u64 s) : g(s) {}
    double u01() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
    double next() {
        if (have) {
            have = false;
            return spare;
        }
        const double u1 = 1.0 - u01();
        const double u2 = u01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * 3.14159265358979323846 * u2;
        spare = r * std::sin(a);
        have = true;
        return r * std::cos(a);
    }
};

// column-major gaussian block (dense.hpp:86-98)
std::vector<double> gaussian_cm(i64 rows, i64 cols, u64 seed) {
    Gauss g(seed);
    std::vector<double> b(static_cast<size_t>(rows * cols));
    for (i64 j = 0; j < cols; ++j)
        for (i64 i = 0; i < rows; ++i) b[static_cast<size_t>(i + j * rows)] = g.next();
    return b;
}

u64 bounded(std::mt19937_64& rng, u64 n) {  // io.hpp:93-96
    return static_cast<u64>((static_cast<unsigned __int128>(rng()) * static_cast<unsigned __int128>(n)) >> 64);
}

std::vector<u64> sample_positions(u64 total, u64 ns, u64 seed) {  // io.hpp:100-113
    std::vector<u64> idx(total);
    for (u64 i = 0; i < total; ++i) idx[i] = i;
    std::mt19937_64 rng(seed);
    for (u64 i = 0; i < ns; ++i) {
        const u64 j = i + bounded(rng, total - i);
        std::swap(idx[i], idx[j]);
    }
    idx.resize(ns);
    return idx;
}

template <typename F>
void parallel_for(i64 n, F&& f) {
    const int T = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    if (n < 1024 || T == 1) {
        f(0, n);
        return;
    }
    std::vector<std::thread> th;
    const i64 chunk = (n + T - 1) / T;
    for (int t = 0; t < T; ++t) {
        const i64 a = t * chunk, b = std::min(n, a + chunk);
        if (a >= b) break;
        th.emplace_back([&f, a, b] { f(a, b); });
    }
    for (auto& x : th) x.join();
}

struct Triples {
    i64 m = 0, n = 0;
    std::vector<i64> r, c;
    std::vector<double> v;
    i64 size() const { return static_cast<i64>(v.size()); }
};

// config 1: M = L R^T, L, R (1000 x 10) iid N(0, 1) (unscaled), 20% observed
void gen_config1(u64 seed, Triples& tr) {
    const i64 m = 1000, n = 1000, r = 10;
    const auto L = gaussian_cm(m, r, derive_seed_u(seed, 1));
    const auto R = gaussian_cm(n, r, derive_seed_u(seed, 2));
    const u64 ns = 200000;
    const auto pos = sample_positions(static_cast<u64>(m * n), ns, derive_seed_u(seed, 3));
    tr.m = m;
    tr.n = n;
    tr.r.resize(ns);
    tr.c.resize(ns);
    tr.v.resize(ns);
    for (u64 k = 0; k < ns; ++k) {
        const i64 i = static_cast<i64>(pos[k] / n), j = static_cast<i64>(pos[k] % n);
        double s = 0.0;
        for (i64 q = 0; q < r; ++q) s += L[static_cast<size_t>(i + q * m)] * R[static_cast<size_t>(j + q * n)];
        tr.r[k] = i;
        tr.c[k] = j;
        tr.v[k] = s;
    }
}

// config 2: 512 x 512 image = 40 Gaussian blobs + 10 low-frequency cosines,
// min-max scaled to [0, 255]; 50% of pixels observed
void gen_config2(u64 seed, Triples& tr) {
    const i64 H = 512, W = 512;
    Gauss g(derive_seed_u(seed, 1));
    std::vector<double> img(static_cast<size_t>(H * W), 0.0);
    const double two_pi = 2.0 * 3.14159265358979323846;
    for (int b = 0; b < 40; ++b) {
        const double cy = g.u01() * H, cx = g.u01() * W;
        const double sg = 8.0 + 56.0 * g.u01();
        const double amp = g.u01();
        const double inv = 1.0 / (2.0 * sg * sg);
        for (i64 y = 0; y < H; ++y)
            for (i64 x = 0; x < W; ++x) {
                const double dy = static_cast<double>(y) - cy, dx = static_cast<double>(x) - cx;
                img[static_cast<size_t>(y * W + x)] += amp * std::exp(-(dx * dx + dy * dy) * inv);
            }
    }
    for (int q = 0; q < 10; ++q) {
        const int fy = 1 + static_cast<int>(bounded(g.g, 6)), fx = 1 + static_cast<int>(bounded(g.g, 6));
        const double py = two_pi * g.u01(), px = two_pi * g.u01();
        const double amp = 0.5 * g.u01();
        for (i64 y = 0; y < H; ++y)
            for (i64 x = 0; x < W; ++x)
                img[static_cast<size_t>(y * W + x)] +=
                    amp * std::cos(two_pi * fy * static_cast<double>(y) / H + py) *
                    std::cos(two_pi * fx * static_cast<double>(x) / W + px);
    }
    const auto mm = std::minmax_element(img.begin(), img.end());
    const double lo = *mm.first, span = *mm.second - *mm.first;
    for (double& v : img) v = (span > 0.0) ? 255.0 * (v - lo) / span : 0.0;
    const u64 ns = static_cast<u64>(H * W / 2);
    const auto pos = sample_positions(static_cast<u64>(H * W), ns, derive_seed_u(seed, 3));
    tr.m = H;
    tr.n = W;
    tr.r.resize(ns);
    tr.c.resize(ns);
    tr.v.resize(ns);
    for (u64 k = 0; k < ns; ++k) {
        tr.r[k] = static_cast<i64>(pos[k] / W);
        tr.c[k] = static_cast<i64>(pos[k] % W);
        tr.v[k] = img[pos[k]];
    }
}

// configs 3 / 4: recommender-shaped ratings.  Per-user degrees follow a
// power law with exponent 1.6 (Pareto tail d_min * U^{-1/0.6}, d_min = 20),
// rescaled to the exact total; items are drawn Zipf(1.1)-weighted without
// replacement (exponential-key sampling) over a random item order; values are
// round/clip of 3.5 + U V^T + N(0, 0.5^2).
void gen_ratings(u64 seed, i64 m, i64 n, i64 total, int rank, double fsd, bool half_star, Triples& tr) {
    std::mt19937_64 rng(derive_seed_u(seed, 1));
    auto u01 = [&] { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
    std::vector<double> raw(static_cast<size_t>(m));
    for (i64 u = 0; u < m; ++u) {
        const double x = 1.0 - u01();  // (0, 1]
        raw[static_cast<size_t>(u)] = std::min(static_cast<double>(n), 20.0 * std::pow(x, -1.0 / 0.6));
    }
    // rescale the excess over the minimum so the degrees sum to `total`
    double excess = 0.0;
    for (double d : raw) excess += d - 20.0;
    const double want = static_cast<double>(total - 20 * m);
    std::vector<i64> deg(static_cast<size_t>(m));
    i64 sum = 0;
    for (i64 u = 0; u < m; ++u) {
        const double d = 20.0 + (raw[static_cast<size_t>(u)] - 20.0) * want / excess;
        deg[static_cast<size_t>(u)] = std::min<i64>(n, std::max<i64>(20, static_cast<i64>(std::floor(d))));
        sum += deg[static_cast<size_t>(u)];
    }
    for (i64 u = 0; sum != total; u = (u + 1) % m) {  // deterministic remainder fix
        i64& d = deg[static_cast<size_t>(u)];
        if (sum < total && d < n) {
            ++d;
            ++sum;
        } else if (sum > total && d > 20) {
            --d;
            --sum;
        }
    }
    // Zipf(1.1) weights over a random item order
    std::vector<i64> perm(static_cast<size_t>(n));
    for (i64 j = 0; j < n; ++j) perm[static_cast<size_t>(j)] = j;
    for (i64 j = n - 1; j > 0; --j) std::swap(perm[static_cast<size_t>(j)], perm[bounded(rng, static_cast<u64>(j + 1))]);
    std::vector<double> wgt(static_cast<size_t>(n));
    for (i64 j = 0; j < n; ++j) wgt[static_cast<size_t>(perm[static_cast<size_t>(j)])] = std::pow(static_cast<double>(j + 1), -1.1);
    // latent factors
    const auto Uf = gaussian_cm(m, rank, derive_seed_u(seed, 2));
    const auto Vf = gaussian_cm(n, rank, derive_seed_u(seed, 3));
    std::vector<i64> off(static_cast<size_t>(m + 1), 0);
    for (i64 u = 0; u < m; ++u) off[static_cast<size_t>(u + 1)] = off[static_cast<size_t>(u)] + deg[static_cast<size_t>(u)];
    tr.m = m;
    tr.n = n;
    tr.r.resize(static_cast<size_t>(total));
    tr.c.resize(static_cast<size_t>(total));
    tr.v.resize(static_cast<size_t>(total));
    const u64 base_items = derive_seed_u(seed, 4), base_noise = derive_seed_u(seed, 5);
    parallel_for(m, [&](i64 a, i64 b) {
        std::vector<std::pair<double, i64>> keys;
        for (i64 u = a; u < b; ++u) {
            const i64 d = deg[static_cast<size_t>(u)];
            std::mt19937_64 ir(derive_seed_u(base_items, static_cast<u64>(u)));
            std::vector<i64> items;
            items.reserve(static_cast<size_t>(d));
            if (d * 4 >= n) {
                keys.resize(static_cast<size_t>(n));
                for (i64 j = 0; j < n; ++j) {
                    const double x = 1.0 - static_cast<double>(ir() >> 11) * 0x1.0p-53;
                    keys[static_cast<size_t>(j)] = {-std::log(x) / wgt[static_cast<size_t>(j)], j};
                }
                std::nth_element(keys.begin(), keys.begin() + d, keys.end());
                for (i64 q = 0; q < d; ++q) items.push_back(keys[static_cast<size_t>(q)].second);
            } else {
                // sequential weighted draws rejecting repeats == successive
                // sampling without replacement
                static thread_local std::vector<double> cdf;
                if (static_cast<i64>(cdf.size()) != n) {
                    cdf.resize(static_cast<size_t>(n));
                    double acc = 0.0;
                    for (i64 j = 0; j < n; ++j) cdf[static_cast<size_t>(j)] = (acc += wgt[static_cast<size_t>(j)]);
                }
                std::unordered_set<i64> seen;
                seen.reserve(static_cast<size_t>(2 * d));
                while (static_cast<i64>(items.size()) < d) {
                    const double x = static_cast<double>(ir() >> 11) * 0x1.0p-53 * cdf.back();
                    const i64 j = static_cast<i64>(std::upper_bound(cdf.begin(), cdf.end(), x) - cdf.begin());
                    const i64 jj = std::min(j, n - 1);
                    if (seen.insert(jj).second) items.push_back(jj);
                }
            }
            std::sort(items.begin(), items.end());
            Gauss noise(derive_seed_u(base_noise, static_cast<u64>(u)));
            for (i64 q = 0; q < d; ++q) {
                const i64 j = items[static_cast<size_t>(q)];
                double s = 3.5;
                for (int t = 0; t < rank; ++t)
                    s += fsd * fsd * Uf[static_cast<size_t>(u + t * m)] * Vf[static_cast<size_t>(j + t * n)];
                s += 0.5 * noise.next();
                double v;
                if (half_star)
                    v = std::clamp(std::round(2.0 * s) / 2.0, 0.5, 5.0);
                else
                    v = std::clamp(std::round(s), 1.0, 5.0);
                const size_t k = static_cast<size_t>(off[static_cast<size_t>(u)] + q);
                tr.r[k] = u;
                tr.c[k] = j;
                tr.v[k] = v;
            }
        }
    });
}

// split_ratings (io.hpp:474-495): a seeded shuffle, the first
// floor(0.9 ns) triples train, the rest test
void split(const Triples& all, double frac, u64 seed, Triples& train, Triples& test) {
    const u64 ns = static_cast<u64>(all.size());
    const u64 n_train = static_cast<u64>(std::floor(frac * static_cast<double>(ns) + 1e-9));
    const auto order = sample_positions(ns, ns, seed);
    train.m = test.m = all.m;
    train.n = test.n = all.n;
    for (u64 k = 0; k < ns; ++k) {
        Triples& t = (k < n_train) ? train : test;
        const u64 o = order[k];
        t.r.push_back(all.r[o]);
        t.c.push_back(all.c[o]);
        t.v.push_back(all.v[o]);
    }
}

// config 5: m = n = 1e5, rank 50, M = L R^T / sqrt(50); every row samples
// its columns uniformly without replacement (Floyd) with a per-row count from
// the normal approximation of Binomial(n, 0.01) (~1e8 entries in total; the
// reference's m*n-index sampler would need 80 GB, io.hpp:100-113).
void gen_config5(u64 seed, i64& m, i64& n, std::vector<i64>& rowptr, std::vector<i64>& col, std::vector<double>& val) {
    m = 100000;
    n = 100000;
    const int r = 50;
    const double p = 0.01;
    const auto L = gaussian_cm(m, r, derive_seed_u(seed, 1));
    const auto R = gaussian_cm(n, r, derive_seed_u(seed, 2));
    // row-major copies for the dot products
    std::vector<double> Lr(static_cast<size_t>(m * r)), Rr(static_cast<size_t>(n * r));
    for (i64 i = 0; i < m; ++i)
        for (int q = 0; q < r; ++q) Lr[static_cast<size_t>(i * r + q)] = L[static_cast<size_t>(i + q * m)];
    for (i64 j = 0; j < n; ++j)
        for (int q = 0; q < r; ++q) Rr[static_cast<size_t>(j * r + q)] = R[static_cast<size_t>(j + q * n)];
    Gauss cg(derive_seed_u(seed, 3));
    rowptr.assign(static_cast<size_t>(m + 1), 0);
    const double mu = static_cast<double>(n) * p, sd = std::sqrt(static_cast<double>(n) * p * (1.0 - p));
    for (i64 i = 0; i < m; ++i) {
        const i64 cnt = std::clamp<i64>(static_cast<i64>(std::llround(mu + sd * cg.next())), 0, n);
        rowptr[static_cast<size_t>(i + 1)] = rowptr[static_cast<size_t>(i)] + cnt;
    }
    const i64 nnz = rowptr[static_cast<size_t>(m)];
    col.resize(static_cast<size_t>(nnz));
    val.resize(static_cast<size_t>(nnz));
    const u64 base = derive_seed_u(seed, 4);
    const double scale = 1.0 / std::sqrt(static_cast<double>(r));
    parallel_for(m, [&](i64 a, i64 b) {
        std::unordered_set<i64> s;
        std::vector<i64> cols;
        for (i64 i = a; i < b; ++i) {
            const i64 k = rowptr[static_cast<size_t>(i + 1)] - rowptr[static_cast<size_t>(i)];
            std::mt19937_64 rng(derive_seed_u(base, static_cast<u64>(i)));
            s.clear();
            s.reserve(static_cast<size_t>(2 * k));
            cols.clear();
            for (i64 j = n - k; j < n; ++j) {  // Floyd's algorithm
                const i64 t = static_cast<i64>(bounded(rng, static_cast<u64>(j + 1)));
                if (s.insert(t).second)
                    cols.push_back(t);
                else {
                    s.insert(j);
                    cols.push_back(j);
                }
            }
            std::sort(cols.begin(), cols.end());
            const i64 o = rowptr[static_cast<size_t>(i)];
            const double* li = Lr.data() + i * r;
            for (i64 q = 0; q < k; ++q) {
                const i64 j = cols[static_cast<size_t>(q)];
                const double* rj = Rr.data() + j * r;
                double acc = 0.0;
                for (int t = 0; t < r; ++t) acc += li[t] * rj[t];
                col[static_cast<size_t>(o + q)] = j;
                val[static_cast<size_t>(o + q)] = acc * scale;
            }
        }
    });
}

std::mutex g_cache_mu;
struct Cache {
    int config = -1;
    u64 seed = 0;
    Triples train, test;
    std::vector<i64> rowptr, col;
    std::vector<double> val;
    i64 m = 0, n = 0;
} g_cache;

void build(int config, u64 seed) {
    if (g_cache.config == config && g_cache.seed == seed) return;
    g_cache = Cache{};
    Triples all;
    switch (config) {
        case 1:
            gen_config1(seed, g_cache.train);
            break;
        case 2:
            gen_config2(seed, g_cache.train);
            break;
        case 3:
            gen_ratings(seed, 6040, 3706, 1000209, 10, 0.35, false, all);
            split(all, 0.9, derive_seed_u(seed, 6), g_cache.train, g_cache.test);
            break;
        case 4:
            gen_ratings(seed, 69878, 10677, 10000054, 20, 0.35, true, all);
            split(all, 0.9, derive_seed_u(seed, 6), g_cache.train, g_cache.test);
            break;
        case 5:
            gen_config5(seed, g_cache.m, g_cache.n, g_cache.rowptr, g_cache.col, g_cache.val);
            break;
        default:
            throw std::invalid_argument("synth: config must be 1..5");
    }
    g_cache.config = config;
    g_cache.seed = seed;
}

}  // namespace

void synth_config(int config, u64 seed, i64* m, i64* n, i64* nnz_train, i64* nnz_test, i64* train_rows,
                  i64* train_cols, double* train_vals, i64* test_rows, i64* test_cols, double* test_vals) {
    if (config == 5) throw std::invalid_argument("synth: config 5 is generated as CSR (svt_synth_config_csr)");
    std::lock_guard<std::mutex> lk(g_cache_mu);
    build(config, seed);
    const Triples& tr = g_cache.train;
    const Triples& te = g_cache.test;
    if (m) *m = tr.m;
    if (n) *n = tr.n;
    if (nnz_train) *nnz_train = tr.size();
    if (nnz_test) *nnz_test = te.size();
    if (train_rows) std::memcpy(train_rows, tr.r.data(), sizeof(i64) * tr.r.size());
    if (train_cols) std::memcpy(train_cols, tr.c.data(), sizeof(i64) * tr.c.size());
    if (train_vals) std::memcpy(train_vals, tr.v.data(), sizeof(double) * tr.v.size());
    if (test_rows && te.size()) std::memcpy(test_rows, te.r.data(), sizeof(i64) * te.r.size());
    if (test_cols && te.size()) std::memcpy(test_cols, te.c.data(), sizeof(i64) * te.c.size());
    if (test_vals && te.size()) std::memcpy(test_vals, te.v.data(), sizeof(double) * te.v.size());
}

void synth_config_csr(int config, u64 seed, i64* m, i64* n, i64* nnz, i64* rowptr, i64* col, double* val) {
    if (config != 5) throw std::invalid_argument("synth: only config 5 is generated as CSR");
    std::lock_guard<std::mutex> lk(g_cache_mu);
    build(config, seed);
    if (m) *m = g_cache.m;
    if (n) *n = g_cache.n;
    if (nnz) *nnz = static_cast<i64>(g_cache.val.size());
    if (rowptr) std::memcpy(rowptr, g_cache.rowptr.data(), sizeof(i64) * g_cache.rowptr.size());
    if (col) std::memcpy(col, g_cache.col.data(), sizeof(i64) * g_cache.col.size());
    if (val) std::memcpy(val, g_cache.val.data(), sizeof(double) * g_cache.val.size());
}

// --- the reference's experiment generators (synth.hpp), used by the CLI -----

// synth.hpp:21-28: G1 G2^T / sqrt(rank), column-major m x n
std::vector<double> make_low_rank_cm(i64 m, i64 n, i64 rank, u64 seed) {
    if (rank < 1 || rank > std::min(m, n)) throw std::invalid_argument("make_low_rank: rank out of range");
    const std::vector<double> G1 = gaussian_cm(m, rank, derive_seed_u(seed, 0));
    const std::vector<double> G2 = gaussian_cm(n, rank, derive_seed_u(seed, 1));
    const double s = std::sqrt(static_cast<double>(rank));
    std::vector<double> A(static_cast<size_t>(m * n));
    parallel_for(n, [&](i64 j0, i64 j1) {
        for (i64 j = j0; j < j1; ++j)
            for (i64 i = 0; i < m; ++i) {
                double acc = 0.0;
                for (i64 k = 0; k < rank; ++k) acc += G1[static_cast<size_t>(i + k * m)] * G2[static_cast<size_t>(j + k * n)];
                A[static_cast<size_t>(i + j * m)] = acc / s;
            }
    });
    return A;
}

// synth.hpp:64-84: exactly floor(fraction m n) uniformly drawn cells
void sample_dense(i64 m, i64 n, const double* A_cm, double fraction, u64 seed, std::vector<i64>& r,
                  std::vector<i64>& c, std::vector<double>& v) {
    if (!(fraction > 0.0 && fraction <= 1.0)) throw std::invalid_argument("sample_dense: fraction must lie in (0, 1]");
    const u64 total = static_cast<u64>(m) * static_cast<u64>(n);
    const u64 ns = static_cast<u64>(std::floor(fraction * static_cast<double>(total) + 1e-9));
    if (ns < 1) throw std::invalid_argument("sample_dense: fraction selects no entries");
    r.clear(), c.clear(), v.clear();
    for (u64 pos : sample_positions(total, ns, seed)) {
        const i64 i = static_cast<i64>(pos / static_cast<u64>(n)), j = static_cast<i64>(pos % static_cast<u64>(n));
        r.push_back(i);
        c.push_back(j);
        v.push_back(A_cm[static_cast<size_t>(i + j * m)]);
    }
}

// synth.hpp:89-114: sum of rank-1 sine-profile products, rescaled to
// [0, 255], rounded and clamped (io.hpp:367-381); row-major pixels
std::vector<unsigned char> synthetic_image(i64 size, i64 rank, u64 seed) {
    if (size < 2 || rank < 1 || rank > size) throw std::invalid_argument("synthetic_image: bad size/rank");
    Gauss stream(derive_seed_u(seed, 2));
    const double pi = 3.14159265358979323846;
    auto profile = [&](int term) {
        std::vector<double> v(static_cast<size_t>(size));
        const double freq = 0.5 + 0.35 * static_cast<double>(term) + 0.25 * std::abs(stream.next());
        const double phase = pi * stream.next();
        for (i64 i = 0; i < size; ++i) {
            const double x = static_cast<double>(i) / static_cast<double>(size - 1);
            v[static_cast<size_t>(i)] = std::sin(2.0 * pi * freq * x + phase);
        }
        return v;
    };
    std::vector<double> M(static_cast<size_t>(size * size), 0.0);
    double weight = 1.0;
    for (i64 t = 0; t < rank; ++t, weight *= 0.8) {
        // the reference's expression evaluates its left profile first
        const std::vector<double> a = profile(static_cast<int>(t));
        const std::vector<double> b = profile(static_cast<int>(t));
        for (i64 i = 0; i < size; ++i)
            for (i64 j = 0; j < size; ++j)
                M[static_cast<size_t>(i * size + j)] += (weight * a[static_cast<size_t>(i)]) * b[static_cast<size_t>(j)];
    }
    double lo = M[0], hi = M[0];
    for (double x : M) lo = std::min(lo, x), hi = std::max(hi, x);
    const double span = (hi > lo) ? (hi - lo) : 1.0;
    std::vector<unsigned char> px(M.size());
    for (size_t k = 0; k < M.size(); ++k)
        px[k] = static_cast<unsigned char>(std::clamp(std::round(255.0 * (M[k] - lo) / span), 0.0, 255.0));
    return px;
}

// synth.hpp:119-160: 3 + U V^T + noise on a uniform cell subset, half-star
// steps clipped to [1, 5]
void synthetic_ratings(i64 users, i64 items, i64 rank, double fill, double noise, u64 seed, std::vector<i64>& r,
                       std::vector<i64>& c, std::vector<double>& v) {
    if (users < 1 || items < 1 || rank < 1 || rank > std::min(users, items))
        throw std::invalid_argument("synthetic_ratings: bad dimensions/rank");
    if (!(fill > 0.0 && fill <= 1.0)) throw std::invalid_argument("synthetic_ratings: fill must lie in (0, 1]");
    std::vector<double> U = gaussian_cm(users, rank, derive_seed_u(seed, 0));
    const double sr = std::sqrt(static_cast<double>(rank));
    for (double& x : U) x /= sr;
    const std::vector<double> V = gaussian_cm(items, rank, derive_seed_u(seed, 1));
    Gauss noise_stream(derive_seed_u(seed, 2));
    const u64 total = static_cast<u64>(users) * static_cast<u64>(items);
    const u64 ns = static_cast<u64>(std::floor(fill * static_cast<double>(total) + 1e-9));
    if (ns < 2) throw std::invalid_argument("synthetic_ratings: fill selects fewer than 2 cells");
    r.clear(), c.clear(), v.clear();
    for (u64 pos : sample_positions(total, ns, derive_seed_u(seed, 3))) {
        const i64 u = static_cast<i64>(pos / static_cast<u64>(items)), i = static_cast<i64>(pos % static_cast<u64>(items));
        double dot = 0.0;
        for (i64 k = 0; k < rank; ++k) dot += U[static_cast<size_t>(u + k * users)] * V[static_cast<size_t>(i + k * items)];
        double x = 3.0 + dot + noise * noise_stream.next();
        x = std::round(x * 2.0) / 2.0;
        x = std::clamp(x, 1.0, 5.0);
        r.push_back(u);
        c.push_back(i);
        v.push_back(x);
    }
}

// the partial Fisher-Yates sampler for the formats module (io.cpp)
std::vector<u64> sample_positions_exported(u64 total, u64 ns, u64 seed) { return sample_positions(total, ns, seed); }

}  // namespace svtb
