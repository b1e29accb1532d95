// Harness-side synthetic inputs for the BASELINE configs (not the product path;
// the reference's own generator src/matgen.cpp is missing).
// Host-only C++; the RNG is this repo's own xoshiro256** + SplitMix64 +
// Box-Muller, stream-compatible with the reference RngStream
// (/root/reference/proj/src/rng.cpp:28-79) so inputs can be regenerated anywhere.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <unordered_set>
#include <vector>

namespace {

constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

struct Rng {
    std::uint64_t s[4];
    double cache = 0.0;
    bool has_cache = false;

    static std::uint64_t sm(std::uint64_t& x) {
        std::uint64_t z = (x += kGolden);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    Rng(std::uint64_t seed, std::uint64_t stream) {
        std::uint64_t x = seed;
        std::uint64_t base = sm(x);
        std::uint64_t y = base + stream * kGolden;
        for (auto& w : s) w = sm(y);
    }
    static std::uint64_t rotl(std::uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
    std::uint64_t u64() {
        const std::uint64_t r = rotl(s[1] * 5, 7) * 9;
        const std::uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl(s[3], 45);
        return r;
    }
    double uniform() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
    double normal() {
        if (has_cache) {
            has_cache = false;
            return cache;
        }
        const double u1 = static_cast<double>((u64() >> 11) + 1) * 0x1.0p-53;
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double th = 2.0 * std::numbers::pi * u2;
        cache = r * std::sin(th);
        has_cache = true;
        return r * std::cos(th);
    }
};

}  // namespace

extern "C" {

// next_gaussian() draws skip .. skip+count-1 of RngStream(seed, stream).
int qbm_gaussian(std::uint64_t seed, std::uint64_t stream, std::int64_t skip, std::int64_t count, double* out) {
    Rng r(seed, stream);
    for (std::int64_t i = 0; i < skip; ++i) r.normal();
    for (std::int64_t i = 0; i < count; ++i) out[i] = r.normal();
    return 0;
}

int qbm_u64(std::uint64_t seed, std::uint64_t stream, std::int64_t count, std::uint64_t* out) {
    Rng r(seed, stream);
    for (std::int64_t i = 0; i < count; ++i) out[i] = r.u64();
    return 0;
}

// Config 3 recipe: every row has exactly `per_row` distinct columns,
// uniform without replacement (Floyd's method on next_u64), sorted ascending; values
// next_double() in [0, 1) drawn after the row's columns. row_ptr has m+1 entries,
// col_idx/values m*per_row.
int qbm_csr_uniform(std::uint64_t seed, std::int64_t m, std::int64_t n, std::int64_t per_row, std::int64_t* rp,
                    std::int32_t* ci, double* v) {
    if (per_row > n) return 1;
    Rng r(seed, 0);
    std::vector<std::int64_t> cols;
    cols.reserve(per_row);
    std::unordered_set<std::int64_t> seen;
    rp[0] = 0;
    for (std::int64_t i = 0; i < m; ++i) {
        cols.clear();
        seen.clear();
        for (std::int64_t j = n - per_row; j < n; ++j) {
            const std::int64_t t = static_cast<std::int64_t>(r.u64() % static_cast<std::uint64_t>(j + 1));
            if (seen.count(t)) {
                seen.insert(j);
                cols.push_back(j);
            } else {
                seen.insert(t);
                cols.push_back(t);
            }
        }
        std::sort(cols.begin(), cols.end());
        const std::int64_t base = i * per_row;
        for (std::int64_t q = 0; q < per_row; ++q) {
            ci[base + q] = static_cast<std::int32_t>(cols[q]);
            v[base + q] = r.uniform();
        }
        rp[i + 1] = base + per_row;
    }
    return 0;
}

// Config 5 recipe (term-document-like, builder's choices recorded in
// DESIGN.md): row lengths L_r = clamp(round(c * rank_r^-alpha), 1, n) over a seeded
// random row permutation (rank_r = position of row r in the permutation, 1-based);
// columns drawn from Zipf(alpha) popularity over a seeded column permutation, with
// replacement then de-duplicated (so a row may end with fewer than L_r entries);
// rows with L_r >= n/2 take every column. Values log(1+k), k ~ Poisson(3), redrawn
// while k == 0. Pass 1 (rp == nullptr) only returns nnz.
std::int64_t qbm_csr_zipf(std::uint64_t seed, std::int64_t m, std::int64_t n, double alpha, double c,
                          std::int64_t* rp, std::int32_t* ci, double* v) {
    Rng rperm(seed, 1), rcol(seed, 2), rval(seed, 3), rpick(seed, 4);
    // row permutation (Fisher-Yates)
    std::vector<std::int64_t> rank_of(m);
    {
        std::vector<std::int64_t> perm(m);
        for (std::int64_t i = 0; i < m; ++i) perm[i] = i;
        for (std::int64_t i = m - 1; i > 0; --i) std::swap(perm[i], perm[rperm.u64() % static_cast<std::uint64_t>(i + 1)]);
        for (std::int64_t i = 0; i < m; ++i) rank_of[perm[i]] = i + 1;
    }
    std::vector<std::int32_t> colperm(n);
    for (std::int64_t j = 0; j < n; ++j) colperm[j] = static_cast<std::int32_t>(j);
    for (std::int64_t j = n - 1; j > 0; --j) std::swap(colperm[j], colperm[rcol.u64() % static_cast<std::uint64_t>(j + 1)]);
    // Zipf CDF over popularity ranks 1..n
    std::vector<double> cdf(n);
    double acc = 0.0;
    for (std::int64_t j = 0; j < n; ++j) {
        acc += std::pow(static_cast<double>(j + 1), -alpha);
        cdf[j] = acc;
    }
    for (auto& x : cdf) x /= acc;
    std::int64_t nnz = 0;
    std::vector<std::int32_t> row;
    std::vector<char> mark(n, 0);
    if (rp) rp[0] = 0;
    for (std::int64_t i = 0; i < m; ++i) {
        const double lr = std::round(c * std::pow(static_cast<double>(rank_of[i]), -alpha));
        const std::int64_t L = std::max<std::int64_t>(1, std::min<std::int64_t>(n, static_cast<std::int64_t>(lr)));
        row.clear();
        if (2 * L >= n) {
            for (std::int64_t j = 0; j < n; ++j) row.push_back(static_cast<std::int32_t>(j));
        } else {
            for (std::int64_t t = 0; t < L; ++t) {
                const double u = rpick.uniform();
                const std::int64_t k = std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin();
                const std::int32_t col = colperm[std::min<std::int64_t>(k, n - 1)];
                if (!mark[col]) {
                    mark[col] = 1;
                    row.push_back(col);
                }
            }
            for (auto col : row) mark[col] = 0;
            std::sort(row.begin(), row.end());
        }
        if (rp) {
            for (std::size_t q = 0; q < row.size(); ++q) {
                ci[nnz + static_cast<std::int64_t>(q)] = row[q];
                // Poisson(3) by inversion, redrawn while 0
                std::int64_t k = 0;
                do {
                    const double u = rval.uniform();
                    double p = std::exp(-3.0), cdfp = p;
                    k = 0;
                    while (u > cdfp && k < 64) {
                        ++k;
                        p *= 3.0 / static_cast<double>(k);
                        cdfp += p;
                    }
                } while (k == 0);
                v[nnz + static_cast<std::int64_t>(q)] = std::log1p(static_cast<double>(k));
            }
            rp[i + 1] = nnz + static_cast<std::int64_t>(row.size());
        }
        nnz += static_cast<std::int64_t>(row.size());
    }
    return nnz;
}

}  // extern "C"
