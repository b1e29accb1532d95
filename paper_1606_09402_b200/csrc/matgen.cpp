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

// out[i] += alpha * (draw skip + i of RngStream(seed, stream)), i < count: the noise term
// of config 4 added in place (no count-sized temporary). alpha * g is rounded before the
// add (no FMA contraction: built without -mfma).
int qbm_gaussian_add(std::uint64_t seed, std::uint64_t stream, std::int64_t skip, std::int64_t count, double alpha,
                     double* out) {
    Rng r(seed, stream);
    for (std::int64_t i = 0; i < skip; ++i) r.normal();
    for (std::int64_t i = 0; i < count; ++i) {
        const double t = alpha * r.normal();
        out[i] += t;
    }
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
// each row holds exactly L_r distinct columns drawn from Zipf(alpha) popularity over a
// seeded column permutation WITHOUT replacement: light rows (L_r <= n/16) redraw a
// column already taken, heavy rows (n/16 < L_r < n) take the L_r largest
// Efraimidis-Spirakis keys log(u_j)/w_j over all n columns, rows with L_r = n take every
// column. So nnz = sum_r L_r exactly. Values log(1+k), k ~ Poisson(3), redrawn while
// k == 0. Pass 1 (rp == nullptr) only returns nnz (no column draws).
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
    auto row_len = [&](std::int64_t i) {
        const double lr = std::round(c * std::pow(static_cast<double>(rank_of[i]), -alpha));
        return std::max<std::int64_t>(1, std::min<std::int64_t>(n, static_cast<std::int64_t>(std::min(lr, 9.0e18))));
    };
    if (!rp) {
        std::int64_t nnz = 0;
        for (std::int64_t i = 0; i < m; ++i) nnz += row_len(i);
        return nnz;
    }
    std::vector<std::int32_t> colperm(n);
    for (std::int64_t j = 0; j < n; ++j) colperm[j] = static_cast<std::int32_t>(j);
    for (std::int64_t j = n - 1; j > 0; --j) std::swap(colperm[j], colperm[rcol.u64() % static_cast<std::uint64_t>(j + 1)]);
    // Zipf weights / CDF over popularity ranks 1..n
    std::vector<double> cdf(n), logw(n);
    double acc = 0.0;
    for (std::int64_t j = 0; j < n; ++j) {
        const double w = std::pow(static_cast<double>(j + 1), -alpha);
        logw[j] = std::log(w);
        acc += w;
        cdf[j] = acc;
    }
    for (auto& x : cdf) x /= acc;
    std::int64_t nnz = 0;
    std::vector<std::int32_t> row;
    std::vector<char> mark(n, 0);
    std::vector<std::pair<double, std::int32_t>> keys;
    rp[0] = 0;
    for (std::int64_t i = 0; i < m; ++i) {
        const std::int64_t L = row_len(i);
        row.clear();
        if (L >= n) {
            for (std::int64_t j = 0; j < n; ++j) row.push_back(static_cast<std::int32_t>(j));
        } else if (16 * L > n) {
            // weighted sampling without replacement: the L largest log(u)/w (u in (0,1])
            keys.resize(n);
            for (std::int64_t k = 0; k < n; ++k) {
                const double u = static_cast<double>((rpick.u64() >> 11) + 1) * 0x1.0p-53;
                keys[k] = {std::log(-std::log(u)) - logw[k], colperm[k]};  // ascending = largest key
            }
            std::nth_element(keys.begin(), keys.begin() + (L - 1), keys.end());
            for (std::int64_t q = 0; q < L; ++q) row.push_back(keys[q].second);
            std::sort(row.begin(), row.end());
        } else {
            while (static_cast<std::int64_t>(row.size()) < L) {
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
        nnz += static_cast<std::int64_t>(row.size());
        rp[i + 1] = nnz;
    }
    return nnz;
}

}  // extern "C"
