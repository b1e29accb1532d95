// Counter-parallel Gaussian generator that reproduces the reference RNG stream.
//
// Reference: RngStream (/root/reference/proj/src/rng.cpp:28-79): xoshiro256**
// seeded through SplitMix64 (rng.cpp:12-34), next_u64 (rng.cpp:36-47), and a
// trigonometric Box-Muller transform with a one-value cache (rng.cpp:53-66)
// that persists across gaussian() calls; gaussian(rows, cols) fills column-major
// (rng.cpp:72-79). Gaussian number g of a stream is therefore a pure function of
// the u64 pair (2*floor(g/2), 2*floor(g/2)+1) and the parity of g.
//
// B200 design: xoshiro256's state transition T is linear over GF(2), so the state
// at u64 index u is T^u * s0. The host precomputes T^(2^k) (k < 64) once, jumps the
// call's base state, and keeps on the device nibble lookup tables of T^(d*16^(pos+1))
// (6 hex positions x 15 digits, 2.9 MB); every thread derives its own start state with
// one 64-lookup mat-vec per non-zero hex digit of its global index (<= 6, no barriers)
// and runs the generator over 8 pairs. The integer stream is bit-identical to the
// reference; log/sin/cos come from CUDA's libdevice.

#include <algorithm>
#include <array>
#include <cstring>
#include <mutex>
#include <vector>

#include "rng.cuh"

namespace qbgpu {

namespace {

constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

inline std::uint64_t splitmix_next(std::uint64_t& x) {
    std::uint64_t z = (x += kGolden);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__host__ __device__ inline std::uint64_t rotl64(std::uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

// One xoshiro256** step; returns the output, advances s.
__host__ __device__ inline std::uint64_t xoshiro_next(std::uint64_t (&s)[4]) {
    const std::uint64_t result = rotl64(s[1] * 5, 7) * 9;
    const std::uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

// GF(2) 256x256 matrix as 256 columns of 4 words: col c = M * e_c.
using Mat256 = std::vector<std::uint64_t>;  // 256*4

void matvec_host(const Mat256& m, const std::uint64_t (&v)[4], std::uint64_t (&out)[4]) {
    std::uint64_t r[4] = {0, 0, 0, 0};
    for (int c = 0; c < 256; ++c) {
        if ((v[c >> 6] >> (c & 63)) & 1ULL) {
            const std::uint64_t* col = &m[c * 4];
            r[0] ^= col[0]; r[1] ^= col[1]; r[2] ^= col[2]; r[3] ^= col[3];
        }
    }
    std::memcpy(out, r, sizeof(r));
}

Mat256 matmul_host(const Mat256& a, const Mat256& b) {  // a * b
    Mat256 c(256 * 4);
    for (int j = 0; j < 256; ++j) {
        std::uint64_t col[4] = {b[j * 4], b[j * 4 + 1], b[j * 4 + 2], b[j * 4 + 3]};
        std::uint64_t out[4];
        matvec_host(a, col, out);
        std::memcpy(&c[j * 4], out, sizeof(out));
    }
    return c;
}

const std::vector<std::uint64_t>& jump_tables_host() {
    static std::vector<std::uint64_t> tables;
    static std::once_flag once;
    std::call_once(once, [] {
        Mat256 t(256 * 4);
        for (int c = 0; c < 256; ++c) {
            std::uint64_t s[4] = {0, 0, 0, 0};
            s[c >> 6] = 1ULL << (c & 63);
            xoshiro_next(s);
            std::memcpy(&t[c * 4], s, sizeof(s));
        }
        tables.resize(static_cast<std::size_t>(kJumpLevels) * 256 * 4);
        Mat256 cur = t;
        for (int k = 0; k < kJumpLevels; ++k) {
            std::memcpy(&tables[static_cast<std::size_t>(k) * 1024], cur.data(), 1024 * 8);
            if (k + 1 < kJumpLevels) cur = matmul_host(cur, cur);
        }
    });
    return tables;
}

// ---------------------------------------------------------------------------------
constexpr int kGenThreads = 256;
constexpr int kMinPairsPerThread = 8; // thread g starts at u64 offset 2 * ppt * g = 16 * (g * ppt / 8)
constexpr int kDigitPositions = 6;    // hex digits of the global thread index (16^6 threads)

// Nibble ("four Russians") table of a GF(2) 256x256 matrix M: entry [p][v] is the XOR of
// the columns of M selected by nibble value v at nibble position p (64 x 16 x 4 words =
// 32 KB). y = M x is 64 independent 32-byte lookups.
__device__ __forceinline__ void nib_matvec(const std::uint64_t* __restrict__ tab, std::uint64_t& s0,
                                           std::uint64_t& s1, std::uint64_t& s2, std::uint64_t& s3) {
    std::uint64_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll
    for (int p = 0; p < 64; ++p) {
        const std::uint64_t w = p < 16 ? s0 : (p < 32 ? s1 : (p < 48 ? s2 : s3));
        const unsigned v = static_cast<unsigned>(w >> ((p & 15) * 4)) & 15u;
        const ulonglong2* e = reinterpret_cast<const ulonglong2*>(tab + (p * 16 + v) * 4);
        const ulonglong2 lo = __ldg(e), hi = __ldg(e + 1);
        r0 ^= lo.x; r1 ^= lo.y; r2 ^= hi.x; r3 ^= hi.y;
    }
    s0 = r0; s1 = r1; s2 = r2; s3 = r3;
}

struct GenArgs {
    std::uint64_t s0[4];       // state at u64 index 2 * floor(g0 / 2) (jumped on the host)
    std::uint64_t g0;          // first gaussian index written
    std::int64_t count;        // gaussians written
    std::int64_t rows;         // output matrix rows (column-major fill order)
    int ppt;                   // pairs per thread (power of two >= 8)
    std::int64_t e_off;        // output element index of gaussian g0
    MatView out;
};

// Thread g (global index) starts at u64 offset 16 g from the call's base state: one
// table mat-vec T^(d * 16^(pos+1)) per non-zero hex digit d of g (<= 6, independent of
// any other thread: no shared memory, no barrier), then 8 sequential Box-Muller pairs.
__global__ void __launch_bounds__(kGenThreads)
gaussian_kernel(GenArgs a, const std::uint64_t* __restrict__ dig) {
    const std::uint64_t gt = static_cast<std::uint64_t>(blockIdx.x) * kGenThreads + threadIdx.x;
    const std::uint64_t unit = gt * static_cast<std::uint64_t>(a.ppt / kMinPairsPerThread);  // in 16-u64 units
    std::uint64_t s0 = a.s0[0], s1 = a.s0[1], s2 = a.s0[2], s3 = a.s0[3];
#pragma unroll 1
    for (int pos = 0; pos < kDigitPositions; ++pos) {
        const unsigned d = static_cast<unsigned>(unit >> (4 * pos)) & 15u;
        if (d) nib_matvec(dig + static_cast<std::size_t>(pos * 15 + d - 1) * 4096, s0, s1, s2, s3);
    }
    std::uint64_t s[4] = {s0, s1, s2, s3};
    const std::uint64_t p_first = a.g0 >> 1;
    const std::uint64_t g_end = a.g0 + static_cast<std::uint64_t>(a.count);  // exclusive
    const std::uint64_t pair0 = p_first + gt * static_cast<std::uint64_t>(a.ppt);
    constexpr double kTwoPi = 2.0 * 3.141592653589793;  // (2.0 * pi) as in rng.cpp:63
#pragma unroll 1
    for (int q = 0; q < a.ppt; ++q) {
        const std::uint64_t p = pair0 + q;
        const std::uint64_t g = 2 * p;
        if (g >= g_end) break;
        const std::uint64_t x1 = xoshiro_next(s);
        const std::uint64_t x2 = xoshiro_next(s);
        const double u1 = static_cast<double>((x1 >> 11) + 1) * 0x1.0p-53;
        const double u2 = static_cast<double>(x2 >> 11) * 0x1.0p-53;
        const double r = sqrt(-2.0 * log(u1));
        const double theta = __dmul_rn(kTwoPi, u2);
        double sn, cs;
        sincos(theta, &sn, &cs);
        if (g >= a.g0) {
            const std::int64_t e = a.e_off + static_cast<std::int64_t>(g - a.g0);
            *a.out.at(e % a.rows, e / a.rows) = __dmul_rn(r, cs);
        }
        if (g + 1 >= a.g0 && g + 1 < g_end) {
            const std::int64_t e = a.e_off + static_cast<std::int64_t>(g + 1 - a.g0);
            *a.out.at(e % a.rows, e / a.rows) = __dmul_rn(r, sn);
        }
    }
}

}  // namespace

void stream_origin(std::uint64_t seed, std::uint64_t stream, std::uint64_t (&s)[4]) {
    std::uint64_t x = seed;
    const std::uint64_t base = splitmix_next(x);
    std::uint64_t y = base + stream * kGolden;
    for (auto& w : s) w = splitmix_next(y);
}

std::uint64_t host_next_u64(std::uint64_t (&s)[4]) { return xoshiro_next(s); }

const std::uint64_t* RngTables::device() {
    if (!dev_) {
        // digit tables: for hex position pos (thread-index digit) and value d = 1..15, the
        // nibble table of T^(d * 16^(pos+1)) (a thread covers 16 u64).
        const auto& h = jump_tables_host();
        auto level = [&](int k) { return Mat256(h.begin() + static_cast<std::size_t>(k) * 1024,
                                                h.begin() + static_cast<std::size_t>(k + 1) * 1024); };
        std::vector<std::uint64_t> tabs(static_cast<std::size_t>(kDigitPositions) * 15 * 4096);
        for (int pos = 0; pos < kDigitPositions; ++pos) {
            Mat256 m;
            for (int d = 1; d <= 15; ++d) {
                // T^(d * 2^(4 + 4 pos)) = T^(2^(4+4pos)) * T^((d-1) * 2^(4+4pos))
                m = d == 1 ? level(4 + 4 * pos) : matmul_host(level(4 + 4 * pos), m);
                std::uint64_t* t = &tabs[static_cast<std::size_t>(pos * 15 + d - 1) * 4096];
                for (int p = 0; p < 64; ++p)
                    for (int v = 0; v < 16; ++v) {
                        std::uint64_t r[4] = {0, 0, 0, 0};
                        for (int bit = 0; bit < 4; ++bit)
                            if ((v >> bit) & 1) {
                                const std::uint64_t* col = &m[(p * 4 + bit) * 4];
                                for (int w = 0; w < 4; ++w) r[w] ^= col[w];
                            }
                        std::memcpy(t + (p * 16 + v) * 4, r, sizeof(r));
                    }
            }
        }
        QB_CUDA(cudaMalloc(&dev_, tabs.size() * sizeof(std::uint64_t)));
        QB_CUDA(cudaMemcpy(dev_, tabs.data(), tabs.size() * sizeof(std::uint64_t), cudaMemcpyHostToDevice));
    }
    return dev_;
}

RngTables::~RngTables() {
    if (dev_) cudaFree(dev_);
}

namespace {
void gaussian_chunk(cudaStream_t st, RngTables& tables, std::uint64_t seed, std::uint64_t stream, std::uint64_t g0,
                    std::int64_t count, std::int64_t e_off, const MatView& out) {
    GenArgs a{};
    stream_origin(seed, stream, a.s0);
    {
        // base state of this call: T^(2 * floor(g0 / 2)) s0, jumped on the host
        const auto& tab = jump_tables_host();
        std::uint64_t e = 2 * (g0 >> 1);
        int k = 0;
        while (e) {
            if (e & 1ULL) {
                std::uint64_t y[4];
                Mat256 m(tab.begin() + static_cast<std::size_t>(k) * 1024, tab.begin() + static_cast<std::size_t>(k + 1) * 1024);
                matvec_host(m, a.s0, y);
                std::memcpy(a.s0, y, sizeof(y));
            }
            e >>= 1;
            ++k;
        }
    }
    a.g0 = g0;
    a.count = count;
    a.rows = out.rows;
    a.e_off = e_off;
    a.out = out;
    const std::uint64_t pairs = ((g0 + count - 1) >> 1) - (g0 >> 1) + 1;
    // enough threads to fill the GPU, then longer runs per thread
    int ppt = kMinPairsPerThread;
    while (ppt < 64 && pairs / static_cast<std::uint64_t>(ppt) > 40000) ppt *= 2;
    a.ppt = ppt;
    const std::uint64_t per_cta = static_cast<std::uint64_t>(kGenThreads) * ppt;
    const unsigned grid = static_cast<unsigned>((pairs + per_cta - 1) / per_cta);
    gaussian_kernel<<<grid, kGenThreads, 0, st>>>(a, tables.device());
    QB_LAUNCH_CHECK();
}
}  // namespace

void gaussian_fill(cudaStream_t st, RngTables& tables, std::uint64_t seed, std::uint64_t stream,
                   std::uint64_t g0, const MatView& out) {
    const std::int64_t count = out.rows * out.cols;
    // one launch covers < 16^6 thread-units of 8 pairs; larger requests are chunked
    const std::int64_t chunk = std::int64_t(1) << 26;  // gaussians per launch (even)
    for (std::int64_t done = 0; done < count; done += chunk) {
        const std::int64_t c = std::min(chunk, count - done);
        gaussian_chunk(st, tables, seed, stream, g0 + static_cast<std::uint64_t>(done), c, done, out);
    }
}

}  // namespace qbgpu
