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
// at u64 index u is T^u * s0. Host code precomputes T^(2^k) (k < 64) once; each CTA
// jumps its anchor with a warp-cooperative GF(2) mat-vec (lanes split the 256
// input bits, XOR-butterfly combine), then the CTA's 256 threads derive their own
// starting states with an 8-level doubling scan. Each thread then runs the
// generator sequentially over kPairsPerThread pairs. The integer stream is
// bit-identical to the reference; log/sin/cos come from CUDA's libdevice.

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
constexpr int kPairsPerThread = 32;            // 64 u64 per thread => per-thread jump = t * 2^6
constexpr int kThreadJumpLevel0 = 6;           // log2(2 * kPairsPerThread)

// Warp-cooperative y = M * x for a table matrix M (global, 256 cols x 4 words).
__device__ __forceinline__ void warp_matvec(const std::uint64_t* __restrict__ m, const std::uint64_t (&x)[4],
                                            std::uint64_t (&y)[4]) {
    const int lane = threadIdx.x & 31;
    std::uint64_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
    const int word = lane >> 3;              // bits [8*lane, 8*lane+8)
    const std::uint64_t bits = (x[word] >> ((lane & 7) * 8)) & 0xFFULL;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if ((bits >> k) & 1ULL) {
            const std::uint64_t* col = m + (lane * 8 + k) * 4;
            r0 ^= __ldg(col); r1 ^= __ldg(col + 1); r2 ^= __ldg(col + 2); r3 ^= __ldg(col + 3);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        r0 ^= __shfl_xor_sync(0xffffffffu, r0, o);
        r1 ^= __shfl_xor_sync(0xffffffffu, r1, o);
        r2 ^= __shfl_xor_sync(0xffffffffu, r2, o);
        r3 ^= __shfl_xor_sync(0xffffffffu, r3, o);
    }
    y[0] = r0; y[1] = r1; y[2] = r2; y[3] = r3;
}

__device__ __forceinline__ void thread_matvec(const std::uint64_t* __restrict__ m, const std::uint64_t* x,
                                              std::uint64_t* y) {
    std::uint64_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll 1
    for (int w = 0; w < 4; ++w) {
        std::uint64_t bits = x[w];
        while (bits) {
            const int b = __ffsll(static_cast<long long>(bits)) - 1;
            bits &= bits - 1;
            const std::uint64_t* col = m + (w * 64 + b) * 4;
            r0 ^= __ldg(col); r1 ^= __ldg(col + 1); r2 ^= __ldg(col + 2); r3 ^= __ldg(col + 3);
        }
    }
    y[0] = r0; y[1] = r1; y[2] = r2; y[3] = r3;
}

struct GenArgs {
    std::uint64_t s0[4];       // stream state at u64 index 0
    std::uint64_t g0;          // first gaussian index written
    std::int64_t count;        // gaussians written
    std::int64_t rows;         // output matrix rows (column-major fill order)
    MatView out;
};

// The jump matrices T^(64 * 2^j), j < 8, used by the in-CTA doubling scan are staged
// in shared memory (64 KB); the CTA anchor jumps from the call's base state (computed
// on the host) by blockIdx * 2^14 u64 steps, i.e. only the bits of blockIdx.
constexpr int kScanLevels = 8;  // 2^8 = kGenThreads
constexpr int kGenSmem = kScanLevels * 1024 * 8 + kGenThreads * 4 * 8;

__device__ __forceinline__ void smem_matvec(const std::uint64_t* m, const std::uint64_t* x, std::uint64_t* y) {
    std::uint64_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        std::uint64_t bits = x[w];
        while (bits) {
            const int b = __ffsll(static_cast<long long>(bits)) - 1;
            bits &= bits - 1;
            const std::uint64_t* col = m + (w * 64 + b) * 4;
            r0 ^= col[0]; r1 ^= col[1]; r2 ^= col[2]; r3 ^= col[3];
        }
    }
    y[0] = r0; y[1] = r1; y[2] = r2; y[3] = r3;
}

__global__ void __launch_bounds__(kGenThreads)
gaussian_kernel(GenArgs a, const std::uint64_t* __restrict__ tables) {
    extern __shared__ std::uint64_t gsm[];
    std::uint64_t* stab = gsm;                              // kScanLevels x 1024 words
    std::uint64_t (*st)[4] = reinterpret_cast<std::uint64_t (*)[4]>(gsm + kScanLevels * 1024);
    const std::uint64_t p_first = a.g0 >> 1;
    const std::uint64_t g_end = a.g0 + static_cast<std::uint64_t>(a.count);  // exclusive
    const std::uint64_t cta_pair0 = p_first + static_cast<std::uint64_t>(blockIdx.x) * kGenThreads * kPairsPerThread;
    for (int i = threadIdx.x; i < kScanLevels * 1024; i += kGenThreads)
        stab[i] = __ldg(tables + static_cast<std::size_t>(kThreadJumpLevel0) * 1024 + i);
    // CTA anchor: T^(2 * 8192 * blockIdx) * base, by warp 0 (levels 14 + bit of blockIdx).
    if (threadIdx.x < 32) {
        std::uint64_t x[4] = {a.s0[0], a.s0[1], a.s0[2], a.s0[3]};
        unsigned e = blockIdx.x;
        int k = kThreadJumpLevel0 + kScanLevels;
        while (e) {
            if (e & 1u) {
                std::uint64_t y[4];
                warp_matvec(tables + static_cast<std::size_t>(k) * 1024, x, y);
                x[0] = y[0]; x[1] = y[1]; x[2] = y[2]; x[3] = y[3];
            }
            e >>= 1;
            ++k;
        }
        if (threadIdx.x == 0) { st[0][0] = x[0]; st[0][1] = x[1]; st[0][2] = x[2]; st[0][3] = x[3]; }
    }
    __syncthreads();
    // Doubling scan: st[t] = T^(64 t) st[0].
#pragma unroll 1
    for (int j = 0; j < kScanLevels; ++j) {
        const int t = threadIdx.x;
        if (t >= (1 << j) && t < (2 << j)) smem_matvec(stab + j * 1024, st[t - (1 << j)], st[t]);
        __syncthreads();
    }
    std::uint64_t s[4] = {st[threadIdx.x][0], st[threadIdx.x][1], st[threadIdx.x][2], st[threadIdx.x][3]};
    const std::uint64_t pair0 = cta_pair0 + static_cast<std::uint64_t>(threadIdx.x) * kPairsPerThread;
    constexpr double kTwoPi = 2.0 * 3.141592653589793;  // (2.0 * pi) as in rng.cpp:63
#pragma unroll 1
    for (int q = 0; q < kPairsPerThread; ++q) {
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
            const std::int64_t e = static_cast<std::int64_t>(g - a.g0);
            *a.out.at(e % a.rows, e / a.rows) = __dmul_rn(r, cs);
        }
        if (g + 1 >= a.g0 && g + 1 < g_end) {
            const std::int64_t e = static_cast<std::int64_t>(g + 1 - a.g0);
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
        const auto& h = jump_tables_host();
        QB_CUDA(cudaMalloc(&dev_, h.size() * sizeof(std::uint64_t)));
        QB_CUDA(cudaMemcpy(dev_, h.data(), h.size() * sizeof(std::uint64_t), cudaMemcpyHostToDevice));
    }
    return dev_;
}

RngTables::~RngTables() {
    if (dev_) cudaFree(dev_);
}

void gaussian_fill(cudaStream_t st, RngTables& tables, std::uint64_t seed, std::uint64_t stream,
                   std::uint64_t g0, const MatView& out) {
    const std::int64_t count = out.rows * out.cols;
    if (count == 0) return;
    GenArgs a{};
    stream_origin(seed, stream, a.s0);
    {
        // base state of this call: T^(2 * p_first) s0, jumped on the host
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
    a.out = out;
    const std::uint64_t p_first = g0 >> 1;
    const std::uint64_t p_last = (g0 + count - 1) >> 1;
    const std::uint64_t pairs = p_last - p_first + 1;
    const std::uint64_t per_cta = static_cast<std::uint64_t>(kGenThreads) * kPairsPerThread;
    const unsigned grid = static_cast<unsigned>((pairs + per_cta - 1) / per_cta);
    static bool configured = false;
    if (!configured) {
        QB_CUDA(cudaFuncSetAttribute(gaussian_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kGenSmem));
        configured = true;
    }
    gaussian_kernel<<<grid, kGenThreads, kGenSmem, st>>>(a, tables.device());
    QB_LAUNCH_CHECK();
}

}  // namespace qbgpu
