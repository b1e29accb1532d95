// Small dense kernels and deterministic reductions for the per-block work of
// randQB_EI / randQB_FP:
//  * sum of squares (||A||_F^2, matrix_handle.cpp:104-110 / kernels_avx2.cpp:36-53)
//  * per-column sums of squares (row norms of B_i, the indicator E -= ||B_i(j,:)||^2,
//    PAPER.md:206-220)
//  * CholQR pieces: in-CTA Cholesky of a b x b Gram with R^{-1} from the same
//    elimination, upper-triangular products (steps 9a-9b)
//  * Householder panel QR (the exact-semantics fallback of orth_qr, qr.hpp:15-18)
// All reductions use fixed partitions and fixed combination order, so results
// are bitwise reproducible.

#include <cooperative_groups.h>
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>

#include "gemm.cuh"

namespace cg = cooperative_groups;

namespace qbgpu {

namespace {

constexpr int kRedThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum with a fixed tree; result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < 32) {
        s = threadIdx.x < NT / 32 ? sh[threadIdx.x] : 0.0;
        s = warp_sum(s);
    }
    __syncthreads();
    return s;
}

__global__ void scale_kernel(MatView c, double beta) {
    pdl_wait();
    const std::int64_t total = c.rows * c.cols;
    for (std::int64_t idx = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
         idx < total; idx += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        std::int64_t i, j;
        if (c.rowmajor) { i = idx / c.cols; j = idx % c.cols; }
        else { i = idx % c.rows; j = idx / c.rows; }
        double* p = c.at(i, j);
        *p = beta == 0.0 ? 0.0 : beta * (*p);
    }
}

__global__ void copy_kernel(MatView s, MatView d) {
    pdl_wait();
    const std::int64_t total = s.rows * s.cols;
    for (std::int64_t idx = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
         idx < total; idx += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        std::int64_t i, j;
        if (d.rowmajor) { i = idx / d.cols; j = idx % d.cols; }
        else { i = idx % d.rows; j = idx / d.rows; }
        *d.at(i, j) = *s.at(i, j);
    }
}

__global__ void add_kernel(MatView s, MatView d, double alpha) {
    pdl_wait();
    const std::int64_t total = s.rows * s.cols;
    for (std::int64_t idx = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
         idx < total; idx += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        std::int64_t i, j;
        if (d.rowmajor) { i = idx / d.cols; j = idx % d.cols; }
        else { i = idx % d.rows; j = idx / d.rows; }
        *d.at(i, j) = fma(alpha, *s.at(i, j), *d.at(i, j));
    }
}

__global__ void identity_kernel(MatView c) {
    const std::int64_t total = c.rows * c.cols;
    for (std::int64_t idx = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
         idx < total; idx += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int64_t i = idx % c.rows, j = idx / c.rows;
        *c.at(i, j) = i == j ? 1.0 : 0.0;
    }
}

// Stage 1: each CTA owns a fixed set of segments (outer index s = cta, cta+G, ...);
// within a segment the lanes stride the contiguous inner dimension.
__global__ void sumsq_stage1(const double* __restrict__ p, std::int64_t outer, std::int64_t inner,
                             std::int64_t ld, double* __restrict__ partial) {
    __shared__ double sh[32];
    double acc = 0.0;
    const int gsz = gridDim.x;
    // Split each segment into pieces so that few long segments still spread over CTAs.
    const std::int64_t piece = 4096;
    const std::int64_t pieces_per_seg = (inner + piece - 1) / piece;
    const std::int64_t units = outer * pieces_per_seg;
    for (std::int64_t u = blockIdx.x; u < units; u += gsz) {
        const std::int64_t s = u / pieces_per_seg;
        const std::int64_t i0 = (u % pieces_per_seg) * piece;
        const std::int64_t i1 = min(inner, i0 + piece);
        const double* seg = p + s * ld;
        // 8 independent loads in flight per thread (a single dependent chain ran at ~2.3 TB/s)
        double a8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        std::int64_t i = i0 + threadIdx.x;
        for (; i + 7 * static_cast<std::int64_t>(blockDim.x) < i1; i += 8 * static_cast<std::int64_t>(blockDim.x)) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = __ldg(seg + i + q * static_cast<std::int64_t>(blockDim.x));
#pragma unroll
            for (int q = 0; q < 8; ++q) a8[q] = fma(v[q], v[q], a8[q]);
        }
        for (; i < i1; i += blockDim.x) {
            const double v = seg[i];
            a8[0] = fma(v, v, a8[0]);
        }
        acc += ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
    }
    const double s = block_sum<kRedThreads>(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// Contiguous operand (ld == inner): a flat grid-stride sweep with 16-byte loads, 4 in flight per
// thread (the segment/piece walk above reached only ~2.7 TB/s on the 512 MB config-2 matrix).
__global__ void __launch_bounds__(kRedThreads) sumsq_flat_stage1(const double2* __restrict__ p, std::int64_t n2,
                                                                  double* __restrict__ partial) {
    __shared__ double sh[32];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
    for (; i + 3 * stride < n2; i += 4 * stride) {
        const double2 v0 = __ldg(p + i), v1 = __ldg(p + i + stride), v2 = __ldg(p + i + 2 * stride),
                      v3 = __ldg(p + i + 3 * stride);
        a0 = fma(v0.x, v0.x, fma(v0.y, v0.y, a0));
        a1 = fma(v1.x, v1.x, fma(v1.y, v1.y, a1));
        a2 = fma(v2.x, v2.x, fma(v2.y, v2.y, a2));
        a3 = fma(v3.x, v3.x, fma(v3.y, v3.y, a3));
    }
    for (; i < n2; i += stride) {
        const double2 v = __ldg(p + i);
        a0 = fma(v.x, v.x, fma(v.y, v.y, a0));
    }
    const double s = block_sum<kRedThreads>((a0 + a1) + (a2 + a3), sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void sumsq_stage2(const double* __restrict__ partial, int n, double* out) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
    const double s = block_sum<kRedThreads>(acc, sh);
    if (threadIdx.x == 0) *out = s;
}

// Per-column sums of squares. CTA c owns rows [c*chunk, (c+1)*chunk); thread j owns
// columns j, j+blockDim, ...
__global__ void colsumsq_stage1(MatView v, std::int64_t chunk, double* __restrict__ partial) {
    pdl_wait();
    const std::int64_t r0 = blockIdx.x * chunk;
    const std::int64_t r1 = min(v.rows, r0 + chunk);
    for (std::int64_t j = threadIdx.x; j < v.cols; j += blockDim.x) {
        double a8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // 8 rows in flight per thread
        std::int64_t i = r0;
        for (; i + 8 <= r1; i += 8) {
            double x[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) x[q] = *v.at(i + q, j);
#pragma unroll
            for (int q = 0; q < 8; ++q) a8[q] = fma(x[q], x[q], a8[q]);
        }
        for (; i < r1; ++i) {
            const double x = *v.at(i, j);
            a8[0] = fma(x, x, a8[0]);
        }
        partial[blockIdx.x * v.cols + j] = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
    }
}

// One CTA per column: threads take partials tid, tid+256, ... (all loads in flight), then the
// fixed block tree (deterministic).
__global__ void __launch_bounds__(kRedThreads) colsumsq_stage2(const double* __restrict__ partial, int nblk,
                                                               std::int64_t cols, double* __restrict__ out) {
    pdl_wait();
    __shared__ double sh[32];
    const std::int64_t j = blockIdx.x;
    double s = 0.0;
    for (int c = threadIdx.x; c < nblk; c += kRedThreads) s += partial[c * cols + j];
    s = block_sum<kRedThreads>(s, sh);
    if (threadIdx.x == 0) out[j] = s;
}

constexpr int kCholThreads = 288;  // 9 warps: 8 DMMA warps + 1
constexpr double kFirstOrderDev = 1e-8;
// A panel whose Gram is within 1e-2 of the identity is what the SECOND pass of CholQR2 is handed
// anyway (it accepts up to kCholGramDevMax = 0.5): one pass with the true Cholesky factor leaves
// u kappa^2 <= 1.02 u of orthogonality loss, so such a panel takes one pass (below 1e-8 the factor
// is the first-order one, chol_tile_block).
constexpr double kOnePassDev = 1e-2;
// One CholQR pass leaves ||Q^T Q - I|| ~ u kappa(Y)^2. Where only span(Y) matters (the sketches inside
// the power iteration: the next pass multiplies them by A or A^T and re-orthonormalises), the second
// pass is skipped when that loss is <= 1e-6, kappa estimated by the diagonal ratio of R_a — the rule
// orth_wide_cholqr2 applies to randQB_FP's power-step sketches (qb.cu).
__device__ __forceinline__ bool span_pass_enough(double dmin, double dmax) {
    return dmin > 0.0 && 2.220446049250313e-16 * dmax * dmax <= 1e-6 * dmin * dmin;
}

// 1/x to full double precision: MUFU reciprocal seed + two Newton steps (no IEEE
// division slow path on the Cholesky's critical path).
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}

// 1/sqrt(x) to ~1 ulp: MUFU seed + two Newton steps (no IEEE sqrt/divide slow-path calls).
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = y * fma(-0.5 * x, y * y, 1.5);
    return y * fma(-0.5 * x, y * y, 1.5);
}

__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a0), "d"(a1), "d"(b0));
}

// ---- blocked in-CTA Cholesky + inverse (b <= 112) -----------------------------------
// G (upper triangle, b x b) is copied into shared memory W (BP x BP, BP = b rounded up to
// 16, padded with the identity). Right-looking over 16-column panels:
//   1. warp 0 factors the 16 x 16 diagonal block by symmetric elimination of [D | I] in
//      registers (lane j < 16 holds column j of D, lane 16 + j column j of I; rows move by
//      warp shuffles, no CTA barrier), giving R_pp and R_pp^{-1};
//   2. the row panel R_p,rest = R_pp^{-T} W_p,rest and 3. the trailing update
//      W_rest -= R_p,rest^T R_p,rest are DMMA (m16n8k4) tile products over all 8 warps.
// R is written out, then inverted in place block column by block column
// (Rinv[:c, c:c+16] = -Rinv[:c, :c] R[:c, c:c+16] Rinv_cc). Per 16 columns: one register
// elimination and 2 tile products, instead of 16 CTA-wide barrier steps.
// A near-identity Gram (max|G - I| <= 1e-8: every second CholQR pass / re-orthogonalisation)
// takes the first-order path R = I + F, R^{-1} = I - F, F = triu(G - I) - diag(G - I)/2.
template <int BP>
struct CholCfg {
    static constexpr int LD = BP + 4;   // = 4 mod 16 doubles: conflict-free DMMA fragment loads
    static constexpr int TLD = 20;
    static constexpr int P = BP / 16;
    static constexpr int SMEM_DOUBLES = BP * LD + BP * TLD + P * 16 * TLD + BP;
    static constexpr int SMEM = SMEM_DOUBLES * 8;
};

// C(16 mi + ., 8 ni + .) = alpha * sum_k A(16 mi + ., k) B(k, 8 ni + .) (+ C if accumulate)
// A(m, k) = a[m * am + k * ak], B(k, n) = bsrc[k * bk + n * bn], C(m, n) = c[m * cm + n], k in [k0, k1).
__device__ __forceinline__ void ct_frag(const double* a, int am, int ak, const double* bsrc, int bk, int bn, double* c,
                                        int cm, int mi, int ni, int k0, int k1, double alpha, bool accumulate) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int kk = k0; kk < k1; kk += 4) {
        const double a0 = a[(16 * mi + g) * am + (kk + t) * ak];
        const double a1 = a[(16 * mi + g + 8) * am + (kk + t) * ak];
        const double b0 = bsrc[(kk + t) * bk + (8 * ni + g) * bn];
        dmma_16x8x4(acc, a0, a1, b0);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int m = 16 * mi + g + (e >= 2 ? 8 : 0), n = 8 * ni + 2 * t + (e & 1);
        double* cp = c + m * cm + n;
        *cp = accumulate ? *cp + alpha * acc[e] : alpha * acc[e];
    }
}

// clock64 stamps of the last in-CTA Cholesky run by CTA 0 (thread 0), for the per-step
// breakdown (qbfac_gpu_test_chol_trace): 0 start, 1 loaded, 2+3p / 3+3p / 4+3p panel p
// eliminated / row panel / trailing update, 16 R written, 17+jb inverse block column jb, 31 end.
__device__ long long g_chol_trace[32];
__device__ __forceinline__ void chol_mark(int slot, bool on = true) {
    if (on && blockIdx.x == 0 && threadIdx.x == 0) g_chol_trace[slot] = clock64();
}

template <int BP, bool SRC_SHARED = false>
__device__ __forceinline__ void chol_tile_block(const double* __restrict__ gsrc, std::int64_t ldg, int b,
                                             double* __restrict__ r, double* __restrict__ rinv, std::int64_t ldr,
                                             SmallStatus* status, double* sm, bool trace = true) {
    using C = CholCfg<BP>;
    double* W = sm;                       // BP x LD, row-major; upper = G, then R, then R^{-1}
    double* Tm = W + BP * C::LD;          // BP x TLD scratch
    double* Dall = Tm + BP * C::TLD;      // P x (16 x TLD): Rinv_pp, row-major
    double* dg = Dall + C::P * 16 * C::TLD;  // diag(R)
    __shared__ double s_red[kCholThreads / 32];
    __shared__ double s_dev;
    __shared__ int s_bad;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nthr = blockDim.x;
    double dev = 0.0;
    chol_mark(0, trace);
    // column-major source: consecutive threads take consecutive rows i of one column j;
    // 8 loads in flight per thread per round
    for (int base = 0; base < BP * BP; base += 8 * nthr) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int idx = base + q * nthr + tid;
            const int j = idx / BP, i = idx - j * BP;
            if constexpr (SRC_SHARED)
                v[q] = (idx < BP * BP && i <= j && j < b) ? gsrc[i + static_cast<std::int64_t>(j) * ldg] : 0.0;
            else
                v[q] = (idx < BP * BP && i <= j && j < b) ? __ldcg(gsrc + i + static_cast<std::int64_t>(j) * ldg) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int idx = base + q * nthr + tid;
            if (idx >= BP * BP) continue;
            const int j = idx / BP, i = idx - j * BP;
            double x = v[q];
            if (i <= j && j < b) dev = fmax(dev, fabs(x - (i == j ? 1.0 : 0.0)));
            if (j >= b) x = (i == j) ? 1.0 : 0.0;
            W[i * C::LD + j] = i <= j ? x : 0.0;
        }
    }
    for (int o = 16; o > 0; o >>= 1) dev = fmax(dev, __shfl_down_sync(0xffffffffu, dev, o));
    if (lane == 0) s_red[warp] = dev;
    if (tid == 0) s_bad = -1;
    __syncthreads();
    if (tid == 0) {
        double dv = 0.0;
        for (int w = 0; w < nthr / 32; ++w) dv = fmax(dv, s_red[w]);
        s_dev = isfinite(dv) ? dv : INFINITY;
    }
    __syncthreads();
    chol_mark(1, trace);
    if (s_dev <= kFirstOrderDev) {
        for (int idx = tid; idx < b * b; idx += nthr) {
            const int i = idx % b, j = idx / b;
            double rv = 0.0, iv = 0.0;
            if (i <= j) {
                const double e = W[i * C::LD + j] - (i == j ? 1.0 : 0.0);
                rv = (i == j) ? 1.0 + 0.5 * e : e;
                iv = (i == j) ? 1.0 - 0.5 * e : -e;
                if (i == j) dg[i] = rv;
            }
            r[i + static_cast<std::int64_t>(j) * ldr] = rv;
            rinv[i + static_cast<std::int64_t>(j) * ldr] = iv;
        }
    } else {
        // not unrolled: one copy of the (fully unrolled) 16 x 16 elimination serves every panel, so
        // the instruction stream stays cache-resident (unrolled copies missed the instruction
        // cache on every call inside chol_wide: 27k clk for the first panel, 44 us per 64 x 64)
#pragma unroll 1
        for (int pnl = 0; pnl < C::P; ++pnl) {
            const int c0 = 16 * pnl, c1 = c0 + 16;
            double* Dv = Dall + pnl * 16 * C::TLD;
            if (warp == 0) {
                // [D | I] elimination, one column per lane
                const int j = lane & 15;
                const bool left = lane < 16;
                double x[16];
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    x[i] = left ? W[(c0 + min(i, j)) * C::LD + c0 + max(i, j)] : (i == j ? 1.0 : 0.0);
                double pv[16];
                // pivots past b (identity padding) are no-op steps: their column of D is e_k, so every
                // multiplier is 0 and the pivot is 1 (b = 20: 4 steps in the second panel, not 16)
                const int nval = min(16, b - c0);
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    if (k >= nval) {
                        pv[k] = 1.0;
                        continue;
                    }
                    double piv = __shfl_sync(0xffffffffu, x[k], k);
                    const bool bad = !(piv > 0.0) || !isfinite(piv);
                    if (bad) {
                        if (lane == 0 && s_bad < 0 && c0 + k < b) s_bad = c0 + k;
                        piv = 1.0;
                        if (lane == k) x[k] = 1.0;
                    }
                    pv[k] = piv;
                    const double pinv = rcp_nr(piv);
#pragma unroll
                    for (int i = k + 1; i < 16; ++i) {
                        const double f = __shfl_sync(0xffffffffu, x[i], k) * pinv;
                        x[i] = fma(-f, x[k], x[i]);
                    }
                }
                double rsq[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) rsq[k] = rsqrt_nr(pv[k]);  // independent: pipelined
                // branch-free write-out (left lanes: row k of R_pp; right lanes: R_pp^{-1}(j, k) =
                // (R_pp^{-T})(k, j) = E(k, j) / sqrt(piv_k), k >= j)
                double* wcol = W + c0 * C::LD + c0 + j;
                double* drow = Dv + j * C::TLD;
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const double sq = pv[k] * rsq[k], v = x[k] * rsq[k];
                    double* dst = left ? wcol + k * C::LD : drow + k;
                    const double val = left ? (k == j ? sq : v) : (k >= j ? v : 0.0);
                    if (!left || k <= j) *dst = val;
                    if (lane == 0) dg[c0 + k] = sq;
                }
            }
            __syncthreads();
            chol_mark(2 + 3 * pnl, trace);
            if (c1 < BP) {
                // 2. row panel (in place): W[c0+m][c1+n] = sum_k Rinv_pp(k, m) W[c0+k][c1+n]
                const int nf = (BP - c1) / 8;
                if (warp < 8)
                    for (int ni = warp; ni < nf; ni += 8)
                        ct_frag(Dv, 1, C::TLD, W + c0 * C::LD + c1, C::LD, 1, W + c0 * C::LD + c1, C::LD, 0, ni, 0, 16,
                                1.0, false);
                __syncthreads();
                chol_mark(3 + 3 * pnl, trace);
                // 3. trailing update on upper fragments: W[c1+m][c1+n] -= sum_k W[c0+k][c1+m] W[c0+k][c1+n]
                const int nb8 = (BP - c1) / 8;
                int nfu = 0;
                for (int mi = 0; mi < (BP - c1) / 16; ++mi) nfu += nb8 - 2 * mi;
                if (warp < 8)
                    for (int f = warp; f < nfu; f += 8) {
                        int e = f, mi = 0;
                        while (e >= nb8 - 2 * mi) { e -= nb8 - 2 * mi; ++mi; }
                        const int ni = 2 * mi + e;
                        ct_frag(W + c0 * C::LD + c1, 1, C::LD, W + c0 * C::LD + c1, C::LD, 1, W + c1 * C::LD + c1, C::LD,
                                mi, ni, 0, 16, -1.0, true);
                    }
                __syncthreads();
                chol_mark(4 + 3 * pnl, trace);
            }
        }
        // R out
        for (int idx = tid; idx < b * b; idx += nthr) {
            const int i = idx % b, j = idx / b;
            r[i + static_cast<std::int64_t>(j) * ldr] = i <= j ? W[i * C::LD + j] : 0.0;
        }
        __syncthreads();
        chol_mark(23, trace);
        // in-place inversion, block column by block column
#pragma unroll 1
        for (int jb = 0; jb < C::P; ++jb) {
            const int cj = 16 * jb;
            const double* Dj = Dall + jb * 16 * C::TLD;
            if (jb > 0) {
                // T[0:cj][0:16] = R[0:cj][cj:cj+16] * Rinv_jj
                const int nfr = jb * 2;
                if (warp < 8)
                    for (int f = warp; f < nfr; f += 8)
                        ct_frag(W + cj, C::LD, 1, Dj, C::TLD, 1, Tm, C::TLD, f >> 1, f & 1, 0, 16, 1.0, false);
                __syncthreads();
                // W[0:cj][cj:cj+16] = -Rinv[0:cj][0:cj] * T  (Rinv upper: k from 16 mi)
                if (warp < 8)
                    for (int f = warp; f < nfr; f += 8) {
                        const int mi = f >> 1;
                        ct_frag(W, C::LD, 1, Tm, C::TLD, 1, W + cj, C::LD, mi, f & 1, 16 * mi, cj, -1.0, false);
                    }
            }
            for (int idx = tid; idx < 256; idx += nthr) {
                const int i = idx >> 4, k = idx & 15;
                W[(cj + i) * C::LD + cj + k] = Dj[i * C::TLD + k];
            }
            __syncthreads();
            chol_mark(24 + jb, trace);
        }
        for (int idx = tid; idx < b * b; idx += nthr) {
            const int i = idx % b, j = idx / b;
            rinv[i + static_cast<std::int64_t>(j) * ldr] = i <= j ? W[i * C::LD + j] : 0.0;
        }
    }
    __syncthreads();
    if (warp == 0 && status) {
        double dmin = INFINITY, dmax = 0.0;
        for (int j = lane; j < b; j += 32) {
            dmin = fmin(dmin, dg[j]);
            dmax = fmax(dmax, dg[j]);
        }
        for (int o = 16; o > 0; o >>= 1) {
            dmin = fmin(dmin, __shfl_down_sync(0xffffffffu, dmin, o));
            dmax = fmax(dmax, __shfl_down_sync(0xffffffffu, dmax, o));
        }
        if (lane == 0) {
            status->breakdown = s_bad >= 0 ? 1 : 0;
            status->bad_index = s_bad;
            status->diag_min = dmin;
            status->diag_max = dmax;
            status->gram_dev = s_dev;
        }
    }
    __syncthreads();
    chol_mark(31, trace);
}

template <int BP>
__global__ void __launch_bounds__(kCholThreads)
chol_small_kernel(const double* __restrict__ g, std::int64_t ldg, int b, double* __restrict__ r,
                  double* __restrict__ rinv, std::int64_t ldr, SmallStatus* status) {
    extern __shared__ __align__(16) double ch_smem[];
    chol_tile_block<BP>(g, ldg, b, r, rinv, ldr, status, ch_smem);
}

// ---- blocked Cholesky + inverse of an l x l Gram in ONE cooperative launch -----------
// Right-looking over 64 x 64 tiles (nt = ceil(l/64)) of the upper triangle of W (col-major):
//   step k:  [CTA 0]  R_kk, R_kk^{-1} = chol_small_block(W_kk)          (phase 1)
//            grid.sync
//            R_kj   = R_kk^{-T} W_kj            for j > k                (phase 2, left)
//            F_pk   = F_pk R_kk^{-1}            for p < k                (phase 2, right)
//            grid.sync
//            W_ij  -= R_ki^T R_kj               for k < i <= j           (phase 3, left)
//            F_pi  -= F_pk R_ki                 for p <= k < i           (phase 3, right)
//            [CTA 0 takes only W_{k+1,k+1} and runs phase 1 of step k+1 right after it]
//            grid.sync
// F (in `rinv`, zero-initialised) ends as R^{-1}: the right half of the elimination of
// [W | I] kept transposed (F_kk = R_kk^{-1} from phase 1). Two grid barriers per step
// instead of ~5 dependent launches per 64-column panel.
// chol_wide's diagonal factorization as an out-of-line call: its own register allocation instead
// of sharing chol_wide_kernel's (the inlined copy spilled and ran ~2x slower than standalone)
template <int BP>
__device__ __noinline__ void chol_tile_block_call(const double* __restrict__ g, std::int64_t ldg, int b,
                                                  double* __restrict__ r, double* __restrict__ rinv, std::int64_t ldr,
                                                  SmallStatus* status, double* sm, bool trace = true) {
    chol_tile_block<BP>(g, ldg, b, r, rinv, ldr, status, sm, trace);
}
__device__ __forceinline__ void chol_tile_block64_call(const double* __restrict__ g, std::int64_t ldg, int b,
                                                       double* __restrict__ r, double* __restrict__ rinv,
                                                       std::int64_t ldr, SmallStatus* status, double* sm) {
    chol_tile_block_call<64>(g, ldg, b, r, rinv, ldr, status, sm);
}

constexpr int kCwNb = 64;
constexpr int kCwLd = 68;   // padded shared stride (= 4 mod 16 doubles: conflict-free fragments)
constexpr int kCwSmemBytes = 2 * kCwNb * kCwLd * 8;

// Stage a 64 x 64 operand X(u, v) = x[u*su + v*sv] (u < ur, v < vr; zero elsewhere) in
// shared memory along its contiguous global dimension. Threads 0..255 each gather 16
// elements into registers first (all loads in flight at once), then store.
__device__ __forceinline__ void cw_stage(double* s, const double* __restrict__ x, std::int64_t su,
                                         std::int64_t sv, int ur, int vr, int& ssu, int& ssv) {
    const bool u_contig = su == 1;
    ssu = u_contig ? 1 : kCwLd;
    ssv = u_contig ? kCwLd : 1;
    const int tid = threadIdx.x;
    if (tid >= 256) return;
    // thread -> fixed index `fast` along the contiguous dimension, `slow` = slow0 + 4q
    const int fast = tid & (kCwNb - 1), slow0 = tid >> 6;
    const std::int64_t s_fast = u_contig ? su : sv, s_slow = u_contig ? sv : su;
    const int lim_fast = u_contig ? ur : vr, lim_slow = u_contig ? vr : ur;
    const int ss_fast = u_contig ? ssu : ssv, ss_slow = u_contig ? ssv : ssu;
    const double* src = x + fast * s_fast + slow0 * s_slow;
    const bool fast_ok = fast < lim_fast;
    double vals[16];
#pragma unroll
    for (int q = 0; q < 16; ++q)
        vals[q] = (fast_ok && slow0 + 4 * q < lim_slow) ? __ldcg(src + 4 * q * s_slow) : 0.0;
    double* dst = s + fast * ss_fast + slow0 * ss_slow;
#pragma unroll
    for (int q = 0; q < 16; ++q) dst[4 * q * ss_slow] = vals[q];
}

// C(m, n) = alpha * sum_q A(m, q) B(q, n) + beta * C(m, n) on one 64 x 64 tile (m < mr,
// n < nc, q < kd): A(m, q) = a[m*a_sm + q*a_sq], B(q, n) = b[q*b_sq + n*b_sn], C col-major.
// Both operands are staged before any store, so C may alias A. DMMA m16n8k4, 8 warps of
// 16 x 32 outputs; the C tile is read into registers (beta != 0) before the MMAs.
__device__ __noinline__ void cw_tile_gemm(double* smem, const double* a, std::int64_t a_sm, std::int64_t a_sq, const double* b,
                             std::int64_t b_sq, std::int64_t b_sn, double* c, std::int64_t ldc, int mr, int nc,
                             int kd, double alpha, double beta) {
    double* sa = smem;
    double* sb = smem + kCwNb * kCwLd;
    int am, aq, bn, bq;
    cw_stage(sa, a, a_sm, a_sq, mr, kd, am, aq);
    cw_stage(sb, b, b_sn, b_sq, nc, kd, bn, bq);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp & 3, wn = warp >> 2;
    const int g = lane >> 2, t = lane & 3;
    double cv[4][4];
    if (warp < 8 && beta != 0.0) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int row = wm * 16 + g + (e >= 2 ? 8 : 0);
                const int col = wn * 32 + j * 8 + 2 * t + (e & 1);
                cv[j][e] = (row < mr && col < nc) ? __ldcg(c + row + static_cast<std::int64_t>(col) * ldc) : 0.0;
            }
    }
    __syncthreads();
    if (warp < 8) {
        double acc[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[j][e] = 0.0;
        const int kq = (kd + 3) & ~3;
        for (int kk = 0; kk < kq; kk += 4) {
            const int r0 = wm * 16 + g;
            const double a0 = sa[r0 * am + (kk + t) * aq];
            const double a1 = sa[(r0 + 8) * am + (kk + t) * aq];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const double bf = sb[(wn * 32 + j * 8 + g) * bn + (kk + t) * bq];
                dmma_16x8x4(acc[j], a0, a1, bf);
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int row = wm * 16 + g + (e >= 2 ? 8 : 0);
                const int col = wn * 32 + j * 8 + 2 * t + (e & 1);
                if (row < mr && col < nc) {
                    const double v = alpha * acc[j][e];
                    c[row + static_cast<std::int64_t>(col) * ldc] = beta == 0.0 ? v : v + beta * cv[j][e];
                }
            }
    }
    __syncthreads();
}

struct CholWideArgs {
    double* w;
    std::int64_t ldw;
    double* r;
    double* rinv;
    std::int64_t ldr;
    int l, nt;
    SmallStatus* stats;
};

// per-step %globaltimer stamps of CTA 0 (qbfac_gpu_test_chol_wide_trace): [k][0] step start,
// [k][1] phase 2 done, [k][2] phase 3 (CTA 0: W_{k+1,k+1} + its Cholesky) done, [k][3] step end
__device__ unsigned long long g_cw_trace[64][4];
__device__ __forceinline__ void cw_mark(int k, int slot) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && k < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_cw_trace[k][slot] = t;
    }
}

__global__ void __launch_bounds__(kCholThreads, 1) chol_wide_kernel(CholWideArgs p) {
    extern __shared__ __align__(16) double cw_smem[];
    cg::grid_group grid = cg::this_grid();
    const int G = gridDim.x, cta = blockIdx.x;
    const int nt = p.nt, l = p.l;
    auto sz = [&](int t) { return min(kCwNb, l - t * kCwNb); };
    auto W = [&](int i, int j) { return p.w + static_cast<std::int64_t>(i) * kCwNb + static_cast<std::int64_t>(j) * kCwNb * p.ldw; };
    auto R = [&](int i, int j) { return p.r + static_cast<std::int64_t>(i) * kCwNb + static_cast<std::int64_t>(j) * kCwNb * p.ldr; };
    auto F = [&](int i, int j) { return p.rinv + static_cast<std::int64_t>(i) * kCwNb + static_cast<std::int64_t>(j) * kCwNb * p.ldr; };
    // item e >= 1 of a phase -> CTA 1 + (e-1) % (G-1); item 0 (phase 3: W_{k+1,k+1}) -> CTA 0
    const int e_first = G == 1 ? 1 : cta, e_step = G == 1 ? 1 : G - 1;
    static_assert(CholCfg<64>::SMEM <= kCwSmemBytes, "chol workspace");
    if (cta == 0) chol_tile_block64_call(W(0, 0), p.ldw, sz(0), R(0, 0), F(0, 0), p.ldr, p.stats, cw_smem);
    grid.sync();
    for (int k = 0; k < nt; ++k) {
        cw_mark(k, 0);
        const int bk = sz(k);
        const int n = nt - k - 1;
        // phase 2: items 1..n left (j = k + e), n+1..n+k right (p = e - n - 1)
        for (int e = e_first; e >= 1 && e <= n + k; e += e_step) {
            if (e <= n) {
                const int j = k + e;
                // R_kj(a, c) = sum_q Rinv_kk(q, a) W_kj(q, c)
                cw_tile_gemm(cw_smem, F(k, k), p.ldr, 1, W(k, j), 1, p.ldw, R(k, j), p.ldr, bk, sz(j), bk, 1.0, 0.0);
            } else {
                const int pp = e - n - 1;
                // F_pk(a, c) = sum_q F_pk(a, q) Rinv_kk(q, c)   (in place)
                cw_tile_gemm(cw_smem, F(pp, k), 1, p.ldr, F(k, k), 1, p.ldr, F(pp, k), p.ldr, sz(pp), bk, bk, 1.0, 0.0);
            }
        }
        cw_mark(k, 1);
        grid.sync();
        if (n == 0) break;
        // phase 3: item 0 = (k+1, k+1); then the other left tiles, then the right tiles
        const int n_left = n * (n + 1) / 2;
        const int items = n_left + (k + 1) * n;
        for (int e = (G == 1 || cta == 0) ? 0 : cta; e < items; e = (G == 1) ? e + 1 : (e == 0 ? items : e + e_step)) {
            if (e < n_left) {
                // e -> (i, j), k < i <= j, enumerated row by row starting at (k+1, k+1)
                int t = e, i = k + 1;
                while (t >= nt - i) { t -= nt - i; ++i; }
                const int j = i + t;
                // W_ij(a, c) -= sum_q R_ki(q, a) R_kj(q, c)
                cw_tile_gemm(cw_smem, R(k, i), p.ldr, 1, R(k, j), 1, p.ldr, W(i, j), p.ldw, sz(i), sz(j), bk, -1.0, 1.0);
            } else {
                const int t = e - n_left;
                const int pp = t / n, i = k + 1 + t % n;
                // F_pi(a, c) -= sum_q F_pk(a, q) R_ki(q, c)
                cw_tile_gemm(cw_smem, F(pp, k), 1, p.ldr, R(k, i), 1, p.ldr, F(pp, i), p.ldr, sz(pp), sz(i), bk, -1.0, 1.0);
            }
            if (e == 0)
                chol_tile_block64_call(W(k + 1, k + 1), p.ldw, sz(k + 1), R(k + 1, k + 1), F(k + 1, k + 1), p.ldr,
                                       p.stats + k + 1, cw_smem);
        }
        cw_mark(k, 2);
        grid.sync();
        cw_mark(k, 3);
    }
}

// ---- fused CholQR2 of a tall panel in ONE cooperative launch -----------------------
// Y (rows x b, row-major) -> Q = Y Ra^{-1} Rb^{-1} with Ra = chol(Y^T Y), Rb = chol(T1^T T1),
// T1 = Y Ra^{-1}: the same arithmetic as the launch sequence Gram / chol_small / Y R^{-1}
// twice, without its 11 launches and split-K round trips. 64-row sub-tiles are staged in
// shared memory (CTA c takes sub-tiles c, c+G, ...); Grams are accumulated with DMMA on
// the upper fragments only, written per CTA and reduced over CTAs in a fixed order (so the
// result is deterministic for a given device); the b x b Choleskies run on CTA 0 between
// grid barriers. Phase B writes T1 and accumulates its Gram from the same registers.
// Sub-tiles stream through a STAGES-deep cp.async ring (~64 KB of rows in flight per SM).
// Grid-wide barrier for cooperative launches (all CTAs co-resident): an arrival counter and
// a generation word in global memory (bar[0], bar[1]; zero-initialised once per context).
// Waiting CTAs poll with __nanosleep backoff so the CTA doing serial work between barriers
// (the Cholesky on CTA 0) does not compete with a storm of polling loads.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            unsigned ns = 32;
            while (*gen == g) {
                __nanosleep(ns);
                ns = ns < 512 ? 2 * ns : 512;
            }
        }
        __threadfence();
    }
    __syncthreads();
}
// Tight-polling variant for kernels whose CTAs all wait (no CTA does serial work between
// barriers): the backoff of grid_barrier would only add wake-up latency.
__device__ __forceinline__ void grid_barrier_tight(unsigned* bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) {}
        }
        __threadfence();
    }
    __syncthreads();
}

struct PanelArgs {
    CUtensorMap tm_y;   // Y as rows x b (row stride ldy), box {BP + 4, SUB}: one TMA per sub-tile
    CUtensorMap tm_t1;  // T1 as rows x b (row stride b)
    int use_tm_y, use_tm_t1;
    const double* y;
    std::int64_t ldy;
    double* t1;  // rows x b, ld b
    double* q;
    std::int64_t ldq;
    std::int64_t rows;
    int b, nsub;
    double* part;  // gridDim.x x BP x BP partial Grams
    double* g;     // b x b Gram (ld kSmallMax)
    double *ra, *rainv, *rb, *rbinv;  // ld kSmallMax
    SmallStatus *st0, *st1;
    unsigned* gbar;  // grid barrier words
    int nstages;     // sub-tile ring depth (<= PanelCfg<BP>::STAGES; fewer -> 2 CTAs per SM)
    int span_only;   // the caller needs span(Y) only (a power-iteration sketch): stop after the first
                     // pass when its loss of orthogonality u kappa^2 (kappa from diag(R_a)) is <= 1e-6
};

template <int BP>
struct PanelCfg {
    static constexpr int SUB = BP >= 96 ? 32 : 64;  // rows per sub-tile
    static constexpr int LD = BP + 4;               // = 4 mod 16 doubles (BP multiple of 16)
    static constexpr int MI = SUB / 16;             // m16 blocks per sub-tile
    static constexpr int NG = 8 / MI;               // warps sharing one m16 block
    static constexpr int NFG = (BP / 16) * (BP / 8) - (BP / 16) * (BP / 16 - 1);  // upper Gram fragments
    static constexpr int MAXG = (NFG + 7) / 8;
    static constexpr int MAXT = (BP / 8 + NG - 1) / NG;  // product fragments per warp: mi = w % MI, ni = w / MI + NG j
    // independent accumulator chains per fragment along k (the FP64 MMA pipe needs ~40
    // MMAs in flight per SM to cover its latency)
    static constexpr int KSG = MAXG >= 5 ? 1 : (MAXG >= 3 ? 2 : 4);
    static constexpr int KST = (MAXT >= 5 || BP >= 96) ? 1 : 2;  // wide panels: registers go to the Gram fragments
    // sub-tile copies in flight: as many as fit next to the triangular factor (~64 KB of rows)
    static constexpr int STAGES = (4 * SUB + BP) * LD * 8 <= 220 * 1024 ? 4 : 3;
    static constexpr int SMEM = (STAGES * SUB + BP) * LD * 8;
};

// Panel sub-tile ring: the producer warp moves each sub-tile row (b contiguous doubles) with a
// TMA bulk copy (cp.async.bulk ... mbarrier::complete_tx, SASS UBLKCP) into the padded
// shared layout; full/empty mbarrier pairs replace the CTA-wide barriers of a cp.async ring.
__device__ __forceinline__ unsigned sm_addr(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void pb_init(std::uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sm_addr(bar)), "r"(count));
}
__device__ __forceinline__ void pb_arrive(std::uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sm_addr(bar)) : "memory");
}
__device__ __forceinline__ void pb_arrive_tx(std::uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void pb_wait(std::uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "PB_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra PB_WAIT_%=;\n"
        "}\n" ::"r"(sm_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void pb_bulk(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(sm_addr(dst)),
        "l"(src), "r"(bytes), "r"(sm_addr(bar))
        : "memory");
}
__device__ __forceinline__ void pb_fence_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// named barrier over the 8 DMMA (consumer) warps only
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }

// acc += Ys^T Ys on this warp's first NV upper fragments (KSG interleaved chains along the
// rows). NV is the warp's count of valid fragments, dispatched at compile time: a predicated-off
// DMMA still occupies the FP64 tensor pipe, so invalid fragments must not be issued at all.
template <int BP, int NV>
__device__ __forceinline__ void panel_gram_n(const double* ys, double (&acc)[PanelCfg<BP>::MAXG][PanelCfg<BP>::KSG][4],
                                             const int (&fm)[PanelCfg<BP>::MAXG], const int (&fn)[PanelCfg<BP>::MAXG]) {
    using C = PanelCfg<BP>;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll 2
    for (int kk = 0; kk < C::SUB; kk += 4 * C::KSG) {
#pragma unroll
        for (int c = 0; c < C::KSG; ++c) {
            const double* row = ys + (kk + 4 * c + t) * C::LD;  // A = Ys^T: a(m, k) = Ys(k, m)
#pragma unroll
            for (int f = 0; f < NV; ++f)
                dmma_16x8x4(acc[f][c], row[16 * fm[f] + g], row[16 * fm[f] + g + 8], row[8 * fn[f] + g]);
        }
    }
}
template <int BP, int NV = PanelCfg<BP>::MAXG>
__device__ __forceinline__ void panel_gram(const double* ys, double (&acc)[PanelCfg<BP>::MAXG][PanelCfg<BP>::KSG][4],
                                           const int (&fm)[PanelCfg<BP>::MAXG], const int (&fn)[PanelCfg<BP>::MAXG],
                                           int nvf) {
    if constexpr (NV > 0) {
        if (nvf == NV) panel_gram_n<BP, NV>(ys, acc, fm, fn);
        else panel_gram<BP, NV - 1>(ys, acc, fm, fn, nvf);
    }
}

// out fragments = Ys (SUB x BP) * Rs (BP x BP, upper), mi = warp % MI, ni = warp / MI + NG j.
// Fragment by fragment with the exact triangular k range (k < 8 ni + 8): no predicated-off
// DMMAs; two interleaved chains along k, summed at the end.
template <int BP>
__device__ __forceinline__ void panel_trmm(const double* ys, const double* rs, double (&out)[PanelCfg<BP>::MAXT][4],
                                           int b) {
    using C = PanelCfg<BP>;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int mi = warp % C::MI, h = warp / C::MI;
    const int nb8 = (b + 7) >> 3, kmax = (b + 3) & ~3;
    const double* a0p = ys + (16 * mi + g) * C::LD + t;
    const double* a1p = a0p + 8 * C::LD;
    // fragments in pairs (n-blocks h + NG j and h + NG (j+1)): over the shorter triangular k range
    // both share the A-fragment loads (4 shared loads per 2 DMMAs instead of 6), the longer one
    // then continues alone; every accumulation runs in ascending k (deterministic)
#pragma unroll
    for (int jp = 0; jp < C::MAXT; jp += 2) {
        const int ni0 = h + C::NG * jp, ni1 = h + C::NG * (jp + 1);
        const bool v1 = (jp + 1 < C::MAXT) && ni1 < nb8;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            out[jp][e] = 0.0;
            if (jp + 1 < C::MAXT) out[jp + 1][e] = 0.0;
        }
        if (ni0 >= nb8) continue;  // warp-uniform; ni1 > ni0 is then invalid too
        const int kend0 = min(kmax, 8 * ni0 + 8);
        const double* bp0 = rs + t * C::LD + 8 * ni0 + g;
        double acc0[4] = {0.0, 0.0, 0.0, 0.0};
        if (v1) {
            const int kend1 = min(kmax, 8 * ni1 + 8);
            const double* bp1 = rs + t * C::LD + 8 * ni1 + g;
            double acc1[4] = {0.0, 0.0, 0.0, 0.0};
            int kk = 0;
            for (; kk < kend0; kk += 4) {
                const double x0 = a0p[kk], x1 = a1p[kk];
                dmma_16x8x4(acc0, x0, x1, bp0[kk * C::LD]);
                dmma_16x8x4(acc1, x0, x1, bp1[kk * C::LD]);
            }
            for (; kk < kend1; kk += 4) dmma_16x8x4(acc1, a0p[kk], a1p[kk], bp1[kk * C::LD]);
#pragma unroll
            for (int e = 0; e < 4; ++e) out[jp + 1][e] = acc1[e];
        } else {
            for (int kk = 0; kk < kend0; kk += 4) dmma_16x8x4(acc0, a0p[kk], a1p[kk], bp0[kk * C::LD]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) out[jp][e] = acc0[e];
    }
}

// A DMMA accumulator's column pair (2t, 2t + 1) to row-major global memory: one 16-byte store when the
// destination allows it (an 8-byte store per element touches every 32-byte sector twice).
__device__ __forceinline__ void store_col_pair(double* dst, bool vec, bool ok0, bool ok1, double v0, double v1) {
    if (vec && ok1) {
        *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
    } else {
        if (ok0) dst[0] = v0;
        if (ok1) dst[1] = v1;
    }
}

// Phase timestamps of the last panel launch (CTA 0, %globaltimer ns): read by
// qbfac_gpu_test_panel_trace for the per-phase breakdown in profiles/.
__device__ unsigned long long g_panel_trace[kPanelTraceSlots];
__device__ __forceinline__ void panel_mark(int slot) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_panel_trace[slot] = t;
    }
}

template <int BP>
__global__ void __launch_bounds__(kCholThreads, 1) cholqr2_panel_kernel(const __grid_constant__ PanelArgs p) {
    pdl_wait();
    using C = PanelCfg<BP>;
    extern __shared__ __align__(128) double psm[];
    const int NST = p.nstages;
    double* ys2 = psm;                         // NST sub-tile buffers (SUB x LD)
    double* rs = psm + NST * C::SUB * C::LD;   // BP x LD triangular factor
    __shared__ __align__(8) std::uint64_t full[C::STAGES], empty[C::STAGES];
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const bool mma_warp = warp < 8;
    const bool vec_q = (p.ldq & 1) == 0 && (reinterpret_cast<std::uintptr_t>(p.q) & 15) == 0;
    const bool vec_t1 = (p.b & 1) == 0 && (reinterpret_cast<std::uintptr_t>(p.t1) & 15) == 0;
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            pb_init(&full[s], 1);
            pb_init(&empty[s], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // The bulk copies fill columns [0, b) only. Columns [b, kmax) enter the triangular products
    // (times zero rows of R^{-1}) and must hold zeros; columns past kmax only reach discarded
    // Gram entries.
    const int kpad = ((p.b + 3) & ~3) - p.b;
    auto zero_pad = [&]() {
        for (int idx = tid; idx < NST * C::SUB * kpad; idx += blockDim.x)
            ys2[(idx / kpad) * C::LD + p.b + idx % kpad] = 0.0;
    };
    zero_pad();
    // this warp's upper Gram fragments
    int fm[C::MAXG], fn[C::MAXG];
#pragma unroll
    for (int f = 0; f < C::MAXG; ++f) {
        int e = warp + 8 * f, mi = 0;
        fm[f] = -1;
        fn[f] = 0;
        // upper fragments (mi, ni >= 2 mi) with column blocks inside b only
        const int nb8 = (p.b + 7) >> 3;
        int nf = 0;
        for (int m2 = 0; m2 < BP / 16; ++m2) nf += max(0, nb8 - 2 * m2);
        if (!mma_warp || e >= nf) continue;
        while (e >= nb8 - 2 * mi) { e -= nb8 - 2 * mi; ++mi; }
        fm[f] = mi;
        fn[f] = 2 * mi + e;
    }
    int nvf = 0;  // valid fragments form a prefix
#pragma unroll
    for (int f = 0; f < C::MAXG; ++f) nvf += fm[f] >= 0 ? 1 : 0;
    double acc[C::MAXG][C::KSG][4];
    auto zero_acc = [&]() {
#pragma unroll
        for (int f = 0; f < C::MAXG; ++f)
#pragma unroll
            for (int c = 0; c < C::KSG; ++c)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[f][c][e] = 0.0;
    };
    auto write_part = [&]() {
        double* dst = p.part + static_cast<std::size_t>(cta) * BP * BP;
#pragma unroll
        for (int f = 0; f < C::MAXG; ++f) {
            if (fm[f] < 0) continue;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int row = 16 * fm[f] + g + (e >= 2 ? 8 : 0), col = 8 * fn[f] + 2 * t + (e & 1);
                double v = acc[f][0][e];
#pragma unroll
                for (int c = 1; c < C::KSG; ++c) v += acc[f][c][e];
                dst[row + col * BP] = v;
            }
        }
    };
    // fixed-order sum of the CTA partials into the b x b Gram slot (upper triangle)
    // one warp per Gram entry: lanes load partials lane, lane+32, ... (all in flight at once) and
    // a fixed shuffle tree sums them (deterministic); a thread per entry walking all G partials
    // serially cost 6-10 us per reduction
    auto reduce_parts = [&]() {
        const int nwg = (G * blockDim.x) >> 5;
        for (int e = (cta * blockDim.x + tid) >> 5; e < BP * BP; e += nwg) {
            const int i = e % BP, j = e / BP;
            if (i > j || j >= p.b) continue;  // warp-uniform
            double v[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                const int c = lane + 32 * q;
                v[q] = c < G ? __ldcg(p.part + static_cast<std::size_t>(c) * BP * BP + e) : 0.0;
            }
            double s = ((v[0] + v[1]) + (v[2] + v[3])) + v[4];
            for (int c = lane + 160; c < G; c += 32) s += __ldcg(p.part + static_cast<std::size_t>(c) * BP * BP + e);
            s = warp_sum(s);
            if (lane == 0) p.g[i + j * kSmallMax] = s;
        }
    };
    auto stage_r = [&](const double* rinv) {
        for (int idx = tid; idx < BP * BP; idx += blockDim.x) {
            const int k = idx / BP, n = idx - k * BP;
            rs[k * C::LD + n] = (k < p.b && n < p.b && k <= n) ? __ldcg(rinv + k + n * kSmallMax) : 0.0;
        }
    };
    // sub-tile loop: warp 8 produces (TMA bulk row copies, or generic copies when rows are not
    // 16-byte aligned), warps 0-7 consume; the ring position persists across the phases.
    int ring_stage = 0;
    unsigned ring_phase = 0;
    auto sub_loop = [&](const double* src, std::int64_t ld, const CUtensorMap* tm, auto&& body) {
        const bool bulk = (ld % 2 == 0) && (p.b % 2 == 0) && ((reinterpret_cast<std::uintptr_t>(src) & 15) == 0);
        if (cta == 0) zero_pad();  // the Cholesky used the ring as its workspace
        pb_fence_async();  // generic shared writes of the previous phase before async-proxy copies
        __syncthreads();
        if (!mma_warp) {
            for (int sub = cta; sub < p.nsub; sub += G) {
                pb_wait(&empty[ring_stage], ring_phase ^ 1);
                double* buf = ys2 + ring_stage * C::SUB * C::LD;
                const std::int64_t r0 = static_cast<std::int64_t>(sub) * C::SUB;
                const int nr = static_cast<int>(min(static_cast<std::int64_t>(C::SUB), p.rows - r0));
                if (tm) {
                    // one 2-D tensor TMA lands the padded sub-tile; columns >= b and rows past the
                    // end are zero-filled by the TMA unit (the full box counts toward the tx bytes)
                    if (lane == 0) {
                        pb_arrive_tx(&full[ring_stage], static_cast<unsigned>(C::SUB * C::LD * 8));
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                                sm_addr(buf)),
                            "l"(reinterpret_cast<std::uint64_t>(tm)), "r"(0), "r"(static_cast<int>(r0)),
                            "r"(sm_addr(&full[ring_stage]))
                            : "memory");
                    }
                    __syncwarp();
                } else if (bulk) {
                    if (nr < C::SUB) {  // rows past the end: zero (stale data of an earlier sub-tile)
                        for (int idx = lane; idx < (C::SUB - nr) * BP; idx += 32)
                            buf[(nr + idx / BP) * C::LD + idx % BP] = 0.0;
                        pb_fence_async();
                    }
                    __syncwarp();
                    if (lane == 0) pb_arrive_tx(&full[ring_stage], static_cast<unsigned>(nr * p.b * 8));
                    __syncwarp();
                    for (int r = lane; r < nr; r += 32)
                        pb_bulk(buf + r * C::LD, src + (r0 + r) * ld, static_cast<unsigned>(p.b * 8), &full[ring_stage]);
                } else {
                    for (int idx = lane; idx < C::SUB * BP; idx += 32) {
                        const int r = idx / BP, c = idx - r * BP;
                        buf[r * C::LD + c] = (r < nr && c < p.b) ? src[(r0 + r) * ld + c] : 0.0;
                    }
                    __syncwarp();
                    if (lane == 0) pb_arrive(&full[ring_stage]);
                }
                if (++ring_stage == NST) { ring_stage = 0; ring_phase ^= 1; }
            }
        } else {
            for (int sub = cta; sub < p.nsub; sub += G) {
                pb_wait(&full[ring_stage], ring_phase);
                body(ys2 + ring_stage * C::SUB * C::LD, static_cast<std::int64_t>(sub) * C::SUB);
                pb_fence_async();  // phase B writes T into the buffer before the next bulk copy lands there
                __syncwarp();
                if (lane == 0) pb_arrive(&empty[ring_stage]);
                if (++ring_stage == NST) { ring_stage = 0; ring_phase ^= 1; }
            }
        }
        __syncthreads();
    };
    // ---- phase A: Gram of Y
    panel_mark(0);
    zero_acc();
    sub_loop(p.y, p.ldy, p.use_tm_y ? &p.tm_y : nullptr, [&](double* cur, std::int64_t) {
        if (mma_warp) panel_gram<BP>(cur, acc, fm, fn, nvf);
    });
    panel_mark(1);
    if (mma_warp) write_part();
    grid_barrier(p.gbar, G);
    panel_mark(2);
    reduce_parts();
    grid_barrier(p.gbar, G);
    panel_mark(3);
    static_assert(CholCfg<BP>::SMEM <= C::SMEM, "chol workspace");
    if (cta == 0) chol_tile_block<BP>(p.g, kSmallMax, p.b, p.ra, p.rainv, kSmallMax, p.st0, psm);
    panel_mark(4);
    grid_barrier(p.gbar, G);
    panel_mark(5);
    // A near-orthonormal panel (Gram within 1e-8 of I: every re-orthogonalisation) needs one
    // pass: Q = Y Ra^{-1} is orthonormal to O(u) already, so phase B writes Q and the second
    // Gram / Cholesky / product are skipped (Rb = I, its status reports a clean identity).
    const bool one_pass = __ldcg(&p.st0->breakdown) == 0 &&
                          (__ldcg(&p.st0->gram_dev) <= kOnePassDev ||
                           (p.span_only && span_pass_enough(__ldcg(&p.st0->diag_min), __ldcg(&p.st0->diag_max))));
    if (one_pass) {
        stage_r(p.rainv);
        sub_loop(p.y, p.ldy, p.use_tm_y ? &p.tm_y : nullptr, [&](double* cur, std::int64_t r0) {
            if (mma_warp) {
                double tacc[C::MAXT][4];
                panel_trmm<BP>(cur, rs, tacc, p.b);
                const int mi = warp % C::MI, h = warp / C::MI;
#pragma unroll
                for (int j = 0; j < C::MAXT; ++j)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int row = 16 * mi + g + 8 * hh, col = 8 * (h + C::NG * j) + 2 * t;
                        const bool rok = r0 + row < p.rows;
                        store_col_pair(p.q + (r0 + row) * p.ldq + col, vec_q, rok && col < p.b, rok && col + 1 < p.b,
                                       tacc[j][2 * hh], tacc[j][2 * hh + 1]);
                    }
            }
        });
        if (cta == 0) {
            for (int idx = tid; idx < p.b * p.b; idx += blockDim.x) {
                const int i = idx % p.b, j = idx / p.b;
                p.rb[i + j * kSmallMax] = i == j ? 1.0 : 0.0;
                p.rbinv[i + j * kSmallMax] = i == j ? 1.0 : 0.0;
            }
            if (tid == 0) {
                p.st1->breakdown = 0;
                p.st1->bad_index = -1;
                p.st1->diag_min = 1.0;
                p.st1->diag_max = 1.0;
                p.st1->gram_dev = 0.0;
            }
        }
        panel_mark(11);
        return;
    }
    // ---- phase B: T1 = Y Ra^{-1} (written out) and the Gram of T1
    stage_r(p.rainv);
    zero_acc();
    sub_loop(p.y, p.ldy, p.use_tm_y ? &p.tm_y : nullptr, [&](double* cur, std::int64_t r0) {
        double tacc[C::MAXT][4];
        if (mma_warp) panel_trmm<BP>(cur, rs, tacc, p.b);
        consumer_sync();
        if (mma_warp) {
            const int mi = warp % C::MI, h = warp / C::MI;
#pragma unroll
            for (int j = 0; j < C::MAXT; ++j)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int row = 16 * mi + g + 8 * hh, col = 8 * (h + C::NG * j) + 2 * t;
                    if (col >= BP) continue;
                    cur[row * C::LD + col] = tacc[j][2 * hh];
                    cur[row * C::LD + col + 1] = tacc[j][2 * hh + 1];
                    const bool rok = r0 + row < p.rows;
                    store_col_pair(p.t1 + (r0 + row) * p.b + col, vec_t1, rok && col < p.b, rok && col + 1 < p.b,
                                   tacc[j][2 * hh], tacc[j][2 * hh + 1]);
                }
        }
        consumer_sync();
        if (mma_warp) panel_gram<BP>(cur, acc, fm, fn, nvf);
    });
    panel_mark(6);
    if (mma_warp) write_part();
    grid_barrier(p.gbar, G);
    reduce_parts();
    grid_barrier(p.gbar, G);
    panel_mark(7);
    if (cta == 0) chol_tile_block<BP>(p.g, kSmallMax, p.b, p.rb, p.rbinv, kSmallMax, p.st1, psm, false);
    panel_mark(8);
    grid_barrier(p.gbar, G);
    panel_mark(9);
    // ---- phase D: Q = T1 Rb^{-1}
    stage_r(p.rbinv);
    sub_loop(p.t1, p.b, p.use_tm_t1 ? &p.tm_t1 : nullptr, [&](double* cur, std::int64_t r0) {
        if (mma_warp) {
            double tacc[C::MAXT][4];
            panel_trmm<BP>(cur, rs, tacc, p.b);
            const int mi = warp % C::MI, h = warp / C::MI;
#pragma unroll
            for (int j = 0; j < C::MAXT; ++j)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int row = 16 * mi + g + 8 * hh, col = 8 * (h + C::NG * j) + 2 * t;
                    const bool rok = r0 + row < p.rows;
                    store_col_pair(p.q + (r0 + row) * p.ldq + col, vec_q, rok && col < p.b, rok && col + 1 < p.b,
                                   tacc[j][2 * hh], tacc[j][2 * hh + 1]);
                }
        }
    });
    panel_mark(10);
}

// ---- CholQR2 of a small panel in ONE thread-block cluster -------------------------------
// Panels with b <= 32 and rows <= 8 x 512 (config 1's 2000 x 20 sketches, the re-orthogonalised
// Q_i of every small block): the cluster's C <= 8 CTAs each keep their row slice of Y resident in
// shared memory for the whole factorization (Y is read from HBM once, Q written once). The b x b
// partial Grams are summed over the cluster through distributed shared memory in rank order (the
// same bits in every CTA), and every CTA factors the reduced Gram itself (the in-CTA blocked
// Cholesky + inverse on a shared-memory source), so no grid barrier, no global partials and no
// broadcast of R are needed; CTA 0 publishes R_a, R_a^{-1}, R_b, R_b^{-1}, the Gram and the two
// statuses exactly as cholqr2_panel_kernel does (same one-pass rule for a near-identity Gram).
constexpr int kClusterRowsPerCta = 512;
constexpr int kClusterMaxCtas = 8;

template <int BP>
struct ClusterPanelCfg {
    using P = PanelCfg<BP>;
    static constexpr int LD = P::LD;
    static constexpr int YS = kClusterRowsPerCta * LD;      // resident row slice
    static constexpr int SQ = BP * BP;
    static constexpr int DOUBLES = YS + 4 * SQ + BP * LD + CholCfg<BP>::SMEM_DOUBLES;
    static constexpr int SMEM = DOUBLES * 8;
};

template <int BP>
__global__ void __launch_bounds__(256, 1) cholqr2_cluster_kernel(const __grid_constant__ PanelArgs p, int rr) {
    pdl_wait();
    panel_mark(0);
    using C = PanelCfg<BP>;
    using K = ClusterPanelCfg<BP>;
    cg::cluster_group cluster = cg::this_cluster();
    const int crank = static_cast<int>(cluster.block_rank()), ncta = static_cast<int>(cluster.num_blocks());
    extern __shared__ __align__(128) double csm[];
    double* ys = csm;                       // rr_pad x LD rows of Y (then T)
    double* gpart = ys + K::YS;              // this CTA's partial Gram (BP x BP, col-major)
    double* gsum = gpart + K::SQ;            // the reduced Gram (identical in every CTA)
    double* rloc = gsum + K::SQ;             // R (col-major, ld BP)
    double* rinvloc = rloc + K::SQ;          // R^{-1}
    double* rs = rinvloc + K::SQ;            // R^{-1} staged for the triangular products (BP x LD)
    double* ws = rs + BP * K::LD;            // in-CTA Cholesky workspace
    __shared__ SmallStatus sst;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const bool vec_q = (p.ldq & 1) == 0 && (reinterpret_cast<std::uintptr_t>(p.q) & 15) == 0;
    const std::int64_t r0 = static_cast<std::int64_t>(crank) * rr;
    const std::int64_t left = p.rows - r0;
    const int nr = left <= 0 ? 0 : static_cast<int>(left < rr ? left : rr);
    const int nsub = (nr + C::SUB - 1) / C::SUB;
    const int b = p.b;
    // load the slice (zero-padded to whole sub-tiles and to BP columns): every element an 8-byte
    // cp.async straight into shared memory, all in flight at once (no register round trip)
    for (int idx = tid; idx < nsub * C::SUB * BP; idx += blockDim.x) {
        const int i = idx / BP, c = idx - i * BP;
        double* dst = ys + i * K::LD + c;
        if (i < nr && c < b) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sm_addr(dst)), "l"(p.y + (r0 + i) * p.ldy + c)
                         : "memory");
        } else {
            *dst = 0.0;
        }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    // this warp's upper Gram fragments (as cholqr2_panel_kernel)
    int fm[C::MAXG], fn[C::MAXG];
#pragma unroll
    for (int f = 0; f < C::MAXG; ++f) {
        int e = warp + 8 * f, mi = 0;
        fm[f] = -1;
        fn[f] = 0;
        const int nb8 = (b + 7) >> 3;
        int nf = 0;
        for (int m2 = 0; m2 < BP / 16; ++m2) nf += max(0, nb8 - 2 * m2);
        if (e >= nf) continue;
        while (e >= nb8 - 2 * mi) { e -= nb8 - 2 * mi; ++mi; }
        fm[f] = mi;
        fn[f] = 2 * mi + e;
    }
    int nvf = 0;
#pragma unroll
    for (int f = 0; f < C::MAXG; ++f) nvf += fm[f] >= 0 ? 1 : 0;
    double acc[C::MAXG][C::KSG][4];
    auto zero_acc = [&]() {
#pragma unroll
        for (int f = 0; f < C::MAXG; ++f)
#pragma unroll
            for (int c = 0; c < C::KSG; ++c)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[f][c][e] = 0.0;
    };
    // partial Gram -> gpart; cluster-wide fixed-order sum -> gsum (every CTA); factor -> rloc, rinvloc
    auto gram_reduce_factor = [&](SmallStatus* st_out, double* r_out, double* rinv_out, bool first) {
        for (int idx = tid; idx < K::SQ; idx += blockDim.x) gpart[idx] = 0.0;
        __syncthreads();
#pragma unroll
        for (int f = 0; f < C::MAXG; ++f) {
            if (fm[f] < 0) continue;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int row = 16 * fm[f] + g + (e >= 2 ? 8 : 0), col = 8 * fn[f] + 2 * t + (e & 1);
                double v = acc[f][0][e];
#pragma unroll
                for (int c = 1; c < C::KSG; ++c) v += acc[f][c][e];
                gpart[row + col * BP] = v;
            }
        }
        cluster.sync();
        panel_mark(first ? 2 : 6);
        for (int idx = tid; idx < K::SQ; idx += blockDim.x) {
            const int i = idx % BP, j = idx / BP;
            double sum = 0.0;
            if (i <= j && j < b)
                for (int c = 0; c < ncta; ++c) sum += cluster.map_shared_rank(gpart, c)[idx];
            gsum[idx] = sum;
        }
        cluster.sync();  // every CTA has read every partial before any gpart is reused
        panel_mark(first ? 3 : 7);
        chol_tile_block<BP, true>(gsum, BP, b, rloc, rinvloc, BP, &sst, ws, false);
        if (crank == 0) {
            for (int idx = tid; idx < b * b; idx += blockDim.x) {
                const int i = idx % b, j = idx / b;
                r_out[i + j * kSmallMax] = rloc[i + j * BP];
                rinv_out[i + j * kSmallMax] = rinvloc[i + j * BP];
                if (first) p.g[i + j * kSmallMax] = gsum[i + j * BP];
            }
            if (tid == 0) *st_out = sst;
        }
        __syncthreads();
        panel_mark(first ? 4 : 8);
        panel_mark(first ? 5 : 9);
    };
    auto stage_r = [&]() {
        for (int idx = tid; idx < BP * BP; idx += blockDim.x) {
            const int k = idx / BP, n = idx - k * BP;
            rs[k * K::LD + n] = (k < b && n < b && k <= n) ? rinvloc[k + n * BP] : 0.0;
        }
        __syncthreads();
    };
    // out rows of this slice = ys * rs, to global (q) or back into ys
    auto product = [&](bool to_q, bool gram_after) {
        for (int sub = 0; sub < nsub; ++sub) {
            double* cur = ys + sub * C::SUB * K::LD;
            double tacc[C::MAXT][4];
            panel_trmm<BP>(cur, rs, tacc, b);
            __syncthreads();
            const int mi = warp % C::MI, h = warp / C::MI;
#pragma unroll
            for (int j = 0; j < C::MAXT; ++j)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int row = 16 * mi + g + 8 * hh, col = 8 * (h + C::NG * j) + 2 * t;
                    if (col >= BP) continue;
                    if (to_q) {
                        const std::int64_t gr = r0 + sub * C::SUB + row;
                        const bool rok = sub * C::SUB + row < nr;
                        store_col_pair(p.q + gr * p.ldq + col, vec_q, rok && col < b, rok && col + 1 < b, tacc[j][2 * hh],
                                       tacc[j][2 * hh + 1]);
                    } else {
                        cur[row * K::LD + col] = tacc[j][2 * hh];
                        cur[row * K::LD + col + 1] = tacc[j][2 * hh + 1];
                    }
                }
            __syncthreads();
            if (gram_after) panel_gram<BP>(cur, acc, fm, fn, nvf);
        }
    };
    __syncthreads();
    // ---- Gram of Y, R_a
    zero_acc();
    for (int sub = 0; sub < nsub; ++sub) panel_gram<BP>(ys + sub * C::SUB * K::LD, acc, fm, fn, nvf);
    panel_mark(1);
    gram_reduce_factor(p.st0, p.ra, p.rainv, true);
    const bool one_pass = sst.breakdown == 0 &&
                          (sst.gram_dev <= kOnePassDev || (p.span_only && span_pass_enough(sst.diag_min, sst.diag_max)));
    stage_r();
    if (one_pass) {  // near-orthonormal Y: Q = Y R_a^{-1}, R_b = I (as the panel kernel)
        product(true, false);
        if (crank == 0) {
            for (int idx = tid; idx < b * b; idx += blockDim.x) {
                const int i = idx % b, j = idx / b;
                p.rb[i + j * kSmallMax] = i == j ? 1.0 : 0.0;
                p.rbinv[i + j * kSmallMax] = i == j ? 1.0 : 0.0;
            }
            if (tid == 0) {
                p.st1->breakdown = 0;
                p.st1->bad_index = -1;
                p.st1->diag_min = 1.0;
                p.st1->diag_max = 1.0;
                p.st1->gram_dev = 0.0;
            }
        }
        panel_mark(11);
        return;
    }
    // ---- T = Y R_a^{-1} (kept in shared memory) and its Gram, R_b
    zero_acc();
    product(false, true);
    gram_reduce_factor(p.st1, p.rb, p.rbinv, false);
    stage_r();
    // ---- Q = T R_b^{-1}
    product(true, false);
    panel_mark(10);
}

template <int BP>
void launch_cholqr2_cluster(cudaStream_t st, PanelArgs& a) {
    using K = ClusterPanelCfg<BP>;
    auto kern = cholqr2_cluster_kernel<BP>;
    static PerDevice<bool> setup;
    setup.get([&] {
        QB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM));
        return true;
    });
    const int ncta = static_cast<int>(std::min<std::int64_t>(kClusterMaxCtas, std::max<std::int64_t>(1, ceil_div(a.rows, 128))));
    const int rr = static_cast<int>(ceil_div(a.rows, ncta));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(ncta));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = K::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = static_cast<unsigned>(ncta);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    QB_CUDA(cudaLaunchKernelEx(&cfg, kern, a, rr));
}

bool cluster_panel_enabled() {
    const char* e = std::getenv("QBFAC_PANEL_CLUSTER");
    return !(e && e[0] == '0');
}

// ---- one-sided Jacobi SVD of a small square matrix (qb_to_svd) ---------
// Hestenes one-sided Jacobi on the columns of N (r x r, column-major): rotations from the
// right orthogonalise the columns, N W = U Sigma, W accumulates the rotations (W starts as
// I). Round-robin (circle method) ordering: each step rotates r/2 disjoint column pairs,
// one warp per pair (column dots reduced in a fixed order: deterministic), steps separated
// by the nanosleep grid barrier; a sweep without any rotation above tol ends the loop.
// One-sided Jacobi keeps high relative accuracy for the small singular values.
struct JacobiArgs {
    double* nmat;
    double* w;
    int r, rp, max_sweeps;
    double tol;
    unsigned* gbar;
    unsigned* rotated;  // per-sweep rotation counters (zeroed before the launch)
    int* sweeps_out;
};

__global__ void __launch_bounds__(256) jacobi_svd_kernel(JacobiArgs p) {
    const int lane = threadIdx.x & 31;
    const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    const int r = p.r, rp = p.rp, half = rp / 2;
    int sweep = 0;
    for (; sweep < p.max_sweeps; ++sweep) {
        for (int step = 0; step < rp - 1; ++step) {
            for (int t = gwarp; t < half; t += nwarps) {
                // circle method: player rp-1 fixed, the others rotate
                int a, b;
                if (t == 0) {
                    a = step;
                    b = rp - 1;
                } else {
                    a = (step + t) % (rp - 1);
                    b = (step - t + (rp - 1)) % (rp - 1);
                }
                if (a > b) { const int x = a; a = b; b = x; }
                if (b >= r) continue;
                double* cp = p.nmat + static_cast<std::int64_t>(a) * r;
                double* cq = p.nmat + static_cast<std::int64_t>(b) * r;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int i = lane; i < r; i += 32) {
                    const double x = cp[i], y = cq[i];
                    al = fma(x, x, al);
                    be = fma(y, y, be);
                    ga = fma(x, y, ga);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o);
                }
                if (!(fabs(ga) > p.tol * sqrt(al * be))) continue;
                const double zeta = (be - al) / (2.0 * ga);
                const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + tt * tt), sn = c * tt;
                for (int i = lane; i < r; i += 32) {
                    const double x = cp[i], y = cq[i];
                    cp[i] = c * x - sn * y;
                    cq[i] = sn * x + c * y;
                }
                double* wp = p.w + static_cast<std::int64_t>(a) * r;
                double* wq = p.w + static_cast<std::int64_t>(b) * r;
                for (int i = lane; i < r; i += 32) {
                    const double x = wp[i], y = wq[i];
                    wp[i] = c * x - sn * y;
                    wq[i] = sn * x + c * y;
                }
                if (lane == 0) atomicAdd(p.rotated + sweep, 1u);
            }
            grid_barrier(p.gbar, gridDim.x);
        }
        if (*reinterpret_cast<volatile unsigned*>(p.rotated + sweep) == 0) break;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *p.sweeps_out = sweep;
}

// ---- block one-sided Jacobi (qb_to_svd at large r) -------------------------------------
// The columns of N are grouped into nblk blocks of nb (nblk even; padding blocks are empty).
// An outer sweep runs the circle method over the blocks: nblk - 1 steps, each with nblk / 2
// disjoint block pairs, one CTA per pair. The CTA stages the pair's 2 nb columns of N in shared
// memory, runs ONE inner one-sided Jacobi sweep over them (circle method on the 2 nb local
// columns, one warp per disjoint column pair, fixed-order warp dots: deterministic) while
// accumulating the 2nb x 2nb rotation V, writes the columns back and applies V to the same
// columns of W (W[:, pair] = W[:, pair] V, row by row). Every pair of global columns meets once
// per outer sweep; the sweep count of the scalar kernel drops by the inner sweeps, and each grid
// barrier now covers nb^2 more rotations (r = 1000: 125 barriers per sweep instead of 999).
struct JacobiBlockArgs {
    double* nmat;
    double* w;
    int r, nb, nblk, max_sweeps;
    double tol;
    unsigned* gbar;
    unsigned* rotated;
    int* sweeps_out;
    int trace;  // QBFAC_JACOBI_TRACE=1: CTA 0 prints its per-phase time split at the end
};

__device__ __forceinline__ unsigned long long jb_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void circle_pair(int round, int t, int n, int& a, int& b) {
    if (t == 0) {
        a = round;
        b = n - 1;
    } else {
        a = (round + t) % (n - 1);
        b = (round - t + (n - 1)) % (n - 1);
    }
    if (a > b) { const int x = a; a = b; b = x; }
}

constexpr int kJbMaxCols = 16;  // 2 nb <= 16

// 16 warps per CTA: the staging, write-back and W-update loops are latency-bound (r = 1000:
// 8 -> 16 warps took the Jacobi kernel 130 -> 106 ms; `QBFAC_JACOBI_TRACE=1` prints the split)
constexpr int kJbThreads = 512;

__global__ void __launch_bounds__(kJbThreads) jacobi_block_kernel(JacobiBlockArgs p) {
    extern __shared__ __align__(16) double jsm[];
    const int r = p.r, nb = p.nb, nc = 2 * nb;
    double* cols = jsm;                                   // nc columns of r (column c at cols + c r)
    double* V = jsm + static_cast<std::size_t>(nc) * r;  // nc x nc, column-major
    __shared__ unsigned s_cnt;
    unsigned long long ph[5] = {0, 0, 0, 0, 0};  // per-phase time (thread 0; printed when p.trace)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
    const int half = p.nblk / 2;
    int sweep = 0;
    for (; sweep < p.max_sweeps; ++sweep) {
        for (int step = 0; step < p.nblk - 1; ++step) {
            for (int t = blockIdx.x; t < half; t += gridDim.x) {
                unsigned long long tp = jb_now();
                int bi, bj;
                circle_pair(step, t, p.nblk, bi, bj);
                const int i0 = bi * nb, j0 = bj * nb;
                const int ni = max(0, min(nb, r - i0)), nj = max(0, min(nb, r - j0));
                auto gcol = [&](int c) -> int {  // local column -> global column (-1: empty)
                    return c < nb ? (c < ni ? i0 + c : -1) : (c - nb < nj ? j0 + c - nb : -1);
                };
                // 8 loads in flight per thread (a load -> store chain per element serialises on L2 latency)
                for (int base = tid; base < nc * r; base += 8 * blockDim.x) {
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int idx = base + u * blockDim.x;
                        v[u] = 0.0;
                        if (idx < nc * r) {
                            const int c = idx / r, g = gcol(c);
                            if (g >= 0) v[u] = p.nmat[static_cast<std::int64_t>(g) * r + (idx - c * r)];
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int idx = base + u * blockDim.x;
                        if (idx < nc * r) cols[idx] = v[u];
                    }
                }
                for (int idx = tid; idx < nc * nc; idx += blockDim.x) V[idx] = (idx % nc == idx / nc) ? 1.0 : 0.0;
                if (tid == 0) s_cnt = 0;
                __syncthreads();
                if (tid == 0) { const unsigned long long q = jb_now(); ph[0] += q - tp; tp = q; }
                for (int rd = 0; rd < nc - 1; ++rd) {
                    for (int q = warp; q < nb; q += nwarps) {
                        int a, b;
                        circle_pair(rd, q, nc, a, b);
                        double* ca = cols + static_cast<std::size_t>(a) * r;
                        double* cb = cols + static_cast<std::size_t>(b) * r;
                        double al = 0.0, be = 0.0, ga = 0.0;
                        for (int i = lane; i < r; i += 32) {
                            const double x = ca[i], y = cb[i];
                            al = fma(x, x, al);
                            be = fma(y, y, be);
                            ga = fma(x, y, ga);
                        }
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            al += __shfl_xor_sync(0xffffffffu, al, o);
                            be += __shfl_xor_sync(0xffffffffu, be, o);
                            ga += __shfl_xor_sync(0xffffffffu, ga, o);
                        }
                        if (!(fabs(ga) > p.tol * sqrt(al * be))) continue;
                        const double zeta = (be - al) / (2.0 * ga);
                        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                        const double c = 1.0 / sqrt(1.0 + tt * tt), sn = c * tt;
                        for (int i = lane; i < r; i += 32) {
                            const double x = ca[i], y = cb[i];
                            ca[i] = c * x - sn * y;
                            cb[i] = sn * x + c * y;
                        }
                        if (lane < nc) {
                            const double x = V[lane + a * nc], y = V[lane + b * nc];
                            V[lane + a * nc] = c * x - sn * y;
                            V[lane + b * nc] = sn * x + c * y;
                        }
                        if (lane == 0) atomicAdd(&s_cnt, 1u);
                    }
                    __syncthreads();
                }
                if (tid == 0) { const unsigned long long q = jb_now(); ph[1] += q - tp; tp = q; }
                for (int idx = tid; idx < nc * r; idx += blockDim.x) {
                    const int c = idx / r, i = idx - c * r, g = gcol(c);
                    if (g >= 0) p.nmat[static_cast<std::int64_t>(g) * r + i] = cols[idx];
                }
                if (tid == 0) { const unsigned long long q = jb_now(); ph[2] += q - tp; tp = q; }
                if (s_cnt) {
                    for (int i = tid; i < r; i += blockDim.x) {
                        double wv[kJbMaxCols];
#pragma unroll
                        for (int c = 0; c < kJbMaxCols; ++c) {
                            const int g = c < nc ? gcol(c) : -1;
                            wv[c] = g >= 0 ? p.w[static_cast<std::int64_t>(g) * r + i] : 0.0;
                        }
#pragma unroll
                        for (int c = 0; c < kJbMaxCols; ++c) {
                            if (c >= nc) break;
                            const int g = gcol(c);
                            if (g < 0) continue;
                            double acc = 0.0;
#pragma unroll
                            for (int k = 0; k < kJbMaxCols; ++k)
                                if (k < nc) acc = fma(wv[k], V[k + c * nc], acc);
                            p.w[static_cast<std::int64_t>(g) * r + i] = acc;
                        }
                    }
                    if (tid == 0) atomicAdd(p.rotated + sweep, s_cnt);
                }
                __syncthreads();
                if (tid == 0) { const unsigned long long q = jb_now(); ph[3] += q - tp; }
            }
            const unsigned long long tb = jb_now();
            grid_barrier(p.gbar, gridDim.x);
            if (tid == 0) ph[4] += jb_now() - tb;
        }
        if (*reinterpret_cast<volatile unsigned*>(p.rotated + sweep) == 0) break;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *p.sweeps_out = sweep;
        if (p.trace)
            printf("jacobi_block r=%d nb=%d CTAs=%d sweeps=%d: load %.1f  inner %.1f  writeback %.1f  W %.1f  barrier %.1f us\n",
                   r, nb, gridDim.x, sweep, ph[0] * 1e-3, ph[1] * 1e-3, ph[2] * 1e-3, ph[3] * 1e-3, ph[4] * 1e-3);
    }
}

// ---- block one-sided Jacobi with a Gram-based inner solver (qb_to_svd at large r) ----------
// Same outer schedule as jacobi_block_kernel (circle method over nb = 8 column blocks, one CTA per
// block pair, one grid barrier per outer round), but the sequential inner rounds no longer touch
// the r-long columns: the CTA forms the 16 x 16 Gram G = X^T X of the pair's staged columns once
// (fresh, fixed-order dots), ONE warp diagonalises G by two-sided Jacobi rotations on the 16 x 16
// shared-memory tile (`inner` cyclic sweeps, 8 disjoint rotations per round, each lane transforms
// two 2 x 2 blocks of G in place) while accumulating V, and the whole CTA applies V once to the
// columns of N (from shared memory) and of W (global). Convergence is judged on the fresh Gram
// only (pairs with |g_pq| > tol sqrt(g_pp g_qq) before any rotation), so the stopping rule is the
// scalar kernel's; a pair block with no such pair is left untouched.
constexpr int kJgNc = 16;
constexpr int kJgMaxCta = 2;  // CTAs per block pair (cluster size)
constexpr int kJgGramWarps = 8;   // warps forming the Gram (one partial buffer each)
constexpr int kJgInnerWarps = 6;  // warps of the inner two-sided Jacobi (2 on G, 4 on V)

struct JacobiGramArgs {
    double* nmat;
    double* w;
    int r, nblk, max_sweeps, inner;
    double tol;
    unsigned* gbar;
    unsigned* rotated;
    unsigned* ver;  // per column block: CTA-visits completed (zeroed before the launch)
    int* sweeps_out;
    int trace;
};

// rows A and 15 - A of the upper triangle of G over this warp's row range (17 dots)
template <int A>
__device__ __forceinline__ void jg_gram_rows(const double* __restrict__ cols, int r, int i0, int i1, int lane,
                                             double* __restrict__ out) {
    constexpr int B = kJgNc - 1 - A;
    double ra[kJgNc - A], rb[kJgNc - B];
#pragma unroll
    for (int c = 0; c < kJgNc - A; ++c) ra[c] = 0.0;
#pragma unroll
    for (int c = 0; c < kJgNc - B; ++c) rb[c] = 0.0;
#pragma unroll 1
    for (int i = i0 + lane; i < i1; i += 32) {
        double x[kJgNc - A];
#pragma unroll
        for (int c = 0; c < kJgNc - A; ++c) x[c] = cols[static_cast<std::size_t>(A + c) * r + i];
#pragma unroll
        for (int c = 0; c < kJgNc - A; ++c) ra[c] = fma(x[0], x[c], ra[c]);
#pragma unroll
        for (int c = 0; c < kJgNc - B; ++c) rb[c] = fma(x[B - A], x[B - A + c], rb[c]);
    }
#pragma unroll
    for (int c = 0; c < kJgNc - A; ++c) {
        double v = ra[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) out[A * kJgNc + A + c] = v;
    }
#pragma unroll
    for (int c = 0; c < kJgNc - B; ++c) {
        double v = rb[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) out[B * kJgNc + B + c] = v;
    }
}

__global__ void __launch_bounds__(kJbThreads, 1) jacobi_gram_kernel(JacobiGramArgs p) {
    extern __shared__ __align__(16) double jsm[];
    constexpr int NC = kJgNc, nb = NC / 2;
    cg::cluster_group cluster = cg::this_cluster();
    const int crank = static_cast<int>(cluster.block_rank()), ncta = static_cast<int>(cluster.num_blocks());
    const int r = p.r;
    // this CTA's rows of the pair's columns: [row0, row0 + rl); slices start on even rows so a
    // column slice is one 16-byte aligned bulk copy when r is even
    const int rs = ((r + ncta - 1) / ncta + 1) & ~1;
    const int row0 = min(r, crank * rs), rl = min(r, row0 + rs) - row0;
    double* cols = jsm;                                        // NC column slices of N (column c at cols + c rs)
    double* wcols = jsm + static_cast<std::size_t>(NC) * rs;  // the same slices of W (prefetched for the apply)
    double* V = wcols + static_cast<std::size_t>(NC) * rs;    // NC x NC, column-major
    double* G = V + NC * NC;                                   // NC x NC, symmetric
    double* Gp = G + NC * NC;                                  // kJgGramWarps partial Grams (row steps w mod 8)
    double* Gx = Gp + kJgGramWarps * NC * NC;                  // [parity][rank] partial Grams pushed by the cluster
    __shared__ unsigned s_cnt;
    __shared__ __align__(8) std::uint64_t s_bar, s_wbar;
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // per-phase time of the traced CTA (thread 0)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int half = p.nblk / 2;
    const int cid = blockIdx.x / ncta, ncl = gridDim.x / ncta;
    const int g8 = lane >> 2, t4 = lane & 3;  // DMMA m16n8k4 fragment coordinates
    const bool bulk = (r & 1) == 0 && rl > 0;
    const double tol2 = p.tol * p.tol;
    unsigned parity = 0, visit = 0;
    int gstep = 0;  // outer rounds completed (over all sweeps)
    if (tid == 0) {
        pb_init(&s_bar, 1);
        pb_init(&s_wbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    int sweep = 0;
    for (; sweep < p.max_sweeps; ++sweep) {
        for (int step = 0; step < p.nblk - 1; ++step) {
            for (int t = cid; t < half; t += ncl) {
                unsigned long long tp = jb_now();
                int bi, bj;
                circle_pair(step, t, p.nblk, bi, bj);
                const int i0 = bi * nb, j0 = bj * nb;
                const int ni = max(0, min(nb, r - i0)), nj = max(0, min(nb, r - j0));
                auto gcol = [&](int c) -> int {
                    return c < nb ? (c < ni ? i0 + c : -1) : (c - nb < nj ? j0 + c - nb : -1);
                };
                // Block dataflow instead of a grid barrier per outer round: every block is visited once
                // per round, by one cluster; ver[b] counts the CTA-visits of block b completed so far,
                // so this visit may start once both of its blocks have seen ncta * (rounds so far).
                const unsigned need = static_cast<unsigned>(ncta) * static_cast<unsigned>(gstep);
                if (tid == 0) {
                    volatile unsigned* vi = p.ver + bi;
                    volatile unsigned* vj = p.ver + bj;
                    while (*vi < need || *vj < need) {}
                    __threadfence();
                }
                __syncthreads();
                if (tid == 0) { const unsigned long long q = jb_now(); ph[4] += q - tp; tp = q; }
                if (bulk) {
                    if (tid == 0) {
                        // the columns were written by other CTAs (generic proxy) before the grid barrier
                        asm volatile("fence.proxy.async;\n" ::: "memory");
                        pb_arrive_tx(&s_bar, static_cast<unsigned>((ni + nj) * rl * 8));
                        for (int c = 0; c < NC; ++c) {
                            const int g = gcol(c);
                            if (g >= 0)
                                pb_bulk(cols + static_cast<std::size_t>(c) * rs,
                                        p.nmat + static_cast<std::int64_t>(g) * r + row0, static_cast<unsigned>(rl * 8), &s_bar);
                        }
                        pb_arrive_tx(&s_wbar, static_cast<unsigned>((ni + nj) * rl * 8));
                        for (int c = 0; c < NC; ++c) {
                            const int g = gcol(c);
                            if (g >= 0)
                                pb_bulk(wcols + static_cast<std::size_t>(c) * rs,
                                        p.w + static_cast<std::int64_t>(g) * r + row0, static_cast<unsigned>(rl * 8), &s_wbar);
                        }
                    }
                    if (ni + nj < NC)
                        for (int idx = tid; idx < NC * rl; idx += kJbThreads) {
                            const int c = idx / rl;
                            if (gcol(c) < 0) cols[static_cast<std::size_t>(c) * rs + (idx - c * rl)] = 0.0;
                        }
                } else {
                    for (int base = tid; base < NC * rl; base += 8 * kJbThreads) {
                        double v[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int idx = base + u * kJbThreads;
                            v[u] = 0.0;
                            if (idx < NC * rl) {
                                const int c = idx / rl, g = gcol(c);
                                if (g >= 0) v[u] = p.nmat[static_cast<std::int64_t>(g) * r + row0 + (idx - c * rl)];
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int idx = base + u * kJbThreads;
                            if (idx < NC * rl) {
                                const int c = idx / rl;
                                cols[static_cast<std::size_t>(c) * rs + (idx - c * rl)] = v[u];
                            }
                        }
                    }
                }
                if (tid < NC * NC) V[tid] = (tid % NC == tid / NC) ? 1.0 : 0.0;
                if (bulk) {
                    pb_wait(&s_bar, parity);
                    parity ^= 1u;
                }
                __syncthreads();
                if (tid == 0) { const unsigned long long q = jb_now(); ph[5] += q - tp; tp = q; }
                if (warp < kJgGramWarps) {
                    // fresh Gram G = X^T X on the FP64 tensor pipe (m16n8k4: A = X^T, B = X, so the B
                    // fragments are the A fragments); warp w takes the 4-row steps w, w + 8, ...
                    double acc0[4] = {0.0, 0.0, 0.0, 0.0}, acc1[4] = {0.0, 0.0, 0.0, 0.0};
                    const double* c0 = cols + static_cast<std::size_t>(g8) * rs;
                    const double* c1 = cols + static_cast<std::size_t>(g8 + 8) * rs;
                    for (int i = 4 * warp + t4; i < ((rl + 3) & ~3); i += 4 * kJgGramWarps) {
                        const double v0 = i < rl ? c0[i] : 0.0, v1 = i < rl ? c1[i] : 0.0;
                        dmma_16x8x4(acc0, v0, v1, v0);
                        dmma_16x8x4(acc1, v0, v1, v1);
                    }
                    double* out = Gp + warp * NC * NC;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int m = g8 + (e >= 2 ? 8 : 0), n = 2 * t4 + (e & 1);
                        out[m * NC + n] = acc0[e];
                        out[m * NC + 8 + n] = acc1[e];
                    }
                }
                __syncthreads();
                if (tid == 0) { const unsigned long long q = jb_now(); ph[6] += q - tp; tp = q; }
                // every CTA pushes its partial into every CTA's Gx[visit parity][its rank]; one cluster
                // barrier; the sum runs in rank order (identical G on every CTA). The buffer of this
                // parity is rewritten two visits later, behind the next visit's cluster barrier.
                {
                    double* gx = Gx + (visit & 1u) * (kJgMaxCta * NC * NC);
                    if (tid < NC * NC && tid / NC <= tid % NC) {
                        double v = 0.0;
#pragma unroll
                        for (int w8 = 0; w8 < kJgGramWarps; ++w8) v += Gp[w8 * NC * NC + tid];  // fixed order
                        for (int c = 0; c < ncta; ++c) cluster.map_shared_rank(gx, c)[crank * NC * NC + tid] = v;
                    }
                    cluster.sync();
                    if (tid < NC * NC) {
                        const int a = tid / NC, b = tid % NC;
                        const int e = min(a, b) * NC + max(a, b);
                        double sum = 0.0;
                        for (int c = 0; c < ncta; ++c) sum += gx[c * NC * NC + e];
                        G[tid] = sum;
                    }
                    ++visit;
                    __syncthreads();
                }
                if (tid == 0) { const unsigned long long q = jb_now(); ph[0] += q - tp; tp = q; }
                if (warp < kJgInnerWarps) {
                    // pairs above the threshold in the fresh Gram (over 32 lanes; every inner warp
                    // counts for itself). The first outer round of a sweep rotates all 120 pairs of the
                    // 16 columns (circle order, 15 rounds); the others only the 64 cross pairs of the
                    // two blocks (8 rounds): every global pair is then rotated exactly once per sweep,
                    // as in the scalar kernel.
                    const bool full = step == 0;
                    unsigned cnt = 0;
                    for (int e = lane; e < NC * (NC - 1) / 2; e += 32) {
                        int a = 0, rem = e;
                        while (rem >= NC - 1 - a) { rem -= NC - 1 - a; ++a; }
                        const int b = a + 1 + rem;
                        if (!full && !(a < nb && b >= nb)) continue;  // not rotated in this visit
                        const double al = G[a * NC + a], be = G[b * NC + b], ga = G[a * NC + b];
                        cnt += fabs(ga) > p.tol * sqrt(al * be) ? 1u : 0u;
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
                    if (tid == 0) s_cnt = cnt;
                    if (cnt) {
                        // Two-sided Jacobi on G over kJgInnerWarps warps (every CTA of the cluster runs
                        // the same sequence on the same G: identical V). Per round, lanes 0-7 of EVERY
                        // inner warp compute the 8 rotations redundantly (no shared-memory hand-off):
                        // cos 2t = |x| / h, h = sqrt(x^2 + y^2), x = g_bb - g_aa, y = 2 g_ab, from two
                        // reciprocal square roots; the other lanes fetch (c, s) by shuffle. Warps 0-1:
                        // one 2 x 2 block of G per lane (row pair qi x column pair qj, in place);
                        // warps 2-5: one (row, pair) of V per lane. One named barrier per round.
                        const int item = warp * 32 + lane;
                        const bool isg = warp < 2;
                        const int qi = isg ? item >> 3 : 0, qj = isg ? item & 7 : (item - 64) >> 4;
                        const int vrow = (item - 64) & 15;
                        for (int isw = 0; isw < p.inner; ++isw) {
                            for (int rd = 0; rd < (full ? NC - 1 : nb); ++rd) {
                                auto pair_of = [&](int q, int& a, int& b) {
                                    if (full) {
                                        circle_pair(rd, q, NC, a, b);
                                    } else {
                                        a = q;
                                        b = nb + ((q + rd) & (nb - 1));
                                    }
                                };
                                int ai, bi2, aj, bj2;
                                pair_of(qi, ai, bi2);
                                pair_of(qj, aj, bj2);
                                // data of this lane's item (independent of the rotation parameters)
                                double g00, g01, g10, g11;
                                if (isg) {
                                    g00 = G[ai * NC + aj]; g01 = G[ai * NC + bj2];
                                    g10 = G[bi2 * NC + aj]; g11 = G[bi2 * NC + bj2];
                                } else {
                                    g00 = V[vrow + aj * NC]; g01 = V[vrow + bj2 * NC];
                                    g10 = 0.0; g11 = 0.0;
                                }
                                double c = 1.0, sn = 0.0;
                                {
                                    int a, b;
                                    pair_of(lane & (nb - 1), a, b);
                                    const double al = G[a * NC + a], be = G[b * NC + b], ga = G[a * NC + b];
                                    if (ga * ga > tol2 * (al * be)) {
                                        const double x = be - al, y = 2.0 * ga;
                                        const double rh = rsqrt(fma(x, x, y * y));
                                        const double c2 = fma(0.5 * fabs(x), rh, 0.5);
                                        const double rc = rsqrt(c2);
                                        c = c2 * rc;
                                        const double sa = 0.5 * fabs(y) * rh * rc;
                                        sn = ((x >= 0.0) == (y >= 0.0)) ? sa : -sa;
                                    }
                                }
                                const double cj = __shfl_sync(0xffffffffu, c, qj), sj = __shfl_sync(0xffffffffu, sn, qj);
                                const double ci = __shfl_sync(0xffffffffu, c, qi), si = __shfl_sync(0xffffffffu, sn, qi);
                                // every read of G for this round is done before any lane overwrites it
                                asm volatile("bar.sync 2, %0;\n" ::"n"(kJgInnerWarps * 32) : "memory");
                                if (isg) {
                                    const double t00 = cj * g00 - sj * g01, t01 = sj * g00 + cj * g01;
                                    const double t10 = cj * g10 - sj * g11, t11 = sj * g10 + cj * g11;
                                    G[ai * NC + aj] = ci * t00 - si * t10;
                                    G[ai * NC + bj2] = ci * t01 - si * t11;
                                    G[bi2 * NC + aj] = si * t00 + ci * t10;
                                    G[bi2 * NC + bj2] = si * t01 + ci * t11;
                                } else {
                                    V[vrow + aj * NC] = cj * g00 - sj * g01;
                                    V[vrow + bj2 * NC] = sj * g00 + cj * g01;
                                }
                                asm volatile("bar.sync 2, %0;\n" ::"n"(kJgInnerWarps * 32) : "memory");
                            }
                        }
                    }
                }
                __syncthreads();
                if (tid == 0) { const unsigned long long q = jb_now(); ph[1] += q - tp; tp = q; }
                if (bulk) {  // the W slices have landed (waited for even when unused: the barrier phase must advance)
                    pb_wait(&s_wbar, parity ^ 1u);
                    if (tid == 0) { const unsigned long long q = jb_now(); ph[7] += q - tp; tp = q; }
                }
                if (s_cnt) {
                    // N[rows, pair] = X V and W[rows, pair] = W[rows, pair] V on the FP64 tensor pipe:
                    // 16-row tiles (m16n8k4, K = 16: four steps, two 8-column halves), V fragments held
                    // in registers; the N slices come from shared memory, W's too when prefetched
                    double bv[4][2];
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {
                        bv[ks][0] = V[(4 * ks + t4) + g8 * NC];
                        bv[ks][1] = V[(4 * ks + t4) + (8 + g8) * NC];
                    }
                    int gk[4];
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) gk[ks] = gcol(4 * ks + t4);
                    const int ntile = (rl + 15) >> 4;
                    for (int tile = warp; tile < 2 * ntile; tile += kJbThreads / 32) {
                        const bool isw = tile >= ntile;
                        const int rbase = 16 * (isw ? tile - ntile : tile);
                        const double* src = isw ? wcols : cols;
                        double* dstm = isw ? p.w : p.nmat;
                        const int ra = rbase + g8, rb = ra + 8;
                        double acc0[4] = {0.0, 0.0, 0.0, 0.0}, acc1[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks) {
                            double a0 = 0.0, a1 = 0.0;
                            if (isw && !bulk) {
                                if (gk[ks] >= 0) {
                                    const double* wc = p.w + static_cast<std::int64_t>(gk[ks]) * r + row0;
                                    if (ra < rl) a0 = wc[ra];
                                    if (rb < rl) a1 = wc[rb];
                                }
                            } else if (gk[ks] >= 0) {
                                const double* sc = src + static_cast<std::size_t>(4 * ks + t4) * rs;
                                if (ra < rl) a0 = sc[ra];
                                if (rb < rl) a1 = sc[rb];
                            }
                            dmma_16x8x4(acc0, a0, a1, bv[ks][0]);
                            dmma_16x8x4(acc1, a0, a1, bv[ks][1]);
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int row = e >= 2 ? rb : ra;
                            if (row >= rl) continue;
                            const int n0 = 2 * t4 + (e & 1);
                            const int ga = gcol(n0), gb2 = gcol(8 + n0);
                            if (ga >= 0) dstm[static_cast<std::int64_t>(ga) * r + row0 + row] = acc0[e];
                            if (gb2 >= 0) dstm[static_cast<std::int64_t>(gb2) * r + row0 + row] = acc1[e];
                        }
                    }
                    if (tid == 0 && crank == 0) atomicAdd(p.rotated + sweep, s_cnt);
                }
                __syncthreads();
                if (tid == 0) {  // this CTA's rows of both blocks are written: publish the visit
                    __threadfence();
                    atomicAdd(p.ver + bi, 1u);
                    atomicAdd(p.ver + bj, 1u);
                    const unsigned long long q = jb_now(); ph[3] += q - tp;
                }
            }
            ++gstep;
        }
        // one grid barrier per sweep: the sweep's rotation count is complete
        const unsigned long long tb = jb_now();
        grid_barrier_tight(p.gbar, gridDim.x);
        if (tid == 0) ph[4] += jb_now() - tb;
        if (*reinterpret_cast<volatile unsigned*>(p.rotated + sweep) == 0) break;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *p.sweeps_out = sweep;
    if (p.trace && blockIdx.x == (gridDim.x > ncta ? ncta : 0) && threadIdx.x == 0)
        printf("jacobi_gram r=%d CTAs=%d cluster=%d inner=%d sweeps=%d (CTA %d): load %.1f  gram %.1f  exchange %.1f  inner %.1f  "
               "w-wait %.1f  apply %.1f  barrier %.1f us\n",
               r, gridDim.x, ncta, p.inner, sweep, blockIdx.x, ph[5] * 1e-3, ph[6] * 1e-3, ph[0] * 1e-3, ph[1] * 1e-3, ph[7] * 1e-3,
               ph[3] * 1e-3, ph[4] * 1e-3);
}

// C = A * B for upper-triangular n x n operands staged in shared memory; blockIdx.x
// selects one of two independent products so R = Rb*Ra and Rinv = Ra^{-1} Rb^{-1}
// are formed in one launch.
struct TrmmPair {
    const double* a[2];
    const double* b[2];
    double* c[2];
};

__global__ void __launch_bounds__(1024) trmm_upper_kernel(TrmmPair prm, int n, std::int64_t ld) {
    pdl_wait();
    extern __shared__ double sm[];
    const int z = blockIdx.x;
    const double* __restrict__ a = prm.a[z];
    const double* __restrict__ bm = prm.b[z];
    double* __restrict__ c = prm.c[z];
    if (!c) return;
    const int lds = n + 1;
    double* sa = sm;              // sa[i * lds + p] = A(i, p)
    double* sb = sm + n * lds;    // sb[j * lds + p] = B(p, j)
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    // staged with explicit zeros outside the triangles, so the product can run over the full p
    // range: adding exact zeros in the same ascending-p order leaves every sum bit-identical to the
    // triangular loop, and each thread's 16 outputs become 16 independent FMA chains
    for (int j = ty; j < n; j += 32)
        for (int i = tx; i < n; i += 32) {
            sa[i * lds + j] = j >= i ? a[i + j * ld] : 0.0;
            sb[j * lds + i] = i <= j ? bm[i + j * ld] : 0.0;
        }
    __syncthreads();
    double acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
    for (int p = 0; p < n; ++p) {
        double av[4], bv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = tx + 32 * u, j = ty + 32 * u;
            av[u] = i < n ? sa[i * lds + p] : 0.0;
            bv[u] = j < n ? sb[j * lds + p] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int i = tx + 32 * u, j = ty + 32 * v;
            if (i < n && j < n) c[i + j * ld] = i <= j ? acc[u][v] : 0.0;
        }
}

// Column j of R^{-1} by back substitution; one thread per column.
__global__ void tri_inverse_kernel(const double* __restrict__ r, double* __restrict__ x, int n,
                                   std::int64_t ld) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        for (int i = n - 1; i >= 0; --i) {
            double v = 0.0;
            if (i <= j) {
                double s = (i == j) ? 1.0 : 0.0;
                for (int p = i + 1; p <= j; ++p) s = fma(-r[i + p * ld], x[p + j * ld], s);
                v = s / r[i + i * ld];
            }
            x[i + j * ld] = v;
        }
    }
}

__global__ void indicator_kernel(double* e_dev, const double* __restrict__ norms, int b, double eps2,
                                 int check, IndicatorOut* out) {
    pdl_wait();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double e = *e_dev;
    int keep = b, met = 0;
    for (int j = 0; j < b; ++j) {
        e -= norms[j];
        if (check && e < eps2) {
            keep = j + 1;
            met = 1;
            break;
        }
    }
    *e_dev = e;
    out->e = e;
    out->keep = keep;
    out->met = met;
}

// ---- Householder panel (cooperative) -------------------------------------------
constexpr int kHhThreads = 256;

__device__ double grid_reduce_sum(cg::grid_group& grid, double v, double* part, double* sh) {
    const double s = block_sum<kHhThreads>(v, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
    grid.sync();
    double tot = 0.0;
    if (threadIdx.x == 0) {
        for (int c = 0; c < static_cast<int>(gridDim.x); ++c) tot += part[c];
        sh[0] = tot;
    }
    __syncthreads();
    tot = sh[0];
    __syncthreads();
    return tot;
}

// Vector version: partials part[cta * nv + c], totals into out_sh (shared, nv values).
__device__ void grid_reduce_vec(cg::grid_group& grid, int nv, double* part, double* out_sh) {
    grid.sync();
    for (int c = threadIdx.x; c < nv; c += blockDim.x) {
        double tot = 0.0;
        for (int q = 0; q < static_cast<int>(gridDim.x); ++q) tot += part[q * nv + c];
        out_sh[c] = tot;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kHhThreads)
householder_panel_kernel(double* y, std::int64_t m, int b, std::int64_t ld, double* r,
                         std::int64_t ldr, double* part, double* qs, double* taus) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[32];
    __shared__ double wv[kSmallMax];
    __shared__ double sgn[kSmallMax];
    const std::int64_t chunk = (m + gridDim.x - 1) / gridDim.x;
    const std::int64_t r0 = blockIdx.x * chunk;
    const std::int64_t r1 = min(m, r0 + chunk);
    // Forward: reflectors H_j = I - tau_j v_j v_j^T, v_j = [1; y(j+1:, j)] (LAPACK dgeqr2 order).
    for (int j = 0; j < b; ++j) {
        double* col = y + static_cast<std::int64_t>(j) * ld;
        const std::int64_t lo = max(r0, static_cast<std::int64_t>(j));
        double acc = 0.0;
        for (std::int64_t i = max(lo, static_cast<std::int64_t>(j) + 1) + threadIdx.x; i < r1; i += blockDim.x)
            acc = fma(col[i], col[i], acc);
        const double sigma = grid_reduce_sum(grid, acc, part, sh);
        const double alpha = col[j];
        double beta, tau, scale;
        if (sigma == 0.0) {
            tau = 0.0; beta = alpha; scale = 1.0;
        } else {
            const double nrm = sqrt(alpha * alpha + sigma);
            beta = alpha >= 0.0 ? -nrm : nrm;
            tau = (beta - alpha) / beta;
            scale = 1.0 / (alpha - beta);
        }
        for (std::int64_t i = max(lo, static_cast<std::int64_t>(j) + 1) + threadIdx.x; i < r1; i += blockDim.x)
            col[i] *= scale;
        __syncthreads();
        const int nv = b - j - 1;
        // w_c = v^T y(j:, c), the v_j = 1 term taken by the owner of row j
        for (int c = 0; c < nv; ++c) {
            const double* yc = y + static_cast<std::int64_t>(j + 1 + c) * ld;
            double a2 = 0.0;
            for (std::int64_t i = lo + threadIdx.x; i < r1; i += blockDim.x)
                a2 = fma(i == j ? 1.0 : col[i], yc[i], a2);
            const double s = block_sum<kHhThreads>(a2, sh);
            if (threadIdx.x == 0) part[blockIdx.x * nv + c] = s;
        }
        grid_reduce_vec(grid, nv, part, wv);
        for (int c = 0; c < nv; ++c) {
            double* yc = y + static_cast<std::int64_t>(j + 1 + c) * ld;
            const double f = tau * wv[c];
            for (std::int64_t i = lo + threadIdx.x; i < r1; i += blockDim.x)
                yc[i] = fma(-f, i == j ? 1.0 : col[i], yc[i]);
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            taus[j] = tau;
            r[j + static_cast<std::int64_t>(j) * ldr] = beta;
        }
        grid.sync();
    }
    // R strictly-upper part = y(i, c), i < c; zeros below the diagonal.
    if (blockIdx.x == 0) {
        for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
            const int i = idx % b, c = idx / b;
            if (i < c) r[i + static_cast<std::int64_t>(c) * ldr] = y[i + static_cast<std::int64_t>(c) * ld];
            else if (i > c) r[i + static_cast<std::int64_t>(c) * ldr] = 0.0;
        }
    }
    // Q = H_0 ... H_{b-1} [I; 0] into qs (m x b, ld m), backward accumulation (dorg2r order).
    for (int c = 0; c < b; ++c)
        for (std::int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x)
            qs[i + static_cast<std::int64_t>(c) * m] = (i == c) ? 1.0 : 0.0;
    grid.sync();
    for (int j = b - 1; j >= 0; --j) {
        const double tau = taus[j];
        const double* v = y + static_cast<std::int64_t>(j) * ld;
        const std::int64_t lo = max(r0, static_cast<std::int64_t>(j));
        const int nv = b - j;
        for (int c = 0; c < nv; ++c) {
            const double* qc = qs + static_cast<std::int64_t>(j + c) * m;
            double a2 = 0.0;
            for (std::int64_t i = lo + threadIdx.x; i < r1; i += blockDim.x)
                a2 = fma(i == j ? 1.0 : v[i], qc[i], a2);
            const double s = block_sum<kHhThreads>(a2, sh);
            if (threadIdx.x == 0) part[blockIdx.x * nv + c] = s;
        }
        grid_reduce_vec(grid, nv, part, wv);
        for (int c = 0; c < nv; ++c) {
            double* qc = qs + static_cast<std::int64_t>(j + c) * m;
            const double f = tau * wv[c];
            for (std::int64_t i = lo + threadIdx.x; i < r1; i += blockDim.x)
                qc[i] = fma(-f, i == j ? 1.0 : v[i], qc[i]);
        }
        grid.sync();
    }
    // Sign post-pass (qr.hpp:15-18): diag(R) >= 0. Copy Q back into y.
    for (int c = threadIdx.x; c < b; c += blockDim.x)
        sgn[c] = r[c + static_cast<std::int64_t>(c) * ldr] < 0.0 ? -1.0 : 1.0;
    __syncthreads();
    for (int c = 0; c < b; ++c)
        for (std::int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x)
            y[i + static_cast<std::int64_t>(c) * ld] = sgn[c] * qs[i + static_cast<std::int64_t>(c) * m];
    if (blockIdx.x == 0) {
        for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
            const int i = idx % b, c = idx / b;
            if (i <= c) r[i + static_cast<std::int64_t>(c) * ldr] *= sgn[i];
        }
    }
}

int grid_for(std::int64_t total, int threads) {
    const std::int64_t want = ceil_div(total, threads);
    return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(want, 8L * gemm_num_sms())));
}

}  // namespace

void scale_matrix(cudaStream_t st, const MatView& c, double beta) {
    if (c.rows * c.cols == 0) return;
    launch_pdl(scale_kernel, dim3(grid_for(c.rows * c.cols, 256)), dim3(256), 0, st, c, beta);
    QB_LAUNCH_CHECK();
}

void copy_matrix(cudaStream_t st, const MatView& s, const MatView& d) {
    if (s.rows != d.rows || s.cols != d.cols) throw QbError(kDimensionError, "copy_matrix: shape");
    if (s.rows * s.cols == 0) return;
    launch_pdl(copy_kernel, dim3(grid_for(s.rows * s.cols, 256)), dim3(256), 0, st, s, d);
    QB_LAUNCH_CHECK();
}

void add_matrix(cudaStream_t st, const MatView& s, const MatView& d, double alpha) {
    if (s.rows != d.rows || s.cols != d.cols) throw QbError(kDimensionError, "add_matrix: shape");
    if (s.rows * s.cols == 0) return;
    launch_pdl(add_kernel, dim3(grid_for(s.rows * s.cols, 256)), dim3(256), 0, st, s, d, alpha);
    QB_LAUNCH_CHECK();
}

void set_identity(cudaStream_t st, const MatView& c) {
    if (c.rows * c.cols == 0) return;
    identity_kernel<<<grid_for(c.rows * c.cols, 256), 256, 0, st>>>(c);
    QB_LAUNCH_CHECK();
}

void sum_squares(cudaStream_t st, Workspace& ws, const MatView& v, double* out) {
    const std::int64_t outer = v.rowmajor ? v.rows : v.cols;
    const std::int64_t inner = v.rowmajor ? v.cols : v.rows;
    if (outer * inner == 0) {
        QB_CUDA(cudaMemsetAsync(out, 0, sizeof(double), st));
        return;
    }
    const int nblk = static_cast<int>(std::min<std::int64_t>(
        std::max<std::int64_t>(1, ceil_div(outer * inner, 8 * kRedThreads)), 4L * gemm_num_sms()));
    double* part = ws.get(static_cast<std::size_t>(nblk));
    const std::int64_t total = outer * inner;
    if (v.ld == inner && total % 2 == 0 && (reinterpret_cast<std::uintptr_t>(v.p) & 15) == 0 && total >= 65536)
        sumsq_flat_stage1<<<nblk, kRedThreads, 0, st>>>(reinterpret_cast<const double2*>(v.p), total / 2, part);
    else
        sumsq_stage1<<<nblk, kRedThreads, 0, st>>>(v.p, outer, inner, v.ld, part);
    QB_LAUNCH_CHECK();
    sumsq_stage2<<<1, kRedThreads, 0, st>>>(part, nblk, out);
    QB_LAUNCH_CHECK();
}

void sum_squares_vec(cudaStream_t st, Workspace& ws, const double* x, std::int64_t n, double* out) {
    MatView v{const_cast<double*>(x), n, 1, n, false};
    sum_squares(st, ws, v, out);
}

void column_sumsq(cudaStream_t st, Workspace& ws, const MatView& v, double* out) {
    if (v.cols == 0) return;
    if (v.rows == 0) {
        QB_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * v.cols, st));
        return;
    }
    // many short row chunks: each thread walks only ~16-32 rows (8 loads in flight), the fixed-order
    // stage-2 warp sums the chunk partials (was 2 x SMs chunks: 27 us for a 5e4 x 50 block)
    const std::int64_t target = 16L * gemm_num_sms();
    const std::int64_t chunk = std::max<std::int64_t>(16, ceil_div(v.rows, target));
    const int nblk = static_cast<int>(ceil_div(v.rows, chunk));
    double* part = ws.get(static_cast<std::size_t>(nblk) * v.cols);
    const int thr = static_cast<int>(std::min<std::int64_t>(256, round_up(v.cols, 32)));
    launch_pdl(colsumsq_stage1, dim3(nblk), dim3(thr), 0, st, v, chunk, part);
    QB_LAUNCH_CHECK();
    launch_pdl(colsumsq_stage2, dim3(static_cast<unsigned>(v.cols)), dim3(kRedThreads), 0, st,
               static_cast<const double*>(part), nblk, static_cast<std::int64_t>(v.cols), out);
    QB_LAUNCH_CHECK();
}

template <int BP>
void launch_chol_small(cudaStream_t st, const double* g, std::int64_t ldg, int b, double* r, double* rinv,
                       std::int64_t ldr, SmallStatus* status) {
    static PerDevice<bool> setup;
    setup.get([] {
        QB_CUDA(cudaFuncSetAttribute(chol_small_kernel<BP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     CholCfg<BP>::SMEM));
        return true;
    });
    chol_small_kernel<BP><<<1, kCholThreads, CholCfg<BP>::SMEM, st>>>(g, ldg, b, r, rinv, ldr, status);
}

void chol_small(cudaStream_t st, const double* g, std::int64_t ldg, int b, double* r, double* rinv,
                std::int64_t ldr, SmallStatus* status) {
    if (b < 1 || b > kSmallMax) throw QbError(kDimensionError, "chol_small: block width out of range");
    // tile edge T with 16 * T >= b
    switch (static_cast<int>(round_up(b, 16))) {
        case 16: launch_chol_small<16>(st, g, ldg, b, r, rinv, ldr, status); break;
        case 32: launch_chol_small<32>(st, g, ldg, b, r, rinv, ldr, status); break;
        case 48: launch_chol_small<48>(st, g, ldg, b, r, rinv, ldr, status); break;
        case 64: launch_chol_small<64>(st, g, ldg, b, r, rinv, ldr, status); break;
        case 80: launch_chol_small<80>(st, g, ldg, b, r, rinv, ldr, status); break;
        case 96: launch_chol_small<96>(st, g, ldg, b, r, rinv, ldr, status); break;
        default: launch_chol_small<112>(st, g, ldg, b, r, rinv, ldr, status); break;
    }
    QB_LAUNCH_CHECK();
}

void chol_wide(cudaStream_t st, double* w, std::int64_t ldw, int l, double* r, double* rinv, std::int64_t ldr,
               SmallStatus* stats) {
    if (l < 1) throw QbError(kDimensionError, "chol_wide: empty");
    static PerDevice<int> setup;
    const int grid = setup.get([] {
        QB_CUDA(cudaFuncSetAttribute(chol_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kCwSmemBytes));
        int per_sm = 0;
        QB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chol_wide_kernel, kCholThreads, kCwSmemBytes));
        return std::max(1, std::min(per_sm, 1) * gemm_num_sms());
    });
    CholWideArgs a{w, ldw, r, rinv, ldr, l, static_cast<int>(ceil_div(l, kCwNb)), stats};
    void* args[] = {&a};
    QB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(chol_wide_kernel), grid, kCholThreads, args,
                                        kCwSmemBytes, st));
    QB_LAUNCH_CHECK();
}

template <int BP>
void launch_cholqr2_panel(cudaStream_t st, PanelArgs& a, int grid_cap) {
    using C = PanelCfg<BP>;
    auto kern = cholqr2_panel_kernel<BP>;
    a.nsub = static_cast<int>(ceil_div(a.rows, C::SUB));
    // ring depth: QBFAC_PANEL_STAGES (2..STAGES) trades in-flight sub-tiles for a second CTA per SM
    const char* st_env = std::getenv("QBFAC_PANEL_STAGES");
    a.nstages = st_env ? std::max(2, std::min(C::STAGES, std::atoi(st_env))) : C::STAGES;
    const int smem = std::max<int>((a.nstages * C::SUB + BP) * C::LD * 8, CholCfg<BP>::SMEM);
    static PerDevice<bool> setup;
    setup.get([&] {
        QB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
        return true;
    });
    int per_sm = 0;
    QB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCholThreads, smem));
    if (per_sm < 1) throw QbError(kError, "cholqr2_panel: kernel does not fit on an SM");
    const int grid = std::max(1, std::min(std::min(a.nsub, grid_cap), per_sm * gemm_num_sms()));
    static const bool tm_on = [] {
        const char* e = std::getenv("QBFAC_PANEL_TM");
        return !(e && e[0] == '0');
    }();
    a.use_tm_y = a.use_tm_t1 = 0;
    // tensor-map sub-tiles (same-box A/B against the bulk row copies): 1e5 x 50 Gram 26.6 -> 15.9 us,
    // 2e6 x 100 panel 4.41 -> 4.33 ms
    if (tm_on && a.rows > 0) {
        if (a.ldy % 2 == 0 && (reinterpret_cast<std::uintptr_t>(a.y) & 15) == 0) {
            make_tensor_map_2d(&a.tm_y, a.y, a.b, a.rows, a.ldy, C::LD, C::SUB);
            a.use_tm_y = 1;
        }
        if (a.b % 2 == 0 && (reinterpret_cast<std::uintptr_t>(a.t1) & 15) == 0) {
            make_tensor_map_2d(&a.tm_t1, a.t1, a.b, a.rows, a.b, C::LD, C::SUB);
            a.use_tm_t1 = 1;
        }
    }
    // cooperative + programmatic stream serialization: the panel's CTAs may become resident while the
    // previous kernel drains (the kernel waits on griddepcontrol before touching memory)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kCholThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    QB_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    QB_LAUNCH_CHECK();
}

void cholqr2_panel(cudaStream_t st, Workspace& ws, const double* y, std::int64_t rows, int b, std::int64_t ldy,
                   double* t1, double* q, std::int64_t ldq, double* g, double* ra, double* rainv, double* rb,
                   double* rbinv, SmallStatus* st0, SmallStatus* st1, unsigned* gbar, bool span_only) {
    if (b < 1 || b > kSmallMax) throw QbError(kDimensionError, "cholqr2_panel: width out of range");
    const int bp = static_cast<int>(round_up(b, 16));
    PanelArgs a{};
    a.span_only = span_only ? 1 : 0;
    a.y = y; a.ldy = ldy; a.t1 = t1; a.q = q; a.ldq = ldq; a.rows = rows; a.b = b;
    a.g = g; a.ra = ra; a.rainv = rainv; a.rb = rb; a.rbinv = rbinv; a.st0 = st0; a.st1 = st1; a.gbar = gbar;
    if (bp <= 32 && rows > 0 && rows <= static_cast<std::int64_t>(kClusterMaxCtas) * kClusterRowsPerCta &&
        cluster_panel_enabled()) {
        if (bp == 16) launch_cholqr2_cluster<16>(st, a);
        else launch_cholqr2_cluster<32>(st, a);
        QB_LAUNCH_CHECK();
        return;
    }
    const int cap = 2 * gemm_num_sms();  // up to 2 CTAs per SM with a shallow ring
    a.part = ws.get(static_cast<std::size_t>(cap) * bp * bp);
    switch (bp) {
        case 16: launch_cholqr2_panel<16>(st, a, cap); break;
        case 32: launch_cholqr2_panel<32>(st, a, cap); break;
        case 48: launch_cholqr2_panel<48>(st, a, cap); break;
        case 64: launch_cholqr2_panel<64>(st, a, cap); break;
        case 80: launch_cholqr2_panel<80>(st, a, cap); break;
        case 96: launch_cholqr2_panel<96>(st, a, cap); break;
        default: launch_cholqr2_panel<112>(st, a, cap); break;
    }
}

void chol_wide_trace(unsigned long long* out) {
    QB_CUDA(cudaMemcpyFromSymbol(out, g_cw_trace, sizeof(unsigned long long) * 64 * 4));
}

void panel_trace(unsigned long long* out) {
    QB_CUDA(cudaMemcpyFromSymbol(out, g_panel_trace, sizeof(unsigned long long) * kPanelTraceSlots));
    QB_CUDA(cudaMemcpyFromSymbol(out + kPanelTraceSlots, g_chol_trace, sizeof(long long) * 32));
}

int jacobi_svd(cudaStream_t st, double* nmat, double* w, int r, unsigned* gbar, int max_sweeps) {
    if (r < 1) return 0;
    const int rp = r + (r & 1);
    const int grid = std::max(1, std::min(gemm_num_sms(), (rp / 2 + 7) / 8));
    unsigned* rotated = nullptr;
    int* sweeps = nullptr;
    const int nver = r / 8 + 4;  // per-block visit counters of the Gram-based kernel
    const std::size_t ctl_bytes = sizeof(unsigned) * (max_sweeps + 1) + sizeof(int) + sizeof(unsigned) * nver;
    QB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rotated), ctl_bytes, st));
    sweeps = reinterpret_cast<int*>(rotated + max_sweeps + 1);
    unsigned* ver = reinterpret_cast<unsigned*>(sweeps + 1);
    QB_CUDA(cudaMemsetAsync(rotated, 0, ctl_bytes, st));
    // block Jacobi when 2 nb columns of N fit in shared memory (nb = 8, 4, 2 or 1)
    int nb = 0;
    const char* nb_env = std::getenv("QBFAC_JACOBI_NB");
    const int nb_max = nb_env ? std::max(1, std::min(8, std::atoi(nb_env))) : 8;
    for (int cand : {8, 4, 2, 1})
        if (cand <= nb_max && (2 * cand * static_cast<std::int64_t>(r) + 4 * cand * cand) * 8 <= 200 * 1024 &&
            r > 2 * cand) {
            nb = cand;
            break;
        }
    // rotation threshold |g_pq| <= tol sqrt(g_pp g_qq): sqrt(r) eps (LAPACK dgesvj's choice), the
    // rounding level of an r-long dot product; a tighter threshold only chases that noise
    const double tol = std::max(1e-15, 2.220446049250313e-16 * std::sqrt(static_cast<double>(r)));
    const char* force_scalar = std::getenv("QBFAC_JACOBI_SCALAR");
    const char* gram_env = std::getenv("QBFAC_JACOBI_GRAM");
    const bool use_gram = nb == 8 && r <= 1568 && !(gram_env && gram_env[0] == '0');
    if (use_gram && !(force_scalar && force_scalar[0] == '1')) {
        const int nblk = static_cast<int>(2 * ceil_div(ceil_div(r, 8), 2));
        // one cluster of 2 CTAs per block pair (each stages half of the rows) when the pairs fit the
        // SMs twice; QBFAC_JACOBI_CLUSTER=1 keeps one CTA per pair
        const char* cl_env = std::getenv("QBFAC_JACOBI_CLUSTER");
        int ncta = cl_env ? std::max(1, std::min(kJgMaxCta, std::atoi(cl_env))) : kJgMaxCta;
        if (r < 64) ncta = 1;
        auto smem_for = [&](int nc) {
            return static_cast<int>(
                (2 * kJgNc * round_up(ceil_div(r, nc), 2) + (2 + kJgGramWarps + 2 * kJgMaxCta) * kJgNc * kJgNc) * 8);
        };
        if (smem_for(ncta) > 224 * 1024) ncta = kJgMaxCta;
        const int smem = smem_for(ncta);
        static PerDevice<bool> setup;
        setup.get([] {
            QB_CUDA(cudaFuncSetAttribute(jacobi_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));
            return true;
        });
        const int gb = std::max(1, std::min(nblk / 2, gemm_num_sms() / ncta)) * ncta;
        const char* tr = std::getenv("QBFAC_JACOBI_TRACE");
        const char* in_env = std::getenv("QBFAC_JACOBI_INNER");
        const int inner = in_env ? std::max(1, std::min(8, std::atoi(in_env))) : 1;
        JacobiGramArgs a{nmat, w, r, nblk, max_sweeps, inner, tol, gbar, rotated, ver, sweeps, tr && tr[0] == '1' ? 1 : 0};
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(gb));
        cfg.blockDim = dim3(kJbThreads);
        cfg.dynamicSmemBytes = static_cast<size_t>(smem);
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = static_cast<unsigned>(ncta);
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        QB_CUDA(cudaLaunchKernelEx(&cfg, jacobi_gram_kernel, a));
    } else if (nb > 0 && !(force_scalar && force_scalar[0] == '1')) {
        const int nblk = static_cast<int>(2 * ceil_div(ceil_div(r, nb), 2));
        const int smem = static_cast<int>((2 * nb * static_cast<std::int64_t>(r) + 4 * nb * nb) * 8);
        static PerDevice<bool> setup;
        setup.get([] {
            QB_CUDA(cudaFuncSetAttribute(jacobi_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            return true;
        });
        int per_sm = 0;
        QB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_block_kernel, kJbThreads, smem));
        const int gb = std::max(1, std::min(nblk / 2, std::max(per_sm, 1) * gemm_num_sms()));
        const char* tr = std::getenv("QBFAC_JACOBI_TRACE");
        JacobiBlockArgs a{nmat, w, r, nb, nblk, max_sweeps, tol, gbar, rotated, sweeps, tr && tr[0] == '1' ? 1 : 0};
        void* args[] = {&a};
        QB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(jacobi_block_kernel), gb, kJbThreads, args, smem, st));
    } else {
        JacobiArgs a{nmat, w, r, rp, max_sweeps, tol, gbar, rotated, sweeps};
        void* args[] = {&a};
        QB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(jacobi_svd_kernel), grid, 256, args, 0, st));
    }
    QB_LAUNCH_CHECK();
    int h = 0;
    QB_CUDA(cudaMemcpyAsync(&h, sweeps, sizeof(int), cudaMemcpyDeviceToHost, st));
    QB_CUDA(cudaStreamSynchronize(st));
    QB_CUDA(cudaFreeAsync(rotated, st));
    return h;
}

void trmm_upper_small(cudaStream_t st, const double* a, const double* b, double* c, int n,
                      std::int64_t ld) {
    trmm_upper_pair(st, a, b, c, nullptr, nullptr, nullptr, n, ld);
}

void trmm_upper_pair(cudaStream_t st, const double* a0, const double* b0, double* c0, const double* a1,
                     const double* b1, double* c1, int n, std::int64_t ld) {
    if (n < 1 || n > kSmallMax) throw QbError(kDimensionError, "trmm_upper: size out of range");
    static PerDevice<bool> setup;
    setup.get([] {
        QB_CUDA(cudaFuncSetAttribute(trmm_upper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     2 * kSmallMax * (kSmallMax + 1) * 8));
        return true;
    });
    TrmmPair p{{a0, a1}, {b0, b1}, {c0, c1}};
    const int smem = 2 * n * (n + 1) * static_cast<int>(sizeof(double));
    launch_pdl(trmm_upper_kernel, dim3(c1 ? 2 : 1), dim3(1024), static_cast<std::size_t>(smem), st, p, n, ld);
    QB_LAUNCH_CHECK();
}

void tri_inverse_small(cudaStream_t st, const double* r, double* rinv, int n, std::int64_t ld) {
    tri_inverse_kernel<<<1, 128, 0, st>>>(r, rinv, n, ld);
    QB_LAUNCH_CHECK();
}

void indicator_step(cudaStream_t st, double* e_dev, const double* norms, int b, double eps2, int check,
                    IndicatorOut* out) {
    launch_pdl(indicator_kernel, dim3(1), dim3(32), 0, st, e_dev, norms, b, eps2, check, out);
    QB_LAUNCH_CHECK();
}

void householder_panel(cudaStream_t st, Workspace& ws, double* y, std::int64_t m, int b, std::int64_t ld,
                       double* r, std::int64_t ldr) {
    if (b < 1 || b > kSmallMax) throw QbError(kDimensionError, "householder_panel: width out of range");
    if (m < b) throw QbError(kDimensionError, "orth_qr: rows < cols");
    int per_sm = 0;
    QB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, householder_panel_kernel, kHhThreads, 0));
    int grid = std::max(1, std::min<int>(per_sm * gemm_num_sms(), static_cast<int>(ceil_div(m, 512))));
    grid = std::min(grid, 2 * gemm_num_sms());
    const std::size_t part_n = static_cast<std::size_t>(grid) * kSmallMax;
    double* base = ws.get(part_n + static_cast<std::size_t>(m) * b + kSmallMax);
    double* part = base;
    double* qs = base + part_n;
    double* taus = qs + static_cast<std::size_t>(m) * b;
    void* args[] = {&y, &m, &b, &ld, &r, &ldr, &part, &qs, &taus};
    QB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(householder_panel_kernel), grid, kHhThreads,
                                        args, 0, st));
    QB_LAUNCH_CHECK();
}

}  // namespace qbgpu
