// CSR passes over a sparse A for sm_100a.
//
// Replaces the reference drivers csr_gemm_n (Y = A X, one column of X at a
// time, A swept p times; /root/reference/proj/src/kernels_drivers.cpp:67-79 with
// sparse_dot kernels_avx2.cpp:123-135) and csr_gemm_t (Y += A^T X by scalar
// scatter, kernels_drivers.cpp:81-94).
//
// B200 design: A is read ONCE per pass for all w right-hand sides. Block vectors
// are row-major so that every nonzero gathers one contiguous row of X (8*w
// bytes, coalesced across the warp) and every output row is one coalesced store.
// A warp owns a row; lanes load 32 (col, val) pairs at a time and broadcast them
// with shuffles. A^T X runs the same gather kernel over a transposed CSR built on
// the device in a stable (row-ascending) order, so there are no atomics and the
// result is bitwise reproducible.

#include "sparse.cuh"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace qbgpu {

namespace {

// acc += sum_{e in [e0, e1)} v[e] * X[ci[e], :] for this lane's columns. Lanes load 32
// (col, val) pairs at once and broadcast them; four nonzeros are gathered per step
// into four independent accumulator sets (more loads in flight, no serial FMA chain),
// combined in a fixed order at the end (deterministic).
template <int NQ>
__device__ __forceinline__ void row_dot(const std::int32_t* __restrict__ ci, const double* __restrict__ v,
                                        const double* __restrict__ x, std::int64_t ldx, int w, std::int64_t e0,
                                        std::int64_t e1, int lane, double (&acc)[NQ]) {
    double a1[NQ], a2[NQ], a3[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) a1[q] = a2[q] = a3[q] = 0.0;
    for (std::int64_t eb = e0; eb < e1; eb += 32) {
        const int cnt = static_cast<int>(e1 - eb < 32 ? e1 - eb : 32);
        std::int32_t my_c = 0;
        double my_v = 0.0;
        if (lane < cnt) {
            my_c = __ldg(ci + eb + lane);
            my_v = __ldg(v + eb + lane);
        }
        int j = 0;
        for (; j + 4 <= cnt; j += 4) {
            const double* x0 = x + static_cast<std::int64_t>(__shfl_sync(0xffffffffu, my_c, j)) * ldx;
            const double* x1 = x + static_cast<std::int64_t>(__shfl_sync(0xffffffffu, my_c, j + 1)) * ldx;
            const double* x2 = x + static_cast<std::int64_t>(__shfl_sync(0xffffffffu, my_c, j + 2)) * ldx;
            const double* x3 = x + static_cast<std::int64_t>(__shfl_sync(0xffffffffu, my_c, j + 3)) * ldx;
            const double v0 = __shfl_sync(0xffffffffu, my_v, j), v1 = __shfl_sync(0xffffffffu, my_v, j + 1);
            const double v2 = __shfl_sync(0xffffffffu, my_v, j + 2), v3 = __shfl_sync(0xffffffffu, my_v, j + 3);
            double g0[NQ], g1[NQ], g2[NQ], g3[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int col = lane + 32 * q;
                const bool ok = col < w;
                g0[q] = ok ? __ldg(x0 + col) : 0.0;
                g1[q] = ok ? __ldg(x1 + col) : 0.0;
                g2[q] = ok ? __ldg(x2 + col) : 0.0;
                g3[q] = ok ? __ldg(x3 + col) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                acc[q] = fma(v0, g0[q], acc[q]);
                a1[q] = fma(v1, g1[q], a1[q]);
                a2[q] = fma(v2, g2[q], a2[q]);
                a3[q] = fma(v3, g3[q], a3[q]);
            }
        }
        for (; j < cnt; ++j) {
            const double* xr = x + static_cast<std::int64_t>(__shfl_sync(0xffffffffu, my_c, j)) * ldx;
            const double a = __shfl_sync(0xffffffffu, my_v, j);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int col = lane + 32 * q;
                if (col < w) acc[q] = fma(a, __ldg(xr + col), acc[q]);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = (acc[q] + a1[q]) + (a2[q] + a3[q]);
}

// 16-byte variant: lane owns the column pairs (2 lane + 64 q, +1), so one load instruction
// moves a 512-byte slice of an X row (half the L2 requests of the 8-byte version). Needs
// ldx even and a 16-byte aligned x; for odd w the pair straddling w reads the row padding,
// whose lane-local accumulator is never stored.
template <int NQ2>
__device__ __forceinline__ void row_dot2(const std::int32_t* __restrict__ ci, const double* __restrict__ v,
                                         const double* __restrict__ x, std::int64_t ldx, int w, std::int64_t e0,
                                         std::int64_t e1, int lane, double2 (&acc)[NQ2]) {
    double2 a1[NQ2], a2[NQ2], a3[NQ2];
#pragma unroll
    for (int q = 0; q < NQ2; ++q) a1[q] = a2[q] = a3[q] = make_double2(0.0, 0.0);
    for (std::int64_t eb = e0; eb < e1; eb += 32) {
        const int cnt = static_cast<int>(e1 - eb < 32 ? e1 - eb : 32);
        std::int32_t my_c = 0;
        double my_v = 0.0;
        if (lane < cnt) {
            my_c = __ldg(ci + eb + lane);
            my_v = __ldg(v + eb + lane);
        }
        int j = 0;
        for (; j + 4 <= cnt; j += 4) {
            const double2* x0 = reinterpret_cast<const double2*>(x + static_cast<std::int64_t>(__shfl_sync(0xffffffffu, my_c, j)) * ldx);
            const double2* x1 = reinterpret_cast<const double2*>(x + static_cast<std::int64_t>(__shfl_sync(0xffffffffu, my_c, j + 1)) * ldx);
            const double2* x2 = reinterpret_cast<const double2*>(x + static_cast<std::int64_t>(__shfl_sync(0xffffffffu, my_c, j + 2)) * ldx);
            const double2* x3 = reinterpret_cast<const double2*>(x + static_cast<std::int64_t>(__shfl_sync(0xffffffffu, my_c, j + 3)) * ldx);
            const double v0 = __shfl_sync(0xffffffffu, my_v, j), v1 = __shfl_sync(0xffffffffu, my_v, j + 1);
            const double v2 = __shfl_sync(0xffffffffu, my_v, j + 2), v3 = __shfl_sync(0xffffffffu, my_v, j + 3);
            double2 g0[NQ2], g1[NQ2], g2[NQ2], g3[NQ2];
#pragma unroll
            for (int q = 0; q < NQ2; ++q) {
                const int pc = lane + 32 * q;  // pair index
                const bool ok = 2 * pc < w;
                const double2 z = make_double2(0.0, 0.0);
                g0[q] = ok ? __ldg(x0 + pc) : z;
                g1[q] = ok ? __ldg(x1 + pc) : z;
                g2[q] = ok ? __ldg(x2 + pc) : z;
                g3[q] = ok ? __ldg(x3 + pc) : z;
            }
#pragma unroll
            for (int q = 0; q < NQ2; ++q) {
                acc[q].x = fma(v0, g0[q].x, acc[q].x);
                acc[q].y = fma(v0, g0[q].y, acc[q].y);
                a1[q].x = fma(v1, g1[q].x, a1[q].x);
                a1[q].y = fma(v1, g1[q].y, a1[q].y);
                a2[q].x = fma(v2, g2[q].x, a2[q].x);
                a2[q].y = fma(v2, g2[q].y, a2[q].y);
                a3[q].x = fma(v3, g3[q].x, a3[q].x);
                a3[q].y = fma(v3, g3[q].y, a3[q].y);
            }
        }
        for (; j < cnt; ++j) {
            const double2* xr = reinterpret_cast<const double2*>(x + static_cast<std::int64_t>(__shfl_sync(0xffffffffu, my_c, j)) * ldx);
            const double a = __shfl_sync(0xffffffffu, my_v, j);
#pragma unroll
            for (int q = 0; q < NQ2; ++q) {
                const int pc = lane + 32 * q;
                if (2 * pc < w) {
                    const double2 g = __ldg(xr + pc);
                    acc[q].x = fma(a, g.x, acc[q].x);
                    acc[q].y = fma(a, g.y, acc[q].y);
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NQ2; ++q) {
        acc[q].x = (acc[q].x + a1[q].x) + (a2[q].x + a3[q].x);
        acc[q].y = (acc[q].y + a1[q].y) + (a2[q].y + a3[q].y);
    }
}

template <int NQ2>
__device__ __forceinline__ void store_row2(double* __restrict__ yr, int w, int lane, const double2 (&acc)[NQ2],
                                           double alpha, double beta) {
#pragma unroll
    for (int q = 0; q < NQ2; ++q) {
        const int col = 2 * (lane + 32 * q);
        if (col + 1 < w) {
            double2 r = make_double2(alpha * acc[q].x, alpha * acc[q].y);
            if (beta != 0.0) {
                const double2 o = *reinterpret_cast<const double2*>(yr + col);
                r.x += beta * o.x;
                r.y += beta * o.y;
            }
            *reinterpret_cast<double2*>(yr + col) = r;
        } else if (col < w) {
            const double r = alpha * acc[q].x;
            yr[col] = beta == 0.0 ? r : r + beta * yr[col];
        }
    }
}

template <int NQ2, int MINB = 4>
__global__ void __launch_bounds__(256, MINB)
csr_spmm_kernel2(std::int64_t rows, const std::int64_t* __restrict__ rp, const std::int32_t* __restrict__ ci,
                 const double* __restrict__ v, const double* __restrict__ x, std::int64_t ldx,
                 double* __restrict__ y, std::int64_t ldy, int w, double alpha, double beta, bool y_vec,
                 std::int64_t heavy_thr, std::int64_t nseg, const std::int64_t* __restrict__ seg,
                 double* __restrict__ partial) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const std::int64_t warp = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const std::int64_t nwarps = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (std::int64_t s = warp; s < nseg; s += nwarps) {  // heavy-row segments first (see csr_spmm_kernel)
        double2 acc[NQ2];
#pragma unroll
        for (int q = 0; q < NQ2; ++q) acc[q] = make_double2(0.0, 0.0);
        row_dot2<NQ2>(ci, v, x, ldx, w, seg[nseg + s], seg[2 * nseg + s], lane, acc);
#pragma unroll
        for (int q = 0; q < NQ2; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = 2 * (lane + 32 * q) + h;
                if (col < w) partial[s * w + col] = h ? acc[q].y : acc[q].x;
            }
    }
    for (std::int64_t i = (warp + nwarps - nseg % nwarps) % nwarps; i < rows; i += nwarps) {
        const std::int64_t e0 = rp[i], e1 = rp[i + 1];
        if (e1 - e0 > heavy_thr) continue;  // heavy rows: segment kernels
        double2 acc[NQ2];
#pragma unroll
        for (int q = 0; q < NQ2; ++q) acc[q] = make_double2(0.0, 0.0);
        row_dot2<NQ2>(ci, v, x, ldx, w, e0, e1, lane, acc);
        double* yr = y + i * ldy;
        if (y_vec) {
            store_row2<NQ2>(yr, w, lane, acc, alpha, beta);
        } else {
#pragma unroll
            for (int q = 0; q < NQ2; ++q)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int col = 2 * (lane + 32 * q) + h;
                    if (col < w) {
                        const double r = alpha * (h ? acc[q].y : acc[q].x);
                        yr[col] = beta == 0.0 ? r : r + beta * yr[col];
                    }
                }
        }
    }
}



// Heavy rows: y[row] = alpha * sum over its segments (in order) + beta * y[row].
__global__ void csr_heavy_combine_kernel(std::int64_t nrows, const std::int64_t* __restrict__ hr,
                                         const double* __restrict__ partial, double* __restrict__ y, std::int64_t ldy,
                                         int w, double alpha, double beta) {
    for (std::int64_t h = blockIdx.x; h < nrows; h += gridDim.x) {
        const std::int64_t row = hr[h], s0 = hr[nrows + h], ns = hr[2 * nrows + h];
        for (int col = threadIdx.x; col < w; col += blockDim.x) {
            double s = 0.0;
            for (std::int64_t q = 0; q < ns; ++q) s += partial[(s0 + q) * w + col];
            double* yp = y + row * ldy + col;
            const double r = alpha * s;
            *yp = beta == 0.0 ? r : r + beta * (*yp);
        }
    }
}

template <int NQ>
__global__ void __launch_bounds__(256)
csr_spmm_kernel(std::int64_t rows, const std::int64_t* __restrict__ rp, const std::int32_t* __restrict__ ci,
                const double* __restrict__ v, const double* __restrict__ x, std::int64_t ldx,
                double* __restrict__ y, std::int64_t ldy, int w, double alpha, double beta, std::int64_t heavy_thr,
                std::int64_t nseg, const std::int64_t* __restrict__ seg, double* __restrict__ partial) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const std::int64_t warp = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const std::int64_t nwarps = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
    // heavy-row segments first (uniform 256-entry work), then the light rows fill the tail; one
    // launch, so warps that draw short rows move on instead of idling behind a second kernel
    for (std::int64_t s = warp; s < nseg; s += nwarps) {
        double acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
        row_dot<NQ>(ci, v, x, ldx, w, seg[nseg + s], seg[2 * nseg + s], lane, acc);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int col = lane + 32 * q;
            if (col < w) partial[s * w + col] = acc[q];
        }
    }
    for (std::int64_t i = (warp + nwarps - nseg % nwarps) % nwarps; i < rows; i += nwarps) {
        double acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
        const std::int64_t e0 = rp[i], e1 = rp[i + 1];
        if (e1 - e0 > heavy_thr) continue;  // heavy rows: segment kernels
        row_dot<NQ>(ci, v, x, ldx, w, e0, e1, lane, acc);
        double* yr = y + i * ldy;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int col = lane + 32 * q;
            if (col < w) {
                const double r = alpha * acc[q];
                yr[col] = beta == 0.0 ? r : r + beta * yr[col];
            }
        }
    }
}

// ---- transposed CSR (stable, deterministic) ---------------------------------------
__global__ void count_cols_kernel(std::int64_t nnz, const std::int32_t* __restrict__ ci, int* __restrict__ cnt) {
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < nnz;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        atomicAdd(cnt + ci[e], 1);
}

// Per-chunk column counts: chunk b owns rows [b*rows_per, (b+1)*rows_per).
__global__ void chunk_count_kernel(std::int64_t m, std::int64_t rows_per, const std::int64_t* __restrict__ rp,
                                   const std::int32_t* __restrict__ ci, std::int64_t n, int* __restrict__ cc) {
    const std::int64_t r0 = blockIdx.x * rows_per;
    const std::int64_t r1 = min(m, r0 + rows_per);
    if (r0 >= r1) return;
    int* mine = cc + static_cast<std::int64_t>(blockIdx.x) * n;
    for (std::int64_t e = rp[r0] + threadIdx.x; e < rp[r1]; e += blockDim.x) atomicAdd(mine + ci[e], 1);
}

// Exclusive scan over n column counts -> ct_ptr (single CTA, chunked).
__global__ void scan_kernel(std::int64_t n, const int* __restrict__ cnt, std::int64_t* __restrict__ ptr) {
    __shared__ std::int64_t part[1024];
    const std::int64_t per = (n + blockDim.x - 1) / blockDim.x;
    const std::int64_t c0 = threadIdx.x * per;
    const std::int64_t c1 = min(n, c0 + per);
    std::int64_t s = 0;
    for (std::int64_t c = c0; c < c1; ++c) s += cnt[c];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        std::int64_t run = 0;
        for (int t = 0; t < static_cast<int>(blockDim.x); ++t) {
            const std::int64_t v = part[t];
            part[t] = run;
            run += v;
        }
        ptr[n] = run;
    }
    __syncthreads();
    std::int64_t run = part[threadIdx.x];
    for (std::int64_t c = c0; c < c1; ++c) {
        ptr[c] = run;
        run += cnt[c];
    }
}

// cc[b][c] -> starting offset of chunk b inside column c (in place).
__global__ void chunk_offsets_kernel(std::int64_t n, int nchunks, const std::int64_t* __restrict__ ptr,
                                     int* __restrict__ cc, std::int64_t* __restrict__ off) {
    for (std::int64_t c = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; c < n;
         c += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        std::int64_t run = ptr[c];
        for (int b = 0; b < nchunks; ++b) {
            const int v = cc[static_cast<std::int64_t>(b) * n + c];
            off[static_cast<std::int64_t>(b) * n + c] = run;
            run += v;
        }
    }
}

// Stable placement: rows of a chunk are visited in order; within a row every column
// is distinct, so the chunk's threads can place a row's entries concurrently.
__global__ void place_kernel(std::int64_t m, std::int64_t rows_per, const std::int64_t* __restrict__ rp,
                             const std::int32_t* __restrict__ ci, const double* __restrict__ v, std::int64_t n,
                             std::int64_t* __restrict__ off, std::int32_t* __restrict__ ct_ci,
                             double* __restrict__ ct_v) {
    const std::int64_t r0 = blockIdx.x * rows_per;
    const std::int64_t r1 = min(m, r0 + rows_per);
    std::int64_t* mine = off + static_cast<std::int64_t>(blockIdx.x) * n;
    for (std::int64_t i = r0; i < r1; ++i) {
        for (std::int64_t e = rp[i] + threadIdx.x; e < rp[i + 1]; e += blockDim.x) {
            const std::int32_t c = ci[e];
            const std::int64_t pos = mine[c]++;
            ct_ci[pos] = static_cast<std::int32_t>(i);
            ct_v[pos] = v[e];
        }
        __syncthreads();
    }
}

// from_parts validation (sparse_csr.cpp:10-40): flags |= 1 structure, |= 2 non-finite.
__global__ void validate_kernel(std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* __restrict__ rp,
                                const std::int32_t* __restrict__ ci, const double* __restrict__ v,
                                int* __restrict__ flags) {
    const std::int64_t tid = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t i = tid; i < m; i += stride) {
        const std::int64_t a = rp[i], b = rp[i + 1];
        if (a > b || a < 0 || b > nnz) { atomicOr(flags, 1); continue; }
        for (std::int64_t e = a; e < b; ++e) {
            const std::int32_t c = ci[e];
            if (c < 0 || c >= n) atomicOr(flags, 1);
            if (e > a && c <= ci[e - 1]) atomicOr(flags, 1);
        }
    }
    for (std::int64_t e = tid; e < nnz; e += stride)
        if (!isfinite(v[e])) atomicOr(flags, 2);
    if (tid == 0 && (rp[0] != 0 || rp[m] != nnz)) atomicOr(flags, 1);
}

}  // namespace

std::int64_t heavy_row_threshold() {
    static const std::int64_t t = [] {
        const char* e = std::getenv("QBFAC_HEAVY_ROW");
        const long long v = e ? std::atoll(e) : 0;
        return v > 0 ? static_cast<std::int64_t>(v) : kHeavyRow;
    }();
    return t;
}

HeavyPlan make_heavy_plan(const std::int64_t* rp, std::int64_t rows, cudaStream_t st) {
    const std::int64_t thr = heavy_row_threshold();
    std::vector<std::int64_t> sr, slo, shi, hr, hs0, hns;
    for (std::int64_t i = 0; i < rows; ++i) {
        const std::int64_t len = rp[i + 1] - rp[i];
        if (len <= thr) continue;
        hr.push_back(i);
        hs0.push_back(static_cast<std::int64_t>(sr.size()));
        std::int64_t cnt = 0;
        for (std::int64_t e = rp[i]; e < rp[i + 1]; e += thr, ++cnt) {
            sr.push_back(i);
            slo.push_back(e);
            shi.push_back(std::min(rp[i + 1], e + thr));
        }
        hns.push_back(cnt);
    }
    HeavyPlan p;
    p.thr = thr;
    p.nseg = static_cast<std::int64_t>(sr.size());
    p.nrows = static_cast<std::int64_t>(hr.size());
    if (p.nseg == 0) return p;
    std::vector<std::int64_t> seg(3 * p.nseg), hrows(3 * p.nrows);
    std::copy(sr.begin(), sr.end(), seg.begin());
    std::copy(slo.begin(), slo.end(), seg.begin() + p.nseg);
    std::copy(shi.begin(), shi.end(), seg.begin() + 2 * p.nseg);
    std::copy(hr.begin(), hr.end(), hrows.begin());
    std::copy(hs0.begin(), hs0.end(), hrows.begin() + p.nrows);
    std::copy(hns.begin(), hns.end(), hrows.begin() + 2 * p.nrows);
    QB_CUDA(cudaMalloc(&p.seg, sizeof(std::int64_t) * seg.size()));
    QB_CUDA(cudaMalloc(&p.rows, sizeof(std::int64_t) * hrows.size()));
    QB_CUDA(cudaMemcpyAsync(p.seg, seg.data(), sizeof(std::int64_t) * seg.size(), cudaMemcpyHostToDevice, st));
    QB_CUDA(cudaMemcpyAsync(p.rows, hrows.data(), sizeof(std::int64_t) * hrows.size(), cudaMemcpyHostToDevice, st));
    QB_CUDA(cudaStreamSynchronize(st));
    return p;
}

void free_heavy_plan(HeavyPlan& p) {
    if (p.seg) cudaFree(p.seg);
    if (p.rows) cudaFree(p.rows);
    p = HeavyPlan{};
}

namespace {
template <int NQ2, int MINB = 4>
void spmm_launch2(cudaStream_t st, const CsrView& a, const double* x, std::int64_t ldx, double* y, std::int64_t ldy,
                  int w, double alpha, double beta, int sms, double* partial) {
    const int threads = 256;
    const int blocks = static_cast<int>(std::max<std::int64_t>(
        1, std::min<std::int64_t>(ceil_div((a.rows + a.heavy.nseg) * 32, threads), 16L * sms)));
    const bool y_vec = (ldy % 2 == 0) && ((reinterpret_cast<std::uintptr_t>(y) & 15) == 0);
    launch_pdl(csr_spmm_kernel2<NQ2, MINB>, dim3(blocks), dim3(threads), 0, st, a.rows, a.rp, a.ci, a.v, x, ldx, y, ldy, w,
               alpha, beta, y_vec, a.heavy.thr, a.heavy.nseg, static_cast<const std::int64_t*>(a.heavy.seg), partial);
    QB_LAUNCH_CHECK();
    if (a.heavy.nseg > 0) {
        csr_heavy_combine_kernel<<<static_cast<int>(std::min<std::int64_t>(a.heavy.nrows, 65535)), 128, 0, st>>>(
            a.heavy.nrows, a.heavy.rows, partial, y, ldy, w, alpha, beta);
        QB_LAUNCH_CHECK();
    }
}

template <int NQ>
void spmm_launch(cudaStream_t st, const CsrView& a, const double* x, std::int64_t ldx, double* y, std::int64_t ldy,
                 int w, double alpha, double beta, int sms, double* partial) {
    const int threads = 256;
    const int blocks = static_cast<int>(std::max<std::int64_t>(
        1, std::min<std::int64_t>(ceil_div((a.rows + a.heavy.nseg) * 32, threads), 16L * sms)));
    launch_pdl(csr_spmm_kernel<NQ>, dim3(blocks), dim3(threads), 0, st, a.rows, a.rp, a.ci, a.v, x, ldx, y, ldy, w, alpha,
               beta, a.heavy.thr, a.heavy.nseg, static_cast<const std::int64_t*>(a.heavy.seg), partial);
    QB_LAUNCH_CHECK();
    if (a.heavy.nseg > 0) {
        csr_heavy_combine_kernel<<<static_cast<int>(std::min<std::int64_t>(a.heavy.nrows, 65535)), 128, 0, st>>>(
            a.heavy.nrows, a.heavy.rows, partial, y, ldy, w, alpha, beta);
        QB_LAUNCH_CHECK();
    }
}
}  // namespace

void csr_spmm(cudaStream_t st, const CsrView& a, const double* x, std::int64_t ldx, double* y, std::int64_t ldy,
              int w, double alpha, double beta, int sms, double* partial) {
    if (a.rows == 0 || w == 0) return;
    if (a.heavy.nseg > 0 && !partial) throw QbError(kInternal, "csr_spmm: heavy rows need scratch");
    const bool x_vec = (ldx % 2 == 0) && ((reinterpret_cast<std::uintptr_t>(x) & 15) == 0) && (ldx >= w + (w & 1));
    // 16-byte gathers measured faster for 32 < w <= 64 only (config 3: +10-16 %); wider blocks
    // (config 5, w = 100) lose occupancy to the larger register footprint
    if (x_vec && w > 32 && w <= 64) return spmm_launch2<1>(st, a, x, ldx, y, ldy, w, alpha, beta, sms, partial);
    if (w <= 32) return spmm_launch<1>(st, a, x, ldx, y, ldy, w, alpha, beta, sms, partial);
    if (w <= 64) return spmm_launch<2>(st, a, x, ldx, y, ldy, w, alpha, beta, sms, partial);
    if (w <= 128) return spmm_launch<4>(st, a, x, ldx, y, ldy, w, alpha, beta, sms, partial);
    if (w <= 256) return spmm_launch<8>(st, a, x, ldx, y, ldy, w, alpha, beta, sms, partial);
    // Wide right-hand sides (randQB_FP sketches): column slabs of 256.
    for (int c0 = 0; c0 < w; c0 += 256) {
        const int wc = std::min(256, w - c0);
        spmm_launch<8>(st, a, x + c0, ldx, y + c0, ldy, wc, alpha, beta, sms, partial);
    }
}

int csr_validate(cudaStream_t st, std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                 const std::int32_t* ci, const double* v, int sms) {
    int* d_flags = nullptr;
    QB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_flags), sizeof(int), st));
    QB_CUDA(cudaMemsetAsync(d_flags, 0, sizeof(int), st));
    const int blocks = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(ceil_div(std::max(m, nnz), 256), 8L * sms)));
    validate_kernel<<<blocks, 256, 0, st>>>(m, n, nnz, rp, ci, v, d_flags);
    QB_LAUNCH_CHECK();
    int flags = 0;
    QB_CUDA(cudaMemcpyAsync(&flags, d_flags, sizeof(int), cudaMemcpyDeviceToHost, st));
    QB_CUDA(cudaFreeAsync(d_flags, st));
    QB_CUDA(cudaStreamSynchronize(st));
    return flags;
}

namespace {
// warp per row: kept entries of row i (rowmap[i] < 0 and colmap[col] < 0)
__global__ void split_count_kernel(std::int64_t m, const std::int64_t* __restrict__ rp, const std::int32_t* __restrict__ ci,
                                   const std::int32_t* __restrict__ rowmap, const std::int32_t* __restrict__ colmap,
                                   int* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const std::int64_t warp = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const std::int64_t nwarps = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (std::int64_t i = warp; i < m; i += nwarps) {
        int c = 0;
        if (rowmap[i] < 0)
            for (std::int64_t e = rp[i] + lane; e < rp[i + 1]; e += 32) c += colmap[ci[e]] < 0 ? 1 : 0;
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) cnt[i] = c;
    }
}

// warp per row: order-preserving compaction into S, dense entries into D_r / D_c
__global__ void split_fill_kernel(std::int64_t m, std::int64_t n, const std::int64_t* __restrict__ rp,
                                  const std::int32_t* __restrict__ ci, const double* __restrict__ v,
                                  const std::int32_t* __restrict__ rowmap, const std::int32_t* __restrict__ colmap,
                                  const std::int64_t* __restrict__ s_rp, std::int32_t* __restrict__ s_ci,
                                  double* __restrict__ s_v, double* __restrict__ d_r, double* __restrict__ d_c) {
    const int lane = threadIdx.x & 31;
    const std::int64_t warp = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const std::int64_t nwarps = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (std::int64_t i = warp; i < m; i += nwarps) {
        const int r = rowmap[i];
        std::int64_t out = s_rp[i];
        for (std::int64_t eb = rp[i]; eb < rp[i + 1]; eb += 32) {
            const std::int64_t e = eb + lane;
            const bool in = e < rp[i + 1];
            const std::int32_t c = in ? ci[e] : 0;
            const double x = in ? v[e] : 0.0;
            const int j = in ? colmap[c] : -1;
            if (r >= 0) {
                if (in) d_r[static_cast<std::int64_t>(r) * n + c] = x;
                continue;
            }
            if (in && j >= 0) d_c[i + static_cast<std::int64_t>(j) * m] = x;
            const bool keep = in && j < 0;
            const unsigned mask = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const std::int64_t pos = out + __popc(mask & ((1u << lane) - 1u));
                s_ci[pos] = c;
                s_v[pos] = x;
            }
            out += __popc(mask);
        }
    }
}

__global__ void gather_rows_kernel(const double* __restrict__ src, std::int64_t lds, const std::int64_t* __restrict__ idx,
                                   std::int64_t k, int w, double* __restrict__ dst) {
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < k * w;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int64_t r = e / w;
        dst[e] = src[idx[r] * lds + (e - r * w)];
    }
}

__global__ void scatter_add_rows_kernel(const double* __restrict__ src, const std::int64_t* __restrict__ idx, std::int64_t k,
                                        int w, double alpha, double* __restrict__ dst, std::int64_t ldd) {
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < k * w;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int64_t r = e / w;
        double* d = dst + idx[r] * ldd + (e - r * w);
        *d = fma(alpha, src[e], *d);
    }
}
}  // namespace

std::int64_t csr_split_dense(cudaStream_t st, std::int64_t m, std::int64_t n, const std::int64_t* rp,
                             const std::int32_t* ci, const double* v, const std::int32_t* rowmap,
                             const std::int32_t* colmap, std::int64_t* s_rp, std::int32_t** s_ci, double** s_v,
                             double* d_r, double* d_c, int sms) {
    int* cnt = nullptr;
    QB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cnt), sizeof(int) * std::max<std::int64_t>(m, 1), st));
    const int blocks = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(ceil_div(m * 32, 256), 16L * sms)));
    split_count_kernel<<<blocks, 256, 0, st>>>(m, rp, ci, rowmap, colmap, cnt);
    QB_LAUNCH_CHECK();
    scan_kernel<<<1, 1024, 0, st>>>(m, cnt, s_rp);
    QB_LAUNCH_CHECK();
    QB_CUDA(cudaFreeAsync(cnt, st));
    std::int64_t snnz = 0;
    QB_CUDA(cudaMemcpyAsync(&snnz, s_rp + m, sizeof(std::int64_t), cudaMemcpyDeviceToHost, st));
    QB_CUDA(cudaStreamSynchronize(st));
    QB_CUDA(cudaMalloc(s_ci, sizeof(std::int32_t) * std::max<std::int64_t>(snnz, 1)));
    QB_CUDA(cudaMalloc(s_v, sizeof(double) * std::max<std::int64_t>(snnz, 1)));
    split_fill_kernel<<<blocks, 256, 0, st>>>(m, n, rp, ci, v, rowmap, colmap, s_rp, *s_ci, *s_v, d_r, d_c);
    QB_LAUNCH_CHECK();
    return snnz;
}

void gather_rows(cudaStream_t st, const double* src, std::int64_t lds, const std::int64_t* idx, std::int64_t k, int w,
                 double* dst) {
    if (k * w == 0) return;
    gather_rows_kernel<<<static_cast<int>(std::min<std::int64_t>(ceil_div(k * w, 256), 4096)), 256, 0, st>>>(
        src, lds, idx, k, w, dst);
    QB_LAUNCH_CHECK();
}

void scatter_add_rows(cudaStream_t st, const double* src, const std::int64_t* idx, std::int64_t k, int w, double alpha,
                      double* dst, std::int64_t ldd) {
    if (k * w == 0) return;
    scatter_add_rows_kernel<<<static_cast<int>(std::min<std::int64_t>(ceil_div(k * w, 256), 4096)), 256, 0, st>>>(
        src, idx, k, w, alpha, dst, ldd);
    QB_LAUNCH_CHECK();
}

void csr_transpose(cudaStream_t st, std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                   const std::int32_t* ci, const double* v, std::int64_t* ct_rp, std::int32_t* ct_ci,
                   double* ct_v, int sms) {
    if (n == 0) return;
    int* cnt = nullptr;
    QB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cnt), sizeof(int) * n, st));
    QB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * n, st));
    if (nnz > 0) {
        const int blocks = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(ceil_div(nnz, 256), 8L * sms)));
        count_cols_kernel<<<blocks, 256, 0, st>>>(nnz, ci, cnt);
        QB_LAUNCH_CHECK();
    }
    scan_kernel<<<1, 1024, 0, st>>>(n, cnt, ct_rp);
    QB_LAUNCH_CHECK();
    QB_CUDA(cudaFreeAsync(cnt, st));
    if (nnz == 0 || m == 0) return;
    // Chunked stable placement.
    const int nchunks = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(2L * sms, m)));
    const std::int64_t rows_per = ceil_div(m, nchunks);
    int* cc = nullptr;
    std::int64_t* off = nullptr;
    QB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cc), sizeof(int) * n * nchunks, st));
    QB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&off), sizeof(std::int64_t) * n * nchunks, st));
    QB_CUDA(cudaMemsetAsync(cc, 0, sizeof(int) * n * nchunks, st));
    chunk_count_kernel<<<nchunks, 256, 0, st>>>(m, rows_per, rp, ci, n, cc);
    QB_LAUNCH_CHECK();
    chunk_offsets_kernel<<<static_cast<int>(std::min<std::int64_t>(ceil_div(n, 256), 8L * sms)), 256, 0, st>>>(
        n, nchunks, ct_rp, cc, off);
    QB_LAUNCH_CHECK();
    place_kernel<<<nchunks, 256, 0, st>>>(m, rows_per, rp, ci, v, n, off, ct_ci, ct_v);
    QB_LAUNCH_CHECK();
    QB_CUDA(cudaFreeAsync(cc, st));
    QB_CUDA(cudaFreeAsync(off, st));
}

}  // namespace qbgpu
