// FP64 tensor-core (DMMA) GEMM for sm_100a.
//
// Replaces the reference's blocked CPU drivers gemm_nn / gemm_tn
// (/root/reference/proj/src/kernels_drivers.cpp:21-65) and every dense product
// the algorithm layer issues through them (dense_matrix.cpp:68-92,
// matrix_handle.cpp:12-19): the passes over A (G = A*Omega, H = A^T*G, power
// products) and the per-block tall-skinny products (Q*M, Q^T*Y, B^T*Omega, ...).
//
// tcgen05.mma has no FP64 kind on sm_100a, so the FP64 tensor path is the
// warp-level mma.sync.m16n8k4.f64 (SASS DMMA.8x8x4). Tiles are staged
// global -> shared with multi-stage cp.async (LDGSTS) pipelines; every shared
// tile uses a leading dimension == 4 (mod 16) doubles, which makes all four
// operand layouts' fragment loads bank-conflict free. Split-K partials are
// reduced in a fixed order, so results are bitwise reproducible run to run.

#include "gemm.cuh"

#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>

#ifndef QB_WIDE_BK
#define QB_WIDE_BK 32
#define QB_WIDE_STAGES 3
#endif

namespace qbgpu {

namespace {

// Output tiles of an M x N product; with kGemmUpperC only those reaching the diagonal
// or above (tile row mt starts at tile column mt*bm/bn).
std::int64_t output_tiles(std::int64_t M, std::int64_t N, int bm, int bn, int flags) {
    const std::int64_t tm = ceil_div(M, bm), tn = ceil_div(N, bn);
    if (!(flags & kGemmUpperC)) return tm * tn;
    std::int64_t t = 0;
    for (std::int64_t mt = 0; mt < tm; ++mt) t += std::max<std::int64_t>(0, tn - (mt * bm) / bn);
    return t;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <int VEC>
__device__ __forceinline__ void cp_async(double* dst, const double* src, int valid) {
    // valid = number of doubles to fetch (0..VEC); the rest is zero-filled.
    const unsigned d = smem_u32(dst);
    if constexpr (VEC == 2) {
        const int bytes = valid * 8;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
    } else {
        const int bytes = valid * 8;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
    }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};\n"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a0), "d"(a1), "d"(b0));
}

constexpr int pad_to4(int base) { return ((4 - base % 16) + 16) % 16; }

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AR, bool BR>
struct Tile {
    static constexpr int NT = WM * WN * 32;
    static constexpr int WTM = BM / WM, WTN = BN / WN;
    static constexpr int MI = WTM / 16, NI = WTN / 8;
    // A shared tile: AR ? [BM][LDA] (m-major) : [BK][LDA] (k-major)
    static constexpr int A_INNER = AR ? BK : BM;
    static constexpr int A_OUTER = AR ? BM : BK;
    static constexpr int LDA = A_INNER + pad_to4(A_INNER);
    // B shared tile: BR ? [BK][LDB] (k-major) : [BN][LDB] (n-major)
    static constexpr int B_INNER = BR ? BN : BK;
    static constexpr int B_OUTER = BR ? BK : BN;
    static constexpr int LDB = B_INNER + pad_to4(B_INNER);
    static constexpr int A_STAGE = A_OUTER * LDA;
    static constexpr int B_STAGE = B_OUTER * LDB;
    static constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 8;
    static_assert(WTM % 16 == 0 && WTN % 8 == 0 && BK % 4 == 0, "tile shape");
    static_assert(LDA % 16 == 4 && LDB % 16 == 4, "conflict-free leading dims");
};

// Loads one (A_OUTER x A_INNER) or (B_OUTER x B_INNER) tile: `outer` segments of
// `inner` contiguous doubles. Segment s starts at base + s*seg_stride (global);
// element e of a segment is valid while (inner0 + e) < inner_lim and the
// segment index (outer0 + s) < outer_lim.
template <int OUTER, int INNER, int LDS, int NT, int VEC>
__device__ __forceinline__ void load_tile(double* smem, const double* __restrict__ base,
                                          std::int64_t seg_stride, std::int64_t inner0,
                                          std::int64_t inner_lim, std::int64_t outer0,
                                          std::int64_t outer_lim) {
    constexpr int CH_PER_SEG = INNER / VEC;
    constexpr int CHUNKS = OUTER * CH_PER_SEG;
#pragma unroll
    for (int it = 0; it < (CHUNKS + NT - 1) / NT; ++it) {
        const int idx = threadIdx.x + it * NT;
        if ((CHUNKS % NT) != 0 && idx >= CHUNKS) break;
        const int s = idx / CH_PER_SEG;
        const int e = (idx % CH_PER_SEG) * VEC;
        const std::int64_t gi = inner0 + e;
        const std::int64_t go = outer0 + s;
        int valid = 0;
        if (go < outer_lim) {
            const std::int64_t rem = inner_lim - gi;
            valid = rem >= VEC ? VEC : (rem > 0 ? static_cast<int>(rem) : 0);
        }
        const double* src = valid ? base + static_cast<std::int64_t>(s) * seg_stride + e : base;
        cp_async<VEC>(smem + s * LDS + e, src, valid);
    }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AR, bool BR, int VEC>
__global__ void __launch_bounds__(WM * WN * 32)
dgemm_kernel(const double* __restrict__ A, std::int64_t lda, const double* __restrict__ B,
             std::int64_t ldb, double* __restrict__ C, std::int64_t ldc, int c_row, int M, int N,
             int K, int k_split_len, double alpha, double beta, double* __restrict__ partial, int flags) {
    using T = Tile<BM, BN, BK, WM, WN, STAGES, AR, BR>;
    extern __shared__ __align__(16) double smem[];
    double* sA = smem;
    double* sB = smem + STAGES * T::A_STAGE;

    const int m0 = blockIdx.x * BM;
    const int n0 = blockIdx.y * BN;
    const int kz = blockIdx.z;
    if ((flags & kGemmUpperC) && m0 >= n0 + BN) return;  // tile strictly below the diagonal
    const int k_begin = kz * k_split_len;
    int k_end = min(K, k_begin + k_split_len);
    if (flags & kGemmTriB) k_end = min(k_end, n0 + BN);   // B upper triangular: rows >= n0+BN are 0
    const int ntiles = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp % WM, wn = warp / WM;
    const int g = lane >> 2, t = lane & 3;

    double acc[T::MI][T::NI][4];
#pragma unroll
    for (int i = 0; i < T::MI; ++i)
#pragma unroll
        for (int j = 0; j < T::NI; ++j)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

    auto issue = [&](int stage, int kt) {
        const int k0 = k_begin + kt * BK;
        double* a_dst = sA + stage * T::A_STAGE;
        double* b_dst = sB + stage * T::B_STAGE;
        if constexpr (AR) {  // A(i,k) = A[i*lda + k]: BM segments (rows) of BK
            load_tile<BM, BK, T::LDA, T::NT, VEC>(a_dst, A + static_cast<std::int64_t>(m0) * lda + k0,
                                                  lda, k0, k_end, m0, M);
        } else {             // A(i,k) = A[i + k*lda]: BK segments (columns) of BM
            load_tile<BK, BM, T::LDA, T::NT, VEC>(a_dst, A + m0 + static_cast<std::int64_t>(k0) * lda,
                                                  lda, m0, M, k0, k_end);
        }
        if constexpr (BR) {  // B(k,j) = B[k*ldb + j]: BK segments of BN
            load_tile<BK, BN, T::LDB, T::NT, VEC>(b_dst, B + static_cast<std::int64_t>(k0) * ldb + n0,
                                                  ldb, n0, N, k0, k_end);
        } else {             // B(k,j) = B[k + j*ldb]: BN segments of BK
            load_tile<BN, BK, T::LDB, T::NT, VEC>(b_dst, B + k0 + static_cast<std::int64_t>(n0) * ldb,
                                                  ldb, k0, k_end, n0, N);
        }
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ntiles) issue(s, s);
        cp_async_commit();
    }

    for (int kt = 0; kt < ntiles; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nk = kt + STAGES - 1;
            if (nk < ntiles) issue(nk % STAGES, nk);
            cp_async_commit();
        }
        const double* a_s = sA + (kt % STAGES) * T::A_STAGE;
        const double* b_s = sB + (kt % STAGES) * T::B_STAGE;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[T::MI][2];
            double bf[T::NI];
#pragma unroll
            for (int i = 0; i < T::MI; ++i) {
                const int r = wm * T::WTM + i * 16 + g;
                if constexpr (AR) {
                    af[i][0] = a_s[r * T::LDA + kk + t];
                    af[i][1] = a_s[(r + 8) * T::LDA + kk + t];
                } else {
                    af[i][0] = a_s[(kk + t) * T::LDA + r];
                    af[i][1] = a_s[(kk + t) * T::LDA + r + 8];
                }
            }
#pragma unroll
            for (int j = 0; j < T::NI; ++j) {
                const int c = wn * T::WTN + j * 8 + g;
                if constexpr (BR) bf[j] = b_s[(kk + t) * T::LDB + c];
                else bf[j] = b_s[c * T::LDB + kk + t];
            }
#pragma unroll
            for (int i = 0; i < T::MI; ++i)
#pragma unroll
                for (int j = 0; j < T::NI; ++j) dmma_16x8x4(acc[i][j], af[i][0], af[i][1], bf[j]);
        }
    }
    cp_async_wait<0>();

    // Epilogue: C fragment rows g / g+8, cols 2t / 2t+1.
#pragma unroll
    for (int i = 0; i < T::MI; ++i) {
#pragma unroll
        for (int j = 0; j < T::NI; ++j) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int row = m0 + wm * T::WTM + i * 16 + g + (r >= 2 ? 8 : 0);
                const int col = n0 + wn * T::WTN + j * 8 + 2 * t + (r & 1);
                if (row < M && col < N) {
                    if (partial) {
                        partial[static_cast<std::int64_t>(kz) * M * N + row +
                                static_cast<std::int64_t>(col) * M] = acc[i][j][r];
                    } else {
                        double* cp = c_row ? C + static_cast<std::int64_t>(row) * ldc + col
                                           : C + row + static_cast<std::int64_t>(col) * ldc;
                        const double v = alpha * acc[i][j][r];
                        *cp = beta == 0.0 ? v : v + beta * (*cp);
                    }
                }
            }
        }
    }
}

// Deterministic split-K reduction: a CTA owns 32 consecutive outputs (lanes); warp g
// sums splits g, g+8, ... in order, then warp 0 adds the 8 group sums in order.

__global__ void __launch_bounds__(256)
splitk_reduce_kernel(const double* __restrict__ partial, int splits, int M, int N, double alpha, double beta,
                     double* __restrict__ C, std::int64_t ldc, int c_row, int flags, int bm, int bn) {
    pdl_wait();
    __shared__ double sh[8][33];
    const std::int64_t total = static_cast<std::int64_t>(M) * N;
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    const std::int64_t idx = static_cast<std::int64_t>(blockIdx.x) * 32 + lane;
    double s = 0.0;
    if (idx < total)
        for (int z = g; z < splits; z += 8) s += partial[z * total + idx];
    sh[g][lane] = s;
    __syncthreads();
    if (g == 0 && idx < total) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) t += sh[q][lane];
        const std::int64_t row = idx % M, col = idx / M;
        if ((flags & kGemmUpperC) && (row / bm) * bm >= (col / bn) * bn + bn) return;
        double* cp = c_row ? C + row * ldc + col : C + row + col * ldc;
        const double v = alpha * t;
        *cp = beta == 0.0 ? v : v + beta * (*cp);
    }
}

#include "gemm_ws.cuh"

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        QB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        if (!f || q != cudaDriverEntryPointSuccess) throw QbError(kError, "cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<EncodeTiledFn>(f);
    }();
    return fn;
}

// 2-D FP64 tensor map over a strided matrix: dim0 (contiguous) of extent inner, dim1 of
// extent outer with a row pitch of ld doubles; box {box0, box1}; zero fill out of range.
void make_tmap(CUtensorMap* map, const double* base, std::int64_t inner, std::int64_t outer, std::int64_t ld,
               int box0, int box1) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(std::max<std::int64_t>(inner, 1)),
                                static_cast<cuuint64_t>(std::max<std::int64_t>(outer, 1))};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box0), static_cast<cuuint32_t>(box1)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_tiled()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides,
                                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw QbError(kError, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
}

// Resident CTAs per SM of one warp-specialised instance (opts its shared memory in once per device).
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AR, bool BR, int NP>
int ws_per_sm() {
    using T = Tile<BM, BN, BK, WM, WN, STAGES, AR, BR>;
    auto kern = dgemm_ws_kernel<BM, BN, BK, WM, WN, STAGES, AR, BR, NP>;
    constexpr int smem = T::SMEM_BYTES + 2 * STAGES * 8;
    static PerDevice<int> setup;
    return setup.get([&] {
        int v = 0;
        QB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        QB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, (WM * WN + NP) * 32, smem));
        return v < 1 ? 1 : v;
    });
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AR, bool BR, int NP>
void launch_ws(cudaStream_t st, const MatView& a, const MatView& b, double* c, std::int64_t ldc, bool c_row, int M,
               int N, int K, int splits, int klen, double alpha, double beta, double* partial, int flags,
               Workspace* tws) {
    using T = Tile<BM, BN, BK, WM, WN, STAGES, AR, BR>;
    auto kern = dgemm_ws_kernel<BM, BN, BK, WM, WN, STAGES, AR, BR, NP>;
    constexpr int smem = T::SMEM_BYTES + 2 * STAGES * 8;
    const int per_sm = ws_per_sm<BM, BN, BK, WM, WN, STAGES, AR, BR, NP>();
    WsArgs p{};
    p.A = a.p; p.lda = a.ld; p.B = b.p; p.ldb = b.ld; p.C = c; p.ldc = ldc; p.c_row = c_row ? 1 : 0;
    p.M = M; p.N = N; p.K = K; p.k_split_len = klen; p.splits = splits;
    p.tiles_m = static_cast<int>(ceil_div(M, BM)); p.tiles_n = static_cast<int>(ceil_div(N, BN));
    p.flags = flags; p.alpha = alpha; p.beta = beta; p.partial = partial;
    p.tiles = static_cast<int>(output_tiles(M, N, BM, BN, flags));
    if (AR) make_tmap(&p.tmA, a.p, K, M, a.ld, T::LDA, BM);               // A(i,k) at A + i*lda + k
    if (BR && BN < 64) make_tmap(&p.tmB, b.p, N, K, b.ld, T::LDB, BK);    // B(k,j) at B + k*ldb + j
    if (!BR) make_tmap(&p.tmB, b.p, K, N, b.ld, T::LDB, BN);              // B(k,j) at B + k + j*ldb
    std::int64_t items = static_cast<std::int64_t>(p.tiles) * splits;
    const int gmax = per_sm * gemm_num_sms();
    // Last-wave balancing: when the whole tiles leave a partial last wave (e.g. 1575 tiles on
    // 148 CTAs: 10 waves + 95 tiles), the tail tiles are cut along K into s pieces so the tail
    // takes ceil(tail*s/G)/s of a wave instead of one; pieces write partial tiles and the
    // last-arriving piece sums them in piece order (deterministic) and runs the epilogue.
    p.full_items = p.tiles;
    p.tail_s = 0;
    if (splits == 1 && !partial && tws && !(flags & (kGemmUpperC | kGemmTriB)) && p.tiles > gmax) {
        const int tail = p.tiles % gmax;
        double best = 1.0;
        int best_s = 1;
        for (int s = 2; s <= 16 && K / s >= 8 * BK; ++s) {
            const double cost = static_cast<double>((tail * s + gmax - 1) / gmax) * (1.0 / s + 0.02);
            if (cost < best - 0.05) { best = cost; best_s = s; }
        }
        if (tail > 0 && best_s > 1) {
            p.full_items = p.tiles - tail;
            p.tail_s = best_s;
            p.tail_klen = static_cast<int>(round_up(ceil_div(K, best_s), BK));
            const std::size_t part = static_cast<std::size_t>(tail) * best_s * BM * BN;
            double* w = tws->get(part + (tail + 7) / 8 + 8);
            p.tail_part = w;
            p.tail_cnt = reinterpret_cast<unsigned*>(w + part);
            QB_CUDA(cudaMemsetAsync(p.tail_cnt, 0, sizeof(unsigned) * tail, st));
            items = p.full_items + static_cast<std::int64_t>(tail) * best_s;
        }
    }
    const int grid = static_cast<int>(std::min<std::int64_t>(items, gmax));
    launch_pdl(kern, dim3(grid), dim3((WM * WN + NP) * 32), smem, st, p);
    QB_LAUNCH_CHECK();
}

// ws_per_sm for the instance dispatch_ws would launch
template <bool AR, bool BR>
int ws_occupancy(int fam) {
    constexpr int NP = (!AR && BR) ? 1 : 2;
    if (fam == 0) return ws_per_sm<128, 128, 32, 2, 4, 3, AR, BR, NP>();
    if (fam == 1) return ws_per_sm<128, 64, 32, 4, 2, 4, AR, BR, NP>();
    if (fam == 3) return ws_per_sm<128, 56, 32, 8, 1, 4, AR, BR, 2>();
    if (fam == 4) return ws_per_sm<128, 80, 32, 4, 2, 3, AR, BR, NP>();
    if (fam == 5) return ws_per_sm<128, 112, 32, 4, 2, 3, AR, BR, NP>();
    if (fam == 6) return ws_per_sm<128, 104, 32, 8, 1, 3, AR, BR, NP>();
    return ws_per_sm<64, 32, 32, 2, 2, 4, AR, BR, 2>();
}

template <bool AR, bool BR>
bool dispatch_ws(int fam, cudaStream_t st, const MatView& a, const MatView& b, double* c, std::int64_t ldc, bool c_row,
                 int M, int N, int K, int splits, int klen, double alpha, double beta, double* partial, int flags,
                 Workspace* tws) {
    // one producer warp when both operands move by bulk TMA, two when cp.async chunks are involved
    constexpr int NP = (!AR && BR) ? 1 : 2;
    if (fam == 0) launch_ws<128, 128, 32, 2, 4, 3, AR, BR, NP>(st, a, b, c, ldc, c_row, M, N, K, splits, klen, alpha, beta, partial, flags, tws);
    else if (fam == 1) launch_ws<128, 64, 32, 4, 2, 4, AR, BR, NP>(st, a, b, c, ldc, c_row, M, N, K, splits, klen, alpha, beta, partial, flags, tws);
    else if (fam == 3) launch_ws<128, 56, 32, 8, 1, 4, AR, BR, 2>(st, a, b, c, ldc, c_row, M, N, K, splits, klen, alpha, beta, partial, flags, tws);
    else if (fam == 4) launch_ws<128, 80, 32, 4, 2, 3, AR, BR, NP>(st, a, b, c, ldc, c_row, M, N, K, splits, klen, alpha, beta, partial, flags, tws);
    else if (fam == 5) launch_ws<128, 112, 32, 4, 2, 3, AR, BR, NP>(st, a, b, c, ldc, c_row, M, N, K, splits, klen, alpha, beta, partial, flags, tws);
    else if (fam == 6) launch_ws<128, 104, 32, 8, 1, 3, AR, BR, NP>(st, a, b, c, ldc, c_row, M, N, K, splits, klen, alpha, beta, partial, flags, tws);
    else launch_ws<64, 32, 32, 2, 2, 4, AR, BR, 2>(st, a, b, c, ldc, c_row, M, N, K, splits, klen, alpha, beta, partial, flags, tws);
    return true;
}

struct Launch {
    int bm, bn, bk;
    int threads;
    int smem;
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AR, bool BR, int VEC>
void launch_cfg(cudaStream_t st, const MatView& a, const MatView& b, double* c, std::int64_t ldc,
                bool c_row, int M, int N, int K, int splits, int klen, double alpha, double beta,
                double* partial, int flags) {
    using T = Tile<BM, BN, BK, WM, WN, STAGES, AR, BR>;
    auto kern = dgemm_kernel<BM, BN, BK, WM, WN, STAGES, AR, BR, VEC>;
    static PerDevice<bool> setup;  // per template instance and device
    setup.get([&] {
        QB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM_BYTES));
        return true;
    });
    dim3 grid(static_cast<unsigned>(ceil_div(M, BM)), static_cast<unsigned>(ceil_div(N, BN)),
              static_cast<unsigned>(splits));
    kern<<<grid, T::NT, T::SMEM_BYTES, st>>>(a.p, a.ld, b.p, b.ld, c, ldc, c_row ? 1 : 0, M, N, K,
                                            klen, alpha, beta, partial, flags);
    QB_LAUNCH_CHECK();
}

// Tile families. "wide": 128x128 CTA tiles (warp 64x32) for the passes over A at
// large widths; "skinny": 128x64 (warp 32x32) for widths ~50-100; "narrow":
// 64x32 for the thinnest products (b = 20, Gram-like outputs).
enum class Family { kWide, kSkinny, kNarrow, kSkinny56, kWide80 };

template <Family F, bool AR, bool BR, int VEC>
void launch_family(cudaStream_t st, const MatView& a, const MatView& b, double* c, std::int64_t ldc,
                   bool c_row, int M, int N, int K, int splits, int klen, double alpha, double beta,
                   double* partial, int flags) {
#ifndef QB_WIDE_BK
#define QB_WIDE_BK 16
#define QB_WIDE_STAGES 4
#endif
    if constexpr (F == Family::kWide)
        launch_cfg<128, 128, QB_WIDE_BK, 2, 4, QB_WIDE_STAGES, AR, BR, VEC>(st, a, b, c, ldc, c_row, M, N, K, splits, klen,
                                                       alpha, beta, partial, flags);
    else if constexpr (F == Family::kSkinny)
        launch_cfg<128, 64, 16, 4, 2, 4, AR, BR, VEC>(st, a, b, c, ldc, c_row, M, N, K, splits, klen,
                                                      alpha, beta, partial, flags);
    else if constexpr (F == Family::kWide80)  // widths that are multiples of 80 (l = 400): no 128-column padding
        launch_cfg<128, 80, 32, 4, 2, 3, AR, BR, VEC>(st, a, b, c, ldc, c_row, M, N, K, splits, klen,
                                                      alpha, beta, partial, flags);
    else if constexpr (F == Family::kSkinny56)  // b = 50-56: 7 n8 tiles per warp, no 64-column padding
        launch_cfg<128, 56, 32, 8, 1, 4, AR, BR, VEC>(st, a, b, c, ldc, c_row, M, N, K, splits, klen,
                                                      alpha, beta, partial, flags);
    else
        launch_cfg<64, 32, 32, 2, 2, 4, AR, BR, VEC>(st, a, b, c, ldc, c_row, M, N, K, splits, klen,
                                                     alpha, beta, partial, flags);
}

template <Family F>
void dispatch_layout(cudaStream_t st, const MatView& a, const MatView& b, double* c,
                     std::int64_t ldc, bool c_row, int M, int N, int K, int splits, int klen,
                     double alpha, double beta, double* partial, bool vec2, int flags) {
#define QB_DISPATCH(AR_, BR_)                                                                    \
    if (vec2) launch_family<F, AR_, BR_, 2>(st, a, b, c, ldc, c_row, M, N, K, splits, klen, alpha, \
                                            beta, partial, flags);                               \
    else launch_family<F, AR_, BR_, 1>(st, a, b, c, ldc, c_row, M, N, K, splits, klen, alpha, beta, \
                                       partial, flags);
    if (a.rowmajor) {
        if (b.rowmajor) { QB_DISPATCH(true, true) } else { QB_DISPATCH(true, false) }
    } else {
        if (b.rowmajor) { QB_DISPATCH(false, true) } else { QB_DISPATCH(false, false) }
    }
#undef QB_DISPATCH
}

bool aligned16(const MatView& v) {
    return (reinterpret_cast<std::uintptr_t>(v.p) % 16 == 0) && (v.ld % 2 == 0);
}

}  // namespace

void make_tensor_map_2d(void* map, const double* base, std::int64_t inner, std::int64_t outer, std::int64_t ld,
                        int box0, int box1) {
    make_tmap(reinterpret_cast<CUtensorMap*>(map), base, inner, outer, ld, box0, box1);
}

void make_tensor_map_rows(void* map, const double* base, std::int64_t rows, int w, std::int64_t ld) {
    // one row of w doubles per box (tile::gather4 requires box height 1)
    make_tmap(reinterpret_cast<CUtensorMap*>(map), base, w, rows, ld, w, 1);
}

int gemm_num_sms() {
    static PerDevice<int> sms;
    return sms.get([] {
        int dev = 0, n = 148;
        QB_CUDA(cudaGetDevice(&dev));
        QB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
        return n;
    });
}

void gemm(cudaStream_t st, Workspace& ws, double alpha, const MatView& a, const MatView& b,
          double beta, const MatView& c, int flags) {
    const std::int64_t M = a.rows, K = a.cols, N = b.cols;
    if (b.rows != K || c.rows != M || c.cols != N)
        throw QbError(kDimensionError, "gemm: inner dimension mismatch");
    if (M == 0 || N == 0) return;
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
        throw QbError(kDimensionError, "gemm: dimension exceeds 2^31");
    if (K == 0) {
        // C = beta*C
        scale_matrix(st, c, beta);
        return;
    }
    Family fam;
    int bm, bn, bk;
    // wide widths: 128-column tiles unless 80-column tiles pad less (e.g. l = 400: 4 x 128 = 512
    // vs 5 x 80 = 400; l = 2000: 2048 vs 2000)
    // (A column-major only: the A^T passes measured faster on 128-wide tiles)
    // (N = 2000: 25 x 80 columns, no padding, measured 0.8-5 % faster than 16 x 128 on the
    // cfg2 passes, Gram and X R^-1)
    // (not for upper-triangular outputs: the 128 x 80 tiles straddling the diagonal waste more)
    const bool use80 = N >= 96 && round_up(N, 80) < round_up(N, 128) && !(flags & kGemmUpperC);
    if (use80) { fam = Family::kWide80; bm = 128; bn = 80; bk = 32; }
    else if (N >= 96) { fam = Family::kWide; bm = 128; bn = 128; bk = QB_WIDE_BK; }
    else if (N > 48 && N <= 56) { fam = Family::kSkinny56; bm = 128; bn = 56; bk = 32; }
    else if (N > 32) { fam = Family::kSkinny; bm = 128; bn = 64; bk = 16; }
    else { fam = Family::kNarrow; bm = 64; bn = 32; bk = 32; }
    const bool vec2 = aligned16(a) && aligned16(b);
    static const bool use_ws = [] {
        const char* e = std::getenv("QBFAC_GEMM_LEGACY");
        return !(e && e[0] == '1');
    }();
    // Warp-specialised TMA path where it measured faster (tools/gemm_bench.py): A column-major
    // (long bulk segments), or both operands row-major with wide tiles (A^T G passes).
    const bool tiny = false;  // (a no-split plain path for tiny products measured slower: split-K keeps SMs busy)
    const bool ws_path = use_ws && vec2 && !tiny;
    if (ws_path) bk = 32;  // the warp-specialised kernels use BK = 32 in every family
    // b = 100: 112-column tiles (14 n8 fragments, 12 % padding) instead of 128 (28 %)
    if (ws_path && fam == Family::kWide && N > 96 && N <= 112) bn = 112;
    // b = 97..104: 104-column tiles (13 n8 fragments, 8 x 1 warps of 16 x 104): 4 % padding at b = 100
    // instead of 12 % (QBFAC_GEMM_104=0 keeps the 112-column tile)
    static const bool use104 = [] {
        const char* e = std::getenv("QBFAC_GEMM_104");
        return !(e && e[0] == '0');
    }();
    if (ws_path && fam == Family::kWide && N > 96 && N <= 104 && use104 && !(flags & kGemmUpperC)) bn = 104;
    // A column-major (the k x b coefficient products Q^T Y, B Omega_i): the 56-column tile too
    // (config 3: Q^T Y 9.19 -> 8.08 ms and B Omega 5.10 -> 4.54 ms per factorization, tools/gemm_cfg3.py;
    // QBFAC_GEMM_TN56=0 restores the 64-column tile, which measured faster before the split-K count
    // followed the kernel's real occupancy)
    static const bool tn56 = [] {
        const char* e = std::getenv("QBFAC_GEMM_TN56");
        return !(e && e[0] == '0');
    }();
    if (ws_path && fam == Family::kSkinny56 && !a.rowmajor && !tn56) bn = 64;
    const std::int64_t tiles = output_tiles(M, N, bm, bn, flags);
    const int sms = gemm_num_sms();
    // the same famid dispatch_ws uses below
    const int famid = fam == Family::kWide ? (bn == 112 ? 5 : bn == 104 ? 6 : 0) : fam == Family::kWide80 ? 4
                      : fam == Family::kSkinny56 ? ((a.rowmajor || tn56) ? 3 : 1) : fam == Family::kSkinny ? 1 : 2;
    // Resident CTAs per SM: the warp-specialised instance's real occupancy (the 64 x 32 tiles:
    // 2 per SM, not 3 — splitting for 3 left a second partial wave); legacy kernels ~1, narrow ~3.
    int resident = fam == Family::kNarrow ? 3 : 1;
    static const bool occ_split = [] {
        const char* e = std::getenv("QBFAC_GEMM_OCC_SPLIT");
        return !(e && e[0] == '0');
    }();
    if (ws_path && occ_split)
        resident = a.rowmajor ? (b.rowmajor ? ws_occupancy<true, true>(famid) : ws_occupancy<true, false>(famid))
                              : (b.rowmajor ? ws_occupancy<false, true>(famid) : ws_occupancy<false, false>(famid));
    const std::int64_t want = static_cast<std::int64_t>(resident) * sms;
    int splits = 1;
    if (tiles < want && !tiny) {
        const std::int64_t max_by_k = std::max<std::int64_t>(1, K / (4 * bk));  // >= 4 k-tiles/split
        const std::int64_t cap = (M * N <= 65536) ? 512 : 64;  // small outputs (Grams): deep split-K
        // floor: tiles * splits must not exceed one wave of resident CTAs (a 2nd partial wave
        // doubles the time; measured on Q^T Y 1000x50x1e5)
        const std::int64_t fit = std::max<std::int64_t>(1, want / tiles);
        splits = static_cast<int>(std::min<std::int64_t>(std::min<std::int64_t>(fit, max_by_k), cap));
    }
    int klen = static_cast<int>(round_up(ceil_div(K, splits), bk));
    splits = static_cast<int>(ceil_div(K, klen));
    double* partial = nullptr;
    if (splits > 1) partial = ws.get(static_cast<std::size_t>(splits) * M * N);
    if (ws_path) {
        // warp-specialised TMA/mbarrier pipeline (gemm_ws.cuh)
        {
            if (a.rowmajor) {
                if (b.rowmajor) dispatch_ws<true, true>(famid, st, a, b, c.p, c.ld, c.rowmajor, (int)M, (int)N, (int)K, splits, klen, alpha, beta, partial, flags, &ws);
                else dispatch_ws<true, false>(famid, st, a, b, c.p, c.ld, c.rowmajor, (int)M, (int)N, (int)K, splits, klen, alpha, beta, partial, flags, &ws);
            } else {
                if (b.rowmajor) dispatch_ws<false, true>(famid, st, a, b, c.p, c.ld, c.rowmajor, (int)M, (int)N, (int)K, splits, klen, alpha, beta, partial, flags, &ws);
                else dispatch_ws<false, false>(famid, st, a, b, c.p, c.ld, c.rowmajor, (int)M, (int)N, (int)K, splits, klen, alpha, beta, partial, flags, &ws);
            }
        }
    } else {
    switch (fam) {
        case Family::kWide:
            dispatch_layout<Family::kWide>(st, a, b, c.p, c.ld, c.rowmajor, (int)M, (int)N, (int)K, splits,
                                           klen, alpha, beta, partial, vec2, flags);
            break;
        case Family::kSkinny:
            dispatch_layout<Family::kSkinny>(st, a, b, c.p, c.ld, c.rowmajor, (int)M, (int)N, (int)K,
                                             splits, klen, alpha, beta, partial, vec2, flags);
            break;
        case Family::kWide80:
            dispatch_layout<Family::kWide80>(st, a, b, c.p, c.ld, c.rowmajor, (int)M, (int)N, (int)K,
                                             splits, klen, alpha, beta, partial, vec2, flags);
            break;
        case Family::kSkinny56:
            dispatch_layout<Family::kSkinny56>(st, a, b, c.p, c.ld, c.rowmajor, (int)M, (int)N, (int)K,
                                               splits, klen, alpha, beta, partial, vec2, flags);
            break;
        default:
            dispatch_layout<Family::kNarrow>(st, a, b, c.p, c.ld, c.rowmajor, (int)M, (int)N, (int)K,
                                             splits, klen, alpha, beta, partial, vec2, flags);
    }
    }
    if (splits > 1) {
        const std::int64_t total = M * N;
        launch_pdl(splitk_reduce_kernel, dim3(static_cast<unsigned>(ceil_div(total, 32))), dim3(256), 0, st,
                   static_cast<const double*>(partial), static_cast<int>(splits), static_cast<int>(M), static_cast<int>(N),
                   alpha, beta, c.p, static_cast<std::int64_t>(c.ld), c.rowmajor ? 1 : 0, flags, bm, bn);
        QB_LAUNCH_CHECK();
    }
}

}  // namespace qbgpu
