// Warp-specialised persistent FP64 DMMA GEMM (included by gemm.cu, inside its
// anonymous namespace; uses Tile<>, dmma_16x8x4).
//
// One producer warp streams A/B tiles global -> shared with TMA bulk copies
// (cp.async.bulk ... mbarrier::complete_tx, SASS UBLKCP) into a STAGES-deep ring;
// each smem row gets its own copy so the padded, bank-conflict-free layout of
// Tile<> is kept. Consumer warps wait on the stage's full mbarrier, run the DMMA
// k-steps and release the stage through its empty mbarrier — there is no
// CTA-wide barrier in the main loop, so the FP64 tensor pipe never drains at
// k-tile boundaries. CTAs are persistent over (m, n, k-split) work items, ordered
// n-fastest so concurrently running CTAs share A panels in L2; the epilogue of one
// item overlaps the producer's prefetch of the next.
//
// Operands whose contiguous segments are long (A column-major: BM rows; B row-major:
// BN >= 64 columns) move by TMA bulk copies; those with short segments (BK along
// the reduction dimension) by 16-byte cp.async chunks whose completion arrives on
// the same full barrier (cp.async.mbarrier.arrive.noinc).
// Edges: rows/cols beyond M/N are never copied (their garbage only reaches
// discarded outputs); the K tail is zeroed (generic stores before the stage's
// arrive for bulk operands, cp.async zero-fill otherwise); bulk segments that are
// not 16-byte aligned / even-length fall back to per-element copies.
#pragma once

__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(std::uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned parity) {
    const unsigned a = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_arrive_noinc(std::uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Short segments (inner extent < 512 B, here always the reduction dimension): 16-byte
// cp.async chunks (LDGSTS) spread over the producer lanes, zero-filled past the K
// limit through the src-size operand; completion is tracked by the stage's full
// barrier via cp.async.mbarrier.arrive.noinc (one per lane per stage).
template <int OUTER, int INNER, int LDS, bool OUTER_IS_K>
__device__ __forceinline__ void produce_async(double* smem, const double* __restrict__ base, std::int64_t seg_stride,
                                              std::int64_t inner0, std::int64_t inner_lim, std::int64_t outer0,
                                              std::int64_t outer_lim, int lane, int nthr) {
    constexpr int CH = INNER / 2;
    for (int idx = lane; idx < OUTER * CH; idx += nthr) {
        const int s = idx / CH, e = (idx % CH) * 2;
        const bool outer_ok = outer0 + s < outer_lim;
        if (!outer_ok && !OUTER_IS_K) continue;  // beyond M/N: only feeds discarded outputs
        const std::int64_t rem = inner_lim - (inner0 + e);
        const int valid = !outer_ok ? 0 : (rem >= 2 ? 2 : (rem > 0 ? static_cast<int>(rem) : 0));
        const double* src = valid ? base + static_cast<std::int64_t>(s) * seg_stride + e : base;
        const unsigned d = smem_u32(smem + s * LDS + e);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(valid * 8) : "memory");
    }
}

// Producer side of one tile operand: OUTER segments of INNER contiguous doubles,
// segment s at base + s*seg_stride (global). Valid inner extent [inner0, inner_lim),
// valid outer extent [outer0, outer_lim). `inner_is_k`: the inner dimension is the
// reduction dimension (its tail must be zero); otherwise the OUTER one is.
// Returns the bulk bytes this lane issued (summed by the caller for expect_tx).
template <int OUTER, int INNER, int LDS>
__device__ __forceinline__ unsigned produce_operand(double* smem, const double* __restrict__ base,
                                                    std::int64_t seg_stride, std::int64_t inner0,
                                                    std::int64_t inner_lim, std::int64_t outer0,
                                                    std::int64_t outer_lim, bool inner_is_k, int lane,
                                                    bool issue_bulk, std::uint64_t* bar, int nthr) {
    unsigned bytes = 0;
    for (int s = lane; s < OUTER; s += nthr) {
        double* dst = smem + s * LDS;
        const std::int64_t go = outer0 + s;
        const bool outer_ok = go < outer_lim;
        std::int64_t valid = inner_lim - inner0;
        valid = valid < 0 ? 0 : (valid > INNER ? INNER : valid);
        if (!outer_ok) {
            if (!inner_is_k) {  // beyond K along the outer dimension: zero the whole segment
                if (!issue_bulk)
                    for (int e = 0; e < INNER; ++e) dst[e] = 0.0;
            }
            continue;  // beyond M/N: leave stale data (only feeds discarded outputs)
        }
        const double* src = base + static_cast<std::int64_t>(s) * seg_stride;
        const bool bulk_ok = valid > 0 && (valid % 2 == 0) && ((reinterpret_cast<std::uintptr_t>(src) & 15) == 0);
        if (!issue_bulk) {
            // generic pass (before the arrive): odd/misaligned segments and the K tail
            if (!bulk_ok)
                for (int e = 0; e < valid; ++e) dst[e] = src[e];
            if (inner_is_k)
                for (int e = static_cast<int>(valid); e < INNER; ++e) dst[e] = 0.0;
        } else if (bulk_ok) {
            bulk_g2s(dst, src, static_cast<unsigned>(valid * 8), bar);
            bytes += static_cast<unsigned>(valid * 8);
        }
    }
    return bytes;
}

template <int OUTER, int INNER>
__device__ __forceinline__ unsigned operand_bulk_bytes(const double* __restrict__ base, std::int64_t seg_stride,
                                                       std::int64_t inner0, std::int64_t inner_lim, std::int64_t outer0,
                                                       std::int64_t outer_lim, int lane, int nthr) {
    unsigned bytes = 0;
    for (int s = lane; s < OUTER; s += nthr) {
        if (outer0 + s >= outer_lim) continue;
        std::int64_t valid = inner_lim - inner0;
        valid = valid < 0 ? 0 : (valid > INNER ? INNER : valid);
        const double* src = base + static_cast<std::int64_t>(s) * seg_stride;
        if (valid > 0 && valid % 2 == 0 && ((reinterpret_cast<std::uintptr_t>(src) & 15) == 0))
            bytes += static_cast<unsigned>(valid * 8);
    }
    return bytes;
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, std::uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

struct WsArgs {
    CUtensorMap tmA;  // used when A's contiguous segments are short (A row-major)
    CUtensorMap tmB;  // used when B's contiguous segments are short (B column-major, or BN < 64)
    const double* A;
    std::int64_t lda;
    const double* B;
    std::int64_t ldb;
    double* C;
    std::int64_t ldc;
    int c_row, M, N, K, k_split_len, splits, tiles_m, tiles_n, flags;
    int tiles;  // output tiles per k-split (kGemmUpperC: only those on/above the diagonal)
    double alpha, beta;
    double* partial;
    // last-wave balancing (launch_ws): items >= full_items are K-pieces of the tail tiles
    int full_items, tail_s, tail_klen;
    double* tail_part;    // (tail tiles x tail_s) partial tiles, fragment order
    unsigned* tail_cnt;   // arrivals per tail tile (zeroed per launch)
};

// Work item -> tile and K range; tail_j >= 0 marks a K-piece of a tail tile.
template <int BM, int BN>
__device__ __forceinline__ void ws_item(const WsArgs& p, int it, int& mt, int& nt, int& kz, int& k_begin, int& k_end,
                                        int& tail_j);

// Work item -> (m tile, n tile, k split), n-fastest. For kGemmUpperC only the tiles
// reaching the diagonal or above are enumerated (row mt starts at n tile mt*BM/BN),
// so the static persistent schedule stays balanced on Gram/SYRK outputs.
template <int BM, int BN>
__device__ __forceinline__ void ws_decode_item(const WsArgs& p, int it, int& mt, int& nt, int& kz) {
    kz = it / p.tiles;
    int t = it - kz * p.tiles;
    if (p.flags & kGemmTriB) {
        // triangular B: tile column nt needs (nt + 1) * BN of K; longest tiles first (LPT),
        // m-fastest, so the static persistent schedule ends on the short ones
        mt = t % p.tiles_m;
        nt = p.tiles_n - 1 - t / p.tiles_m;
        return;
    }
    if (!(p.flags & kGemmUpperC)) {
        nt = t % p.tiles_n;
        mt = t / p.tiles_n;
        return;
    }
    for (mt = 0; mt < p.tiles_m - 1; ++mt) {
        const int cnt = max(0, p.tiles_n - (mt * BM) / BN);
        if (t < cnt) break;
        t -= cnt;
    }
    nt = (mt * BM) / BN + t;
}

template <int BM, int BN>
__device__ __forceinline__ void ws_item(const WsArgs& p, int it, int& mt, int& nt, int& kz, int& k_begin, int& k_end,
                                        int& tail_j) {
    tail_j = -1;
    if (p.tail_s && it >= p.full_items) {
        const int j = it - p.full_items;
        ws_decode_item<BM, BN>(p, p.full_items + j / p.tail_s, mt, nt, kz);
        k_begin = (j % p.tail_s) * p.tail_klen;
        k_end = min(p.K, k_begin + p.tail_klen);
        tail_j = j;
        return;
    }
    ws_decode_item<BM, BN>(p, it, mt, nt, kz);
    k_begin = kz * p.k_split_len;
    k_end = min(p.K, k_begin + p.k_split_len);
    if (p.flags & kGemmTriB) k_end = min(k_end, nt * BN + BN);
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AR, bool BR, int NP>
__global__ void __launch_bounds__((WM * WN + NP) * 32, 1) dgemm_ws_kernel(const __grid_constant__ WsArgs p) {
    using T = Tile<BM, BN, BK, WM, WN, STAGES, AR, BR>;
    constexpr int NC = WM * WN;  // consumer warps
    pdl_wait();  // launched with programmatic stream serialization: wait for the previous kernel's memory
    extern __shared__ __align__(128) double smem[];
    double* sA = smem;
    double* sB = smem + STAGES * T::A_STAGE;
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(sB + STAGES * T::B_STAGE);
    std::uint64_t* empty = full + STAGES;
    __shared__ unsigned s_bytes[NP];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);  // one arrive carrying expect_tx (bulk + tensor TMA bytes)
            mbar_init(&empty[s], NC);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int items = p.tail_s ? p.full_items + (p.tiles - p.full_items) * p.tail_s : p.tiles * p.splits;
    __shared__ int s_last;
    if (warp >= NC) {
        // ===== producer warps =====
        const int pt = threadIdx.x - NC * 32;  // producer thread index
        constexpr int PT = NP * 32;
        int stage = 0;
        unsigned phase = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
            int mt, nt, kz, k_begin, k_end, tail_j;
            ws_item<BM, BN>(p, it, mt, nt, kz, k_begin, k_end, tail_j);
            const int m0 = mt * BM, n0 = nt * BN;
            const int ntiles = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;
            for (int kt = 0; kt < ntiles; ++kt) {
                mbar_wait(&empty[stage], phase ^ 1);
                const int k0 = k_begin + kt * BK;
                double* a_dst = sA + stage * T::A_STAGE;
                double* b_dst = sB + stage * T::B_STAGE;
                const double* a_src = AR ? p.A + static_cast<std::int64_t>(m0) * p.lda + k0
                                         : p.A + m0 + static_cast<std::int64_t>(k0) * p.lda;
                const double* b_src = BR ? p.B + static_cast<std::int64_t>(k0) * p.ldb + n0
                                         : p.B + k0 + static_cast<std::int64_t>(n0) * p.ldb;
                // Long contiguous segments (A column-major: BM rows; B row-major: BN >= 64
                // columns) go by per-row TMA bulk copies into the padded layout; short ones
                // (BK along the reduction dimension, or BN < 64) by ONE 2-D tensor TMA per
                // operand whose box is the padded row length (the extra 4 doubles per row are
                // an over-read that keeps the layout bank-conflict free); out-of-range
                // elements are zero-filled by the TMA unit.
                constexpr bool A_BULK = !AR;
                constexpr bool B_BULK = BR && BN >= 64;
                // 1) generic pass for bulk operands: K-tail zero segments and unaligned/odd segments
                if constexpr (A_BULK)
                    produce_operand<BK, BM, T::LDA>(a_dst, a_src, p.lda, m0, p.M, k0, k_end, false, pt, false, nullptr, PT);
                if constexpr (B_BULK)
                    produce_operand<BK, BN, T::LDB>(b_dst, b_src, p.ldb, n0, p.N, k0, k_end, false, pt, false, nullptr, PT);
                // 2) expected bytes, then one arrive carrying expect_tx
                unsigned bytes = 0;
                if constexpr (A_BULK) bytes += operand_bulk_bytes<BK, BM>(a_src, p.lda, m0, p.M, k0, k_end, pt, PT);
                if constexpr (B_BULK) bytes += operand_bulk_bytes<BK, BN>(b_src, p.ldb, n0, p.N, k0, k_end, pt, PT);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
                if constexpr (NP > 1) {
                    // combine the producer warps' byte counts (named barrier over producers only)
                    if (lane == 0) s_bytes[warp - NC] = bytes;
                    asm volatile("bar.sync 1, %0;\n" ::"n"(NP * 32) : "memory");
                    bytes = 0;
#pragma unroll
                    for (int q = 0; q < NP; ++q) bytes += s_bytes[q];
                    asm volatile("bar.sync 1, %0;\n" ::"n"(NP * 32) : "memory");
                }
                if constexpr (!A_BULK) bytes += T::A_STAGE * 8;   // full box, zero-filled where out of range
                if constexpr (!B_BULK) bytes += T::B_STAGE * 8;
                fence_proxy_async();
                __syncwarp();
                if (pt == 0) mbar_arrive_tx(&full[stage], bytes);
                if constexpr (NP > 1) asm volatile("bar.sync 1, %0;\n" ::"n"(NP * 32) : "memory");
                __syncwarp();
                // 3) copies
                if constexpr (A_BULK)
                    produce_operand<BK, BM, T::LDA>(a_dst, a_src, p.lda, m0, p.M, k0, k_end, false, pt, true, &full[stage], PT);
                else if (pt == 0)
                    tma_2d(a_dst, &p.tmA, k0, m0, &full[stage]);          // box {LDA, BM} at (k0, m0)
                if constexpr (B_BULK)
                    produce_operand<BK, BN, T::LDB>(b_dst, b_src, p.ldb, n0, p.N, k0, k_end, false, pt, true, &full[stage], PT);
                else if (pt == 0) {
                    if constexpr (BR) tma_2d(b_dst, &p.tmB, n0, k0, &full[stage]);   // box {LDB, BK} at (n0, k0)
                    else tma_2d(b_dst, &p.tmB, k0, n0, &full[stage]);                // box {LDB, BN} at (k0, n0)
                }
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
        pdl_trigger();
        return;
    }
    // ===== consumers =====
    const int wm = warp % WM, wn = warp / WM;
    const int g = lane >> 2, t = lane & 3;
    int stage = 0;
    unsigned phase = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        int mt, nt, kz, k_begin, k_end, tail_j;
        ws_item<BM, BN>(p, it, mt, nt, kz, k_begin, k_end, tail_j);
        const int m0 = mt * BM, n0 = nt * BN;
        const int ntiles = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;
        double acc[T::MI][T::NI][4];
#pragma unroll
        for (int i = 0; i < T::MI; ++i)
#pragma unroll
            for (int j = 0; j < T::NI; ++j)
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;
        // beta != 0 (skinny updates Y -= Q M): the C fragment is loaded before the main loop
        // so its latency hides behind the MMAs instead of stalling the epilogue
        constexpr bool kPrefetchC = T::MI * T::NI * 4 <= 32;
        double cpre[kPrefetchC ? T::MI : 1][kPrefetchC ? T::NI : 1][4];
        const bool use_pre = kPrefetchC && p.beta != 0.0 && !p.partial;
        const bool vec_c = !p.partial && p.c_row && (p.ldc & 1) == 0 && (reinterpret_cast<std::uintptr_t>(p.C) & 15) == 0;
        if constexpr (kPrefetchC) {
            if (use_pre && vec_c) {  // 16-byte loads of the fragment's column pairs
#pragma unroll
                for (int i = 0; i < T::MI; ++i)
#pragma unroll
                    for (int j = 0; j < T::NI; ++j)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int row = m0 + wm * T::WTM + i * 16 + g + 8 * h;
                            const int col = n0 + wn * T::WTN + j * 8 + 2 * t;
                            double2 v = make_double2(0.0, 0.0);
                            if (row < p.M && col + 1 < p.N)
                                v = __ldcg(reinterpret_cast<const double2*>(p.C + static_cast<std::int64_t>(row) * p.ldc + col));
                            else if (row < p.M && col < p.N)
                                v.x = __ldcg(p.C + static_cast<std::int64_t>(row) * p.ldc + col);
                            cpre[i][j][2 * h] = v.x;
                            cpre[i][j][2 * h + 1] = v.y;
                        }
            } else if (use_pre) {
#pragma unroll
                for (int i = 0; i < T::MI; ++i)
#pragma unroll
                    for (int j = 0; j < T::NI; ++j)
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const int row = m0 + wm * T::WTM + i * 16 + g + (r >= 2 ? 8 : 0);
                            const int col = n0 + wn * T::WTN + j * 8 + 2 * t + (r & 1);
                            cpre[i][j][r] = (row < p.M && col < p.N)
                                                ? __ldcg(p.c_row ? p.C + static_cast<std::int64_t>(row) * p.ldc + col
                                                                 : p.C + row + static_cast<std::int64_t>(col) * p.ldc)
                                                : 0.0;
                        }
            }
        }
        for (int kt = 0; kt < ntiles; ++kt) {
            mbar_wait(&full[stage], phase);
            const double* a_s = sA + stage * T::A_STAGE;
            const double* b_s = sB + stage * T::B_STAGE;
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
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (tail_j >= 0) {
            // K-piece of a tail tile: publish the partial; the last piece to arrive sums all
            // pieces in piece order and falls through to the epilogue
            const int tt = tail_j / p.tail_s, piece = tail_j % p.tail_s;
            constexpr int FR = T::MI * T::NI * 4 * 32;  // doubles per warp
            double* mine = p.tail_part + (static_cast<std::size_t>(tt) * p.tail_s + piece) * (NC * FR) + warp * FR;
#pragma unroll
            for (int i = 0; i < T::MI; ++i)
#pragma unroll
                for (int j = 0; j < T::NI; ++j)
#pragma unroll
                    for (int r = 0; r < 4; ++r) __stcg(mine + ((i * T::NI + j) * 4 + r) * 32 + lane, acc[i][j][r]);
            __threadfence();
            asm volatile("bar.sync 2, %0;\n" ::"n"(NC * 32) : "memory");
            if (threadIdx.x == 0) s_last = atomicAdd(p.tail_cnt + tt, 1u) == static_cast<unsigned>(p.tail_s - 1);
            asm volatile("bar.sync 2, %0;\n" ::"n"(NC * 32) : "memory");
            if (!s_last) continue;
            __threadfence();
            const double* all = p.tail_part + static_cast<std::size_t>(tt) * p.tail_s * (NC * FR) + warp * FR;
#pragma unroll
            for (int i = 0; i < T::MI; ++i)
#pragma unroll
                for (int j = 0; j < T::NI; ++j)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        double v = 0.0;
                        for (int q = 0; q < p.tail_s; ++q)
                            v += __ldcg(all + static_cast<std::size_t>(q) * (NC * FR) + ((i * T::NI + j) * 4 + r) * 32 + lane);
                        acc[i][j][r] = v;
                    }
        }
        // epilogue (registers -> global); the producer is already prefetching the next item.
        // Row-major C with an even, 16-byte aligned row stride: the fragment's column pairs (2t, 2t + 1)
        // leave as one 16-byte store (a full half-sector per lane instead of two 8-byte pieces).
        if (vec_c) {
#pragma unroll
            for (int i = 0; i < T::MI; ++i) {
#pragma unroll
                for (int j = 0; j < T::NI; ++j) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int row = m0 + wm * T::WTM + i * 16 + g + 8 * h;
                        const int col = n0 + wn * T::WTN + j * 8 + 2 * t;
                        if (row >= p.M || col >= p.N) continue;
                        double* cp = p.C + static_cast<std::int64_t>(row) * p.ldc + col;
                        double v0 = p.alpha * acc[i][j][2 * h], v1 = p.alpha * acc[i][j][2 * h + 1];
                        if (p.beta != 0.0) {
                            double o0, o1;
                            if constexpr (kPrefetchC) {
                                o0 = use_pre ? cpre[i][j][2 * h] : cp[0];
                                o1 = use_pre ? cpre[i][j][2 * h + 1] : (col + 1 < p.N ? cp[1] : 0.0);
                            } else {
                                o0 = cp[0];
                                o1 = col + 1 < p.N ? cp[1] : 0.0;
                            }
                            v0 += p.beta * o0;
                            v1 += p.beta * o1;
                        }
                        if (col + 1 < p.N) *reinterpret_cast<double2*>(cp) = make_double2(v0, v1);
                        else cp[0] = v0;
                    }
                }
            }
            continue;
        }
#pragma unroll
        for (int i = 0; i < T::MI; ++i) {
#pragma unroll
            for (int j = 0; j < T::NI; ++j) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int row = m0 + wm * T::WTM + i * 16 + g + (r >= 2 ? 8 : 0);
                    const int col = n0 + wn * T::WTN + j * 8 + 2 * t + (r & 1);
                    if (row < p.M && col < p.N) {
                        if (p.partial) {
                            p.partial[static_cast<std::int64_t>(kz) * p.M * p.N + row +
                                      static_cast<std::int64_t>(col) * p.M] = acc[i][j][r];
                        } else {
                            double* cp = p.c_row ? p.C + static_cast<std::int64_t>(row) * p.ldc + col
                                                 : p.C + row + static_cast<std::int64_t>(col) * p.ldc;
                            const double v = p.alpha * acc[i][j][r];
                            double old_c = 0.0;
                            if constexpr (kPrefetchC) old_c = use_pre ? cpre[i][j][r] : (p.beta == 0.0 ? 0.0 : *cp);
                            else old_c = p.beta == 0.0 ? 0.0 : *cp;
                            *cp = p.beta == 0.0 ? v : v + p.beta * old_c;
                        }
                    }
                }
            }
        }
    }
}
