// Micro: which part of chol_small's elimination step costs the ~900 clocks.
// Same thread/tile mapping (T=4, 288 threads), variants toggle pieces of the step.
#include <cstdio>
constexpr int kThr = 288, kMax = 128;
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double lds64(unsigned a) { double v; asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a)); return v; }
__device__ __forceinline__ void sts64p(bool p, unsigned a, double v) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.shared.f64 [%1], %2; }" :: "r"((unsigned)p), "r"(a), "d"(v));
}
__device__ __forceinline__ void sts64(unsigned a, double v) { asm volatile("st.shared.f64 [%0], %1;" :: "r"(a), "d"(v)); }
template <int T, int V, int kG = 16>
__global__ void __launch_bounds__(kThr) kern(const double* g, int b, double* out, long long* cyc) {
    constexpr int kTiles = kG * (kG + 1);
    __shared__ __align__(16) double bufL[2][kMax];
    __shared__ __align__(16) double bufR[2][kMax];
    __shared__ double s_sq[kMax];
    const int tid = threadIdx.x;
    int side = -1, ti = 0, tj = 0;
    if (tid < kTiles) {
        int t = tid < kTiles / 2 ? tid : tid - kTiles / 2;
        int row = 0;
        while (t >= kG - row) { t -= kG - row; ++row; }
        if (tid < kTiles / 2) { side = 0; ti = row; tj = row + t; } else { side = 1; ti = row + t; tj = row; }
    }
    const int i0 = ti * T, j0 = tj * T;
    double v[T][T];
#pragma unroll
    for (int a = 0; a < T; ++a)
#pragma unroll
        for (int c = 0; c < T; ++c) {
            const int i = i0 + a, j = j0 + c;
            v[a][c] = (side == 0 && i < b && j < b && i <= j) ? g[i + j * b] : (side == 1 && i == j ? 1.0 : 0.0);
        }
    for (int idx = tid; idx < 2 * kMax; idx += kThr) { (&bufL[0][0])[idx] = 0.0; (&bufR[0][0])[idx] = 0.0; }
    unsigned uL, uR, uS;
    asm volatile("mov.u32 %0, %1;" : "=r"(uL) : "r"((unsigned)__cvta_generic_to_shared(&bufL[0][0])));
    asm volatile("mov.u32 %0, %1;" : "=r"(uR) : "r"((unsigned)__cvta_generic_to_shared(&bufR[0][0])));
    asm volatile("mov.u32 %0, %1;" : "=r"(uS) : "r"((unsigned)__cvta_generic_to_shared(&s_sq[0])));
    auto publish4 = [&](int k, int buf) {
        const int a = k - i0;
        if (side < 0 || a < 0 || a >= T) return;
#pragma unroll
        for (int c = 0; c < T; ++c) {
            double x = v[0][c];
#pragma unroll
            for (int aa = 1; aa < T; ++aa) x = (a == aa) ? v[aa][c] : x;
            const int j = j0 + c;
            if (side == 0) {
                if (j == k) sts64(uS + 8 * k, x > 0.0 ? x : 1.0);
                sts64(uL + 8 * (buf * kMax + j), j > k ? x : 0.0);
            } else {
                sts64(uR + 8 * (buf * kMax + j), x);
            }
        }
    };
    auto publish = [&](int k, int buf) {
        const int a = k - i0;
        if (side < 0 || a < 0 || a >= T) return;
#pragma unroll
        for (int c = 0; c < T; ++c) {
            double x = v[0][c];
#pragma unroll
            for (int aa = 1; aa < T; ++aa) x = (a == aa) ? v[aa][c] : x;
            const int j = j0 + c;
            if (side == 0) {
                if (j == k) s_sq[k] = x > 0.0 ? x : 1.0;
                bufL[buf][j] = j > k ? x : 0.0;
            } else {
                bufR[buf][j] = x;
            }
        }
    };
    __syncthreads();
    publish(0, 0);
    __syncthreads();
    long long c0 = clock64();
    for (int k = 0; k < b; ++k) {
        const int p = k & 1;
        if (V == 5) { __syncthreads(); continue; }
        if (V == 6) {
            const double pinv = rcp_nr(lds64(uS + 8 * (k & 63)));
            v[0][0] += pinv;
            __syncthreads();
            continue;
        }
        if (V == 7) {
            const double pinv = rcp_nr(lds64(uS + 8 * (k & 63)));
            v[0][0] += pinv;
            if (tid == 37) sts64(uS + 8 * ((k + 1) & 63), v[0][0]);
            __syncthreads();
            continue;
        }
        if (V == 8) {
            if (side >= 0 && i0 + T - 1 > k) {
                const double pinv = rcp_nr(lds64(uS + 8 * k));
                const double* rbp = (side == 0 ? bufL[p] : bufR[p]) + j0;
                const double* fbp = bufL[p] + i0;
                const double2 r01 = *reinterpret_cast<const double2*>(rbp), r23 = *reinterpret_cast<const double2*>(rbp + 2);
                const double2 f01 = *reinterpret_cast<const double2*>(fbp), f23 = *reinterpret_cast<const double2*>(fbp + 2);
                double f[4] = {f01.x, f01.y, f23.x, f23.y}, rowk[4] = {r01.x, r01.y, r23.x, r23.y};
#pragma unroll
                for (int a = 0; a < T; ++a) f[a] = (i0 + a > k) ? f[a] * pinv : 0.0;
#pragma unroll
                for (int a = 0; a < T; ++a)
#pragma unroll
                    for (int c = 0; c < T; ++c) v[a][c] = fma(-f[a], rowk[c], v[a][c]);
            }
            if (k + 1 < b) publish4(k + 1, p ^ 1);
            __syncthreads();
            continue;
        }
        if (V == 9) {
            if (side >= 0 && i0 + T - 1 > k) {
                const double pinv = rcp_nr(lds64(uS + 8 * k));
                const double* rbp = (side == 0 ? bufL[p] : bufR[p]) + j0;
                const double* fbp = bufL[p] + i0;
                const double2 r01 = *reinterpret_cast<const double2*>(rbp), r23 = *reinterpret_cast<const double2*>(rbp + 2);
                const double2 f01 = *reinterpret_cast<const double2*>(fbp), f23 = *reinterpret_cast<const double2*>(fbp + 2);
                double f[4] = {f01.x, f01.y, f23.x, f23.y}, rowk[4] = {r01.x, r01.y, r23.x, r23.y};
#pragma unroll
                for (int a = 0; a < T; ++a) f[a] = (i0 + a > k) ? f[a] * pinv : 0.0;
#pragma unroll
                for (int a = 0; a < T; ++a)
#pragma unroll
                    for (int c = 0; c < T; ++c) v[a][c] = fma(-f[a], rowk[c], v[a][c]);
            }
            __syncthreads();
            continue;
        }
        if (V == 10 || V == 11) {
            if (side >= 0 && i0 + T - 1 > k) {
                const double pinv = rcp_nr(lds64(uS + 8 * k));
                const double* rbp = (side == 0 ? bufL[p] : bufR[p]) + (V == 10 ? 0 : j0);
                const double* fbp = bufL[p] + (V == 10 ? 0 : i0);
                const double2 r01 = *reinterpret_cast<const double2*>(rbp), r23 = *reinterpret_cast<const double2*>(rbp + 2);
                const double2 f01 = *reinterpret_cast<const double2*>(fbp), f23 = *reinterpret_cast<const double2*>(fbp + 2);
                double f[4] = {f01.x, f01.y, f23.x, f23.y}, rowk[4] = {r01.x, r01.y, r23.x, r23.y};
                if (V == 10) {
#pragma unroll
                    for (int a = 0; a < T; ++a) f[a] = (i0 + a > k) ? f[a] * pinv : 0.0;
#pragma unroll
                    for (int a = 0; a < T; ++a)
#pragma unroll
                        for (int c = 0; c < T; ++c) v[a][c] = fma(-f[a], rowk[c], v[a][c]);
                } else {
                    v[0][0] += f[0] + f[1] + f[2] + f[3] + rowk[0] + rowk[1] + rowk[2] + rowk[3];
                }
            }
            __syncthreads();
            continue;
        }
        if (V == 12) {
            if (side >= 0 && i0 + T - 1 > k) {
                const double pinv = rcp_nr(lds64(uS + 8 * k));
                const double* rbp = (side == 0 ? bufL[p] : bufR[p]) + j0;
                const double* fbp = bufL[p] + i0;
                const double2 r01 = *reinterpret_cast<const double2*>(rbp), r23 = *reinterpret_cast<const double2*>(rbp + 2);
                const double2 f01 = *reinterpret_cast<const double2*>(fbp), f23 = *reinterpret_cast<const double2*>(fbp + 2);
                double f[4] = {f01.x, f01.y, f23.x, f23.y}, rowk[4] = {r01.x, r01.y, r23.x, r23.y};
#pragma unroll
                for (int a = 0; a < T; ++a) f[a] = (i0 + a > k) ? f[a] * pinv : 0.0;
#pragma unroll
                for (int a = 0; a < T; ++a)
#pragma unroll
                    for (int c = 0; c < T; ++c) v[a][c] = fma(-f[a], rowk[c], v[a][c]);
            }
            {   // branch-free publish of row k+1
                const int kk = k + 1;
                const int a = kk - i0;
                const bool own = side >= 0 && a >= 0 && a < T && kk < b;
                const unsigned base = (side == 0 ? uL : uR) + 8 * ((p ^ 1) * kMax + j0);
#pragma unroll
                for (int c = 0; c < T; ++c) {
                    double x = v[0][c];
#pragma unroll
                    for (int aa = 1; aa < T; ++aa) x = (a == aa) ? v[aa][c] : x;
                    const int j = j0 + c;
                    const bool piv = own && side == 0 && j == kk;
                    sts64p(piv, uS + 8 * kk, x > 0.0 ? x : 1.0);
                    sts64p(own, base + 8 * c, (side == 1 || j > kk) ? x : 0.0);
                }
            }
            __syncthreads();
            continue;
        }
        if (V == 4) {
            if (side >= 0 && i0 + T - 1 > k) {
                const double pinv = rcp_nr(lds64(uS + 8 * k));
                const unsigned rb = (side == 0 ? uL : uR) + 8 * (p * kMax + j0);
                const unsigned fb = uL + 8 * (p * kMax + i0);
                double f[T], rowk[T];
#pragma unroll
                for (int a = 0; a < T; ++a) f[a] = (i0 + a > k) ? lds64(fb + 8 * a) * pinv : 0.0;
#pragma unroll
                for (int c = 0; c < T; ++c) rowk[c] = lds64(rb + 8 * c);
#pragma unroll
                for (int a = 0; a < T; ++a)
#pragma unroll
                    for (int c = 0; c < T; ++c) v[a][c] = fma(-f[a], rowk[c], v[a][c]);
            }
            if (k + 1 < b) publish4(k + 1, p ^ 1);
            __syncthreads();
            continue;
        }
        if (side >= 0 && i0 + T - 1 > k) {
            const double pinv = (V == 2) ? 0.5 : rcp_nr(s_sq[k]);
            const double* rb = side == 0 ? bufL[p] : bufR[p];
            double f[T], rowk[T];
#pragma unroll
            for (int a = 0; a < T; ++a) f[a] = (i0 + a > k) ? bufL[p][i0 + a] * pinv : 0.0;
#pragma unroll
            for (int c = 0; c < T; ++c) rowk[c] = rb[j0 + c];
            if (V != 1) {
#pragma unroll
                for (int a = 0; a < T; ++a)
#pragma unroll
                    for (int c = 0; c < T; ++c) v[a][c] = fma(-f[a], rowk[c], v[a][c]);
            } else {
                v[0][0] += f[0] * rowk[0];
            }
        }
        if (V != 3 && k + 1 < b) publish(k + 1, p ^ 1);
        if (V == 3 && tid == 0) { bufL[p ^ 1][k] = v[0][0]; s_sq[k + 1] = 2.0; }
        __syncthreads();
    }
    long long c1 = clock64();
    if (tid == 0) *cyc = c1 - c0;
    double s = 0;
#pragma unroll
    for (int a = 0; a < T; ++a)
#pragma unroll
        for (int c = 0; c < T; ++c) s += v[a][c];
    out[tid] = s;
}
int main() {
    const int b = 64;
    double *g, *o; long long* c;
    cudaMalloc(&g, 8 * b * b); cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 64);
    double h[64 * 64];
    for (int i = 0; i < b; ++i) for (int j = 0; j < b; ++j) h[i + j * b] = (i == j ? 3.0 * b : 0.0) + 1.0 / (1 + i + j);
    cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
    long long cy;
    const char* names[] = {"full", "no DFMA update", "no rcp", "no publish", "explicit smem addr", "bar only", "lds+rcp+bar", "lds+rcp+1 sts+bar", "vector lds", "vector lds, no publish", "broadcast lds, no publish", "vector lds no math", "branch-free publish"};
    for (int r = 0; r < 2; ++r) kern<8, 0, 8><<<1, kThr>>>(g, b, o, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("T=8 grid 8 full   %.0f clk/step (%s)\n", cy / (double)b, cudaGetErrorString(cudaGetLastError()));
    for (int r = 0; r < 2; ++r) kern<8, 3, 8><<<1, kThr>>>(g, b, o, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("T=8 grid 8 no publish %.0f clk/step\n", cy / (double)b);
#define RUN(V) for (int r = 0; r < 2; ++r) kern<4, V><<<1, kThr>>>(g, b, o, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); \
    printf("%-16s %.0f clk/step\n", names[V], cy / (double)b);
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8) RUN(9) RUN(10) RUN(11) RUN(12)
}
