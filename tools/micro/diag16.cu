// Micro: cost of the one-warp 16x16 [D | I] elimination used by chol_tile_block.
#include <cstdio>
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = y * fma(-0.5 * x, y * y, 1.5);
    return y * fma(-0.5 * x, y * y, 1.5);
}
template <int V>
__global__ void diag(const double* W, double* out, long long* cyc) {
    __shared__ double Ws[16 * 20], Dv[16 * 20], dg[16];
    const int lane = threadIdx.x & 31, j = lane & 15;
    const bool left = lane < 16;
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = left ? W[min(i, j) * 16 + max(i, j)] : (i == j ? 1.0 : 0.0);
    __syncwarp();
    long long c0 = clock64();
    double pv[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        double piv = __shfl_sync(0xffffffffu, x[k], k);
        if (V == 0) {
            const bool bad = !(piv > 0.0) || !isfinite(piv);
            if (bad) { piv = 1.0; if (lane == k) x[k] = 1.0; }
        }
        pv[k] = piv;
        const double pinv = rcp_nr(piv);
#pragma unroll
        for (int i = k + 1; i < 16; ++i) {
            const double f = __shfl_sync(0xffffffffu, x[i], k) * pinv;
            x[i] = fma(-f, x[k], x[i]);
        }
    }
    long long c1 = clock64();
    if (V == 2) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const double rsq = rsqrt_nr(pv[k]), sq = pv[k] * rsq;
            if (left) {
                if (k < j) Ws[k * 20 + j] = x[k] * rsq;
                else if (k == j) Ws[k * 20 + j] = sq;
            } else {
                Dv[j * 20 + k] = k >= j ? x[k] * rsq : 0.0;
            }
            if (lane == 0) dg[k] = sq;
        }
        __syncwarp();
        c1 = clock64();
        out[lane + 32] = Ws[lane] + Dv[lane] + dg[lane & 15];
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += x[k] + pv[k];
    out[lane] = s;
    if (lane == 0) *cyc = c1 - c0;
}
int main() {
    double h[256];
    for (int i = 0; i < 16; ++i) for (int j = 0; j < 16; ++j) h[i * 16 + j] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
    double *w, *o; long long* c; cudaMalloc(&w, sizeof(h)); cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 8);
    cudaMemcpy(w, h, sizeof(h), cudaMemcpyHostToDevice);
    long long cy;
    for (int r = 0; r < 2; ++r) diag<0><<<1, 32>>>(w, o, c);
    cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("with bad check: %lld clk\n", cy);
    for (int r = 0; r < 2; ++r) diag<1><<<1, 32>>>(w, o, c);
    cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("no bad check:   %lld clk\n", cy);
    for (int r = 0; r < 2; ++r) diag<2><<<1, 32>>>(w, o, c);
    cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("with writeout:  %lld clk\n", cy);
}
