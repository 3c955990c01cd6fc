// Single-warp 32x32 complex GEMV with the matrix in registers and x broadcast by shuffles
// (the chain warp of trsv.cu v6), alone on an SM, and with other warps loading the SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 cfma(double2 acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
    return acc;
}

template <int MODE>
__global__ void k_gemv(double2* out, long long* cyc, int reps, int busy_warps) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp > 0) {   // load the SM: DFMA-heavy warps
        if (warp > busy_warps) return;
        double a = lane, b = 1.0 + lane;
        for (int i = 0; i < reps * 200; i++) { a = fma(a, 0.999, 1e-9); b = fma(b, 0.999, 1e-9); }
        if (a + b == 0.123) out[1000] = make_double2(a, b);
        return;
    }
    double2 g[32];
#pragma unroll
    for (int j = 0; j < 32; j++) g[j] = make_double2(1e-3 * (lane + j), 1e-3 * (lane - j));
    double2 xprev = make_double2(1.0 + lane, 0.5);
    long long t0 = clock64();
    for (int r = 0; r < reps; r++) {
        double2 acc[4] = {make_double2(0, 0), make_double2(0, 0), make_double2(0, 0), make_double2(0, 0)};
        if (MODE == 0) {
#pragma unroll
            for (int j = 0; j < 32; j++) {
                double2 xj;
                xj.x = __shfl_sync(0xffffffffu, xprev.x, j);
                xj.y = __shfl_sync(0xffffffffu, xprev.y, j);
                acc[j & 3] = cfma(acc[j & 3], g[j], xj);
            }
        } else {   // batches of 8 shuffles ahead of their FMAs
#pragma unroll
            for (int j0 = 0; j0 < 32; j0 += 8) {
                double2 xs[8];
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    xs[u].x = __shfl_sync(0xffffffffu, xprev.x, j0 + u);
                    xs[u].y = __shfl_sync(0xffffffffu, xprev.y, j0 + u);
                }
#pragma unroll
                for (int u = 0; u < 8; u++) acc[u & 3] = cfma(acc[u & 3], g[j0 + u], xs[u]);
            }
        }
        const double2 v = make_double2(acc[0].x + acc[1].x + acc[2].x + acc[3].x, acc[0].y + acc[1].y + acc[2].y + acc[3].y);
        xprev = make_double2(v.x * 1e-3 + 1.0, v.y * 1e-3);
    }
    long long t1 = clock64();
    if (lane == 0) *cyc = (t1 - t0) / reps;
    out[lane] = xprev;
}

int main() {
    double2* o; long long* c; long long h;
    cudaMalloc(&o, 2048 * 16); cudaMalloc(&c, 8);
    for (int busy : {0, 3, 9}) {
        k_gemv<0><<<1, 320>>>(o, c, 1000, busy); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("gemv interleaved, %d busy warps: %lld cycles\n", busy, h);
        k_gemv<1><<<1, 320>>>(o, c, 1000, busy); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("gemv batched,     %d busy warps: %lld cycles\n", busy, h);
    }
    return 0;
}
