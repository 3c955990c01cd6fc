// Microbenchmark: the y warps' triangular mat-vec y = D^{-1} s (B = 32, packed lower,
// column-major) in shared memory, one warp, lane = row (trsv.cu), cycles per mat-vec.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 cfma(double2 acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
    return acc;
}

// var 0: predicated loop (trsv.cu), 1: unpredicated (zero-padded full 32x32 column-major),
// 2: as 1 with 4 accumulators
__global__ void k(int var, int iters, long long* out, double2* sink) {
    constexpr int B = 32;
    __shared__ __align__(16) double2 inv[B * (B + 1) / 2];
    __shared__ __align__(16) double2 full[B * B];
    __shared__ __align__(16) double2 sR[B];
    const int r = threadIdx.x;
    for (int i = r; i < B * (B + 1) / 2; i += 32) inv[i] = make_double2(1e-3 * i, 0.5);
    for (int i = r; i < B * B; i += 32) full[i] = make_double2(1e-3 * i, 0.25);
    sR[r] = make_double2(1.0, 0.1 * r);
    __syncwarp();
    double2 acc = make_double2(0, 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        double2 y0 = make_double2(0, 0), y1 = make_double2(0, 0), y2 = y0, y3 = y0;
        if (var == 0) {
#pragma unroll
            for (int j = 0; j < B; j += 2) {
                if (j <= r) y0 = cfma(y0, inv[j * B - (j * (j - 1)) / 2 + (r - j)], sR[j]);
                if (j + 1 <= r) y1 = cfma(y1, inv[(j + 1) * B - ((j + 1) * j) / 2 + (r - j - 1)], sR[j + 1]);
            }
        } else if (var == 1) {
#pragma unroll
            for (int j = 0; j < B; j += 2) {
                y0 = cfma(y0, full[j * B + r], sR[j]);
                y1 = cfma(y1, full[(j + 1) * B + r], sR[j + 1]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < B; j += 4) {
                y0 = cfma(y0, full[j * B + r], sR[j]);
                y1 = cfma(y1, full[(j + 1) * B + r], sR[j + 1]);
                y2 = cfma(y2, full[(j + 2) * B + r], sR[j + 2]);
                y3 = cfma(y3, full[(j + 3) * B + r], sR[j + 3]);
            }
        }
        acc.x += y0.x + y1.x + y2.x + y3.x;
        acc.y += y0.y + y1.y + y2.y + y3.y;
        sR[r].x += 1e-30 * acc.x;   // next mat-vec depends on this one
        __syncwarp();
    }
    long long t1 = clock64();
    if (r == 0) out[0] = (t1 - t0) / iters;
    sink[r] = acc;
}

int main() {
    long long* d;
    double2* s;
    cudaMalloc(&d, 8);
    cudaMalloc(&s, 32 * 16);
    const char* vn[] = {"packed, predicated", "full 32x32, 2 acc", "full 32x32, 4 acc"};
    for (int v = 0; v < 3; v++) {
        k<<<1, 32>>>(v, 1000, d, s);
        long long c;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("%-24s %lld cycles per mat-vec\n", vn[v], c);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
