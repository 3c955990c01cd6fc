// Microbenchmark: one warp's DFMA dependent-chain latency and issue rate, and LDS.128 latency
// on sm_100a (clock64 cycles).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int NC>
__global__ void k_chain(int iters, long long* out, double* sink, double a, double b) {
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; c++) acc[c] = threadIdx.x * 1e-3 + c;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 16; u++)
#pragma unroll
            for (int c = 0; c < NC; c++) acc[c] = fma(acc[c], a, b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < NC; c++) s += acc[c];
    sink[threadIdx.x] = s;
    if (threadIdx.x == 0) out[0] = t1 - t0;
}

__global__ void k_lds(int iters, long long* out, int* sink) {
    __shared__ int buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i + 1) & 1023;
    __syncthreads();
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) p = buf[p];
    long long t1 = clock64();
    sink[threadIdx.x] = p;
    if (threadIdx.x == 0) out[0] = t1 - t0;
}

int main() {
    long long* d;
    double* s;
    int* si;
    cudaMalloc(&d, 8);
    cudaMalloc(&s, 1024 * 8);
    cudaMalloc(&si, 1024 * 4);
    const int iters = 1000;
    long long c;
    k_chain<1><<<1, 32>>>(iters, d, s, 1.0000001, 1e-9);
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("1 chain, 1 warp: %.2f cycles per dependent DFMA\n", (double)c / (iters * 16));
    k_chain<8><<<1, 32>>>(iters, d, s, 1.0000001, 1e-9);
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("8 chains, 1 warp: %.2f cycles per DFMA instruction\n", (double)c / (iters * 16 * 8));
    k_chain<8><<<1, 128>>>(iters, d, s, 1.0000001, 1e-9);
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("8 chains, 4 warps (1 per SMSP): %.2f cycles per warp DFMA instruction\n", (double)c / (iters * 16 * 8));
    k_chain<8><<<1, 256>>>(iters, d, s, 1.0000001, 1e-9);
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("8 chains, 8 warps (2 per SMSP): %.2f cycles per warp DFMA instruction (per warp)\n",
           (double)c / (iters * 16 * 8));
    k_lds<<<1, 32>>>(iters, d, si);
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("LDS.32 dependent latency: %.2f cycles\n", (double)c / iters);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
