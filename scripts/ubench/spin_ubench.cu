// Microbenchmark: cost of a 16-term complex FMA section (the y warps' G2 product in
// trsv.cu) on one warp while another warp of the same SMSP spins on
//   mode 0: nothing (spinner exits), 1: mbarrier.try_wait on a barrier that never completes,
//   2: ld.acquire.cta.shared polling, 3: try_wait with a suspend-time hint, 4: nanosleep(32) polling
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 cfma(double2 acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
    return acc;
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(int mode, int iters, long long* out, double2* sink) {
    __shared__ __align__(16) double2 G[32 * 32];
    __shared__ __align__(16) double2 X[32];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ volatile int stop;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 1024; i += blockDim.x) G[i] = make_double2(1e-3 * i, 0.5);
    if (tid < 32) X[tid] = make_double2(0.25, 1e-2 * tid);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1) : "memory");
        stop = 0;
    }
    __syncthreads();
    if (warp == 4) {   // same SMSP as warp 0
        if (mode == 1) {
            while (!stop) {
                uint32_t ok;
                asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}"
                             : "=r"(ok) : "r"(su32(&bar)) : "memory");
            }
        } else if (mode == 2) {
            int v;
            do asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(su32((const void*)&stop)) : "memory");
            while (!v);
        } else if (mode == 3) {
            while (!stop) {
                uint32_t ok;
                asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0, 1000;\nselp.u32 %0, 1, 0, p;\n}"
                             : "=r"(ok) : "r"(su32(&bar)) : "memory");
            }
        } else if (mode == 4) {
            while (!stop) __nanosleep(32);
        }
        return;
    }
    if (warp != 0) return;
    const int r = lane >> 1, q = lane & 1;
    double2 acc = make_double2(0, 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        double2 g0 = make_double2(0, 0), g1 = make_double2(0, 0);
#pragma unroll
        for (int t = 0; t < 16; t += 2) {
            g0 = cfma(g0, G[(q + 2 * t) * 32 + r], X[q + 2 * t]);
            g1 = cfma(g1, G[(q + 2 * (t + 1)) * 32 + r], X[q + 2 * (t + 1)]);
        }
        acc.x += g0.x + g1.x; acc.y += g0.y + g1.y;
        X[lane & 31].x += 0.0 * acc.x;   // keep iterations dependent through smem
        __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) {
        out[0] = (t1 - t0) / iters;
        stop = 1;
    }
    sink[lane] = acc;
}

// variants of the section without a spinner: 0 as k mode 0, 1 no smem store, 2 loads only,
// 3 FMAs on registers only, 4 loads hoisted into registers before the FMAs
__global__ void k2(int var, int iters, long long* out, double2* sink) {
    __shared__ __align__(16) double2 G[32 * 32];
    __shared__ __align__(16) double2 X[32];
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < 1024; i += blockDim.x) G[i] = make_double2(1e-3 * i, 0.5);
    if (tid < 32) X[tid] = make_double2(0.25, 1e-2 * tid);
    __syncthreads();
    const int r = lane >> 1, q = lane & 1;
    double2 acc = make_double2(0, 0);
    double2 gr[16], xr[16];
#pragma unroll
    for (int t = 0; t < 16; t++) {
        gr[t] = G[(q + 2 * t) * 32 + r];
        xr[t] = X[q + 2 * t];
    }
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        double2 g0 = make_double2(0, 0), g1 = make_double2(0, 0);
        if (var == 2) {
#pragma unroll
            for (int t = 0; t < 16; t++) {
                const double2 a = G[(q + 2 * t) * 32 + r], b = X[q + 2 * t];
                g0.x += a.x + b.x;
                g0.y += a.y + b.y;
            }
        } else if (var == 4) {
#pragma unroll
            for (int t = 0; t < 16; t++) {
                const double2 a = G[(q + 2 * t) * 32 + r];
                g0.x += a.x;
                g0.y += a.y;
            }
        } else if (var == 5) {
#pragma unroll
            for (int t = 0; t < 16; t++) {
                const double2 b = X[q + 2 * t];
                g0.x += b.x;
                g0.y += b.y;
            }
        } else if (var == 6) {
#pragma unroll
            for (int t = 0; t < 16; t++) {
                const double2 a = G[t * 64 + lane];
                g0.x += a.x;
                g0.y += a.y;
            }
        } else if (var == 7) {   // conflict-free G, x by shuffles from one register per lane
            const double2 xl = X[lane];
#pragma unroll
            for (int t = 0; t < 16; t += 2) {
                double2 b0, b1;
                b0.x = __shfl_sync(0xffffffffu, xl.x, q + 2 * t);
                b0.y = __shfl_sync(0xffffffffu, xl.y, q + 2 * t);
                b1.x = __shfl_sync(0xffffffffu, xl.x, q + 2 * t + 2);
                b1.y = __shfl_sync(0xffffffffu, xl.y, q + 2 * t + 2);
                g0 = cfma(g0, G[t * 64 + lane], b0);
                g1 = cfma(g1, G[(t + 1) * 64 + lane], b1);
            }
        } else if (var == 8) {   // conflict-free G, x broadcast loads
#pragma unroll
            for (int t = 0; t < 16; t += 2) {
                g0 = cfma(g0, G[t * 64 + lane], X[q + 2 * t]);
                g1 = cfma(g1, G[(t + 1) * 64 + lane], X[q + 2 * t + 2]);
            }
        } else if (var == 3) {
#pragma unroll
            for (int t = 0; t < 16; t += 2) {
                g0 = cfma(g0, gr[t], xr[t]);
                g1 = cfma(g1, gr[t + 1], xr[t + 1]);
            }
        } else {
#pragma unroll
            for (int t = 0; t < 16; t += 2) {
                g0 = cfma(g0, G[(q + 2 * t) * 32 + r], X[q + 2 * t]);
                g1 = cfma(g1, G[(q + 2 * (t + 1)) * 32 + r], X[q + 2 * (t + 1)]);
            }
        }
        acc.x += g0.x + g1.x;
        acc.y += g0.y + g1.y;
        if (var == 0) X[lane & 31].x += 0.0 * acc.x;
        __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) out[0] = (t1 - t0) / iters;
    sink[lane] = acc;
}

int main() {
    long long* d;
    double2* s;
    cudaMalloc(&d, 8);
    cudaMalloc(&s, 32 * 16);
    const char* names[] = {"none", "try_wait", "ld.acquire poll", "try_wait+hint", "nanosleep(32) poll"};
    for (int mode = 0; mode < 5; mode++) {
        k<<<1, 256>>>(mode, 1000, d, s);
        long long c;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("mode %d (%s): %lld cycles per 16-cfma section\n", mode, names[mode], c);
    }
    const char* vn[] = {"with smem store", "no store", "loads only", "register FMAs only", "G loads only (2-way)",
                        "X broadcast loads only", "G loads conflict-free", "cf G + shfl x", "cf G + bcast x"};
    for (int v = 0; v < 9; v++) {
        k2<<<1, 32>>>(v, 1000, d, s);
        long long c;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("variant %s: %lld cycles\n", vn[v], c);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
