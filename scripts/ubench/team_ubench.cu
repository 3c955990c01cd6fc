// Microbenchmark of the chain team's step (trsv.cu): 4 warps, lane = row, each warp owns 8
// columns of a 32x32 complex G held in registers; per step: x slice by shuffles (or smem
// broadcast), 8 complex FMAs, partial to smem, mbarrier handoff, every warp reduces the 4
// partials.  Reports cycles per step for the variants.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 cfma(double2 acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
    return acc;
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                     su32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// var 0: shuffles + mbarrier; 1: per-warp smem copy of x + broadcast loads + mbarrier;
// 2: shuffles + named barrier; 3: no handoff (each warp alone: shuffles + FMAs only)
__global__ void k(int var, int steps, long long* out, double2* sink) {
    __shared__ __align__(16) double2 tpart[2][4][32];
    __shared__ __align__(16) double2 xw[4][32];
    __shared__ __align__(8) uint64_t pready[2];
    const int tid = threadIdx.x, lane = tid & 31, tw = tid >> 5, j0 = tw * 8;
    if (tid == 0) { mbar_init(&pready[0], 4); mbar_init(&pready[1], 4); }
    __syncthreads();
    double2 g1[8];
#pragma unroll
    for (int u = 0; u < 8; u++) g1[u] = make_double2(1e-3 * (lane + u), 1e-4 * u);
    double2 xk = make_double2(1.0 + lane, 0.5);
    const double2 y = make_double2(0.1 * lane, 0.2);
    long long t0 = clock64();
    for (int k = 0; k < steps; k++) {
        double2 xs[8];
        if (var == 1) {
            xw[tw][lane] = xk;
            __syncwarp();
#pragma unroll
            for (int u = 0; u < 8; u++) xs[u] = xw[tw][j0 + u];
        } else {
#pragma unroll
            for (int u = 0; u < 8; u++) {
                xs[u].x = __shfl_sync(0xffffffffu, xk.x, j0 + u);
                xs[u].y = __shfl_sync(0xffffffffu, xk.y, j0 + u);
            }
        }
        double2 p0 = make_double2(0, 0), p1 = make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
            p0 = cfma(p0, g1[u], xs[u]);
            p1 = cfma(p1, g1[u + 1], xs[u + 1]);
        }
        if (var == 3) {
            xk = make_double2(y.x - p0.x - p1.x, y.y - p0.y - p1.y);
            continue;
        }
        tpart[k & 1][tw][lane] = make_double2(p0.x + p1.x, p0.y + p1.y);
        if (var == 2) {
            bar_named(1, 128);
        } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(&pready[k & 1]);
            mbar_wait(&pready[k & 1], (k >> 1) & 1);
        }
        double2 s = tpart[k & 1][0][lane];
#pragma unroll
        for (int w = 1; w < 4; w++) s = make_double2(s.x + tpart[k & 1][w][lane].x, s.y + tpart[k & 1][w][lane].y);
        xk = make_double2(y.x - 1e-3 * s.x, y.y - 1e-3 * s.y);
    }
    long long t1 = clock64();
    if (tid == 0) out[0] = (t1 - t0) / steps;
    sink[tid] = xk;
}

int main() {
    long long* d;
    double2* s;
    cudaMalloc(&d, 8);
    cudaMalloc(&s, 128 * 16);
    const char* vn[] = {"shfl + mbarrier", "smem bcast + mbarrier", "shfl + bar.sync", "shfl + FMAs only (no handoff)"};
    for (int v = 0; v < 4; v++) {
        k<<<1, 128>>>(v, 10000, d, s);
        long long c;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("%-32s %lld cycles per step\n", vn[v], c);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
