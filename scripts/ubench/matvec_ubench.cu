// Microbenchmarks for the block substitution's critical path (diagnostic, not product):
//  1. packed lower-triangular B x B complex mat-vec out of shared memory (the trsv.cu mapping)
//  2. DFMA throughput per SM
//  3. cross-CTA ping-pong latency through global memory (st.relaxed / ld.relaxed polling)
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1411_4356_b200/csrc/trimv.cuh"

__device__ __forceinline__ double2 cfma(double2 acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
    return acc;
}

template <int B, int NT, int MODE>
__global__ void k_matvec(double2* out, long long* cyc, int reps) {
    extern __shared__ double2 sm[];
    constexpr int PK = B * (B + 1) / 2;
    double2* sInv = sm;
    double2* sR = sm + PK;
    double2* sPart = sR + B;
    const int tid = threadIdx.x;
    for (int i = tid; i < PK; i += NT) sInv[i] = make_double2(1e-3 * (i % 7), 1e-3 * (i % 5));
    for (int i = tid; i < B; i += NT) sR[i] = make_double2(1.0 + i, 0.5);
    __syncthreads();
    long long t0 = clock64();
    for (int rep = 0; rep < reps; rep++) {
        if (MODE == 4) {
        } else if (MODE == 6 || MODE == 7 || MODE == 8 || MODE == 9) {
            constexpr int CW = MODE == 6 ? 16 : (MODE == 7 ? 32 : (MODE == 8 ? 8 : 4));
            ssb::trimv::matvec_tiles<B, CW, NT / 32>(sInv, sR, sPart, threadIdx.x >> 5, threadIdx.x & 31);
            __syncthreads();
            if (tid < B) {
                double2 s = ssb::trimv::sum_row<B, CW>(sPart, tid);
                sR[tid] = make_double2(s.x * 1e-3, s.y * 1e-3);
            }
            __syncthreads();
            continue;
        } else if (MODE == 5) {   // warp owns row pairs; lanes stride columns; shuffle reduce
            constexpr int W = NT / 32, RPW = B / W;
            const int lane = tid & 31, w = tid >> 5;
            for (int q = 0; q < RPW / 2; q++) {
                const int i1 = w * (RPW / 2) + q, i2 = B - 1 - i1;
                double2 s1 = make_double2(0, 0), s2 = s1;
                for (int j = lane; j <= i2; j += 32) {
                    const double2 rj = sR[j];
                    const int o2 = (i2 * (i2 + 1)) / 2 + j;          // row-major packed
                    s2 = cfma(s2, sInv[o2], rj);
                    if (j <= i1) s1 = cfma(s1, sInv[(i1 * (i1 + 1)) / 2 + j], rj);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    s1.x += __shfl_xor_sync(0xffffffffu, s1.x, o);
                    s1.y += __shfl_xor_sync(0xffffffffu, s1.y, o);
                    s2.x += __shfl_xor_sync(0xffffffffu, s2.x, o);
                    s2.y += __shfl_xor_sync(0xffffffffu, s2.y, o);
                }
                if (lane == 0) { sPart[i1] = s1; sPart[i2] = s2; }
            }
        } else if (MODE == 2 || MODE == 3) {
            constexpr int kPairs = B / 2, TP = NT / kPairs;
            const int pr = tid % kPairs, sub = tid / kPairs;
            const int i1 = pr, i2 = B - 1 - pr;
            double2 s1 = make_double2(0, 0), s2 = s1;
            const double2 cst = make_double2(1e-3 * pr, 2e-3);
            for (int j = sub; j <= i2; j += TP) {
                const int cs = j * B - (j * (j - 1)) / 2;
                if (MODE == 2) {
                    s2 = cfma(s2, cst, cst);
                    if (j <= i1) s1 = cfma(s1, cst, cst);
                } else {
                    const double2 v = sInv[cs + (i2 - j)];
                    s2.x += v.x; s2.y += v.y;
                    if (j <= i1) { const double2 u = sInv[cs + (i1 - j)]; s1.x += u.x; s1.y += u.y; }
                }
            }
            sPart[sub * B + i1] = s1;
            sPart[sub * B + i2] = s2;
        } else if (MODE == 0) {   // trsv.cu mapping: row pairs, TP threads per pair
            constexpr int kPairs = B / 2, TP = NT / kPairs;
            const int pr = tid % kPairs, sub = tid / kPairs;
            const int i1 = pr, i2 = B - 1 - pr;
            double2 s1 = make_double2(0, 0), s2 = s1, t1 = s1, t2 = s1;
            int j = sub;
            for (; j + TP <= i1; j += 2 * TP) {
                const int ja = j, jb = j + TP;
                const int ca = ja * B - (ja * (ja - 1)) / 2, cb = jb * B - (jb * (jb - 1)) / 2;
                const double2 ra = sR[ja], rb = sR[jb];
                s2 = cfma(s2, sInv[ca + (i2 - ja)], ra);
                t2 = cfma(t2, sInv[cb + (i2 - jb)], rb);
                s1 = cfma(s1, sInv[ca + (i1 - ja)], ra);
                t1 = cfma(t1, sInv[cb + (i1 - jb)], rb);
            }
            for (; j <= i2; j += TP) {
                const int cs = j * B - (j * (j - 1)) / 2;
                const double2 rj = sR[j];
                s2 = cfma(s2, sInv[cs + (i2 - j)], rj);
                if (j <= i1) s1 = cfma(s1, sInv[cs + (i1 - j)], rj);
            }
            sPart[sub * B + i1] = make_double2(s1.x + t1.x, s1.y + t1.y);
            sPart[sub * B + i2] = make_double2(s2.x + t2.x, s2.y + t2.y);
        } else {   // column-oriented: thread owns row i = tid % B, strided columns, 4 accumulators
            constexpr int P = NT / B;
            const int i = tid % B, part = tid / B;
            double2 a0 = make_double2(0, 0), a1 = a0, a2 = a0, a3 = a0;
            int j = part;
            for (; j + 3 * P <= i; j += 4 * P) {
                a0 = cfma(a0, sInv[j * B - (j * (j - 1)) / 2 + i - j], sR[j]);
                const int j1 = j + P, j2 = j + 2 * P, j3 = j + 3 * P;
                a1 = cfma(a1, sInv[j1 * B - (j1 * (j1 - 1)) / 2 + i - j1], sR[j1]);
                a2 = cfma(a2, sInv[j2 * B - (j2 * (j2 - 1)) / 2 + i - j2], sR[j2]);
                a3 = cfma(a3, sInv[j3 * B - (j3 * (j3 - 1)) / 2 + i - j3], sR[j3]);
            }
            for (; j <= i; j += P) a0 = cfma(a0, sInv[j * B - (j * (j - 1)) / 2 + i - j], sR[j]);
            sPart[part * B + i] = make_double2(a0.x + a1.x + a2.x + a3.x, a0.y + a1.y + a2.y + a3.y);
        }
        __syncthreads();
        if (tid < B) {
            double2 s = sPart[tid];
            constexpr int Q = MODE == 5 ? 1 : (MODE == 1 ? NT / B : NT / (B / 2));  // unused for tiles
            for (int q = 1; q < Q; q++) { s.x += sPart[q * B + tid].x; s.y += sPart[q * B + tid].y; }
            sR[tid] = make_double2(s.x * 1e-3, s.y * 1e-3);
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
    if (tid < B) out[blockIdx.x * B + tid] = sR[tid];
}

__global__ void k_dfma(double* out, long long* cyc) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double m = 0.999999, c = 1e-9;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < 4096; i++) {
        a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
        a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_pingpong(volatile unsigned long long* box, long long* res, int iters) {
    // CTA 0 and CTA 1 bounce a counter through global memory
    const int me = blockIdx.x;
    if (threadIdx.x != 0) return;
    unsigned long long* p = (unsigned long long*)box;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (me == 0) {
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"((unsigned long long)(2 * i + 1)) : "memory");
            unsigned long long v;
            do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p + 16) : "memory"); } while (v != (unsigned long long)(2 * i + 2));
        } else {
            unsigned long long v;
            do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); } while (v != (unsigned long long)(2 * i + 1));
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p + 16), "l"((unsigned long long)(2 * i + 2)) : "memory");
        }
    }
    long long t1 = clock64();
    if (me == 0) res[0] = (t1 - t0) / iters;
}

template <int B, int NT, int MODE>
void run_mv(const char* name) {
    constexpr int PK = B * (B + 1) / 2;
    size_t smem = (PK + B + 17 * B) * sizeof(double2);
    double2* out;
    long long* cyc;
    cudaMalloc(&out, 148 * B * sizeof(double2));
    cudaMalloc(&cyc, 148 * sizeof(long long));
    cudaFuncSetAttribute(k_matvec<B, NT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_matvec<B, NT, MODE><<<148, NT, smem>>>(out, cyc, 200);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double2 o[2];
    cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
    printf("%s B=%d NT=%d mode=%d: %lld cycles per mat-vec+reduce (%s) out0=%.12e\n", name, B, NT, MODE, h[0], cudaGetErrorString(e), o[0].x);
    cudaFree(out);
    cudaFree(cyc);
}

__global__ void k_lat(double* out, long long* cyc) {
    double a = threadIdx.x * 1e-3;
    const double m = 0.999999, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < 1024; i++) a = fma(a, m, c);
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int B, int CW, int A, int S>
__global__ void k_onetile(double2* out, long long* cyc) {
    extern __shared__ double2 sm[];
    constexpr int PK = B * (B + 1) / 2;
    double2* sInv = sm;
    double2* sR = sm + PK;
    double2* sPart = sR + B;
    for (int i = threadIdx.x; i < PK; i += blockDim.x) sInv[i] = make_double2(1e-3 * (i % 7), 1e-3 * (i % 5));
    for (int i = threadIdx.x; i < B; i += blockDim.x) sR[i] = make_double2(1.0 + i, 0.5);
    __syncwarp();
    long long t0 = clock64();
    for (int rep = 0; rep < 100; rep++) {
        ssb::trimv::tile<B, CW>(A, S, sInv, sR, sPart, threadIdx.x);
        __syncwarp();
        sR[threadIdx.x % B] = sPart[S * B + 32 * A + threadIdx.x];
        __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 100;
    out[threadIdx.x] = sR[threadIdx.x];
}

int main() {
    {
        double* o; long long* c; long long h;
        cudaMalloc(&o, 4096 * 8); cudaMalloc(&c, 64);
        k_lat<<<1, 32>>>(o, c); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("DFMA dependent latency: %.2f cycles\n", h / 1024.0);
        double2* o2; cudaMalloc(&o2, 4096 * 16);
        cudaFuncSetAttribute(k_onetile<64, 16, 1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
        k_onetile<64, 16, 1, 0><<<1, 32, 100000>>>(o2, c); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("one full tile (16 CMAC/lane) single warp: %lld cycles\n", h);
        cudaFuncSetAttribute(k_onetile<64, 16, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
        k_onetile<64, 16, 1, 2><<<1, 32, 100000>>>(o2, c); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("one diagonal tile single warp: %lld cycles (%s)\n", h, cudaGetErrorString(cudaGetLastError()));
    }
    run_mv<128, 512, 0>("matvec");
    run_mv<128, 512, 6>("tiles16");
    run_mv<128, 512, 7>("tiles32");
    run_mv<128, 256, 6>("tiles16");
    run_mv<64, 256, 6>("tiles16");
    run_mv<64, 256, 7>("tiles32");
    run_mv<64, 128, 6>("tiles16");
    run_mv<64, 256, 8>("tiles8");
    run_mv<64, 512, 8>("tiles8");
    run_mv<64, 512, 9>("tiles4");
    run_mv<64, 512, 6>("tiles16");
    run_mv<128, 512, 8>("tiles8");
    run_mv<128, 1024, 8>("tiles8");
    run_mv<128, 512, 2>("matvec-noload");
    run_mv<128, 512, 3>("matvec-loadonly");
    run_mv<128, 512, 4>("barriers+reduce");
    run_mv<128, 512, 5>("matvec-warprow");
    run_mv<128, 256, 5>("matvec-warprow");
    run_mv<64, 256, 5>("matvec-warprow");
    run_mv<128, 512, 1>("matvec");
    run_mv<128, 256, 0>("matvec");
    run_mv<128, 256, 1>("matvec");
    run_mv<64, 256, 0>("matvec");
    run_mv<64, 256, 1>("matvec");
    {
        double* o;
        long long* c;
        cudaMalloc(&o, 148 * 1024 * sizeof(double));
        cudaMalloc(&c, 148 * sizeof(long long));
        for (int nt : {128, 256, 512, 1024}) {
            k_dfma<<<148, nt>>>(o, c);
            cudaDeviceSynchronize();
            long long h;
            cudaMemcpy(&h, c, sizeof(h), cudaMemcpyDeviceToHost);
            printf("dfma NT=%d: %.1f DFMA/cycle/SM\n", nt, 4096.0 * 8 * nt / h);
        }
    }
    {
        unsigned long long* box;
        long long* r;
        cudaMalloc(&box, 4096);
        cudaMemset(box, 0, 4096);
        cudaMalloc(&r, 8);
        k_pingpong<<<2, 32>>>(box, r, 1000);
        cudaDeviceSynchronize();
        long long h;
        cudaMemcpy(&h, r, 8, cudaMemcpyDeviceToHost);
        printf("pingpong round trip: %lld cycles (two one-way handoffs)\n", h);
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock %d kHz\n", clk);
    return 0;
}
