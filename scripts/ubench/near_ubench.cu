// Microbenchmark of the chain CTA's near phase (trsv.cu) in isolation: 256 threads, B rows,
// near list of L entries per row in shared memory, x ring in shared memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 cfma(double2 acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
    return acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int B, int TPR>
__global__ void k_near(int per_row, long long* cyc, double2* out, const double2* gsrc, int tma_bytes) {
    extern __shared__ __align__(16) unsigned char sm[];
    double2* ring = (double2*)sm;                      // 8*B
    double2* nval = ring + 8 * B;                      // B*per_row
    int* nloc = (int*)(nval + B * per_row);            // B+1
    int* ncol = nloc + B + 4;                          // B*per_row
    double2* sR = (double2*)(ncol + B * per_row + 4);
    const int tid = threadIdx.x;
    for (int i = tid; i < 8 * B; i += blockDim.x) ring[i] = make_double2(1e-3 * i, 1.0);
    for (int i = tid; i < B * per_row; i += blockDim.x) { nval[i] = make_double2(0.5, 0.25); ncol[i] = (i * 37) % (7 * B); }
    for (int i = tid; i <= B; i += blockDim.x) nloc[i] = i * per_row;
    __shared__ __align__(8) unsigned long long bar;
    __shared__ volatile int stop;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1) : "memory");
        stop = 0;
    }
    __syncthreads();
    if (tid >= 256) {   // TMA streamer warp
        if (tid == 256 && tma_bytes > 0) {
            unsigned char* dst = (unsigned char*)(sR + B + 16);
            uint32_t ph = 0;
            while (!stop) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(tma_bytes) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su32(dst)), "l"(gsrc), "r"(tma_bytes), "r"(su32(&bar)) : "memory");
                asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(&bar)), "r"(ph) : "memory");
                ph ^= 1;
            }
        }
        return;
    }
    __shared__ __align__(8) unsigned long long bar2;
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2)), "r"(1) : "memory");
    asm volatile("bar.sync 1, 256;" ::: "memory");
    long long t0 = clock64();
    long long tw = 0;
    for (int rep = 0; rep < 100; rep++) {
        if (tma_bytes < 0) {   // restage the near values (written by TMA) every step, like trsv.cu
            const uint32_t nb = (uint32_t)(B * per_row * 16);
            if (tid == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar2)), "r"(nb) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su32(nval)), "l"(gsrc), "r"(nb), "r"(su32(&bar2)) : "memory");
            }
            asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(&bar2)), "r"((uint32_t)(rep & 1)) : "memory");
        }
        long long ta = clock64();
        const int r = tid / TPR, q = tid % TPR;
        const int lo = nloc[r], hi = nloc[r + 1], len = hi - lo;
        const int e0 = lo + (q * len) / TPR, e1 = lo + ((q + 1) * len) / TPR;
        double2 acc = make_double2(0.0, 0.0), acc2 = acc;
        int e = e0;
        for (; e + 4 <= e1; e += 4) {
            const int c0 = ncol[e], c1 = ncol[e + 1], c2 = ncol[e + 2], c3 = ncol[e + 3];
            const double2 v0 = nval[e], v1 = nval[e + 1], v2 = nval[e + 2], v3 = nval[e + 3];
            const double2 x0 = ring[c0 & (8 * B - 1)], x1 = ring[c1 & (8 * B - 1)];
            const double2 x2 = ring[c2 & (8 * B - 1)], x3 = ring[c3 & (8 * B - 1)];
            acc = cfma(acc, v0, x0); acc2 = cfma(acc2, v1, x1); acc = cfma(acc, v2, x2); acc2 = cfma(acc2, v3, x3);
        }
        for (; e < e1; e++) acc = cfma(acc, nval[e], ring[ncol[e] & (8 * B - 1)]);
        acc.x += acc2.x; acc.y += acc2.y;
        for (int o = 1; o < TPR; o <<= 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        }
        if (q == 0) sR[r] = acc;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        tw += clock64() - ta;
        if (tid < B) ring[(rep * B + tid) & (8 * B - 1)] = make_double2(sR[tid].x * 1e-9, 1.0);
        asm volatile("bar.sync 1, 256;" ::: "memory");
    }
    long long t1 = clock64();
    if (tid == 0) { *cyc = (t1 - t0) / 100; cyc[1] = tw / 100; stop = 1; }
    if (tid < B) out[tid] = sR[tid];
}

__global__ void k_hog(const double4* __restrict__ src, size_t n, double* out, int loops) {
    double acc = 0;
    for (int l = 0; l < loops; l++)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            double2 v = __ldcs((const double2*)(src + i));
            acc += v.x + v.y;
        }
    if (acc == 1.2345) out[0] = acc;
}

int main() {
    long long* c; double2* o; long long h; double2* g;
    cudaMalloc(&c, 8); cudaMalloc(&o, 1024 * 16); cudaMalloc(&g, 1 << 20);
    cudaMalloc(&c, 16);
    double4* big; double* dout; size_t nbig = (size_t)1 << 27;   // 4 GiB
    cudaMalloc(&big, nbig * sizeof(double4)); cudaMalloc(&dout, 8); cudaMemset(big, 0, nbig * sizeof(double4));
    cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    for (int hog : {0, 1}) for (int tb : {0, -1}) for (int pr : {4, 35}) {
        if (hog) k_hog<<<147 * 2, 512, 0, s2>>>(big, nbig, dout, 3);
        size_t smem = 8 * 32 * 16 + 32 * pr * 16 + (33 + 4) * 4 + 32 * pr * 4 + 16 + 32 * 16 + 64 + 16 * 16 + 65536;
        cudaFuncSetAttribute(k_near<32, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_near<32, 8><<<1, 288, smem, s1>>>(pr, c, o, g, tb);
        cudaError_t e = cudaStreamSynchronize(s1);
        cudaDeviceSynchronize();
        long long hh[2];
        cudaMemcpy(hh, c, 16, cudaMemcpyDeviceToHost);
        printf("hog=%d near B=32 per_row=%d TMA mode %d: %lld cycles per step, %lld in near+barrier (%s)\n", hog, pr, tb, hh[0], hh[1], cudaGetErrorString(e));
    }
    return 0;
}
