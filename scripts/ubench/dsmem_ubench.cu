// Microbenchmark: DSMEM ping-pong latency between two CTAs of a cluster (sm_100a): one warp
// st.asyncs 512 B (32 x 16 B) into the peer's shared memory completing the peer's mbarrier
// transaction (+ one remote arrive.expect_tx), the peer waits and answers the same way.
// Reports the round trip in cycles (clock64 of CTA 0).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t par) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                     su32(bar)), "r"(par) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) k(int iters, long long* out, int mode) {
    __shared__ __align__(16) double2 buf[32];
    __shared__ __align__(8) uint64_t bar;
    const int lane = threadIdx.x;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;" ::: "memory");
    const uint32_t peer = rank ^ 1;
    const uint32_t pbuf = mapa(su32(buf), peer), pbar = mapa(su32(&bar), peer);
    double2 v = make_double2(lane, 1.0);
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        if (rank == 0) {
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(pbar), "r"(512)
                             : "memory");
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                             pbuf + lane * 16), "d"(v.x), "d"(v.y), "r"(pbar) : "memory");
            wait(&bar, it & 1);
            v = buf[lane];
        } else {
            wait(&bar, it & 1);
            v = buf[lane];
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(pbar), "r"(512)
                             : "memory");
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                             pbuf + lane * 16), "d"(v.x), "d"(v.y), "r"(pbar) : "memory");
        }
    }
    long long t1 = clock64();
    if (rank == 0 && lane == 0) out[0] = (t1 - t0) / iters;
    asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;" ::: "memory");
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    k<<<2, 32>>>(10000, d, 0);
    long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("DSMEM st.async ping-pong: %lld cycles round trip (%.0f ns at 1.965 GHz)\n", c, c / 1.965);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
