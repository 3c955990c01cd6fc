// common.cuh -- shared device/host helpers of the B200 steady-state library.
//
// complex128 is carried as double2 (x = re, y = im), 16-byte aligned, so a
// complex vector streams as 128-bit loads (LDG.E.128).  No FMA contraction is
// relied upon for parity: kernels whose results are compared bit-for-bit with
// the oracle use the explicit __dmul_rn/__dadd_rn/__dsub_rn intrinsics.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

namespace ssb {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
std::atomic<int64_t>& launch_counter();

struct Error {
    int code;
    std::string msg;
};

#define SSB_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw ::ssb::Error{2, std::string(#call) + ": " + cudaGetErrorString(e_)};  \
    } while (0)

#define SSB_CHECK(cond, code, msg)                         \
    do {                                                   \
        if (!(cond)) throw ::ssb::Error{(code), (msg)};    \
    } while (0)

// count every launch of our kernels (gpu_launches evidence) and check it
#define SSB_LAUNCHED()                                                         \
    do {                                                                       \
        ::ssb::launch_counter().fetch_add(1, std::memory_order_relaxed);       \
        SSB_CUDA(cudaGetLastError());                                          \
    } while (0)

// ------------------------------------------------------------------ complex
__host__ __device__ __forceinline__ double2 cmk(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
// conj(a) * b
__host__ __device__ __forceinline__ double2 cdotc(double2 a, double2 b) {
    return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
#ifdef __CUDACC__
// acc - a*b  (FMA-friendly; used where bit-parity is not required)
__device__ __forceinline__ double2 cfms(double2 acc, double2 a, double2 b) {
    acc.x = fma(-a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(-a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
    return acc;
}
__device__ __forceinline__ double2 cfma(double2 acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
    return acc;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    return v;
}

#endif  // __CUDACC__

constexpr int kNumSMs = 148;

inline int grid_for(int64_t work, int threads, int max_blocks = 148 * 8) {
    int64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return (int)b;
}

}  // namespace ssb
