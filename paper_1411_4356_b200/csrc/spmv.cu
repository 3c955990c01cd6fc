// spmv.cu -- y = A x for the complex128 CSR Liouvillian (L~_RCM).
//
// The GMRES operator of Eq. (8) applies L~_RCM once per Arnoldi
// step.  L~ has ~10-13 entries per row (Eq. (3): 5-point H on each side of rho plus
// three dissipator jumps) and one long row (row of rho_00: + N trace entries).
// Four lanes cooperate on a row: a warp covers 8 consecutive rows, i.e. ~100
// contiguous (col, val) entries, so the int32 column and 16-byte value streams are
// read fully coalesced; x is gathered through L2 (x of the largest config is
// 33 MB, L2-resident).  HBM-bound: algorithmic bytes per launch =
// nnz*(16+4) + (n+1)*8 + 2*n*16 (values, columns, row pointers, x once, y).
#include "problem.h"

namespace ssb {

namespace {
constexpr int kTPR = 4;   // threads per row

__global__ void __launch_bounds__(256) k_spmv(int64_t n, const int64_t* __restrict__ rowptr,
                                              const int32_t* __restrict__ col,
                                              const double2* __restrict__ val,
                                              const double2* __restrict__ x, double2* __restrict__ y) {
    const int sub = threadIdx.x & (kTPR - 1);
    const unsigned gmask = 0xFu << ((threadIdx.x & 31) & ~(kTPR - 1));   // the row's 4 lanes
    const int64_t stride = (int64_t)gridDim.x * blockDim.x / kTPR;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kTPR; r < n; r += stride) {
        const int64_t b = rowptr[r], e = rowptr[r + 1];
        double2 acc = make_double2(0.0, 0.0);
        for (int64_t q = b + sub; q < e; q += kTPR) {
            const double2 a = __ldg(val + q);
            const double2 v = __ldg(x + __ldg(col + q));
            acc = cfma(acc, a, v);
        }
#pragma unroll
        for (int o = kTPR / 2; o > 0; o >>= 1) {
            acc.x += __shfl_xor_sync(gmask, acc.x, o);
            acc.y += __shfl_xor_sync(gmask, acc.y, o);
        }
        if (sub == 0) y[r] = acc;
    }
}
}  // namespace

void spmv(const DevCSR& A, const double2* x, double2* y, cudaStream_t s) {
    const int T = 256;
    const int64_t threads = A.n * kTPR;
    int blocks = (int)std::min<int64_t>((threads + T - 1) / T, (int64_t)kNumSMs * 16);
    k_spmv<<<blocks, T, 0, s>>>(A.n, A.rowptr, A.col, A.val, x, y);
    SSB_LAUNCHED();
}

}  // namespace ssb
