// spmv.cu -- y = A x for the complex128 Liouvillian operator of the hot path
// (A' = Pi^T L~_RCM, setup.cpp).
//
// The GMRES operator of Eq. (8) applies the Liouvillian once per Arnoldi
// step.  L~ has ~10-13 entries per row (Eq. (3): 5-point H on each side of rho plus
// three dissipator jumps) and one long row (row of rho_00: + N trace entries, Eq. (5)).
//
// Layout: SELL-32 (built at setup, problem.h): a warp owns a slice of 32 consecutive rows,
// lane = row, and walks the slice's columns e = 0 .. width-1; entry e of the 32 rows is
// one contiguous 128 B column-index line and one 512 B value line, so both streams are
// read fully coalesced with no per-row pointer chase, and the x gathers of a step are
// independent (2 entries in flight per lane).  x is gathered through L2 (RCM-banded,
// L2-resident).  The rows longer than kSellLong (the trace row) are summed from the CSR
// by one warp each (extra blocks of the same launch).
// HBM-bound: algorithmic bytes per launch = nnz*(16+4) + (n+1)*8 + 2*n*16 (values,
// columns, row pointers, x once, y); the SELL padding is real traffic beyond that.
#include "problem.h"

namespace ssb {

namespace {
constexpr int kTPR = 4;        // CSR fallback: threads per row
constexpr int kSellT = 256;    // SELL: threads per block (8 slices)

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

// blocks [0, sblocks): slices (8 per block); blocks [sblocks, ...): the long rows, one warp each
__global__ void __launch_bounds__(kSellT) k_spmv_sell(int64_t n, int64_t nslices, const int64_t* __restrict__ sptr,
                                                      const int32_t* __restrict__ scol,
                                                      const double2* __restrict__ sval, int64_t nlong,
                                                      const int64_t* __restrict__ lrows,
                                                      const int64_t* __restrict__ rowptr,
                                                      const int32_t* __restrict__ col,
                                                      const double2* __restrict__ val, int sblocks,
                                                      const double2* __restrict__ x, double2* __restrict__ y) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if ((int)blockIdx.x >= sblocks) {
        const int64_t j = (int64_t)(blockIdx.x - sblocks) * (kSellT / 32) + warp;
        if (j >= nlong) return;
        const int64_t r = lrows[j];
        double2 acc = make_double2(0.0, 0.0);
        for (int64_t q = rowptr[r] + lane; q < rowptr[r + 1]; q += 32) acc = cfma(acc, __ldg(val + q), __ldg(x + __ldg(col + q)));
        acc = warp_sum2(acc);
        if (lane == 0) y[r] = acc;
        return;
    }
    const int64_t s = (int64_t)blockIdx.x * (kSellT / 32) + warp;
    if (s >= nslices) return;
    const int64_t b = __ldg(sptr + s), w = (__ldg(sptr + s + 1) - b) >> 5;
    const int32_t* cp = scol + b + lane;
    const double2* vp = sval + b + lane;
    const int32_t c0 = __ldcs(cp);
    double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
    if (c0 >= 0) {
        acc0 = cfma(acc0, __ldcs(vp), __ldg(x + c0));
        int64_t e = 1;
        for (; e + 1 < w; e += 2) {
            const int32_t ca = __ldcs(cp + 32 * e), cb = __ldcs(cp + 32 * (e + 1));
            const double2 va = __ldcs(vp + 32 * e), vb = __ldcs(vp + 32 * (e + 1));
            acc1 = cfma(acc1, va, __ldg(x + ca));
            acc0 = cfma(acc0, vb, __ldg(x + cb));
        }
        if (e < w) acc1 = cfma(acc1, __ldcs(vp + 32 * e), __ldg(x + __ldcs(cp + 32 * e)));
    }
    const int64_t r = s * 32 + lane;
    if (r < n && c0 >= 0) y[r] = cadd(acc0, acc1);
}
}  // namespace

void spmv(const DevCSR& A, const double2* x, double2* y, cudaStream_t s) {
    if (A.sptr) {
        const int sblocks = (int)((A.nslices + kSellT / 32 - 1) / (kSellT / 32));
        const int lblocks = (int)((A.nlong + kSellT / 32 - 1) / (kSellT / 32));
        k_spmv_sell<<<sblocks + lblocks, kSellT, 0, s>>>(A.n, A.nslices, A.sptr, A.scol, A.sval, A.nlong, A.lrows,
                                                         A.rowptr, A.col, A.val, sblocks, x, y);
        SSB_LAUNCHED();
        return;
    }
    const int T = 256;
    const int64_t threads = A.n * kTPR;
    int blocks = (int)std::min<int64_t>((threads + T - 1) / T, (int64_t)kNumSMs * 16);
    k_spmv<<<blocks, T, 0, s>>>(A.n, A.rowptr, A.col, A.val, x, y);
    SSB_LAUNCHED();
}

}  // namespace ssb
