// trsv.cu -- forward / backward substitution with the ILU factors (M^{-1} = U^{-1} L^{-1}).
//
// Applying the incomplete-LU preconditioner of sec. II inside the
// left-preconditioned GMRES of Eq. (8) is one forward
// substitution with the unit lower factor and one backward substitution with the
// upper factor per Arnoldi step.
//
// v1 (this file): level-scheduled substitution by ONE persistent CTA.  The rows of
// each dependency level (computed at setup, DevTri::lev_*) are independent; the CTA
// walks the levels in order, its warps take the rows of a level (one row per warp,
// lanes stride the row's entries), and a block barrier separates levels.  The
// factors of RCM-ordered Liouvillians have ~n/4 levels, so this
// kernel is latency-bound; it is the correctness baseline the faster substitution
// kernels are checked against.
#include "problem.h"

namespace ssb {

namespace {

template <bool kUpper>
__global__ void __launch_bounds__(1024, 1)
k_trsv_levels(int64_t nlev, const int64_t* __restrict__ lev_ptr, const int32_t* __restrict__ lev_rows,
              const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
              const double2* __restrict__ val, const double2* __restrict__ inv_diag,
              const double2* __restrict__ b, double2* x) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    for (int64_t l = 0; l < nlev; l++) {
        const int64_t p0 = lev_ptr[l], p1 = lev_ptr[l + 1];
        for (int64_t p = p0 + warp; p < p1; p += nwarps) {
            const int32_t i = lev_rows[p];
            const int64_t q0 = rowptr[i], q1 = rowptr[i + 1];
            double2 acc = make_double2(0.0, 0.0);
            for (int64_t q = q0 + lane; q < q1; q += 32) {
                const double2 a = val[q];
                const double2 v = x[col[q]];   // written by this CTA in an earlier level
                acc = cfma(acc, a, v);
            }
            acc = warp_sum2(acc);
            if (lane == 0) {
                double2 r = csub(b[i], acc);
                if (kUpper) r = cmul(r, inv_diag[i]);
                x[i] = r;
            }
        }
        __syncthreads();
    }
}

}  // namespace

void trsv_lower(const DevTri& L, const double2* b, double2* x, cudaStream_t s) {
    k_trsv_levels<false><<<1, 1024, 0, s>>>(L.nlev, L.lev_ptr, L.lev_rows, L.rowptr, L.col, L.val,
                                            nullptr, b, x);
    SSB_LAUNCHED();
}

void trsv_upper(const DevTri& U, const double2* b, double2* x, cudaStream_t s) {
    k_trsv_levels<true><<<1, 1024, 0, s>>>(U.nlev, U.lev_ptr, U.lev_rows, U.rowptr, U.col, U.val,
                                           U.inv_diag, b, x);
    SSB_LAUNCHED();
}

}  // namespace ssb
