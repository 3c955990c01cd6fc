// trimv.cuh -- dense lower-triangular complex mat-vec x = D^{-1} r out of shared memory,
// the step of the block substitution (trsv.cu) that sits on the dependency chain.
//
// D^{-1} is stored packed, column-major (column j holds rows j..B-1 at cs(j) = jB - j(j-1)/2),
// complex128.  The mat-vec is bound by shared-memory bandwidth (B(B+1)/2 x 16 bytes at
// 128 B/clk) and by instruction issue (an FP64 FMA takes 2 issue slots of an SMSP), so the
// work is cut into compile-time tiles: a warp owns 32 consecutive rows and a segment of
// CW consecutive columns; with the column index a compile-time constant every shared
// load is [row register + immediate] and carries no address arithmetic.  The
// (row block, column segment) tiles that touch the lower triangle are enumerated at
// compile time and dealt round-robin to the warps; tile partial sums land in
// sPart[segment][row] and are added in segment order (deterministic).
#pragma once

#include "common.cuh"

namespace ssb {
namespace trimv {

template <int B, int CW>
struct Tiles {
    static constexpr int kRowBlocks = B / 32;
    static constexpr int kSegs = B / CW;
    // tiles of row block a: segments s with s*CW <= 32a + 31
    __host__ __device__ static constexpr int segs_of(int a) { return (32 * a + 31) / CW + 1; }
    static constexpr int count() {
        int c = 0;
        for (int a = 0; a < kRowBlocks; a++) c += segs_of(a);
        return c;
    }
    static constexpr int kCount = count();
    static constexpr int row_block(int t) {
        for (int a = 0; a < kRowBlocks; a++) {
            if (t < segs_of(a)) return a;
            t -= segs_of(a);
        }
        return -1;
    }
    static constexpr int seg(int t) {
        for (int a = 0; a < kRowBlocks; a++) {
            if (t < segs_of(a)) return t;
            t -= segs_of(a);
        }
        return -1;
    }
};

// Shared-memory load that ptxas may not sink next to its use (asm volatile keeps the
// batch of loads together at the head of the group).
__device__ __forceinline__ double2 lds2(const double2* p) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}

__device__ __forceinline__ double2 cfma2(double2 acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
    return acc;
}

// One tile, generic in (A, S) so that every warp runs the same code (I-cache friendly):
// rows i = 32A + lane, columns j0 .. j0+CW-1 (j0 = CW*S).  Entry (i, j0+jj) sits at
// p + jj*st - jj(jj-1)/2 with p = &(i, j0) and st = B - j0 - 1, so each column costs one
// IMAD.  Loads are issued 8 columns ahead of their FMAs (asm volatile keeps them
// batched), and a diagonal tile zeroes its j > i terms by select (those reads land in
// the tail of column j-1, inside the array).
template <int B, int CW>
__device__ __forceinline__ void tile(int A, int S, const double2* __restrict__ sInv,
                                     const double2* __restrict__ sR, double2* __restrict__ sPart, int lane) {
    const int i = 32 * A + lane;
    const int j0 = CW * S;
    const double2* p = sInv + (j0 * B - (j0 * (j0 - 1)) / 2 - j0 + i);
    const double2* r = sR + j0;
    const int st = B - j0 - 1;
    const bool diag = j0 + CW - 1 > 32 * A;
    double2 acc[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0),
                      make_double2(0.0, 0.0)};
#pragma unroll
    for (int g = 0; g < CW; g += 8) {
        double2 m[8], rv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int jj = g + u;
            m[u] = lds2(p + (jj * st - (jj * (jj - 1)) / 2));
            rv[u] = lds2(r + jj);
        }
        if (diag) {
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const bool off = j0 + g + u > i;
                m[u].x = off ? 0.0 : m[u].x;
                m[u].y = off ? 0.0 : m[u].y;
            }
        }
#pragma unroll
        for (int u = 0; u < 8; u++) acc[u & 3] = cfma2(acc[u & 3], m[u], rv[u]);
    }
    sPart[S * B + i] = make_double2((acc[0].x + acc[1].x) + (acc[2].x + acc[3].x),
                                    (acc[0].y + acc[1].y) + (acc[2].y + acc[3].y));
}

// All tiles of the lower triangle, dealt round-robin to the warps w0 .. w0+NW-1 of the
// calling group (warp-uniform).  The caller synchronises, then sums with sum_row().
template <int B, int CW, int NW>
__device__ __forceinline__ void matvec_tiles(const double2* sInv, const double2* sR, double2* sPart, int warp,
                                             int lane) {
    using TL = Tiles<B, CW>;
    for (int t = warp; t < TL::kCount; t += NW) {
        int a = 0, s = t;
        while (s >= TL::segs_of(a)) {
            s -= TL::segs_of(a);
            a++;
        }
        tile<B, CW>(a, s, sInv, sR, sPart, lane);
    }
}

// x_i = sum over the segments that row i's tiles cover, in segment order.
template <int B, int CW>
__device__ __forceinline__ double2 sum_row(const double2* sPart, int i) {
    const int nseg = (32 * (i / 32) + 31) / CW + 1;
    double2 s = sPart[i];
    for (int q = 1; q < nseg; q++) s = make_double2(s.x + sPart[q * B + i].x, s.y + sPart[q * B + i].y);
    return s;
}

}  // namespace trimv
}  // namespace ssb
