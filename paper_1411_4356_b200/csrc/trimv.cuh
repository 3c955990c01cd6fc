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
    static constexpr int segs_of(int a) { return (32 * a + 31) / CW + 1; }
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

__device__ __forceinline__ double2 cfma2(double2 acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
    return acc;
}

// One tile: rows 32A + lane, columns CW*S .. CW*S + CW-1 (j <= i only).
template <int B, int CW, int A, int S>
__device__ __forceinline__ void tile(const double2* __restrict__ sInv, const double2* __restrict__ sR,
                                     double2* __restrict__ sPart, int lane) {
    const int i = 32 * A + lane;
    const double2* base = sInv + i;   // + cs(j) - j
    double2 acc[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0),
                      make_double2(0.0, 0.0)};
#pragma unroll
    for (int jj = 0; jj < CW; jj++) {
        const int j = CW * S + jj;
        const int off = j * B - (j * (j - 1)) / 2 - j;
        if (CW * S + CW - 1 <= 32 * A || j <= i) acc[jj & 3] = cfma2(acc[jj & 3], base[off], sR[j]);
    }
    const double2 s = make_double2((acc[0].x + acc[1].x) + (acc[2].x + acc[3].x),
                                   (acc[0].y + acc[1].y) + (acc[2].y + acc[3].y));
    sPart[S * B + i] = s;
}

template <int B, int CW, int T>
__device__ __forceinline__ void dispatch(int t, const double2* sInv, const double2* sR, double2* sPart, int lane) {
    using TL = Tiles<B, CW>;
    if constexpr (T < TL::kCount) {
        if (t == T) {
            tile<B, CW, TL::row_block(T), TL::seg(T)>(sInv, sR, sPart, lane);
            return;
        }
        dispatch<B, CW, T + 1>(t, sInv, sR, sPart, lane);
    }
}

// Whole CTA (NT threads): sPart[s*B + i] = sum over the tile (row block of i, segment s).
// The caller synchronises, then sums with sum_row().
template <int B, int NT, int CW>
__device__ __forceinline__ void matvec_tiles(const double2* sInv, const double2* sR, double2* sPart) {
    using TL = Tiles<B, CW>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
    for (int t = warp; t < TL::kCount; t += NW) dispatch<B, CW, 0>(t, sInv, sR, sPart, lane);
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
