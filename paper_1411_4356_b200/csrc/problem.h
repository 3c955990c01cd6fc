// problem.h -- the handle behind ss_problem* and the internal interfaces.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/ss_b200.h"
#include "common.cuh"

namespace ssb {

// Device CSR matrix: int64 row pointers, int32 columns, complex128 values.
struct DevCSR {
    int64_t n = 0, nnz = 0;
    int64_t* rowptr = nullptr;
    int32_t* col = nullptr;
    double2* val = nullptr;
    void alloc_rowptr(int64_t n_) {
        n = n_;
        SSB_CUDA(cudaMalloc(&rowptr, (n + 1) * sizeof(int64_t)));
    }
    void alloc_entries(int64_t nnz_) {
        nnz = nnz_;
        SSB_CUDA(cudaMalloc(&col, (nnz > 0 ? nnz : 1) * sizeof(int32_t)));
        SSB_CUDA(cudaMalloc(&val, (nnz > 0 ? nnz : 1) * sizeof(double2)));
    }
    // SELL-32 copy for the SpMV (spmv.cu), built at setup: slice s = rows 32s .. 32s+31,
    // entries column-major within the slice (entry e of row 32s+r at sptr[s] + 32e + r),
    // width = the longest row of the slice; padding col 0 / value 0.  Rows longer than
    // kSellLong entries (the trace row) are left out (first col = -1) and summed from
    // the CSR by one warp each (lrows).
    int64_t nslices = 0, nlong = 0, sell_entries = 0;
    int64_t* sptr = nullptr;
    int32_t* scol = nullptr;
    double2* sval = nullptr;
    int64_t* lrows = nullptr;
    void release() {
        cudaFree(rowptr);
        cudaFree(col);
        cudaFree(val);
        cudaFree(sptr);
        cudaFree(scol);
        cudaFree(sval);
        cudaFree(lrows);
        rowptr = nullptr;
        col = nullptr;
        val = nullptr;
        sptr = nullptr;
        scol = nullptr;
        sval = nullptr;
        lrows = nullptr;
        n = nnz = nslices = nlong = sell_entries = 0;
    }
};
constexpr int kSellLong = 64;

// std::vector whose resize() leaves trivial elements uninitialised: the setup fills its
// large arrays in parallel (first touch) instead of zeroing GBs on one thread first.
template <class T>
struct DefaultInitAlloc : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = DefaultInitAlloc<U>;
    };
    DefaultInitAlloc() = default;
    template <class U>
    DefaultInitAlloc(const DefaultInitAlloc<U>&) noexcept {}
    template <class U>
    void construct(U* p) noexcept(std::is_nothrow_default_constructible<U>::value) {
        ::new ((void*)p) U;
    }
    template <class U, class... Args>
    void construct(U* p, Args&&... args) {
        ::new ((void*)p) U(std::forward<Args>(args)...);
    }
};
template <class T>
using hvec = std::vector<T, DefaultInitAlloc<T>>;

// Host CSR (int64 everywhere) used during setup.
struct HostCSR {
    int64_t n = 0;
    std::vector<int64_t> rowptr;
    hvec<int64_t> col;
    hvec<double2> val;
    int64_t nnz() const { return (int64_t)col.size(); }
};

// Triangular factor on the device in the block layout of trsv.cu (kernel index space:
// L as is, U reversed i' = n-1-i so that both are lower triangular; blocks of B rows).
// Source-distance split of the entries left of block k (d = k - source block):
//   d = 1 .. kDense  -> dense G_d = D_k^{-1} T_{k,k-d} (the chain teams)
//   kDense < d < Q_k -> list B, staged per lieutenant CTA and block
//   d >= Q_k         -> far part (helper CTAs)
#ifndef SSB_KDENSE
#define SSB_KDENSE 2   // (build-time experiment knob: 3 moves d = 3 from the lieutenants to the chain teams)
#endif
constexpr int kDense = SSB_KDENSE;
#ifndef SSB_LTCAP
#define SSB_LTCAP 1024   // list-B entries per lieutenant and block (the lieutenants' shared-memory stage)
#endif
constexpr int near_cap_b(int B) { return B > 0 ? SSB_LTCAP : SSB_LTCAP; }   // per lieutenant and block
constexpr int kLieutenants = 7;   // list B CTAs of a chain cluster (trsv.cu; cluster = 1 + 7)
constexpr int lt_rows(int B) { return (B + kLieutenants - 1) / kLieutenants; }   // rows per lieutenant
constexpr int near_nloc(int B) { return 2 * (B + 4); }   // per list: row starts | late-part starts

// one near list on the device (see setup.cpp::build_block_tri)
struct NearDev {
    int64_t* bp = nullptr;    // [nblk+1] start of block k's list (multiple of 4 entries)
    int32_t* col = nullptr;   // kernel-space columns, rows in order
    double2* val = nullptr;
    int32_t* loc = nullptr;   // [list][2(B+4)] row starts, then starts of each row's d = kDense+1
                              // entries (the late part), relative to bp[list]
    void release() {
        cudaFree(bp);
        cudaFree(col);
        cudaFree(val);
        cudaFree(loc);
        *this = NearDev();
    }
};

struct TriArgs {
    int64_t n, nblk;
    int32_t rev, B;
    const int64_t* farptr;    // [n+1] entries of row i' with source block <= k-Q_k (k = i'/B)
    const int32_t* fcol;      //       kernel-space columns, ascending within a row
    const double2* fval;
    const int64_t* itemptr;   // [nblk+1] far work items of block k: items[itemptr[k] .. itemptr[k+1])
    const uint32_t* items;    //          item = (c << 5) | r: entries 32c .. 32c+31 of row r of the
                              //          block's far part, sorted by newest source block (setup.cpp)
    const int64_t* nbpB;      // near list B: [nblk*kLieutenants+1], list of (block k, lieutenant l) at k*kLt+l
    const int32_t* ncolB;
    const double2* nvalB;
    const int32_t* nlocB;
    const double2* dinv;      // [nblk][B(B+1)/2] inverse diagonal blocks, packed lower, column-major
    const double2* G;         // [nblk][kDense][B*B] D_k^{-1} T_{k,k-d}, d = 1 .. kDense, column-major
    double2* yfar;            // [nblk*B] y_k = D_k^{-1} (b_k - far part), written by the helper CTAs
    const int64_t* operm;     // [n] output permutation out[operm[i]] = x[i] (ILUTP columns), or null
    uint32_t* fflag;          // [nblk] "yfar of block k is ready" (value = launch epoch)
    unsigned long long* xfront;   // (epoch << 32) | number of blocks of x published
};

struct DevBlockTri {
    int64_t n = 0, nblk = 0, nnz_far = 0, nnz_near = 0, nnz_strict = 0;
    int B = 0, rev = 0, nt = 0, Q = 0;   // rows per block, reversed (U), threads, smallest Q_k
    int64_t* farptr = nullptr;
    int32_t* fcol = nullptr;
    double2* fval = nullptr;
    int64_t* itemptr = nullptr;
    uint32_t* items = nullptr;
    NearDev nearB;
    double2* dinv = nullptr;
    double2* G = nullptr;
    double2* yfar = nullptr;
    uint32_t* fflag = nullptr;
    unsigned long long* xfront = nullptr;
    int64_t* operm = nullptr;   // U of ILUTP: out[operm[p]] = x[p] (column permutation), else null
    double2* xwork = nullptr;   // position-space x when operm is set
    uint32_t epoch = 0;
    int grid = 0;         // persistent grid on the whole GPU (all co-resident clusters, <= blocks)
    int sm_budget = 0;    // ss_set_sm_budget: at most this many CTAs (whole clusters), 0 = grid
    int64_t nlev = 0;   // row-level dependency levels (diagnostic)
    TriArgs args() const {
        return TriArgs{n,        nblk,      rev,       B,         farptr, fcol, fval,  itemptr, items, nearB.bp,
                       nearB.col, nearB.val, nearB.loc, dinv,      G,      yfar, operm, fflag,   xfront};
    }
    void release() {
        cudaFree(farptr);
        cudaFree(fcol);
        cudaFree(fval);
        cudaFree(itemptr);
        cudaFree(items);
        nearB.release();
        cudaFree(dinv);
        cudaFree(G);
        cudaFree(yfar);
        cudaFree(fflag);
        cudaFree(xfront);
        cudaFree(operm);
        cudaFree(xwork);
        *this = DevBlockTri();
    }
};

// GMRES(m) workspace.
struct Krylov {
    int m = 0;
    int64_t n = 0;
    double2* V = nullptr;      // (m+1) x n basis, row k = v_k
    double2* w = nullptr;      // work vectors
    double2* t = nullptr;
    double2* x = nullptr;      // iterate (RCM order)
    double2* b = nullptr;      // right-hand side (RCM order)
    double2* r = nullptr;
    double2* part = nullptr;   // block partial sums
    int part_cap = 0;
    double2* hcol = nullptr;   // device Hessenberg column accumulators (2 x (m+2))
    double* scal = nullptr;    // device scalars
    double* h_stat = nullptr;  // pinned host mirror of scalars (two 4-double slots: steps j, j+1)
    cudaEvent_t st_ev[2] = {nullptr, nullptr};   // the status copy of step j landed (slot j & 1)
    void release() {
        cudaFree(V);
        cudaFree(w);
        cudaFree(t);
        cudaFree(x);
        cudaFree(b);
        cudaFree(r);
        cudaFree(part);
        cudaFree(hcol);
        cudaFree(scal);
        if (h_stat) cudaFreeHost(h_stat);
        for (auto& e : st_ev)
            if (e) cudaEventDestroy(e);
        *this = Krylov();
    }
};

struct Problem {
    ss_params params{};
    cudaStream_t stream = nullptr;
    int device = 0;
    int64_t N = 0, n = 0, nnz = 0;
    double2 w{0.0, 0.0};

    DevCSR nat;                 // L~ natural order
    DevCSR A;                   // A' = Pi^T L~_RCM: L~_RCM with its rows in iLUTP pivot order (R16)
    std::vector<int64_t> perm;  // new -> old (RCM; the columns of A', the index of x)
    std::vector<int64_t> rowperm;   // row j of A' is row rowperm[j] of L~ (natural index)
    int64_t rhs_pos = -1;       // the row of A' holding w of b = (w, 0, ...)
    int64_t* d_perm = nullptr;
    int64_t* d_rowperm = nullptr;
    bool have_setup = false;

    HostCSR hL, hU;             // iLUTP of L~_RCM^T (export / tests): L~_RCM^T[:, colperm] ~ hL hU
    std::vector<int64_t> colperm;   // its column permutation = the row order of A'
    int sm_budget = 0;          // ss_set_sm_budget (copied into L, U)
    DevBlockTri L, U;           // the substitutions: L <- U'^T (lower, pivots), U <- L'^T (unit upper)
    int64_t bw_nat = 0, bw_rcm = 0;

    Krylov K;
    double2* rho = nullptr;     // normalised solution, natural order (vec(rho))
    bool have_solution = false;

    cudaEvent_t ev0 = nullptr, ev1 = nullptr;

    void release();
};

// build.cu
void build_liouvillian(Problem& P);
// setup.cpp
void setup_problem(Problem& P, double drop_tol, double fill_factor, double permtol, int threads,
                   ss_setup_info* info);
// rcm.cpp
std::vector<int64_t> rcm_order(int64_t n, const std::vector<int64_t>& rowptr, const hvec<int64_t>& col);
// ilut.cpp
struct IlutStats {
    int32_t repaired = 0;
    int32_t swaps = 0;
    int32_t threads = 1;
};
// ILUTP: A[:, colperm] ~ L U (L strict lower, unit diagonal implicit; U diagonal first)
void ilut_factor(const HostCSR& A, double drop_tol, double fill_factor, double permtol, int threads, HostCSR& L,
                 HostCSR& U, std::vector<int64_t>& colperm, IlutStats& st);
// spmv.cu
void spmv(const DevCSR& A, const double2* x, double2* y, cudaStream_t s);
// setup.cpp: the SELL-32 copy of a host CSR into D (D's CSR already uploaded)
void build_sell(const HostCSR& H, DevCSR& D, cudaStream_t s);
// trsv.cu: x = T^{-1} b for one factor (b, x in natural index order; x must not alias b)
// trace (optional, device, SS_TRACE_STAMPS x nblk %globaltimer stamps per block; the
// meaning of each stamp is listed at ss_debug_trace_trsv in include/ss_b200.h).
void block_trsv(DevBlockTri& T, const double2* b, double2* x, cudaStream_t s,
                unsigned long long* trace = nullptr);
size_t block_trsv_packed(int B);
void block_trsv_prepare(DevBlockTri& T);
void poison_shared_memory(cudaStream_t s);   // ss_debug_poison_smem (trsv.cu)   // launch geometry (persistent grid)
// krylov.cu / gmres.cu
void gmres_solve(Problem& P, const double2* b_dev, int restart, double tol, int max_iter,
                 ss_solve_info* info);
void finish_solution(Problem& P, ss_solve_info* info);
void expectations(Problem& P, double* na, double* nb);
void gather_perm(const double2* src, const int64_t* perm, int64_t n, double2* dst, cudaStream_t s);   // dst[k] = src[perm[k]]
void scatter_perm(const double2* src, const int64_t* perm, int64_t n, double2* dst, cudaStream_t s);  // dst[perm[k]] = src[k]
void ensure_krylov(Problem& P, int m);

}  // namespace ssb
