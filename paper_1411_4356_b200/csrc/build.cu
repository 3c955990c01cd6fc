// build.cu -- device assembly of the trace-constrained Liouvillian L~ (Eq. (5)).
//
// PAPER.md:27-29 (Eq. 1), :52-56 (Eq. 3), :62 (column stacking), :67-70 (Eq. 5),
// :100 (a = a (x) I_b, b = I_a (x) b), :119 (w = mean of diag L).
//
// Row r = i + N j of L~ is the equation for rho_ij (N = N_c N_m, i = c N_m + m).
// Its entries follow from vec(A rho B) = (B^T (x) A) vec(rho):
//   -i H_ik        at column k + N j   (k a neighbour of i in H, k != i)
//   +i H_kj        at column i + N k   (k a neighbour of j in H, k != j)
//   r C_ik conj(C_jl) at column k + N l for C in {a, b, b^+} (one entry each)
//   diagonal       -i (H_ii - H_jj) + sum_C r (-1/2 (C^+C)_ii - 1/2 (C^+C)_jj)
// and row 0 additionally carries w at the columns k (N+1) of the diagonal elements.
// Every value is formed with the same IEEE operations, in the same order, as the
// formula reads (explicit __d*_rn intrinsics: no FMA contraction), e.g.
// (a^+a)_kk = sqrt(c)*sqrt(c) rounded, so the assembly is reproducible bit-for-bit.
// Exact zeros are not stored (canonical CSR).
#include <cub/cub.cuh>

#include "problem.h"

namespace ssb {

namespace {

struct Ent {
    int64_t col;
    double2 v;
};

constexpr int kMaxRow = 16;   // rows other than row 0 hold at most 13 entries

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// (C^+ C)_kk for the three channels; 0 where the sparse product has no entry.
__device__ __forceinline__ double num_sq(int q) {   // sqrt(q)*sqrt(q) rounded, q >= 1 else 0
    if (q < 1) return 0.0;
    double s = sqrt((double)q);
    return mul(s, s);
}

struct Dev {
    int Nc, Nm;
    int64_t N;
    double omega, Delta, kappa, g0, E, gam1, gam2;
};

// H_ii  = (-Delta) * (a^+a)_ii + omega * (b^+b)_ii
__device__ double H_diag(const Dev& d, int c, int m) {
    return add(mul(-d.Delta, num_sq(c)), mul(d.omega, num_sq(m)));
}

// neighbours of Hilbert index (c, m) in H with their (real) matrix elements
__device__ int H_nbrs(const Dev& d, int c, int m, int64_t* idx, double* val) {
    int k = 0;
    const int64_t i = (int64_t)c * d.Nm + m;
    // g0 (b + b^+) a^+a : (b+b^+)_{i,k} * (a^+a)_kk, same c, m +- 1
    if (c >= 1) {
        double na = num_sq(c);
        if (m >= 1) {   // k = m-1: (b^+)_{i,i-1} = sqrt(m)
            double v = mul(d.g0, mul(sqrt((double)m), na));
            if (v != 0.0) { idx[k] = i - 1; val[k] = v; k++; }
        }
        if (m + 1 < d.Nm) {   // k = m+1: b_{i,i+1} = sqrt(m+1)
            double v = mul(d.g0, mul(sqrt((double)(m + 1)), na));
            if (v != 0.0) { idx[k] = i + 1; val[k] = v; k++; }
        }
    }
    // E (a + a^+): c +- 1, same m
    if (c >= 1) {
        double v = mul(d.E, sqrt((double)c));
        if (v != 0.0) { idx[k] = i - d.Nm; val[k] = v; k++; }
    }
    if (c + 1 < d.Nc) {
        double v = mul(d.E, sqrt((double)(c + 1)));
        if (v != 0.0) { idx[k] = i + d.Nm; val[k] = v; k++; }
    }
    return k;
}

// Entries of row r of L (without the trace term). Returns count; unsorted.
__device__ int row_entries(const Dev& d, int64_t r, Ent* e) {
    const int64_t N = d.N;
    const int64_t i = r % N, j = r / N;
    const int ci = (int)(i / d.Nm), mi = (int)(i % d.Nm);
    const int cj = (int)(j / d.Nm), mj = (int)(j % d.Nm);
    int n = 0;
    int64_t nb[4];
    double nv[4];

    // diagonal: -1j * (H_ii - H_jj)  ->  (0, -(H_ii - H_jj)), then + r * d_C per channel
    double v = sub(H_diag(d, ci, mi), H_diag(d, cj, mj));
    double re = 0.0;
    {
        double da = sub(mul(-0.5, num_sq(ci)), mul(0.5, num_sq(cj)));
        double db = sub(mul(-0.5, num_sq(mi)), mul(0.5, num_sq(mj)));
        // (b b^+)_mm = sqrt(m+1)^2 for m < N_m - 1, absent for the top level
        double qi = (mi + 1 < d.Nm) ? num_sq(mi + 1) : 0.0;
        double qj = (mj + 1 < d.Nm) ? num_sq(mj + 1) : 0.0;
        double dd = sub(mul(-0.5, qi), mul(0.5, qj));
        if (d.kappa != 0.0) re = add(re, mul(d.kappa, da));
        if (d.gam1 != 0.0) re = add(re, mul(d.gam1, db));
        if (d.gam2 != 0.0) re = add(re, mul(d.gam2, dd));
    }
    double2 dv = make_double2(re, -v);
    if (dv.x != 0.0 || dv.y != 0.0) e[n++] = Ent{r, dv};

    // -i H_ik rho_kj  ->  (0, -H_ik) at k + N j
    int kn = H_nbrs(d, ci, mi, nb, nv);
    for (int t = 0; t < kn; t++) e[n++] = Ent{nb[t] + N * j, make_double2(0.0, -nv[t])};
    // +i rho_ik H_kj  ->  (0, +H_kj) at i + N k
    kn = H_nbrs(d, cj, mj, nb, nv);
    for (int t = 0; t < kn; t++) e[n++] = Ent{i + N * nb[t], make_double2(0.0, nv[t])};

    // r C rho C^+ : r * (conj(C)_jl * C_ik) at k + N l
    if (d.kappa != 0.0 && ci + 1 < d.Nc && cj + 1 < d.Nc) {
        double p = mul(sqrt((double)(cj + 1)), sqrt((double)(ci + 1)));
        double x = mul(d.kappa, p);
        if (x != 0.0) e[n++] = Ent{(i + d.Nm) + N * (j + d.Nm), make_double2(x, 0.0)};
    }
    if (d.gam1 != 0.0 && mi + 1 < d.Nm && mj + 1 < d.Nm) {
        double p = mul(sqrt((double)(mj + 1)), sqrt((double)(mi + 1)));
        double x = mul(d.gam1, p);
        if (x != 0.0) e[n++] = Ent{(i + 1) + N * (j + 1), make_double2(x, 0.0)};
    }
    if (d.gam2 != 0.0 && mi >= 1 && mj >= 1) {
        double p = mul(sqrt((double)mj), sqrt((double)mi));
        double x = mul(d.gam2, p);
        if (x != 0.0) e[n++] = Ent{(i - 1) + N * (j - 1), make_double2(x, 0.0)};
    }
    return n;
}

__device__ void sort_row(Ent* e, int n) {
    for (int a = 1; a < n; a++) {
        Ent t = e[a];
        int b = a - 1;
        while (b >= 0 && e[b].col > t.col) { e[b + 1] = e[b]; b--; }
        e[b + 1] = t;
    }
}

__global__ void k_count(Dev d, int64_t n, int64_t* counts, double2* diag) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        Ent e[kMaxRow];
        int k = row_entries(d, r, e);
        counts[r] = k;
        double2 dg = make_double2(0.0, 0.0);
        for (int t = 0; t < k; t++)
            if (e[t].col == r) dg = e[t].v;
        diag[r] = dg;
    }
}

__global__ void k_fill(Dev d, int64_t n, const int64_t* rowptr, int32_t* col, double2* val) {
    for (int64_t r = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        Ent e[kMaxRow];
        int k = row_entries(d, r, e);
        sort_row(e, k);
        int64_t o = rowptr[r];
        for (int t = 0; t < k; t++) {
            col[o + t] = (int32_t)e[t].col;
            val[o + t] = e[t].v;
        }
    }
}

__global__ void k_row0(Dev d, int64_t* cols, double2* vals, int* count) {
    Ent e[kMaxRow];
    int k = row_entries(d, 0, e);
    sort_row(e, k);
    for (int t = 0; t < k; t++) { cols[t] = e[t].col; vals[t] = e[t].v; }
    *count = k;
}

Dev make_dev(const ss_params& p) {
    Dev d;
    d.Nc = p.N_c;
    d.Nm = p.N_m;
    d.N = (int64_t)p.N_c * p.N_m;
    d.omega = p.omega_m;
    d.Delta = p.Delta;
    d.kappa = p.kappa;
    d.g0 = p.g0;
    d.E = p.E;
    // Gamma_m (1 + n_th) and Gamma_m n_th, rounded once each as in Eq. (3)
    volatile double one_plus = 1.0 + p.n_th;
    d.gam1 = p.Gamma_m * one_plus;
    d.gam2 = p.Gamma_m * p.n_th;
    return d;
}

}  // namespace

void build_liouvillian(Problem& P) {
    const ss_params& p = P.params;
    Dev d = make_dev(p);
    const int64_t N = d.N, n = N * N;
    SSB_CHECK(n < (int64_t)INT32_MAX, SS_ERR_ARG, "Liouvillian dimension must be < 2^31");
    P.N = N;
    P.n = n;
    cudaStream_t s = P.stream;

    int64_t* d_counts = nullptr;
    double2* d_diag = nullptr;
    SSB_CUDA(cudaMalloc(&d_counts, (n + 1) * sizeof(int64_t)));
    SSB_CUDA(cudaMalloc(&d_diag, n * sizeof(double2)));
    const int T = 256;
    k_count<<<grid_for(n, T), T, 0, s>>>(d, n, d_counts, d_diag);
    SSB_LAUNCHED();

    // w = (sum of diag(L), accumulated left to right) / n  -- reading R1
    std::vector<double2> diag(n);
    SSB_CUDA(cudaMemcpyAsync(diag.data(), d_diag, n * sizeof(double2), cudaMemcpyDeviceToHost, s));
    // row 0 of L (to merge with w T on the host)
    int64_t* d_r0c;
    double2* d_r0v;
    int* d_r0n;
    SSB_CUDA(cudaMalloc(&d_r0c, kMaxRow * sizeof(int64_t)));
    SSB_CUDA(cudaMalloc(&d_r0v, kMaxRow * sizeof(double2)));
    SSB_CUDA(cudaMalloc(&d_r0n, sizeof(int)));
    k_row0<<<1, 1, 0, s>>>(d, d_r0c, d_r0v, d_r0n);
    SSB_LAUNCHED();
    int64_t r0c[kMaxRow];
    double2 r0v[kMaxRow];
    int r0n = 0;
    SSB_CUDA(cudaMemcpyAsync(r0c, d_r0c, sizeof(r0c), cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaMemcpyAsync(r0v, d_r0v, sizeof(r0v), cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaMemcpyAsync(&r0n, d_r0n, sizeof(int), cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));

    double2 w;
    if (std::isnan(p.w)) {
        volatile double sr = 0.0, si = 0.0;
        for (int64_t t = 0; t < n; t++) { sr = sr + diag[t].x; si = si + diag[t].y; }
        w = make_double2(sr / (double)n, si / (double)n);
    } else {
        w = make_double2(p.w, 0.0);
    }
    P.w = w;

    // row 0 of L~ = row 0 of L + w * (ones at k (N+1)), exact zeros removed
    std::vector<int64_t> c0;
    std::vector<double2> v0;
    {
        int a = 0;
        for (int64_t k = 0; k <= N; k++) {   // k == N: flush remaining L entries
            int64_t tc = (k < N) ? k * (N + 1) : INT64_MAX;
            while (a < r0n && r0c[a] < tc) { c0.push_back(r0c[a]); v0.push_back(r0v[a]); a++; }
            if (k == N) break;
            double2 x = w;
            if (a < r0n && r0c[a] == tc) {
                volatile double xr = r0v[a].x + w.x, xi = r0v[a].y + w.y;
                x = make_double2(xr, xi);
                a++;
            }
            if (x.x != 0.0 || x.y != 0.0) { c0.push_back(tc); v0.push_back(x); }
        }
    }
    const int64_t n0 = (int64_t)c0.size();
    SSB_CUDA(cudaMemcpyAsync(d_counts, &n0, sizeof(int64_t), cudaMemcpyHostToDevice, s));

    // rowptr = exclusive scan of counts (counts[n] = 0 sentinel)
    int64_t zero = 0;
    SSB_CUDA(cudaMemcpyAsync(d_counts + n, &zero, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    P.nat.alloc_rowptr(n);
    size_t tmp_bytes = 0;
    SSB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_counts, P.nat.rowptr, n + 1, s));
    void* d_tmp = nullptr;
    SSB_CUDA(cudaMalloc(&d_tmp, tmp_bytes));
    SSB_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_counts, P.nat.rowptr, n + 1, s));
    SSB_LAUNCHED();
    int64_t nnz = 0;
    SSB_CUDA(cudaMemcpyAsync(&nnz, P.nat.rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    P.nat.alloc_entries(nnz);
    P.nnz = nnz;
    // row 0 from the host
    {
        std::vector<int32_t> c32(c0.begin(), c0.end());
        SSB_CUDA(cudaMemcpyAsync(P.nat.col, c32.data(), n0 * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaMemcpyAsync(P.nat.val, v0.data(), n0 * sizeof(double2), cudaMemcpyHostToDevice, s));
        k_fill<<<grid_for(n, T), T, 0, s>>>(d, n, P.nat.rowptr, P.nat.col, P.nat.val);
        SSB_LAUNCHED();
        SSB_CUDA(cudaStreamSynchronize(s));
    }
    cudaFree(d_tmp);
    cudaFree(d_counts);
    cudaFree(d_diag);
    cudaFree(d_r0c);
    cudaFree(d_r0v);
    cudaFree(d_r0n);
}

}  // namespace ssb
