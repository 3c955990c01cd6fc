// setup.cpp -- one-time setup of a built Liouvillian: RCM order, permuted L~_RCM,
// ILUT factors, substitution schedules and their device layout (timed separately from
// the GMRES hot path, as the north star asks).
//
// sec. III: RCM of L~ + L~^T applied as a symmetric permutation;
// sec. II: bandwidth B = ub + lb + 1 reported before / after;
// sec. II: ILUT(d, p).
#include <algorithm>
#include <chrono>
#include <cstring>

#include "problem.h"

namespace ssb {

namespace {

double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

int64_t bandwidth(const HostCSR& A) {
    int64_t ub = 0, lb = 0;
    for (int64_t i = 0; i < A.n; i++)
        for (int64_t q = A.rowptr[i]; q < A.rowptr[i + 1]; q++) {
            int64_t d = A.col[q] - i;
            ub = std::max(ub, d);
            lb = std::max(lb, -d);
        }
    return ub + lb + 1;
}

void download(const DevCSR& D, HostCSR& H, cudaStream_t s) {
    H.n = D.n;
    H.rowptr.resize(D.n + 1);
    std::vector<int32_t> c32(D.nnz);
    H.val.resize(D.nnz);
    SSB_CUDA(cudaMemcpyAsync(H.rowptr.data(), D.rowptr, (D.n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaMemcpyAsync(c32.data(), D.col, D.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaMemcpyAsync(H.val.data(), D.val, D.nnz * sizeof(double2), cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    H.col.assign(c32.begin(), c32.end());
}

void upload(const HostCSR& H, DevCSR& D, cudaStream_t s) {
    D.release();
    D.alloc_rowptr(H.n);
    D.alloc_entries(H.nnz());
    std::vector<int32_t> c32(H.col.begin(), H.col.end());
    SSB_CUDA(cudaMemcpyAsync(D.rowptr, H.rowptr.data(), (H.n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(D.col, c32.data(), c32.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(D.val, H.val.data(), H.val.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaStreamSynchronize(s));
}

// A_new[k][*] = A[perm[k]][perm^{-1}(*)], columns re-sorted
HostCSR permute(const HostCSR& A, const std::vector<int64_t>& perm) {
    const int64_t n = A.n;
    std::vector<int64_t> iperm(n);
    for (int64_t k = 0; k < n; k++) iperm[perm[k]] = k;
    HostCSR B;
    B.n = n;
    B.rowptr.assign(n + 1, 0);
    for (int64_t k = 0; k < n; k++) B.rowptr[k + 1] = B.rowptr[k] + (A.rowptr[perm[k] + 1] - A.rowptr[perm[k]]);
    B.col.resize(A.nnz());
    B.val.resize(A.nnz());
    std::vector<std::pair<int64_t, double2>> tmp;
    for (int64_t k = 0; k < n; k++) {
        const int64_t o = perm[k];
        tmp.clear();
        for (int64_t q = A.rowptr[o]; q < A.rowptr[o + 1]; q++) tmp.emplace_back(iperm[A.col[q]], A.val[q]);
        std::sort(tmp.begin(), tmp.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        int64_t p = B.rowptr[k];
        for (auto& e : tmp) {
            B.col[p] = e.first;
            B.val[p] = e.second;
            p++;
        }
    }
    return B;
}

// Level schedule of a triangular dependency graph given as strict rows.
// lower: level(i) = 1 + max level(j), j < i in row i; upper: processed from the bottom.
void levels(const std::vector<int64_t>& rp, const std::vector<int64_t>& col, int64_t n, bool upper,
            int64_t skip_first, std::vector<int64_t>& lev_ptr, std::vector<int32_t>& lev_rows) {
    std::vector<int32_t> lev(n, 0);
    int32_t maxl = 0;
    auto row = [&](int64_t i) {
        int32_t l = 0;
        for (int64_t q = rp[i] + skip_first; q < rp[i + 1]; q++) l = std::max(l, lev[col[q]] + 1);
        lev[i] = l;
        maxl = std::max(maxl, l);
    };
    if (!upper)
        for (int64_t i = 0; i < n; i++) row(i);
    else
        for (int64_t i = n - 1; i >= 0; i--) row(i);
    lev_ptr.assign((size_t)maxl + 2, 0);
    for (int64_t i = 0; i < n; i++) lev_ptr[lev[i] + 1]++;
    for (int32_t l = 0; l <= maxl; l++) lev_ptr[l + 1] += lev_ptr[l];
    lev_rows.resize(n);
    std::vector<int64_t> pos(lev_ptr.begin(), lev_ptr.end() - 1);
    if (!upper)
        for (int64_t i = 0; i < n; i++) lev_rows[pos[lev[i]]++] = (int32_t)i;
    else
        for (int64_t i = n - 1; i >= 0; i--) lev_rows[pos[lev[i]]++] = (int32_t)i;
}

void upload_tri(const HostCSR& F, bool upper, DevTri& T, cudaStream_t s) {
    T.release();
    const int64_t n = F.n;
    T.n = n;
    // strict part (U: drop the leading diagonal entry of each row)
    std::vector<int64_t> rp(n + 1, 0);
    std::vector<int32_t> c32;
    std::vector<double2> v;
    std::vector<double2> invd;
    c32.reserve(F.nnz());
    v.reserve(F.nnz());
    if (upper) invd.resize(n);
    for (int64_t i = 0; i < n; i++) {
        int64_t q0 = F.rowptr[i];
        if (upper) {
            const double2 u = F.val[q0];
            const double d = u.x * u.x + u.y * u.y;
            invd[i] = make_double2(u.x / d, -u.y / d);
            q0++;
        }
        for (int64_t q = q0; q < F.rowptr[i + 1]; q++) {
            c32.push_back((int32_t)F.col[q]);
            v.push_back(F.val[q]);
        }
        rp[i + 1] = (int64_t)c32.size();
    }
    T.nnz = (int64_t)c32.size();
    std::vector<int64_t> lev_ptr;
    std::vector<int32_t> lev_rows;
    levels(F.rowptr, F.col, n, upper, upper ? 1 : 0, lev_ptr, lev_rows);
    T.nlev = (int64_t)lev_ptr.size() - 1;
    SSB_CUDA(cudaMalloc(&T.rowptr, (n + 1) * sizeof(int64_t)));
    SSB_CUDA(cudaMalloc(&T.col, std::max<int64_t>(1, T.nnz) * sizeof(int32_t)));
    SSB_CUDA(cudaMalloc(&T.val, std::max<int64_t>(1, T.nnz) * sizeof(double2)));
    SSB_CUDA(cudaMalloc(&T.lev_ptr, lev_ptr.size() * sizeof(int64_t)));
    SSB_CUDA(cudaMalloc(&T.lev_rows, n * sizeof(int32_t)));
    SSB_CUDA(cudaMemcpyAsync(T.rowptr, rp.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    if (T.nnz) {
        SSB_CUDA(cudaMemcpyAsync(T.col, c32.data(), T.nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaMemcpyAsync(T.val, v.data(), T.nnz * sizeof(double2), cudaMemcpyHostToDevice, s));
    }
    SSB_CUDA(cudaMemcpyAsync(T.lev_ptr, lev_ptr.data(), lev_ptr.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(T.lev_rows, lev_rows.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    if (upper) {
        SSB_CUDA(cudaMalloc(&T.inv_diag, n * sizeof(double2)));
        SSB_CUDA(cudaMemcpyAsync(T.inv_diag, invd.data(), n * sizeof(double2), cudaMemcpyHostToDevice, s));
    }
    SSB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

void setup_problem(Problem& P, double drop_tol, double fill_factor, int threads, ss_setup_info* info) {
    cudaStream_t s = P.stream;
    P.have_setup = false;
    const double t0 = now_ms();
    HostCSR nat;
    download(P.nat, nat, s);
    P.bw_nat = bandwidth(nat);
    P.perm = rcm_order(nat.n, nat.rowptr, nat.col);
    HostCSR A = permute(nat, P.perm);
    P.bw_rcm = bandwidth(A);
    const double t1 = now_ms();
    IlutStats st;
    ilut_factor(A, drop_tol, fill_factor, threads, P.hL, P.hU, st);
    const double t2 = now_ms();
    upload(A, P.A, s);
    if (!P.d_perm) SSB_CUDA(cudaMalloc(&P.d_perm, P.n * sizeof(int64_t)));
    SSB_CUDA(cudaMemcpyAsync(P.d_perm, P.perm.data(), P.n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    upload_tri(P.hL, false, P.L, s);
    upload_tri(P.hU, true, P.U, s);
    const double t3 = now_ms();
    P.have_setup = true;
    P.have_solution = false;
    if (info) {
        info->nnz_L = P.hL.nnz();
        info->nnz_U = P.hU.nnz();
        info->fill = (double)(P.hL.nnz() + P.hU.nnz()) / (double)P.nnz;
        info->bandwidth_nat = P.bw_nat;
        info->bandwidth_rcm = P.bw_rcm;
        info->levels_L = P.L.nlev;
        info->levels_U = P.U.nlev;
        info->pivots_repaired = st.repaired;
        info->threads = st.threads;
        info->rcm_ms = t1 - t0;
        info->ilut_ms = t2 - t1;
        info->upload_ms = t3 - t2;
    }
}

}  // namespace ssb
