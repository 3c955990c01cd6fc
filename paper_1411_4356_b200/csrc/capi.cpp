// capi.cpp -- the extern "C" boundary declared in include/ss_b200.h.
//
// Argument marshalling, error translation and handle lifetime only; every step of the
// method runs in build.cu / setup.cpp / spmv.cu / trsv.cu / krylov.cu / solution.cu.
#include <cstring>
#include <mutex>
#include <string>

#include "problem.h"

namespace ssb {

namespace {
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
std::atomic<int64_t>& launch_counter() { return g_launches; }

void Problem::release() {
    nat.release();
    A.release();
    L.release();
    U.release();
    K.release();
    cudaFree(d_perm);
    cudaFree(d_rowperm);
    cudaFree(rho);
    d_perm = nullptr;
    d_rowperm = nullptr;
    rho = nullptr;
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    ev0 = ev1 = nullptr;
}

void gmres_solve(Problem& P, const double2* b_dev, int restart, double tol, int max_iter, ss_solve_info* info);
void ensure_krylov(Problem& P, int m);

}  // namespace ssb

using namespace ssb;

#define SS_GUARD_BEGIN try {
#define SS_GUARD_END                                         \
    }                                                        \
    catch (const ssb::Error& e) {                            \
        ssb::set_error(e.msg);                               \
        return e.code;                                       \
    }                                                        \
    catch (const std::bad_alloc&) {                          \
        ssb::set_error("host allocation failed");            \
        return SS_ERR_OOM;                                   \
    }                                                        \
    catch (const std::exception& e) {                        \
        ssb::set_error(e.what());                            \
        return SS_ERR_ARG;                                   \
    }                                                        \
    return SS_OK;

struct ss_problem {
    ssb::Problem P;
};

extern "C" {

const char* ss_last_error(void) { return g_last_error.c_str(); }

int64_t ss_kernel_launches(void) { return g_launches.load(); }

int ss_build(const ss_params* p, void* cuda_stream, ss_problem** out, ss_build_info* info) {
    SS_GUARD_BEGIN
    SSB_CHECK(p && out, SS_ERR_ARG, "ss_build: NULL argument");
    SSB_CHECK(p->N_c >= 1 && p->N_m >= 1, SS_ERR_ARG, "ss_build: cut-offs must be >= 1");
    SSB_CHECK(p->kappa >= 0 && p->Gamma_m >= 0 && p->n_th >= 0, SS_ERR_ARG, "ss_build: negative rate");
    int ndev = 0;
    cudaError_t ce = cudaGetDeviceCount(&ndev);
    SSB_CHECK(ce == cudaSuccess && ndev > 0, SS_ERR_CUDA,
              std::string("ss_build: no CUDA device (") + cudaGetErrorString(ce) + "); there is no CPU fallback");
    ss_problem* h = new ss_problem();
    try {
        h->P.params = *p;
        h->P.stream = (cudaStream_t)cuda_stream;
        SSB_CUDA(cudaGetDevice(&h->P.device));
        SSB_CUDA(cudaEventCreate(&h->P.ev0));
        SSB_CUDA(cudaEventCreate(&h->P.ev1));
        SSB_CUDA(cudaEventRecord(h->P.ev0, h->P.stream));
        build_liouvillian(h->P);
        SSB_CUDA(cudaEventRecord(h->P.ev1, h->P.stream));
        SSB_CUDA(cudaEventSynchronize(h->P.ev1));
    } catch (...) {
        h->P.release();
        delete h;
        throw;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->P.ev0, h->P.ev1);
    if (info) {
        info->hilbert_dim = h->P.N;
        info->n = h->P.n;
        info->nnz = h->P.nnz;
        info->w_re = h->P.w.x;
        info->w_im = h->P.w.y;
        info->build_ms = ms;
    }
    *out = h;
    SS_GUARD_END
}

int ss_setup(ss_problem* h, double drop_tol, double fill_factor, double permtol, int32_t n_threads,
             ss_setup_info* info) {
    SS_GUARD_BEGIN
    SSB_CHECK(h, SS_ERR_ARG, "ss_setup: NULL handle");
    setup_problem(h->P, drop_tol, fill_factor, permtol, n_threads, info);
    SS_GUARD_END
}

int ss_solve(ss_problem* h, int32_t restart, double tol, int32_t max_iter, ss_solve_info* info) {
    SS_GUARD_BEGIN
    SSB_CHECK(h, SS_ERR_ARG, "ss_solve: NULL handle");
    Problem& P = h->P;
    SSB_CHECK(P.have_setup, SS_ERR_STATE, "ss_solve before ss_setup");
    ensure_krylov(P, restart);
    // b' = b in the row order of A' (b = (w, 0, ..., 0): w in row rhs_pos, found at setup)
    SSB_CUDA(cudaMemsetAsync(P.K.b, 0, P.n * sizeof(double2), P.stream));
    SSB_CUDA(cudaMemcpyAsync(P.K.b + P.rhs_pos, &P.w, sizeof(double2), cudaMemcpyHostToDevice, P.stream));
    ss_solve_info loc{};
    gmres_solve(P, P.K.b, restart, tol, max_iter, &loc);
    finish_solution(P, &loc);
    if (info) *info = loc;
    SS_GUARD_END
}

int ss_solve_host(ss_problem* h, const double* rhs_host, double* x_host, int32_t restart, double tol,
                  int32_t max_iter, ss_solve_info* info) {
    SS_GUARD_BEGIN
    SSB_CHECK(h && x_host, SS_ERR_ARG, "ss_solve_host: NULL argument");
    Problem& P = h->P;
    SSB_CHECK(P.have_setup, SS_ERR_STATE, "ss_solve_host before ss_setup");
    ensure_krylov(P, restart);
    const int64_t n = P.n;
    cudaStream_t s = P.stream;
    // natural-order rhs -> device (scratch K.r) -> the row order of A' into K.b
    if (rhs_host) {
        SSB_CUDA(cudaMemcpyAsync(P.K.r, rhs_host, n * sizeof(double2), cudaMemcpyHostToDevice, s));
    } else {
        SSB_CUDA(cudaMemsetAsync(P.K.r, 0, n * sizeof(double2), s));
        SSB_CUDA(cudaMemcpyAsync(P.K.r, &P.w, sizeof(double2), cudaMemcpyHostToDevice, s));
    }
    gather_perm(P.K.r, P.d_rowperm, n, P.K.b, s);
    ss_solve_info loc{};
    gmres_solve(P, P.K.b, restart, tol, max_iter, &loc);
    finish_solution(P, &loc);   // also scatters x to natural order (in rho, then normalised)
    scatter_perm(P.K.x, P.d_perm, n, P.K.r, s);
    SSB_CUDA(cudaMemcpyAsync(x_host, P.K.r, n * sizeof(double2), cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    if (info) *info = loc;
    SS_GUARD_END
}

int ss_debug_poison_smem(ss_problem* h) {
    SS_GUARD_BEGIN
    SSB_CHECK(h, SS_ERR_ARG, "ss_debug_poison_smem: NULL handle");
    SSB_CUDA(cudaSetDevice(h->P.device));
    poison_shared_memory(h->P.stream);
    SS_GUARD_END
}

int ss_set_sm_budget(ss_problem* h, int32_t sms) {
    SS_GUARD_BEGIN
    SSB_CHECK(h && sms >= 0, SS_ERR_ARG, "ss_set_sm_budget: NULL handle or negative budget");
    h->P.sm_budget = sms;
    h->P.L.sm_budget = h->P.U.sm_budget = sms;
    SS_GUARD_END
}

int ss_expect(ss_problem* h, double* n_cavity, double* n_mech) {
    SS_GUARD_BEGIN
    SSB_CHECK(h && n_cavity && n_mech, SS_ERR_ARG, "ss_expect: NULL argument");
    expectations(h->P, n_cavity, n_mech);
    SS_GUARD_END
}

int ss_get_rho(ss_problem* h, void* dst, int32_t dst_is_device) {
    SS_GUARD_BEGIN
    SSB_CHECK(h && dst, SS_ERR_ARG, "ss_get_rho: NULL argument");
    SSB_CHECK(h->P.have_solution, SS_ERR_STATE, "ss_get_rho before ss_solve");
    SSB_CUDA(cudaMemcpyAsync(dst, h->P.rho, h->P.n * sizeof(double2),
                             dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->P.stream));
    SSB_CUDA(cudaStreamSynchronize(h->P.stream));
    SS_GUARD_END
}

void ss_destroy(ss_problem* h) {
    if (!h) return;
    h->P.release();
    delete h;
}

int ss_sizes(const ss_problem* h, int64_t* n, int64_t* nnz, int64_t* nnz_L, int64_t* nnz_U) {
    SS_GUARD_BEGIN
    SSB_CHECK(h, SS_ERR_ARG, "ss_sizes: NULL handle");
    if (n) *n = h->P.n;
    if (nnz) *nnz = h->P.nnz;
    if (nnz_L) *nnz_L = h->P.have_setup ? h->P.hL.nnz() : -1;
    if (nnz_U) *nnz_U = h->P.have_setup ? h->P.hU.nnz() : -1;
    SS_GUARD_END
}

int ss_export_matrix(const ss_problem* h, int32_t which, int64_t* rowptr, int64_t* colidx, double* vals) {
    SS_GUARD_BEGIN
    SSB_CHECK(h && rowptr && colidx && vals, SS_ERR_ARG, "ss_export_matrix: NULL argument");
    SSB_CHECK(which == 0 || which == 1, SS_ERR_ARG, "ss_export_matrix: which must be 0 or 1");
    const Problem& P = h->P;
    SSB_CHECK(which == 0 || P.have_setup, SS_ERR_STATE, "ss_export_matrix(1) before ss_setup");
    const DevCSR& D = which == 0 ? P.nat : P.A;
    std::vector<int32_t> c32(D.nnz);
    SSB_CUDA(cudaMemcpyAsync(rowptr, D.rowptr, (D.n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, P.stream));
    SSB_CUDA(cudaMemcpyAsync(c32.data(), D.col, D.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, P.stream));
    SSB_CUDA(cudaMemcpyAsync(vals, D.val, D.nnz * sizeof(double2), cudaMemcpyDeviceToHost, P.stream));
    SSB_CUDA(cudaStreamSynchronize(P.stream));
    for (int64_t q = 0; q < D.nnz; q++) colidx[q] = c32[q];
    SS_GUARD_END
}

int ss_export_perm(const ss_problem* h, int64_t* perm) {
    SS_GUARD_BEGIN
    SSB_CHECK(h && perm, SS_ERR_ARG, "ss_export_perm: NULL argument");
    SSB_CHECK(h->P.have_setup, SS_ERR_STATE, "ss_export_perm before ss_setup");
    std::memcpy(perm, h->P.perm.data(), h->P.n * sizeof(int64_t));
    SS_GUARD_END
}

int ss_export_colperm(const ss_problem* h, int64_t* colperm) {
    SS_GUARD_BEGIN
    SSB_CHECK(h && colperm, SS_ERR_ARG, "ss_export_colperm: NULL argument");
    SSB_CHECK(h->P.have_setup, SS_ERR_STATE, "ss_export_colperm before ss_setup");
    std::memcpy(colperm, h->P.colperm.data(), h->P.n * sizeof(int64_t));
    SS_GUARD_END
}

int ss_export_factors(const ss_problem* h, int32_t which, int64_t* rowptr, int64_t* colidx, double* vals) {
    SS_GUARD_BEGIN
    SSB_CHECK(h && rowptr && colidx && vals, SS_ERR_ARG, "ss_export_factors: NULL argument");
    SSB_CHECK(which == 0 || which == 1, SS_ERR_ARG, "ss_export_factors: which must be 0 or 1");
    SSB_CHECK(h->P.have_setup, SS_ERR_STATE, "ss_export_factors before ss_setup");
    const HostCSR& F = which == 0 ? h->P.hL : h->P.hU;
    std::memcpy(rowptr, F.rowptr.data(), (F.n + 1) * sizeof(int64_t));
    std::memcpy(colidx, F.col.data(), F.nnz() * sizeof(int64_t));
    std::memcpy(vals, F.val.data(), F.nnz() * sizeof(double2));
    SS_GUARD_END
}

int ss_ilutp_host(int64_t n, const int64_t* rowptr, const int64_t* colidx, const double* vals, double drop_tol,
                  double fill_factor, double permtol, int32_t n_threads, int64_t* L_rowptr, int64_t* L_colidx,
                  double* L_vals, int64_t L_cap, int64_t* U_rowptr, int64_t* U_colidx, double* U_vals,
                  int64_t U_cap, int64_t* colperm) {
    SS_GUARD_BEGIN
    SSB_CHECK(n > 0 && rowptr && colidx && vals && L_rowptr && L_colidx && L_vals && U_rowptr && U_colidx &&
                  U_vals && colperm && L_cap >= 0 && U_cap >= 0,
              SS_ERR_ARG, "ss_ilutp_host: NULL or negative argument");
    SSB_CHECK(rowptr[0] == 0, SS_ERR_ARG, "ss_ilutp_host: rowptr[0] must be 0");
    HostCSR A;
    A.n = n;
    A.rowptr.assign(rowptr, rowptr + n + 1);
    std::vector<int64_t> mark(n, -1);
    for (int64_t i = 0; i < n; i++) {
        SSB_CHECK(rowptr[i + 1] >= rowptr[i], SS_ERR_ARG, "ss_ilutp_host: rowptr must be non-decreasing");
        for (int64_t q = rowptr[i]; q < rowptr[i + 1]; q++) {
            const int64_t c = colidx[q];
            SSB_CHECK(c >= 0 && c < n, SS_ERR_ARG, "ss_ilutp_host: column out of range in row " + std::to_string(i));
            SSB_CHECK(mark[c] != i, SS_ERR_ARG, "ss_ilutp_host: duplicate column in row " + std::to_string(i));
            mark[c] = i;
        }
    }
    const int64_t nnz = rowptr[n];
    A.col.assign(colidx, colidx + nnz);
    A.val.resize(nnz);
    std::memcpy(A.val.data(), vals, nnz * sizeof(double2));
    HostCSR L, U;
    std::vector<int64_t> cp;
    IlutStats st;
    ilut_factor(A, drop_tol, fill_factor, permtol, n_threads, L, U, cp, st);
    SSB_CHECK(L.nnz() <= L_cap && U.nnz() <= U_cap, SS_ERR_ARG,
              "ss_ilutp_host: caps too small, need L_cap >= " + std::to_string(L.nnz()) + " and U_cap >= " +
                  std::to_string(U.nnz()));
    std::memcpy(L_rowptr, L.rowptr.data(), (n + 1) * sizeof(int64_t));
    std::memcpy(L_colidx, L.col.data(), L.nnz() * sizeof(int64_t));
    std::memcpy(L_vals, L.val.data(), L.nnz() * sizeof(double2));
    std::memcpy(U_rowptr, U.rowptr.data(), (n + 1) * sizeof(int64_t));
    std::memcpy(U_colidx, U.col.data(), U.nnz() * sizeof(int64_t));
    std::memcpy(U_vals, U.val.data(), U.nnz() * sizeof(double2));
    std::memcpy(colperm, cp.data(), n * sizeof(int64_t));
    SS_GUARD_END
}

int ss_spmv(ss_problem* h, const void* x_dev, void* y_dev) {
    SS_GUARD_BEGIN
    SSB_CHECK(h && x_dev && y_dev, SS_ERR_ARG, "ss_spmv: NULL argument");
    SSB_CHECK(h->P.have_setup, SS_ERR_STATE, "ss_spmv before ss_setup");
    spmv(h->P.A, (const double2*)x_dev, (double2*)y_dev, h->P.stream);
    SSB_CUDA(cudaStreamSynchronize(h->P.stream));
    SS_GUARD_END
}

int ss_precond(ss_problem* h, int32_t which, const void* x_dev, void* y_dev) {
    SS_GUARD_BEGIN
    SSB_CHECK(h && x_dev && y_dev && x_dev != y_dev, SS_ERR_ARG, "ss_precond: bad pointers");
    const bool async = (which & SS_PRECOND_ASYNC) != 0;
    which &= ~SS_PRECOND_ASYNC;
    SSB_CHECK(which >= 0 && which <= 2, SS_ERR_ARG, "ss_precond: which must be 0, 1 or 2");
    Problem& P = h->P;
    SSB_CHECK(P.have_setup, SS_ERR_STATE, "ss_precond before ss_setup");
    const double2* x = (const double2*)x_dev;
    double2* y = (double2*)y_dev;
    if (which == 0) {
        block_trsv(P.L, x, y, P.stream);
    } else if (which == 1) {
        block_trsv(P.U, x, y, P.stream);
    } else {
        ensure_krylov(P, P.K.m > 0 ? P.K.m : 1);
        block_trsv(P.L, x, P.K.t, P.stream);
        block_trsv(P.U, P.K.t, y, P.stream);
    }
    if (!async) SSB_CUDA(cudaStreamSynchronize(P.stream));
    SS_GUARD_END
}

int ss_debug_trace_trsv(ss_problem* h, int32_t which, const void* x_dev, void* y_dev, uint64_t* host_trace,
                        int64_t* nblk_out) {
    SS_GUARD_BEGIN
    SSB_CHECK(h && x_dev && y_dev && x_dev != y_dev && nblk_out, SS_ERR_ARG, "ss_debug_trace_trsv: bad pointers");
    SSB_CHECK(which == 0 || which == 1, SS_ERR_ARG, "ss_debug_trace_trsv: which must be 0 or 1");
    Problem& P = h->P;
    SSB_CHECK(P.have_setup, SS_ERR_STATE, "ss_debug_trace_trsv before ss_setup");
    DevBlockTri& T = which == 0 ? P.L : P.U;
    *nblk_out = T.nblk;
    if (!host_trace) return SS_OK;
    unsigned long long* d = nullptr;
    SSB_CUDA(cudaMalloc(&d, T.nblk * SS_TRACE_STAMPS * sizeof(unsigned long long)));
    try {
        SSB_CUDA(cudaMemsetAsync(d, 0, T.nblk * SS_TRACE_STAMPS * sizeof(unsigned long long), P.stream));
        block_trsv(T, (const double2*)x_dev, (double2*)y_dev, P.stream, d);
        SSB_CUDA(cudaMemcpyAsync(host_trace, d, T.nblk * SS_TRACE_STAMPS * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                 P.stream));
        SSB_CUDA(cudaStreamSynchronize(P.stream));
    } catch (...) {
        cudaFree(d);
        throw;
    }
    cudaFree(d);
    SS_GUARD_END
}

}  // extern "C"
