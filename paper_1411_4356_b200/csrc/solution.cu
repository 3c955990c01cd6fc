// solution.cu -- map the GMRES iterate back to rho and form the observables.
//
// x solves L~_RCM x = b_RCM; the natural-order vector is x_nat[perm[k]] = x[k]
// (sec. III "apply the resulting row and column ordering"), and
// rho = unvec(x_nat) with column stacking (Eq. (4)): rho_ij = x_nat[i + N j].
// Reading R11: rho <- rho / Tr(rho).  Observables <a^+a> = sum_i rho_ii c(i),
// <b^+b> = sum_i rho_ii m(i) with i = c N_m + m.
#include "problem.h"

namespace ssb {

namespace {

__global__ void k_unpermute(const double2* __restrict__ x, const int64_t* __restrict__ perm, int64_t n,
                            double2* __restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        out[perm[k]] = x[k];
}

// one block: tr = sum_k rho[k (N+1)], na = sum Re(rho_kk) c(k), nb = sum Re(rho_kk) m(k)
__global__ void k_diag_sums(const double2* __restrict__ rho, int64_t N, int Nm, double* out) {
    __shared__ double s[4][256];
    double tr = 0, ti = 0, a = 0, b = 0;
    for (int64_t k = threadIdx.x; k < N; k += blockDim.x) {
        const double2 d = rho[k * (N + 1)];
        tr += d.x;
        ti += d.y;
        a += d.x * (double)(k / Nm);
        b += d.x * (double)(k % Nm);
    }
    s[0][threadIdx.x] = tr;
    s[1][threadIdx.x] = ti;
    s[2][threadIdx.x] = a;
    s[3][threadIdx.x] = b;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int q = 0; q < 4; q++) s[q][threadIdx.x] += s[q][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x < 4) out[threadIdx.x] = s[threadIdx.x][0];
}

// rho *= 1 / (tr_re + i tr_im)
__global__ void k_normalise(double2* rho, int64_t n, const double* tr) {
    const double2 t = make_double2(tr[0], tr[1]);
    const double d = t.x * t.x + t.y * t.y;
    const double2 inv = make_double2(t.x / d, -t.y / d);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        rho[k] = cmul(rho[k], inv);
}

__global__ void k_gather(const double2* __restrict__ src, const int64_t* __restrict__ perm, int64_t n,
                         double2* __restrict__ dst) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = src[perm[k]];
}

}  // namespace

void gather_perm(const double2* src, const int64_t* perm, int64_t n, double2* dst, cudaStream_t s) {
    k_gather<<<grid_for(n, 256, kNumSMs * 8), 256, 0, s>>>(src, perm, n, dst);
    SSB_LAUNCHED();
}

void scatter_perm(const double2* src, const int64_t* perm, int64_t n, double2* dst, cudaStream_t s) {
    k_unpermute<<<grid_for(n, 256, kNumSMs * 8), 256, 0, s>>>(src, perm, n, dst);
    SSB_LAUNCHED();
}

void finish_solution(Problem& P, ss_solve_info* info) {
    const int64_t n = P.n;
    cudaStream_t s = P.stream;
    if (!P.rho) SSB_CUDA(cudaMalloc(&P.rho, n * sizeof(double2)));
    k_unpermute<<<grid_for(n, 256, kNumSMs * 8), 256, 0, s>>>(P.K.x, P.d_perm, n, P.rho);
    SSB_LAUNCHED();
    double* d_out = P.K.scal + 4;
    k_diag_sums<<<1, 256, 0, s>>>(P.rho, P.N, P.params.N_m, d_out);
    SSB_LAUNCHED();
    k_normalise<<<grid_for(n, 256, kNumSMs * 8), 256, 0, s>>>(P.rho, n, d_out);
    SSB_LAUNCHED();
    double h[2];
    SSB_CUDA(cudaMemcpyAsync(h, d_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    if (info) {
        info->trace_re = h[0];
        info->trace_im = h[1];
    }
    P.have_solution = true;
}

void expectations(Problem& P, double* na, double* nb) {
    SSB_CHECK(P.have_solution, SS_ERR_STATE, "ss_expect before ss_solve");
    cudaStream_t s = P.stream;
    double* d_out = P.K.scal + 4;
    k_diag_sums<<<1, 256, 0, s>>>(P.rho, P.N, P.params.N_m, d_out);
    SSB_LAUNCHED();
    double h[4];
    SSB_CUDA(cudaMemcpyAsync(h, d_out, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    *na = h[2];
    *nb = h[3];
}

}  // namespace ssb
