/*
 * ss_b200.h -- C ABI of the B200-native steady-state solver for the driven,
 * damped optomechanical Liouvillian of arXiv:1411.4356.
 *
 * The operation the library performs is the paper's statement of the problem:
 *   find rho_ss with  L~ vec(rho_ss) = (w, 0, ..., 0)^T            Eq. (5)
 *   L[rho] = -i[H,rho] + kappa D[a] + Gamma_m(1+n_th) D[b] + Gamma_m n_th D[b^+]
 *                                                                   Eq. (3)
 *   H = -Delta a^+a + omega_m b^+b + g0 (b+b^+) a^+a + E (a+a^+)    Eq. (1)
 * vec() column stacking, a = a (x) I_b, b = I_a (x) b,
 * solved by GMRES(m) on the reverse-Cuthill-McKee permuted L~
 * (sec. III) with an incomplete-LU dual-threshold preconditioner
 * (sec. II) applied from the left (Eq. (8)).
 *
 * Conventions for every entry point
 *  - complex128 values are interleaved (re, im) pairs of IEEE doubles, 16-byte
 *    aligned; "a complex vector of length n" is 2n doubles.
 *  - index arrays are int64 on the host side of the ABI (int32 column indices
 *    are used internally on the device; n and row lengths are < 2^31).
 *  - "device pointer" = a CUDA global-memory address on the handle's device,
 *    owned by the caller (e.g. a torch tensor's data_ptr()); "host pointer" =
 *    ordinary (optionally pinned) host memory owned by the caller.
 *  - the library owns every buffer it allocates inside a handle; they are
 *    released by ss_destroy.  All device work runs on the CUDA stream given to
 *    ss_build (NULL = legacy default stream); every call returns only after
 *    its work on that stream has completed unless stated otherwise.
 *  - return value: SS_OK (0) on success, otherwise one of the SS_ERR_* codes;
 *    ss_last_error() then returns a NUL-terminated, thread-local message.
 *    On error the handle stays valid (it may need ss_setup again).
 *  - there is NO CPU fallback: without a CUDA device every call that computes
 *    returns SS_ERR_CUDA.
 */
#ifndef SS_B200_H
#define SS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_OK 0
#define SS_ERR_ARG 1        /* invalid argument (sizes, NULL, ranges)                */
#define SS_ERR_CUDA 2       /* CUDA runtime error / no device                        */
#define SS_ERR_OOM 3        /* device or host allocation failed                       */
#define SS_ERR_BREAKDOWN 4  /* ILUT zero pivot that cannot be repaired (drop_tol = 0)  */
#define SS_ERR_STATE 5      /* call out of order (e.g. ss_solve before ss_setup)      */

/* Physical parameters, Eq. (1) and Eq. (3); all rates in units of omega_m. */
typedef struct ss_params {
    int32_t N_c;        /* cavity Fock cut-off   (>= 1)                                */
    int32_t N_m;        /* mechanical Fock cut-off (>= 1); Hilbert dim N = N_c N_m     */
    double omega_m;     /* mechanical frequency                                        */
    double Delta;       /* pump-cavity detuning  (H term -Delta a^+a)                  */
    double kappa;       /* cavity decay rate  (>= 0)                                   */
    double g0;          /* vacuum optomechanical coupling                              */
    double E;           /* pump amplitude                                              */
    double Gamma_m;     /* mechanical damping (>= 0)                                   */
    double n_th;        /* bath occupation (>= 0)                                      */
    double w;           /* trace weight of Eq. (5); NaN -> mean of diag(L) */
} ss_params;

typedef struct ss_problem ss_problem;   /* opaque handle: one Liouvillian on one GPU */

typedef struct ss_build_info {
    int64_t hilbert_dim;   /* N = N_c N_m                                  */
    int64_t n;             /* Liouvillian dimension N^2                    */
    int64_t nnz;           /* stored entries of L~ (exact zeros pruned)    */
    double w_re, w_im;     /* the trace weight used                        */
    double build_ms;       /* device time of the assembly                  */
} ss_build_info;

typedef struct ss_setup_info {
    int64_t nnz_L;          /* strict lower entries of the ILU factor (unit diag implicit) */
    int64_t nnz_U;          /* upper entries incl. the diagonal                             */
    double fill;            /* (nnz_L + nnz_U) / nnz(L~)  -- Fig. 3 "fill-factor"            */
    int64_t bandwidth_nat;  /* B(L~), sec. II                                                */
    int64_t bandwidth_rcm;  /* B(L~_RCM)                                                      */
    int64_t levels_L;       /* dependency levels of the forward / backward substitutions    */
    int64_t levels_U;
    int32_t pivots_repaired;/* zero pivots replaced by tau_i (reading R6)                     */
    int32_t pivot_swaps;    /* column exchanges made by the iLUTP pivoting (reading R13)      */
    int32_t pad0;
    int32_t threads;        /* host threads used by the factorisation                        */
    int32_t trsv_block;     /* rows per block B of the block substitution (trsv.cu)          */
    int32_t trsv_grid;      /* persistent CTAs of the block substitution (chain + helpers)   */
    int32_t trsv_q_L;       /* smallest near window Q_k of the L / U substitution (source      */
    int32_t trsv_q_U;       /*   blocks k-Q_k+1..k-1 on the chain SM, older ones on helpers)  */
    double rcm_ms, ilut_ms, upload_ms;
} ss_setup_info;

typedef struct ss_solve_info {
    int32_t iterations;     /* Arnoldi steps = applications of M^{-1} L~                 */
    int32_t cycles;         /* GMRES restarts performed                                  */
    int32_t converged;      /* 1 iff rel_residual <= tol                                 */
    int32_t pad;
    double rel_residual;    /* true ||b - L~ x||_2 / ||b||_2 at exit (x before rescaling) */
    double trace_re, trace_im; /* Tr(rho) before normalisation                            */
    double solve_ms;        /* device time of the whole solve                             */
} ss_solve_info;

/* ---------------- the four calls of the method ---------------- */

/* Assemble L~ of Eq. (5) (natural order, CSR, complex128) on the current CUDA device,
 * on stream `cuda_stream` (a cudaStream_t, may be NULL).  *out receives a new handle. */
int ss_build(const ss_params* p, void* cuda_stream, ss_problem** out, ss_build_info* info);

/* One-time setup: RCM ordering of pattern(L~ + L~^T) (sec. III), the
 * symmetric permutation L~_RCM, the column-oriented iLUTP(drop_tol, fill_factor, permtol)
 * of L~_RCM (sec. II, "dual-threshold and pivoting", SuperLU's orientation,
 * PAPER.md:119; R4-R7, R13, R16): the row-wise iLUTP of its transpose,
 * L~_RCM^T Pi ~ L' U', so Pi^T L~_RCM ~ U'^T L'^T (permtol = 0: no exchanges = plain
 * ILUT); the operator of the hot path A' = Pi^T L~_RCM (rows in pivot order, SELL-32
 * copy for the SpMV), the block layout of the two substitutions and their upload.  n_threads <= 0 -> all host cores (more than the host
 * cores are clamped to that; the factors are the same for any n_threads).  May be called again
 * with other parameters.  Errors: SS_ERR_ARG (negative parameter), SS_ERR_BREAKDOWN
 * (zero pivot with drop_tol = 0). */
int ss_setup(ss_problem* h, double drop_tol, double fill_factor, double permtol, int32_t n_threads,
             ss_setup_info* info);

/* Solve Eq. (5) by left-preconditioned GMRES(restart) (Eq. (8)) from
 * x0 = 0 to the true relative residual tol, at most max_iter Arnoldi steps.  The
 * solution is normalised to Tr rho = 1 (reading R11) and kept on the device. */
int ss_solve(ss_problem* h, int32_t restart, double tol, int32_t max_iter, ss_solve_info* info);

/* Observables of the last solution: <a^+a> = Tr(rho a^+a), <b^+b> = Tr(rho b^+b). */
int ss_expect(ss_problem* h, double* n_cavity, double* n_mech);

/* Copy the last solution rho (N x N complex128, column-major == vec(rho) of Eq. (4))
 * to dst (N*N*16 bytes), a device pointer if dst_is_device else a host pointer. */
int ss_get_rho(ss_problem* h, void* dst, int32_t dst_is_device);

/* End-to-end variant for callers holding HOST buffers: copies rhs (natural order,
 * length n, host) to the device, runs the same GMRES, copies the raw solution x
 * (natural order, length n, not normalised) back to x_host.  rhs_host == NULL uses
 * the Eq. (5) right-hand side.  The copies are part of the call. */
int ss_solve_host(ss_problem* h, const double* rhs_host, double* x_host, int32_t restart,
                  double tol, int32_t max_iter, ss_solve_info* info);

void ss_destroy(ss_problem* h);
const char* ss_last_error(void);

/* ---------------- kernel-level entry points (parity tests, benchmark) ---------------- */

/* Dimensions: n, nnz(L~); after ss_setup also nnz_L, nnz_U (else -1). */
int ss_sizes(const ss_problem* h, int64_t* n, int64_t* nnz, int64_t* nnz_L, int64_t* nnz_U);

/* Copy L~ (which = 0: natural order; 1: the hot path's operator A' = Pi^T L~_RCM, i.e.
 * row j = row colperm[j] of L~_RCM, needs ss_setup) to host CSR arrays: rowptr[n+1],
 * colidx[nnz] (int64), vals[2*nnz] (complex128).  Columns ascending. */
int ss_export_matrix(const ss_problem* h, int32_t which, int64_t* rowptr, int64_t* colidx,
                     double* vals);

/* Copy the RCM permutation perm[n] (new -> old: L~_RCM = L~[perm][:, perm]). */
int ss_export_perm(const ss_problem* h, int64_t* perm);

/* Copy the iLUTP pivot permutation colperm[n]: L~_RCM^T[:, colperm] ~ L' U' (R16), i.e.
 * row j of A' is row colperm[j] of L~_RCM; the identity when nothing was exchanged. */
int ss_export_colperm(const ss_problem* h, int64_t* colperm);

/* Copy an iLUTP factor of L~_RCM^T to host CSR: which = 0: strict lower L' (unit
 * diagonal implicit), rowptr[n+1], colidx[nnz_L], vals[2 nnz_L]; which = 1: U' with its
 * diagonal FIRST in every row then strict upper columns ascending, rowptr[n+1],
 * colidx[nnz_U], vals[2 nnz_U].  M'^{-1} = L'^{-T} U'^{-T}. */
int ss_export_factors(const ss_problem* h, int32_t which, int64_t* rowptr, int64_t* colidx,
                      double* vals);

/* Host-only iLUTP (sec. II; rules R4-R7, R13 of DESIGN.md) of a given CSR
 * matrix A (n rows, int64 rowptr[n+1] / colidx[nnz] with columns in [0, n) and no
 * duplicates in a row, complex128 vals[2 nnz]), with the same multi-threaded code and the
 * same results as ss_setup (bit-identical for any n_threads; n_threads <= 0: all host
 * cores).  Needs no GPU.  Outputs, caller-allocated: L (strict lower, unit diagonal
 * implicit) L_rowptr[n+1], L_colidx[L_cap], L_vals[2 L_cap]; U (diagonal first in every
 * row) U_rowptr[n+1], U_colidx[U_cap], U_vals[2 U_cap]; colperm[n] (A[:, colperm] ~ L U).
 * Enough room: L_cap = sum_i floor(p nnz(a_i) / 2), U_cap = that + n (rule R5).  Errors:
 * SS_ERR_ARG (bad arguments, caps too small: the message states the sizes needed),
 * SS_ERR_BREAKDOWN (zero pivot with drop_tol = 0). */
int ss_ilutp_host(int64_t n, const int64_t* rowptr, const int64_t* colidx, const double* vals, double drop_tol,
                  double fill_factor, double permtol, int32_t n_threads, int64_t* L_rowptr, int64_t* L_colidx,
                  double* L_vals, int64_t L_cap, int64_t* U_rowptr, int64_t* U_colidx, double* U_vals,
                  int64_t U_cap, int64_t* colperm);

/* y = A' x = Pi^T L~_RCM x  (device pointers, complex128 length n).                */
int ss_spmv(ss_problem* h, const void* x_dev, void* y_dev);
/* y = U'^{-T} x (which = 0, the first substitution: lower, the pivots on its diagonal),
 * y = L'^{-T} x (which = 1, unit upper), y = M'^{-1} x = L'^{-T} U'^{-T} x (which = 2);
 * M'^{-1} A' = M^{-1} L~_RCM with M = Pi U'^T L'^T (R16);
 * device pointers, length n, x and y may not alias.  which | SS_PRECOND_ASYNC: return
 * right after the launches (stream-ordered, no host synchronisation; used to time the
 * kernels with events).  which = 2 uses the handle's Krylov scratch vector.          */
#define SS_PRECOND_ASYNC 4
int ss_precond(ss_problem* h, int32_t which, const void* x_dev, void* y_dev);

/* Diagnostic: run the block substitution of factor `which` (0 = L, 1 = U) on x_dev -> y_dev
 * (device pointers, length n) with per-block %globaltimer stamps (ns) copied to host_trace
 * [SS_TRACE_STAMPS * nblk], row k (block k): 0 chain team: partials of block k reduced,
 * 2 lieutenant 6: its q_k sent, 3 x_k stored in the chain ring, 4 helper: y_k published,
 * 5 producer: y_k staged (flag seen), 6 chain team: the lieutenants' q_k landed,
 * 7 lieutenant 0: x_{k-3} landed, 8 chain team: x_k pushed to the lieutenants,
 * 9 lieutenant 0: q_k sent, 10 chain team: off-chain work of block k done, 11 lieutenant
 * 0: early part done, 12 lieutenant 0: stage of block k ready, 13 chain team: x_{k-1}
 * read; 1, 14, 15 zero (14: only in -DSSB_LT_G3 experiment builds, lieutenant 0 saw
 * x_{k-3}).  *nblk_out receives the number of blocks (host_trace may be NULL to query it). */
#define SS_TRACE_STAMPS 16
int ss_debug_trace_trsv(ss_problem* h, int32_t which, const void* x_dev, void* y_dev, uint64_t* host_trace,
                        int64_t* nblk_out);

/* Test hook: fill the shared memory of every SM with 0xFF bytes (a NaN pattern as complex128) on
 * the problem's stream.  Shared memory is not cleared between kernels, so this stands in for
 * "whatever another kernel left there": a substitution that multiplies a zeroed value by a
 * ring slot or partial it has not written in this launch (0 * NaN = NaN) fails after it
 * (tests/test_gpu_parity.py::test_precond_ignores_stale_shared_memory).  Errors: SS_ERR_ARG,
 * SS_ERR_CUDA. */
int ss_debug_poison_smem(ss_problem* h);

/* Limit the substitution kernels of this problem to `sms` SMs (rounded down to whole
 * 8-CTA clusters, at least 2 clusters; 0 = the whole GPU, the default), so that several
 * problems can run their solves concurrently on one GPU from different host threads and
 * streams (the detuning sweep: "several simulations to be
 * run in parallel").  The launches of one problem spin on each other's CTAs, so the
 * budgets of the problems solved at the same time must add up to at most the GPU's
 * co-resident clusters.  Takes effect at the next substitution.  Errors: SS_ERR_ARG. */
int ss_set_sm_budget(ss_problem* h, int32_t sms);

/* Number of CUDA kernels this library has launched since load (gpu_launches evidence). */
int64_t ss_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* SS_B200_H */
