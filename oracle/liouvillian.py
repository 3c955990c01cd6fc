"""Oracle: Hamiltonian, Lindblad Liouvillian and trace-constrained system.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows PAPER.md line-by-line:
  * Eq. (1), PAPER.md:27-29 -- H/hbar = -Delta a^+a + omega_m b^+b
      + g0 (b + b^+) a^+a + E (a + a^+).
  * Eq. (3), PAPER.md:52-56 -- L[rho] = -i[H, rho] + kappa D[a, rho]
      + Gamma_m (1+n_th) D[b, rho] + Gamma_m n_th D[b^+, rho],
      D[O, rho] = 1/2 [2 O rho O^+ - rho O^+O - O^+O rho].
  * Eq. (4), PAPER.md:62 -- vec(rho) is column stacking; hence
      vec(A rho B) = (B^T kron A) vec(rho).
  * sec. III, PAPER.md:100 -- a == a (x) I_b, b == I_a (x) b  (cavity is the
      outer tensor factor: Hilbert index i = c * N_m + m).
  * Eq. (5), PAPER.md:67-70 -- L~ = L + w T, T has ones in row 0 at the columns
      of the diagonal elements of rho (index k (N+1)), right-hand side (w,0,...).
  * sec. IV, PAPER.md:119 -- "we set the weighting factor w ... to be the
      average of the diagonal elements in L" (used when Params.w is None).

The matrices are assembled with scipy.sparse.kron (a library primitive) exactly
as the formulas read; explicit zeros are removed (a canonical CSR, as needed
for the NNZ(L~) = 8957 count in the Fig. 1 caption).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def destroy(n: int) -> sp.csr_matrix:
    """Truncated annihilation operator: <k-1| a |k> = sqrt(k), k = 1..n-1."""
    if n < 1:
        raise ValueError("Fock cut-off must be >= 1")
    k = np.arange(1, n)
    return sp.csr_matrix((np.sqrt(k).astype(np.complex128), (k - 1, k)), shape=(n, n))


def operators(N_c: int, N_m: int):
    """a = a (x) I_{N_m}, b = I_{N_c} (x) b."""
    a = sp.kron(destroy(N_c), sp.identity(N_m, dtype=np.complex128), format="csr")
    b = sp.kron(sp.identity(N_c, dtype=np.complex128), destroy(N_m), format="csr")
    return a, b


def dag(A):
    return A.conj().T.tocsr()


def hamiltonian(p) -> sp.csr_matrix:
    """Eq. (1)."""
    a, b = operators(p.N_c, p.N_m)
    ad, bd = dag(a), dag(b)
    n_a = ad @ a
    H = (-p.Delta) * n_a + p.omega_m * (bd @ b) + p.g0 * ((b + bd) @ n_a) + p.E * (a + ad)
    H = H.tocsr()
    H.eliminate_zeros()
    return H


def collapse_ops(p):
    """The three Lindblad channels of Eq. (3), with their rates."""
    a, b = operators(p.N_c, p.N_m)
    return [(a, p.kappa), (b, p.Gamma_m * (1.0 + p.n_th)), (dag(b), p.Gamma_m * p.n_th)]


def liouvillian(p) -> sp.csr_matrix:
    """Matrix of Eq. (3) acting on column-stacked vec(rho) (Eq. (4)).

    -i[H, rho]          -> -i (I kron H  -  H^T kron I)
    r D[C, rho]         -> r (conj(C) kron C - 1/2 I kron C^+C - 1/2 (C^+C)^T kron I)
    """
    N = p.hilbert_dim
    I = sp.identity(N, dtype=np.complex128, format="csr")
    H = hamiltonian(p)
    L = -1j * (sp.kron(I, H) - sp.kron(H.T, I))
    for C, r in collapse_ops(p):
        if r == 0.0:
            continue
        CdC = dag(C) @ C
        L = L + r * (sp.kron(C.conj(), C) - 0.5 * sp.kron(I, CdC) - 0.5 * sp.kron(CdC.T, I))
    L = sp.csr_matrix(L)
    L.eliminate_zeros()
    L.sort_indices()
    return L


def trace_matrix(N: int) -> sp.csr_matrix:
    """T of Eq. (5): ones in row 0 at columns k (N+1), k = 0..N-1."""
    n = N * N
    cols = np.arange(N) * (N + 1)
    return sp.csr_matrix((np.ones(N, dtype=np.complex128), (np.zeros(N, dtype=np.int64), cols)),
                         shape=(n, n))


def trace_weight(L: sp.csr_matrix, p) -> complex:
    """w of Eq. (5): Params.w if given, else mean(diag(L)).

    Reading R1: the mean is (sum of the n diagonal elements accumulated
    left to right, index 0 first) / n -- np.cumsum is that sequential sum.
    """
    if p.w is not None:
        return complex(p.w)
    d = L.diagonal()
    n = d.shape[0]
    return complex(np.cumsum(d.real)[-1] / n, np.cumsum(d.imag)[-1] / n)


def constrained_system(p):
    """Eq. (5): returns (L~, rhs, w, L) with L~ = L + w T and rhs = (w, 0, ..., 0)."""
    L = liouvillian(p)
    w = trace_weight(L, p)
    T = trace_matrix(p.hilbert_dim)
    Lt = sp.csr_matrix(L + w * T)
    Lt.eliminate_zeros()
    Lt.sort_indices()
    rhs = np.zeros(Lt.shape[0], dtype=np.complex128)
    rhs[0] = w
    return Lt, rhs, w, L


def unvec(x: np.ndarray, N: int) -> np.ndarray:
    """Inverse of column stacking (Eq. (4)): rho[i, j] = x[i + N j]."""
    return np.asarray(x).reshape((N, N), order="F")


def vec(rho: np.ndarray) -> np.ndarray:
    return np.asarray(rho).reshape(-1, order="F")
