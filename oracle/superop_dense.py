"""Oracle pin helper: the Liouvillian built by APPLYING Eq. (3) to basis matrices.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Independent of oracle/liouvillian.py's kron identities: the Hamiltonian and the
collapse operators are written here as dense Fock-basis matrices from their
matrix elements (<c-1|a|c> = sqrt(c), PAPER.md:30 operators, ordering of
PAPER.md:100), and column (k + N l) of the superoperator is vec(L[E_kl]) with
E_kl the basis matrix and L[.] evaluated literally as in Eq. (3), PAPER.md:52-56,
vec = column stacking.  Only usable for tiny Hilbert spaces.
"""
from __future__ import annotations

import numpy as np


def dense_ops(N_c: int, N_m: int):
    N = N_c * N_m
    a = np.zeros((N, N), dtype=np.complex128)
    b = np.zeros((N, N), dtype=np.complex128)
    for c in range(N_c):
        for m in range(N_m):
            i = c * N_m + m
            if c >= 1:
                a[(c - 1) * N_m + m, i] = np.sqrt(c)
            if m >= 1:
                b[c * N_m + (m - 1), i] = np.sqrt(m)
    return a, b


def dense_H(p):
    a, b = dense_ops(p.N_c, p.N_m)
    ad, bd = a.conj().T, b.conj().T
    return -p.Delta * ad @ a + p.omega_m * bd @ b + p.g0 * (b + bd) @ ad @ a + p.E * (a + ad)


def apply_L(p, rho: np.ndarray) -> np.ndarray:
    """L[rho] of Eq. (3) evaluated with dense matrix products."""
    a, b = dense_ops(p.N_c, p.N_m)
    H = dense_H(p)
    out = -1j * (H @ rho - rho @ H)
    for C, r in ((a, p.kappa), (b, p.Gamma_m * (1 + p.n_th)), (b.conj().T, p.Gamma_m * p.n_th)):
        Cd = C.conj().T
        out = out + r * 0.5 * (2 * C @ rho @ Cd - rho @ Cd @ C - Cd @ C @ rho)
    return out


def dense_liouvillian(p) -> np.ndarray:
    N = p.N_c * p.N_m
    L = np.zeros((N * N, N * N), dtype=np.complex128)
    for l in range(N):
        for k in range(N):
            E = np.zeros((N, N), dtype=np.complex128)
            E[k, l] = 1.0
            L[:, k + N * l] = apply_L(p, E).reshape(-1, order="F")
    return L


def nullspace_steady_state(p) -> np.ndarray:
    """Eq. (2)/(4): rho_ss spans the null space of L; via the smallest right
    singular vector of the dense matrix, normalised to unit trace."""
    L = dense_liouvillian(p)
    _, s, vh = np.linalg.svd(L)
    x = vh[-1].conj()
    N = p.N_c * p.N_m
    rho = x.reshape((N, N), order="F")
    return rho / np.trace(rho), s
