"""Oracle: applying the ILU preconditioner M^{-1} of Eq. (8).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:84-87 (Eq. (8)): the preconditioned system M^{-1} L~ rho = M^{-1} b
with M = L U from the incomplete factorisation.  Applying M^{-1}
is a forward substitution with the unit lower factor followed by a backward
substitution with the upper factor.  ``forward``/``backward`` are the textbook
loops (small inputs); ``apply_preconditioner`` uses scipy's
spsolve_triangular (a library primitive) for large ones.

Two orientations (R13, R16):
  row-wise iLUTP      A Pi = L U:        M^{-1} v = Pi U^{-1} L^{-1} v
  column-wise iLUTP   A^T Pi = L U:      M^{-1} v = L^{-T} U^{-T} (Pi^T v)
(L unit lower, U upper with its diagonal first in each row, perm[p] = the column of
A (A^T) at position p.)
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as sla


def forward(F, b: np.ndarray) -> np.ndarray:
    """y_i = b_i - sum_{j<i} l_ij y_j   (unit diagonal)."""
    y = np.array(b, dtype=np.complex128)
    for i in range(F.n):
        s = y[i]
        for q in range(F.Lp[i], F.Lp[i + 1]):
            s -= F.Lx[q] * y[F.Lj[q]]
        y[i] = s
    return y


def backward(F, y: np.ndarray) -> np.ndarray:
    """x_i = (y_i - sum_{j>i} u_ij x_j) / u_ii."""
    x = np.array(y, dtype=np.complex128)
    for i in range(F.n - 1, -1, -1):
        q0 = F.Up[i]
        s = x[i]
        for q in range(q0 + 1, F.Up[i + 1]):
            s -= F.Ux[q] * x[F.Uj[q]]
        x[i] = s / F.Ux[q0]
    return x


def forward_transposed(F, y: np.ndarray) -> np.ndarray:
    """Solve U^T z = y (U^T lower, non-unit), column sweep over the rows of U:
    z_i = y_i / u_ii, then y_j -= u_ij z_i for the entries j > i of row i of U."""
    y = np.array(y, dtype=np.complex128)
    z = np.zeros_like(y)
    for i in range(F.n):
        q0 = F.Up[i]
        z[i] = y[i] / F.Ux[q0]
        for q in range(q0 + 1, F.Up[i + 1]):
            y[F.Uj[q]] -= F.Ux[q] * z[i]
    return z


def backward_transposed(F, z: np.ndarray) -> np.ndarray:
    """Solve L^T x = z (L^T unit upper), column sweep over the rows of L from the last:
    x_i = z_i, then z_j -= l_ij x_i for the entries j < i of row i of L."""
    z = np.array(z, dtype=np.complex128)
    x = np.zeros_like(z)
    for i in range(F.n - 1, -1, -1):
        x[i] = z[i]
        for q in range(F.Lp[i], F.Lp[i + 1]):
            z[F.Lj[q]] -= F.Lx[q] * x[i]
    return x


def lower_unit_matrix(F) -> sp.csr_matrix:
    return sp.csr_matrix(F.L() + sp.identity(F.n, dtype=np.complex128, format="csr"))


def unpivot(F, y: np.ndarray) -> np.ndarray:
    """ILUTP: A Pi = L U, so M^{-1} = Pi U^{-1} L^{-1}: x[perm[p]] = y[p] (identity for ILUT)."""
    if getattr(F, "perm", None) is None:
        return y
    x = np.empty_like(y)
    x[F.perm] = y
    return x


def pivot_gather(F, v: np.ndarray) -> np.ndarray:
    """Column-wise iLUTP: (Pi^T v)[j] = v[perm[j]] (identity without exchanges)."""
    if getattr(F, "perm", None) is None:
        return np.asarray(v, dtype=np.complex128)
    return np.asarray(v, dtype=np.complex128)[F.perm]


def apply_preconditioner(F, v: np.ndarray, small_loops: bool = False) -> np.ndarray:
    if getattr(F, "columns", False):
        y = pivot_gather(F, v)
        if small_loops:
            return backward_transposed(F, forward_transposed(F, y))
        Lt = sp.csr_matrix(lower_unit_matrix(F).T)
        Ut = sp.csr_matrix(F.U().T)
        z = sla.spsolve_triangular(Ut, y, lower=True)
        return sla.spsolve_triangular(Lt, z, lower=False, unit_diagonal=True)
    if small_loops:
        return unpivot(F, backward(F, forward(F, v)))
    Lm = lower_unit_matrix(F)
    Um = F.U()
    y = sla.spsolve_triangular(Lm, np.asarray(v, dtype=np.complex128), lower=True, unit_diagonal=True)
    return unpivot(F, sla.spsolve_triangular(Um, y, lower=False))
