"""Oracle: dual-threshold incomplete LU (sec. II) -- Python face of ilut.c.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:94: "incomplete LU factorization with dual-threshold ... a drop
tolerance d and allowed fill-in p are specified such that all fill-in smaller
than d times the infinity-norm of a row are dropped, and at most only
p NNZ(L~) fill-in elements are allowed ... In the limit where d=0, the iLU
preconditioner returns the complete LU factorization".
The arithmetic is in oracle/ilut.c (rules R4-R7 of DESIGN.md, restated there).

Also: condest(), the paper's estimate ||M e||_inf of the approximate inverse,
PAPER.md:126 -- read (R8) as ||(LU)^{-1} e||_inf, e = (1,...,1)^T.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _clib


@dataclass
class IluFactors:
    n: int
    Lp: np.ndarray   # unit lower triangular, strict part only, CSR (cols ascending)
    Lj: np.ndarray
    Lx: np.ndarray
    Up: np.ndarray   # upper triangular, diagonal FIRST in each row, then cols ascending
    Uj: np.ndarray
    Ux: np.ndarray
    perm: np.ndarray | None = None   # ILUTP column permutation: A[:, perm] ~ L U (None: identity)
    columns: bool = False            # True: the factors of A^T (column-oriented iLUTP, R16):
                                     #   A^T[:, perm] ~ L U, i.e. A ~ Pi U^T L^T

    @property
    def nnz(self) -> int:
        return len(self.Lj) + len(self.Uj)

    def L(self) -> sp.csr_matrix:
        """Strictly lower part as a canonical CSR (unit diagonal not stored)."""
        return sp.csr_matrix((self.Lx, self.Lj, self.Lp), shape=(self.n, self.n))

    def U(self) -> sp.csr_matrix:
        M = sp.csr_matrix((self.Ux, self.Uj, self.Up), shape=(self.n, self.n))
        M = M.copy()
        M.sort_indices()
        return M

    def diag(self) -> np.ndarray:
        return self.Ux[self.Up[:-1]]


def ilut(A, drop_tol: float, fill_factor: float) -> IluFactors:
    A = sp.csr_matrix(A)
    A.sort_indices()
    n = A.shape[0]
    rp = np.ascontiguousarray(A.indptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.indices, dtype=np.int64)
    v = np.ascontiguousarray(A.data, dtype=np.complex128)
    P64 = ctypes.POINTER(ctypes.c_int64)
    PD = ctypes.POINTER(ctypes.c_double)
    Lp, Lj, Up, Uj = P64(), P64(), P64(), P64()
    Lx, Ux = PD(), PD()
    Ln, Un = ctypes.c_int64(), ctypes.c_int64()
    lib = _clib.lib()
    rc = lib.oracle_ilut(n, rp.ctypes.data_as(P64), ci.ctypes.data_as(P64), v.view(np.float64).ctypes.data_as(PD),
                         float(drop_tol), float(fill_factor),
                         ctypes.byref(Lp), ctypes.byref(Lj), ctypes.byref(Lx), ctypes.byref(Ln),
                         ctypes.byref(Up), ctypes.byref(Uj), ctypes.byref(Ux), ctypes.byref(Un))
    if rc != 0:
        raise RuntimeError(f"oracle ILUT failed (rc={rc}): zero pivot at row {-rc - 1}" if rc > -2000000000
                           else "oracle ILUT: out of memory")

    def take(pp, jj, xx, nn):
        p = np.ctypeslib.as_array(pp, (n + 1,)).copy()
        j = np.ctypeslib.as_array(jj, (nn,)).copy() if nn else np.zeros(0, np.int64)
        x = np.ctypeslib.as_array(xx, (2 * nn,)).copy().view(np.complex128) if nn else np.zeros(0, np.complex128)
        for q in (pp, jj, xx):
            lib.oracle_free(ctypes.cast(q, ctypes.c_void_p))
        return p, j, x

    lp, lj, lx = take(Lp, Lj, Lx, Ln.value)
    up, uj, ux = take(Up, Uj, Ux, Un.value)
    return IluFactors(n, lp, lj, lx, up, uj, ux)


def ilutp(A, drop_tol: float, fill_factor: float, permtol: float) -> IluFactors:
    """ILUT with column pivoting ("iLUTP"; oracle_ilutp in ilut.c, reading R13):
    A[:, perm] ~ L U.  permtol = 0 reproduces ilut() exactly (perm = identity)."""
    A = sp.csr_matrix(A)
    A.sort_indices()
    n = A.shape[0]
    rp = np.ascontiguousarray(A.indptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.indices, dtype=np.int64)
    v = np.ascontiguousarray(A.data, dtype=np.complex128)
    P64 = ctypes.POINTER(ctypes.c_int64)
    PD = ctypes.POINTER(ctypes.c_double)
    Lp, Lj, Up, Uj, Pm = P64(), P64(), P64(), P64(), P64()
    Lx, Ux = PD(), PD()
    Ln, Un = ctypes.c_int64(), ctypes.c_int64()
    lib = _clib.lib()
    rc = lib.oracle_ilutp(n, rp.ctypes.data_as(P64), ci.ctypes.data_as(P64), v.view(np.float64).ctypes.data_as(PD),
                          float(drop_tol), float(fill_factor), float(permtol),
                          ctypes.byref(Lp), ctypes.byref(Lj), ctypes.byref(Lx), ctypes.byref(Ln),
                          ctypes.byref(Up), ctypes.byref(Uj), ctypes.byref(Ux), ctypes.byref(Un), ctypes.byref(Pm))
    if rc != 0:
        raise RuntimeError(f"oracle ILUTP failed (rc={rc}): zero pivot at row {-rc - 1}" if rc > -2000000000
                           else "oracle ILUTP: out of memory")

    def take(pp, jj, xx, nn):
        p = np.ctypeslib.as_array(pp, (n + 1,)).copy()
        j = np.ctypeslib.as_array(jj, (nn,)).copy() if nn else np.zeros(0, np.int64)
        x = np.ctypeslib.as_array(xx, (2 * nn,)).copy().view(np.complex128) if nn else np.zeros(0, np.complex128)
        for q in (pp, jj, xx):
            lib.oracle_free(ctypes.cast(q, ctypes.c_void_p))
        return p, j, x

    lp, lj, lx = take(Lp, Lj, Lx, Ln.value)
    up, uj, ux = take(Up, Uj, Ux, Un.value)
    perm = np.ctypeslib.as_array(Pm, (n,)).copy()
    lib.oracle_free(ctypes.cast(Pm, ctypes.c_void_p))
    return IluFactors(n, lp, lj, lx, up, uj, ux, perm)


def ilutp_columns(A, drop_tol: float, fill_factor: float, permtol: float) -> IluFactors:
    """Column-oriented iLUTP (reading R16 of DESIGN.md): the factorisation works on the
    columns of A -- each column's fill is dropped against d times the infinity norm of
    that column of A, its L and U parts are capped at floor(p nnz(A[:, j]) / 2), and the
    pivot is exchanged along the column (rows) -- which is exactly the row-wise iLUTP
    above applied to A^T.  This is the orientation of SuperLU's ILU ("the
    SuperLU solver from SciPy", which the paper's iLUTP is).

    With A^T Pi = L U (perm: A^T[:, perm] = L U):  Pi^T A = U^T L^T, so
    M = Pi U^T L^T  and  M^{-1} v = L^{-T} U^{-T} (Pi^T v),  (Pi^T v)[j] = v[perm[j]].
    """
    A = sp.csr_matrix(A)
    F = ilutp(sp.csr_matrix(A.T), drop_tol, fill_factor, permtol)
    F.columns = True
    return F


def condest(F: IluFactors) -> float:
    """||(LU)^{-1} e||_inf, PAPER.md:126 (reading R8)."""
    from .trisolve import apply_preconditioner
    return float(np.abs(apply_preconditioner(F, np.ones(F.n, dtype=np.complex128))).max())
