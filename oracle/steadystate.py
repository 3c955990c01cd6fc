"""Oracle: the end-to-end steady-state computation and its observables.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Pipeline (sec. II-IV):
  build L~, rhs          Eq. (5)                         oracle.liouvillian
  RCM of L~ + L~^T       sec. III, PAPER.md:98            oracle.rcm / rcm_ref.c
  iLUTP of L~_RCM        sec. II, PAPER.md:94, :119       oracle.ilut (ilutp_columns: the
                         column-oriented iLUTP of SuperLU, R16; ilutp: row-wise)
  GMRES(m), left prec.   sec. IV, Eq. (8)    oracle.gmres
  un-permute, unvec      Eq. (4) column stacking
and the reference answer of the linear system itself:
  direct solve           Eq. (5) "direct (i.e non-iterative) solution ... via
                         sparse LU decomposition" PAPER.md:66 (scipy's SuperLU,
                         a library primitive, as in the paper PAPER.md:119).
Normalisation (R11): rho <- rho / Tr(rho) after the solve.
Observables: <a^+a> = Tr(rho a^+a), <b^+b> = Tr(rho b^+b) (the <n>, <b^+b> the
north star gathers); both are sums of diagonal elements weighted by the Fock
numbers c(i), m(i) of i = c N_m + m (PAPER.md:100 ordering).
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as sla

from . import liouvillian as lv
from . import rcm as rcm_py
from . import _clib
from .ilut import ilutp, ilutp_columns, IluFactors
from .trisolve import apply_preconditioner
from .gmres import gmres, GmresResult


def rcm_c(S: sp.csr_matrix) -> np.ndarray:
    """Order with oracle/rcm_ref.c (same rule as oracle.rcm.rcm, fast)."""
    S = sp.csr_matrix(S)
    S.sort_indices()
    n = S.shape[0]
    rp = np.ascontiguousarray(S.indptr, dtype=np.int64)
    ci = np.ascontiguousarray(S.indices, dtype=np.int64)
    perm = np.empty(n, dtype=np.int64)
    P64 = ctypes.POINTER(ctypes.c_int64)
    rc = _clib.lib().oracle_rcm(n, rp.ctypes.data_as(P64), ci.ctypes.data_as(P64), perm.ctypes.data_as(P64))
    if rc != 0:
        raise RuntimeError(f"oracle_rcm failed rc={rc}")
    return perm


def order(Lt: sp.csr_matrix, use_c: bool = True) -> np.ndarray:
    S = rcm_py.symmetrized_pattern(Lt)
    return rcm_c(S) if use_c else rcm_py.rcm(S)


def normalise(x: np.ndarray, N: int) -> np.ndarray:
    rho = lv.unvec(x, N)
    return rho / np.trace(rho)


def solve_direct(p) -> np.ndarray:
    Lt, rhs, w, L = lv.constrained_system(p)
    x = sla.spsolve(sp.csc_matrix(Lt), rhs)
    return normalise(x, p.hilbert_dim)


@dataclass
class IterativeResult:
    rho: np.ndarray
    x: np.ndarray               # raw solution (natural order, before normalisation)
    perm: np.ndarray
    factors: IluFactors
    gmres: GmresResult
    times: dict


def factor(A: sp.csr_matrix, p, orientation: str = "columns") -> IluFactors:
    """The iLUTP(d, p, permtol) of L~_RCM: column-oriented (the reading R16, default) or
    row-oriented (R13; kept for the study of DESIGN.md R16)."""
    if orientation == "columns":
        return ilutp_columns(A, p.drop_tol, p.fill_factor, p.permtol)
    if orientation == "rows":
        return ilutp(A, p.drop_tol, p.fill_factor, p.permtol)
    raise ValueError(f"orientation must be 'columns' or 'rows', not {orientation!r}")


def solve_iterative(p, use_c_rcm: bool = True, orientation: str = "columns") -> IterativeResult:
    t0 = time.perf_counter()
    Lt, rhs, w, L = lv.constrained_system(p)
    t1 = time.perf_counter()
    perm = order(Lt, use_c=use_c_rcm)
    A = rcm_py.permute(Lt, perm)
    t2 = time.perf_counter()
    F = factor(A, p, orientation)
    t3 = time.perf_counter()
    res = gmres(lambda v: A @ v, lambda v: apply_preconditioner(F, v), rhs[perm], p.restart, p.tol,
                p.max_iter)
    t4 = time.perf_counter()
    x = np.empty_like(res.x)
    x[perm] = res.x
    return IterativeResult(normalise(x, p.hilbert_dim), x, perm, F, res,
                           dict(build=t1 - t0, rcm=t2 - t1, ilut=t3 - t2, gmres=t4 - t3))


def fock_numbers(p):
    i = np.arange(p.hilbert_dim)
    return i // p.N_m, i % p.N_m          # c(i), m(i)


def expect(rho: np.ndarray, p) -> tuple[float, float]:
    """(<a^+a>, <b^+b>) = (Tr rho a^+a, Tr rho b^+b)."""
    c, m = fock_numbers(p)
    d = np.real(np.diag(rho))
    return float(d @ c), float(d @ m)


def liouvillian_residual(rho: np.ndarray, p, L: sp.csr_matrix | None = None, w: complex | None = None) -> float:
    """||L vec(rho)||_2 / ||b||_2 with ||b|| = |w| (north-star residual)."""
    if L is None or w is None:
        _, _, w, L = lv.constrained_system(p)
    return float(np.linalg.norm(L @ lv.vec(rho)) / abs(w))
