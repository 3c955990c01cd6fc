"""Oracle: restarted GMRES(m) with left preconditioning (sec. IV, Eq. (8)).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:126: "we perform preconditioned iterations using the Restarted
Generalized Minimum Residual (GMRES) solver [saad:1986] ... we restart the
algorithm after 10 steps" (the BASELINE configs fix m = 30/40/50 instead).
Eq. (8): left preconditioning, M^{-1} L~ x = M^{-1} b.

Written as in Saad & Schultz (1986) / Saad (2003) Alg. 6.9-6.11: Arnoldi with
modified Gram-Schmidt, complex Givens rotations on the Hessenberg matrix, a
triangular solve for y and x <- x + V_k y at the end of each cycle.

Stopping rule (R9): at the start of cycle c the true residual
r_c = b - A x_c is formed; the run has converged when ||r_c||/||b|| <= tol.
Otherwise z = M^{-1} r_c, beta = ||z||, and the cycle's inner loop stops early
once the preconditioned residual estimate |g_{j+1}| <= beta * tol ||b|| / ||r_c||
(the same relative reduction the true residual still needs), or after m steps.
``iterations`` counts Arnoldi steps (applications of M^{-1} A).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class GmresResult:
    x: np.ndarray
    iterations: int
    converged: bool
    rel_residual: float                      # true ||b - A x|| / ||b||
    history: list = field(default_factory=list)   # true relative residual per cycle start


def givens(a: complex, b: complex):
    """(c, s, r) with c real, [[c, s], [-conj(s), c]] @ [a, b] = [r, 0]."""
    aa, bb = abs(a), abs(b)
    if bb == 0.0:
        return 1.0, 0.0 + 0.0j, a
    if aa == 0.0:
        return 0.0, 1.0 + 0.0j, b
    nu = np.sqrt(aa * aa + bb * bb)
    ph = a / aa
    return aa / nu, ph * np.conj(b) / nu, ph * nu


def gmres(A_mv, M_solve, b: np.ndarray, m: int, tol: float, max_iter: int,
          x0: np.ndarray | None = None) -> GmresResult:
    n = b.shape[0]
    x = np.zeros(n, dtype=np.complex128) if x0 is None else np.array(x0, dtype=np.complex128)
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return GmresResult(np.zeros(n, dtype=np.complex128), 0, True, 0.0, [0.0])
    total = 0
    hist = []
    while True:
        r = b - A_mv(x)
        rn = np.linalg.norm(r)
        rel = rn / bnorm
        hist.append(rel)
        if rel <= tol:
            return GmresResult(x, total, True, rel, hist)
        if total >= max_iter:
            return GmresResult(x, total, False, rel, hist)
        z = M_solve(r)
        beta = np.linalg.norm(z)
        target = beta * tol * bnorm / rn
        V = np.zeros((m + 1, n), dtype=np.complex128)
        H = np.zeros((m + 1, m), dtype=np.complex128)
        cs = np.zeros(m)
        sn = np.zeros(m, dtype=np.complex128)
        g = np.zeros(m + 1, dtype=np.complex128)
        g[0] = beta
        V[0] = z / beta
        k = 0
        for j in range(m):
            w = M_solve(A_mv(V[j]))
            total += 1
            for i in range(j + 1):                      # modified Gram-Schmidt
                H[i, j] = np.vdot(V[i], w)
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] != 0.0:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):                          # previous rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -np.conj(sn[i]) * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            c, s, rr = givens(H[j, j], H[j + 1, j])
            cs[j], sn[j] = c, s
            H[j, j], H[j + 1, j] = rr, 0.0
            g[j + 1] = -np.conj(s) * g[j]
            g[j] = c * g[j]
            k = j + 1
            if abs(g[j + 1]) <= target or total >= max_iter or H[j, j] == 0.0:
                break
        y = np.zeros(k, dtype=np.complex128)
        for i in range(k - 1, -1, -1):                  # back substitution H y = g
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        x = x + V[:k].T @ y
