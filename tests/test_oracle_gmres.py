"""Oracle pins for restarted GMRES(m) (sec. IV) and the end-to-end oracle pipeline."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import gmres as G
from oracle import ilut as I
from oracle import steadystate as ss
from oracle import trisolve as T
from workloads import CONFIGS, rand_cvec


def test_identity_one_step():
    b = rand_cvec(50, 1)
    r = G.gmres(lambda v: v, lambda v: v, b, 10, 1e-12, 100)
    assert r.converged and r.iterations == 1 and np.allclose(r.x, b, atol=1e-14)


def test_exact_preconditioner_converges_in_one_step():
    """With d = 0 the ILU is the complete LU, so M^{-1} A = I: one Arnoldi step."""
    n = 80
    rng = np.random.default_rng(4)
    A = sp.random(n, n, density=0.08, random_state=4, format="csr") + sp.diags(5 + rng.random(n))
    A = sp.csr_matrix(A, dtype=complex)
    F = I.ilut(A, 0.0, 1e9)
    b = rand_cvec(n, 5)
    r = G.gmres(lambda v: A @ v, lambda v: T.apply_preconditioner(F, v), b, 20, 1e-13, 50)
    assert r.converged and r.iterations == 1
    assert np.abs(r.x - np.linalg.solve(A.toarray(), b)).max() < 1e-11


def test_unpreconditioned_matches_dense_solve_and_finite_termination():
    """Full GMRES (m >= n) terminates in at most n steps in exact arithmetic (Saad-Schultz)."""
    n = 30
    rng = np.random.default_rng(8)
    A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) + 6 * np.eye(n)
    b = rand_cvec(n, 9)
    r = G.gmres(lambda v: A @ v, lambda v: v, b, n, 1e-12, 10 * n)
    assert r.converged and r.iterations <= n
    assert np.abs(r.x - np.linalg.solve(A, b)).max() < 1e-10


def test_restarted_residual_history_non_increasing():
    n = 200
    rng = np.random.default_rng(3)
    A = sp.random(n, n, density=0.05, random_state=3, format="csr") + sp.diags(4 + rng.random(n) + 1j)
    A = sp.csr_matrix(A, dtype=complex)
    b = rand_cvec(n, 3)
    r = G.gmres(lambda v: A @ v, lambda v: v, b, 5, 1e-10, 2000)
    h = np.array(r.history)
    assert r.converged and np.all(h[1:] <= h[:-1] * (1 + 1e-12))
    assert np.linalg.norm(A @ r.x - b) / np.linalg.norm(b) <= 1e-10


def test_givens_rotation():
    for a, b in [(1 + 2j, 3.0 + 0j), (0j, 2.0 + 0j), (1.5 - 1j, 0j)]:
        c, s, r = G.givens(a, b)
        M = np.array([[c, s], [-np.conj(s), c]])
        out = M @ np.array([a, b])
        assert abs(out[1]) < 1e-15 and abs(out[0] - r) < 1e-15 and abs(abs(c) ** 2 + abs(s) ** 2 - 1) < 1e-15


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_iterative_pipeline_equals_direct(name):
    """The paper's pipeline (RCM + ILUT + GMRES) reaches the Eq. (5) solution."""
    p = CONFIGS[name]
    it = ss.solve_iterative(p)
    d = ss.solve_direct(p)
    assert it.gmres.converged and it.gmres.rel_residual <= p.tol
    assert np.abs(it.rho - d).sum() < 1e-6
    assert ss.liouvillian_residual(it.rho, p) < 1e-9
    assert abs(np.trace(it.rho) - 1) < 1e-12
