"""Oracle pins for the steady state itself: closed forms, invariants, brute force.

North star: "the closed forms at g0=0 (cavity coherent state alpha = E/(Delta + i kappa/2),
mechanical thermal state with mean n_th); the invariants Tr rho = 1, rho = rho^+, rho >= 0;
brute-force dense null-space on tiny inputs".
"""
import numpy as np
import pytest

from oracle import liouvillian as lv
from oracle import steadystate as ss
from oracle import superop_dense as sd
from workloads import CONFIGS, tiny_params


def reduced(rho, p, keep):
    r = rho.reshape(p.N_c, p.N_m, p.N_c, p.N_m)
    return np.einsum("imjm->ij", r) if keep == "cav" else np.einsum("cicj->ij", r)


def test_coherent_cavity_state_at_g0_zero():
    """g0 = 0: cavity -> |alpha><alpha|, alpha = E / (Delta + i kappa/2) (d<a>/dt = 0 of Eq. (1)+(3))."""
    # N_c = 20: the truncation error ~ |alpha|^N_c / sqrt(N_c!) is ~1e-13 here
    p = tiny_params(20, 2, g0=0.0, E=0.4, Delta=-0.6, kappa=0.5, n_th=0.3)
    rho = ss.solve_direct(p)
    rc = reduced(rho, p, "cav")
    alpha = p.E / (p.Delta + 0.5j * p.kappa)
    a = lv.destroy(p.N_c).toarray()
    assert abs(np.trace(rc @ a) - alpha) < 1e-9
    assert abs(np.trace(rc @ a.conj().T @ a).real - abs(alpha) ** 2) < 1e-9
    # the state itself: truncated coherent state
    n = np.arange(p.N_c)
    from math import factorial
    psi = np.exp(-abs(alpha) ** 2 / 2) * alpha ** n / np.sqrt([float(factorial(k)) for k in n])
    assert np.abs(rc - np.outer(psi, psi.conj())).max() < 1e-9


@pytest.mark.parametrize("nth", [0.2, 1.0, 3.0])
def test_thermal_mechanics_closed_form(nth):
    """E = 0, g0 = 0: mechanics relaxes to the (truncated) Bose-Einstein state p_m ~ (n/(1+n))^m;
    detailed balance of the D[b], D[b^+] ladder holds exactly level by level."""
    p = tiny_params(2, 40, g0=0.0, E=0.0, n_th=nth, Gamma_m=0.01)
    rho = ss.solve_direct(p)
    rm = reduced(rho, p, "mech")
    r = nth / (1 + nth)
    pm = r ** np.arange(p.N_m)
    pm /= pm.sum()
    assert np.abs(np.diag(rm).real - pm).max() < 1e-10
    assert np.abs(rm - np.diag(np.diag(rm))).max() < 1e-12
    _, nb = ss.expect(rho, p)
    assert abs(nb - (np.arange(p.N_m) @ pm)) < 1e-9
    if nth <= 1.0:                  # (n/(1+n))^40 <= 1e-12: the truncation is invisible
        assert abs(nb - nth) < 1e-8


@pytest.mark.parametrize("Nc,Nm,kw", [(2, 3, {}), (3, 3, dict(n_th=0.0)), (2, 4, dict(g0=1.5, Delta=0.2))])
def test_direct_solve_equals_dense_nullspace(Nc, Nm, kw):
    """Eq. (4): rho_ss spans the null space of L; independent dense SVD vs the Eq. (5) solve."""
    p = tiny_params(Nc, Nm, **kw)
    rho_null, s = sd.nullspace_steady_state(p)
    assert s[-1] < 1e-10 * s[0] and s[-2] > 1e-8 * s[0]     # one-dimensional null space
    rho = ss.solve_direct(p)
    assert np.abs(rho - rho_null).sum() < 1e-9


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_invariants_direct(name):
    p = CONFIGS[name]
    rho = ss.solve_direct(p)
    assert abs(np.trace(rho) - 1) < 1e-13
    assert np.abs(rho - rho.conj().T).max() < 1e-10
    ev = np.linalg.eigvalsh(0.5 * (rho + rho.conj().T))
    assert ev.min() > -1e-10


def test_nth_1e15_equals_nth0():
    """n_th = 1e-15 keeps the thermal structure yet 'the calculated density matrix is
    numerically identical to the n_th=0 solution'."""
    p0 = tiny_params(3, 10, n_th=0.0)
    p1 = tiny_params(3, 10, n_th=1e-15)
    assert np.abs(ss.solve_direct(p0) - ss.solve_direct(p1)).max() < 1e-10
