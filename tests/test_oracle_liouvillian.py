"""Oracle pins: Hamiltonian, Liouvillian, trace-constrained system (Eqs. (1), (3), (5)).

Each test pins oracle/liouvillian.py to something other than itself: the paper's
printed NNZ (Fig. 1), an independent dense construction that applies Eq. (3) to
basis matrices (oracle/superop_dense.py), closed forms and invariants.
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import liouvillian as lv
from oracle import superop_dense as sd
from workloads import CONFIGS, tiny_params

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_destroy_matrix_elements():
    a = lv.destroy(4).toarray()
    ref = np.zeros((4, 4))
    ref[0, 1], ref[1, 2], ref[2, 3] = 1.0, np.sqrt(2), np.sqrt(3)
    assert np.array_equal(a, ref)
    n = (a.conj().T @ a).real
    assert np.allclose(np.diag(n), [0, 1, 2, 3], atol=1e-15) and np.count_nonzero(n - np.diag(np.diag(n))) == 0


def test_fig1_nnz_golden():
    """PAPER.md:90 (Fig. 1 caption): N_c=4, N_m=8, thermal bath, all terms present -> NNZ(L~) = 8957."""
    g = json.load(open(os.path.join(GOLD, "fig1_structure.json")))
    p = tiny_params(g["N_c"], g["N_m"], n_th=0.5)
    Lt, _, _, _ = lv.constrained_system(p)
    assert Lt.nnz == g["nnz_Ltilde"]


def test_nnz_drops_without_thermal_channel():
    """n_th = 0 removes the D[b^+] jump entries ('setting n_th to zero ... eliminating some elements')."""
    a, _, _, _ = lv.constrained_system(tiny_params(4, 8, n_th=0.5))
    b, _, _, _ = lv.constrained_system(tiny_params(4, 8, n_th=0.0))
    c, _, _, _ = lv.constrained_system(tiny_params(4, 8, n_th=1e-15))
    assert b.nnz < a.nnz and c.nnz == a.nnz


@pytest.mark.parametrize("Nc,Nm,kw", [(2, 3, {}), (3, 2, dict(Delta=0.7, n_th=2.0)),
                                      (2, 2, dict(g0=1.3, E=0.0)), (3, 3, dict(kappa=0.0, n_th=0.0))])
def test_kron_liouvillian_equals_superoperator_applied_to_basis(Nc, Nm, kw):
    """Column k + N l of the matrix must be vec(L[E_kl]) with L[.] evaluated literally (Eq. (3))."""
    p = tiny_params(Nc, Nm, **kw)
    L = lv.liouvillian(p).toarray()
    D = sd.dense_liouvillian(p)
    assert np.abs(L - D).max() <= 1e-13 * max(1.0, np.abs(D).max())


def test_hamiltonian_hermitian_and_uncoupled_diagonal():
    p = tiny_params(4, 5, g0=0.0, E=0.0, Delta=0.3)
    H = lv.hamiltonian(p)
    c = np.arange(20) // 5
    m = np.arange(20) % 5
    assert sp.csr_matrix(H - H.getH()).nnz == 0
    assert np.allclose(H.diagonal(), -0.3 * c + 1.0 * m, atol=1e-15)
    p2 = tiny_params(4, 5)
    H2 = lv.hamiltonian(p2)
    assert abs(H2 - H2.getH()).max() == 0.0


def test_two_level_decay_toy():
    """N_c = 2, N_m = 1, only kappa: L = [[0,0,0,k],[0,-k/2,0,0],[0,0,-k/2,0],[0,0,0,-k]] (vec column stacking)."""
    k = 0.7
    p = tiny_params(2, 1, kappa=k, g0=0.0, E=0.0, Delta=0.0, omega_m=0.0, Gamma_m=0.0, n_th=0.0)
    L = lv.liouvillian(p).toarray()
    ref = np.zeros((4, 4), complex)
    ref[0, 3] = k
    ref[1, 1] = ref[2, 2] = -k / 2
    ref[3, 3] = -k
    assert np.allclose(L, ref, atol=1e-15)


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_trace_preservation(name):
    """Lindblad generators preserve the trace: sum over diagonal rows of L vanishes."""
    p = CONFIGS[name]
    L = lv.liouvillian(p)
    N = p.hilbert_dim
    rows = np.arange(N) * (N + 1)
    s = np.asarray(L[rows].sum(axis=0)).ravel()
    assert np.abs(s).max() <= 1e-12 * abs(L).max()


def test_trace_matrix_structure():
    """Eq. (5): T has ones in row 0 at the diagonal-element columns, incl. the final column."""
    N = 7
    T = lv.trace_matrix(N)
    assert T.nnz == N
    r, c = T.nonzero()
    assert set(r) == {0} and sorted(c) == [k * (N + 1) for k in range(N)]
    assert (N * N - 1) in set(c)


@pytest.mark.parametrize("name", ["small", "medium"])
def test_trace_weight_closed_form(name):
    """mean(diag L) = -[kappa (N_c-1) + Gamma_m (1+2 n_th) (N_m-1)] / 2 (the -i[H,.] part is traceless on the diagonal)."""
    p = CONFIGS[name]
    L = lv.liouvillian(p)
    w = lv.trace_weight(L, p)
    ref = -(p.kappa * (p.N_c - 1) + p.Gamma_m * (1 + 2 * p.n_th) * (p.N_m - 1)) / 2
    assert abs(w.real - ref) <= 1e-13 * abs(ref) and abs(w.imag) <= 1e-15


def test_given_weight_and_rhs():
    p = CONFIGS["tiny"]
    Lt, rhs, w, L = lv.constrained_system(p)
    assert w == 1.0 and rhs[0] == w and np.count_nonzero(rhs) == 1
    D = (Lt - L).tocoo()
    assert set(D.row) == {0}
