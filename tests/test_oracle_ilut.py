"""Oracle pins for the dual-threshold ILU (sec. II) and the condition estimate (sec. IV)."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import ilut as I
from oracle import trisolve as T


def rand_dd(n, density, seed, complex_=True):
    rng = np.random.default_rng(seed)
    A = sp.random(n, n, density=density, random_state=seed, format="csr")
    if complex_:
        B = sp.random(n, n, density=density, random_state=seed + 100, format="csr")
        A = A + 1j * B
    A = A + sp.diags(4.0 + rng.random(n) + 1j * rng.random(n))
    A = sp.csr_matrix(A)
    A.sort_indices()
    return A


def full_LU(F):
    L = (F.L() + sp.identity(F.n)).toarray()
    U = F.U().toarray()
    return L, U


@pytest.mark.parametrize("seed", [0, 1])
def test_d0_unbounded_fill_is_complete_lu(seed):
    """'In the limit where d=0, the iLU preconditioner returns the complete LU factorization'.
    A unit-lower/upper LU without pivoting is unique, so L U = A pins every entry."""
    A = rand_dd(40, 0.1, seed)
    F = I.ilut(A, 0.0, 1e9)
    L, U = full_LU(F)
    assert np.allclose(np.tril(L, -1), L - np.eye(40)) and np.allclose(np.triu(U), U)
    assert np.abs(L @ U - A.toarray()).max() <= 1e-12 * np.abs(A).max()
    x = np.random.default_rng(seed).standard_normal(40) + 0j
    assert np.abs(T.apply_preconditioner(F, A @ x, small_loops=True) - x).max() < 1e-12


def test_identity():
    F = I.ilut(sp.identity(5, dtype=complex, format="csr"), 1e-3, 10)
    assert F.Lj.size == 0 and np.array_equal(F.Uj, np.arange(5)) and np.allclose(F.Ux, 1)


def test_lower_triangular_input_is_exact():
    """ILUT of a lower-triangular matrix with no fill: l_ij = a_ij / a_jj, U = diag(A) (for d = 0)."""
    A = sp.csr_matrix(np.array([[2, 0, 0], [1, 4, 0], [0, 3, 5.0]], dtype=complex))
    F = I.ilut(A, 0.0, 100)
    L, U = full_LU(F)
    assert np.allclose(L, [[1, 0, 0], [0.5, 1, 0], [0, 0.75, 1]]) and np.allclose(U, np.diag([2, 4, 5]))


def test_tridiagonal_no_fill():
    n = 12
    A = sp.diags([np.full(n - 1, 1.0), np.full(n, 4.0), np.full(n - 1, 1.0 + 1j)], [-1, 0, 1], format="csr",
                 dtype=complex)
    F = I.ilut(A, 1e-12, 10)
    assert F.nnz == A.nnz
    L, U = full_LU(F)
    assert np.abs(L @ U - A.toarray()).max() < 1e-14


def test_hand_worked_drop():
    """3x3 with d = 0.01 (worked by hand, R4-R5):
    row 2: multiplier 0.001/4 = 2.5e-4 < 0.01*4 -> dropped, no update; multiplier 1/3.75 kept."""
    A = sp.csr_matrix(np.array([[4, 1, 0], [1, 4, 1], [0.001, 1, 4]], dtype=complex))
    F = I.ilut(A, 0.01, 100)
    L, U = full_LU(F)
    u11 = 4 - 0.25
    l21 = 1.0 / u11
    assert np.allclose(L, [[1, 0, 0], [0.25, 1, 0], [0, l21, 1]], rtol=0, atol=1e-15)
    assert np.allclose(U, [[4, 1, 0], [0, u11, 1], [0, 0, 4 - l21]], rtol=0, atol=1e-15)
    # the complete factorisation keeps the small multiplier
    Fe = I.ilut(A, 0.0, 100)
    assert abs(full_LU(Fe)[0][2, 0] - 0.001 / 4) < 1e-18


def test_fill_cap_keeps_largest():
    """p caps each part of a row at floor(p nnz(a_i) / 2) entries, the largest |.|."""
    n = 6
    dense = np.eye(n, dtype=complex) * 10
    dense[5, :5] = [1, 5, 2, 4, 3]          # L part of row 5 (no fill from rows 0-4: they are diagonal)
    dense[0, 1:] = [3, 1, 4, 1, 5]          # U part of row 0
    A = sp.csr_matrix(dense)
    F = I.ilut(A, 0.0, 0.7)                 # row 5: nnz 6 -> lfil = floor(0.7*6/2) = 2
    L = F.L().toarray()
    assert np.count_nonzero(L[5]) == 2 and set(np.nonzero(L[5])[0]) == {1, 3}
    U = F.U().toarray()
    assert set(np.nonzero(U[0, 1:])[0] + 1) == {3, 5} and U[0, 0] == 10


def test_drop_rule_and_cap_on_random():
    A = rand_dd(200, 0.05, 3)
    d, p = 0.05, 3.0
    F = I.ilut(A, d, p)
    rowmax = abs(A).max(axis=1).toarray().ravel()
    nnz_row = np.diff(A.indptr)
    for i in range(200):
        lv = F.Lx[F.Lp[i]:F.Lp[i + 1]]
        uv = F.Ux[F.Up[i] + 1:F.Up[i + 1]]
        lfil = int(p * nnz_row[i] / 2)
        assert len(lv) <= lfil and len(uv) <= lfil
        assert np.all(np.abs(lv) >= d * rowmax[i] * (1 - 1e-15))
        assert np.all(np.abs(uv) >= d * rowmax[i] * (1 - 1e-15))
    assert F.nnz <= p * A.nnz + 200


def test_zero_pivot_repair_and_error():
    A = sp.csr_matrix(np.array([[1, 1], [1, 1.0]], dtype=complex))
    F = I.ilut(A, 0.1, 10)
    assert F.diag()[1] == 0.1
    with pytest.raises(RuntimeError):
        I.ilut(A, 0.0, 10)


def test_condest():
    """condition estimate ||M e||_inf (reading R8: (LU)^{-1} e)."""
    F = I.ilut(sp.identity(4, dtype=complex, format="csr"), 0.0, 10)
    assert I.condest(F) == 1.0
    F = I.ilut(sp.diags([1.0, 1e-8]).tocsr().astype(complex), 0.0, 10)
    assert abs(I.condest(F) - 1e8) < 1e-6


def test_triangular_solves_against_dense():
    A = rand_dd(60, 0.1, 11)
    F = I.ilut(A, 1e-3, 5)
    L, U = full_LU(F)
    b = np.random.default_rng(2).standard_normal(60) + 1j
    ref = np.linalg.solve(U, np.linalg.solve(L, b))
    assert np.abs(T.apply_preconditioner(F, b, small_loops=True) - ref).max() < 1e-11
    assert np.abs(T.apply_preconditioner(F, b) - ref).max() < 1e-11


# ---------------------------------------------------------------- iLUTP (reading R13)
def random_sparse(rng, n, density):
    """Random complex sparse matrix, far from diagonally dominant (a scaled random
    permutation is added so that it is nonsingular and pivoting is needed)."""
    seed = int(rng.integers(1 << 30))
    A = sp.random(n, n, density=density, random_state=seed, format="csr")
    A = A + 1j * sp.random(n, n, density=density, random_state=seed + 1, format="csr")
    perm = rng.permutation(n)
    A = A + sp.csr_matrix((3.0 + rng.random(n), (np.arange(n), perm)), shape=(n, n))
    A = sp.csr_matrix(A)
    A.sort_indices()
    return A


def test_ilutp_permtol0_is_ilut():
    """permtol = 0 never exchanges columns: bit-identical to ilut (two code paths), and
    both raise on the same unrecoverable zero pivot."""
    rng = np.random.default_rng(3)
    for seed in range(3):
        for A in (rand_dd(60, 0.15, seed), random_sparse(rng, 60, 0.15)):
            for d, p in ((0.0, 1e9), (0.05, 3), (1e-3, 10)):
                try:
                    F0 = I.ilut(A, d, p)
                except RuntimeError:
                    with pytest.raises(RuntimeError):
                        I.ilutp(A, d, p, 0.0)
                    continue
                F1 = I.ilutp(A, d, p, 0.0)
                assert np.array_equal(F1.perm, np.arange(60))
                for k in ("Lp", "Lj", "Lx", "Up", "Uj", "Ux"):
                    assert np.array_equal(getattr(F0, k), getattr(F1, k))


def test_ilutp_complete_lu_with_column_pivoting():
    """d = 0 and unbounded fill: complete LU of A[:, perm] (Saad's ILUTP with no dropping)."""
    rng = np.random.default_rng(4)
    for seed in range(3):
        A = random_sparse(rng, 40, 0.2)
        F = I.ilutp(A, 0.0, 1e9, 0.5)
        Lm = (F.L() + sp.identity(40)).toarray()
        assert np.abs(Lm @ F.U().toarray() - A.toarray()[:, F.perm]).max() <= 1e-10 * np.abs(A.toarray()).max()
        assert sorted(F.perm.tolist()) == list(range(40))
        # pivot rule: after the exchange every diagonal is >= permtol * the largest entry of its U row
        U = F.U().toarray()
        for i in range(40):
            assert abs(U[i, i]) >= 0.5 * np.abs(U[i, i:]).max() * (1 - 1e-12)


def test_ilutp_factors_zero_diagonal():
    """[[0, 2], [3, 0]]: ILUT meets an exactly zero pivot (error with d = 0); ILUTP
    exchanges the columns: A[:, [1, 0]] = I * diag(2, 3)."""
    A = sp.csr_matrix(np.array([[0, 2], [3, 0]], dtype=complex))
    with pytest.raises(RuntimeError):
        I.ilut(A, 0.0, 10)
    F = I.ilutp(A, 0.0, 10, 0.5)
    assert F.perm.tolist() == [1, 0]
    assert np.array_equal(F.U().toarray(), np.array([[2, 0], [0, 3]], dtype=complex))
    assert F.L().nnz == 0


def test_ilutp_hand_worked_exchange():
    """3x3 by hand, permtol = 0.5, d = 0:
    A = [[1, 4, 0], [2, 1, 1], [0, 1, 3]]
    row 0: U part (1, 4, 0); 0.5*4 > 1 -> exchange columns 0 and 1 (perm = [1, 0, 2]);
           U row 0 = (4 | 1, 0) in positions (0 | 1, 2).
    row 1 in positions: (a11, a10, a12) = (1, 2, 1); l = 1/4; w = (2 - 1/4, 1 - 0) = (1.75, 1);
           0.5*1 < 1.75 -> no exchange.  U row 1 = (1.75 | 1).
    row 2: positions (1, 0, 3); l20 = 1/4; w1 = 0 - 1/4*1 = -0.25, w2 = 3;
           l21 = -0.25/1.75 = -1/7; w2 = 3 - (-1/7)*1 = 22/7."""
    A = sp.csr_matrix(np.array([[1, 4, 0], [2, 1, 1], [0, 1, 3]], dtype=complex))
    F = I.ilutp(A, 0.0, 100, 0.5)
    assert F.perm.tolist() == [1, 0, 2]
    U = F.U().toarray()
    assert np.allclose(U, [[4, 1, 0], [0, 1.75, 1], [0, 0, 22 / 7]], rtol=0, atol=1e-15)
    Lm = F.L().toarray()
    assert np.allclose(Lm, [[0, 0, 0], [0.25, 0, 0], [0.25, -1 / 7, 0]], rtol=0, atol=1e-15)


def perm_matrix(perm):
    """Pi with B Pi = B[:, perm]: Pi[perm[j], j] = 1 (built from the definition)."""
    n = len(perm)
    P = np.zeros((n, n))
    P[perm, np.arange(n)] = 1.0
    return P


def cycle_lengths(perm):
    seen, out = set(), []
    for s in range(len(perm)):
        if s in seen:
            continue
        k, c = s, 0
        while k not in seen:
            seen.add(k)
            k = perm[k]
            c += 1
        out.append(c)
    return out


def small_diagonal(n, seed):
    """Dense-ish complex matrix with a tiny diagonal: iLUTP must exchange at most rows,
    and the exchanges compose into permutation cycles longer than 2."""
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    M[rng.random((n, n)) < 0.4] = 0.0
    np.fill_diagonal(M, 1e-3 * (1 + rng.random(n)))
    A = sp.csr_matrix(M)
    A.sort_indices()
    return A


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_row_ilutp_unpivot_with_long_cycles(seed):
    """Pins the Pi of M^{-1} = Pi U^{-1} L^{-1} (row-wise iLUTP, R13): with d = 0 and
    unbounded fill the factors are complete, so M^{-1} (A x) = x for every x -- only if
    Pi (not Pi^{-1}) is applied, which differs once perm has a cycle longer than 2."""
    A = small_diagonal(24, seed)
    F = I.ilutp(A, 0.0, 1e9, 0.5)
    assert max(cycle_lengths(F.perm)) > 2
    Ad = A.toarray()
    Lm = (F.L() + sp.identity(24)).toarray()
    assert np.abs(Lm @ F.U().toarray() - Ad @ perm_matrix(F.perm)).max() <= 1e-9 * np.abs(Ad).max()
    x = np.random.default_rng(seed + 7).standard_normal(24) + 1j
    for loops in (True, False):
        assert np.abs(T.apply_preconditioner(F, Ad @ x, small_loops=loops) - x).max() <= 1e-9 * np.abs(x).max()
    y = T.backward(F, T.forward(F, Ad @ x))
    right = np.empty(24, complex)
    right[F.perm] = y                    # x = Pi y: x[perm[p]] = y[p]
    assert np.abs(right - x).max() <= 1e-9 * np.abs(x).max()
    wrong = y[F.perm]                    # Pi^{-1} y instead
    assert np.abs(wrong - x).max() > 1e-3


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_column_ilutp_complete_with_long_cycles(seed):
    """Column-oriented iLUTP (R16): A^T Pi = L U, hence A = Pi U^T L^T; with d = 0 and
    unbounded fill this is exact, so M^{-1} (A x) = L^{-T} U^{-T} Pi^T A x = x (textbook
    column-sweep loops and library triangular solves), and the pivot rule holds along the
    COLUMNS of A (every pivot >= permtol times the largest entry of its column of the
    lower factor)."""
    A = small_diagonal(24, seed)
    F = I.ilutp_columns(A, 0.0, 1e9, 0.5)
    assert F.columns and max(cycle_lengths(F.perm)) > 2
    Ad = A.toarray()
    Lm = (F.L() + sp.identity(24)).toarray()
    U = F.U().toarray()
    assert np.abs(perm_matrix(F.perm) @ U.T @ Lm.T - Ad).max() <= 1e-9 * np.abs(Ad).max()
    lower = U.T   # the factor of A that carries the pivots
    for j in range(24):
        assert abs(lower[j, j]) >= 0.5 * np.abs(lower[j:, j]).max() * (1 - 1e-12)
    x = np.random.default_rng(seed + 9).standard_normal(24) + 1j
    for loops in (True, False):
        assert np.abs(T.apply_preconditioner(F, Ad @ x, small_loops=loops) - x).max() <= 1e-9 * np.abs(x).max()


def test_column_ilutp_hand_worked_drop():
    """Column orientation, by hand: A = [[4, 1, 0.001], [1, 4, 1], [0, 1, 4]], d = 0.01.
    Column 0 = (4, 1, 0): pivot 4, no exchange (permtol 0.01).  Column 1 = (1, 4, 1): its
    entry above the diagonal gives the multiplier 1/4 (kept), then 4 - 1/4 = 3.75.
    Column 2 = (0.001, 1, 4), threshold 0.01 * ||A[:, 2]||_inf = 0.04: the multiplier
    0.001/4 = 2.5e-4 is dropped (no update), 1/3.75 is kept, pivot 4 - 1/3.75.
    (The multipliers land in the unit UPPER factor of A: the column orientation.)
    """
    A = sp.csr_matrix(np.array([[4, 1, 0.001], [1, 4, 1], [0, 1, 4]], dtype=complex))
    F = I.ilutp_columns(A, 0.01, 100, 0.01)
    assert F.perm.tolist() == [0, 1, 2]
    u11 = 4 - 0.25
    lower = F.U().toarray().T            # lower factor of A, pivots on the diagonal
    upper = (F.L() + sp.identity(3)).toarray().T   # unit upper factor of A
    assert np.allclose(upper, [[1, 0.25, 0], [0, 1, 1 / u11], [0, 0, 1]], rtol=0, atol=1e-15)
    assert np.allclose(lower, [[4, 0, 0], [1, u11, 0], [0, 1, 4 - 1 / u11]], rtol=0, atol=1e-15)
