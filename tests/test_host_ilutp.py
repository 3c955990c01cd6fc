"""The product's multi-threaded iLUTP (csrc/ilut.cpp, through the host-only C-ABI call
ss_ilutp_host) against the oracle's serial iLUTP (oracle/ilut.c), on CPU.

PAPER.md:94 (sec. II, "iLUTP"), rules R4-R7, R13 of DESIGN.md.  The threaded code must be
bit-identical to the serial algorithm for every thread count: the frontier pipeline, the
position bitmap, the U-candidate snapshot and the column exchanges are host logic, so
they are covered here without a GPU (the GPU suite checks the same factors after
ss_setup).  Column exchanges are forced with permtol 0.3-1.0 (hundreds of exchanges), and
the multi-threaded cases are repeated to give races a chance to show.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import ilut as I
from oracle import liouvillian as lv
from oracle import rcm as R
from oracle import steadystate as ss
from workloads import CONFIGS, tiny_params


def pb():
    import paper_1411_4356_b200 as m
    return m


def rcm_matrix(p):
    Lt, _, _, _ = lv.constrained_system(p)
    A = R.permute(Lt, ss.rcm_c(R.symmetrized_pattern(Lt))).tocsr()
    A.sort_indices()
    return A


def random_banded(n, bw, density, seed):
    """Random complex matrix with a dominant-ish diagonal inside a band (plus a few
    far entries), a general stand-in for the Liouvillian's RCM profile."""
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for i in range(n):
        k = max(1, int(density * 2 * bw))
        c = rng.integers(max(0, i - bw), min(n, i + bw + 1), size=k)
        rows += [i] * len(c)
        cols += list(c)
    far = rng.integers(0, n, size=(n // 10, 2))
    rows += list(far[:, 0])
    cols += list(far[:, 1])
    rows += list(range(n))
    cols += list(range(n))
    v = rng.normal(size=len(rows)) + 1j * rng.normal(size=len(rows))
    A = sp.csr_matrix((v, (rows, cols)), shape=(n, n))
    A.sum_duplicates()
    A.sort_indices()
    return A


def check(A, d, p, permtol, threads, F=None):
    F = F if F is not None else I.ilutp(A, d, p, permtol)
    (Lp, Lj, Lx), (Up, Uj, Ux), cp = pb().ss_ilutp_host(A.indptr, A.indices, A.data, d, p, permtol, threads)
    assert np.array_equal(cp, F.perm if F.perm is not None else np.arange(A.shape[0]))
    assert np.array_equal(Lp, F.Lp) and np.array_equal(Lj, F.Lj) and np.array_equal(Lx, F.Lx)
    assert np.array_equal(Up, F.Up) and np.array_equal(Uj, F.Uj) and np.array_equal(Ux, F.Ux)
    return F


@pytest.mark.parametrize("name", ["tiny", "ragged", "nth0", "Nc1"])
@pytest.mark.parametrize("threads", [1, 2, 5])
def test_liouvillian_bit_exact(name, threads):
    p = CONFIGS["tiny"] if name == "tiny" else {
        "ragged": tiny_params(7, 13, Delta=0.37, g0=0.55),
        "nth0": tiny_params(3, 7, n_th=0.0),
        "Nc1": tiny_params(1, 6)}[name]
    check(rcm_matrix(p), p.drop_tol, p.fill_factor, p.permtol, threads)


@pytest.mark.parametrize("permtol", [0.3, 1.0])
def test_column_exchanges_every_thread_count(permtol):
    p = CONFIGS["tiny"]
    A = rcm_matrix(p)
    F = I.ilutp(A, p.drop_tol, p.fill_factor, permtol)
    assert F.perm is not None and np.count_nonzero(F.perm != np.arange(A.shape[0])) > 50
    for threads in (1, 2, 3, 4, 8, 8, 8, 16):
        check(A, p.drop_tol, p.fill_factor, permtol, threads, F)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_banded_bit_exact(seed):
    A = random_banded(1500, 40, 0.15, seed)
    for d, p, permtol in ((1e-3, 10, 0.0), (1e-4, 20, 0.5), (0.0, 1000, 0.1)):
        F = I.ilutp(A, d, p, permtol)
        for threads in (1, 4, 7):
            check(A, d, p, permtol, threads, F)


def test_small_config_many_threads():
    """configs[1] (n = 32,400, 7.4 M factor entries) with forced exchanges, 8 threads."""
    p = CONFIGS["small"]
    A = rcm_matrix(p)
    check(A, p.drop_tol, p.fill_factor, 0.5, 8)


def test_errors():
    p = CONFIGS["tiny"]
    A = rcm_matrix(p)
    m = pb()
    n = A.shape[0]
    rp, ci, va = A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data.astype(np.complex128)
    bufs = [np.empty(n + 1, np.int64), np.empty(1, np.int64), np.empty(1, np.complex128),
            np.empty(n + 1, np.int64), np.empty(1, np.int64), np.empty(1, np.complex128), np.empty(n, np.int64)]
    with pytest.raises(m.SSError) as e:   # caps too small
        m._lib._check(m._lib.load().ss_ilutp_host(
            n, rp.ctypes.data, ci.ctypes.data, va.ctypes.data, 1e-4, 20.0, 0.01, 2, bufs[0].ctypes.data,
            bufs[1].ctypes.data, bufs[2].ctypes.data, 1, bufs[3].ctypes.data, bufs[4].ctypes.data,
            bufs[5].ctypes.data, 1, bufs[6].ctypes.data))
    assert e.value.code == 1 and "need L_cap" in str(e.value)
    bad = A.copy()
    bad.indices[1] = bad.indices[0]   # duplicate column in row 0
    with pytest.raises(m.SSError) as e:
        m.ss_ilutp_host(bad.indptr, bad.indices, bad.data, 1e-4, 20, 0.01)
    assert e.value.code == 1
    with pytest.raises(m.SSError) as e:   # zero row, d = 0: zero pivot cannot be repaired
        Z = sp.csr_matrix((np.ones(2, np.complex128), [0, 2], [0, 1, 1, 2]), shape=(3, 3))
        m.ss_ilutp_host(Z.indptr, Z.indices, Z.data, 0.0, 10, 0.0)
    assert e.value.code == 4


@pytest.mark.parametrize("threads", [1, 8])
def test_breakdown_with_later_rows_referencing_drained_rows(threads):
    """d = 0 and a zero pivot at row 1 (rows 0 and 1 equal); rows 2, 3 reference the
    rows before them.  The oracle reports the zero pivot; the threaded code must return
    SS_ERR_BREAKDOWN (never eliminate against a row drained after the breakdown)."""
    m = pb()
    A = sp.csr_matrix(np.array([[1, 1, 0, 0], [1, 1, 0, 0], [0, 1, 1, 0], [0, 0, 1, 1]], np.complex128))
    with pytest.raises(RuntimeError, match="zero pivot at row 1"):
        I.ilutp(A, 0.0, 10, 0.0)
    for _ in range(5):
        with pytest.raises(m.SSError) as e:
            m.ss_ilutp_host(A.indptr, A.indices, A.data, 0.0, 10, 0.0, threads=threads)
        assert e.value.code == 4
