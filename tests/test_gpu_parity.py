"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Bars: index work (structure, permutation, factor patterns)
bit-exact; assembled values and ILUT values bit-exact (same IEEE operations in the
same order, no FMA); SpMV / substitutions within a rounding-order tolerance; the
steady state within the north-star tolerances ||rho_gpu - rho_oracle||_1 <= 1e-6,
||L rho|| / ||b|| <= 1e-9, |Tr rho - 1| <= 1e-12.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import ilut as I
from oracle import liouvillian as lv
from oracle import rcm as R
from oracle import steadystate as ss
from oracle import trisolve as T
from workloads import CONFIGS, jittered, rand_cvec, tiny_params

pytestmark = pytest.mark.gpu


def pb():
    import paper_1411_4356_b200 as m
    return m


EDGE = {
    "Nc1": tiny_params(1, 6),                       # no cavity dynamics
    "Nm1": tiny_params(5, 1),                       # no mechanics
    "nth0": tiny_params(3, 7, n_th=0.0),            # D[b^+] absent
    "E0": tiny_params(3, 5, E=0.0),
    "g00": tiny_params(4, 5, g0=0.0),
    "Delta0": tiny_params(3, 6, Delta=0.0),
    "w_given": tiny_params(3, 4, w=2.5),
    "ragged": tiny_params(7, 13, Delta=0.37, g0=0.55),
}
BUILD_CASES = {**{k: CONFIGS[k] for k in ("tiny", "small")}, **EDGE,
               "jit1": jittered(CONFIGS["small"], 11), "jit2": jittered(CONFIGS["tiny"], 12)}


@pytest.mark.parametrize("name", list(BUILD_CASES))
def test_build_bit_exact(cuda, name):
    p = BUILD_CASES[name]
    s = pb().SteadyState(p)
    Lt, _, w, _ = lv.constrained_system(p)
    rp, ci, va = pb().ss_export_matrix(s.handle, 0)
    assert np.array_equal(rp, Lt.indptr) and np.array_equal(ci, Lt.indices)
    assert np.array_equal(va, Lt.data)                      # bit-exact values (+0/-0 compare equal)
    assert complex(s.build_info["w_re"], s.build_info["w_im"]) == w
    s.close()


@pytest.mark.parametrize("name", ["tiny", "small", "ragged", "nth0", "Nc1"])
def test_setup_bit_exact(cuda, name):
    p = {**CONFIGS, **EDGE}[name]
    s = pb().SteadyState(p).setup()
    Lt, _, _, _ = lv.constrained_system(p)
    perm = ss.rcm_c(R.symmetrized_pattern(Lt))
    assert np.array_equal(pb().ss_export_perm(s.handle), perm)
    if Lt.shape[0] <= 2000:
        assert np.array_equal(R.rcm(R.symmetrized_pattern(Lt)), perm)
    A = R.permute(Lt, perm)
    F = I.ilutp_columns(A, p.drop_tol, p.fill_factor, p.permtol)
    assert np.array_equal(pb().ss_export_colperm(s.handle), F.perm)
    # the operator of the hot path: L~_RCM with its rows in pivot order, A' = Pi^T L~_RCM
    Ar = sp.csr_matrix(A[F.perm])
    rp, ci, va = pb().ss_export_matrix(s.handle, 1)
    assert np.array_equal(rp, Ar.indptr) and np.array_equal(ci, Ar.indices) and np.array_equal(va, Ar.data)
    for which, (P_, J_, X_) in ((0, (F.Lp, F.Lj, F.Lx)), (1, (F.Up, F.Uj, F.Ux))):
        gp, gj, gx = pb().ss_export_factors(s.handle, which)
        assert np.array_equal(gp, P_) and np.array_equal(gj, J_)
        assert np.array_equal(gx, X_)
    assert s.setup_info["nnz_L"] + s.setup_info["nnz_U"] == F.nnz
    s.close()


@pytest.mark.parametrize("name,permtol,threads", [("tiny", 0.5, 0), ("small", 0.5, 1), ("small", 0.5, 5),
                                                   ("small", 0.01, 3)])
def test_setup_bit_exact_pivoting(cuda, name, permtol, threads):
    """Multi-threaded iLUTP (ilut.cpp) with many pivot exchanges (permtol 0.5) and odd
    thread counts: factors and permutation bit-identical to the serial oracle."""
    p = CONFIGS[name].with_(permtol=permtol)
    s = pb().SteadyState(p).setup(threads=threads)
    Lt, _, _, _ = lv.constrained_system(p)
    A = R.permute(Lt, ss.rcm_c(R.symmetrized_pattern(Lt)))
    F = I.ilutp_columns(A, p.drop_tol, p.fill_factor, p.permtol)
    if permtol >= 0.5:
        assert not np.array_equal(F.perm, np.arange(A.shape[0])) and s.setup_info["pivot_swaps"] > 0
    assert np.array_equal(pb().ss_export_colperm(s.handle), F.perm)
    for which, (P_, J_, X_) in ((0, (F.Lp, F.Lj, F.Lx)), (1, (F.Up, F.Uj, F.Ux))):
        gp, gj, gx = pb().ss_export_factors(s.handle, which)
        assert np.array_equal(gp, P_) and np.array_equal(gj, J_)
        assert np.array_equal(gx, X_)
    s.close()


def check_substitutions(s, F, x, torch, tol_tri=1e-11, tol_m=1e-10):
    """The two substitutions of M'^{-1} = L^{-T} U^{-T} (R16) and their product against
    scipy's triangular solves of the oracle's factors, and against the oracle's M^{-1}
    (which also gathers by Pi^T: M^{-1} v = M'^{-1} (Pi^T v))."""
    xd = torch.from_numpy(x).cuda()
    Ut = sp.csr_matrix(F.U().T)
    Lt = sp.csr_matrix(T.lower_unit_matrix(F).T)
    y1 = s.precond(xd, 0).cpu().numpy()
    r1 = sp.linalg.spsolve_triangular(Ut, x, lower=True)
    assert np.abs(y1 - r1).max() <= tol_tri * np.abs(r1).max()
    y2 = s.precond(xd, 1).cpu().numpy()
    r2 = sp.linalg.spsolve_triangular(Lt, x, lower=False, unit_diagonal=True)
    assert np.abs(y2 - r2).max() <= tol_tri * np.abs(r2).max()
    ym = s.precond(xd, 2).cpu().numpy()
    v = np.empty_like(x)
    v[F.perm] = x                                   # Pi^T v = x
    rm = T.apply_preconditioner(F, v)
    assert np.abs(ym - rm).max() <= tol_m * np.abs(rm).max()


@pytest.mark.parametrize("name,permtol", [("tiny", None), ("small", None), ("ragged", None), ("small", 0.5),
                                          ("ragged", 0.5)])
def test_spmv_and_substitutions(cuda, name, permtol):
    """permtol 0.5: hundreds of pivot exchanges, so Pi (as opposed to Pi^{-1} or no
    permutation) is exercised by the gathered operator and M^{-1}."""
    torch = cuda
    p = {**CONFIGS, **EDGE}[name]
    if permtol is not None:
        p = p.with_(permtol=permtol)
    s = pb().SteadyState(p).setup()
    Lt, _, _, _ = lv.constrained_system(p)
    perm = pb().ss_export_perm(s.handle)
    A = R.permute(Lt, perm)
    F = I.ilutp_columns(A, p.drop_tol, p.fill_factor, p.permtol)
    if permtol:
        assert s.setup_info["pivot_swaps"] > 20
    Ar = sp.csr_matrix(A[F.perm])
    n = A.shape[0]
    for seed in (1, 2):
        x = rand_cvec(n, seed)
        y = s.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
        ref = Ar @ x
        assert np.abs(y - ref).max() <= 1e-13 * np.abs(ref).max()
        check_substitutions(s, F, x, torch)
    s.close()


@pytest.mark.parametrize("knobs", [{"SSB_TRSV_Q": "4"}, {"SSB_TRSV_Q": "5"}, {"SSB_TRSV_Q": "9"}])
def test_substitution_split_variants(cuda, monkeypatch, knobs):
    """The same substitutions with the source-distance split moved:
    Q = 4 leaves the lieutenants' list B empty (everything beyond the dense G blocks goes
    to the helper CTAs), Q = 5 gives list B only its late part, Q = 9 a shorter window."""
    torch = cuda
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    p = CONFIGS["small"]
    s = pb().SteadyState(p).setup()
    Lt, _, _, _ = lv.constrained_system(p)
    A = R.permute(Lt, pb().ss_export_perm(s.handle))
    F = I.ilutp_columns(A, p.drop_tol, p.fill_factor, p.permtol)
    x = rand_cvec(A.shape[0], 5)
    for _ in range(2):   # relaunch: epochs advance
        check_substitutions(s, F, x, torch)
    assert max(s.setup_info["trsv_q_L"], s.setup_info["trsv_q_U"]) <= int(knobs["SSB_TRSV_Q"])
    s.close()


@pytest.mark.parametrize("name", ["tiny", "small", "ragged", "nth0", "g00", "w_given"])
def test_steady_state_parity(cuda, name):
    p = {**CONFIGS, **EDGE}[name]
    s = pb().SteadyState(p).setup().solve()
    info = s.solve_info
    assert info["converged"] == 1 and info["rel_residual"] <= p.tol
    rho = s.rho().cpu().numpy()
    ref = ss.solve_direct(p)
    assert np.abs(rho - ref).sum() <= 1e-6
    assert ss.liouvillian_residual(rho, p) <= 1e-9
    assert abs(np.trace(rho) - 1) <= 1e-12
    na, nb = s.expect()
    ra, rb = ss.expect(ref, p)
    # |<n> - <n>_ref| = |sum_i n_i (rho - ref)_ii| <= max(n_i) ||rho - ref||_1
    l1 = np.abs(rho - ref).sum()
    assert abs(na - ra) <= (p.N_c - 1) * l1 + 1e-14 and abs(nb - rb) <= (p.N_m - 1) * l1 + 1e-14
    # and, tighter than that bound, what both converged solutions give (measured ~1e-9)
    assert abs(na - ra) <= 1e-8 and abs(nb - rb) <= 1e-8
    # same algorithm as the oracle: iteration counts agree closely (CGS2 vs MGS rounding)
    it = ss.solve_iterative(p)
    assert abs(info["iterations"] - it.gmres.iterations) <= max(2, it.gmres.iterations // 10)
    s.close()


@pytest.mark.parametrize("restart", [5, 8])
def test_multi_cycle_gmres_parity(cuda, restart):
    """configs[1] with GMRES(5) / GMRES(8): several restart cycles, so the true-residual
    recompute at each cycle start, the x update across cycles and the step enqueued
    speculatively at a cycle boundary all run.  rho against the oracle's GMRES(m) and
    direct solve, iteration counts against the oracle's GMRES(m) (R9, R10)."""
    p = CONFIGS["small"].with_(restart=restart)
    s = pb().SteadyState(p).setup().solve()
    info = s.solve_info
    assert info["converged"] == 1 and info["rel_residual"] <= p.tol
    it = ss.solve_iterative(p)
    assert it.gmres.converged and len(it.gmres.history) >= 3          # >= 2 restarts
    assert info["iterations"] > restart
    assert abs(info["iterations"] - it.gmres.iterations) <= max(2, it.gmres.iterations // 10)
    rho = s.rho().cpu().numpy()
    assert np.abs(rho - it.rho).sum() <= 1e-6
    assert np.abs(rho - ss.solve_direct(p)).sum() <= 1e-6
    s.close()


def test_solve_host_e2e(cuda):
    p = CONFIGS["small"]
    s = pb().SteadyState(p).setup()
    n = s.n
    x = np.empty(n, np.complex128)
    info = pb().ss_solve_host(s.handle, None, x.ctypes.data, p.restart, p.tol, p.max_iter)
    assert info["converged"] == 1
    rho = lv.unvec(x, p.hilbert_dim)
    rho = rho / np.trace(rho)
    assert np.abs(rho - ss.solve_direct(p)).sum() <= 1e-6
    # arbitrary right-hand side through host buffers: L~ x = r
    Lt, _, _, _ = lv.constrained_system(p)
    r = rand_cvec(n, 5)
    info = pb().ss_solve_host(s.handle, r.ctypes.data, x.ctypes.data, 50, 1e-11, 3000)
    assert info["converged"] == 1
    assert np.linalg.norm(Lt @ x - r) / np.linalg.norm(r) <= 1e-11
    s.close()


def test_errors_are_reported(cuda):
    m = pb()
    h, _ = m.ss_build(CONFIGS["tiny"])
    with pytest.raises(m.SSError) as e:
        m.ss_solve(h, 30, 1e-10, 100)
    assert e.value.code == 5
    m.ss_setup(h, 1e-4, 20)
    with pytest.raises(m.SSError) as e:
        m.ss_solve(h, 0, 1e-10, 100)
    assert e.value.code == 1
    with pytest.raises(m.SSError):
        m.ss_setup(h, -1.0, 20)
    m.ss_destroy(h)
    bad = CONFIGS["tiny"].with_(kappa=-1.0)
    with pytest.raises(m.SSError) as e:
        m.ss_build(bad)
    assert e.value.code == 1


def test_zero_pivot_breakdown_reported(cuda):
    """d = 0 with an exactly singular pivot cannot be repaired (R6): SS_ERR_BREAKDOWN."""
    m = pb()
    p = tiny_params(1, 2, kappa=0.0, Gamma_m=0.0, n_th=0.0, g0=0.0, E=0.0, Delta=0.0, omega_m=0.0, w=1.0)
    h, _ = m.ss_build(p)      # L = 0: L~ = T only -> singular
    with pytest.raises(m.SSError) as e:
        m.ss_setup(h, 0.0, 10)
    assert e.value.code == 4
    m.ss_destroy(h)


def test_kernel_launch_counter_moves(cuda):
    m = pb()
    before = m.ss_kernel_launches()
    s = m.SteadyState(CONFIGS["tiny"]).setup().solve()
    assert m.ss_kernel_launches() > before + 10
    s.close()


def test_sweep_points_on_gpu(cuda):
    """The detuning sweep driver (sweep.py, world size 1) on a few jittered tiny points:
    every point's observables equal the oracle's direct solve within the bound above."""
    from paper_1411_4356_b200.sweep import run_sweep
    pts = [tiny_params(3, 8, Delta=d, n_th=0.2) for d in (-1.0, -0.25, 0.5)]
    table = run_sweep(pts)
    for row, p in zip(table, pts):
        assert row[0] == p.Delta and row[5] == 1.0 and row[4] <= p.tol
        ref = ss.solve_direct(p)
        ra, rb = ss.expect(ref, p)
        assert abs(row[1] - ra) <= 1e-7 and abs(row[2] - rb) <= 1e-6


def test_concurrent_points_identical_to_sequential(cuda):
    """Several points solved at the same time on one GPU (sweep.concurrent_solver: host
    threads, own streams, SM budgets for the persistent substitutions) give exactly the
    table of the one-at-a-time sweep: the block substitution's reductions have a fixed
    order whatever the number of helper CTAs, so the results are bit-identical."""
    from paper_1411_4356_b200.sweep import run_sweep, concurrent_solver
    pts = [CONFIGS["small"].with_(Delta=d) for d in (-1.0, -0.5, 0.0, 0.5, 1.0)]
    seq = run_sweep(pts)
    # default: setups overlap, solves one at a time; overlap_solves: the solves share the GPU too
    for overlap in (False, True):
        con = run_sweep(pts, solve=concurrent_solver(3, overlap_solves=overlap), concurrent=3)
        assert np.array_equal(seq[:, :6], con[:, :6])      # all but the timing column
        assert np.all(con[:, 5] == 1.0)


def test_sm_budget_same_result(cuda):
    """ss_set_sm_budget (2 clusters: chain + one helper cluster) leaves M^{-1} bit-identical."""
    torch = cuda
    s = pb().SteadyState(CONFIGS["small"]).setup()
    x = torch.from_numpy(rand_cvec(s.n, 3)).cuda()
    y0 = s.precond(x, 2)
    pb().ss_set_sm_budget(s.handle, 16)
    y1 = s.precond(x, 2)
    assert torch.equal(y0, y1)
    with pytest.raises(pb().SSError):
        pb().ss_set_sm_budget(s.handle, -1)
    s.close()


def test_precond_ignores_stale_shared_memory(cuda):
    """Shared memory is not cleared between kernels.  With every SM's shared memory filled with a
    NaN pattern (ss_debug_poison_smem: what another problem's kernels may leave behind when several
    sweep points share a GPU), M^{-1}, its two factors and the whole solve give bit-identical,
    finite results: no term of the substitution may multiply a zeroed value by a ring slot or a
    partial that this launch has not written (0 * NaN = NaN).  Regression test for the sweep
    points that lost their first M^{-1} application."""
    torch = cuda
    for name in ("tiny", "small"):
        s = pb().SteadyState(CONFIGS[name]).setup()
        x = torch.from_numpy(rand_cvec(s.n, 5)).cuda()
        ref = [s.precond(x, w) for w in (0, 1, 2)]
        for rep in range(3):
            for w in (0, 1, 2):
                pb().ss_debug_poison_smem(s.handle)
                y = s.precond(x, w)
                assert bool(torch.isfinite(torch.view_as_real(y)).all()), (name, w, rep)
                assert torch.equal(y, ref[w]), (name, w, rep)
        s.solve()
        it0, rho0 = s.solve_info["iterations"], s.rho().clone()
        pb().ss_debug_poison_smem(s.handle)
        s.solve()
        assert s.solve_info["converged"] == 1 and s.solve_info["iterations"] == it0
        assert torch.equal(s.rho(), rho0)
        s.close()


def test_trace_abi(cuda):
    """ss_debug_trace_trsv returns one row of SS_TRACE_STAMPS (16) stamps per block."""
    torch = cuda
    s = pb().SteadyState(CONFIGS["tiny"]).setup()
    x = torch.randn(s.n, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    tr = pb().ss_debug_trace_trsv(s.handle, 0, x.data_ptr(), y.data_ptr())
    assert tr.shape == ((s.n + 31) // 32, 16)
    assert np.all(tr[:, 3] > 0) and np.all(tr[:, 14:] == 0)
    ref = s.precond(x, 0)
    assert torch.equal(y, ref)      # tracing does not change the result
    s.close()


def test_full_size_medium(cuda):
    """BASELINE configs[2] (n = 360,000) at full size through the C ABI, in the launch
    configuration bench.py times: rho element by element against the oracle's iterative
    steady state (tests/golden/medium_rho.npy, written by a committed oracle-only script;
    the oracle's direct solve does not fit here), the north-star residual computed with
    the oracle's own Liouvillian, Tr rho = 1, rho = rho^H, a real non-negative diagonal,
    and both substitutions checked row by row on sampled rows against their plain
    definitions with the exported factors."""
    torch = cuda
    p = CONFIGS["medium"]
    s = pb().SteadyState(p).setup().solve()
    info = s.solve_info
    assert info["converged"] == 1 and info["rel_residual"] <= p.tol
    rho = s.rho().cpu().numpy()
    assert ss.liouvillian_residual(rho, p) <= 1e-9
    assert abs(np.trace(rho) - 1) <= 1e-12
    # element-wise against the ORACLE's steady state (scripts/make_golden_medium.py: oracle
    # RCM + column iLUTP + GMRES(50), converged to 3.2e-11; north-star bar 1e-6)
    import os
    ref = np.load(os.path.join(os.path.dirname(__file__), "golden", "medium_rho.npy"))
    assert np.abs(rho - ref).sum() <= 1e-6
    na, nb = s.expect()
    ra, rb = ss.expect(ref, p)
    assert abs(na - ra) <= 1e-8 and abs(nb - rb) <= 1e-8
    # the exact steady state is Hermitian with a real non-negative diagonal, so these
    # deviations are bounded by 2 ||rho - rho_exact||_1, which the north star bounds by
    # 2e-6 (measured: 7e-10)
    assert np.abs(rho - rho.conj().T).sum() <= 2e-6
    d = np.diag(rho)
    assert np.abs(d.imag).sum() <= 2e-6 and d.real.min() >= -2e-6
    # first substitution (U'^T z = x, lower with the pivots on its diagonal), sampled rows
    # against its plain definition with the exported factor U' of the column-oriented iLUTP
    n = s.n
    x = rand_cvec(n, 21)
    z = s.precond(torch.from_numpy(x).cuda(), 0).cpu().numpy()
    rp, ci, va = pb().ss_export_factors(s.handle, 1)
    Ut = sp.csr_matrix((va, ci, rp), shape=(n, n)).T.tocsr()   # row i of U'^T = column i of U'
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([rng.integers(0, n, 400), [0, 1, 31, 32, n - 33, n - 1]]))
    for i in rows:
        lhs = np.dot(Ut.data[Ut.indptr[i]:Ut.indptr[i + 1]], z[Ut.indices[Ut.indptr[i]:Ut.indptr[i + 1]]])
        assert abs(lhs - x[i]) <= 1e-10 * (np.abs(x).max() + np.abs(Ut.data).max() * np.abs(z).max())
    # second substitution (L'^T y = x, unit upper), sampled rows
    y = s.precond(torch.from_numpy(x).cuda(), 1).cpu().numpy()
    rp, ci, va = pb().ss_export_factors(s.handle, 0)
    Lt = sp.csr_matrix((va, ci, rp), shape=(n, n)).T.tocsr()
    for i in rows:
        lhs = y[i] + np.dot(Lt.data[Lt.indptr[i]:Lt.indptr[i + 1]], y[Lt.indices[Lt.indptr[i]:Lt.indptr[i + 1]]])
        assert abs(lhs - x[i]) <= 1e-10 * (np.abs(x).max() + np.abs(Lt.data).max() * np.abs(y).max())
    s.close()


def test_full_size_sweep_points(cuda):
    """BASELINE configs[4] (n = 230,400 per point) at full size through the sweep driver
    (sweep.py, world size 1) on the two end points and the centre of the detuning range,
    with the sweep's iLUTP parameters (R15/R16).  Each point converges to the BASELINE
    tolerance (the paper: RCM iLU "converges ... at all detunings" for n_th > 0,
    PAPER.md:128), the driver's converged flag agrees with its residual, and the
    north-star residual recomputed with the oracle's own Liouvillian holds (the oracle's
    direct solve does not fit at this size)."""
    from paper_1411_4356_b200.sweep import run_sweep
    from workloads import sweep_params
    allp = sweep_params()
    pts = [allp[0], allp[len(allp) // 2], allp[-1]]
    table = run_sweep(pts)
    for row, p in zip(table, pts):
        assert row[0] == p.Delta
        assert row[5] == float(row[4] <= p.tol)
        assert row[5] == 1.0
    s = pb().SteadyState(pts[-1]).setup().solve()
    rho = s.rho().cpu().numpy()
    assert ss.liouvillian_residual(rho, pts[-1]) <= 1e-9 and abs(np.trace(rho) - 1) <= 1e-12
    na, nb = s.expect()
    assert abs(na - table[-1][1]) <= 1e-12 and abs(nb - table[-1][2]) <= 1e-12   # the driver's numbers
    s.close()
