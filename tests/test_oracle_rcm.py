"""Oracle pins for the RCM ordering (sec. III) and the structure metrics (sec. II)."""
import itertools
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import liouvillian as lv
from oracle import metrics as M
from oracle import rcm as R
from oracle import steadystate as ss
from workloads import CONFIGS, tiny_params

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def graph(n, edges, diag=True):
    r = [a for a, b in edges] + [b for a, b in edges]
    c = [b for a, b in edges] + [a for a, b in edges]
    if diag:
        r += list(range(n))
        c += list(range(n))
    return sp.csr_matrix((np.ones(len(r)), (r, c)), shape=(n, n))


def test_hand_derived_example():
    g = json.load(open(os.path.join(GOLD, "rcm_hand_example.json")))
    S = graph(g["n"], g["edges"])
    assert R.rcm(S).tolist() == g["rcm_perm_new_to_old"]
    assert ss.rcm_c(S).tolist() == g["rcm_perm_new_to_old"]


def test_path_graph_keeps_bandwidth_one():
    n = 9
    S = graph(n, [(i, i + 1) for i in range(n - 1)])
    p = R.rcm(S)
    assert sorted(p.tolist()) == list(range(n))
    assert M.bandwidth(R.permute(S, p))[2] == 3          # ub = lb = 1


def test_rcm_not_worse_than_optimum_bound_bruteforce():
    """Brute force over all 6! orders of small random graphs: RCM is a bijection and its bandwidth
    is >= the true minimum (sanity) and <= the natural one for these banded-ish graphs."""
    rng = np.random.default_rng(7)
    for trial in range(5):
        n = 6
        edges = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.35]
        S = graph(n, edges)
        p = R.rcm(S)
        assert sorted(p.tolist()) == list(range(n))
        best = min(M.bandwidth(R.permute(S, np.array(q)))[2] for q in itertools.permutations(range(n)))
        assert M.bandwidth(R.permute(S, p))[2] >= best


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_python_and_c_rcm_bit_exact_random(seed):
    rng = np.random.default_rng(seed)
    n = 300
    A = sp.random(n, n, density=0.01, random_state=seed, format="csr")
    S = R.symmetrized_pattern(A + sp.identity(n))
    assert np.array_equal(R.rcm(S), ss.rcm_c(S))


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_python_and_c_rcm_bit_exact_liouvillian(name):
    Lt, _, _, _ = lv.constrained_system(CONFIGS[name])
    S = R.symmetrized_pattern(Lt)
    assert np.array_equal(R.rcm(S), ss.rcm_c(S))


def test_fig1_reduction_factors():
    """RCM lowers the total bandwidth ~5x and the profile ~2.5x at N_c=4, N_m=8."""
    g = json.load(open(os.path.join(GOLD, "fig1_structure.json")))
    p = tiny_params(g["N_c"], g["N_m"], n_th=0.5)
    Lt, _, _, L = lv.constrained_system(p)
    A = R.permute(Lt, R.rcm(R.symmetrized_pattern(Lt)))
    rb = M.bandwidth(Lt)[2] / M.bandwidth(A)[2]
    rp = M.profile(Lt)[2] / M.profile(A)[2]
    assert 4.0 <= rb <= 6.0 and 2.0 <= rp <= 3.0
    # "The bandwidth and profile of L~_RCM are ... also less than that of L itself"
    assert M.bandwidth(A)[2] < M.bandwidth(L)[2] and M.profile(A)[2] < M.profile(L)[2]


@pytest.mark.parametrize("Nc,Nm", [(2, 3), (3, 5), (4, 8), (5, 7)])
def test_bandwidth_exceeds_hilbert_dim_squared(Nc, Nm):
    """'the total bandwidth must satisfy B(L~) > (N_c N_m)^2' (T reaches the last column)."""
    Lt, _, _, _ = lv.constrained_system(tiny_params(Nc, Nm))
    assert M.bandwidth(Lt)[2] > (Nc * Nm) ** 2


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_rcm_bandwidth_not_above_natural(name):
    Lt, _, _, _ = lv.constrained_system(CONFIGS[name])
    A = R.permute(Lt, ss.rcm_c(R.symmetrized_pattern(Lt)))
    assert M.bandwidth(A)[2] <= M.bandwidth(Lt)[2]
    assert A.nnz == Lt.nnz and np.allclose(np.sort_complex(A.diagonal()), np.sort_complex(Lt.diagonal()))


def test_metrics_definitions():
    A = sp.csr_matrix(np.array([[1, 0, 2], [0, 1, 0], [0, 0, 1.0]]))
    assert M.bandwidth(A) == (2, 0, 3)
    assert M.profile(A) == (2, 0, 2)
    D = sp.identity(4, format="csr")
    assert M.bandwidth(D) == (0, 0, 1) and M.profile(D) == (0, 0, 0)
