"""Oracle: reverse Cuthill-McKee ordering of sec. III (pure Python).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:98 (sec. III): "CM ordering does a breadth-first search of the graph
starting with a node (row) of lowest degree, where the degree of the i-th node
is defined to be the number of nonzero elements in the i-th matrix row, and
visiting neighboring nodes in each level-set in order from lowest to highest
degree.  This is repeated for each connected component of the graph. ...
reversing the CM order, the RCM ordering ...  we calculate the RCM ordering of
the symmetrized form L~ + L~^T and apply the resulting row and column ordering
to L~".

Readings (R3): the graph is the STRUCTURAL union pattern(L~) U
pattern(L~^T) (values irrelevant, "only the locations of nonzero
matrix elements"); degree = stored entries of the row of that pattern
(diagonal included, as the quote says); ties in degree are broken by the
smaller original index, both for the start node of every component and for the
order in which a node's unvisited neighbours are appended to the queue.
Output ``perm`` maps new -> old: A_rcm = A[perm][:, perm].

A second, independently written implementation of the same rule is
oracle/rcm_ref.c (used for large inputs and as the bit-exact cross-check the
north star asks for).  Pure-Python loops: small inputs only.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def symmetrized_pattern(A) -> sp.csr_matrix:
    """pattern(A + A^T) as a 0/1 CSR matrix (structural union)."""
    P = sp.csr_matrix(A, copy=True)
    P.data = np.ones_like(P.data, dtype=np.float64)
    S = sp.csr_matrix(P + P.T)
    S.data[:] = 1.0
    S.sort_indices()
    return S


def rcm(S: sp.csr_matrix) -> np.ndarray:
    S = sp.csr_matrix(S)
    S.sort_indices()
    n = S.shape[0]
    ptr, idx = S.indptr, S.indices
    deg = [int(ptr[i + 1] - ptr[i]) for i in range(n)]
    visited = [False] * n
    order: list[int] = []
    for s in sorted(range(n), key=lambda i: (deg[i], i)):
        if visited[s]:
            continue
        visited[s] = True
        queue = [s]
        head = 0
        while head < len(queue):
            v = queue[head]
            head += 1
            nbrs = [int(u) for u in idx[ptr[v]:ptr[v + 1]] if u != v and not visited[u]]
            nbrs.sort(key=lambda u: (deg[u], u))
            for u in nbrs:
                visited[u] = True
                queue.append(u)
        order.extend(queue)
    return np.array(order[::-1], dtype=np.int64)


def permute(A, perm: np.ndarray) -> sp.csr_matrix:
    """Symmetric permutation A[perm][:, perm] (new index k <- old perm[k])."""
    A = sp.csr_matrix(A)
    B = sp.csr_matrix(A[perm][:, perm])
    B.sort_indices()
    return B
