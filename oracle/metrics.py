"""Oracle: sparse-matrix bandwidth and profile of sec. II.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:73-81:  ub = max_{a_ij != 0} (j - i),  lb = max_{a_ij != 0} (i - j),
B = ub + lb + 1;  up = sum_i max_{a_ij != 0} (j - i),
lp = sum_j max_{a_ij != 0} (i - j),  P = up + lp.
Reading R2: a row (column) whose entries all lie on the other side
of the diagonal contributes 0 to up (lp), i.e. the per-row max is clamped at 0.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def bandwidth(A) -> tuple[int, int, int]:
    C = sp.coo_matrix(A)
    if C.nnz == 0:
        raise ValueError("bandwidth undefined for an empty matrix")
    d = C.col.astype(np.int64) - C.row.astype(np.int64)
    ub = int(max(d.max(), 0))
    lb = int(max((-d).max(), 0))
    return ub, lb, ub + lb + 1


def profile(A) -> tuple[int, int, int]:
    C = sp.coo_matrix(A)
    n = A.shape[0]
    d = C.col.astype(np.int64) - C.row.astype(np.int64)
    up_row = np.zeros(n, dtype=np.int64)
    np.maximum.at(up_row, C.row, d)          # clamp at 0 through the zero init
    lp_col = np.zeros(A.shape[1], dtype=np.int64)
    np.maximum.at(lp_col, C.col, -d)
    up, lp = int(up_row.sum()), int(lp_col.sum())
    return up, lp, up + lp
