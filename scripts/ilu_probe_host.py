"""Host-side probe of the iLUTP parameters on configs[3]/[4]-shaped problems (R14-R16).

Diagnostic only.  L~ (Eq. (5)) and its RCM order come from oracle/, the column-oriented
iLUTP (R16) from the product's threaded host factorisation `ss_ilutp_host` (bit-identical
to oracle/ilut.c: tests/test_host_ilutp.py) so that problems the serial oracle takes
~15 min for run in ~1 min; the stability estimate ||M^{-1} e||_inf (R8) and
GMRES(m) (R9) are the oracle's.  No GPU needed.

usage: python scripts/ilu_probe_host.py "CONFIG N_m DELTA d p permtol [n_th]" ...
Prints one JSON line per job.
"""
from __future__ import annotations

import json
import os
import sys
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402


def run(job: str, max_iter: int = 400) -> dict:
    warnings.filterwarnings("ignore")
    import paper_1411_4356_b200 as pb
    from oracle import liouvillian as lv, rcm as rcm_py
    from oracle.gmres import gmres
    from oracle.ilut import IluFactors
    from oracle.steadystate import order
    from oracle.trisolve import apply_preconditioner
    from workloads import CONFIGS, SWEEP_BASE

    f = job.split()
    cfg, nm, D, d, p, pt = f[0], int(f[1]), float(f[2]), float(f[3]), float(f[4]), float(f[5])
    base = SWEEP_BASE if cfg == "sweep" else CONFIGS[cfg]
    P = base.with_(N_m=nm, Delta=D, drop_tol=d, fill_factor=p, permtol=pt)
    if len(f) > 6:
        P = P.with_(n_th=float(f[6]))
    out = dict(config=cfg, N_c=P.N_c, N_m=nm, Delta=D, d=d, p=p, permtol=pt, n_th=P.n_th)
    Lt, rhs, w, L = lv.constrained_system(P)
    perm = order(Lt)
    A = rcm_py.permute(Lt, perm)
    At = sp.csr_matrix(A.T)
    At.sort_indices()
    t0 = time.perf_counter()
    (Lp, Lj, Lx), (Up, Uj, Ux), cp = pb.ss_ilutp_host(At.indptr, At.indices, At.data, d, p, pt)
    t1 = time.perf_counter()
    F = IluFactors(A.shape[0], Lp, Lj, Lx, Up, Uj, Ux, cp, columns=True)
    M = lambda v: apply_preconditioner(F, v)  # noqa: E731
    ce = float(np.abs(M(np.ones(A.shape[0], complex))).max())
    r = gmres(lambda v: A @ v, M, rhs[perm], P.restart, P.tol, max_iter) if np.isfinite(ce) else None
    out.update(n=A.shape[0], fill=round(F.nnz / A.nnz, 2), swaps=int((cp != np.arange(F.n)).sum()),
               condest=ce, iterations=r.iterations if r else 0, converged=bool(r and r.converged),
               rel_residual=float(r.rel_residual) if r else float("nan"), ilu_s=round(t1 - t0, 1))
    return out


if __name__ == "__main__":
    for job in sys.argv[1:]:
        print(json.dumps(run(job)), flush=True)
