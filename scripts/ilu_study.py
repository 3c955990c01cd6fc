"""Oracle-only study of the iLUTP reading (R13-R16): which orientation and
parameters give stable preconditioners on configs[3]/[4]-shaped problems.

Calls ONLY oracle/ and workloads.py (no product code).  For each case it builds L~
(Eq. (5)), orders it by RCM (sec. III), factors L~_RCM with the oracle's iLUTP in the
given orientation ("rows": row-wise ILUTP of L~_RCM, R13; "columns": row-wise ILUTP of
L~_RCM^T, R16), and records the fill, the paper's stability estimate ||M^{-1} e||_inf
(R8) and GMRES(m) (R9) to the config's tolerance, at most
400 Arnoldi steps.

usage: python scripts/ilu_study.py OUT.jsonl [JOBS]       (default: the built-in grid)
  a job line: CONFIG N_m DELTA ORIENT d p permtol [n_th]
"""
from __future__ import annotations

import json
import os
import sys
import time
import warnings
from concurrent.futures import ProcessPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

GRID = [
    # configs[4]-shaped (N_c = 8, g0 = 0.8, kappa = 0.5, n_th = 0.2) at growing N_m
    *[f"sweep {nm} {D} {o} 1e-5 40 0.01" for nm in (20, 30) for D in (-2, 0, 2) for o in ("rows", "columns")],
    *[f"sweep 40 {D} columns 1e-5 40 0.01" for D in (-2, -1, 0, 2)],
    "sweep 40 2 columns 1e-5 40 0.5", "sweep 40 2 columns 1e-5 100 0.01",
    "sweep 40 2 rows 1e-5 40 0.5", "sweep 40 2 rows 1e-5 100 0.01",
    "sweep 20 0 rows 1e-5 1e6 0.01", "sweep 20 0 columns 1e-5 1e6 0.01",
    # configs[3]-shaped (N_c = 12, g0/kappa = 2), n_th = 0 and the paper's 1e-15 (R12)
    "large 20 -1 rows 1e-5 80 0.01 0", "large 20 -1 columns 1e-5 80 0.01 0",
    "large 20 -1 columns 1e-5 80 0.01 1e-15",
]


def run(job: str) -> dict:
    warnings.filterwarnings("ignore")
    import numpy as np
    from oracle import liouvillian as lv, rcm as rcm_py
    from oracle.gmres import gmres
    from oracle.steadystate import order, factor
    from oracle.trisolve import apply_preconditioner
    from workloads import CONFIGS, SWEEP_BASE

    f = job.split()
    cfg, nm, D, orient, d, p, pt = f[0], int(f[1]), float(f[2]), f[3], float(f[4]), float(f[5]), float(f[6])
    base = SWEEP_BASE if cfg == "sweep" else CONFIGS[cfg]
    P = base.with_(N_m=nm, Delta=D, drop_tol=d, fill_factor=p, permtol=pt)
    if len(f) > 7:
        P = P.with_(n_th=float(f[7]))
    out = dict(config=cfg, N_c=P.N_c, N_m=nm, Delta=D, orientation=orient, d=d, p=p, permtol=pt, n_th=P.n_th)
    try:
        Lt, rhs, w, L = lv.constrained_system(P)
        perm = order(Lt)
        A = rcm_py.permute(Lt, perm)
        t0 = time.perf_counter()
        F = factor(A, P, orient)
        t1 = time.perf_counter()
        M = lambda v: apply_preconditioner(F, v)
        ce = float(np.abs(M(np.ones(A.shape[0], complex))).max())
        ok = np.isfinite(ce)
        r = gmres(lambda v: A @ v, M, rhs[perm], P.restart, P.tol, 400) if ok else None
        out.update(n=A.shape[0], fill=round(F.nnz / A.nnz, 2),
                   swaps=int((F.perm != np.arange(F.n)).sum()), condest=ce,
                   iterations=r.iterations if r else 0, converged=bool(r and r.converged),
                   rel_residual=float(r.rel_residual) if r else float("nan"), ilu_s=round(t1 - t0, 1))
    except Exception as ex:  # noqa: BLE001
        out["error"] = str(ex)
    return out


def main():
    out_path = sys.argv[1]
    jobs = GRID if len(sys.argv) < 3 else [l.strip() for l in open(sys.argv[2]) if l.strip()]
    with ProcessPoolExecutor(max_workers=max(1, (os.cpu_count() or 2) - 1)) as ex, open(out_path, "a") as fo:
        for res in ex.map(run, jobs):
            fo.write(json.dumps(res) + "\n")
            fo.flush()
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
