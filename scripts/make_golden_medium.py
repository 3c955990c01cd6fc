"""Write tests/golden/medium_rho.npy: the ORACLE's steady state of BASELINE configs[2]
(N_c = 10, N_m = 60, Liouvillian dim 360,000), for the element-wise GPU parity test
(tests/test_gpu_parity.py::test_full_size_medium).

Calls only oracle/ and workloads.py: RCM (sec. III), the column-oriented iLUTP (R16),
GMRES(50) to tol 1e-10 (sec. IV), rho / Tr rho (R11).  The oracle's direct solve does not
fit at this size; its iterative solve does (about half an hour on one core).  The
north-star residual ||L rho|| / ||b|| of the stored rho is checked before writing.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import steadystate as ss  # noqa: E402
from workloads import CONFIGS  # noqa: E402


def main():
    p = CONFIGS["medium"]
    t0 = time.perf_counter()
    r = ss.solve_iterative(p)
    res = ss.liouvillian_residual(r.rho, p)
    meta = dict(config="medium", iterations=r.gmres.iterations, converged=bool(r.gmres.converged),
                rel_residual_rcm=float(r.gmres.rel_residual), liouvillian_residual=res,
                fill=r.factors.nnz / 3918797, times=r.times, wall_s=time.perf_counter() - t0)
    print(json.dumps(meta))
    assert r.gmres.converged and res <= 1e-9, "oracle did not converge"
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
    np.save(os.path.join(out, "medium_rho.npy"), r.rho)
    with open(os.path.join(out, "medium_rho.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    main()
