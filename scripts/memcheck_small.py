"""Diagnostic: one configs[1]-shaped solve (and, with an argument, 4 concurrent sweep points at N_m = 12)
for compute-sanitizer memcheck."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1411_4356_b200 as pb  # noqa: E402
from workloads import CONFIGS, SWEEP_BASE, sweep_params  # noqa: E402

s = pb.SteadyState(CONFIGS["small"].with_(N_m=12)).setup().solve()
print("seq", s.solve_info["iterations"], s.solve_info["converged"], flush=True)
s.close()
if len(sys.argv) > 1:
    from paper_1411_4356_b200.sweep import concurrent_solver, run_sweep
    pts = sweep_params(8, base=SWEEP_BASE.with_(N_m=12))
    tab = run_sweep(pts, solve=concurrent_solver(4), concurrent=4)
    print("conc converged", tab[:, 5].tolist(), flush=True)
