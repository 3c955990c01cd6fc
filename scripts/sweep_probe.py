"""Probe ILU parameters for the detuning sweep (BASELINE configs[4]) on the GPU.

usage: python scripts/sweep_probe.py DELTA d p [d p ...]     (env PERMTOL overrides permtol)
Prints one line per (d, p): setup time, fill, iterations, converged, residual, solve ms.
Diagnostic only (reading R15 in DESIGN.md).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1411_4356_b200 as pb  # noqa: E402
from workloads import SWEEP_BASE  # noqa: E402


def main():
    delta = float(sys.argv[1])
    rest = sys.argv[2:]
    for d, f in zip(rest[0::2], rest[1::2]):
        p = SWEEP_BASE.with_(Delta=delta, drop_tol=float(d), fill_factor=float(f),
                             permtol=float(os.environ.get("PERMTOL", SWEEP_BASE.permtol)))
        t0 = time.perf_counter()
        s = pb.SteadyState(p).setup()
        t1 = time.perf_counter()
        s.solve()
        i = s.solve_info
        print(json.dumps({"Delta": delta, "d": float(d), "p": float(f), "permtol": p.permtol,
                          "setup_s": round(t1 - t0, 2),
                          "fill": s.setup_info["fill"], "iterations": i["iterations"],
                          "converged": i["converged"], "rel_residual": i["rel_residual"],
                          "solve_ms": round(i["solve_ms"], 1)}), flush=True)
        s.close()


if __name__ == "__main__":
    main()
