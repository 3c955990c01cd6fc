"""Probe iLUTP parameters on full-size points on the GPU (R15/R16 study).

usage: python scripts/sweep_probe.py CONFIG "DELTAS" "d:p:permtol ..." [n_th]
  CONFIG  sweep | large | medium | small  (BASELINE configs; sweep = configs[4] base point)
  DELTAS  comma-separated detunings, or "-" for the config's own
Prints one JSON line per (Delta, d, p, permtol): setup time, fill, pivot exchanges,
||M^{-1} e||_inf (reading R8), iterations, converged, residual, solve ms.
The factors are bit-identical to the oracle's (tests/test_host_ilutp.py,
tests/test_gpu_parity.py), so this is the oracle's iLUTP at sizes the oracle takes
hours for.  Diagnostic only.
"""
import json
import sys
import time
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1411_4356_b200 as pb  # noqa: E402
from workloads import CONFIGS, SWEEP_BASE  # noqa: E402


def main():
    cfg = sys.argv[1]
    base = SWEEP_BASE if cfg == "sweep" else CONFIGS[cfg]
    deltas = [base.Delta] if sys.argv[2] == "-" else [float(x) for x in sys.argv[2].split(",")]
    combos = [tuple(float(v) for v in c.split(":")) for c in sys.argv[3].split()]
    if len(sys.argv) > 4:
        base = base.with_(n_th=float(sys.argv[4]))
    for delta in deltas:
        for d, f, pt in combos:
            p = base.with_(Delta=delta, drop_tol=d, fill_factor=f, permtol=pt)
            out = {"config": cfg, "Delta": delta, "d": d, "p": f, "permtol": pt, "n_th": p.n_th}
            try:
                t0 = time.perf_counter()
                s = pb.SteadyState(p).setup()
                t1 = time.perf_counter()
                e = torch.ones(s.n, dtype=torch.complex128, device="cuda")
                ce = float(s.precond(e, 2).abs().max())
                s.solve()
                i = s.solve_info
                # device ms of one L / U substitution and one SpMV (roofline evidence)
                kms = {}
                y = torch.empty_like(e)
                for nm, fn in (("trsv_lower", lambda: pb.ss_precond(s.handle, 0 | 4, e.data_ptr(), y.data_ptr())),
                               ("trsv_upper", lambda: pb.ss_precond(s.handle, 1 | 4, e.data_ptr(), y.data_ptr())),
                               ("spmv", lambda: s.spmv(e))):
                    fn()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(3):
                        fn()
                    b.record()
                    b.synchronize()
                    kms[nm] = a.elapsed_time(b) / 3
                out["kernel_ms"] = kms
                out["nnz_L"], out["nnz_U"] = s.setup_info["nnz_L"], s.setup_info["nnz_U"]
                out["n"], out["nnz"] = s.n, s.build_info["nnz"]
                out.update(setup_s=round(t1 - t0, 2), fill=round(s.setup_info["fill"], 2),
                           swaps=s.setup_info["pivot_swaps"], repaired=s.setup_info["pivots_repaired"],
                           condest=ce, iterations=i["iterations"], converged=i["converged"],
                           rel_residual=i["rel_residual"], solve_ms=round(i["solve_ms"], 1))
                s.close()
            except Exception as ex:   # noqa: BLE001 -- report and carry on
                out["error"] = str(ex)
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
