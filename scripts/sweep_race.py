"""Diagnostic: concurrent sweep points on one GPU vs the same points one at a time.

usage: python scripts/sweep_race.py N_m POINTS CONCURRENT MODE [reps]
  MODE  full        setup and solve concurrently (sweep.concurrent_solver)
        lock_solve  setups concurrent, solves one at a time (a lock around solve)
        lock_setup  setups one at a time, solves concurrent
Prints the number of points whose observables / iteration counts differ from the
sequential run, and the failing points.
"""
import json
import os
import sys
import threading
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1411_4356_b200 as pb  # noqa: E402
from workloads import SWEEP_BASE, sweep_params  # noqa: E402


def main():
    nm, npts, conc, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
    pts = sweep_params(npts, base=SWEEP_BASE.with_(N_m=nm))
    dev = torch.cuda.current_device()
    cores = os.cpu_count() or 1

    def one(p, stream, threads, budget, lock_setup=None, lock_solve=None):
        ctx = lock_setup or threading.Lock()
        with ctx if lock_setup else _null():
            s = pb.SteadyState(p, stream=stream).setup(threads=threads)
        try:
            if budget:
                pb.ss_set_sm_budget(s.handle, budget)
            with lock_solve if lock_solve else _null():
                s.solve()
            i = s.solve_info
            na, nb = s.expect()
            out = dict(Delta=p.Delta, it=i["iterations"], conv=i["converged"], res=i["rel_residual"], na=na, nb=nb,
                       nnzL=s.setup_info["nnz_L"], nnzU=s.setup_info["nnz_U"], swaps=s.setup_info["pivot_swaps"])
            if i["converged"] != 1:
                # transient (the launch) or persistent (the data on the device)?  M^{-1} e twice, then
                # the solve again, on the same handle, with nothing else running in this thread
                torch.cuda.synchronize()
                e = torch.ones(s.n, dtype=torch.complex128, device="cuda")
                e1, e2 = e.clone(), e.clone()
                torch.cuda.synchronize()
                y1, y2 = s.precond(e1), s.precond(e2)
                out["again_precond_finite"] = [bool(torch.isfinite(torch.view_as_real(y)).all()) for y in (y1, y2)]
                out["again_precond_equal"] = bool(torch.equal(y1, y2))
                s.solve()
                out["again_solve"] = [s.solve_info["iterations"], s.solve_info["converged"]]
            return out
        finally:
            s.close()

    seq = [one(p, torch.cuda.current_stream(), cores, 0) for p in pts]
    s0 = pb.SteadyState(pts[0]).setup()
    grid = s0.setup_info["trsv_grid"]
    s0.close()
    local = threading.local()
    ls = threading.Lock() if mode == "lock_setup" else None
    lv = threading.Lock() if mode == "lock_solve" else None

    def worker(p):
        torch.cuda.set_device(dev)
        if not hasattr(local, "stream"):
            local.stream = torch.cuda.Stream(device=dev)
        return one(p, local.stream, max(1, cores // conc), 8 * max(2, grid // 8 // conc), ls, lv)

    bad_total = 0
    for r in range(reps):
        with ThreadPoolExecutor(conc) as ex:
            got = list(ex.map(worker, pts))
        bad = [(a, b) for a, b in zip(seq, got) if a["it"] != b["it"] or abs(a["na"] - b["na"]) > 1e-9
               or a["nnzL"] != b["nnzL"] or a["swaps"] != b["swaps"] or b["conv"] != 1]
        bad_total += len(bad)
        print(json.dumps({"rep": r, "mode": mode, "N_m": nm, "points": npts, "concurrent": conc, "bad": len(bad),
                          "examples": bad[:3]}), flush=True)
    print(json.dumps({"mode": mode, "bad_total": bad_total, "reps": reps}), flush=True)


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


if __name__ == "__main__":
    main()
