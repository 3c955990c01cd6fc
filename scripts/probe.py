"""Probe one BASELINE config on the GPU: setup statistics, per-kernel times, a capped solve.

usage: python scripts/probe.py NAME [max_iter] [field=value ...]
Prints one JSON line (setup_info, per-kernel device ms, solve_info).  Diagnostic only.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1411_4356_b200 as pb  # noqa: E402
from workloads import CONFIGS  # noqa: E402


def timed(fn, stream, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    name = sys.argv[1]
    max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
    p = CONFIGS[name]
    for kv in sys.argv[3:]:
        k, v = kv.split("=")
        p = p.with_(**{k: type(getattr(p, k))(float(v)) if getattr(p, k) is not None else float(v)})
    st = torch.cuda.current_stream()
    t0 = time.perf_counter()
    s = pb.SteadyState(p, stream=st)
    t1 = time.perf_counter()
    s.setup()
    t2 = time.perf_counter()
    out = {"name": name, "params": p.as_dict(), "n": s.n, "build": s.build_info, "build_s": t1 - t0, "setup_s": t2 - t1,
           "setup": s.setup_info}
    x = torch.randn(s.n, dtype=torch.complex128, device="cuda")
    out["ms"] = {"spmv": timed(lambda: s.spmv(x), st), "trsv_lower": timed(lambda: s.precond(x, 0), st, 2),
                 "trsv_upper": timed(lambda: s.precond(x, 1), st, 2)}
    print(json.dumps(out), flush=True)
    t3 = time.perf_counter()
    s.solve(max_iter=max_iter)
    out["solve"] = s.solve_info
    out["solve_wall_s"] = time.perf_counter() - t3
    out["expect"] = s.expect()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
