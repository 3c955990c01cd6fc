"""Benchmark: preconditioned GMRES iterations/s for the steady state of the optomechanical
Liouvillian (BASELINE.json metric), on the CUDA path of include/ss_b200.h.

One step = one full solve of Eq. (5) on the rank's Liouvillian: GMRES(m) from x0 = 0 to
the configured tolerance (every Arnoldi step = SpMV + forward + backward substitution
with the ILUT factors + CGS2 orthogonalisation), the un-permutation/normalisation of
rho, and the NCCL all-gather of the observables (<a^+a>, <b^+b>) across ranks.
Setup (build, RCM, ILUT) is done once before the timed region and reported separately.

Default (N = 1): BASELINE configs[1] (N_c=6, N_m=30, Liouvillian dim 32,400).
N > 1 (torchrun): every rank solves its own detuning point of the same shape (the
sweep axis of the north star): weak scaling, no data-path collective except the
observable gather.  --impl reference times the oracle (oracle/) on host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from workloads import CONFIGS, CONFIG_ORDER  # noqa: E402

METRIC = "preconditioned GMRES iterations/s & time-to-steady-state vs Liouvillian dim"
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="small", choices=["tiny", "small", "medium", "large"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--threads", type=int, default=0, help="host threads for the ILUT setup")
    ap.add_argument("--dims", default="tiny,small,medium",
                    help="configs for the time-to-steady-state vs Liouvillian-dim table (rank 0, N = 1)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def rank_params(name: str, rank: int, world: int):
    """Rank 0 runs the BASELINE config verbatim; other ranks shift the detuning (sweep axis)."""
    p = CONFIGS[name]
    if rank == 0:
        return p
    return p.with_(Delta=p.Delta + 0.25 * rank)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str):
    """Per-launch dram bytes of `kernel` from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(path))
        return d.get(kernel)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = f"/tmp/ss_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(name: str, budget_s: float = 20.0):
    """The oracle as it stands (numpy/scipy + plain C), timed on host cores: setup untimed,
    then GMRES Arnoldi steps until ~budget_s; reports oracle GMRES iterations/s."""
    from threadpoolctl import threadpool_limits

    from oracle import liouvillian as lv
    from oracle import rcm as R
    from oracle import steadystate as ss
    from oracle.ilut import ilutp
    from oracle.trisolve import apply_preconditioner
    from oracle import gmres as G

    p = CONFIGS[name]
    Lt, rhs, w, L = lv.constrained_system(p)
    perm = ss.order(Lt)
    A = R.permute(Lt, perm)
    F = ilutp(A, p.drop_tol, p.fill_factor, p.permtol)
    with threadpool_limits(limits=1):
        # calibrate: time a bounded number of Arnoldi steps (max_iter cap), one cycle at most
        t0 = time.perf_counter()
        G.gmres(lambda v: A @ v, lambda v: apply_preconditioner(F, v), rhs[perm], p.restart, p.tol, 2)
        per = (time.perf_counter() - t0) / 2
        k = max(2, min(p.max_iter, int(budget_s / max(per, 1e-6))))
        t0 = time.perf_counter()
        r = G.gmres(lambda v: A @ v, lambda v: apply_preconditioner(F, v), rhs[perm], p.restart, p.tol, k)
        dt = time.perf_counter() - t0
    return {"value": r.iterations / dt, "unit": "iterations/s", "cores": 1, "kind": "oracle",
            "sample": f"{r.iterations} oracle GMRES({p.restart}) Arnoldi steps on {name} "
                      f"(n={p.liouvillian_dim}) after an untimed oracle setup; {dt:.1f} s, 1 thread"}


# oracle GMRES iterations to tol from x0 = 0 (tests/test_oracle_gmres.py, oracle.steadystate);
# the reference arm's ms_per_step is that many steps at its sampled rate
ORACLE_ITERATIONS = {"tiny": 11, "small": 26}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    base = CONFIGS[args.workload]
    vals = []
    cb = None
    for step in range(args.warmup + args.steps):
        cb = cpu_baseline(args.workload, budget_s=max(5.0, 120.0 / (args.warmup + args.steps)))
        if step >= args.warmup:
            vals.append(cb["value"])
    v = statistics.mean(vals)
    # a step of the b200 arm is one solve of the workload from x0 = 0; the oracle's time for
    # it at the sampled rate (iterations per solve from the oracle's own full solve count,
    # one restart cycle: configs[1] converges in 26)
    its = ORACLE_ITERATIONS.get(args.workload)
    ms_step = 1e3 * its / v if its else None
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "iterations/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": workload_config(args.workload, base, world),
            "cpu_baseline": {**cb, "value": v},
            "e2e": {"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(name, p, world):
    return {"workload": f"configs[{CONFIG_ORDER.index(name)}] {name}: N_c={p.N_c}, N_m={p.N_m}, "
                        f"Liouvillian dim {p.liouvillian_dim}",
            "N_c": p.N_c, "N_m": p.N_m, "liouvillian_dim": p.liouvillian_dim, "omega_m": p.omega_m,
            "Delta": p.Delta, "kappa": p.kappa, "g0": p.g0, "E": p.E, "Gamma_m": p.Gamma_m, "n_th": p.n_th,
            "drop_tol": p.drop_tol, "fill_factor": p.fill_factor, "restart": p.restart, "tol": p.tol,
            "ranks": world, "rank_detuning_shift": 0.25,
            "l2": "flushed (256 MiB write) before every timed step, outside the step's events"}


def precond_bytes(si, n):
    """Algorithmic bytes of one M^{-1} application (both substitutions), DESIGN.md sec. 5:
    every strict factor entry once (16 B value + 4 B column), U's diagonal, the row
    pointers, and per factor the right-hand side read, x written and x read back once."""
    strict = si["nnz_L"] + si["nnz_U"] - n
    return strict * 20 + n * 16 + 2 * ((n + 1) * 8 + 3 * n * 16)


def steady_state_vs_dim(names, threads):
    """Time to steady state (build + setup, then the GMRES solve from x0 = 0) per config;
    the second half of the BASELINE metric.  Device time of the solve from ss_solve_info,
    host wall time of build/setup."""
    import paper_1411_4356_b200 as pb

    rows = []
    for name in names:
        p = CONFIGS[name]
        t0 = time.perf_counter()
        s = pb.SteadyState(p)
        s.setup(threads=threads)
        t1 = time.perf_counter()
        s.solve()
        si = s.solve_info
        rows.append({"config": name, "liouvillian_dim": p.liouvillian_dim, "nnz": s.build_info["nnz"],
                     "setup_s": t1 - t0, "solve_ms": si["solve_ms"], "iterations": si["iterations"],
                     "converged": bool(si["converged"]), "rel_residual": si["rel_residual"],
                     "iterations_per_s": si["iterations"] / (si["solve_ms"] * 1e-3) if si["solve_ms"] else None})
        s.close()
    return rows


def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_1411_4356_b200 as pb

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    p = rank_params(args.workload, rank, world)

    t0 = time.perf_counter()
    s = pb.SteadyState(p, stream=stream)
    s.setup(threads=args.threads)
    setup_s = time.perf_counter() - t0
    n = s.n
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    obs = torch.zeros(2, dtype=torch.float64, device=dev)
    gathered = torch.zeros(2 * world, dtype=torch.float64, device=dev)

    def step():
        s.solve()
        na, nb = s.expect()
        obs[0], obs[1] = na, nb
        if world > 1:
            dist.all_gather_into_tensor(gathered, obs)
        return s.solve_info["iterations"]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = pb.ss_kernel_launches()
    evs = []
    iters = 0
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for _ in range(args.steps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        iters += step()
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = pb.ss_kernel_launches() - launches0
    ms_total = sum(a.elapsed_time(b) for a, b in evs)
    clk = clocks.stop()

    # --- kernel-level timing of the hot-path pieces on the same stream (roofline evidence)
    x = torch.randn(n, dtype=torch.complex128, device=dev)
    lvl = {}
    y = torch.empty_like(x)
    for name, fn in (("trsv_lower", lambda: pb.ss_precond(s.handle, 0 | 4, x.data_ptr(), y.data_ptr())),
                     ("trsv_upper", lambda: pb.ss_precond(s.handle, 1 | 4, x.data_ptr(), y.data_ptr())),
                     ("spmv", lambda: s.spmv(x))):
        fn()
        reps = 5
        tot = 0.0
        for _ in range(reps):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            tot += a.elapsed_time(b)
        lvl[name] = tot / reps

    # --- end to end through the C ABI with HOST buffers (H2D rhs + D2H x inside the region)
    rhs = torch.zeros(n, dtype=torch.complex128).pin_memory()
    rhs[0] = complex(s.build_info["w_re"], s.build_info["w_im"])
    xh = torch.empty(n, dtype=torch.complex128).pin_memory()
    e2e_ms, e2e_it = 0.0, 0
    for _ in range(max(1, args.steps // 2)):
        torch.cuda.synchronize()
        t = time.perf_counter()
        info = pb.ss_solve_host(s.handle, rhs.data_ptr(), xh.data_ptr(), p.restart, p.tol, p.max_iter)
        e2e_ms += (time.perf_counter() - t) * 1e3
        e2e_it += info["iterations"]

    # max over ranks of the device time
    tt = torch.tensor([ms_total, float(iters), e2e_ms, float(e2e_it)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = tt.clone()
        dist.all_reduce(mx[0:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(mx[2:3], op=dist.ReduceOp.MAX)
        dist.all_reduce(mx[1:2], op=dist.ReduceOp.SUM)
        dist.all_reduce(mx[3:4], op=dist.ReduceOp.SUM)
        tt = mx
    ms_max, it_sum, e2e_max, e2e_it_sum = [float(v) for v in tt.tolist()]

    if rank == 0:
        si = s.setup_info
        peak, peak_src = peaks()
        nlL, nlU = si["levels_L"], si["levels_U"]
        bytes_pc = precond_bytes(si, n)
        ms_pc = lvl["trsv_lower"] + lvl["trsv_upper"]
        achieved = bytes_pc / (ms_pc * 1e-3) / 1e9
        tr = ncu_traffic("k_chain_trsv")
        line = {
            "metric": METRIC, "value": it_sum / (ms_max * 1e-3), "unit": "iterations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (BASELINE parameter set; no dataset exists for this method)",
            "config": {**workload_config(args.workload, p if rank == 0 else CONFIGS[args.workload], world),
                       "setup_s": setup_s, "iterations_per_solve": it_sum / (args.steps * world),
                       "fill": si["fill"], "nnz_L": si["nnz_L"], "nnz_U": si["nnz_U"],
                       "levels_L": nlL, "levels_U": nlU, "bandwidth_rcm": si["bandwidth_rcm"],
                       "time_to_steady_state_ms": ms_max / args.steps},
            "roofline": {"bound": "hbm", "kernel": "k_chain_trsv (L then U launch: one M^-1 application)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "peak_source": peak_src, "traffic": tr,
                         "algorithmic_bytes_per_apply": bytes_pc, "ms_per_apply": ms_pc,
                         "kernel_ms": lvl, "trsv_block": si.get("trsv_block"),
                         "trsv_q": [si.get("trsv_q_L"), si.get("trsv_q_U")],
                         "note": "chain-latency bound: n/B dependent block steps per factor (DESIGN.md sec. 5)"},
            "e2e": {"value": e2e_it_sum / (e2e_max * 1e-3), "unit": "iterations/s",
                    "h2d_bytes_per_step": n * 16, "d2h_bytes_per_step": n * 16},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if world == 1 and args.dims:
            line["time_to_steady_state_vs_dim"] = steady_state_vs_dim(args.dims.split(","), args.threads)
        if not args.no_cpu_baseline and world == 1:
            try:
                line["cpu_baseline"] = cpu_baseline(args.workload)
            except Exception as e:  # the baseline is reported, never required
                line["cpu_baseline"] = {"value": None, "error": str(e)}
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
