"""Benchmark: preconditioned GMRES iterations/s for the steady state of the optomechanical
Liouvillian (BASELINE.json metric), on the CUDA path of include/ss_b200.h.

One step = one full solve of Eq. (5) on the rank's Liouvillian: GMRES(m) from x0 = 0 to
the configured tolerance (every Arnoldi step = SpMV + forward + backward substitution
with the ILUT factors + CGS2 orthogonalisation), the un-permutation/normalisation of
rho, and the NCCL all-gather of the observables (<a^+a>, <b^+b>) across ranks.
Setup (build, RCM, ILUT) is done once before the timed region and reported separately.

Default (N = 1): BASELINE configs[2] (N_c=10, N_m=60, Liouvillian dim 360,000), the
largest single Liouvillian whose setup fits the bench's time budget (configs[3] is
measured with --workload large).
N > 1 (torchrun): every rank solves its own detuning point of the same shape (the
sweep axis of the north star): weak scaling, no data-path collective except the
observable gather.
--workload sweep: BASELINE configs[4], the 64-point detuning sweep through
paper_1411_4356_b200.sweep.run_sweep (contiguous shards over the ranks, observables
all-gathered over NCCL); a step is the whole sweep, per point build + setup + solve.
--impl reference times the oracle (oracle/) on host cores.
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
    ap.add_argument("--workload", default="medium", choices=["tiny", "small", "medium", "large", "sweep"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-baseline-only", default=None, help=argparse.SUPPRESS)   # internal: the oracle leg
    ap.add_argument("--threads", type=int, default=0, help="host threads for the ILUT setup")
    ap.add_argument("--concurrent", type=int, default=4,
                    help="sweep: points solved at the same time per GPU (host threads, SM budgets)")
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


def cpu_baseline(name: str, budget_s: float = 20.0, oracle_state: dict | None = None):
    """The oracle as it stands (numpy/scipy + plain C), timed on host cores: setup untimed
    (RCM + the column-oriented iLUTP of R16, cached in oracle_state across calls), then
    GMRES Arnoldi steps until ~budget_s; reports oracle GMRES iterations/s."""
    from threadpoolctl import threadpool_limits

    from oracle import liouvillian as lv
    from oracle import rcm as R
    from oracle import steadystate as ss
    from oracle.trisolve import apply_preconditioner
    from oracle import gmres as G

    p = CONFIGS[name]
    st = oracle_state if oracle_state is not None else {}
    if "A" not in st:
        t0 = time.perf_counter()
        Lt, rhs, w, L = lv.constrained_system(p)
        perm = ss.order(Lt)
        A = R.permute(Lt, perm)
        st.update(A=A, F=ss.factor(A, p), b=rhs[perm], setup_s=time.perf_counter() - t0)
    A, F, b = st["A"], st["F"], st["b"]
    with threadpool_limits(limits=1):
        # calibrate: time a bounded number of Arnoldi steps (max_iter cap), one cycle at most
        t0 = time.perf_counter()
        G.gmres(lambda v: A @ v, lambda v: apply_preconditioner(F, v), b, p.restart, p.tol, 2)
        per = (time.perf_counter() - t0) / 2
        k = max(2, min(p.max_iter, int(budget_s / max(per, 1e-6))))
        t0 = time.perf_counter()
        r = G.gmres(lambda v: A @ v, lambda v: apply_preconditioner(F, v), b, p.restart, p.tol, k)
        dt = time.perf_counter() - t0
    return {"value": r.iterations / dt, "unit": "iterations/s", "cores": 1, "kind": "oracle",
            "sample": f"{r.iterations} oracle GMRES({p.restart}) Arnoldi steps on {name} "
                      f"(n={p.liouvillian_dim}) after an untimed oracle setup ({st['setup_s']:.0f} s); "
                      f"{dt:.1f} s, 1 thread"}


# oracle GMRES iterations to tol from x0 = 0 (tests/test_oracle_gmres.py, oracle.steadystate);
# the reference arm's ms_per_step is that many steps at its sampled rate
ORACLE_ITERATIONS = {"tiny": 11, "small": 26, "medium": 33}   # medium: tests/golden/medium_rho.json


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    base = CONFIGS[args.workload]
    vals = []
    cb = None
    ost = {}
    for step in range(args.warmup + args.steps):
        cb = cpu_baseline(args.workload, budget_s=max(5.0, 120.0 / (args.warmup + args.steps)), oracle_state=ost)
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


def spmv_bytes(nnz, n):
    """One L~x: values + columns, row pointers, x read, y written."""
    return nnz * 20 + (n + 1) * 8 + 2 * n * 16


def cgs_bytes(nv, n):
    """CGS2 at Arnoldi step j (nv = j + 1 basis vectors): three streaming passes over V,
    w read three times and written twice (krylov.cu)."""
    return 3 * nv * n * 16 + 5 * n * 16


def solve_bytes(si, build, iterations, restart):
    """Algorithmic bytes of the Arnoldi steps of one solve (the north star's per-iteration
    roofline: L~, L, U and the Krylov vectors): every step SpMV + M^{-1} + CGS2 with the
    basis size of its position in its restart cycle."""
    n, nnz = build["n"], build["nnz"]
    per = spmv_bytes(nnz, n) + precond_bytes(si, n)
    tot = 0
    for it in range(int(iterations)):
        tot += per + cgs_bytes(it % restart + 1, n)
    return tot


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
    # the oracle's CPU baseline runs in its own process on the host cores meanwhile (its
    # untimed iLUTP setup alone takes minutes on the larger configs); one core of work
    cpu_proc = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_proc = subprocess.Popen([sys.executable, os.path.abspath(__file__), "--cpu-baseline-only",
                                     args.workload], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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
        its_per_solve = it_sum / (args.steps * world)
        sb = solve_bytes(si, s.build_info, round(its_per_solve), p.restart)
        ach_it = sb / (ms_max / args.steps * 1e-3) / 1e9
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
            "roofline_iteration": {"bound": "hbm", "what": "whole Arnoldi steps of the solve (SpMV + M^-1 + CGS2): "
                                   "algorithmic bytes of L~, the factors and the Krylov vectors / solve time",
                                   "achieved": ach_it, "peak": peak, "unit": "GB/s", "frac": ach_it / peak,
                                   "bytes_per_solve": sb, "bytes_per_iteration": sb / max(1, round(its_per_solve)),
                                   "spmv_bytes": spmv_bytes(s.build_info["nnz"], n),
                                   "precond_bytes": bytes_pc},
            "e2e": {"value": e2e_it_sum / (e2e_max * 1e-3), "unit": "iterations/s",
                    "h2d_bytes_per_step": n * 16, "d2h_bytes_per_step": n * 16},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if world == 1 and args.dims:
            line["time_to_steady_state_vs_dim"] = steady_state_vs_dim(args.dims.split(","), args.threads)
        if cpu_proc is not None:
            try:
                out, _ = cpu_proc.communicate(timeout=1500)
                line["cpu_baseline"] = json.loads(out.strip().splitlines()[-1])
            except Exception as e:  # the baseline is reported, never required
                cpu_proc.kill()
                line["cpu_baseline"] = {"value": None, "error": repr(e)}
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()


def sweep_roofline(pinfo, ms_step, world):
    """configs[4]: algorithmic bytes of every Arnoldi step of every solve of the sweep (SpMV +
    M^-1 + CGS2, solve_bytes) over (a) the summed per-point solve times -- the average
    bandwidth of one point's solve, which shares the GPU with the concurrent points -- and (b)
    the sweep step (setup included: the whole-job rate).  Rank 0's points only."""
    peak, src = peaks()
    tot_b = tot_ms = 0.0
    for r in pinfo:
        si = {"nnz_L": r["nnz_L"], "nnz_U": r["nnz_U"]}
        tot_b += solve_bytes(si, {"n": r["n"], "nnz": r["nnz"]}, r["iterations"], r["restart"])
        tot_ms += r["solve_ms"]
    ach = tot_b / (tot_ms * 1e-3) / 1e9 if tot_ms else None
    return {"bound": "hbm", "kernel": "whole Arnoldi steps of each point's solve (SpMV + M^-1 + CGS2)",
            "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak if ach else None,
            "peak_source": src, "traffic": None, "points_rank0": len(pinfo), "bytes_rank0": tot_b,
            "solve_ms_sum_rank0": tot_ms,
            "achieved_over_step": tot_b * world / (ms_step * 1e-3) / 1e9 if ms_step else None,
            "note": "per-point solve bandwidth; the sweep step itself is bound by the host iLUTP setups"}


def run_sweep_bench(args):
    """configs[4]: the 64-point detuning sweep through sweep.run_sweep.  A step is the whole
    sweep: every rank builds, sets up and solves its contiguous shard, one Liouvillian at a
    time, and the observables of all points are all-gathered over NCCL.  Timed with CUDA
    events on the rank's stream around the step (host setup included: time to steady
    state), max over ranks; value = points of the whole job per second."""
    import torch
    import torch.distributed as dist

    import paper_1411_4356_b200 as pb
    from paper_1411_4356_b200.sweep import run_sweep, shard_range
    from workloads import SWEEP_BASE, sweep_params

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    import threading

    from paper_1411_4356_b200.sweep import concurrent_solver

    points = sweep_params()
    rec = {"solve_ms": 0.0, "iterations": 0, "points": 0}
    lock = threading.Lock()
    conc = max(1, min(args.concurrent, 8))
    pinfo: list = []
    inner = concurrent_solver(conc, info=pinfo)

    def solve(p):
        row = inner(p)
        with lock:
            rec["solve_ms"] += row[6]
            rec["iterations"] += row[3]
            rec["points"] += 1
        return row

    for _ in range(args.warmup):   # warm-up: one point of the rank's shard (context, kernels, allocator)
        solve(points[shard_range(len(points), rank, world).start])
    rec.update(solve_ms=0.0, iterations=0, points=0)
    pinfo.clear()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = pb.ss_kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    tab = None
    ms = 0.0
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tab = run_sweep(points, rank, world, group=group, solve=solve, concurrent=conc)
        e1.record(stream)
        e1.synchronize()
        ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = pb.ss_kernel_launches() - launches0
    tt = torch.tensor([ms, rec["solve_ms"], float(rec["iterations"])], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt[0:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:3], op=dist.ReduceOp.SUM)
    ms_max, solve_ms_sum, its_sum = [float(v) for v in tt.tolist()]
    if rank == 0:
        npts = len(points) * args.steps
        conv = int(np.nansum(tab[:, 5]))
        line = {
            "metric": METRIC, "value": npts / (ms_max * 1e-3), "unit": "steady states/s (64-point sweep)",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (BASELINE configs[4] parameter sweep)",
            "config": {"workload": "configs[4] sweep: 64 detunings in [-2, 2], N_c=8, N_m=60, Liouvillian dim 230400",
                       "N_c": SWEEP_BASE.N_c, "N_m": SWEEP_BASE.N_m, "drop_tol": SWEEP_BASE.drop_tol,
                       "fill_factor": SWEEP_BASE.fill_factor, "permtol": SWEEP_BASE.permtol,
                       "restart": SWEEP_BASE.restart, "tol": SWEEP_BASE.tol, "ranks": world,
                       "sharding": "contiguous blocks of points per rank; observables all-gathered (NCCL)",
                       "concurrent_per_gpu": conc,
                       "concurrency": "setups (host iLUTP) of concurrent_per_gpu points overlap; GMRES solves one at a time on the whole GPU",
                       "l2": "inputs (factors of every point) larger than L2"},
            "converged": conv, "points": len(points),
            "roofline": sweep_roofline(pinfo, ms_max / args.steps, world),
            "concurrent_per_gpu": conc,
            "gmres_iterations_per_s_per_point": its_sum / (solve_ms_sum * 1e-3) if solve_ms_sum else None,
            "solve_s_sum": solve_ms_sum * 1e-3,
            "table": {"fields": ["Delta", "n_cavity", "n_mech", "iterations", "rel_residual", "converged",
                                 "solve_ms"], "rows": tab.tolist()},
            "e2e": {"value": npts / (ms_max * 1e-3), "unit": "steady states/s (64-point sweep)",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": int(len(points) * 7 * 8),
                    "note": "parameters in, observables out: the step is already end to end"},
            "gpu_launches": int(launches), "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.cpu_baseline_only:
        print(json.dumps(cpu_baseline(args.cpu_baseline_only)), flush=True)
        return
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "sweep":
        run_sweep_bench(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
