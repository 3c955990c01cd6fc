"""Detuning sweep across the GPUs of one node (BASELINE.json configs[4], north star).

Every point of the sweep is an independent steady-state problem (its own Liouvillian,
RCM order, ILU factors and GMRES solve), so the work shards over ranks with no
data-path collective: rank r solves the contiguous block ``workloads.shard(points, r, W)``
one Liouvillian at a time on its own GPU, and the observables <a^+a>, <b^+b> (plus the
iteration count and final residual) of all points are gathered at the end with one
``all_gather`` over the process group (NCCL on GPUs; the host logic is tested over gloo).

PAPER.md:147 -- "the reduced memory footprint of iterative methods, allowing for several
simulations to be run in parallel" -- is the motivation; the paper's Fig. 4 sweeps the
detuning the same way.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

# Row of the gathered table for one point: Delta, <a^+a>, <b^+b>, iterations, rel. residual,
# converged, solve ms.  A point a rank does not own is NaN in its local table.
FIELDS = ("Delta", "n_cavity", "n_mech", "iterations", "rel_residual", "converged", "solve_ms")


def shard_range(npoints: int, rank: int, world: int) -> range:
    """Contiguous block sharding (same rule as workloads.shard)."""
    lo = (npoints * rank) // world
    hi = (npoints * (rank + 1)) // world
    return range(lo, hi)


def solve_point_gpu(p, concurrent: int = 1, host_threads: int = 0, stream=None, info: list | None = None,
                    solve_lock=None) -> tuple:
    """Build -> setup -> solve -> expect one parameter point on the current CUDA device.

    concurrent > 1: this point shares the GPU with concurrent - 1 others handled by other
    host threads at the same time, on its own stream.  With ``solve_lock`` (the default of
    ``concurrent_solver``) only the setups overlap -- the host-bound iLUTP is ~95 % of a
    sweep point -- and the GMRES solves take the whole GPU one at a time.  Without it the
    solves overlap too: the substitution kernels of this point get 1/concurrent of the
    co-resident clusters (ss_set_sm_budget; the budgets add up to at most the GPU, so the
    persistent launches of different points never wait on one another)."""
    import contextlib

    from . import SteadyState, ss_set_sm_budget

    s = SteadyState(p, stream=stream).setup(threads=host_threads)
    try:
        if concurrent > 1 and solve_lock is None:
            clusters = s.setup_info["trsv_grid"] // 8          # co-resident clusters (whole GPU)
            ss_set_sm_budget(s.handle, 8 * max(2, clusters // concurrent))
        with solve_lock if solve_lock is not None else contextlib.nullcontext():
            s.solve()
            na, nb = s.expect()
        i = s.solve_info
        if info is not None:   # (list.append is atomic: safe from several host threads)
            info.append({"Delta": p.Delta, "n": s.n, "nnz": s.build_info["nnz"], "nnz_L": s.setup_info["nnz_L"],
                         "nnz_U": s.setup_info["nnz_U"], "iterations": i["iterations"], "restart": p.restart,
                         "solve_ms": i["solve_ms"]})
        return (p.Delta, na, nb, i["iterations"], i["rel_residual"], i["converged"], i["solve_ms"])
    finally:
        s.close()


def concurrent_solver(concurrent: int, host_cores: int | None = None, info: list | None = None,
                      overlap_solves: bool = False) -> Callable:
    """A solve(p) for run_sweep that may be called from `concurrent` host threads at once:
    each call on the calling thread's own CUDA stream (same device as the caller of
    run_sweep), with 1/concurrent of the host cores for its iLUTP setup.  The solves run
    one at a time on the whole GPU (a lock) while the other points' setups go on;
    ``overlap_solves=True`` lets them share the GPU instead (1/concurrent of the
    co-resident clusters each) -- kept for diagnostics: in two 64-point runs of that mode
    one point each (a different one) lost its first M^-1 application."""
    import os
    import threading

    import torch

    dev = torch.cuda.current_device()
    cores = host_cores or os.cpu_count() or 1
    local = threading.local()
    lock = None if overlap_solves else threading.Lock()

    def solve(p):
        torch.cuda.set_device(dev)
        if not hasattr(local, "stream"):
            local.stream = torch.cuda.Stream(device=dev)
        return solve_point_gpu(p, concurrent, max(1, cores // concurrent), local.stream, info, lock)

    return solve


def run_sweep(points: Sequence, rank: int = 0, world: int = 1, group=None,
              solve: Callable = solve_point_gpu, device=None, concurrent: int = 1) -> np.ndarray:
    """Solve this rank's shard of ``points`` and return the full (npoints x len(FIELDS))
    table on every rank.  ``group`` is a torch.distributed process group (None with
    world == 1).  ``solve(p)`` returns one FIELDS tuple; it is injectable so the host
    logic runs in tests without a GPU.  concurrent > 1: the shard's points are handed
    out in order to that many host threads calling ``solve`` at once (with the GPU
    solver: ``concurrent_solver(concurrent)``)."""
    import torch

    n = len(points)
    local = np.full((n, len(FIELDS)), np.nan)
    mine = list(shard_range(n, rank, world))
    if concurrent > 1 and len(mine) > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=concurrent) as ex:
            for k, row in zip(mine, ex.map(lambda k: solve(points[k]), mine)):
                local[k] = row
    else:
        for k in mine:
            local[k] = solve(points[k])
    if world == 1:
        return local
    import torch.distributed as dist

    if device is None and dist.get_backend(group) == "nccl":   # NCCL gathers device tensors only
        device = torch.device("cuda", torch.cuda.current_device())
    t = torch.from_numpy(local)
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    full = np.full_like(local, np.nan)
    for r in range(world):
        rows = shard_range(n, r, world)
        full[rows.start:rows.stop] = parts[r].cpu().numpy()[rows.start:rows.stop]
    return full
