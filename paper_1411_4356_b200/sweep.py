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


def solve_point_gpu(p) -> tuple:
    """Build -> setup -> solve -> expect one parameter point on the current CUDA device."""
    from . import SteadyState

    s = SteadyState(p).setup().solve()
    try:
        na, nb = s.expect()
        i = s.solve_info
        return (p.Delta, na, nb, i["iterations"], i["rel_residual"], i["converged"], i["solve_ms"])
    finally:
        s.close()


def run_sweep(points: Sequence, rank: int = 0, world: int = 1, group=None,
              solve: Callable = solve_point_gpu, device=None) -> np.ndarray:
    """Solve this rank's shard of ``points`` and return the full (npoints x len(FIELDS))
    table on every rank.  ``group`` is a torch.distributed process group (None with
    world == 1).  ``solve(p)`` returns one FIELDS tuple; it is injectable so the host
    logic runs in tests without a GPU."""
    import torch

    n = len(points)
    local = np.full((n, len(FIELDS)), np.nan)
    for k in shard_range(n, rank, world):
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
