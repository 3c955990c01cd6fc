"""Multi-rank host logic of the detuning sweep (paper_1411_4356_b200/sweep.py) over gloo.

The sweep shards independent parameter points (BASELINE configs[4]) over ranks and
gathers the observables; here the per-point GPU solve is replaced by a deterministic
stand-in so the sharding and the gather are checked on CPU with world size 2 and 3.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from workloads import sweep_params, SWEEP_POINTS


def fake_solve(p):
    # deterministic, point-dependent stand-in for one steady-state solve
    return (p.Delta, 0.1 + p.Delta ** 2, 1.0 + abs(p.Delta), 7.0, 1e-11, 1.0, 0.5)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, npoints, out_dir, explicit_device=False, concurrent=1):
    import torch
    import torch.distributed as dist

    from paper_1411_4356_b200.sweep import run_sweep

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pts = sweep_params(npoints)
        # explicit_device: the branch an NCCL group takes (gather from a tensor on a given
        # device, then back to the host); gloo can only use the CPU device
        table = run_sweep(pts, rank, world, solve=fake_solve,
                          device=torch.device("cpu") if explicit_device else None, concurrent=concurrent)
        np.save(os.path.join(out_dir, f"r{rank}.npy"), table)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,npoints,explicit_device,concurrent",
                         [(2, SWEEP_POINTS, False, 1), (3, 10, False, 1), (2, 1, False, 1),
                          (2, SWEEP_POINTS, True, 1), (3, SWEEP_POINTS, False, 4)])
def test_sweep_gather_gloo(tmp_path, world, npoints, explicit_device, concurrent):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, npoints, str(tmp_path), explicit_device, concurrent), nprocs=world,
             join=True)
    pts = sweep_params(npoints)
    ref = np.array([fake_solve(p) for p in pts])
    for r in range(world):
        t = np.load(tmp_path / f"r{r}.npy")
        assert t.shape == ref.shape
        assert np.array_equal(t, ref)   # every rank holds every point, exactly once


def test_shards_partition_the_points():
    from paper_1411_4356_b200.sweep import shard_range
    for n in (1, 5, 64):
        for w in (1, 2, 3, 8):
            seen = [k for r in range(w) for k in shard_range(n, r, w)]
            assert seen == list(range(n))


def test_sweep_points_match_baseline():
    pts = sweep_params()
    assert len(pts) == 64
    assert pts[0].Delta == -2.0 and pts[-1].Delta == 2.0
    d = np.diff([p.Delta for p in pts])
    assert np.allclose(d, 4.0 / 63)
    assert all(p.N_c == 8 and p.N_m == 60 and p.liouvillian_dim == 230400 for p in pts)


def test_concurrent_threads_fill_the_same_table():
    """concurrent > 1 hands the rank's points to host threads: every point solved once,
    each row where the sequential sweep puts it."""
    import threading

    from paper_1411_4356_b200.sweep import run_sweep
    pts = sweep_params(13)
    seen = []
    lock = threading.Lock()

    def solve(p):
        with lock:
            seen.append(p.Delta)
        return fake_solve(p)

    seq = run_sweep(pts, solve=fake_solve)
    con = run_sweep(pts, solve=solve, concurrent=4)
    assert np.array_equal(seq, con)
    assert sorted(seen) == sorted(p.Delta for p in pts)
