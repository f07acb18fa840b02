"""N>1 path on CPU: two gloo ranks shard a batch by solve index, each solves its contiguous
range (with the oracle standing in for the rank's GPU engine) and rank 0 gathers.  The
gathered result must equal the unsharded one bitwise and be in input order."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _oracle_engine(h, settings):
    """solve_fn with the PackedBatch -> PackedResult contract of BatchEngine.solve."""
    from oracle import trajopt_np as orc
    from oracle.iiwa14_np import Iiwa14
    from paper_2510_07625_b200.engine import PackedResult

    def solve(batch):
        M = batch.size
        max_it = settings.max_sqp_iterations
        X, U = batch.X.copy(), batch.U.copy()
        trace = np.zeros((M, max_it, 8))
        info = np.zeros((M, 8), dtype=np.int32)
        for b in range(M):
            p = orc.Problem(Iiwa14(), batch.Q[b], batch.R[b], batch.QN[b], batch.goal[b], X.shape[1] - 1, h,
                            batch.x_start[b], batch.force[b])
            import dataclasses
            res = orc.solve(p, batch.X[b], batch.U[b], dataclasses.replace(settings, rho_init=float(batch.rho_init[b])))
            X[b], U[b] = res.X, res.U
            for r in res.trace:
                trace[b, r.iteration] = [r.merit, r.constraint_l1, np.nan if r.alpha is None else r.alpha, r.rho,
                                         r.pcg_iterations, float(r.accepted), r.step_inf_norm, r.iteration]
            info[b, 0], info[b, 1] = len(res.trace), int(res.converged)
        return PackedResult(X, U, trace, info, 1.0 + M)
    return solve


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, str(ROOT))
    from oracle import trajopt_np as orc
    from paper_2510_07625_b200 import sharding, workloads
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        batch = workloads.iiwa14_reach_arrays(5, 4)
        settings = orc.Settings(max_sqp_iterations=2, step_tolerance=None, pcg_tolerance=1e-6)
        res = sharding.solve_sharded(batch, _oracle_engine(0.02, settings), rank, world)
        if rank == 0:
            np.savez(out_path, X=res.X, U=res.U, trace=res.trace, info=res.info, ms=res.device_ms)
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(600)
def test_two_rank_shard_and_gather_equals_unsharded(tmp_path):
    from oracle import trajopt_np as orc
    from paper_2510_07625_b200 import sharding, workloads
    out = tmp_path / "gathered.npz"
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    got = np.load(out)
    batch = workloads.iiwa14_reach_arrays(5, 4)
    settings = orc.Settings(max_sqp_iterations=2, step_tolerance=None, pcg_tolerance=1e-6)
    whole = _oracle_engine(0.02, settings)(batch)
    assert np.array_equal(got["X"], whole.X) and np.array_equal(got["U"], whole.U)
    assert np.array_equal(got["trace"], whole.trace, equal_nan=True) and np.array_equal(got["info"], whole.info)
    # shards [0,2) and [2,5): device time is the max over ranks
    assert float(got["ms"]) == 4.0
    assert sharding.local_shard(batch, 1, 2)[1] == (2, 5)


def test_sharded_solve_rejects_more_ranks_than_solves():
    from paper_2510_07625_b200 import sharding, workloads
    with pytest.raises(ValueError):
        sharding.solve_sharded(workloads.iiwa14_reach_arrays(1, 4), lambda b: None, 0, 2)
