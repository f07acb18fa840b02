"""N > 1 path with real engines on ONE GPU: two gloo ranks, each with its own BatchEngine on cuda:0, shard a
batch by contiguous solve-index range through sharding.solve_sharded; rank 0's gathered result must be
bitwise the unsharded solve (the analogue of pkg/tests/test_batch.py:48-57: worker counts do not change
results).  Also: batch_solve(devices=[0, 0]) (two shards in one process), and `bench.py --gpus 2` launched
WITHOUT torchrun must spawn its two ranks itself and report n_gpus = 2."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

M_TOTAL, N, H, ITERS = 7, 16, 0.02, 3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    import paper_2510_07625_b200 as gb
    from paper_2510_07625_b200 import sharding, workloads
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        batch = workloads.iiwa14_reach_arrays(M_TOTAL, N)
        lo, hi = sharding.shard_bounds(M_TOTAL, world)[rank]
        eng = gb.BatchEngine(gb.Iiwa14(), hi - lo, N, H, workloads.fixed_budget_settings(ITERS))
        try:
            res = sharding.solve_sharded(batch, eng.solve, rank, world)
        finally:
            eng.close()
        if rank == 0:
            np.savez(out_path, X=res.X, U=res.U, trace=res.trace, info=res.info)
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_engines_shard_and_gather_equals_unsharded(tmp_path):
    import torch.multiprocessing as mp

    import paper_2510_07625_b200 as gb
    from paper_2510_07625_b200 import workloads
    out = tmp_path / "gathered.npz"
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    got = np.load(out)
    batch = workloads.iiwa14_reach_arrays(M_TOTAL, N)
    eng = gb.BatchEngine(gb.Iiwa14(), M_TOTAL, N, H, workloads.fixed_budget_settings(ITERS))
    try:
        whole = eng.solve(batch)
    finally:
        eng.close()
    assert got["X"].shape[0] == M_TOTAL
    assert np.array_equal(got["X"], whole.X) and np.array_equal(got["U"], whole.U)
    assert np.array_equal(got["trace"], whole.trace, equal_nan=True) and np.array_equal(got["info"], whole.info)


def test_batch_solve_two_shards_in_one_process():
    """batch_solve(devices=[0, 0]): two shards of one call on the same device use two engines (not one engine
    twice) and give the single-shard result bit for bit."""
    import paper_2510_07625_b200 as gb
    from paper_2510_07625_b200 import workloads
    batch = workloads.iiwa14_reach_arrays(6, 8)
    spec = workloads.arrays_to_spec(batch, H, workloads.fixed_budget_settings(2))
    one = gb.batch_solve(spec)
    two = gb.batch_solve(spec, devices=[0, 0])
    assert one.ok and two.ok
    for a, b in zip(one.results, two.results):
        assert np.array_equal(a.X, b.X) and np.array_equal(a.U, b.U)
        assert [r.pcg_iterations for r in a.trace] == [r.pcg_iterations for r in b.trace]
    gb.batch.clear_engine_cache()


@pytest.mark.timeout(900)
def test_bench_gpus_2_spawns_two_ranks():
    """`python bench.py --gpus 2` without torchrun's environment launches its own two ranks; on a one-GPU box
    they share the device and talk through gloo."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    env["GATO_DIST_BACKEND"] = "gloo"
    proc = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1",
                           "--batch", "16", "--no-cpu-baseline"], env=env, capture_output=True, text=True,
                          timeout=850, cwd=str(ROOT))
    assert proc.returncode == 0, proc.stdout[-2000:] + proc.stderr[-2000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, proc.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["dist"]["ranks"] == 2 and line["dist"]["backend"] == "gloo"
    assert line["config"]["global_batch"] == 32 and line["dist"]["gathered_rows"] == 32
    assert line["all_solves_ok"] and line["stream_launch_check"]["bitwise_equal"]
    assert line["strong"]["global_batch"] == 4096 and line["strong"]["gathered_rows"] == 4096
    assert line["n1"]["weak"]["value"] > 0 and line["n1"]["strong"]["value"] > 0
    assert line["value"] > 0 and line["e2e"]["value"] > 0
