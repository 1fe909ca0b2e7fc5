"""Host-side sweep logic on CPU: batch packing, LPT sharding, the sharded
runner's gather over gloo (world size 2) with the oracle standing in for the
per-rank device run (the product never calls the oracle)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
from paper_1903_06631_b200 import sweep, workloads
from paper_1903_06631_b200.trace import as_arrays


def oracle_runner(batch, params):
    recs, brecs, offs, orders = orc.sweep(batch, params)
    Nev = int(batch.ev_off[-1])
    o = np.zeros(max(Nev, 1), np.int64)
    c = np.zeros(max(Nev, 1), np.int32)
    for t in range(batch.ntraces):
        e0 = int(batch.ev_off[t])
        o[e0:e0 + len(offs[t])] = offs[t]
        c[e0:e0 + len(orders[t])] = orders[t]
    return sweep.SweepResult(recs, brecs, o[:Nev], c[:Nev], batch.ev_off, params, batch)


def test_batch_round_trips_every_trace():
    traces = workloads.sweep_traces(n_models=5, n_scales=2)
    batch = sweep.SweepBatch.from_traces(traces)
    assert batch.ntraces == 10
    for t, tr in enumerate(traces):
        a, b = as_arrays(tr), batch.trace(t)
        assert a.names == b.names
        for col in ("kind", "var", "size", "t_us"):
            assert np.array_equal(getattr(a, col), getattr(b, col))
    sub = batch.subset([7, 2])
    assert sub.ntraces == 2 and sub.trace(0).names == batch.trace(7).names


def test_shard_is_a_balanced_deterministic_partition():
    rng = np.random.default_rng(0)
    costs = rng.integers(100, 3000, size=1024).tolist()
    for world in (1, 2, 4, 8):
        parts = sweep.shard(costs, world)
        assert parts == sweep.shard(costs, world)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(1024))
        loads = [sum(costs[i] for i in p) for p in parts]
        # LPT: within the largest unit of the ideal share
        assert max(loads) - min(loads) <= max(costs)
    assert sweep.shard([5, 1], 4)[2:] == [[], []]


def test_params_validation():
    with pytest.raises(ValueError):
        sweep.SweepParams(policy="worst_fit").struct()
    with pytest.raises(ValueError):
        sweep.SweepParams(budgets=(0.9,) * 9).struct()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    batch = sweep.SweepBatch.from_traces(workloads.sweep_traces(n_models=6, n_scales=3))
    res = sweep.run_sweep_sharded(batch, sweep.SweepParams(), rank, world, runner=oracle_runner)
    if rank == 0:
        np.save(out + ".traces.npy", res.traces)
        np.save(out + ".budgets.npy", res.budgets)
        np.save(out + ".offsets.npy", res.offsets)
    else:
        assert res is None
    dist.destroy_process_group()


def test_sharded_sweep_gathers_over_gloo(tmp_path):
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    batch = sweep.SweepBatch.from_traces(workloads.sweep_traces(n_models=6, n_scales=3))
    whole = oracle_runner(batch, sweep.SweepParams())
    assert np.load(out + ".traces.npy").tobytes() == whole.traces.tobytes()
    assert np.load(out + ".budgets.npy").tobytes() == whole.budgets.tobytes()
    assert np.array_equal(np.load(out + ".offsets.npy"), whole.offsets)


def test_bench_launcher_runs_the_sharded_sweep_on_two_ranks(tmp_path):
    """bench.py --gpus N re-launches itself with bench.torchrun_cmd; the same
    launch line drives a 2-rank gloo sweep whose gathered records equal one
    process planning the whole batch."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    out = str(tmp_path / "res")
    cmd = bench.torchrun_cmd(2, os.path.join(root, "tests", "_torchrun_sweep_worker.py"), [out])
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1" and "--nproc-per-node=2" in cmd
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    subprocess.run(cmd, check=True, timeout=300, env=env, cwd=root)
    batch = sweep.SweepBatch.from_traces(workloads.sweep_traces(n_models=6, n_scales=3))
    whole = oracle_runner(batch, sweep.SweepParams())
    assert np.load(out + ".traces.npy").tobytes() == whole.traces.tobytes()
    assert np.load(out + ".budgets.npy").tobytes() == whole.budgets.tobytes()
    assert np.array_equal(np.load(out + ".offsets.npy"), whole.offsets)
