"""One rank of the sharded sweep under torchrun (env rendezvous, gloo), with
the C oracle standing in for the per-rank device run — launched by
test_cpu_sweep.py through bench.torchrun_cmd, the launcher `bench.py --gpus N`
uses.  Rank 0 saves the gathered records to argv[1]."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.join(os.path.dirname(HERE), "oracle"), HERE]

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1903_06631_b200 import sweep, workloads  # noqa: E402
from test_cpu_sweep import oracle_runner  # noqa: E402

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
assert world == int(os.environ["WORLD_SIZE"]) == 2
batch = sweep.SweepBatch.from_traces(workloads.sweep_traces(n_models=6, n_scales=3))
res = sweep.run_sweep_sharded(batch, sweep.SweepParams(), rank, world, runner=oracle_runner)
if rank == 0:
    np.save(sys.argv[1] + ".traces.npy", res.traces)
    np.save(sys.argv[1] + ".budgets.npy", res.budgets)
    np.save(sys.argv[1] + ".offsets.npy", res.offsets)
else:
    assert res is None
dist.destroy_process_group()
