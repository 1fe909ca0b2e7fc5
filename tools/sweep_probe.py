"""Run the config-5 sweep kernel a few times (for ncu captures)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]

from paper_1903_06631_b200 import _native as N  # noqa: E402
from paper_1903_06631_b200 import sweep, workloads  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
batch = sweep.SweepBatch.from_traces(workloads.sweep_traces())
ds = sweep.DeviceSweep(batch)
for _ in range(reps):
    ds.run(sweep.SweepParams(budgets=workloads.SWEEP_BUDGETS))
N.sync()
print("ok", batch.ntraces)
