"""Run the config-5 sweep kernel on its largest trace alone (for ncu)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_1903_06631_b200 import _native as N, sweep, workloads  # noqa: E402
batch = sweep.SweepBatch.from_traces(workloads.sweep_traces())
prm = sweep.SweepParams(budgets=workloads.SWEEP_BUDGETS)
big = int(np.argmax([batch.events_of(t) for t in range(batch.ntraces)]))
ds = sweep.DeviceSweep(batch.subset([big]))
for _ in range(3):
    ds.run(prm)
N.sync()
print("ok")
