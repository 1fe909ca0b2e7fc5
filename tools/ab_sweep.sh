#!/bin/bash
# Interleaved A/B of ab/ library variants on the config-5 sweep kernel time
R=$1; shift
for r in $(seq $R); do
  for n in "$@"; do
    printf "%-8s " $n
    MEMPLAN_LIB=paper_1903_06631_b200/ab/lib_$n.so python - <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1903_06631_b200 import _native as N, sweep, workloads
batch = sweep.SweepBatch.from_traces(workloads.sweep_traces())
ds = sweep.DeviceSweep(batch)
prm = sweep.SweepParams(budgets=workloads.SWEEP_BUDGETS)
stream = torch.cuda.ExternalStream(N.stream_ptr())
ts = []
for i in range(12):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream); ds.run(prm); e.record(stream); e.synchronize()
    if i >= 2: ts.append(s.elapsed_time(e))
print(f"{np.median(ts):.4f} ms (min {min(ts):.4f})")
PY
  done
done
