"""Host-side breakdown of the single-trace plan call (BASELINE configs[0]):
where the microseconds of pipeline.plan_arrays on the ResNet-50 b32 trace go.

    python tools/c1_probe.py [--reps 200]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]

import numpy as np  # noqa: E402

from paper_1903_06631_b200 import _native as N  # noqa: E402
from paper_1903_06631_b200 import sweep, synth, workloads  # noqa: E402
from paper_1903_06631_b200.pipeline import plan_arrays  # noqa: E402
from paper_1903_06631_b200.trace import as_arrays  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=200)
a = ap.parse_args()
arrays = as_arrays(synth.generate_synthetic_trace(workloads.resnet50_spec(32)))
prm = sweep.SweepParams(budgets=())
for _ in range(10):
    plan_arrays(arrays)
N.sync()
tt = {k: [] for k in ("from_traces", "upload", "run", "sync", "download", "close", "plan_arrays")}
for _ in range(a.reps):
    t0 = time.perf_counter()
    b = sweep.SweepBatch.from_traces([arrays])
    t1 = time.perf_counter()
    ds = sweep.DeviceSweep(b)
    t2 = time.perf_counter()
    ds.run(prm)
    t3 = time.perf_counter()
    N.sync()
    t4 = time.perf_counter()
    ds.download()
    t5 = time.perf_counter()
    ds.close()
    t6 = time.perf_counter()
    plan_arrays(arrays)
    N.sync()
    t7 = time.perf_counter()
    for k, v in zip(tt, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5, t7 - t6)):
        tt[k].append(v * 1e6)
for k, v in tt.items():
    print(f"{k:12s} median {np.median(v):8.1f} us  p90 {np.percentile(v, 90):8.1f} us")
