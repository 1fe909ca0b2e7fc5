"""Per-stage device timing of the pool path on the config-4 interval trace.

Usage: python tools/stage_probe.py [--nvars N] [--accesses] [--oracle]
Prints per-stage device ms (CUDA events on the library stream) and checks
the plan against the CPU oracle when --oracle is given.
"""
import argparse
import hashlib
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import numpy as np  # noqa: E402

from paper_1903_06631_b200 import _native as N  # noqa: E402
from paper_1903_06631_b200 import workloads  # noqa: E402
from paper_1903_06631_b200.pipeline import plan_arrays  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nvars", type=int, default=1_000_000)
ap.add_argument("--accesses", action="store_true")
ap.add_argument("--oracle", action="store_true")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--max-size", type=int, default=64 << 20, help="largest variable size (bytes)")
a = ap.parse_args()
t0 = time.time()
arrays, window = workloads.interval_trace(a.nvars, seed=0, accesses=a.accesses, max_size=a.max_size)
print(f"trace n={len(arrays)} window={window} built in {time.time() - t0:.1f}s", flush=True)
for _ in range(2):
    plan = plan_arrays(arrays)
N.sync()
N.set_timing(True)
walls = []
for _ in range(a.reps):
    t0 = time.perf_counter()
    plan = plan_arrays(arrays)
    N.sync()
    walls.append(time.perf_counter() - t0)
tm = N.timings()
N.set_timing(False)
print(f"plan: period={plan.period} nvars={plan.nvars} nnz={plan.nnz} levels={plan.levels} "
      f"peak={plan.peak_bytes} footprint={plan.footprint_bytes} alpha={plan.competitive_ratio:.6f}")
tot = sum(v[0] for v in tm.values()) / a.reps
for k, (ms, c) in tm.items():
    print(f"  {k:14s} {ms / a.reps:9.3f} ms/step  ({c // a.reps} intervals/step) {100 * ms / a.reps / tot:5.1f}%")
print(f"  staged total {tot:.3f} ms; wall per step {1e3 * min(walls):.3f} ms; "
      f"{plan.nvars / min(walls) / 1e6:.2f} M vars/s (wall)")
sha = hashlib.sha256(plan.offsets.tobytes()).hexdigest()[:16]
print("offsets sha", sha)
if a.oracle:
    import oracle as orc
    t0 = time.perf_counter()
    rc, p = orc.detect(arrays)
    t1 = time.perf_counter()
    rc, fp = orc.extract(arrays, len(arrays) - p, len(arrays))
    t2 = time.perf_counter()
    off, lo, hi = orc.profile_segments(fp)
    h, row, col = orc.conflict(off, lo, hi)
    t3 = time.perf_counter()
    rc, offs, foot = orc.plan(h, fp.size, fp.alloc.astype(np.int64), fp.base, fp.name_ralloc(),
                              fp.name_blob, fp.name_off, 1)
    t4 = time.perf_counter()
    print(f"oracle: detect {t1 - t0:.2f}s extract {t2 - t1:.2f}s conflict {t3 - t2:.2f}s plan {t4 - t3:.2f}s "
          f"total {t4 - t0:.2f}s -> {fp.nvars / (t4 - t0):.0f} vars/s; footprint {foot}; nnz {row[-1]}")
    print("PARITY offsets", np.array_equal(offs, plan.offsets), "footprint", foot == plan.footprint_bytes,
          "peak", fp.peak_bytes == plan.peak_bytes)
