"""Config 4 through the drop-in object API (dev tool).

  python tools/object_api_probe.py [--nvars N] [--out FILE]

Builds the config-4 trace as the reference's own objects (a Trace of 4 M
TraceEvent, names "v<id>"), then times each layer a user of
``PoolPlanner().fit(trace)`` goes through: the Trace -> columns conversion
(host Python, cached on the Trace while its event list is unchanged), the
estimator fit (device plan + the Python-side profile, plan dict and lookup
table the reference API returns), a second fit on the same Trace (cached
columns), and the columnar ``plan_arrays`` call the bench's headline uses.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1903_06631_b200 import workloads  # noqa: E402
from paper_1903_06631_b200.estimators import PoolPlanner  # noqa: E402
from paper_1903_06631_b200.pipeline import plan_arrays  # noqa: E402
from paper_1903_06631_b200.trace import EventKind, Trace, TraceEvent, as_arrays  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nvars", type=int, default=1_000_000)
    ap.add_argument("--out", default=None)
    ap.add_argument("--profile", action="store_true", help="cProfile a third fit (top functions by own time)")
    a = ap.parse_args()
    arrays, window = workloads.interval_trace(a.nvars, seed=0)
    kinds = [EventKind.MALLOC, EventKind.FREE, EventKind.READ, EventKind.WRITE]
    t0 = time.perf_counter()
    names = arrays.names
    ev = [TraceEvent(i, int(t), kinds[k], names[v], int(s))
          for i, (t, k, v, s) in enumerate(zip(arrays.t_us.tolist(), arrays.kind.tolist(),
                                                arrays.var.tolist(), arrays.size.tolist()))]
    trace = Trace(ev)
    build_s = time.perf_counter() - t0
    n = len(trace)

    t0 = time.perf_counter()
    cols = as_arrays(trace)
    conv_s = time.perf_counter() - t0
    assert np.array_equal(cols.var, arrays.var) and np.array_equal(cols.size, arrays.size)

    t0 = time.perf_counter()
    pp = PoolPlanner().fit(trace)
    fit1_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    pp2 = PoolPlanner().fit(trace)
    fit2_s = time.perf_counter() - t0
    assert pp2.footprint_bytes_ == pp.footprint_bytes_

    if a.profile:
        import cProfile
        import pstats
        pr = cProfile.Profile()
        pr.enable()
        PoolPlanner().fit(trace)
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(14)
    plan_arrays(arrays)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        pl = plan_arrays(arrays)
        ts.append(time.perf_counter() - t0)
    cols_ms = float(np.median(ts)) * 1e3
    res = {
        "workload": f"interval_trace_{a.nvars} (BASELINE configs[3]) as {n} TraceEvent objects",
        "events": n,
        "build_objects_s": round(build_s, 3),
        "trace_to_columns_s": round(conv_s, 3),
        "poolplanner_fit_first_s": round(fit1_s, 3),
        "poolplanner_fit_cached_columns_s": round(fit2_s, 3),
        "plan_arrays_ms": round(cols_ms, 3),
        "footprint_bytes": int(pp.footprint_bytes_),
        "footprint_equal_plan_arrays": int(pp.footprint_bytes_) == int(pl.footprint_bytes),
        "lookup_entries": len(pp.lookup_),
    }
    print(json.dumps(res))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
