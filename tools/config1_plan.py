"""Config 1 (BASELINE configs[0]): SmartPool plan of the ResNet-50 b32
trace — the per-trace device path (plan_arrays), the same trace as a
one-trace sweep, and the C oracle on one host core; bit-exact check.

  python tools/config1_plan.py [--reps 50]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import numpy as np  # noqa: E402

import oracle as orc  # noqa: E402
from paper_1903_06631_b200 import _native as N  # noqa: E402
from paper_1903_06631_b200 import sweep, synth, workloads  # noqa: E402
from paper_1903_06631_b200.pipeline import plan_arrays  # noqa: E402
from paper_1903_06631_b200.trace import as_arrays  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    tr = synth.generate_synthetic_trace(workloads.resnet50_spec(32))
    arrays = as_arrays(tr)
    def timed(path):
        for _ in range(3):
            plan_arrays(arrays, path=path)
        N.sync()
        t0 = time.perf_counter()
        for _ in range(args.reps):
            pl = plan_arrays(arrays, path=path)
        return pl, (time.perf_counter() - t0) / args.reps

    plan, per_trace = timed("auto")
    gplan, grid_s = timed("grid")
    batch = sweep.SweepBatch.from_traces([arrays])
    prm = sweep.SweepParams(budgets=())
    ds = sweep.DeviceSweep(batch)
    for _ in range(3):
        ds.run(prm)
    N.sync()
    t0 = time.perf_counter()
    for _ in range(args.reps):
        ds.run(prm)
    N.sync()
    one_sweep = (time.perf_counter() - t0) / args.reps
    res = ds.download()
    # the C oracle: detect + extract + conflict + plan, one core
    t0 = time.perf_counter()
    rc, p = orc.detect(arrays)
    rc, fp = orc.extract(arrays, len(arrays) - p, len(arrays))
    off, lo, hi = orc.profile_segments(fp)
    h, _r, _c = orc.conflict(off, lo, hi)
    rc, offs, foot = orc.plan(h, fp.size, fp.alloc.astype(np.int64), fp.base, fp.name_ralloc(), fp.name_blob,
                              fp.name_off, 1)
    oracle_s = time.perf_counter() - t0
    orc.graph_free(h)
    out = {"config": "resnet50_b32 (BASELINE configs[0])", "events": len(arrays), "period": plan.period,
           "nvars": plan.nvars, "edges": plan.nnz // 2, "peak_bytes": plan.peak_bytes,
           "footprint_bytes": plan.footprint_bytes, "alpha": plan.competitive_ratio,
           "plan_arrays_us": per_trace * 1e6, "grid_stages_us": grid_s * 1e6,
           "one_trace_sweep_kernel_us": one_sweep * 1e6,
           "oracle_1core_us": oracle_s * 1e6,
           "parity": {"offsets": bool(np.array_equal(offs, plan.offsets)), "footprint": foot == plan.footprint_bytes,
                      "peak": fp.peak_bytes == plan.peak_bytes,
                      "sweep_offsets": bool(np.array_equal(res.offsets_of(0), plan.offsets)),
                      "grid_offsets": bool(np.array_equal(gplan.offsets, plan.offsets))}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
