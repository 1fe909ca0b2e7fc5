"""Device sweep vs the CPU oracle on config-5 style batches (dev tool).

  python tools/sweep_check.py [--models M] [--scales S] [--policy best_fit] [--bw 12e9]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import numpy as np  # noqa: E402

import oracle as orc  # noqa: E402
from paper_1903_06631_b200 import sweep, workloads  # noqa: E402


def compare(res, recs, brecs, offs, orders, limit=10):
    bad = 0
    for t in range(len(recs)):
        a, b = res.traces[t], recs[t]
        if a.tobytes() != b.tobytes():
            bad += 1
            if bad <= limit:
                print("trace", t, "\n dev", a, "\n orc", b)
            continue
        if not np.array_equal(res.offsets_of(t), offs[t]):
            bad += 1
            if bad <= limit:
                print("offsets", t, res.offsets_of(t)[:10], offs[t][:10])
            continue
        if not np.array_equal(res.order_of(t), orders[t]):
            bad += 1
            if bad <= limit:
                print("order", t, res.order_of(t), orders[t])
            continue
        if res.budgets[t].tobytes() != brecs[t].tobytes():
            bad += 1
            if bad <= limit:
                print("budgets", t, "\n dev", res.budgets[t], "\n orc", brecs[t])
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", type=int, default=64)
    ap.add_argument("--scales", type=int, default=16)
    ap.add_argument("--policy", default="best_fit")
    ap.add_argument("--bw", type=float, default=12e9)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    tr = workloads.sweep_traces(args.models, args.scales)
    batch = sweep.SweepBatch.from_traces(tr)
    prm = sweep.SweepParams(policy=args.policy, bandwidth_bytes_per_s=args.bw)
    ds = sweep.DeviceSweep(batch)
    import torch
    from paper_1903_06631_b200 import _native as N
    stream = torch.cuda.ExternalStream(N.stream_ptr())
    times = []
    for _ in range(args.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        ds.run(prm)
        e.record(stream)
        e.synchronize()
        times.append(s.elapsed_time(e))
    res = ds.download()
    ds.set_profile(True)
    ds.run(prm)
    prof = ds.profile()
    names = ("group+validate+detect", "extract+loads", "prep+cand+loadmin", "greedy", "sim prep+publish", "to join", "tail")
    tot = prof.sum(axis=1)
    top = np.argsort(-tot)[:5]
    print("phase cycles: median over traces / the 5 slowest traces")
    for j, nm in enumerate(names):
        print(f"  {nm:24s} med {int(np.median(prof[:, j])):>9d}  " + " ".join(f"{int(prof[t, j]):>9d}" for t in top))
    ex = ds.profile_extra
    raw = ds.profile_raw
    print("  placement start / end after CTA start (5 slowest):",
          [(int(raw[t, 8] - raw[t, 0]), int(raw[t, 9] - raw[t, 0])) for t in top], "CTA end",
          [int(raw[t, 7] - raw[t, 0]) for t in top])
    print("  placement loop cycles (5 slowest):", [int(ex[t, 1] - ex[t, 0]) for t in top],
          "scan", [int(ex[t, 2]) for t in top], "insert", [int(ex[t, 3]) for t in top])
    print("  budget 0 (5 slowest): sched+overlay", [int(ex[t, 4]) for t in top], "replay", [int(ex[t, 5]) for t in top],
          "rounds", [int(ex[t, 6]) for t in top], "nsel", [int(ex[t, 7]) for t in top])
    print("  slowest traces:", [(int(t), batch.events_of(int(t)), int(res.traces['nvars'][t]), int(res.traces['ncand'][t])) for t in top])
    t0 = time.perf_counter()
    recs, brecs, offs, orders = orc.sweep(batch, prm)
    tc = time.perf_counter() - t0
    bad = compare(res, recs, brecs, offs, orders)
    print(f"traces={batch.ntraces} device ms={times} oracle s={tc:.3f} mismatching units={bad}")
    print("budget status", np.unique(res.budgets["status"], return_counts=True))


if __name__ == "__main__":
    main()
