"""Where the placement kernel's time goes: per DAG level, how many variables
it holds and when (device %globaltimer) its first and last variable were
placed; plus the placement rate over time.

    python tools/place_trace.py [--nvars N]

Runs the config-4 pool path once with MP_PLACE_TRACE set (a debug dump the
placement launch writes: level and completion time per variable).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]

import numpy as np  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nvars", type=int, default=1_000_000)
ap.add_argument("--out", default="gpurun_out/place_trace.bin")
a = ap.parse_args()

from paper_1903_06631_b200 import workloads  # noqa: E402
from paper_1903_06631_b200.pipeline import plan_arrays  # noqa: E402
from paper_1903_06631_b200 import _native as N  # noqa: E402

arrays, window = workloads.interval_trace(a.nvars, seed=0)
for _ in range(2):
    plan_arrays(arrays)
N.sync()
os.environ["MP_PLACE_TRACE"] = a.out
plan_arrays(arrays)
N.sync()
del os.environ["MP_PLACE_TRACE"]
with open(a.out, "rb") as fh:
    V = int(np.frombuffer(fh.read(8), np.int64)[0])
    lvl = np.frombuffer(fh.read(4 * V), np.int32)
    m = np.frombuffer(fh.read(4 * V), np.int32)
    t = np.frombuffer(fh.read(8 * V), np.uint64).astype(np.int64)
    t0 = np.frombuffer(fh.read(8 * V), np.uint64).astype(np.int64)
    tr = np.frombuffer(fh.read(8 * V), np.uint64).astype(np.int64)
    tg = np.frombuffer(fh.read(8 * V), np.uint64).astype(np.int64)
    ts = np.frombuffer(fh.read(8 * V), np.uint64).astype(np.int64)
base = t0.min()
tr = np.where(tr == 0, 0.0, (tr - base) / 1e3)
t = (t - base) / 1e3  # us
t0 = (t0 - base) / 1e3
dur = t - t0
span = t.max()
print(f"V={V} levels={lvl.max()} span={span:.1f} us")
order = np.argsort(lvl, kind="stable")
ls = lvl[order]
bounds = np.searchsorted(ls, np.arange(1, lvl.max() + 2))
print(f"{'level':>5} {'count':>7} {'first_us':>9} {'last_us':>9} {'median':>9}")
rows = []
for L in range(1, lvl.max() + 1):
    sel = order[bounds[L - 1]:bounds[L]]
    tt = t[sel]
    rows.append((L, len(sel), tt.min(), tt.max(), np.median(tt)))
for r in rows:
    if r[0] <= 12 or r[0] % 8 == 0 or r[0] > lvl.max() - 6:
        print(f"{r[0]:5d} {r[1]:7d} {r[2]:9.1f} {r[3]:9.1f} {r[4]:9.1f}")
# throughput over time
hist, edges = np.histogram(t, bins=30)
print("placed per bucket (%.1f us):" % (edges[1] - edges[0]))
print(" ".join(str(int(h)) for h in hist))
# the chain of last finishers: the level-L variable placed last, per level
last = [r[3] for r in rows]
gaps = np.diff(last)
print(f"per-level advance of the last finisher: mean {gaps.mean():.2f} us, median {np.median(gaps):.2f} us")

print("predecessor-count histogram (all / placed after 0.66*span):")
late = t > 0.66 * span
for lo, hi in ((0, 0), (1, 32), (33, 64), (65, 128), (129, 256), (257, 1 << 30)):
    s = (m >= lo) & (m <= hi)
    if s.any():
        print(f"  m {lo:4d}-{hi:<10d} n={s.sum():7d} late={int((s & late).sum()):6d} "
              f"dur med {np.median(dur[s]):7.2f} us p99 {np.percentile(dur[s], 99):7.2f} max {dur[s].max():7.2f}")
print(f"max m {m.max()}")

wait = (t0 - base / 1e3 * 0) if False else None
qwait = ((t0 * 1e3 + 0) / 1e3) - tr
print(f"ready->claim wait: med {np.median(qwait):.2f} us p90 {np.percentile(qwait, 90):.2f} p99 {np.percentile(qwait, 99):.2f}")
for lo, hi in ((0, 0.25), (0.25, 0.5), (0.5, 0.66), (0.66, 0.8), (0.8, 1.01)):
    s = (t >= lo * span) & (t < hi * span)
    if s.any():
        print(f"  placed in [{lo:.2f},{hi:.2f})*span: n={s.sum():7d} wait med {np.median(qwait[s]):6.2f} "
              f"p90 {np.percentile(qwait[s], 90):6.2f}  dur med {np.median(dur[s]):6.2f} p90 {np.percentile(dur[s], 90):6.2f}"
              f"  m med {np.median(m[s]):.0f}")
# the critical chain: walk back from the last-placed variable through the
# predecessor that made it ready is not recorded; show the last 15 placed
idx = np.argsort(t)[-15:]
print("last placed: level m ready claim done")
for i in idx:
    print(f"  {lvl[i]:4d} {m[i]:4d} {tr[i]:8.1f} {t0[i]:8.1f} {t[i]:8.1f}")

ok = (tg > 0) & (ts > 0)
tg = (tg - base) / 1e3
ts = (ts - base) / 1e3
print("phases (claim->gathered, gathered->sorted, sorted->placed) by time window, m>32 only:")
for lo, hi in ((0, 0.25), (0.25, 0.5), (0.5, 0.66), (0.66, 0.8), (0.8, 1.01)):
    s = ok & (m > 32) & (t >= lo * span) & (t < hi * span)
    if s.any():
        a1, a2, a3 = tg[s] - t0[s], ts[s] - tg[s], t[s] - ts[s]
        print(f"  [{lo:.2f},{hi:.2f}) n={s.sum():6d} gather med {np.median(a1):6.2f} p90 {np.percentile(a1, 90):6.2f} | "
              f"sort med {np.median(a2):6.2f} p90 {np.percentile(a2, 90):6.2f} | hole med {np.median(a3):6.2f} "
              f"p90 {np.percentile(a3, 90):6.2f}")
