"""Summarize an ncu --metrics gpu__time_duration.sum launch list (CSV):
per-kernel totals over one config-4 pipeline pass — the launches between the
last two launches of a once-per-pass kernel (default k_period_quick; the
grouping sort of the next pass stands in for this pass's)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
idx = {k: i for i, k in enumerate(h)}
data = rows[hi + 1:]
names = [r[idx["Kernel Name"]] for r in data]
pre = sys.argv[2] if len(sys.argv) > 2 else "k_period_quick"
hits = [i for i, n in enumerate(names) if n.startswith(pre) or n.startswith("void " + pre)]
first, last = (hits[-2], hits[-1]) if len(hits) > 1 else (hits[-1], len(data))
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in data[first:last]:
    n = r[idx["Kernel Name"]].split("(")[0]
    v = float(r[idx["Metric Value"]].replace(",", ""))
    u = r[idx["Metric Unit"]]
    us = v / 1000 if u in ("nsecond", "ns") else (v if u in ("usecond", "us") else v * 1000)
    agg[n][0] += 1
    agg[n][1] += us
    tot += us
for n, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:58]:58s} {c:4d} {us:10.1f} us {100 * us / tot:5.1f}%")
print(f"total {tot:.1f} us in {last - first} launches")
