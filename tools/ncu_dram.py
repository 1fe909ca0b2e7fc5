"""Per-kernel duration and DRAM bytes from an ncu --csv launch list taken
with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum.

  python tools/ncu_dram.py <csv> [first-kernel-prefix] [--json out.json] [--peak GBps]

With a prefix naming a kernel launched once per pass, keeps the last pass
(as many launches as separate the prefix kernel's last two launches), groups by kernel name, and prints per kernel: launches,
total us, DRAM read/write MB, DRAM GB/s (measured bytes / duration) and the
fraction of the HBM peak.  ncu serialises launches and runs them cold-cache,
so the absolute times are upper bounds; shares and bytes are what count."""
import collections
import csv
import json
import sys

args = [a for a in sys.argv[1:]]
out_json = None
peak = 6547.2
if "--json" in args:
    i = args.index("--json"); out_json = args[i + 1]; del args[i:i + 2]
if "--peak" in args:
    i = args.index("--peak"); peak = float(args[i + 1]); del args[i:i + 2]
rows = list(csv.reader(open(args[0])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    lid = r[ix["ID"]]
    d = launch.setdefault(lid, {"name": r[ix["Kernel Name"]].split("(")[0]})
    v = float(r[ix["Metric Value"]].replace(",", ""))
    u = r[ix["Metric Unit"]]
    m = r[ix["Metric Name"]]
    if m == "gpu__time_duration.sum":
        d["us"] = v / 1000 if u in ("nsecond", "ns") else (v if u in ("usecond", "us") else v * 1000)
    else:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
        d["rd" if "read" in m else "wr"] = v * scale
L = list(launch.values())
pre = args[1] if len(args) > 1 else None
if pre:
    # the prefix names a kernel launched once per pass: the last pass is the
    # last (distance between its last two launches) launches of the list
    hits = [i for i, d in enumerate(L) if d["name"].startswith(pre) or d["name"].startswith("void " + pre)]
    per = hits[-1] - hits[-2] if len(hits) > 1 else len(L) - hits[-1]
    L = L[len(L) - per:] if len(hits) > 1 else L[hits[-1]:]
agg = collections.OrderedDict()
for d in L:
    a = agg.setdefault(d["name"], {"launches": 0, "us": 0.0, "rd": 0.0, "wr": 0.0})
    a["launches"] += 1
    a["us"] += d.get("us", 0.0)
    a["rd"] += d.get("rd", 0.0)
    a["wr"] += d.get("wr", 0.0)
tot = sum(a["us"] for a in agg.values())
print(f"{'kernel':52s} {'n':>3s} {'us':>9s} {'share':>6s} {'rd MB':>8s} {'wr MB':>8s} {'GB/s':>7s} {'frac':>6s}")
for n, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
    gbs = (a["rd"] + a["wr"]) / (a["us"] * 1e-6) / 1e9 if a["us"] else 0.0
    a["dram_gbs"] = gbs
    print(f"{n[:52]:52s} {a['launches']:3d} {a['us']:9.1f} {100 * a['us'] / tot:5.1f}% {a['rd'] / 1e6:8.1f} "
          f"{a['wr'] / 1e6:8.1f} {gbs:7.0f} {gbs / peak:6.3f}")
print(f"total {tot:.1f} us in {len(L)} launches")
if out_json:
    kern = {}
    for n, a in agg.items():
        short = (n[5:] if n.startswith("void ") else n).split("<")[0]
        k = kern.setdefault(short, {"launches": 0, "us": 0.0, "dram_read_bytes": 0.0, "dram_write_bytes": 0.0})
        k["launches"] += a["launches"]; k["us"] += a["us"]; k["dram_read_bytes"] += a["rd"]; k["dram_write_bytes"] += a["wr"]
    for k in kern.values():
        n = k["launches"]
        k["us_per_launch"] = k["us"] / n
        k["dram_read_bytes"] /= n
        k["dram_write_bytes"] /= n
        k["note"] = "per launch (averaged over launches of the kernel in the pass)"
    json.dump({"source": args[0], "peak_gbs": peak, "total_us": tot, "kernels": kern}, open(out_json, "w"), indent=1)
