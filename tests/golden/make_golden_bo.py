"""Golden fixtures for SwapPlanner(score="bo"), produced by the REFERENCE.

Run in the build container only:  python tests/golden/make_golden_bo.py

For each scenario the reference's SwapPlanner(limit, score="bo", bo_budget,
seed).fit(profile) runs (estimators.py:85-130: the BO loop of
autoswap.optimize_weights over bo.minimize, each evaluation a combined-score
select_by_score + build_schedule + simulate); the tuned weights, the final
selection and the simulated result are stored (floats as float.hex).
"""
from __future__ import annotations

import gzip
import json
import os
import platform
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import memplan as mp  # noqa: E402  (the reference)

from make_golden import err, fhex, ref_trace, trace_block  # noqa: E402
from paper_1903_06631_b200 import synth, workloads  # noqa: E402


def scenarios():
    out = []
    # (depth, scale, seed) x runs (frac, bw, lat, threshold, budget, seed): the
    # first five make BO explore (non-zero overhead, a non-corner optimum)
    shapes = {(7, 0.4, 2): [(0.88, 1e9, 5.0, 1 << 20, 10, 0), (0.9, 12e9, 10.0, 1 << 20, 8, 0)],
              (9, 0.3, 3): [(0.88, 1e9, 5.0, 1 << 20, 10, 0), (0.8, 1e9, 5.0, 1 << 20, 10, 0),
                            (0.75, 2e9, 5.0, 1 << 20, 10, 1)],
              (6, 1.0, 4): [(0.93, 1e9, 5.0, 1 << 20, 10, 0), (0.88, 1e9, 5.0, 1 << 20, 10, 0),
                            (0.88, 1e9, 5.0, 1 << 20, 14, 3)],
              (5, 0.5, 1): [(0.75, 2e9, 5.0, 1 << 20, 10, 1)]}
    for (d, sc, seed), runs in shapes.items():
        t = synth.generate_synthetic_trace(synth.vgg_like(depth=d, scale=sc, iterations=3, seed=seed, temp_ratio=0.5))
        out.append((f"vgg_like_d{d}_s{sc}", t, runs))
    for seed in range(3):
        rng = random.Random(9000 + seed)
        t = workloads.random_periodic_trace(seed + 50, slots=rng.choice((24, 40)), nvars=rng.randrange(4, 12),
                                            iterations=5, n_persistent=1)
        out.append((f"periodic_{seed}", t, [(0.8, 1e9, 1.0, 1000, 8, seed)]))
    return out


def main():
    t0 = time.time()
    scen = []
    for name, t, runs in scenarios():
        rt = ref_trace(t)
        det = mp.detect_iteration(rt)
        prof = mp.extract_lifetimes(rt, det.window)
        res = []
        for frac, bw, lat, thr, budget, seed in runs:
            limit = int(prof.load.peak_bytes * frac)
            sp = mp.SwapPlanner(limit_bytes=limit, score="bo", threshold_bytes=thr, bandwidth_bytes_per_s=bw,
                                latency_us=lat, bo_budget=budget, seed=seed)
            rec = {"limit": limit, "bw": fhex(bw), "lat": fhex(lat), "threshold": thr, "budget": budget,
                   "seed": seed}
            try:
                sp.fit(prof)
            except Exception as ex:  # noqa: BLE001
                rec["error"] = err(ex)
                res.append(rec)
                continue
            rec.update({"weights": [fhex(x) for x in sp.weights_.as_tuple()],
                        "selection": [c.var for c in sp.selection_],
                        "overhead_us": fhex(sp.overhead_us_), "achieved": sp.achieved_peak_bytes_})
            res.append(rec)
        scen.append({"name": name, "trace": trace_block(t), "runs": res})
    meta = {"python": sys.version, "platform": platform.platform(), "seconds": time.time() - t0}
    with gzip.open(os.path.join(HERE, "bo.json.gz"), "wt") as fh:
        json.dump({"meta": meta, "scenarios": scen}, fh, separators=(",", ":"))
    print(f"{sum(len(s['runs']) for s in scen)} BO runs in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
