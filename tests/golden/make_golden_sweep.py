"""Golden fixtures for the batched sweep unit, produced by the REFERENCE.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden_sweep.py

A sweep unit is what the reference's estimators do for one trace
(pkg/src/memplan/estimators.py:20-130): validate_trace, detect_iteration,
extract_lifetimes, build_conflict_graph + plan_pool, filter_candidates,
compute_load_min, the SWDOA greedy order, and per budget fraction
SwapPlanner(limit_bytes=int(peak * frac), score="swdoa", ...).fit.  This
script runs exactly those reference calls on a set of traces and parameter
sets and writes tests/golden/sweep.json.gz (floats as float.hex), which pins
the CPU oracle's orc_sweep_unit and, through it, the device sweep.
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
from paper_1903_06631_b200.trace import EventKind, Trace, TraceEvent  # noqa: E402

MIB = 1 << 20

PARAMS = [
    dict(name="default", policy="best_fit", threshold=MIB, bw=12e9, lat=10.0, max_rounds=100,
         budgets=[0.95, 0.9, 0.7, 0.5]),
    dict(name="slow_link", policy="first_fit", threshold=1000, bw=1e9, lat=1.0, max_rounds=100,
         budgets=[1.0, 0.99, 0.9, 0.8, 0.7, 0.6, 0.5, 0.0]),
]


def traces():
    out = []
    for i, spec in enumerate(workloads.sweep_specs(n_models=14, n_scales=2)):
        out.append((f"sweep_{i}_{spec.name}", synth.generate_synthetic_trace(spec)))
    for seed in range(12):
        rng = random.Random(5000 + seed)
        kw = dict(slots=rng.choice((12, 24, 40)), nvars=rng.randrange(2, 12),
                  iterations=rng.randrange(4, 6), max_wrap=rng.choice((0.9, 1.5, 2.2)),
                  n_persistent=rng.randrange(0, 3), n_leak=rng.randrange(0, 2),
                  n_reuse=rng.randrange(0, 3), zero_dt=rng.choice((0.0, 0.3)))
        out.append((f"periodic_{seed}", workloads.random_periodic_trace(seed, **kw)))
    # error paths: an invariant violation, a trace without a period, a tiny trace
    good = synth.generate_synthetic_trace(synth.vgg_like(depth=4, scale=0.25, iterations=3, seed=9))
    ev = list(good.events)
    bad = [TraceEvent(e.index, e.t_us, e.kind, e.var, e.size) for e in ev]
    j = next(k for k, e in enumerate(bad) if e.kind == EventKind.FREE and k > len(bad) // 2)
    bad[j] = TraceEvent(bad[j].index, bad[j].t_us, EventKind.FREE, "nosuchvar", 0)
    out.append(("invalid_free", Trace(events=bad)))
    aper = [TraceEvent(i, 10 * i, EventKind.MALLOC if i % 2 == 0 else EventKind.FREE, f"a{i // 2}",
                       (i // 2 + 1) * 100 if i % 2 == 0 else 0) for i in range(40)]
    out.append(("aperiodic", Trace(events=aper)))
    out.append(("single_var", Trace(events=[TraceEvent(0, 0, EventKind.MALLOC, "x", 64),
                                            TraceEvent(1, 5, EventKind.FREE, "x", 0),
                                            TraceEvent(2, 9, EventKind.MALLOC, "x", 64),
                                            TraceEvent(3, 14, EventKind.FREE, "x", 0)])))
    return out


def unit(rt, prm):
    out = {}
    try:
        mp.validate_trace(rt)
        det = mp.detect_iteration(rt)
    except Exception as ex:  # noqa: BLE001
        out["error"] = err(ex)
        return out
    prof = mp.extract_lifetimes(rt, det.window)
    names = [v.var for v in prof.variables]
    pos = {nm: i for i, nm in enumerate(names)}
    g = mp.build_conflict_graph(prof)
    plan = mp.plan_pool(g, prm["policy"])
    tm = mp.TransferModel(bandwidth_bytes_per_s=prm["bw"], latency_us=prm["lat"])
    cands = mp.filter_candidates(prof, threshold_bytes=prm["threshold"], transfer=tm)
    order, _, _ = mp.autoswap._swdoa_greedy(cands, prof, None)
    out.update({
        "period": prof.period, "nvars": len(names),
        "ncarry": sum(v.alloc_index is None for v in prof.variables),
        "naccess": sum(len(v.accesses) for v in prof.variables),
        "peak": prof.load.peak_bytes, "peak_index": prof.load.peak_index,
        "duration": fhex(prof.period_duration_us), "footprint": plan.footprint_bytes,
        "edges": sum(len(s) for s in g.adj) // 2, "ncand": len(cands),
        "load_min": mp.compute_load_min(prof, cands),
        "offsets": [plan.offsets[nm] for nm in names],
        "order": [pos[c.var] for c in order],
    })
    budgets = []
    for frac in prm["budgets"]:
        limit = int(prof.load.peak_bytes * frac)
        rec = {"limit": limit}
        sp = mp.SwapPlanner(limit_bytes=limit, score="swdoa", threshold_bytes=prm["threshold"],
                            bandwidth_bytes_per_s=prm["bw"], latency_us=prm["lat"])
        try:
            sp.fit(prof)
        except Exception as ex:  # noqa: BLE001
            rec["error"] = err(ex)
            budgets.append(rec)
            continue
        res = sp.result_
        rec.update({"selection": [pos[c.var] for c in sp.selection_],
                    "selected_bytes": sum(c.size for c in sp.selection_),
                    "rounds": res.rounds, "overhead_us": fhex(res.overhead_us),
                    "achieved": res.achieved_peak_bytes, "planned": res.load_prime.peak_bytes})
        budgets.append(rec)
    out["budgets"] = budgets
    return out


def main():
    t0 = time.time()
    scen = []
    trs = traces()
    for prm in PARAMS:
        for name, t in trs:
            rt = ref_trace(t)
            scen.append({"name": f"{prm['name']}:{name}", "params": prm, "trace": trace_block(t),
                         "unit": unit(rt, prm)})
    meta = {"python": sys.version, "platform": platform.platform(), "seconds": time.time() - t0,
            "generator": "tests/golden/make_golden_sweep.py"}
    with gzip.open(os.path.join(HERE, "sweep.json.gz"), "wt") as fh:
        json.dump({"meta": meta, "scenarios": scen}, fh, separators=(",", ":"))
    print(f"{len(scen)} sweep units in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
