"""Generate the golden parity fixtures by running the REFERENCE package.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports ``memplan`` from /root/reference/pkg/src, builds every scenario
trace with this repo's own builders (tests/golden/scenarios.py), runs the
reference's pipeline on it — detect_iteration, extract_lifetimes,
build_conflict_graph, plan_pool (both policies), filter_candidates, the
four scores, the SWDOA greedy, select_by_score for every score at a sweep
of limits, build_schedule, simulate, compute_load_min, combine_with_pool —
and writes the results to tests/golden/*.json.gz.  Floats are stored as
``float.hex`` strings so parity is checked bit for bit; arrays longer than
``INLINE`` entries are stored as a SHA-256 of their canonical JSON.
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import platform
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import memplan as mp  # noqa: E402  (the reference)

import scenarios  # noqa: E402

INLINE = 400


def fhex(x):
    return float(x).hex()


def digest(obj) -> str:
    return hashlib.sha256(json.dumps(obj, separators=(",", ":")).encode()).hexdigest()


def pack(lst):
    if len(lst) <= INLINE:
        return lst
    return {"sha256": digest(lst), "n": len(lst)}


def ref_trace(t):
    return mp.Trace(events=[mp.TraceEvent(e.index, e.t_us, mp.EventKind(e.kind.value),
                                          e.var, e.size) for e in t.events])


def err(ex):
    if isinstance(ex, mp.InvariantViolation):
        return ["InvariantViolation", ex.index, ex.reason]
    if isinstance(ex, mp.LimitUnreachable):
        return ["LimitUnreachable", ex.limit_bytes, ex.achievable_bytes]
    if isinstance(ex, mp.SwapDeadlock):
        return ["SwapDeadlock", ex.index, ex.reason]
    if isinstance(ex, mp.PeriodNotFound):
        return ["PeriodNotFound", str(ex)]
    if isinstance(ex, IndexError):
        return ["IndexError"]
    if isinstance(ex, ValueError):
        return ["ValueError", str(ex)]
    raise ex


def canon_profile(prof):
    kinds = {"malloc": 0, "free": 1, "read": 2, "write": 3}
    var = []
    for v in prof.variables:
        var.append([v.var, v.base_var, v.size, v.alloc_index, v.free_index,
                    [list(s) for s in v.segments], v.persistent, v.wraps,
                    [[a.index, fhex(a.t_us), kinds[a.kind.value], a.next_iteration]
                     for a in v.accesses]])
    return {
        "period": prof.period, "window": list(prof.window),
        "vars": pack(var), "nvars": len(var),
        "loads": pack(list(prof.load.loads)), "peak": prof.load.peak_bytes,
        "peak_index": prof.load.peak_index,
        "op_times": pack([fhex(x) for x in prof.op_times_us]),
        "duration": fhex(prof.period_duration_us),
        "op_instance": pack(list(prof.op_instance)),
    }


def canon_graph(g):
    adj = [sorted(s) for s in g.adj]
    return {"nvars": len(g.vars), "edges": sum(len(s) for s in adj) // 2,
            "adj": pack(adj), "peak": g.peak_load_bytes}


def canon_plan(plan, g):
    return {"offsets": pack([plan.offsets[v.var] for v in g.vars]),
            "footprint": plan.footprint_bytes}


def canon_cand(c):
    return [c.var, c.size, c.out_index, fhex(c.out_time_us), fhex(c.out_ready_us),
            c.in_index, fhex(c.in_time_us), fhex(c.delta_out_us), fhex(c.delta_in_us),
            c.spans_iterations]


def canon_sched(s):
    return {"events": [[e.var, e.size, fhex(e.t_start_out), fhex(e.t_end_out),
                        fhex(e.t_start_in), fhex(e.t_end_in)] for e in s.events],
            "order": list(s.order), "duration": fhex(s.period_duration_us)}


def canon_curve(c):
    return {"points": pack([[fhex(t), v] for t, v in c.points]),
            "peak": c.peak_bytes, "peak_t": fhex(c.peak_time_us)}


def canon_sim(r):
    return {"limit": r.limit_bytes, "baseline": fhex(r.baseline_duration_us),
            "duration": fhex(r.duration_us), "overhead_us": fhex(r.overhead_us),
            "overhead_pct": fhex(r.overhead_pct), "peak": r.achieved_peak_bytes,
            "delayed": pack([[d.index, fhex(d.delay_us)] for d in r.delayed_ops]),
            "load_prime": canon_curve(r.load_prime),
            "load_double_prime": canon_curve(r.load_double_prime),
            "schedule": canon_sched(r.schedule), "rounds": r.rounds}


SCORES = ("swdoa", "doa", "aoa", "wdoa", "combined", "combined_w")
ALT_WEIGHTS = (0.3, -0.5, 0.2, 0.8)


def swap_block(prof, bw, lat, threshold, fracs):
    tm = mp.TransferModel(bandwidth_bytes_per_s=bw, latency_us=lat)
    cands = mp.filter_candidates(prof, threshold_bytes=threshold, transfer=tm)
    out = {"bw": fhex(bw), "lat": fhex(lat), "threshold": threshold,
           "candidates": [canon_cand(c) for c in cands]}
    out["load_min"] = mp.compute_load_min(prof, cands)
    if cands:
        mp.attach_scores(cands, prof)
        out["scores"] = [[fhex(c.scores[s]) for s in ("doa", "aoa", "wdoa", "swdoa")]
                         for c in cands]
        order, _, _ = mp.autoswap._swdoa_greedy(cands, prof, None)
        out["swdoa_order"] = [c.var for c in order]
        comb = mp.combined_scores(cands, prof, mp.ScoreWeights(*ALT_WEIGHTS))
        out["combined_w"] = [fhex(comb[c.var]) for c in cands]
    peak = prof.load.peak_bytes
    limits = sorted({max(1, int(peak * f)) for f in fracs} | {out["load_min"], max(1, out["load_min"] - 1)},
                    reverse=True)
    runs = []
    for limit in limits:
        for score in SCORES:
            run = {"limit": limit, "score": score}
            w = mp.ScoreWeights(*ALT_WEIGHTS) if score == "combined_w" else None
            sc = "combined" if score == "combined_w" else score
            fresh = mp.filter_candidates(prof, threshold_bytes=threshold, transfer=tm)
            try:
                sel = mp.select_by_score(fresh, prof, limit, score=sc, weights=w)
            except Exception as ex:  # noqa: BLE001
                run["selection"] = err(ex)
                runs.append(run)
                continue
            run["selection"] = [c.var for c in sel]
            sched = mp.build_schedule(sel, prof)
            run["schedule"] = canon_sched(sched)
            try:
                res = mp.simulate(sched, prof, limit)
            except Exception as ex:  # noqa: BLE001
                run["sim"] = err(ex)
                runs.append(run)
                continue
            run["sim"] = canon_sim(res)
            try:
                comb = mp.combine_with_pool(prof, res.schedule)
                cg = mp.build_conflict_graph(comb)
                run["combined"] = {"profile": canon_profile(comb),
                                   "footprint": mp.plan_pool(cg).footprint_bytes}
            except Exception as ex:  # noqa: BLE001
                run["combined"] = err(ex)
            runs.append(run)
    out["runs"] = runs
    return out


def trace_block(t):
    kinds = {"malloc": "m", "free": "f", "read": "r", "write": "w"}
    return {"kind": "".join(kinds[e.kind.value] for e in t.events),
            "var": [e.var for e in t.events], "size": [e.size for e in t.events],
            "t": [e.t_us for e in t.events], "index": [e.index for e in t.events]}


def run_trace_scenario(sc):
    t = sc["trace"]
    rt = ref_trace(t)
    out = {"name": sc["name"], "kind": "trace", "trace": trace_block(t)}
    try:
        mp.validate_trace(rt)
        out["validate"] = None
    except Exception as ex:  # noqa: BLE001
        out["validate"] = err(ex)
    if sc.get("validate_only"):
        return out
    window = sc.get("window")
    if window is None:
        try:
            det = mp.detect_iteration(rt)
            out["detect"] = [det.period, det.window[0], det.window[1]]
            window = det.window
        except Exception as ex:  # noqa: BLE001
            out["detect"] = err(ex)
            return out
    out["window"] = list(window)
    try:
        prof = mp.extract_lifetimes(rt, tuple(window))
    except Exception as ex:  # noqa: BLE001
        out["profile"] = err(ex)
        return out
    out["profile"] = canon_profile(prof)
    g = mp.build_conflict_graph(prof)
    out["graph"] = canon_graph(g)
    out["plans"] = {pol: canon_plan(mp.plan_pool(g, pol), g) for pol in ("best_fit", "first_fit")}
    out["swap"] = [swap_block(prof, bw, lat, thr, sc.get("fracs", (0.9, 0.75, 0.6)))
                   for bw, lat, thr in sc.get("transfers", ())]
    return out


def run_arcs_scenario(sc):
    arcs = sc["arcs"]
    g = mp.conflict_graph_from_arcs(sc["period"], [(a[0], a[1], a[2], tuple(tuple(s) for s in a[3]), a[4])
                                                   for a in arcs], sc["peak"])
    return {"name": sc["name"], "kind": "arcs", "arcs": arcs, "period": sc["period"],
            "peak": sc["peak"], "graph": canon_graph(g),
            "plans": {pol: canon_plan(mp.plan_pool(g, pol), g) for pol in ("best_fit", "first_fit")}}


def run_synthetic_scenario(sc):
    loads, spacing = sc["loads"], sc["spacing"]
    times = [spacing * r for r in range(len(loads))]
    peak = max(loads)
    prof = mp.IterationProfile(period=len(loads), window=(0, len(loads)), variables=[],
                               load=mp.LoadProfile(loads=list(loads), peak_bytes=peak,
                                                   peak_index=loads.index(peak)),
                               op_times_us=times, period_duration_us=spacing * len(loads),
                               events=[])

    def mk():
        return [mp.SwapCandidate(var=c[0], size=c[1], out_index=c[2], out_time_us=c[3],
                                 out_ready_us=c[4], in_index=c[5], in_time_us=c[6],
                                 delta_out_us=c[7], delta_in_us=c[8], spans_iterations=c[9])
                for c in sc["cands"]]
    cands = mk()
    out = {"name": sc["name"], "kind": "synthetic", "loads": loads, "spacing": fhex(spacing),
           "cands": [[c[0], c[1], c[2], fhex(c[3]), fhex(c[4]), c[5], fhex(c[6]), fhex(c[7]),
                      fhex(c[8]), c[9]] for c in sc["cands"]]}
    out["wdoa"] = [fhex(mp.score_wdoa(c, prof)) for c in cands]
    out["doa"] = [fhex(mp.score_doa(c)) for c in cands]
    out["aoa"] = [fhex(mp.score_aoa(c)) for c in cands]
    sw = mp.swdoa_scores(cands, prof)
    out["swdoa"] = [fhex(sw[c.var]) for c in cands]
    out["load_min"] = mp.compute_load_min(prof, cands)
    runs = []
    for limit in sc["limits"]:
        for score in ("swdoa", "doa", "aoa", "wdoa", "combined"):
            try:
                sel = mp.select_by_score(mk(), prof, limit, score=score)
                runs.append({"limit": limit, "score": score, "selection": [c.var for c in sel]})
            except Exception as ex:  # noqa: BLE001
                runs.append({"limit": limit, "score": score, "selection": err(ex)})
    out["runs"] = runs
    return out


def main():
    os.makedirs(HERE, exist_ok=True)
    meta = {"python": sys.version, "platform": platform.platform(),
            "reference": "/root/reference/pkg/src/memplan", "generated": time.time()}
    groups = scenarios.all_groups()
    for gname, items in groups.items():
        t0 = time.time()
        out = []
        for sc in items:
            kind = sc.get("kind", "trace")
            if kind == "trace":
                out.append(run_trace_scenario(sc))
            elif kind == "arcs":
                out.append(run_arcs_scenario(sc))
            else:
                out.append(run_synthetic_scenario(sc))
        path = os.path.join(HERE, f"{gname}.json.gz")
        with gzip.open(path, "wt") as fh:
            json.dump({"meta": meta, "scenarios": out}, fh, separators=(",", ":"))
        print(f"{gname}: {len(out)} scenarios, {os.path.getsize(path)} B, {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
