"""Golden parity through the public drop-in API (Python objects end to end).

Same fixtures as test_gpu_pool_parity / test_gpu_swap_parity, but every
value is read from the reference-shaped objects the package returns
(IterationProfile, ConflictGraph, PoolPlan, SwapCandidate, SwapSchedule,
SimulationResult) and combine_with_pool is checked too.
"""
import pytest

from golden_util import ALT_WEIGHTS, fhex, load, pack

pytestmark = pytest.mark.gpu

GROUPS = ("hand", "generator", "configs", "periodic", "interval")
KIND = {"malloc": 0, "free": 1, "read": 2, "write": 3}


def _params():
    for g in GROUPS:
        for sc in load(g):
            if "profile" in sc and isinstance(sc["profile"], dict):
                yield pytest.param(g, sc["name"], id=f"{g}:{sc['name']}")


def _get(g, name):
    return next(s for s in load(g) if s["name"] == name)


def to_trace(mp, sc):
    tr = sc["trace"]
    kinds = {"m": "malloc", "f": "free", "r": "read", "w": "write"}
    return mp.Trace(events=[mp.TraceEvent(i, t, mp.EventKind(kinds[k]), v, s) for i, k, v, s, t in
                            zip(tr["index"], tr["kind"], tr["var"], tr["size"], tr["t"])])


def canon_profile(prof):
    var = [[v.var, v.base_var, v.size, v.alloc_index, v.free_index, [list(s) for s in v.segments], v.persistent,
            v.wraps, [[a.index, fhex(a.t_us), KIND[a.kind.value], a.next_iteration] for a in v.accesses]]
           for v in prof.variables]
    return {"period": prof.period, "window": list(prof.window), "vars": pack(var), "nvars": len(var),
            "loads": pack(list(prof.load.loads)), "peak": prof.load.peak_bytes, "peak_index": prof.load.peak_index,
            "op_times": pack([fhex(x) for x in prof.op_times_us]), "duration": fhex(prof.period_duration_us),
            "op_instance": pack(list(prof.op_instance))}


def canon_sched(s):
    return {"events": [[e.var, e.size, fhex(e.t_start_out), fhex(e.t_end_out), fhex(e.t_start_in),
                        fhex(e.t_end_in)] for e in s.events], "order": list(s.order),
            "duration": fhex(s.period_duration_us)}


def canon_curve(c):
    return {"points": pack([[fhex(t), v] for t, v in c.points]), "peak": c.peak_bytes,
            "peak_t": fhex(c.peak_time_us)}


@pytest.mark.parametrize("group,name", list(_params()))
def test_api_matches_reference(group, name):
    import paper_1903_06631_b200 as mp
    sc = _get(group, name)
    trace = to_trace(mp, sc)
    prof = mp.extract_lifetimes(trace, tuple(sc["window"]))
    assert canon_profile(prof) == sc["profile"]
    g = mp.build_conflict_graph(prof)
    adj = [sorted(s) for s in g.adj]
    assert {"edges": sum(len(a) for a in adj) // 2, "adj": pack(adj)} == \
        {k: sc["graph"][k] for k in ("edges", "adj")}
    for pol in ("best_fit", "first_fit"):
        plan = mp.plan_pool(g, pol)
        assert pack([plan.offsets[v.var] for v in g.vars]) == sc["plans"][pol]["offsets"]
        assert plan.footprint_bytes == sc["plans"][pol]["footprint"]
    for blk in sc.get("swap", []):
        tm = mp.TransferModel(float.fromhex(blk["bw"]), float.fromhex(blk["lat"]))
        cands = mp.filter_candidates(prof, threshold_bytes=blk["threshold"], transfer=tm)
        assert [[c.var, c.size, c.out_index, fhex(c.out_time_us), fhex(c.out_ready_us), c.in_index,
                 fhex(c.in_time_us), fhex(c.delta_out_us), fhex(c.delta_in_us), c.spans_iterations]
                for c in cands] == blk["candidates"]
        assert mp.compute_load_min(prof, cands) == blk["load_min"]
        for run in blk["runs"]:
            score = "combined" if run["score"] == "combined_w" else run["score"]
            w = mp.ScoreWeights(*ALT_WEIGHTS) if run["score"] == "combined_w" else None
            fresh = mp.filter_candidates(prof, threshold_bytes=blk["threshold"], transfer=tm)
            try:
                sel = mp.select_by_score(fresh, prof, run["limit"], score=score, weights=w)
            except mp.LimitUnreachable as ex:
                assert run["selection"] == ["LimitUnreachable", ex.limit_bytes, ex.achievable_bytes]
                continue
            assert [c.var for c in sel] == run["selection"]
            sched = mp.build_schedule(sel, prof)
            assert canon_sched(sched) == run["schedule"]
            try:
                res = mp.simulate(sched, prof, run["limit"])
            except mp.SwapDeadlock as ex:
                assert run["sim"] == ["SwapDeadlock", ex.index, ex.reason]
                continue
            except IndexError:
                assert run["sim"] == ["IndexError"]
                continue
            sim = run["sim"]
            got = {"limit": res.limit_bytes, "baseline": fhex(res.baseline_duration_us),
                   "duration": fhex(res.duration_us), "overhead_us": fhex(res.overhead_us),
                   "overhead_pct": fhex(res.overhead_pct), "peak": res.achieved_peak_bytes,
                   "delayed": pack([[d.index, fhex(d.delay_us)] for d in res.delayed_ops]),
                   "load_prime": canon_curve(res.load_prime),
                   "load_double_prime": canon_curve(res.load_double_prime),
                   "schedule": canon_sched(res.schedule), "rounds": res.rounds}
            assert got == sim
            want = run.get("combined")
            if want is None:
                continue
            try:
                comb = mp.combine_with_pool(prof, res.schedule)
            except mp.InvariantViolation as ex:
                assert want == ["InvariantViolation", ex.index, ex.reason]
                continue
            assert isinstance(want, dict), want
            cp = canon_profile(comb)
            assert cp == want["profile"]
            assert mp.plan_pool(mp.build_conflict_graph(comb)).footprint_bytes == want["footprint"]
