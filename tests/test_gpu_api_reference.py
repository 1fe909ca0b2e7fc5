"""The reference's own test cases, re-expressed against the drop-in package.

Each test restates a case from pkg/tests/test_*.py (cited per test) and
runs it through ``paper_1903_06631_b200`` — i.e. through the device
library.  Goldens are the reference's (pytest.approx where the reference
uses it; exact elsewhere).
"""
import itertools
import json
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MIB = 1 << 20
MB = 10 ** 6


@pytest.fixture(scope="module")
def mp():
    import paper_1903_06631_b200 as m
    return m


def make_trace(mp, ops, spacing_us=10):
    return mp.Trace(events=[mp.TraceEvent(i, spacing_us * i, mp.EventKind(k), v, s)
                            for i, (k, v, s) in enumerate(ops)])


def profile_of(mp, ops):
    t = make_trace(mp, ops)
    return mp.extract_lifetimes(t, mp.detect_iteration(t).window)


def congested(iterations=2):
    one = [("malloc", "w1", 25 * MIB), ("write", "w1", 0), ("malloc", "w2", 25 * MIB), ("write", "w2", 0),
           ("malloc", "w3", 25 * MIB), ("write", "w3", 0), ("malloc", "a", 45 * MIB), ("write", "a", 0),
           ("free", "a", 0), ("malloc", "b", 20 * MIB), ("write", "b", 0), ("free", "b", 0), ("read", "w3", 0),
           ("free", "w3", 0), ("read", "w2", 0), ("free", "w2", 0), ("read", "w1", 0), ("write", "w1", 0),
           ("free", "w1", 0)]
    return one * iterations


def three_var(iterations=2):
    one = [("malloc", "v1", 45 * MB), ("write", "v1", 0), ("malloc", "v2", 40 * MB), ("write", "v2", 0),
           ("malloc", "v3", 34 * MB), ("write", "v3", 0), ("malloc", "t", 1 * MB), ("free", "t", 0),
           ("read", "v1", 0), ("free", "v1", 0), ("read", "v2", 0), ("free", "v2", 0), ("read", "v3", 0),
           ("write", "v3", 0), ("free", "v3", 0)]
    return one * iterations


def filter_instance():
    ops = []
    for k in (1, 2):
        ops += [("malloc", f"F{k}", 2 * MIB), ("write", f"F{k}", 0), ("read", f"F{k}", 0), ("free", f"F{k}", 0),
                ("malloc", f"B{k}", 2 * MIB), ("write", f"B{k}", 0), ("malloc", f"s{k}", 500_000),
                ("write", f"s{k}", 0), ("malloc", f"T{k}", 3 * MIB), ("free", f"T{k}", 0), ("read", f"s{k}", 0),
                ("free", f"s{k}", 0), ("write", f"B{k}", 0), ("free", f"B{k}", 0)]
    return ops


def synthetic_profile(mp, loads, spacing=10.0):
    times = [spacing * r for r in range(len(loads))]
    peak = max(loads)
    return mp.IterationProfile(period=len(loads), window=(0, len(loads)), variables=[],
                               load=mp.LoadProfile(loads=list(loads), peak_bytes=peak,
                                                   peak_index=loads.index(peak)),
                               op_times_us=times, period_duration_us=spacing * len(loads), events=[])


def hand_candidate(mp, gap_us, d_out, d_in, size=MIB, out_index=0, in_index=1, out_time=0.0, spans=False,
                   var="x"):
    return mp.SwapCandidate(var=var, size=size, out_index=out_index, out_time_us=out_time,
                            out_ready_us=out_time, in_index=in_index, in_time_us=out_time + gap_us,
                            delta_out_us=d_out, delta_in_us=d_in, spans_iterations=spans)


# --------------------------------------------------------------- iteration
# pkg/tests/test_iteration.py

def test_exact_doubling_gives_full_period(mp):
    ops = [(k, f"a{c}.{i}", (i + 1) if k == "malloc" else 0) for c in range(2) for i in range(6)
           for k in ("malloc", "free")]
    det = mp.detect_iteration(make_trace(mp, ops))
    assert (det.period, det.window) == (12, (12, 24))


def test_aperiodic_and_short_traces_raise(mp):
    ops = [(k, f"a{i}", (i + 1) if k == "malloc" else 0) for i in range(25) for k in ("malloc", "free")]
    with pytest.raises(mp.PeriodNotFound):
        mp.detect_iteration(make_trace(mp, ops))
    with pytest.raises(mp.PeriodNotFound):
        mp.detect_iteration(make_trace(mp, [("malloc", "a", 5), ("write", "a", 0), ("read", "a", 0)]))


def test_generator_period_matches_metadata(mp):
    for seed in (0, 1, 2):
        spec = mp.vgg_like(depth=5, scale=0.5, iterations=5, seed=seed)
        t = mp.generate_synthetic_trace(spec)
        det = mp.detect_iteration(t)
        p, n = t.meta["period"], len(t)
        assert det.period == p and det.window == (n - p, n)


def test_detection_ignores_variable_names(mp):
    t = mp.generate_synthetic_trace(mp.vgg_like(depth=4, scale=0.5, iterations=4, seed=11))
    names = {}
    renamed = [mp.TraceEvent(e.index, e.t_us, e.kind, names.setdefault(e.var, f"v{len(names)}"), e.size) for e in t]
    a, b = mp.detect_iteration(t), mp.detect_iteration(mp.Trace(renamed))
    assert (a.period, a.window) == (b.period, b.window)


def test_plain_window_lifetime(mp):
    ops = [("malloc", "w", 5), ("write", "w", 0)]
    for k in (1, 2):
        ops += [("read", "w", 0), ("read", "w", 0), ("malloc", f"x{k}", 10), ("write", f"x{k}", 0),
                ("read", f"x{k}", 0), ("read", "w", 0), ("read", "w", 0), ("free", f"x{k}", 0)]
    prof = profile_of(mp, ops)
    assert prof.period == 8
    x = prof.lifetime("x2")
    assert (x.alloc_index, x.free_index, x.segments) == (2, 7, ((2, 7),))
    assert not x.persistent and not x.wraps
    w = prof.lifetime("w")
    assert w.persistent and w.segments == ((0, 8),)
    g = mp.build_conflict_graph(prof)
    idx = {pv.var: i for i, pv in enumerate(g.vars)}
    assert idx["x2"] in g.adj[idx["w"]]


def test_nest_and_coexist_twins(mp):
    ops = [("malloc", "b0", 8), ("write", "b0", 0)]
    for k in (1, 2, 3):
        ops += [("read", f"b{k-1}", 0), ("free", f"b{k-1}", 0), ("malloc", f"b{k}", 8), ("write", f"b{k}", 0),
                ("malloc", f"s{k}", 1), ("free", f"s{k}", 0)]
    prof = profile_of(mp, ops)
    b = prof.lifetime("b3")
    assert b.wraps and b.segments == ((2, 6), (0, 1))
    assert [(a.index, a.kind, a.next_iteration) for a in b.accesses] == \
        [(3, mp.EventKind.WRITE, False), (0, mp.EventKind.READ, True)]
    assert prof.load.loads == [8, 0, 8, 8, 9, 8]
    ops = [("malloc", "a0", 8), ("write", "a0", 0)]
    for k in (1, 2, 3):
        ops += [("malloc", f"a{k}", 8), ("write", f"a{k}", 0), ("free", f"a{k-1}", 0)]
    prof = profile_of(mp, ops)
    old, new = prof.lifetime("a2"), prof.lifetime("a3")
    assert old.segments == ((0, 2),) and not old.wraps
    assert new.segments == ((0, 3),) and new.wraps
    assert prof.load.loads == [16, 16, 8]
    plan = mp.plan_pool(mp.build_conflict_graph(prof), policy="first_fit")
    assert {plan.offsets["a2"], plan.offsets["a3"]} == {0, 8} and plan.footprint_bytes == 16


def test_load_matches_liveness_and_recompute(mp):
    for seed, depth, ratio in ((0, 4, 0.5), (7, 6, 0.0), (3, 3, 0.9)):
        spec = mp.vgg_like(depth=depth, scale=0.3, iterations=4, seed=seed)
        spec.temp_ratio = ratio
        t = mp.generate_synthetic_trace(spec)
        det = mp.detect_iteration(t)
        prof = mp.extract_lifetimes(t, det.window)
        live, loads = {}, []
        for e in t.events[:det.window[0]]:
            if e.kind == mp.EventKind.MALLOC:
                live[e.var] = e.size
            elif e.kind == mp.EventKind.FREE:
                live.pop(e.var, None)
        for e in t.events[det.window[0]:det.window[1]]:
            if e.kind == mp.EventKind.MALLOC:
                live[e.var] = e.size
            elif e.kind == mp.EventKind.FREE:
                live.pop(e.var, None)
            loads.append(sum(live.values()))
        assert prof.load.loads == loads
        again = mp.compute_load_profile(prof)
        assert (again.loads, again.peak_bytes, again.peak_index) == \
            (prof.load.loads, prof.load.peak_bytes, prof.load.peak_index)


def test_persistent_and_unfreed(mp):
    t = mp.generate_synthetic_trace(mp.vgg_like(depth=4, scale=0.5, iterations=3, seed=8))
    prof = mp.extract_lifetimes(t, mp.detect_iteration(t).window)
    g = mp.build_conflict_graph(prof)
    for i, v in enumerate(prof.variables):
        if v.persistent:
            assert g.adj[i] == set(range(len(prof.variables))) - {i}
    ops = []
    for k in (1, 2):
        ops += [("malloc", f"keep{k}", 4), ("write", f"keep{k}", 0), ("malloc", f"tmp{k}", 9),
                ("read", f"tmp{k}", 0), ("free", f"tmp{k}", 0)]
    prof = profile_of(mp, ops)
    keep = prof.lifetime("keep2")
    assert keep.persistent and keep.segments == ((0, prof.period),)


# --------------------------------------------------------------- smartpool
# pkg/tests/test_smartpool.py

def arc(var, size, lo, hi):
    return (var, size, lo, ((lo, hi),), False)


def random_arcs(rng, n, period=100, max_size=64 * MIB):
    arcs, events = [], []
    for i in range(n):
        lo = rng.randrange(0, period - 1)
        hi = rng.randrange(lo + 1, period + 1)
        size = rng.randrange(1024, max_size)
        arcs.append((f"v{i:03d}", size, lo, ((lo, hi),), False))
        events += [(lo, 1, size), (hi, 0, size)]
    events.sort()
    cur = peak = 0
    for _pt, ph, s in events:
        cur = cur + s if ph else cur - s
        peak = max(peak, cur)
    return arcs, peak


def test_touching_vs_overlapping_and_chain(mp):
    g = mp.conflict_graph_from_arcs(100, [arc("a", 10, 0, 5), arc("b", 10, 5, 9)], 0)
    assert g.adj == [set(), set()]
    for policy in ("first_fit", "best_fit"):
        plan = mp.plan_pool(g, policy)
        assert plan.offsets == {"a": 0, "b": 0} and plan.footprint_bytes == 10
    g = mp.conflict_graph_from_arcs(100, [arc("a", 10, 0, 5), arc("b", 10, 3, 9)], 0)
    assert g.adj == [{1}, {0}]
    g = mp.conflict_graph_from_arcs(100, [arc("A", 30, 0, 5), arc("B", 20, 4, 8), arc("C", 25, 6, 9)], 50)
    for policy in ("first_fit", "best_fit"):
        plan = mp.plan_pool(g, policy)
        assert plan.offsets == {"A": 0, "C": 0, "B": 30}
        assert plan.footprint_bytes == 50 and plan.competitive_ratio == 1.0
        mp.check_plan(plan, g)
    assert mp.brute_force_optimal_footprint(g) == 50


def test_clique_weight_equals_peak(mp):
    rng = random.Random(7)
    for _ in range(100):
        n = rng.randint(2, 12)
        arcs, peak = random_arcs(rng, n)
        g = mp.conflict_graph_from_arcs(100, arcs, peak)
        segs = [a[3][0] for a in arcs]
        loads = [sum(a[1] for a, (lo, hi) in zip(arcs, segs) if lo <= r < hi) for r in range(101)]
        pt = max(range(101), key=lambda r: loads[r])
        cover = [i for i, (lo, hi) in enumerate(segs) if lo <= pt < hi]
        for i, j in itertools.combinations(cover, 2):
            assert j in g.adj[i]
        assert loads[pt] == peak


def test_sandwich_largest_at_zero_determinism(mp):
    rng = random.Random(99)
    for _ in range(60):
        arcs, peak = random_arcs(rng, rng.randint(2, 6))
        g = mp.conflict_graph_from_arcs(100, arcs, peak)
        opt = mp.brute_force_optimal_footprint(g)
        for policy in ("first_fit", "best_fit"):
            plan = mp.plan_pool(g, policy)
            mp.check_plan(plan, g)
            assert peak <= opt <= plan.footprint_bytes
            assert plan.offsets[max(g.vars, key=lambda pv: pv.size).var] == 0
    arcs, peak = random_arcs(random.Random(5), 30)
    g = mp.conflict_graph_from_arcs(100, arcs, peak)
    a, b = mp.plan_pool(g, "best_fit"), mp.plan_pool(g, "best_fit")
    assert a.offsets == b.offsets and a.footprint_bytes == b.footprint_bytes
    with pytest.raises(ValueError):
        mp.plan_pool(g, "worst_fit")
    with pytest.raises(mp.GraphTooLarge):
        mp.brute_force_optimal_footprint(mp.conflict_graph_from_arcs(100, random_arcs(random.Random(1), 11)[0], 0))


def test_check_plan_rejects_overlap(mp):
    g = mp.conflict_graph_from_arcs(100, [arc("a", 10, 0, 5), arc("b", 10, 3, 9)], 0)
    plan = mp.plan_pool(g, "best_fit")
    bad = mp.PoolPlan(policy=plan.policy, offsets={"a": 0, "b": 5}, sizes=plan.sizes, footprint_bytes=15,
                      peak_load_bytes=plan.peak_load_bytes)
    with pytest.raises(mp.MemplanError):
        mp.check_plan(bad, g)


def test_lookup_tables(mp):
    ops = []
    for k in (1, 2):
        ops += [("malloc", f"x{k}", 10), ("write", f"x{k}", 0), ("read", f"x{k}", 0), ("read", f"x{k}", 0),
                ("free", f"x{k}", 0), ("malloc", f"y{k}", 3), ("write", f"y{k}", 0), ("free", f"y{k}", 0)]
    prof = profile_of(mp, ops)
    table = mp.make_lookup_table(mp.plan_pool(mp.build_conflict_graph(prof), "best_fit"), prof)
    assert len(table) == 2 and 0 in table and 5 in table
    assert table.offset_for(0) == 0 and table.var_for(0) == "x2"
    empty = mp.PoolPlan(policy="best_fit", offsets={}, sizes={}, footprint_bytes=0, peak_load_bytes=0)
    with pytest.raises(mp.MissingVariable):
        mp.make_lookup_table(empty, prof)


def test_lookup_table_columns_match_loop(mp):
    """make_lookup_table's column path (untouched profile and plan) builds the
    entries the per-variable loop builds; an edited plan or a materialized
    profile takes the loop (smartpool.py:246-254)."""
    from paper_1903_06631_b200 import smartpool
    for seed in (0, 3):
        spec = mp.vgg_like(depth=6, scale=0.5, iterations=3, seed=seed)
        t = mp.generate_synthetic_trace(spec)
        win = mp.detect_iteration(t).window
        prof = mp.extract_lifetimes(t, win)
        plan = mp.plan_pool(mp.build_conflict_graph(prof), "best_fit")
        fast = smartpool._lookup_from_columns(plan, prof)
        assert fast is not None
        prof2 = mp.extract_lifetimes(t, win)
        plan2 = mp.plan_pool(mp.build_conflict_graph(prof2), "best_fit")
        _ = prof2.variables  # materialized: the loop runs
        assert smartpool._lookup_from_columns(plan2, prof2) is None
        slow = mp.make_lookup_table(plan2, prof2)
        assert fast.items() == slow.items() and len(fast) == len(slow)
        some = next(iter(slow._entries))
        assert some in fast and fast.offset_for(some) == slow.offset_for(some)
        assert fast.var_for(some) == slow.var_for(some) and -1 not in fast and "x" not in fast
        assert fast._entries == slow._entries  # the reference's dict, materialized on demand
        assert fast.items() == slow.items()
        # an edited plan is honoured
        plan3 = mp.plan_pool(mp.build_conflict_graph(prof), "best_fit")
        name = next(iter(plan3.offsets))
        plan3.offsets[name] = 12345
        t3 = mp.make_lookup_table(plan3, prof)
        assert any(v == (name, 12345) for _, v in t3.items()) or name not in {v[0] for _, v in slow.items()}


def test_replay_never_double_books_and_alpha(mp):
    for seed in (0, 4):
        spec = mp.vgg_like(depth=5, scale=0.4, iterations=4, seed=seed)
        t = mp.generate_synthetic_trace(spec)
        prof = mp.extract_lifetimes(t, mp.detect_iteration(t).window)
        plan = mp.plan_pool(mp.build_conflict_graph(prof), "best_fit")
        for r in range(prof.period):
            spans = sorted((plan.offsets[v.var], plan.offsets[v.var] + v.size) for v in prof.variables if v.covers(r))
            for (_, hi), (lo, _) in zip(spans, spans[1:]):
                assert hi <= lo
            assert spans[-1][1] <= plan.footprint_bytes
    for seed in (0, 1):
        t = mp.generate_synthetic_trace(mp.vgg_like(depth=7, scale=0.4, iterations=4, seed=seed))
        plan = mp.plan_pool(mp.build_conflict_graph(mp.extract_lifetimes(t, mp.detect_iteration(t).window)))
        assert plan.peak_load_bytes <= plan.footprint_bytes and plan.competitive_ratio <= 1.10


# --------------------------------------------------------------- autoswap
# pkg/tests/test_autoswap.py

def test_filter_threshold_gap_and_spans(mp):
    prof = profile_of(mp, filter_instance())
    assert prof.load.peak_index == 8
    assert [c.var for c in mp.filter_candidates(prof)] == ["B2"]
    assert sorted(c.var for c in mp.filter_candidates(prof, threshold_bytes=500_000)) == ["B2", "s2"]
    cands = mp.filter_candidates(prof, threshold_bytes=1)
    names = {c.var for c in cands}
    assert "F2" not in names and "T2" not in names
    b = next(c for c in cands if c.var == "B2")
    assert (b.out_index, b.in_index, b.spans_iterations) == (5, 12, False)
    c = mp.filter_candidates(prof, transfer=mp.TransferModel(bandwidth_bytes_per_s=1e9, latency_us=3.0))[0]
    assert c.delta_out_us == pytest.approx(2 * MIB / 1e9 * 1e6 + 3.0)
    ops = [("malloc", "w", 2 * MIB), ("write", "w", 0)]
    for k in (1, 2):
        ops += [("malloc", f"a{k}", 5 * MIB), ("write", f"a{k}", 0), ("free", f"a{k}", 0), ("read", "w", 0),
                ("malloc", f"s{k}", 1), ("free", f"s{k}", 0)]
    prof = profile_of(mp, ops)
    cands = mp.filter_candidates(prof)
    assert [c.var for c in cands] == ["w"]
    w = cands[0]
    assert w.spans_iterations and w.out_index == 3 and w.in_index == 3
    assert w.gap_us == pytest.approx(prof.period_duration_us)


def test_doa_aoa_and_wdoa(mp):
    assert mp.score_doa(hand_candidate(mp, 100.0, 30.0, 30.0)) == 40.0
    assert mp.score_aoa(hand_candidate(mp, 100.0, 30.0, 30.0, size=2 * MB)) == pytest.approx(80.0 * MB)
    assert mp.score_aoa(hand_candidate(mp, 50.0, 30.0, 30.0, size=2 * MB)) == pytest.approx(-10.0 / (2 * MB))
    prof = synthetic_profile(mp, [150] * 6)
    c = hand_candidate(mp, 50.0, 1.0, 1.0, out_time=10.0, out_index=1, in_index=5)
    assert mp.score_wdoa(c, prof) == pytest.approx(150 * 50.0)
    c = hand_candidate(mp, 30.0, 1.0, 1.0, out_time=40.0, out_index=4, in_index=1, spans=True)
    assert mp.score_wdoa(c, prof) == pytest.approx(150 * 30.0)
    prof = synthetic_profile(mp, [10, 10, 0, 0, 0, 10])
    assert mp.score_wdoa(hand_candidate(mp, 10.0, 1.0, 1.0, out_time=30.0, out_index=3, in_index=4), prof) == 0.0
    prof = profile_of(mp, congested())
    cands = {c.var: c for c in mp.filter_candidates(prof)}
    assert [x // MIB for x in prof.load.loads] == [25, 25, 50, 50, 75, 75, 120, 120, 75, 95, 95, 75, 75, 50, 50,
                                                   25, 25, 25, 0]
    assert mp.score_wdoa(cands["w2"], prof) == pytest.approx(9050 * MIB)
    assert mp.score_wdoa(cands["w3"], prof) == pytest.approx(6550 * MIB)


def divergence(mp):
    prof = synthetic_profile(mp, [10, 100, 100, 0, 90, 0])
    return prof, [hand_candidate(mp, 30.0, 1.0, 1.0, size=60, out_time=0.0, out_index=0, in_index=3, var="A"),
                  hand_candidate(mp, 20.0, 1.0, 1.0, size=70, out_time=10.0, out_index=1, in_index=3, var="B"),
                  hand_candidate(mp, 20.0, 1.0, 1.0, size=50, out_time=30.0, out_index=3, in_index=5, var="C")]


def test_swdoa_divergence(mp):
    prof, cands = divergence(mp)
    assert {c.var: mp.score_wdoa(c, prof) for c in cands} == {"A": 2100.0, "B": 2000.0, "C": 900.0}
    assert [c.var for c in mp.select_by_swdoa(cands, prof, limit_bytes=45)] == ["A", "C"]
    assert [c.var for c in mp.select_by_score(cands, prof, 45, score="wdoa")] == ["A", "B", "C"]
    assert mp.swdoa_scores(cands, prof) == {"A": 2100.0, "C": 900.0, "B": 800.0}
    assert len(mp.select_by_swdoa(cands, prof, limit_bytes=99)) == 1
    with pytest.raises(ValueError):
        mp.select_by_score(cands, prof, 100, score="random")


def test_selection_limits(mp):
    prof = profile_of(mp, congested())
    cands = mp.filter_candidates(prof)
    for score in ("doa", "aoa", "wdoa", "swdoa"):
        assert mp.select_by_score(cands, prof, 120 * MIB, score=score) == []
    for score in ("doa", "aoa", "wdoa", "swdoa", "combined"):
        sel = mp.select_by_score(cands, prof, 60 * MIB, score=score)
        peaks = [mp.planned_peak(sel[:k], prof) for k in range(len(sel) + 1)]
        assert peaks[0] == 120 * MIB and peaks[-1] <= 60 * MIB
        assert all(a >= b for a, b in zip(peaks, peaks[1:]))
    with pytest.raises(mp.LimitUnreachable) as exc:
        mp.select_by_swdoa(cands, prof, 40 * MIB)
    assert (exc.value.limit_bytes, exc.value.achievable_bytes) == (40 * MIB, 45 * MIB)


def test_standardize_and_combined(mp):
    got = mp.standardize([1.0, 2.0, 3.0])
    assert got[0] == pytest.approx(-1.224744871391589) and got[2] == pytest.approx(1.224744871391589)
    assert mp.standardize([5.0, 5.0, 5.0]) == [0.0, 0.0, 0.0] and mp.standardize([]) == []
    rng = random.Random(3)
    for _ in range(300):
        xs = [rng.uniform(-1e6, 1e6) for _ in range(rng.randrange(1, 30))]
        mean = sum(xs) / len(xs)
        var = sum((x - mean) ** 2 for x in xs) / len(xs)
        want = [0.0] * len(xs) if var <= 0 else [(x - mean) / var ** 0.5 for x in xs]
        assert mp.standardize(xs) == want  # bit-exact with CPython
    prof = profile_of(mp, congested())
    cands = mp.filter_candidates(prof)
    w = mp.ScoreWeights(aoa=0.0, doa=1.0, wdoa=0.0, swdoa=0.0)
    comb = mp.combined_scores(cands, prof, w)
    rank = lambda d: sorted(d, key=lambda v: -d[v])  # noqa: E731
    assert rank(comb) == rank({c.var: c.scores["doa"] for c in cands})
    for limit in (95 * MIB, 60 * MIB, 45 * MIB):
        a = mp.select_by_score(cands, prof, limit, score="doa")
        b = mp.select_by_score(cands, prof, limit, score="combined", weights=w)
        assert [c.var for c in a] == [c.var for c in b]
    with pytest.raises(ValueError):
        mp.ScoreWeights(aoa=1.5)


# --------------------------------------------------------------- swapsim
# pkg/tests/test_swapsim.py

D_W = 25 * MIB / 12e9 * 1e6 + 10.0
D_V1 = 45 * MB / 12e9 * 1e6 + 10.0
D_V3 = 34 * MB / 12e9 * 1e6 + 10.0


def swap_setup(mp, ops, limit, transfer=None, score="swdoa"):
    prof = profile_of(mp, ops)
    cands = mp.filter_candidates(prof) if transfer is None else mp.filter_candidates(prof, transfer=transfer)
    sel = mp.select_by_score(cands, prof, limit, score=score)
    return prof, cands, sel, mp.build_schedule(sel, prof)


def test_three_var_schedule_and_replay_goldens(mp):
    prof, cands, sel, sched = swap_setup(mp, three_var(), 60 * MB)
    assert [c.var for c in sel] == ["v2", "v1", "v3"] and sched.order == ["v2", "v1", "v3"]
    assert [e.var for e in sched.events] == ["v1", "v2", "v3"]
    want = {"v1": (20.0, 20.0 + D_V1, 3780.0, 3780.0 + D_V1),
            "v3": (7123.333333, 7123.333333 + D_V3, 10883.333333, 10883.333333 + D_V3)}
    for e in sched.events:
        if e.var in want:
            assert (e.t_start_out, e.t_end_out, e.t_start_in, e.t_end_in) == pytest.approx(want[e.var])
    res = mp.simulate(sched, prof, 60 * MB)
    assert res.achieved_peak_bytes == 45 * MB and res.overhead_us == pytest.approx(19853.333333)
    assert res.rounds == 2 and res.load_prime.peak_bytes == 120 * MB
    assert [d.index for d in res.delayed_ops] == [17, 19, 23, 25, 27]


def test_congested_replay_golden(mp):
    prof, cands, sel, sched = swap_setup(mp, congested(), 60 * MIB)
    assert [c.var for c in sel] == ["w1", "w2", "w3"]
    res = mp.simulate(sched, prof, 60 * MIB)
    assert res.baseline_duration_us == pytest.approx(190.0)
    assert res.overhead_us == pytest.approx(13047.2)
    assert res.achieved_peak_bytes == 50 * MIB == res.load_double_prime.peak_bytes
    assert res.load_prime.peak_bytes == 120 * MIB and res.rounds == 2
    assert [d.index for d in res.delayed_ops] == [23, 25, 31, 33, 35]
    delay_of = {d.index: d.delay_us for d in res.delayed_ops}
    assert delay_of[23] == pytest.approx(D_W - 20.0) and delay_of[25] == pytest.approx(2 * D_W - 20.0)
    final = {e.var: e for e in res.schedule.events}
    assert final["w1"].t_end_in == pytest.approx(40.0 + 6 * D_W)
    rep = mp.simulation_report(res)
    assert json.loads(json.dumps(rep)) == rep and len(rep["schedule"]) == 3


def test_fast_bus_and_free_transfers(mp):
    fast = mp.TransferModel(bandwidth_bytes_per_s=1e12, latency_us=0.1)
    prof, cands, sel, sched = swap_setup(mp, filter_instance(), 3 * MIB + 500_000, transfer=fast)
    e = sched.events[0]
    assert (e.t_start_out, e.t_end_out, e.t_start_in, e.t_end_in) == \
        pytest.approx((60.0, 62.197152, 117.802848, 120.0))
    res = mp.simulate(sched, prof, prof.load.peak_bytes)
    assert res.overhead_us == 0.0 and res.delayed_ops == [] and res.rounds == 1
    assert res.load_prime.points == res.load_double_prime.points
    instant = mp.TransferModel(bandwidth_bytes_per_s=float("inf"), latency_us=0.0)
    prof, cands, sel, sched = swap_setup(mp, three_var(), 45 * MB, transfer=instant)
    assert mp.compute_load_min(prof, cands) == 45 * MB
    res = mp.simulate(sched, prof, 45 * MB)
    assert res.overhead_us == 0.0 and res.achieved_peak_bytes == 45 * MB


def test_slow_bus_deadlocks(mp):
    t = mp.generate_synthetic_trace(mp.vgg_like(depth=6, scale=0.5, iterations=4, seed=7))
    prof = mp.extract_lifetimes(t, mp.detect_iteration(t).window)
    cands = mp.filter_candidates(prof, transfer=mp.TransferModel(bandwidth_bytes_per_s=2e9, latency_us=10.0))
    limit = int(prof.load.peak_bytes * 0.8)
    sched = mp.build_schedule(mp.select_by_score(cands, prof, limit, score="swdoa"), prof)
    with pytest.raises(mp.SwapDeadlock) as err:
        mp.simulate(sched, prof, limit)
    assert prof.window[0] <= err.value.index < prof.window[1] and "op" in str(err.value)


def test_combine_splits_lifetimes(mp):
    fast = mp.TransferModel(bandwidth_bytes_per_s=1e12, latency_us=0.1)
    prof, _, _, sched = swap_setup(mp, filter_instance(), 3 * MIB + 500_000, transfer=fast)
    res = mp.simulate(sched, prof, 3 * MIB + 500_000)
    before = mp.plan_pool(mp.build_conflict_graph(prof))
    combined = mp.combine_with_pool(prof, res.schedule)
    assert combined.period == prof.period + 2
    after_g = mp.build_conflict_graph(combined)
    names = [v.var for v in after_g.vars]
    assert "B2" not in names and len([n for n in names if n.startswith("B2")]) == 2
    assert mp.plan_pool(after_g).footprint_bytes == before.footprint_bytes - 2 * MIB
    t = mp.generate_synthetic_trace(mp.vgg_like(depth=8, scale=0.5, iterations=3, seed=1, temp_ratio=0.0))
    prof = mp.extract_lifetimes(t, mp.detect_iteration(t).window)
    alone = mp.plan_pool(mp.build_conflict_graph(prof))
    limit = int(prof.load.peak_bytes * 0.75)
    res = mp.simulate(mp.build_schedule(mp.select_by_score(mp.filter_candidates(prof), prof, limit), prof),
                      prof, limit)
    assert res.overhead_us == 0.0
    combined = mp.combine_with_pool(prof, res.schedule)
    both = mp.plan_pool(mp.build_conflict_graph(combined))
    assert res.achieved_peak_bytes <= both.footprint_bytes < alone.footprint_bytes
    assert mp.combine_with_pool(prof, mp.SwapSchedule([], {}, [], 1.0)) is prof


# --------------------------------------------------------------- estimators
# pkg/tests/test_estimators.py

def test_estimators(mp):
    from sklearn.base import clone
    an = mp.IterationAnalyzer().fit(make_trace(mp, three_var()))
    assert (an.period_, an.window_, an.peak_bytes_) == (15, (15, 30), 120 * MB)
    with pytest.raises(TypeError):
        mp.IterationAnalyzer().fit(42)
    with pytest.raises(mp.InvariantViolation):
        mp.IterationAnalyzer().fit(make_trace(mp, [("free", "x", 0), ("malloc", "x", 8)]))
    planner = mp.PoolPlanner().fit(make_trace(mp, three_var()))
    assert planner.footprint_bytes_ == planner.peak_load_bytes_ == 120 * MB and planner.alpha_ == 1.0
    assert planner.predict([0, 2, 4, 6]).tolist() == [0, 45 * MB, 85 * MB, 119 * MB]
    with pytest.raises(KeyError):
        planner.predict([1])
    with pytest.raises(ValueError):
        mp.PoolPlanner(policy="zigzag").fit(make_trace(mp, three_var()))
    sp = mp.SwapPlanner(limit_bytes=60 * MIB).fit(make_trace(mp, congested()))
    assert [c.var for c in sp.candidates_] == ["w1", "w2", "w3"] and sp.load_min_ == 45 * MIB
    assert sp.overhead_us_ == pytest.approx(13047.2) and sp.achieved_peak_bytes_ == 50 * MIB
    assert sp.result_.rounds == 2 and sp.weights_ is None
    assert not hasattr(clone(sp), "overhead_us_")
    with pytest.raises(mp.LimitUnreachable) as err:
        mp.SwapPlanner(limit_bytes=40 * MIB).fit(make_trace(mp, congested()))
    assert err.value.achievable_bytes == 45 * MIB
    sp = mp.SwapPlanner(limit_bytes=3 * MIB + 500_000, bandwidth_bytes_per_s=1e12, latency_us=0.1)
    sp.fit(make_trace(mp, filter_instance()))
    combined = sp.transform()
    assert combined.period == sp.profile_.period + 2
    before = mp.PoolPlanner().fit(sp.profile_).footprint_bytes_
    assert mp.PoolPlanner().fit(combined).footprint_bytes_ == before - 2 * MIB


def test_bo_matches_best_corner(mp):
    trace = make_trace(mp, congested())
    pure = [mp.SwapPlanner(limit_bytes=60 * MIB, score=s).fit(trace).overhead_us_ for s in mp.SCORE_NAMES]
    tuned = mp.SwapPlanner(limit_bytes=60 * MIB, score="bo", bo_budget=8, seed=0).fit(trace)
    assert isinstance(tuned.weights_, mp.ScoreWeights) and tuned.overhead_us_ <= min(pure) + 1e-9


# --------------------------------------------------------------- acceptance
# pkg/tests/test_acceptance.py

def test_a1_no_overlap_1000_graphs(mp):
    rng = random.Random(101)
    for case in range(1000):
        arcs, peak = random_arcs(rng, rng.randrange(5, 501))
        g = mp.conflict_graph_from_arcs(100, arcs, peak)
        plan = mp.plan_pool(g)
        assert plan.footprint_bytes >= peak
        offs = plan.offset_array
        sizes = np.array([a[1] for a in arcs])
        row, col = __import__("paper_1903_06631_b200._native", fromlist=["x"]).graph_csr(g._dev)
        src = np.repeat(np.arange(len(arcs)), np.diff(row))
        lo_i, hi_i = offs[src], offs[src] + sizes[src]
        lo_j, hi_j = offs[col], offs[col] + sizes[col]
        assert np.all((hi_i <= lo_j) | (hi_j <= lo_i)), case


def test_a3_a5_a8(mp):
    for depth in (4, 8, 12):
        for scale in (0.25, 1.0, 4.0):
            t = mp.generate_synthetic_trace(mp.vgg_like(depth=depth, scale=scale, iterations=3, seed=0))
            plan = mp.plan_pool(mp.build_conflict_graph(mp.extract_lifetimes(t, mp.detect_iteration(t).window)))
            assert plan.competitive_ratio <= 1.10
    for depth, scale, iters, seed in ((8, 0.5, 3, 1), (6, 1.0, 3, 2), (10, 0.25, 4, 3)):
        t = mp.generate_synthetic_trace(mp.vgg_like(depth=depth, scale=scale, iterations=iters, seed=seed,
                                                    temp_ratio=0.0))
        prof = mp.extract_lifetimes(t, mp.detect_iteration(t).window)
        peak = prof.load.peak_bytes
        cands = mp.filter_candidates(prof)
        load_min = mp.compute_load_min(prof, cands)
        best = 0.0
        for pct in range(95, 30, -5):
            limit = int(peak * pct / 100)
            if limit < load_min:
                break
            res = mp.simulate(mp.build_schedule(mp.select_by_score(cands, prof, limit), prof), prof, limit)
            if res.overhead_us == 0.0:
                best = max(best, 1.0 - res.achieved_peak_bytes / peak)
        assert best >= 0.25
    rng = random.Random(808)
    for seed in range(100):
        spec = mp.vgg_like(depth=rng.randrange(3, 9), scale=0.25 * rng.randrange(1, 5),
                           iterations=rng.randrange(3, 11), seed=seed)
        t = mp.generate_synthetic_trace(spec)
        assert mp.detect_iteration(t).period == t.meta["period"]
