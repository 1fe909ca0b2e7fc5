"""In-place edit programs: the same steps run against the reference package
(tests/golden/make_golden_edits.py, build container) and against the drop-in
(tests/test_gpu_dropin_edits.py, GPU box).  Each program takes the package
module ``m`` and returns a JSON-ready list of observations.

The reference keeps no cache: ``validate_trace``/``detect_iteration``/
``extract_lifetimes`` re-read ``trace.events`` (trace.py:55-84,
iteration.py:93-301), ``build_conflict_graph`` reads ``profile.variables``
(smartpool.py:82-88) and ``plan_pool`` reads ``graph.vars``/``graph.adj``
(smartpool.py:122-144) on every call.  These programs edit those containers
in place between calls and record what each call returns, so a drop-in that
reuses a device copy after an edit fails them.
"""
from __future__ import annotations

import dataclasses


def _err(m, ex):
    if isinstance(ex, m.InvariantViolation):
        return ["InvariantViolation", ex.index, ex.reason]
    return [type(ex).__name__, str(ex)]


def _guard(m, fn):
    try:
        return ["ok", fn()]
    except (m.MemplanError, ValueError, IndexError, KeyError) as ex:
        return ["err", _err(m, ex)]


def _profile_summary(prof):
    return {"period": prof.period, "window": list(prof.window), "peak": prof.load.peak_bytes,
            "peak_index": prof.load.peak_index, "loads": list(prof.load.loads),
            "vars": [[v.var, v.size, v.alloc_index, v.free_index, [list(s) for s in v.segments], v.persistent,
                      v.wraps, len(v.accesses)] for v in prof.variables]}


def _plans(m, g):
    out = {}
    for pol in ("best_fit", "first_fit"):
        plan = m.plan_pool(g, pol)
        out[pol] = [[pv.var, plan.offsets[pv.var]] for pv in g.vars] + [plan.footprint_bytes]
    return out


def _trace(m, depth=5, seed=3):
    return m.generate_synthetic_trace(m.vgg_like(depth=depth, scale=0.5, iterations=3, seed=seed))


def _first(trace, kind):
    return next(i for i, e in enumerate(trace.events) if e.kind.value == kind)


def trace_replace_event(m):
    """Replace one malloc (and its matching free stays valid) with a larger
    size: detect/extract must see the new size."""
    t = _trace(m)
    obs = []
    d = m.detect_iteration(t)
    obs.append(["detect", d.period, list(d.window)])
    obs.append(["extract", _profile_summary(m.extract_lifetimes(t, d.window))])
    k = [i for i, e in enumerate(t.events) if e.kind.value == "malloc"][-3]
    e = t.events[k]
    t.events[k] = dataclasses.replace(e, size=e.size * 3 + 512)
    obs.append(["validate", _guard(m, lambda: m.validate_trace(t))])
    d2 = _guard(m, lambda: m.detect_iteration(t))
    obs.append(["detect", d2[0], [d2[1].period, list(d2[1].window)] if d2[0] == "ok" else d2[1]])
    obs.append(["extract", _profile_summary(m.extract_lifetimes(t, d.window))])
    return obs


def trace_break_invariant(m):
    """An edit that makes the trace invalid: validation must now raise."""
    t = _trace(m, depth=4, seed=5)
    obs = [["validate", _guard(m, lambda: m.validate_trace(t))]]
    k = _first(t, "free") + 7
    e = t.events[k]
    t.events[k] = dataclasses.replace(e, t_us=-1)
    obs.append(["validate", _guard(m, lambda: m.validate_trace(t))])
    t.events[k] = e
    obs.append(["validate", _guard(m, lambda: m.validate_trace(t))])
    # a free turned into a read of the same id keeps the id live: a later
    # malloc of it is a malloc of a live id
    k = _first(t, "free")
    e = t.events[k]
    t.events[k] = dataclasses.replace(e, kind=m.EventKind.READ)
    obs.append(["validate", _guard(m, lambda: m.validate_trace(t))])
    t.events[k] = e
    k = _first(t, "read")
    t.events[k] = dataclasses.replace(t.events[k], size=4)
    obs.append(["validate", _guard(m, lambda: m.validate_trace(t))])
    return obs


def trace_append_window(m):
    """Events appended after the first analysis: a longer trace."""
    t = _trace(m, depth=4, seed=7)
    d = m.detect_iteration(t)
    obs = [["detect", d.period, list(d.window)]]
    tail = t.events[d.window[0]:d.window[1]]
    base = len(t.events)
    dt = t.events[-1].t_us + 1 - tail[0].t_us
    t.events.extend(dataclasses.replace(e, index=base + i, t_us=e.t_us + dt) for i, e in enumerate(tail))
    d2 = m.detect_iteration(t)
    obs.append(["detect", d2.period, list(d2.window)])
    obs.append(["extract", _profile_summary(m.extract_lifetimes(t, d2.window))])
    return obs


def profile_edit_sizes(m):
    """Variable sizes edited in place after extraction: the conflict graph,
    the plan and the swap candidates follow the new sizes."""
    t = _trace(m, depth=6, seed=11)
    d = m.detect_iteration(t)
    prof = m.extract_lifetimes(t, d.window)
    obs = [["plan", _plans(m, m.build_conflict_graph(prof))]]
    vs = prof.variables
    big = max(range(len(vs)), key=lambda i: vs[i].size)
    vs[big].size = vs[big].size // 3 + 8
    small = min(range(len(vs)), key=lambda i: (vs[i].size, vs[i].var))
    vs[small].size = vs[big].size * 5
    obs.append(["plan", _plans(m, m.build_conflict_graph(prof))])
    return obs


def profile_edit_segments(m):
    """A lifetime's segments edited in place: new conflicts."""
    t = _trace(m, depth=6, seed=13)
    d = m.detect_iteration(t)
    prof = m.extract_lifetimes(t, d.window)
    g0 = m.build_conflict_graph(prof)
    obs = [["plan", _plans(m, g0)]]
    v = next(x for x in prof.variables if not x.persistent and len(x.segments) == 1)
    v.segments = ((0, prof.period),)
    g1 = m.build_conflict_graph(prof)
    obs.append(["edges", sum(len(a) for a in g1.adj)])
    obs.append(["plan", _plans(m, g1)])
    # the first graph is a snapshot of the profile before the edit
    obs.append(["plan_old", _plans(m, g0)])
    return obs


def graph_edit_adj(m):
    """Adjacency and sizes of a built graph edited in place between plans."""
    t = _trace(m, depth=5, seed=17)
    d = m.detect_iteration(t)
    prof = m.extract_lifetimes(t, d.window)
    g = m.build_conflict_graph(prof)
    obs = [["plan", _plans(m, g)]]
    n = len(g.vars)
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n) if j not in g.adj[i]][:6]
    for i, j in pairs:
        g.adj[i].add(j)
        g.adj[j].add(i)
    obs.append(["plan", _plans(m, g)])
    g.vars[n // 2].size = g.vars[0].size + 4096
    obs.append(["plan", _plans(m, g)])
    i, j = pairs[0]
    g.adj[i].discard(j)  # now one-sided
    obs.append(["plan", _plans(m, g)])
    return obs


def graph_asymmetric(m):
    """Hand-built graphs whose adjacency is not symmetric, with self loops
    and negative ids: plan_pool reads only adj[i] when placing i."""
    obs = []
    sizes = [96, 64, 64, 48, 32, 32, 16, 8]
    pv = [m.smartpool.PoolVar(f"v{i}", s, i, ((i, i + 3),), False) for i, s in enumerate(sizes)]
    adj = [{1, 2}, set(), {0, 1, 2}, {0, -1}, {3, 2}, {4, 5}, {0, 1, 2, 3, 4, 5}, {6}]
    g = m.ConflictGraph(period=12, vars=pv, adj=adj, peak_load_bytes=160)
    obs.append(["plan", _plans(m, g)])
    g.adj[1].add(0)
    obs.append(["plan", _plans(m, g)])
    bad = m.ConflictGraph(period=12, vars=pv[:3], adj=[{1}, {5}, set()], peak_load_bytes=10)
    obs.append(["bad", _guard(m, lambda: _plans(m, bad))])
    return obs


def _arcs_random(seed, nvars, max_segs, span, offset=0):
    import random
    rng = random.Random(seed)
    arcs = []
    for i in range(nvars):
        segs = []
        for _ in range(rng.choice([1, 2, max_segs // 2, max_segs])):
            lo = rng.randrange(span)
            segs.append((offset + lo, offset + lo + rng.choice([0, 1, 2, rng.randrange(1, span // 4 + 2)])))
        arcs.append((f"a{i:03d}", rng.randrange(1, 1 << 20), rng.randrange(-1, 40), tuple(segs), rng.random() < 0.1))
    return arcs


def _arcs_graph(m, arcs):
    g = m.conflict_graph_from_arcs(64, arcs, 1 << 22)
    return [["adj", [sorted(a) for a in g.adj]], ["plan", _plans(m, g)]]


def arcs_many_segments(m):
    """Variables with up to 300 (self-overlapping, some empty) segments."""
    return _arcs_graph(m, _arcs_random(23, 40, 300, 4000))


def arcs_large_bounds(m):
    """Segment bounds far outside 32 bits."""
    return _arcs_graph(m, _arcs_random(29, 60, 6, 1000, offset=(1 << 40) - 500))


PROGRAMS = {f.__name__: f for f in (arcs_many_segments, arcs_large_bounds, trace_replace_event, trace_break_invariant, trace_append_window,
                                     profile_edit_sizes, profile_edit_segments, graph_edit_adj,
                                     graph_asymmetric)}
