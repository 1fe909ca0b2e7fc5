"""Host logic of the swap executor (swapexec.py): absence windows under a
limit, hook-point feasibility, split pool arcs and served offsets."""
from types import SimpleNamespace

import numpy as np

from paper_1903_06631_b200 import swapexec
from paper_1903_06631_b200.autoswap import SwapCandidate
from paper_1903_06631_b200.iteration import VariableLifetime


def cand(var, size, out_i, in_i, spans=False):
    return SwapCandidate(var=var, size=size, out_index=out_i, out_time_us=float(out_i), out_ready_us=float(out_i),
                         in_index=in_i, in_time_us=float(in_i), delta_out_us=1.0, delta_in_us=1.0,
                         spans_iterations=spans)


def var(name, size, alloc, free, wraps=False):
    segs = ((alloc, free),) if not wraps else ((alloc, 20), (0, free))
    return VariableLifetime(var=name, base_var=name, size=size, alloc_index=alloc, free_index=free,
                            segments=segs, accesses=[], persistent=False, wraps=wraps)


def profile(loads, variables):
    return SimpleNamespace(load=SimpleNamespace(loads=list(loads)), variables=variables, period=len(loads))


def test_absence_covers_exactly_the_over_limit_events():
    loads = [10] * 20
    for r in range(8, 13):
        loads[r] = 30
    prof = profile(loads, [var("x", 15, 1, 18)])
    points = np.arange(20) * 2  # one event per op: event r sits before op r
    acts, skipped = swapexec.plan_actions(prof, [cand("x", 15, 3, 16)], 20, points, {"x": 0})
    assert not skipped
    (x,) = acts
    assert (x.a, x.b) == (8, 13)
    assert x.issue_out == points[3] + 1 and x.wait_out == points[8]
    assert x.issue_in == points[12] + 1 and x.wait_in == points[16]


def test_not_needed_and_spanning_candidates_are_skipped():
    prof = profile([5] * 10, [var("x", 4, 0, 9)])
    acts, skipped = swapexec.plan_actions(prof, [cand("x", 4, 1, 8), cand("y", 4, 1, 8, spans=True)], 10,
                                          np.arange(10) * 2, {"x": 0})
    assert not acts
    assert [s["why"] for s in skipped] == ["not needed under the limit",
                                          "not executable (spans iterations / not pool-served)"]


def test_later_selection_sees_earlier_absences():
    loads = [10] * 20
    for r in range(8, 13):
        loads[r] = 30
    prof = profile(loads, [var("x", 25, 1, 18), var("y", 25, 1, 18)])
    acts, skipped = swapexec.plan_actions(prof, [cand("x", 25, 3, 16), cand("y", 25, 3, 16)], 20,
                                          np.arange(20) * 2, {"x": 0, "y": 1})
    assert [a.var for a in acts] == ["x"]
    assert skipped[0]["why"] == "not needed under the limit"


def test_same_op_events_push_the_window_to_op_boundaries():
    # events 3..5 belong to one op (point 6): the D2H of the access at event
    # 3 can only be waited from the next op on
    loads = [10] * 12
    for r in range(4, 9):
        loads[r] = 30
    points = np.array([0, 2, 4, 6, 6, 6, 8, 10, 12, 14, 16, 18])
    prof = profile(loads, [var("x", 25, 0, 11)])
    acts, _ = swapexec.plan_actions(prof, [cand("x", 25, 3, 10)], 20, points, {"x": 0})
    (x,) = acts
    assert x.a == 6 and x.wait_out >= x.issue_out
    assert x.issue_in <= x.wait_in


def test_split_arcs_and_served_offsets():
    prof = profile([0] * 20, [var("x", 1024, 1, 18), var("w", 512, 9, 12),
                              VariableLifetime("carry", "carry", 64, None, 4, ((0, 4),), [], False, False)])
    act = swapexec.SwapAction("x", 0, 1024, 3, 8, 13, 16, 7, 16, 25, 32)
    arcs = swapexec.split_arcs(prof, [act])
    by = {a[0]: a for a in arcs}
    assert "carry" not in by  # carry-ins are not pool-served
    assert by["x"][3] == ((1, 8), (13, 18)) and by["x"][1] == 1024 + swapexec.SWAP_LEAD
    assert by["w"][3] == ((9, 12),)
    offs = swapexec.served_offsets(arcs, {"x": 0, "w": 0}, [act])
    assert offs == {"x": swapexec.SWAP_LEAD, "w": 0}


def test_window_slots_follow_allocation_order():
    prof = profile([0] * 10, [var("b", 8, 5, 9), var("a", 8, 2, 9), var("~iteration", 1, 7, 8)])
    assert swapexec.window_slots(prof) == {"a": 0, "b": 1}


# ---- select_window_fits: copies must fit the executor's windows ----

def _wf_profile(loads, times):
    return SimpleNamespace(load=SimpleNamespace(loads=list(loads)), op_times_us=list(times), period=len(loads))


def test_window_fits_keeps_a_candidate_whose_copies_fit():
    from paper_1903_06631_b200.errors import LimitUnreachable
    loads = [10] * 20
    for r in range(8, 13):
        loads[r] = 30
    times = [100.0 * r for r in range(20)]          # 100 us per op
    points = np.arange(20) * 2
    c = cand("x", 1000, 1, 18)                       # 1000 B at 1e8 B/s = 10 us each way
    sel = swapexec.select_window_fits(_wf_profile(loads, times), [c], 20, points, {"x": 0}, 1e8, 1e8,
                                      latency_us=0.0, margin=1.0)
    assert [s.var for s in sel] == ["x"]
    # a link too slow for the window: D2H (from t[2]=200) must end by t[8]=800
    try:
        swapexec.select_window_fits(_wf_profile(loads, times), [c], 20, points, {"x": 0}, 1e6, 1e8,
                                    latency_us=0.0, margin=1.0)
        raise AssertionError("expected LimitUnreachable")
    except LimitUnreachable:
        pass
    # ... unless the stall budget covers the predicted wait (1000 us - 600 us)
    sel = swapexec.select_window_fits(_wf_profile(loads, times), [c], 20, points, {"x": 0}, 1e6, 1e8,
                                      latency_us=0.0, margin=1.0, stall_budget_us=400.0)
    assert [s.var for s in sel] == ["x"]


def test_window_fits_serializes_copies_on_one_stream():
    from paper_1903_06631_b200.errors import LimitUnreachable
    loads = [1000] * 20
    for r in range(8, 13):
        loads[r] = 2000
    times = [100.0 * r for r in range(20)]
    points = np.arange(20) * 2
    # each needs 500 us of D2H after t[2] = 200: on one stream the second
    # would end at 1200 > t[8] = 800
    cs = [cand("x", 500, 1, 18), cand("y", 500, 1, 18)]
    try:
        swapexec.select_window_fits(_wf_profile(loads, times), cs, 1000, points, {"x": 0, "y": 1}, 1e6, 1e8,
                                    latency_us=0.0, margin=1.0)
        raise AssertionError("expected LimitUnreachable")
    except LimitUnreachable:
        pass
    # one of them suffices for a looser limit
    sel = swapexec.select_window_fits(_wf_profile(loads, times), cs, 1500, points, {"x": 0, "y": 1}, 1e6, 1e8,
                                      latency_us=0.0, margin=1.0)
    assert len(sel) == 1
