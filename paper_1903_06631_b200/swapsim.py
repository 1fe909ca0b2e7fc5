"""Swap scheduling and discrete-event simulation (drop-in for memplan.swapsim).

Reference: pkg/src/memplan/swapsim.py:1-514.  ``_make_schedule`` and the
LOAD'/LOAD'' replay with its fixed-point deadline refinement run on the
device (csrc/swap.cu); ``combine_with_pool`` rewrites the window's op list
on the host and re-extracts lifetimes on the device with the rewritten op
times (mp_extract_times).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .autoswap import SwapCandidate, _cands
from .errors import SwapDeadlock  # noqa: F401  (re-raised from the device status)
from .iteration import IterationProfile, device_profile
from .trace import EventKind, TraceArrays

INF = float("inf")
_EPS_US = 1e-6


@dataclass(frozen=True)
class SwapEvent:
    var: str
    size: int
    t_start_out: float
    t_end_out: float
    t_start_in: float
    t_end_in: float


@dataclass
class SwapSchedule:
    events: list[SwapEvent]
    candidates: dict[str, SwapCandidate]
    order: list[str]
    period_duration_us: float

    @property
    def by_var(self) -> dict[str, SwapEvent]:
        return {e.var: e for e in self.events}

    def __len__(self) -> int:
        return len(self.events)

    def __iter__(self):
        return iter(self.events)


def _schedule_from(selection, times, event_order, duration) -> SwapSchedule:
    so, eo, si, ei = times
    events = [SwapEvent(selection[s].var, selection[s].size, float(so[s]), float(eo[s]), float(si[s]),
                        float(ei[s])) for s in event_order]
    return SwapSchedule(events=events, candidates={c.var: c for c in selection},
                        order=[c.var for c in selection], period_duration_us=duration)


def _make_schedule(selection: list[SwapCandidate], ready: dict[str, float], deadline: dict[str, float],
                   duration_us: float) -> SwapSchedule:
    """Serialize transfers on one duplex channel (swapsim.py:62-108)."""
    if not selection:
        return SwapSchedule(events=[], candidates={}, order=[], period_duration_us=duration_us)
    times, eorder = N.swap_schedule(_cands(selection), np.arange(len(selection), dtype=np.int32),
                                    [ready[c.var] for c in selection], [deadline[c.var] for c in selection])
    return _schedule_from(selection, times, eorder.tolist(), duration_us)


def build_schedule(selection: list[SwapCandidate], profile: IterationProfile) -> SwapSchedule:
    """Outs from each candidate's ready time, ins back-scheduled from its next
    access (swapsim.py:111-116)."""
    ready = {c.var: c.out_ready_us for c in selection}
    deadline = {c.var: c.in_time_us for c in selection}
    return _make_schedule(list(selection), ready, deadline, profile.period_duration_us)


@dataclass(frozen=True)
class DelayedOp:
    index: int
    delay_us: float


@dataclass
class LoadCurve:
    points: list[tuple[float, int]]
    peak_bytes: int
    peak_time_us: float


@dataclass
class SimulationResult:
    limit_bytes: int | None
    baseline_duration_us: float
    duration_us: float
    overhead_us: float
    overhead_pct: float
    achieved_peak_bytes: int
    delayed_ops: list[DelayedOp]
    load_prime: LoadCurve
    load_double_prime: LoadCurve
    schedule: SwapSchedule
    rounds: int = 1


def _curve(t, v, peak, peak_t) -> LoadCurve:
    return LoadCurve(points=list(zip(t.tolist(), v.tolist())), peak_bytes=int(peak), peak_time_us=float(peak_t))


def simulate(schedule: SwapSchedule, profile: IterationProfile, limit_bytes: int | None,
             max_rounds: int = 100) -> SimulationResult:
    """Replay the window under the plan, refining swap-in deadlines from the
    actual access times until the total delay is stable (swapsim.py:349-395)."""
    d_nat = profile.period_duration_us
    selection = [schedule.candidates[v] for v in schedule.order]
    n = len(selection)
    pos = {c.var: i for i, c in enumerate(selection)}
    by_var = schedule.by_var
    cands = _cands(selection)
    if n:
        # the replay charges each event's own size (swapsim.py:215)
        cands.size = np.array([by_var[c.var].size for c in selection], np.int64)
    so = [by_var[c.var].t_start_out for c in selection]
    eo = [by_var[c.var].t_end_out for c in selection]
    si = [by_var[c.var].t_start_in for c in selection]
    ei = [by_var[c.var].t_end_in for c in selection]
    eorder = [pos[e.var] for e in schedule.events]
    dp = device_profile(profile)
    res = N.swap_simulate(dp, profile.period, cands, np.arange(n, dtype=np.int32), ((so, eo, si, ei), eorder),
                          limit_bytes, max_rounds, cand_names=[c.var for c in selection])
    delay = res["delay"]
    rounds = res["rounds"]
    refined = rounds > 1 or (max_rounds == 1 and n > 0 and delay != 0.0)
    final = schedule
    if refined:
        final = _schedule_from(selection, (res["t_so"], res["t_eo"], res["t_si"], res["t_ei"]),
                               res["event_order"].tolist(), d_nat)
    return SimulationResult(
        limit_bytes=limit_bytes, baseline_duration_us=d_nat, duration_us=d_nat + delay, overhead_us=delay,
        overhead_pct=delay / d_nat * 100.0 if d_nat > 0 else 0.0, achieved_peak_bytes=res["ldp"][2],
        delayed_ops=[DelayedOp(int(i), float(u)) for i, u in zip(*res["delayed"])],
        load_prime=_curve(*res["lp"]), load_double_prime=_curve(*res["ldp"]), schedule=final, rounds=rounds)


def compute_load_min(profile: IterationProfile, candidates: list[SwapCandidate]) -> int:
    """Residual peak with every candidate absent (swapsim.py:398-405)."""
    if not profile.period:
        return 0
    return int(N.swap_planned_peak(device_profile(profile), _cands(candidates)))


def combine_with_pool(profile: IterationProfile, schedule: SwapSchedule) -> IterationProfile:
    """Split each swapped variable's lifetime at its scheduled absence and
    rebuild the profile for pool planning (swapsim.py:408-492).

    The op-list rewrite (synthetic free at the swap-out end, malloc at the
    re-entry) is host bookkeeping over O(p + swaps) tuples; the rebuilt
    lifetimes come from the device extractor, fed the rewritten op times.
    """
    if not schedule.events:
        return profile
    if not profile.events:
        raise ValueError("profile has no raw events to rewrite")
    p = profile.period
    tau = profile.op_times_us
    d = profile.period_duration_us
    variables = profile.variables
    sizes = {v.var: v.size for v in variables}
    var_by = {v.var: v for v in variables}
    op_instance = profile.op_instance
    events = profile.events
    ops = []  # (time, rank, seq, kind, id, size); rank: synthetic malloc < op < synthetic free
    for r in range(p):
        name = op_instance[r]
        kind = events[r].kind
        ops.append((tau[r], 1, r, kind, name, sizes[name] if kind == EventKind.MALLOC else 0))
    seq = p
    span_split: set[str] = set()
    plain_split_seq: dict[str, int] = {}
    for e in schedule.events:
        c = schedule.candidates[e.var]
        v = var_by[e.var]
        s = sizes[e.var]
        if not c.spans_iterations:
            bound = tau[v.free_index] if v.free_index is not None else d
            w_in = min(e.t_start_in, tau[c.in_index])
            if not e.t_end_out < w_in <= bound:
                continue
            ops.append((e.t_end_out, 2, seq, EventKind.FREE, e.var, 0))
            seq += 1
            ops.append((w_in, 0, seq, EventKind.MALLOC, e.var, s))
            plain_split_seq[e.var] = seq
            seq += 1
        else:
            w = min(max(e.t_start_in - d, 0.0), tau[c.in_index])
            if e.t_end_out > d or w >= e.t_end_out:
                continue
            if not v.persistent and (v.free_index is None or w > tau[v.free_index]):
                continue
            span_split.add(e.var)
            ops.append((w, 0, seq, EventKind.MALLOC, e.var, s))
            seq += 1
            ops.append((e.t_end_out, 2, seq, EventKind.FREE, e.var, 0))
            seq += 1
    ops.sort(key=lambda o: (o[0], o[1], o[2]))
    pos_by_seq = {o[2]: i for i, o in enumerate(ops) if o[3] == EventKind.MALLOC}
    live_start: dict[str, tuple[int, int | None]] = {}
    for v in variables:
        if v.var in span_split:
            continue
        if v.alloc_index is None:
            if v.persistent and v.var in plain_split_seq:
                twin = pos_by_seq.get(plain_split_seq[v.var])
            elif v.wraps or v.persistent:
                twin = None
            else:
                continue
            live_start[v.var] = (v.size, twin)
        elif v.wraps and not v.persistent:
            live_start[v.var] = (v.size, pos_by_seq.get(v.alloc_index))
    return _profile_from_ops([(o[3], o[4], o[5]) for o in ops], [o[0] for o in ops], d, live_start,
                             profile.window)


def _profile_from_ops(window_ops, op_times, duration, live_start, window) -> IterationProfile:
    """build_profile (iteration.py:135-272) on the device: the carry-in set
    becomes a synthetic prefix whose mallocs sit where each twin_rel says
    (one period before the window; earlier when there is no twin), then the
    window is extracted with the given op times."""
    q = len(window_ops)
    no_twin = [b for b, (_s, t) in live_start.items() if t is None]
    lead = len(no_twin)
    start = lead + q
    kinds, names, sizes = [], [], []
    slot = [None] * q
    for b, (s, t) in live_start.items():
        if t is not None:
            slot[t] = (b, s)
    filler = "\x00filler"
    for b in no_twin:
        kinds.append(0)
        names.append(b)
        sizes.append(live_start[b][0])
    for r in range(q):
        if slot[r] is None:
            kinds.append(2)  # a read: invisible to the live-set scan
            names.append(filler)
            sizes.append(0)
        else:
            kinds.append(0)
            names.append(slot[r][0])
            sizes.append(slot[r][1])
    code = {EventKind.MALLOC: 0, EventKind.FREE: 1, EventKind.READ: 2, EventKind.WRITE: 3}
    for kind, name, size in window_ops:
        kinds.append(code[kind])
        names.append(name)
        sizes.append(size)
    n = len(kinds)
    arrays = TraceArrays.from_columns(np.array(kinds, np.uint8), names, np.array(sizes, np.int64),
                                      np.zeros(n, np.int64))
    dp = N.extract_times(arrays, start, n, np.asarray(op_times, np.float64), float(duration))
    prof = IterationProfile._from_device(dp, arrays, (start, n))
    prof.__dict__["window"] = tuple(window)
    prof._flat = None
    fp = prof._flat_profile()
    fp.window = tuple(window)
    prof.__dict__["events"] = []
    prof.__dict__["_pending"] = tuple(x for x in prof._pending if x != "events")
    return prof


def simulation_report(result: SimulationResult) -> dict:
    """JSON-ready summary of a simulation pass (swapsim.py:495-514)."""
    return {
        "limit": result.limit_bytes, "baseline_duration_us": result.baseline_duration_us,
        "duration_us": result.duration_us, "overhead_us": result.overhead_us,
        "overhead_pct": result.overhead_pct, "achieved_peak": result.achieved_peak_bytes,
        "rounds": result.rounds,
        "delayed_ops": [{"index": o.index, "delay_us": o.delay_us} for o in result.delayed_ops],
        "schedule": [{"var": e.var, "t_so": e.t_start_out, "t_eo": e.t_end_out, "t_si": e.t_start_in,
                      "t_ei": e.t_end_in} for e in result.schedule.events],
    }
