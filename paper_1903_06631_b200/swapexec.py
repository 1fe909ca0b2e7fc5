"""Execute an AutoSwap plan on a PyTorch training iteration.

The reference stops at the plan: ``SwapSchedule`` + ``simulate``
(swapsim.py:62-395) predict the overhead of moving each selected variable to
host memory during its longest access gap.  This module runs that plan on
the device, next to the SmartPool allocator (torchmem.py):

* every selected variable keeps ONE pool offset; its lifetime splits into two
  segments around the absence ``[a, b)`` (event indices of the window), and
  the pool is planned on those split arcs (``conflict_graph_from_arcs``), so
  other variables reuse its bytes while it is on the host
  (combine_with_pool, swapsim.py:408-492, restated on event indices);
* a ``TorchDispatchMode`` counts the iteration's aten ops; at hook points
  before/after op k the executor issues, on two copy streams (D2H and H2D —
  PCIe/C2C is duplex):
    - after the out access's op: record an event on the compute stream, the
      D2H stream waits on it and copies the variable to pinned host memory;
    - before event a (first malloc that may reuse the bytes): the compute
      stream waits for the D2H;
    - after event b-1 (every variable sharing the bytes is dead): record, the
      H2D stream waits and copies the variable back;
    - before the in access's op: the compute stream waits for the H2D.
  Event ordering makes the execution correct whatever the real timings are;
  ``[a, b)`` is where the memory limit needs the variable gone
  (``plan_actions``), the stalls are the price of the limit.

Hook points: 2k = before op k, 2k+1 = after op k (k = 1-based op ordinal
inside the iteration; point 1 = iteration start).  An event recorded inside
op k sits at 2k, an allocator record between op k and op k+1 at 2k+1.
Only window-allocated, non-wrapping variables are executed (activations and
their gradients); carry-ins (weights, optimizer state) are not pool-served.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from .torchmem import MARK_NAME

_DEBUG = bool(os.environ.get("MP_SWAP_DEBUG"))


@dataclass
class SwapAction:
    var: str
    slot: int          # malloc ordinal in the iteration
    size: int
    out_index: int     # window event indices
    a: int
    b: int
    in_index: int
    issue_out: int     # hook points
    wait_out: int
    issue_in: int
    wait_in: int


def event_points(tracer, window) -> tuple[np.ndarray, int]:
    """Hook point of every window event (see module docstring) and the op
    ordinal the window starts after."""
    start, end = window
    seqs = np.asarray(tracer.event_seq, np.int64)
    mark_seqs = sorted(s for s, _t in tracer.marks)
    # the window starts right after a mark: ops are numbered from it
    base = max([s for s in mark_seqs if s <= seqs[start]] or [seqs[start] - 1])
    # an event whose op ordinal s has span (lo, hi): records inside the op
    # were tagged s; reads/writes too.  A record tagged s that lies outside
    # the op's span happened between op s and op s+1.
    pts = np.zeros(end - start, np.int64)
    kinds = tracer._event_where  # 0 inside/at op, 1 after op
    for i in range(start, end):
        k = int(seqs[i] - base)
        pts[i - start] = 2 * k + int(kinds[i])
    return pts, int(base)


def next_point(pt: int) -> int:
    """First hook point after the event at ``pt`` (its op has been issued)."""
    return pt + 1


def schedule_in_events(profile, sim) -> dict[str, int]:
    """Window event index at which the reference's replay starts each
    swap-in: the first op whose replayed start time (natural time plus the
    delays ``simulate`` charged before it, swapsim.py:303-340) is at or after
    the final schedule's ``t_start_in`` (swapsim.py:84-96).  Spanning
    candidates (swap-in in the next iteration) are not mapped."""
    tau = np.asarray(profile.op_times_us, np.float64)
    delay = np.zeros(len(tau), np.float64)
    w0 = profile.window[0]
    for d in sim.delayed_ops:
        delay[d.index - w0] += d.delay_us
    actual = tau + np.cumsum(delay)
    out = {}
    for e in sim.schedule.events:
        c = sim.schedule.candidates[e.var]
        if c.spans_iterations:
            continue
        out[e.var] = int(np.searchsorted(actual, e.t_start_in - 1e-6, side="left"))
    return out


def plan_actions(profile, selection, limit_bytes: int, points, slot_of,
                 in_events: dict | None = None) -> tuple[list[SwapAction], list[dict]]:
    """Absence of each selected variable, in selection (priority) order:
    from the first to the last event of its access gap where the load,
    with the absences decided so far, is still above the limit.  Leaving as
    late and returning as early as the limit allows keeps the stalls (the
    copy/compute event waits) as short as the memory target permits.
    With ``in_events`` (``schedule_in_events``) a swap-in is issued at the
    reference schedule's start instead, or as soon after it as the pool
    bytes are free, and never after the op that waits for it.
    Returns the executable actions and the skipped ones with the reason."""
    loads = np.asarray(profile.load.loads, np.int64).copy()
    acts, skipped = [], []
    for c in selection:
        if c.spans_iterations or c.var not in slot_of:
            skipped.append({"var": c.var, "why": "not executable (spans iterations / not pool-served)"})
            continue
        r1, r2 = int(c.out_index), int(c.in_index)
        over = np.nonzero(loads[r1 + 1:r2] > limit_bytes)[0]
        if over.size == 0:
            skipped.append({"var": c.var, "why": "not needed under the limit"})
            continue
        a = r1 + 1 + int(over[0])
        b = r1 + 1 + int(over[-1]) + 1
        # the D2H is issued after the out access's op and waited before a;
        # the H2D is issued after event b-1's op and waited before r2
        while a < b and next_point(points[r1]) > points[a]:
            a += 1
        while b > a and next_point(points[b - 1]) > points[r2]:
            b -= 1
        if b <= a:
            skipped.append({"var": c.var, "why": "no absence window at op granularity"})
            continue
        loads[a:b] -= c.size
        issue_in = int(next_point(points[b - 1]))
        if in_events is not None and c.var in in_events:
            ev = in_events[c.var]
            if ev < len(points):
                issue_in = max(issue_in, min(int(points[ev]), int(points[r2])))
        acts.append(SwapAction(c.var, slot_of[c.var], int(c.size), r1, a, b, r2, int(next_point(points[r1])),
                               int(points[a]), issue_in, int(points[r2])))
    return acts, skipped


def select_window_fits(profile, cands, limit_bytes: int, points, slot_of, d2h_bytes_per_s: float,
                       h2d_bytes_per_s: float, latency_us: float = 10.0, margin: float = 0.9,
                       stall_budget_us: float = 0.0, order=None):
    """An executor-aware selection (not the reference's): candidates largest
    first, each kept only if, with the absences chosen so far, its copies fit
    the windows ``plan_actions`` would give it — the D2H (queued behind
    earlier ones on its stream) done before the first op that needs its
    bytes, the H2D done before its in access — at ``margin`` x the measured
    link rates on the traced op times.  Stops once the load is within the
    limit; returns the selection or raises LimitUnreachable.  With
    ``stall_budget_us`` a candidate may also stall the compute stream (copy
    done after the op that waits for it) while the predicted stalls sum to
    at most that budget.
    """
    from .errors import LimitUnreachable
    t = np.asarray(profile.op_times_us, np.float64)
    loads = np.asarray(profile.load.loads, np.int64).copy()
    busy_out, busy_in = [], []  # (start, end) of accepted copies per stream
    chosen = []
    stall = 0.0

    def queue_end(busy, start, dur):
        # first start >= start that does not overlap an accepted copy
        for s0, e0 in sorted(busy):
            if start + dur <= s0:
                break
            if e0 > start:
                start = e0
        return start + dur

    for c in sorted(cands, key=order or (lambda c: (-c.size, c.var))):
        if loads.max() <= limit_bytes:
            break
        if c.spans_iterations or c.var not in slot_of:
            continue
        r1, r2 = int(c.out_index), int(c.in_index)
        over = np.nonzero(loads[r1 + 1:r2] > limit_bytes)[0]
        if over.size == 0:
            continue
        a = r1 + 1 + int(over[0])
        b = r1 + 1 + int(over[-1]) + 1
        while a < b and next_point(points[r1]) > points[a]:
            a += 1
        while b > a and next_point(points[b - 1]) > points[r2]:
            b -= 1
        if b <= a:
            continue
        d_out = c.size / (d2h_bytes_per_s * margin) * 1e6 + latency_us
        d_in = c.size / (h2d_bytes_per_s * margin) * 1e6 + latency_us
        out_start = t[r1 + 1]
        out_end = queue_end(busy_out, out_start, d_out)
        in_start = t[b] if b < len(t) else t[-1]
        in_end = queue_end(busy_in, in_start, d_in)
        st = max(0.0, out_end - t[a]) + max(0.0, in_end - t[r2])
        if st > 0 and stall + st > stall_budget_us:
            continue
        stall += st
        busy_out.append((out_end - d_out, out_end))
        busy_in.append((in_end - d_in, in_end))
        loads[a:b] -= c.size
        chosen.append(c)
    if loads.max() > limit_bytes:
        raise LimitUnreachable(limit_bytes, int(loads.max()))
    return chosen


SWAP_LEAD = 512  # swapped blocks start this far into their arc (see split_arcs)


def split_arcs(profile, actions) -> list[tuple]:
    """Pool arcs of the window-allocated variables, swapped ones split at
    their absence [a, b).  A swapped arc is SWAP_LEAD bytes longer and its
    block starts SWAP_LEAD bytes in: PyTorch keys live blocks by pointer, so
    a co-tenant placed at the arc's start never aliases the absent block
    (the allocator also refuses exact aliases and falls back)."""
    absent = {x.var: (x.a, x.b) for x in actions}
    arcs = []
    for v in profile.variables:
        if v.alloc_index is None or v.var.startswith(MARK_NAME):
            continue
        segs = list(v.segments)
        if v.var in absent:
            a, b = absent[v.var]
            out = []
            for lo, hi in segs:
                if hi <= a or lo >= b:
                    out.append((lo, hi))
                    continue
                if lo < a:
                    out.append((lo, a))
                if b < hi:
                    out.append((b, hi))
            segs = out
            arcs.append((v.var, v.size + SWAP_LEAD, v.alloc_index, tuple(segs), v.persistent))
            continue
        arcs.append((v.var, v.size, v.alloc_index, tuple(segs), v.persistent))
    return arcs


def served_offsets(arcs, plan_offsets: dict, actions) -> dict:
    """Block offset of every arc (swapped blocks sit SWAP_LEAD in)."""
    swapped = {x.var for x in actions}
    return {v: plan_offsets[v] + (SWAP_LEAD if v in swapped else 0) for v, *_ in arcs}


def window_slots(profile) -> dict[str, int]:
    """Var -> malloc ordinal for the window's real allocations."""
    vs = sorted((v.alloc_index, v.var) for v in profile.variables
                if v.alloc_index is not None and not v.var.startswith(MARK_NAME))
    return {name: k for k, (_a, name) in enumerate(vs)}


class SwapExecutor:
    """Issue the copies/waits of a set of SwapActions while an iteration runs.

    ``base`` = device address of the pool, ``offsets`` = var -> pool offset,
    ``n_ops`` = aten ops of one iteration.  Call ``begin()`` right after
    ``torchmem.begin_iteration()`` and ``end()`` when the iteration's ops are
    all issued.
    """

    def __init__(self, actions, base: int, offsets: dict, n_ops: int):
        import torch
        from torch.utils._python_dispatch import TorchDispatchMode
        self.actions = actions
        self.n_ops = n_ops
        self.compute = torch.cuda.current_stream()
        self.s_out = torch.cuda.Stream()
        self.s_in = torch.cuda.Stream()
        self.by_point: dict[int, list] = {}
        self.host = []
        self.dev = []
        self.off = []
        for i, x in enumerate(actions):
            n = x.size
            h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
            self.host.append(h)
            self.dev.append((base + offsets[x.var], n))
            self.off.append(int(offsets[x.var]))
            ev = {k: torch.cuda.Event() for k in ("out_src", "in_src")}
            # timed: the last iteration's copy durations (copy_stats)
            ev.update({k: torch.cuda.Event(enable_timing=True) for k in ("out_t0", "out_done", "in_t0", "in_done")})
            x._ev = ev
            for pt, fn in ((x.issue_out, self._issue_out), (x.wait_out, self._wait_out),
                           (x.issue_in, self._issue_in), (x.wait_in, self._wait_in)):
                self.by_point.setdefault(pt, []).append((fn, i))
        # order at one point: issue before wait (an issue_in and wait_out of
        # different variables may share a point)
        for pt in self.by_point:
            self.by_point[pt].sort(key=lambda t: 0 if t[0] in (self._issue_out, self._issue_in) else 1)
        self.k = 0
        self.bytes_out = 0
        self.bytes_in = 0
        ex = self

        class Mode(TorchDispatchMode):
            def __torch_dispatch__(self, func, types, args=(), kwargs=None):
                ex.k += 1
                ex._run(2 * ex.k)
                if _DEBUG:
                    ex._check(f"before op {ex.k} {func}")
                out = func(*args, **(kwargs or {}))
                if _DEBUG:
                    ex._check(f"after op {ex.k} {func}")
                ex._run(2 * ex.k + 1)
                return out
        self._mode = Mode()

    def _run(self, pt):
        lst = self.by_point.get(pt)
        if lst:
            for fn, i in lst:
                if _DEBUG:
                    self._check(f"before {fn.__name__} {i} at {pt}")
                fn(i)
                if _DEBUG:
                    self._check(f"after {fn.__name__} {i} at {pt}: {self.actions[i]} dev {self.dev[i]} "
                                f"host {self.host[i].data_ptr():#x}")

    def _check(self, what):
        from .torchmem import ctl
        import torch
        e = int(ctl().mp_alloc_peek_error())
        if e:
            raise RuntimeError(f"pending CUDA error {e} {what}")
        torch.cuda.synchronize()

    def _issue_out(self, i):
        x = self.actions[i]
        x._ev["out_src"].record(self.compute)
        self.s_out.wait_event(x._ev["out_src"])
        x._ev["out_t0"].record(self.s_out)
        _copy(self.host[i], self.dev[i], d2h=True, stream=self.s_out)
        x._ev["out_done"].record(self.s_out)
        self.bytes_out += x.size

    def _wait_out(self, i):
        from .torchmem import ctl
        self.compute.wait_event(self.actions[i]._ev["out_done"])
        ctl().mp_alloc_pool_release(C.c_int64(self.off[i]))

    def _issue_in(self, i):
        from .torchmem import ctl
        x = self.actions[i]
        if ctl().mp_alloc_pool_reclaim(C.c_int64(self.off[i]), C.c_int64(x.size)):
            raise RuntimeError(f"swap-in of {x.var}: its pool bytes are still held by a live block "
                               "(the run's lifetimes drifted from the plan)")
        x._ev["in_src"].record(self.compute)
        self.s_in.wait_event(x._ev["in_src"])
        x._ev["in_t0"].record(self.s_in)
        _copy(self.host[i], self.dev[i], d2h=False, stream=self.s_in)
        x._ev["in_done"].record(self.s_in)
        self.bytes_in += x.size

    def _wait_in(self, i):
        self.compute.wait_event(self.actions[i]._ev["in_done"])

    def copy_stats(self) -> dict:
        """Bytes and copy-stream busy time of the LAST iteration's copies
        (call after a synchronize): the achieved host-link rate of the
        executed plan, per direction."""
        out = {}
        for d, (t0, t1) in (("d2h", ("out_t0", "out_done")), ("h2d", ("in_t0", "in_done"))):
            ms = sum(x._ev[t0].elapsed_time(x._ev[t1]) for x in self.actions)
            nb = sum(x.size for x in self.actions)
            out[d] = {"bytes": int(nb), "busy_ms": ms, "bytes_per_s": nb / (ms * 1e-3) if ms > 0 else None}
        return out

    def begin(self):
        self.k = 0
        self._run(0)
        self._run(1)
        self._mode.__enter__()

    def end(self):
        self._mode.__exit__(None, None, None)
        for pt in sorted(p for p in self.by_point if p > 2 * self.k + 1):
            self._run(pt)
        if self.k != self.n_ops:
            raise RuntimeError(f"iteration ran {self.k} ops, the plan was made for {self.n_ops}")


def _copy(host, dev, d2h: bool, stream) -> None:
    """Stream-ordered copy between a pinned host tensor and a raw pool range
    (the pool bytes belong to no tensor while the variable is absent)."""
    import ctypes as C
    from .torchmem import ctl
    ptr, n = dev
    rc = ctl().mp_alloc_copy_async(C.c_void_p(ptr), C.c_void_p(host.data_ptr()), C.c_int64(n), C.c_int(1 if d2h else 0),
                                   C.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"cudaMemcpyAsync failed ({rc})")
