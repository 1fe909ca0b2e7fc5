"""Array-native entry points: the whole pool-planning path in one call.

``plan_arrays`` is what ``PoolPlanner.fit`` does (estimators.py:49-58 of
the reference) without Python object materialization: the columnar trace
goes to the device, validate -> detect_iteration -> extract_lifetimes ->
build_conflict_graph -> plan_pool run there, and only the offsets come
back.  It is the call a batch pipeline (or bench.py's e2e leg) makes.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import MemplanError
from .trace import TraceArrays

# traces up to this many events are planned by one CTA (csrc/sweep.cu) — a
# single launch instead of the grid-wide stages' ~50 launches and host
# round trips (ResNet-50 b32: 0.43 ms vs 4.7 ms)
CTA_PATH_MAX_EVENTS = 1 << 15

POLICY_CODE = {"first_fit": 0, "best_fit": 1}


@dataclass
class ArrayPlan:
    period: int
    window: tuple[int, int]
    nvars: int
    peak_bytes: int
    peak_index: int
    footprint_bytes: int
    offsets: np.ndarray | None  # int64[nvars], profile variable order
    levels: int                 # wavefront depth of the placement DAG
    nnz: int                    # CSR entries of the conflict graph

    @property
    def competitive_ratio(self) -> float:
        return 1.0 if self.peak_bytes <= 0 else self.footprint_bytes / self.peak_bytes


def plan_arrays(arrays: TraceArrays, window: tuple[int, int] | None = None,
                policy: str = "best_fit", validate: bool = True,
                offsets_out: np.ndarray | None = None, keep_on_device: bool = False,
                path: str = "auto") -> ArrayPlan:
    """Plan a static pool for the iteration window of ``arrays``.

    ``offsets_out`` (e.g. a pinned buffer) receives the offsets; with
    ``keep_on_device`` they stay in HBM (``ArrayPlan.offsets`` is None).
    ``path``: "grid" (the grid-wide stages), "cta" (one CTA, detected window
    only) or "auto" (cta for small traces).  Both are bit-identical.
    """
    if policy not in POLICY_CODE:
        raise ValueError(f"unknown policy {policy!r}")
    if path not in ("auto", "grid", "cta"):
        raise ValueError(f"unknown path {path!r}")
    small = window is None and arrays.index is None and not keep_on_device
    if path == "cta" or (path == "auto" and small and len(arrays) <= CTA_PATH_MAX_EVENTS):
        if not small:
            raise ValueError("the one-CTA path plans the detected window of an indexed, host-side plan")
        return _plan_cta(arrays, policy, validate, offsets_out)
    # The upload is asynchronous, column by column (var, kind, size, then
    # the rest): grouping and period detection run while the later columns
    # are still in flight.  Validation still decides first: a detection
    # failure on an invalid trace reports the invariant violation, as the
    # reference (validate -> detect -> extract) would.
    # The timestamps (needed only for op times and their own checks) arrive
    # last: structure is validated before extraction, timestamps after the
    # plan, and any failure in between defers to the timestamp check first.
    fresh = getattr(arrays, "_dev", None) is None
    dev = N.device_trace(arrays, asynchronous=True)
    try:
        N.lib().mp_trace_reset(dev.h)
        if window is None and validate:
            # validation and period detection share one readback; a violation
            # wins, and without a period the full validation decides first
            p = N.detect_validate(arrays, "structure" if fresh else "all")
            window = (len(arrays) - p, len(arrays))
        else:
            if window is None:
                try:
                    p = N.detect(arrays)
                except (MemplanError, ValueError):
                    if validate:
                        N.validate(arrays)
                    raise
                window = (len(arrays) - p, len(arrays))
            if validate:
                # a resident trace has every column: one pass, one readback
                N.validate(arrays, "structure" if fresh else "all")
        try:
            dp = N.extract(arrays, window[0], window[1])
            g = N.conflict_from_profile(dp)
            nv, nnz = N.graph_dims(g)
            if fresh:
                # the timestamps go up during the placement (see mp_trace_flush)
                N.trace_flush(dev)
            if keep_on_device:
                fp, lv = N.plan_pool_device(g, POLICY_CODE[policy])
                offs = None
            else:
                offs, fp, lv = N.plan_pool(g, POLICY_CODE[policy], nv, out=offsets_out)
        except (MemplanError, ValueError):
            if validate and fresh:
                N.validate(arrays, "times")
            raise
        if validate and fresh:
            N.validate(arrays, "times")
        dims = dp.dims()
    finally:
        if fresh:
            N.trace_wait(dev)  # the host arrays are the caller's again
    return ArrayPlan(period=int(dims.period), window=tuple(window), nvars=int(dims.nvars),
                     peak_bytes=int(dims.peak_bytes), peak_index=int(dims.peak_index),
                     footprint_bytes=fp, offsets=offs, levels=lv, nnz=nnz)


def _plan_cta(arrays: TraceArrays, policy: str, validate: bool, offsets_out) -> ArrayPlan:
    from . import sweep
    batch = sweep.SweepBatch.from_traces([arrays])
    res = sweep.run_sweep(batch, sweep.SweepParams(budgets=(), policy=policy, validate=validate))
    res.raise_for(0)
    r = res.traces[0]
    offs = res.offsets_of(0)
    if offsets_out is not None:
        offsets_out[:offs.shape[0]] = offs
        offs = offsets_out[:offs.shape[0]]
    n, p = len(arrays), int(r["period"])
    return ArrayPlan(period=p, window=(n - p, n), nvars=int(r["nvars"]), peak_bytes=int(r["peak_bytes"]),
                     peak_index=int(r["peak_index"]), footprint_bytes=int(r["footprint_bytes"]),
                     offsets=offs.copy() if offsets_out is None else offs, levels=-1, nnz=2 * int(r["edges"]))
