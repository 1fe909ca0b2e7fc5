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
from .trace import TraceArrays

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
                offsets_out: np.ndarray | None = None, keep_on_device: bool = False) -> ArrayPlan:
    """Plan a static pool for the iteration window of ``arrays``.

    ``offsets_out`` (e.g. a pinned buffer) receives the offsets; with
    ``keep_on_device`` they stay in HBM (``ArrayPlan.offsets`` is None).
    """
    if policy not in POLICY_CODE:
        raise ValueError(f"unknown policy {policy!r}")
    dev = N.device_trace(arrays)
    N.lib().mp_trace_reset(dev.h)
    if validate:
        N.validate(arrays)
    if window is None:
        p = N.detect(arrays)
        window = (len(arrays) - p, len(arrays))
    dp = N.extract(arrays, window[0], window[1])
    dims = dp.dims()
    g = N.conflict_from_profile(dp)
    nv, nnz = N.graph_dims(g)
    if keep_on_device:
        fp, lv = N.plan_pool_device(g, POLICY_CODE[policy])
        offs = None
    else:
        offs, fp, lv = N.plan_pool(g, POLICY_CODE[policy], nv, out=offsets_out)
    return ArrayPlan(period=int(dims.period), window=tuple(window), nvars=int(dims.nvars),
                     peak_bytes=int(dims.peak_bytes), peak_index=int(dims.peak_index),
                     footprint_bytes=fp, offsets=offs, levels=lv, nnz=nnz)
