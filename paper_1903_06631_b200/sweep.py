"""Batched planning sweep over many independent traces (BASELINE configs[4]).

A sweep unit is what the reference's estimators run for one trace
(pkg/src/memplan/estimators.py:20-130): ``IterationAnalyzer`` (validate,
detect, extract), ``PoolPlanner`` (conflict graph + ``plan_pool``) and, for
every swap budget, ``SwapPlanner(limit_bytes, score="swdoa").fit`` (the
limit checks, ``select_by_swdoa``, ``build_schedule``, ``simulate``).  The
device runs a whole batch in one launch, one CTA per trace (csrc/sweep.cu);
budgets are fractions of each trace's own peak, ``limit = int(peak * frac)``.

Results come back as numpy structured arrays whose fields mirror
``mp_sweep_trace`` / ``mp_sweep_budget`` (include/memplan_b200.h); status
codes map to the reference's exceptions through ``_abi.raise_for``.

Multi-GPU: traces are independent, so ``shard`` splits a batch across ranks
(longest-processing-time on event counts) with no collective on the data
path; results are gathered on the host at the end.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as N
from ._abi import MP_OK, MpErr, ptr, raise_for
from .trace import TraceArrays, as_arrays

MIB = 1 << 20
MAX_BUDGETS = 8
POLICY_CODE = {"first_fit": 0, "best_fit": 1}

TRACE_DTYPE = np.dtype([
    ("status", np.int32), ("err_code", np.int32), ("err_index", np.int64),
    ("period", np.int64), ("nvars", np.int64), ("ncarry", np.int64), ("naccess", np.int64),
    ("peak_bytes", np.int64), ("peak_index", np.int64), ("duration_us", np.float64),
    ("footprint_bytes", np.int64), ("edges", np.int64), ("ncand", np.int64), ("load_min", np.int64),
    ("norder", np.int64),
], align=True)

BUDGET_DTYPE = np.dtype([
    ("limit_bytes", np.int64), ("status", np.int32), ("rounds", np.int32),
    ("nsel", np.int64), ("selected_bytes", np.int64), ("err_index", np.int64), ("err_aux", np.int64),
    ("overhead_us", np.float64), ("achieved_peak_bytes", np.int64), ("planned_peak_bytes", np.int64),
], align=True)


class MpSweepParams(C.Structure):
    _fields_ = [("policy", C.c_int32), ("nbudget", C.c_int32), ("max_rounds", C.c_int32),
                ("validate", C.c_int32), ("threshold", C.c_int64), ("bw", C.c_double),
                ("lat", C.c_double), ("budget_frac", C.c_double * MAX_BUDGETS)]


class MpSweepIn(C.Structure):
    _fields_ = [("ntraces", C.c_int64)] + [(n, C.c_void_p) for n in (
        "ev_off", "kind", "var", "size", "t_us", "var_off", "name_blob", "name_off")]


assert TRACE_DTYPE.itemsize == 112 and BUDGET_DTYPE.itemsize == 72


@dataclass
class SweepParams:
    """SwapPlanner / PoolPlanner settings shared by every unit of a sweep
    (defaults as estimators.py:41-80 and swapsim.py:350)."""
    budgets: Sequence[float] = (0.9, 0.8, 0.7, 0.6)
    policy: str = "best_fit"
    threshold_bytes: int = MIB
    bandwidth_bytes_per_s: float = 12e9
    latency_us: float = 10.0
    max_rounds: int = 100
    validate: bool = True

    def struct(self) -> MpSweepParams:
        if self.policy not in POLICY_CODE:
            raise ValueError(f"unknown policy {self.policy!r}")
        if len(self.budgets) > MAX_BUDGETS:
            raise ValueError(f"at most {MAX_BUDGETS} budgets per sweep")
        fr = (C.c_double * MAX_BUDGETS)(*[float(b) for b in self.budgets])
        return MpSweepParams(POLICY_CODE[self.policy], len(self.budgets), int(self.max_rounds),
                             1 if self.validate else 0, int(self.threshold_bytes),
                             float(self.bandwidth_bytes_per_s), float(self.latency_us), fr)


class SweepBatch:
    """Traces concatenated column-wise (host numpy); trace t's events are
    rows ev_off[t]:ev_off[t+1], its names ids var_off[t]:var_off[t+1]."""

    COLUMNS = ("kind", "var", "size", "t_us", "ev_off", "var_off", "name_blob", "name_off")

    def copy_to(self, alloc) -> "SweepBatch":
        """The same batch in buffers from ``alloc(nbytes) -> uint8 array`` (e.g.
        pinned host memory, so uploads are asynchronous DMA)."""
        cols = {}
        for c in self.COLUMNS:
            a = getattr(self, c)
            buf = alloc(max(a.nbytes, 1)).view(a.dtype)[:a.size]
            buf[...] = a
            cols[c] = buf
        return SweepBatch(**cols)

    def __init__(self, kind, var, size, t_us, ev_off, var_off, name_blob, name_off):
        self.kind = np.ascontiguousarray(kind, np.uint8)
        self.var = np.ascontiguousarray(var, np.int32)
        self.size = np.ascontiguousarray(size, np.int64)
        self.t_us = np.ascontiguousarray(t_us, np.int64)
        self.ev_off = np.ascontiguousarray(ev_off, np.int64)
        self.var_off = np.ascontiguousarray(var_off, np.int64)
        self.name_blob = np.ascontiguousarray(name_blob, np.uint8)
        self.name_off = np.ascontiguousarray(name_off, np.int64)
        if self.name_blob.size == 0:
            self.name_blob = np.zeros(1, np.uint8)

    @classmethod
    def from_traces(cls, traces: Sequence) -> "SweepBatch":
        arrs = [as_arrays(t) for t in traces]
        for i, a in enumerate(arrs):
            if a.index is not None:
                raise ValueError(f"trace {i}: event indices must equal positions in a sweep")
        T = len(arrs)
        ev_off = np.zeros(T + 1, np.int64)
        var_off = np.zeros(T + 1, np.int64)
        if T:
            ev_off[1:] = np.cumsum([len(a) for a in arrs])
            var_off[1:] = np.cumsum([a.nvars for a in arrs])
        cat = (lambda xs, dt: np.concatenate(xs).astype(dt, copy=False) if xs else np.zeros(0, dt))
        blob_parts, off_parts, base = [], [np.zeros(1, np.int64)], 0
        for a in arrs:
            nb = int(a.name_off[-1])
            blob_parts.append(a.name_blob[:nb])
            off_parts.append(a.name_off[1:] + base)
            base += nb
        return cls(cat([a.kind for a in arrs], np.uint8), cat([a.var for a in arrs], np.int32),
                   cat([a.size for a in arrs], np.int64), cat([a.t_us for a in arrs], np.int64),
                   ev_off, var_off, cat(blob_parts, np.uint8), np.concatenate(off_parts))

    @property
    def ntraces(self) -> int:
        return int(self.ev_off.shape[0] - 1)

    def __len__(self) -> int:
        return self.ntraces

    def events_of(self, t: int) -> int:
        return int(self.ev_off[t + 1] - self.ev_off[t])

    def trace(self, t: int) -> TraceArrays:
        """Trace t as its own TraceArrays (names re-derived from the blob)."""
        e0, e1 = int(self.ev_off[t]), int(self.ev_off[t + 1])
        v0, v1 = int(self.var_off[t]), int(self.var_off[t + 1])
        offs = self.name_off[v0:v1 + 1]
        blob = self.name_blob.tobytes()
        names = [blob[int(offs[i]):int(offs[i + 1])].decode("utf-8") for i in range(v1 - v0)]
        return TraceArrays(self.kind[e0:e1], self.var[e0:e1], self.size[e0:e1], self.t_us[e0:e1], names)

    def subset(self, idx: Sequence[int]) -> "SweepBatch":
        return SweepBatch.from_traces([self.trace(int(i)) for i in idx])

    def sweep_in(self) -> MpSweepIn:
        return MpSweepIn(self.ntraces, ptr(self.ev_off), ptr(self.kind), ptr(self.var), ptr(self.size),
                         ptr(self.t_us), ptr(self.var_off), ptr(self.name_blob), ptr(self.name_off))

    @property
    def nbytes(self) -> int:
        return sum(getattr(self, c).nbytes for c in ("kind", "var", "size", "t_us", "ev_off", "var_off",
                                                     "name_blob", "name_off"))


@dataclass
class SweepResult:
    traces: np.ndarray          # TRACE_DTYPE[T]
    budgets: np.ndarray         # BUDGET_DTYPE[T, B]
    offsets: np.ndarray         # int64[N]: trace t's plan at ev_off[t] (profile variable order)
    cand_order: np.ndarray      # int32[N]: trace t's SWDOA greedy picks (profile variable indices)
    ev_off: np.ndarray
    params: SweepParams = field(default_factory=SweepParams)
    batch: "SweepBatch | None" = None

    def records_only(self) -> "SweepResult":
        """The records without the input batch (what a rank sends in a gather)."""
        return SweepResult(self.traces, self.budgets, self.offsets, self.cand_order, self.ev_off, self.params, None)

    def offsets_of(self, t: int) -> np.ndarray:
        e0 = int(self.ev_off[t])
        return self.offsets[e0:e0 + int(self.traces["nvars"][t])]

    def order_of(self, t: int) -> np.ndarray:
        """The SWDOA greedy picks the budgets needed (a prefix of the full order)."""
        e0 = int(self.ev_off[t])
        return self.cand_order[e0:e0 + int(self.traces["norder"][t])]

    def selection_of(self, t: int, b: int) -> np.ndarray:
        return self.order_of(t)[:int(self.budgets["nsel"][t, b])]

    def overhead_pct(self) -> np.ndarray:
        d = self.traces["duration_us"][:, None]
        with np.errstate(divide="ignore", invalid="ignore"):
            return np.where(d > 0, self.budgets["overhead_us"] / d * 100.0, 0.0)

    @property
    def planned_vars(self) -> int:
        ok = self.traces["status"] == MP_OK
        return int(self.traces["nvars"][ok].sum())

    def raise_for(self, t: int, b: int | None = None) -> None:
        """Re-raise trace t's (or budget b's) failure as the reference exception."""
        rec = self.traces[t] if b is None else self.budgets[t, b]
        code = int(rec["status"])
        if code == MP_OK:
            return
        err = MpErr()
        err.code = code
        err.index = int(rec["err_index"])
        names = None
        if b is None:
            err.aux0 = int(rec["err_code"])
            if code == 1 and self.batch is not None:
                # the offending event: absolute for validate_trace, window-relative
                # for extract_lifetimes (codes >= 9)
                e0 = int(self.batch.ev_off[t])
                pos = err.index + (self.batch.events_of(t) - int(rec["period"]) if err.aux0 >= 9 else 0)
                err.aux1 = int(self.batch.kind[e0 + pos]) if err.aux0 == 6 else int(self.batch.var[e0 + pos])
                names = self.batch.trace(t).names
        else:
            err.aux0 = int(rec["limit_bytes"])
            err.aux1 = int(rec["err_aux"])
        raise_for(code, err, names)


def _lib():
    L = N.lib()
    for name in ("mp_sweep_upload", "mp_sweep_run", "mp_sweep_download", "mp_sweep_free"):
        getattr(L, name).restype = C.c_int
    return L


class DeviceSweep:
    """A batch resident in HBM: upload once, run many times (bench's
    resident leg), download the records."""

    def __init__(self, batch: SweepBatch):
        self.batch = batch
        self._h = C.c_void_p()
        err = MpErr()
        sin = batch.sweep_in()
        rc = _lib().mp_sweep_upload(N.ctx(), C.byref(sin), C.byref(self._h), C.byref(err))
        raise_for(rc, err)
        self.params: SweepParams | None = None

    def run(self, params: SweepParams) -> None:
        err = MpErr()
        prm = params.struct()
        rc = _lib().mp_sweep_run(N.ctx(), self._h, C.byref(prm), C.byref(err))
        raise_for(rc, err)
        self.params = params

    def download(self, traces=None, budgets=None, offsets=None, cand_order=None) -> SweepResult:
        b = self.batch
        T, Nev = b.ntraces, int(b.ev_off[-1])
        nb = len(self.params.budgets) if self.params else 0
        traces = np.zeros(T, TRACE_DTYPE) if traces is None else traces
        budgets = np.zeros((T, nb), BUDGET_DTYPE) if budgets is None else budgets
        offsets = np.zeros(max(Nev, 1), np.int64) if offsets is None else offsets
        cand_order = np.zeros(max(Nev, 1), np.int32) if cand_order is None else cand_order
        err = MpErr()
        rc = _lib().mp_sweep_download(N.ctx(), self._h, ptr(traces), ptr(budgets) if nb else None,
                                      ptr(offsets), ptr(cand_order), C.byref(err))
        raise_for(rc, err)
        return SweepResult(traces, budgets, offsets[:Nev], cand_order[:Nev], b.ev_off, self.params, b)

    def set_profile(self, on: bool = True) -> None:
        """Diagnostics: record clock64() at the kernel's 8 phase marks."""
        L = _lib()
        L.mp_sweep_set_profile.restype = C.c_int
        err = MpErr()
        raise_for(L.mp_sweep_set_profile(N.ctx(), self._h, C.c_int(1 if on else 0), C.byref(err)), err)

    def profile(self) -> np.ndarray:
        """[ntraces, 7] SM cycles spent per phase: group/validate/detect,
        extract, plan, candidates, greedy, simulate prep, budgets."""
        L = _lib()
        L.mp_sweep_profile_download.restype = C.c_int
        out = np.zeros((max(self.batch.ntraces, 1), 16), np.int64)
        err = MpErr()
        raise_for(L.mp_sweep_profile_download(N.ctx(), self._h, ptr(out), C.byref(err)), err)
        self.profile_extra = out[:self.batch.ntraces, 8:]
        self.profile_raw = out[:self.batch.ntraces]
        return np.diff(out[:self.batch.ntraces, :8], axis=1)

    def close(self):
        if self._h:
            _lib().mp_sweep_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def run_sweep(traces, params: SweepParams | None = None, out: SweepResult | None = None) -> SweepResult:
    """Plan every trace of a batch (a SweepBatch or a list of traces) on the
    device: upload, one sweep launch, download.  ``out`` (e.g. pinned
    buffers from ``SweepResult.empty_like``) receives the records."""
    batch = traces if isinstance(traces, SweepBatch) else SweepBatch.from_traces(traces)
    params = params or SweepParams()
    ds = DeviceSweep(batch)
    try:
        ds.run(params)
        if out is None:
            return ds.download()
        return ds.download(out.traces, out.budgets, out.offsets, out.cand_order)
    finally:
        ds.close()


def shard(costs: Sequence[float], world: int) -> list[list[int]]:
    """Longest-processing-time partition of units over `world` ranks:
    units by descending cost, each to the currently lightest rank (ties to
    the lower rank) — deterministic, so every rank computes the same split."""
    load = [0.0] * world
    parts: list[list[int]] = [[] for _ in range(world)]
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    for i in order:
        r = min(range(world), key=lambda q: (load[q], q))
        parts[r].append(i)
        load[r] += float(costs[i])
    return [sorted(p) for p in parts]


def concat_results(parts: Sequence[tuple[Sequence[int], SweepResult]], batch: SweepBatch) -> SweepResult:
    """Reassemble per-shard results (shard trace indices, result) into one
    result in the batch's trace order."""
    T, Nev = batch.ntraces, int(batch.ev_off[-1])
    params = next((r.params for _, r in parts if r is not None), SweepParams())
    nb = len(params.budgets)
    traces = np.zeros(T, TRACE_DTYPE)
    budgets = np.zeros((T, nb), BUDGET_DTYPE)
    offsets = np.zeros(max(Nev, 1), np.int64)
    cand_order = np.zeros(max(Nev, 1), np.int32)
    for idx, res in parts:
        for q, t in enumerate(idx):
            traces[t] = res.traces[q]
            budgets[t] = res.budgets[q]
            e0, n = int(batch.ev_off[t]), batch.events_of(t)
            s0 = int(res.ev_off[q])
            offsets[e0:e0 + n] = res.offsets[s0:s0 + n]
            cand_order[e0:e0 + n] = res.cand_order[s0:s0 + n]
    return SweepResult(traces, budgets, offsets[:Nev], cand_order[:Nev], batch.ev_off, params, batch)


def run_sweep_sharded(batch: SweepBatch, params: SweepParams | None = None, rank: int = 0, world: int = 1,
                      runner=None, group=None) -> SweepResult | None:
    """One rank's share of a sweep, then a gather on rank 0.

    Units are partitioned by ``shard`` on event counts (every rank computes
    the same split), each rank plans its own traces on its own device with
    no collective on the data path, and the fixed-size records are gathered
    to rank 0 with ``torch.distributed.gather_object`` once at the end.
    Returns the whole batch's result on rank 0 and None elsewhere.
    """
    params = params or SweepParams()
    runner = runner or run_sweep
    parts = shard([batch.events_of(t) for t in range(batch.ntraces)], world)
    mine = parts[rank]
    res = runner(batch.subset(mine), params) if mine else None
    if world == 1:
        return concat_results([(mine, res)], batch)
    import torch.distributed as dist
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((mine, res.records_only() if res is not None else None), gathered, dst=0, group=group)
    if rank != 0:
        return None
    return concat_results([g for g in gathered if g[1] is not None], batch)
