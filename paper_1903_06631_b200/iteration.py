"""Iteration detection and lifetime extraction (drop-in for memplan.iteration).

Same dataclasses and functions as the reference (pkg/src/memplan/
iteration.py:21-353).  ``detect_iteration`` and ``extract_lifetimes`` run
on the device (csrc/ingest.cu); the resulting ``IterationProfile`` keeps the
device-resident profile and materializes the reference's Python objects
(variables, accesses, loads, op_instance) only when they are read.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._abi import F_PERSISTENT, F_RENAMED, F_WRAPS, FlatProfile, MpProfileDims
from .errors import MemplanError
from .trace import KIND_BY_CODE, EventKind, Trace, TraceArrays, TraceEvent, as_arrays

Segment = tuple[int, int]


@dataclass(frozen=True)
class Access:
    index: int
    t_us: float
    kind: EventKind
    next_iteration: bool = False


@dataclass
class VariableLifetime:
    var: str
    base_var: str
    size: int
    alloc_index: int | None
    free_index: int | None
    segments: tuple[Segment, ...]
    accesses: list[Access]
    persistent: bool
    wraps: bool

    def covers(self, index: int) -> bool:
        return any(lo <= index < hi for lo, hi in self.segments)


@dataclass
class LoadProfile:
    loads: list[int]
    peak_bytes: int
    peak_index: int

    @property
    def samples(self) -> list[tuple[int, int]]:
        return list(enumerate(self.loads))


@dataclass
class DetectedIteration:
    period: int
    window: tuple[int, int]


_LAZY = ("variables", "load", "op_times_us", "events", "op_instance")
# the fields a device profile is built from (``events`` is not uploaded)
_DEVICE_FIELDS = ("variables", "load", "op_times_us", "op_instance")
_SCALARS = ("period", "window", "period_duration_us")


def _freeze(name, value):
    """Value snapshot of a profile field, for in-place edit detection."""
    if value is None:
        return None
    if name == "variables":
        return tuple((v.var, v.base_var, v.size, v.alloc_index, v.free_index, tuple(v.segments),
                      tuple(v.accesses), v.persistent, v.wraps) for v in value)
    if name == "load":
        return (tuple(value.loads), value.peak_bytes, value.peak_index)
    return tuple(value)


class IterationProfile:
    """One iteration window's lifetimes (iteration.py:63-90).

    Constructed either by the user (plain fields, like the reference
    dataclass) or from a device profile; in the latter case the list-valued
    fields are built on first access from the downloaded columns.
    """

    def __init__(self, period: int, window: tuple[int, int], variables: list[VariableLifetime] | None = None,
                 load: LoadProfile | None = None, op_times_us: list[float] | None = None,
                 period_duration_us: float = 0.0, events: list[TraceEvent] | None = None,
                 op_instance: list[str] | None = None):
        self.period = period
        self.window = window
        self.period_duration_us = period_duration_us
        self.__dict__["variables"] = variables
        self.__dict__["load"] = load
        self.__dict__["op_times_us"] = op_times_us
        self.__dict__["events"] = events if events is not None else []
        self.__dict__["op_instance"] = op_instance if op_instance is not None else []
        self._dev = None        # DProfile (device) when this profile came from / went to the device
        self._flat = None       # FlatProfile columns
        self._arrays = None     # TraceArrays the profile was extracted from
        self._trace_events = None
        self._pending = ()      # lazily materialized fields

    # -- construction from the device ------------------------------------
    @classmethod
    def _from_device(cls, dp, arrays: TraceArrays, window, trace_events=None) -> "IterationProfile":
        dims = dp.dims()
        prof = cls(int(dims.period), tuple(window), period_duration_us=float(dims.duration_us))
        prof._dev = dp
        prof._arrays = arrays
        prof._trace_events = trace_events
        prof._pending = _LAZY
        for name in _LAZY:
            del prof.__dict__[name]
        prof._dims = dims
        return prof

    def _flat_profile(self) -> FlatProfile:
        if self._flat is None:
            if self._dev is not None and self._arrays is not None:
                a = self._arrays
                self._flat = N.download_profile(self._dev, a.names, a.name_blob, a.name_off, self.window)
            else:
                self._flat = _flatten(self)
        return self._flat

    def __getattr__(self, name):
        # only reached for lazily-built fields
        if name in _LAZY and name in self.__dict__.get("_pending", ()):
            value = self._materialize(name)
            self.__dict__[name] = value
            if name in _DEVICE_FIELDS:
                # the device copy stays valid while this value is unedited
                self.__dict__.setdefault("_sig", {})[name] = _freeze(name, value)
            return value
        raise AttributeError(name)

    def _materialize_all(self, skip=None) -> None:
        """Build every still-lazy field (but ``skip``) from the current
        device columns."""
        for name in self.__dict__.get("_pending", ()):
            if name != skip and name not in self.__dict__:
                getattr(self, name)

    def _drop_device(self, skip=None) -> None:
        d = self.__dict__
        if d.get("_dev") is not None or d.get("_flat") is not None:
            self._materialize_all(skip)
        d["_dev"] = None
        d["_flat"] = None
        d["_sig"] = {}

    def __setattr__(self, name, value):
        if name in _LAZY or (name in _SCALARS and self.__dict__.get("_dev") is not None):
            # a user edit invalidates the device copy (the other lazy
            # fields are built from it first)
            self._drop_device(skip=name)
            self.__dict__[name] = value
            return
        object.__setattr__(self, name, value)

    def _device_stale(self) -> bool:
        """True when a field the device copy was built from has been edited
        in place since (the reference reads the fields on every call)."""
        sig = self.__dict__.get("_sig") or {}
        return any(name in self.__dict__ and _freeze(name, self.__dict__[name]) != frozen
                   for name, frozen in sig.items())

    def _materialize(self, name):
        fp = self._flat_profile()
        if name == "op_times_us":
            return fp.op_times.tolist()
        if name == "load":
            return LoadProfile(loads=fp.loads.tolist(), peak_bytes=fp.peak_bytes, peak_index=fp.peak_index)
        if name == "op_instance":
            names = fp.var_names()
            return [names[o] for o in fp.op_owner.tolist()]
        if name == "events":
            if self._trace_events is not None:
                return self._trace_events[self.window[0]:self.window[1]]
            a = self._arrays
            s, e = self.window
            return [TraceEvent(i, int(t), KIND_BY_CODE[int(k)], a.names[int(v)], int(sz))
                    for i, k, v, sz, t in zip(range(s, e), a.kind[s:e].tolist(), a.var[s:e].tolist(),
                                              a.size[s:e].tolist(), a.t_us[s:e].tolist())]
        if name == "variables":
            return _variables_from_flat(fp)
        raise AttributeError(name)

    # -- reference methods ---------------------------------------------------
    def op_end_us(self, r: int) -> float:
        if r + 1 < self.period:
            return self.op_times_us[r + 1]
        return self.period_duration_us

    def lifetime(self, var: str) -> VariableLifetime:
        for v in self.variables:
            if v.var == var:
                return v
        raise KeyError(var)

    @property
    def alloc_instance(self) -> dict[int, str]:
        return {v.alloc_index: v.var for v in self.variables if v.alloc_index is not None}

    def __repr__(self):
        return (f"IterationProfile(period={self.period}, window={self.window}, "
                f"nvars={self.nvars}, peak={self.peak_bytes})")

    def __eq__(self, other):
        if not isinstance(other, IterationProfile):
            return NotImplemented
        return all(getattr(self, f) == getattr(other, f) for f in (
            "period", "window", "variables", "load", "op_times_us", "period_duration_us", "events",
            "op_instance"))

    # -- cheap summaries that avoid materialization -------------------------
    @property
    def nvars(self) -> int:
        if "variables" in self.__dict__ and self.__dict__["variables"] is not None:
            return len(self.__dict__["variables"])
        return int(self._dims.nvars) if self._dev is not None else 0

    @property
    def peak_bytes(self) -> int:
        if "load" in self.__dict__:
            return self.__dict__["load"].peak_bytes
        return int(self._dims.peak_bytes)


def _variables_from_flat(fp: FlatProfile) -> list[VariableLifetime]:
    names = fp.var_names()
    base = [fp.names[b] for b in fp.base.tolist()]
    times = fp.op_times
    ao = fp.acc_off.tolist()
    ai, ak, an = fp.acc_index.tolist(), fp.acc_kind.tolist(), fp.acc_next.tolist()
    seg = fp.seg.tolist()
    out = []
    for i in range(fp.nvars):
        accs = [Access(ai[a], float(times[ai[a]]), KIND_BY_CODE[ak[a]], bool(an[a])) for a in range(ao[i], ao[i + 1])]
        ns = int(fp.nseg[i])
        segs = tuple((seg[4 * i + 2 * s], seg[4 * i + 2 * s + 1]) for s in range(ns))
        al, fr, fl = int(fp.alloc[i]), int(fp.free_[i]), int(fp.flags[i])
        out.append(VariableLifetime(var=names[i], base_var=base[i], size=int(fp.size[i]),
                                    alloc_index=None if al < 0 else al, free_index=None if fr < 0 else fr,
                                    segments=segs, accesses=accs, persistent=bool(fl & F_PERSISTENT),
                                    wraps=bool(fl & F_WRAPS)))
    return out


def _flatten(profile: IterationProfile) -> FlatProfile:
    """Columnar form of a Python-built profile (names interned; no renames)."""
    variables = profile.variables or []
    names = sorted({v.var for v in variables} | set(profile.op_instance or []))
    rank = {n: i for i, n in enumerate(names)}
    V, p = len(variables), profile.period
    nseg = np.array([len(v.segments) for v in variables] or [0], np.int32)[:V]
    if V and nseg.max() > 2:
        raise MemplanError("device profiles hold at most two segments per variable")
    seg = np.zeros(4 * V, np.int32)
    for i, v in enumerate(variables):
        for s, (lo, hi) in enumerate(v.segments):
            seg[4 * i + 2 * s], seg[4 * i + 2 * s + 1] = lo, hi
    acc_off = np.zeros(V + 1, np.int64)
    acc_off[1:] = np.cumsum([len(v.accesses) for v in variables]) if V else []
    accs = [a for v in variables for a in v.accesses]
    code = {k: i for i, k in enumerate(KIND_BY_CODE)}
    loads = profile.load
    op_owner = [rank.get(n, 0) for n in (profile.op_instance or [])]
    arrays = {
        "base": np.array([rank[v.var] for v in variables], np.int32),
        "size": np.array([v.size for v in variables], np.int64),
        "alloc": np.array([-1 if v.alloc_index is None else v.alloc_index for v in variables], np.int32),
        "free_": np.array([-1 if v.free_index is None else v.free_index for v in variables], np.int32),
        "nseg": nseg.astype(np.int32), "seg": seg,
        "flags": np.array([(F_PERSISTENT if v.persistent else 0) | (F_WRAPS if v.wraps else 0)
                           for v in variables], np.uint8),
        "acc_off": acc_off,
        "acc_index": np.array([a.index for a in accs], np.int32),
        "acc_kind": np.array([code[EventKind(a.kind)] for a in accs], np.uint8),
        "acc_next": np.array([bool(a.next_iteration) for a in accs], np.uint8),
        "op_times": np.array(profile.op_times_us or [], np.float64),
        "loads": np.array(loads.loads if loads is not None else [0] * p, np.int64),
        "op_owner": np.array(op_owner + [0] * (p - len(op_owner)), np.int32)[:p],
    }
    arrays = {k: (v if v.size else np.zeros(1, v.dtype)) for k, v in arrays.items()}
    dims = MpProfileDims(p, V, sum(1 for v in variables if v.alloc_index is None), len(accs),
                         loads.peak_bytes if loads is not None else 0,
                         loads.peak_index if loads is not None else 0, float(profile.period_duration_us))
    blobs = [n.encode("utf-8") for n in names]
    off = np.zeros(len(names) + 1, np.int64)
    if blobs:
        off[1:] = np.cumsum([len(b) for b in blobs])
    blob = np.frombuffer(b"".join(blobs) or b"\0", np.uint8).copy()
    fp = FlatProfile(dims, arrays, names, blob, off, profile.window)
    return fp


def device_profile(profile: IterationProfile):
    """Device handle of a profile: the extracted one, or an upload of the
    Python fields — redone whenever a field was edited in place since."""
    if profile._dev is not None and profile._device_stale():
        profile._drop_device()
    if profile._dev is None:
        fp = profile._flat_profile()
        profile.__dict__["_dev"] = N.upload_profile(fp)
        profile.__dict__["_dims"] = fp.dims()
        profile.__dict__["_sig"] = {name: _freeze(name, profile.__dict__.get(name)) for name in _DEVICE_FIELDS}
    return profile._dev


# ---------------------------------------------------------------------------
# the reference's functions


def _events_of(trace):
    return trace.events if isinstance(trace, Trace) else None


def detect_iteration(trace) -> DetectedIteration:
    """Smallest p whose last 2p (kind, size) fingerprints repeat
    (iteration.py:93-105), found on the device."""
    arrays = as_arrays(trace)
    p = N.detect(arrays)
    n = len(arrays)
    return DetectedIteration(period=p, window=(n - p, n))


def extract_lifetimes(trace, window: tuple[int, int]) -> IterationProfile:
    """Per-variable circular lifetimes of one window (iteration.py:275-301)."""
    arrays = as_arrays(trace)
    start, end = window
    n = len(arrays)
    if not (0 <= start < end <= n):
        raise ValueError(f"window {window} out of range for {n} events")
    dp = N.extract(arrays, start, end)
    return IterationProfile._from_device(dp, arrays, (start, end), _events_of(trace))


def compute_load_profile(profile: IterationProfile) -> LoadProfile:
    """Step function of live bytes per op (iteration.py:304-320)."""
    if profile._dev is not None and "variables" not in profile.__dict__:
        fp = profile._flat_profile()
        return LoadProfile(loads=fp.loads.tolist(), peak_bytes=fp.peak_bytes, peak_index=fp.peak_index)
    fp = _flatten(profile)
    dp = N.upload_profile(fp)
    loads, peak, idx = N.profile_loads(dp, profile.period)
    return LoadProfile(loads=loads.tolist(), peak_bytes=peak, peak_index=idx)


def profile_report(profile: IterationProfile) -> dict:
    """JSON-ready summary (iteration.py:323-353)."""
    variables = [{
        "var": v.var, "base_var": v.base_var, "size": v.size, "alloc_index": v.alloc_index,
        "free_index": v.free_index, "segments": [list(s) for s in v.segments], "persistent": v.persistent,
        "wraps": v.wraps,
        "accesses": [{"index": a.index, "t_us": a.t_us, "kind": a.kind.value, "next_iteration": a.next_iteration}
                     for a in v.accesses],
    } for v in profile.variables]
    return {"period": profile.period, "window": list(profile.window),
            "period_duration_us": profile.period_duration_us, "peak_bytes": profile.load.peak_bytes,
            "peak_index": profile.load.peak_index, "variables": variables,
            "load": [{"t_us": profile.op_times_us[r], "bytes": profile.load.loads[r]} for r in range(profile.period)]}


_ = (F_RENAMED, field)
