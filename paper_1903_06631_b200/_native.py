"""ctypes binding of libmemplan_b200.so (the sm_100a device library).

There is no CPU fallback: if the library or a CUDA device is missing, every
call raises.  One context (CUDA stream + scratch) is created per process on
first use; device-resident handles (trace, profile, graph) are freed when
their Python owners are collected.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from ._abi import (MP_OK, FlatProfile, MpErr, MpProfileDims, MpProfileOut, ptr,
                   raise_for, trace_in)

HERE = os.path.dirname(os.path.abspath(__file__))
# MEMPLAN_LIB: an alternative build of the same library (A/B kernel experiments, tools/ab_place.sh)
LIB_PATH = os.environ.get("MEMPLAN_LIB") or os.path.join(HERE, "libmemplan_b200.so")

_lib = None
_ctx = None
_lock = threading.Lock()


class NativeUnavailable(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.mp_ctx_launches.restype = C.c_int64
        L.mp_ctx_stream.restype = C.c_void_p
        for name in ("mp_validate", "mp_detect", "mp_extract", "mp_trace_upload", "mp_trace_upload_async",
                     "mp_trace_wait", "mp_trace_flush", "mp_validate_structure", "mp_validate_times", "mp_profile_download",
                     "mp_profile_upload", "mp_conflict_from_profile", "mp_conflict_from_arcs",
                     "mp_graph_download", "mp_plan_pool", "mp_ctx_create"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def ctx():
    """Process-wide device context (creates it on first use)."""
    global _ctx
    if _ctx is None:
        with _lock:
            if _ctx is None:
                h = C.c_void_p()
                err = MpErr()
                dev = int(os.environ.get("MEMPLAN_DEVICE", "0"))
                rc = lib().mp_ctx_create(dev, C.byref(h), C.byref(err))
                if rc != MP_OK:
                    raise NativeUnavailable(
                        f"CUDA context on device {dev} failed: {err.msg.decode(errors='replace')}")
                _ctx = h
    return _ctx


def launches() -> int:
    return int(lib().mp_ctx_launches(ctx()))


def stream_ptr() -> int:
    return int(lib().mp_ctx_stream(ctx()) or 0)


def sync():
    err = MpErr()
    rc = lib().mp_ctx_sync(ctx(), C.byref(err))
    raise_for(rc, err)


class _Handle:
    _free_fn = None

    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h and _lib is not None:
                getattr(_lib, self._free_fn)(self.h)
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass
        self.h = None


class DTrace(_Handle):
    _free_fn = "mp_trace_free"


class DProfile(_Handle):
    _free_fn = "mp_profile_free"

    def dims(self) -> MpProfileDims:
        d = MpProfileDims()
        lib().mp_profile_get_dims(self.h, C.byref(d))
        return d


class DGraph(_Handle):
    _free_fn = "mp_graph_free"


# ---------------------------------------------------------------------------
# trace stages


def device_trace(arrays, asynchronous: bool = False) -> DTrace:
    """Upload (once) and cache the trace on its TraceArrays.  With
    ``asynchronous`` the copies overlap the first stages; the host arrays
    must stay untouched until ``trace_wait``."""
    cached = getattr(arrays, "_dev", None)
    if cached is not None:
        return cached
    h = C.c_void_p()
    err = MpErr()
    fn = lib().mp_trace_upload_async if asynchronous else lib().mp_trace_upload
    rc = fn(ctx(), C.byref(trace_in(arrays)), C.byref(h), C.byref(err))
    raise_for(rc, err, arrays.names)
    d = DTrace(h)
    try:
        arrays._dev = d
    except AttributeError:
        pass
    return d


def trace_flush(d: DTrace) -> None:
    """Send the deferred timestamp column of an asynchronous upload now."""
    err = MpErr()
    raise_for(lib().mp_trace_flush(d.h, C.byref(err)), err)


def trace_wait(d: DTrace) -> None:
    """Host wait until an asynchronous upload has read its host buffers."""
    err = MpErr()
    raise_for(lib().mp_trace_wait(d.h, C.byref(err)), err)


def validate(arrays, checks: str = "all") -> None:
    """validate_trace on the device: ``checks`` "all", or the two halves of
    an overlapped upload, "structure" (everything but timestamps; reports
    what "all" would on a violation) and "times"."""
    t = device_trace(arrays)
    err = MpErr()
    fn = {"all": lib().mp_validate, "structure": lib().mp_validate_structure,
          "times": lib().mp_validate_times}[checks]
    rc = fn(ctx(), t.h, C.byref(err))
    raise_for(rc, err, arrays.names)


def detect(arrays) -> int:
    t = device_trace(arrays)
    p = C.c_int64(0)
    err = MpErr()
    rc = lib().mp_detect(ctx(), t.h, C.byref(p), C.byref(err))
    raise_for(rc, err, arrays.names)
    return int(p.value)


def detect_validate(arrays, checks: str = "all") -> int:
    """validate_trace then detect_iteration with one device round trip
    (mp_detect_validate); raises what validate, then detect, would."""
    t = device_trace(arrays)
    p = C.c_int64(0)
    err = MpErr()
    rc = lib().mp_detect_validate(ctx(), t.h, C.c_int32(1 if checks == "structure" else 0), C.byref(p),
                                  C.byref(err))
    raise_for(rc, err, arrays.names)
    return int(p.value)


def extract(arrays, start: int, end: int) -> DProfile:
    t = device_trace(arrays)
    h = C.c_void_p()
    err = MpErr()
    rc = lib().mp_extract(ctx(), t.h, C.c_int64(start), C.c_int64(end), C.byref(h), C.byref(err))
    raise_for(rc, err, arrays.names, what=f"window {(start, end)} out of range for {len(arrays)} events")
    return DProfile(h)


def extract_times(arrays, start: int, end: int, op_times: np.ndarray, duration: float) -> DProfile:
    t = device_trace(arrays)
    h = C.c_void_p()
    err = MpErr()
    op_times = np.ascontiguousarray(op_times, np.float64)
    rc = lib().mp_extract_times(ctx(), t.h, C.c_int64(start), C.c_int64(end), ptr(op_times),
                                C.c_double(duration), C.byref(h), C.byref(err))
    raise_for(rc, err, arrays.names)
    return DProfile(h)


def download_profile(dp: DProfile, names, name_blob, name_off, window) -> FlatProfile:
    dims = dp.dims()
    arrays, out = FlatProfile.alloc_arrays(dims)
    err = MpErr()
    rc = lib().mp_profile_download(ctx(), dp.h, C.byref(out), C.byref(err))
    raise_for(rc, err)
    return FlatProfile(dims, FlatProfile.trim(arrays, dims), names, name_blob, name_off, window)


def upload_profile(fp: FlatProfile) -> DProfile:
    h = C.c_void_p()
    err = MpErr()
    rc = lib().mp_profile_upload(ctx(), C.byref(fp.dims()), C.byref(fp.out_struct()), ptr(fp.name_blob),
                                 ptr(fp.name_off), C.c_int32(len(fp.names)), C.byref(h), C.byref(err))
    raise_for(rc, err)
    return DProfile(h)


# ---------------------------------------------------------------------------
# pool planning


def conflict_from_profile(dp: DProfile) -> DGraph:
    h = C.c_void_p()
    err = MpErr()
    rc = lib().mp_conflict_from_profile(ctx(), dp.h, C.byref(h), C.byref(err))
    raise_for(rc, err)
    return DGraph(h)


def conflict_from_arcs(size, tiekey, seg_off, seg_lo, seg_hi) -> DGraph:
    size = np.ascontiguousarray(size, np.int64)
    tiekey = np.ascontiguousarray(tiekey, np.int64)
    seg_off = np.ascontiguousarray(seg_off, np.int64)
    seg_lo = np.ascontiguousarray(seg_lo, np.int32)
    seg_hi = np.ascontiguousarray(seg_hi, np.int32)
    h = C.c_void_p()
    err = MpErr()
    rc = lib().mp_conflict_from_arcs(ctx(), C.c_int32(size.shape[0]), ptr(size), ptr(tiekey), ptr(seg_off),
                                     ptr(seg_lo), ptr(seg_hi), C.byref(h), C.byref(err))
    raise_for(rc, err)
    return DGraph(h)


def graph_csr(g: DGraph):
    nv, nnz = C.c_int64(), C.c_int64()
    lib().mp_graph_dims(g.h, C.byref(nv), C.byref(nnz))
    row = np.zeros(nv.value + 1, np.int64)
    col = np.zeros(max(nnz.value, 1), np.int32)
    err = MpErr()
    rc = lib().mp_graph_download(ctx(), g.h, ptr(row), ptr(col), C.byref(err))
    raise_for(rc, err)
    return row, col[:nnz.value]


def graph_dims(g: DGraph):
    nv, nnz = C.c_int64(), C.c_int64()
    lib().mp_graph_dims(g.h, C.byref(nv), C.byref(nnz))
    return int(nv.value), int(nnz.value)


def plan_pool(g: DGraph, policy: int, nvars: int, out: np.ndarray | None = None):
    offs = np.zeros(max(nvars, 1), np.int64) if out is None else out
    fp = C.c_int64(0)
    lv = C.c_int64(0)
    err = MpErr()
    rc = lib().mp_plan_pool(ctx(), g.h, C.c_int32(policy), ptr(offs), C.byref(fp), C.byref(lv), C.byref(err))
    raise_for(rc, err, what=f"unknown policy {policy!r}")
    return offs[:nvars], int(fp.value), int(lv.value)


def plan_pool_device(g: DGraph, policy: int):
    """Plan and leave the offsets in HBM (mp_graph_offsets_device)."""
    fp = C.c_int64(0)
    lv = C.c_int64(0)
    err = MpErr()
    rc = lib().mp_plan_pool(ctx(), g.h, C.c_int32(policy), None, C.byref(fp), C.byref(lv), C.byref(err))
    raise_for(rc, err, what=f"unknown policy {policy!r}")
    return int(fp.value), int(lv.value)


def graph_from_csr(row_off, col, size, tiekey) -> DGraph:
    row_off = np.ascontiguousarray(row_off, np.int64)
    col = np.ascontiguousarray(col if len(col) else np.zeros(1, np.int32), np.int32)
    size = np.ascontiguousarray(size, np.int64)
    tiekey = np.ascontiguousarray(tiekey, np.int64)
    h = C.c_void_p()
    err = MpErr()
    rc = lib().mp_graph_from_csr(ctx(), C.c_int32(size.shape[0]), ptr(row_off), ptr(col), ptr(size), ptr(tiekey),
                                 C.byref(h), C.byref(err))
    raise_for(rc, err)
    return DGraph(h)


def profile_loads(dp: DProfile, period: int):
    loads = np.zeros(max(period, 1), np.int64)
    pk, pi = C.c_int64(), C.c_int64()
    err = MpErr()
    rc = lib().mp_profile_compute_loads(ctx(), dp.h, ptr(loads), C.byref(pk), C.byref(pi), C.byref(err))
    raise_for(rc, err)
    return loads[:period], int(pk.value), int(pi.value)


# ---------------------------------------------------------------------------
# swap planning


class MpCandsIO(C.Structure):
    _fields_ = [("k", C.c_int64)] + [(n, C.c_void_p) for n in (
        "var", "size", "out_index", "out_t", "out_ready", "in_index", "in_t", "dout", "din", "spans",
        "name_rank")]


CAND_COLS = (("var", np.int32), ("size", np.int64), ("out_index", np.int32), ("out_t", np.float64),
             ("out_ready", np.float64), ("in_index", np.int32), ("in_t", np.float64), ("dout", np.float64),
             ("din", np.float64), ("spans", np.uint8), ("name_rank", np.int32))


class Cands:
    """Columnar candidates handed to the swap kernels."""

    def __init__(self, k: int, **cols):
        self.k = k
        for name, dt in CAND_COLS:
            setattr(self, name, np.ascontiguousarray(cols.get(name, np.zeros(max(k, 1), dt)), dtype=dt))

    def io(self) -> MpCandsIO:
        return MpCandsIO(self.k, *[ptr(getattr(self, n)) for n, _ in CAND_COLS])


class MpSimIO(C.Structure):
    _fields_ = [("t_so", C.c_void_p), ("t_eo", C.c_void_p), ("t_si", C.c_void_p), ("t_ei", C.c_void_p),
                ("event_order", C.c_void_p),
                ("lp_t", C.c_void_p), ("lp_v", C.c_void_p), ("n_lp", C.c_int64), ("lp_peak", C.c_int64),
                ("lp_peak_t", C.c_double),
                ("ldp_t", C.c_void_p), ("ldp_v", C.c_void_p), ("n_ldp", C.c_int64), ("ldp_peak", C.c_int64),
                ("ldp_peak_t", C.c_double),
                ("delayed_index", C.c_void_p), ("delayed_us", C.c_void_p), ("n_delayed", C.c_int64),
                ("delay", C.c_double), ("rounds", C.c_int64)]


def swap_candidates(dp: DProfile, nvars: int, threshold: int, bw: float, lat: float) -> Cands:
    c = Cands(nvars)
    io = c.io()
    err = MpErr()
    rc = lib().mp_swap_candidates(ctx(), dp.h, C.c_int64(threshold), C.c_double(bw), C.c_double(lat),
                                  C.byref(io), C.byref(err))
    raise_for(rc, err)
    c.k = int(io.k)
    for name, _ in CAND_COLS:
        setattr(c, name, getattr(c, name)[:c.k])
    return c


def swap_scores(dp: DProfile, c: Cands):
    k = c.k
    outs = [np.zeros(max(k, 1)) for _ in range(4)]
    order = np.zeros(max(k, 1), np.int32)
    peaks = np.zeros(k + 1)
    err = MpErr()
    rc = lib().mp_swap_scores(ctx(), dp.h, C.byref(c.io()), *[ptr(a) for a in outs], ptr(order), ptr(peaks),
                              C.byref(err))
    raise_for(rc, err)
    return [a[:k] for a in outs], order[:k], peaks


def swap_gap_area(dp: DProfile, c: Cands, loads=None) -> np.ndarray:
    out = np.zeros(max(c.k, 1))
    cur = None if loads is None else np.ascontiguousarray(loads, np.float64)
    err = MpErr()
    rc = lib().mp_swap_gap_area(ctx(), dp.h, C.byref(c.io()), ptr(cur), ptr(out), C.byref(err))
    raise_for(rc, err)
    return out[:c.k]


def swap_select_static(dp: DProfile, c: Cands, ranked, limit: int):
    sel = np.zeros(max(c.k, 1), np.int32)
    n = C.c_int64()
    rk = np.ascontiguousarray(ranked if len(ranked) else np.zeros(1), np.float64)
    err = MpErr()
    rc = lib().mp_swap_select_static(ctx(), dp.h, C.byref(c.io()), ptr(rk), C.c_int64(limit), ptr(sel),
                                     C.byref(n), C.byref(err))
    raise_for(rc, err)
    return sel[:n.value]


def swap_planned_peak(dp: DProfile, c: Cands, subset=None) -> float:
    pk = C.c_double()
    sub = None if subset is None else np.ascontiguousarray(subset if len(subset) else np.zeros(1), np.int32)
    nsub = 0 if subset is None else len(subset)
    err = MpErr()
    rc = lib().mp_swap_planned_peak(ctx(), dp.h, C.byref(c.io()), ptr(sub), C.c_int64(nsub), C.byref(pk),
                                    C.byref(err))
    raise_for(rc, err)
    return float(pk.value)


def swap_schedule(c: Cands, sel, ready, deadline):
    sel = np.ascontiguousarray(sel, np.int32)
    n = sel.shape[0]
    t = [np.zeros(max(n, 1)) for _ in range(4)]
    eo = np.zeros(max(n, 1), np.int32)
    rd = np.ascontiguousarray(ready if n else np.zeros(1), np.float64)
    dl = np.ascontiguousarray(deadline if n else np.zeros(1), np.float64)
    err = MpErr()
    rc = lib().mp_swap_schedule(ctx(), C.byref(c.io()), ptr(sel if n else np.zeros(1, np.int32)), C.c_int64(n),
                                ptr(rd), ptr(dl), *[ptr(a) for a in t], ptr(eo), C.byref(err))
    raise_for(rc, err)
    return [a[:n] for a in t], eo[:n]


def swap_simulate(dp: DProfile, period: int, c: Cands, sel, sched, limit, max_rounds=100, cand_names=None):
    sel = np.ascontiguousarray(sel, np.int32)
    n = sel.shape[0]
    t = [np.array(a, np.float64) if n else np.zeros(1) for a in sched[0]]
    eo = np.array(sched[1], np.int32) if n else np.zeros(1, np.int32)
    cap = 1 + period + 2 * n + 2
    b = dict(lp_t=np.zeros(cap), lp_v=np.zeros(cap, np.int64), ldp_t=np.zeros(cap),
             ldp_v=np.zeros(cap, np.int64), di=np.zeros(period + 1, np.int64), du=np.zeros(period + 1))
    io = MpSimIO(ptr(t[0]), ptr(t[1]), ptr(t[2]), ptr(t[3]), ptr(eo), ptr(b["lp_t"]), ptr(b["lp_v"]), 0, 0, 0.0,
                 ptr(b["ldp_t"]), ptr(b["ldp_v"]), 0, 0, 0.0, ptr(b["di"]), ptr(b["du"]), 0, 0.0, 0)
    err = MpErr()
    rc = lib().mp_swap_simulate(ctx(), dp.h, C.byref(c.io()), ptr(sel if n else np.zeros(1, np.int32)),
                                C.c_int64(n), C.c_int64(0 if limit is None else limit),
                                C.c_int32(limit is not None), C.c_int32(max_rounds), C.byref(io), C.byref(err))
    raise_for(rc, err, cand_names=cand_names)
    return dict(t_so=t[0][:n], t_eo=t[1][:n], t_si=t[2][:n], t_ei=t[3][:n], event_order=eo[:n],
                lp=(b["lp_t"][:io.n_lp], b["lp_v"][:io.n_lp], int(io.lp_peak), float(io.lp_peak_t)),
                ldp=(b["ldp_t"][:io.n_ldp], b["ldp_v"][:io.n_ldp], int(io.ldp_peak), float(io.ldp_peak_t)),
                delayed=(b["di"][:io.n_delayed], b["du"][:io.n_delayed]), delay=float(io.delay),
                rounds=int(io.rounds))


def swap_eval_weights(dp: DProfile, c: Cands, z, weights, limit: int, max_rounds: int = 100):
    """Batched BO objective (mp_swap_eval_weights): per weight vector
    (status, overhead_us, nsel, aux)."""
    w = np.ascontiguousarray(weights, np.float64).reshape(-1, 4)
    m = w.shape[0]
    zz = np.ascontiguousarray(z, np.float64).reshape(4, -1) if c.k else np.zeros((4, 1))
    st = np.zeros(max(m, 1), np.int32)
    ov = np.zeros(max(m, 1))
    ns = np.zeros(max(m, 1), np.int64)
    ax = np.zeros(max(m, 1), np.int64)
    err = MpErr()
    rc = lib().mp_swap_eval_weights(ctx(), dp.h, C.byref(c.io()), ptr(zz), ptr(w), C.c_int64(m), C.c_int64(limit),
                                    C.c_int32(max_rounds), ptr(st), ptr(ov), ptr(ns), ptr(ax), C.byref(err))
    raise_for(rc, err)
    return st[:m], ov[:m], ns[:m], ax[:m]


def standardize(x) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros(max(x.shape[0], 1))
    lib().mp_standardize(ptr(x if x.shape[0] else np.zeros(1)), C.c_int64(x.shape[0]), ptr(out))
    return out[:x.shape[0]]


STAGES = ("group_sort", "validate", "detect", "extract", "loads", "conflict_prep", "conflict_fill",
          "place_order", "place_split", "place", "footprint", "swap", "sweep")


def set_timing(on: bool) -> None:
    lib().mp_ctx_set_timing(ctx(), C.c_int(1 if on else 0))


def timings() -> dict:
    """Accumulated per-stage device ms (CUDA events on the library stream)."""
    ms = (C.c_double * 16)()
    cnt = (C.c_int64 * 16)()
    err = MpErr()
    rc = lib().mp_ctx_timings(ctx(), ms, cnt, C.byref(err))
    raise_for(rc, err)
    return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(STAGES) if cnt[i]}


_ = (MpProfileOut,)
