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
LIB_PATH = os.path.join(HERE, "libmemplan_b200.so")

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
        for name in ("mp_validate", "mp_detect", "mp_extract", "mp_trace_upload", "mp_profile_download",
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


def device_trace(arrays) -> DTrace:
    """Upload (once) and cache the trace on its TraceArrays."""
    cached = getattr(arrays, "_dev", None)
    if cached is not None:
        return cached
    h = C.c_void_p()
    err = MpErr()
    rc = lib().mp_trace_upload(ctx(), C.byref(trace_in(arrays)), C.byref(h), C.byref(err))
    raise_for(rc, err, arrays.names)
    d = DTrace(h)
    try:
        arrays._dev = d
    except AttributeError:
        pass
    return d


def validate(arrays) -> None:
    t = device_trace(arrays)
    err = MpErr()
    rc = lib().mp_validate(ctx(), t.h, C.byref(err))
    raise_for(rc, err, arrays.names)


def detect(arrays) -> int:
    t = device_trace(arrays)
    p = C.c_int64(0)
    err = MpErr()
    rc = lib().mp_detect(ctx(), t.h, C.byref(p), C.byref(err))
    raise_for(rc, err, arrays.names)
    return int(p.value)


def extract(arrays, start: int, end: int) -> DProfile:
    t = device_trace(arrays)
    h = C.c_void_p()
    err = MpErr()
    rc = lib().mp_extract(ctx(), t.h, C.c_int64(start), C.c_int64(end), C.byref(h), C.byref(err))
    raise_for(rc, err, arrays.names, what=f"window {(start, end)} out of range for {len(arrays)} events")
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


STAGES = ("group_sort", "validate", "detect", "extract", "loads", "conflict_prep", "conflict_fill",
          "place_order", "place_split", "place", "footprint", "swap")


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
