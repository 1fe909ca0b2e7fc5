"""ctypes binding of the CPU oracle (liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, by __graft_entry__.smoke()
and by bench.py's cpu_baseline / --impl reference legs, always as the
checker or the CPU baseline — never by the product package.  The oracle is
a sequential C restatement of the reference path (memplan_oracle.c) and is
pinned against tests/golden/, which the reference itself produced.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1903_06631_b200._abi import (MP_OK, FlatProfile, MpErr, MpProfileDims,
                                        MpProfileOut, ptr, trace_in)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = C.CDLL(LIB)
        _lib.orc_graph_nnz.restype = C.c_int64
        _lib.orc_candidates.restype = C.c_int64
        _lib.orc_load_min.restype = C.c_int64
        _lib.orc_gap_area.restype = C.c_double
    return _lib


class Names(C.Structure):
    _fields_ = [("blob", C.c_void_p), ("off", C.c_void_p)]


class Cands(C.Structure):
    _fields_ = [("k", C.c_int64)] + [(n, C.c_void_p) for n in (
        "var", "size", "out_index", "out_t", "out_ready", "in_index", "in_t", "dout", "din",
        "spans", "name_base", "name_ralloc")]


class Load(C.Structure):
    _fields_ = [("period", C.c_int64), ("loads", C.c_void_p), ("op_times", C.c_void_p),
                ("duration", C.c_double)]


class SimOut(C.Structure):
    _fields_ = [("t_so", C.c_void_p), ("t_eo", C.c_void_p), ("t_si", C.c_void_p),
                ("t_ei", C.c_void_p), ("event_order", C.c_void_p),
                ("lp_t", C.c_void_p), ("lp_v", C.c_void_p), ("n_lp", C.c_int64),
                ("lp_peak", C.c_int64), ("lp_peak_t", C.c_double),
                ("ldp_t", C.c_void_p), ("ldp_v", C.c_void_p), ("n_ldp", C.c_int64),
                ("ldp_peak", C.c_int64), ("ldp_peak_t", C.c_double),
                ("delayed_index", C.c_void_p), ("delayed_us", C.c_void_p),
                ("n_delayed", C.c_int64), ("delay", C.c_double), ("rounds", C.c_int64)]


CAND_FIELDS = (("var", np.int32), ("size", np.int64), ("out_index", np.int32),
               ("out_t", np.float64), ("out_ready", np.float64), ("in_index", np.int32),
               ("in_t", np.float64), ("dout", np.float64), ("din", np.float64),
               ("spans", np.uint8), ("name_base", np.int32), ("name_ralloc", np.int32))


class CandArrays:
    """Columnar swap candidates (autoswap.py:34-50)."""

    def __init__(self, k: int, **arrays):
        self.k = k
        for name, dt in CAND_FIELDS:
            setattr(self, name, np.ascontiguousarray(arrays[name], dtype=dt))

    @classmethod
    def empty(cls, n):
        return cls(0, **{name: np.zeros(max(n, 1), dt) for name, dt in CAND_FIELDS})

    def struct(self) -> Cands:
        return Cands(self.k, *[ptr(getattr(self, n)) for n, _ in CAND_FIELDS])

    def trim(self):
        for n, _ in CAND_FIELDS:
            setattr(self, n, getattr(self, n)[:self.k])
        return self


def validate(arrays):
    err = MpErr()
    rc = lib().orc_validate(C.byref(trace_in(arrays)), C.byref(err))
    return rc, err


def detect(arrays, naive=False):
    p = C.c_int64(0)
    err = MpErr()
    f = lib().orc_detect_naive if naive else lib().orc_detect
    rc = f(C.byref(trace_in(arrays)), C.byref(p), C.byref(err))
    return rc, int(p.value)


def extract(arrays, start, end):
    L = lib()
    h = C.c_void_p()
    err = MpErr()
    rc = L.orc_extract(C.byref(trace_in(arrays)), C.c_int64(start), C.c_int64(end),
                       C.byref(h), C.byref(err))
    if rc != MP_OK:
        return rc, err
    dims = MpProfileDims()
    L.orc_profile_dims(h, C.byref(dims))
    arr, out = FlatProfile.alloc_arrays(dims)
    L.orc_profile_copy(h, C.byref(out))
    L.orc_profile_free(h)
    return MP_OK, FlatProfile(dims, FlatProfile.trim(arr, dims), arrays.names,
                              arrays.name_blob, arrays.name_off, (start, end))


def conflict(seg_off, lo, hi):
    L = lib()
    seg_off = np.ascontiguousarray(seg_off, np.int64)
    lo = np.ascontiguousarray(lo, np.int32)
    hi = np.ascontiguousarray(hi, np.int32)
    nv = seg_off.shape[0] - 1
    h = C.c_void_p()
    L.orc_conflict(C.c_int32(nv), ptr(seg_off), ptr(lo), ptr(hi), C.byref(h))
    nnz = L.orc_graph_nnz(h)
    row = np.zeros(nv + 1, np.int64)
    col = np.zeros(max(nnz, 1), np.int32)
    L.orc_graph_copy(h, ptr(row), ptr(col))
    return h, row, col[:nnz]


def graph_free(h):
    lib().orc_graph_free(h)


def profile_segments(fp: FlatProfile):
    nseg = fp.nseg.astype(np.int64)
    off = np.zeros(fp.nvars + 1, np.int64)
    off[1:] = np.cumsum(nseg)
    seg = fp.seg.reshape(-1, 4)
    lo = np.concatenate([seg[:, 0:1], seg[:, 2:3]], axis=1)
    hi = np.concatenate([seg[:, 1:2], seg[:, 3:4]], axis=1)
    mask = np.arange(2)[None, :] < nseg[:, None]
    return off, lo[mask], hi[mask]


def plan(h, size, alloc, name_base, name_ralloc, blob, off, policy):
    size = np.ascontiguousarray(size, np.int64)
    alloc = np.ascontiguousarray(alloc, np.int64)
    nb = np.ascontiguousarray(name_base, np.int32)
    nr = np.ascontiguousarray(name_ralloc, np.int32)
    offs = np.zeros(max(size.shape[0], 1), np.int64)
    fp = C.c_int64(0)
    names = Names(ptr(blob), ptr(off))
    rc = lib().orc_plan(h, ptr(size), ptr(alloc), ptr(nb), ptr(nr), names, C.c_int32(policy),
                        ptr(offs), C.byref(fp))
    return rc, offs[:size.shape[0]], int(fp.value)


def _load(fp: FlatProfile) -> Load:
    return Load(fp.period, ptr(fp.loads), ptr(fp.op_times), fp.duration_us)


def candidates(fp: FlatProfile, threshold, bw, lat) -> CandArrays:
    c = CandArrays.empty(fp.nvars)
    st = c.struct()
    k = lib().orc_candidates(C.byref(fp.dims()), C.byref(fp.out_struct()), C.c_int64(threshold),
                             C.c_double(bw), C.c_double(lat), C.byref(st))
    c.k = int(k)
    return c.trim()


def names_of(fp_or_blob, off=None) -> Names:
    if off is None:
        return Names(ptr(fp_or_blob.name_blob), ptr(fp_or_blob.name_off))
    return Names(ptr(fp_or_blob), ptr(off))


def scores(load: Load, c: CandArrays, names: Names):
    k = max(c.k, 1)
    out = [np.zeros(k) for _ in range(4)]
    order = np.zeros(k, np.int32)
    lib().orc_scores(load, C.byref(c.struct()), names, *[ptr(a) for a in out], ptr(order))
    return [a[:c.k] for a in out], order[:c.k]


def standardize(x):
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros(max(x.shape[0], 1))
    lib().orc_standardize(ptr(x), C.c_int64(x.shape[0]), ptr(out))
    return out[:x.shape[0]]


def select(load: Load, c: CandArrays, names: Names, score: int, weights, limit: int):
    sel = np.zeros(max(c.k, 1), np.int32)
    n = C.c_int64(0)
    w = np.ascontiguousarray(weights if weights is not None else (0.0, 0.0, 0.0, 1.0), np.float64)
    err = MpErr()
    rc = lib().orc_select(load, C.byref(c.struct()), names, C.c_int32(score), ptr(w),
                          C.c_int64(limit), ptr(sel), C.byref(n), C.byref(err))
    return rc, err, sel[:n.value]


def load_min(load: Load, c: CandArrays) -> int:
    return int(lib().orc_load_min(load, C.byref(c.struct())))


def schedule(fp: FlatProfile, c: CandArrays, names: Names, sel):
    sel = np.ascontiguousarray(sel, np.int32)
    n = sel.shape[0]
    t = [np.zeros(max(n, 1)) for _ in range(4)]
    eo = np.zeros(max(n, 1), np.int32)
    lib().orc_schedule(C.byref(fp.dims()), ptr(fp.op_times), C.byref(c.struct()), names, ptr(sel),
                       C.c_int64(n), *[ptr(a) for a in t], ptr(eo))
    return [a[:n] for a in t], eo[:n]


def simulate(fp: FlatProfile, c: CandArrays, names: Names, sel, sched, limit,
             max_rounds=100, window0=None):
    sel = np.ascontiguousarray(sel, np.int32)
    n, p = sel.shape[0], fp.period
    cap = 1 + p + 2 * n + 2
    t = [np.array(a, dtype=np.float64) if n else np.zeros(1) for a in sched[0]]
    eo = np.array(sched[1], np.int32) if n else np.zeros(1, np.int32)
    bufs = dict(lp_t=np.zeros(cap), lp_v=np.zeros(cap, np.int64), ldp_t=np.zeros(cap),
                ldp_v=np.zeros(cap, np.int64), di=np.zeros(p + 1, np.int64), du=np.zeros(p + 1))
    o = SimOut(ptr(t[0]), ptr(t[1]), ptr(t[2]), ptr(t[3]), ptr(eo), ptr(bufs["lp_t"]),
               ptr(bufs["lp_v"]), 0, 0, 0.0, ptr(bufs["ldp_t"]), ptr(bufs["ldp_v"]), 0, 0, 0.0,
               ptr(bufs["di"]), ptr(bufs["du"]), 0, 0.0, 0)
    err = MpErr()
    w0 = fp.window[0] if window0 is None else window0
    rc = lib().orc_simulate(C.byref(fp.dims()), C.byref(fp.out_struct()), C.c_int64(w0),
                            C.byref(c.struct()), names, ptr(sel), C.c_int64(n),
                            C.c_int64(0 if limit is None else limit), C.c_int32(limit is not None),
                            C.c_int32(max_rounds), C.byref(o), C.byref(err))
    if rc != MP_OK:
        return rc, err, None
    res = dict(t_so=t[0][:n], t_eo=t[1][:n], t_si=t[2][:n], t_ei=t[3][:n], event_order=eo[:n],
               lp=(bufs["lp_t"][:o.n_lp], bufs["lp_v"][:o.n_lp], o.lp_peak, o.lp_peak_t),
               ldp=(bufs["ldp_t"][:o.n_ldp], bufs["ldp_v"][:o.n_ldp], o.ldp_peak, o.ldp_peak_t),
               delayed=(bufs["di"][:o.n_delayed], bufs["du"][:o.n_delayed]),
               delay=o.delay, rounds=o.rounds)
    return rc, err, res


lib_loaded = lib
_ = (MpProfileOut,)


# ---------------------------------------------------------------------------
# batched sweep unit (orc_sweep_unit): the checker / CPU baseline of
# paper_1903_06631_b200.sweep


def sweep_unit(arrays, params):
    """One unit of a sweep on the CPU: (trace record, budget records,
    offsets, greedy order) with the dtypes of paper_1903_06631_b200.sweep."""
    from paper_1903_06631_b200.sweep import BUDGET_DTYPE, TRACE_DTYPE
    L = lib()
    L.orc_sweep_unit.restype = C.c_int
    prm = params.struct()
    rec = np.zeros(1, TRACE_DTYPE)
    nb = len(params.budgets)
    brec = np.zeros(max(nb, 1), BUDGET_DTYPE)
    n = len(arrays)
    offs = np.zeros(max(n, 1), np.int64)
    order = np.zeros(max(n, 1), np.int32)
    L.orc_sweep_unit(C.byref(trace_in(arrays)), C.byref(prm), ptr(rec), ptr(brec), ptr(offs), ptr(order))
    r = rec[0]
    return r, brec[:nb], offs[:int(r["nvars"])], order[:int(r["norder"])]


def sweep(batch, params, indices=None):
    """Every unit of a SweepBatch (or the given subset) on one host core."""
    from paper_1903_06631_b200.sweep import BUDGET_DTYPE, TRACE_DTYPE
    idx = range(batch.ntraces) if indices is None else indices
    idx = list(idx)
    nb = len(params.budgets)
    recs = np.zeros(len(idx), TRACE_DTYPE)
    brecs = np.zeros((len(idx), nb), BUDGET_DTYPE)
    offs, orders = [], []
    for q, t in enumerate(idx):
        r, b, o, od = sweep_unit(batch.trace(t), params)
        recs[q] = r
        brecs[q] = b
        offs.append(o)
        orders.append(od)
    return recs, brecs, offs, orders
