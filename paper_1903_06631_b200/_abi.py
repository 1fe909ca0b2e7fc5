"""ctypes mirrors of the structs in include/memplan_b200.h and the flat
host-side containers both the device library and the CPU oracle fill.

``FlatProfile`` is the columnar ``IterationProfile``: per-variable arrays
in the reference variable order, an access CSR, and per-op arrays.  It is
what crosses the C ABI; ``iteration.IterationProfile`` materializes the
reference dataclasses from it lazily.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .errors import (InvariantViolation, LimitUnreachable, MemplanError,
                     PeriodNotFound, SwapDeadlock)

MP_OK = 0
MP_E_INVARIANT = 1
MP_E_PERIOD_NOT_FOUND = 2
MP_E_LIMIT_UNREACHABLE = 3
MP_E_SWAP_DEADLOCK = 4
MP_E_SIM_INDEXERROR = 5
MP_E_VALUE = 6
MP_E_CUDA = 7
MP_E_NOMEM = 8
MP_E_UNSUPPORTED = 9

F_PERSISTENT, F_WRAPS, F_RENAMED = 1, 2, 4

KIND_NAMES = ("malloc", "free", "read", "write")


class MpErr(C.Structure):
    _fields_ = [("code", C.c_int32), ("trace", C.c_int32), ("index", C.c_int64),
                ("aux0", C.c_int64), ("aux1", C.c_int64), ("msg", C.c_char * 192)]


class MpTraceIn(C.Structure):
    _fields_ = [("n", C.c_int64), ("kind", C.c_void_p), ("var", C.c_void_p),
                ("size", C.c_void_p), ("t_us", C.c_void_p), ("index", C.c_void_p),
                ("nvars", C.c_int32), ("name_blob", C.c_void_p), ("name_off", C.c_void_p)]


class MpProfileDims(C.Structure):
    _fields_ = [("period", C.c_int64), ("nvars", C.c_int64), ("ncarry", C.c_int64),
                ("naccess", C.c_int64), ("peak_bytes", C.c_int64), ("peak_index", C.c_int64),
                ("duration_us", C.c_double)]


class MpProfileOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "base", "size", "alloc", "free_", "nseg", "seg", "flags", "acc_off",
        "acc_index", "acc_kind", "acc_next", "op_times", "loads", "op_owner")]


def ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def trace_in(arrays) -> MpTraceIn:
    """Borrowed view of a TraceArrays (keep `arrays` alive during the call)."""
    return MpTraceIn(len(arrays), ptr(arrays.kind), ptr(arrays.var), ptr(arrays.size),
                     ptr(arrays.t_us), ptr(arrays.index), arrays.nvars,
                     ptr(arrays.name_blob), ptr(arrays.name_off))


_PROFILE_ARRAYS = (
    # name, dtype, length-kind
    ("base", np.int32, "V"), ("size", np.int64, "V"), ("alloc", np.int32, "V"),
    ("free_", np.int32, "V"), ("nseg", np.int32, "V"), ("seg", np.int32, "V4"),
    ("flags", np.uint8, "V"), ("acc_off", np.int64, "V1"), ("acc_index", np.int32, "A"),
    ("acc_kind", np.uint8, "A"), ("acc_next", np.uint8, "A"), ("op_times", np.float64, "P"),
    ("loads", np.int64, "P"), ("op_owner", np.int32, "P"))


class FlatProfile:
    """Columnar iteration profile plus the name table of its trace."""

    def __init__(self, dims: MpProfileDims, arrays: dict, names, name_blob, name_off,
                 window=(0, 0)):
        self.period = int(dims.period)
        self.nvars = int(dims.nvars)
        self.ncarry = int(dims.ncarry)
        self.naccess = int(dims.naccess)
        self.peak_bytes = int(dims.peak_bytes)
        self.peak_index = int(dims.peak_index)
        self.duration_us = float(dims.duration_us)
        for k, v in arrays.items():
            setattr(self, k, v)
        self.names = names
        self.name_blob = name_blob
        self.name_off = name_off
        self.window = tuple(window)

    @staticmethod
    def alloc_arrays(dims: MpProfileDims) -> tuple[dict, MpProfileOut]:
        V, A, P = int(dims.nvars), int(dims.naccess), int(dims.period)
        n = {"V": V, "V1": V + 1, "V4": 4 * V, "A": A, "P": P}
        arrays = {k: np.zeros(max(n[kind], 1), dtype=dt) for k, dt, kind in _PROFILE_ARRAYS}
        out = MpProfileOut(**{k: ptr(a) for k, a in arrays.items()})
        # trim views to exact sizes after the fill
        return arrays, out

    @staticmethod
    def trim(arrays: dict, dims: MpProfileDims) -> dict:
        V, A, P = int(dims.nvars), int(dims.naccess), int(dims.period)
        n = {"V": V, "V1": V + 1, "V4": 4 * V, "A": A, "P": P}
        return {k: arrays[k][:n[kind]] for k, _, kind in _PROFILE_ARRAYS}

    def dims(self) -> MpProfileDims:
        return MpProfileDims(self.period, self.nvars, self.ncarry, self.naccess,
                             self.peak_bytes, self.peak_index, self.duration_us)

    def out_struct(self) -> MpProfileOut:
        return MpProfileOut(**{k: ptr(getattr(self, k)) for k, _, _ in _PROFILE_ARRAYS})

    def var_name(self, i: int) -> str:
        base = self.names[int(self.base[i])]
        if self.flags[i] & F_RENAMED:
            return f"{base}#{int(self.alloc[i])}"
        return base

    def var_names(self) -> list[str]:
        names = self.names
        base = self.base.tolist()
        out = [names[b] for b in base]
        ren = np.nonzero(self.flags & F_RENAMED)[0]
        alloc = self.alloc
        for i in ren.tolist():
            out[i] = f"{out[i]}#{int(alloc[i])}"
        return out

    def name_ralloc(self) -> np.ndarray:
        """per var: alloc when the name is renamed, else -1"""
        return np.where(self.flags & F_RENAMED, self.alloc, -1).astype(np.int32)


def invariant_reason(err: MpErr, names) -> str:
    code = int(err.aux0)
    a1 = int(err.aux1)
    if code == 1:
        return f"index {a1} not contiguous"
    if code == 2:
        return "negative timestamp"
    if code == 3:
        return "timestamp decreases"
    if code == 4:
        return "malloc size must be > 0"
    if code == 5:
        return f"malloc of live id {names[a1]!r}"
    if code == 6:
        return f"{KIND_NAMES[a1]} size must be 0"
    if code == 7:
        return f"free of dead id {names[a1]!r}"
    if code == 8:
        return f"use of dead id {names[a1]!r}"
    if code == 9:
        return f"malloc of live id {names[a1]!r} in window"
    if code == 10:
        return f"free of dead id {names[a1]!r} in window"
    if code == 11:
        return f"use of dead id {names[a1]!r} in window"
    return f"invariant {code}"


def raise_for(rc: int, err: MpErr, names=None, what: str = "", cand_names=None):
    """Map a status code onto the reference exception (errors.py)."""
    if rc == MP_OK:
        return
    if rc == MP_E_INVARIANT:
        raise InvariantViolation(int(err.index), invariant_reason(err, names))
    if rc == MP_E_PERIOD_NOT_FOUND:
        raise PeriodNotFound(f"no repeating iteration suffix in {int(err.index)} events")
    if rc == MP_E_LIMIT_UNREACHABLE:
        raise LimitUnreachable(int(err.aux0), int(err.aux1))
    if rc == MP_E_SWAP_DEADLOCK:
        if int(err.aux0) == 1 and cand_names is not None:
            raise SwapDeadlock(int(err.index), f"swap-in of {cand_names[int(err.aux1)]!r} cannot start")
        raise SwapDeadlock(int(err.index))
    if rc == MP_E_SIM_INDEXERROR:
        # the reference's replay raises a bare IndexError here
        # (swapsim.py:266-267); kept for drop-in parity
        raise IndexError("list index out of range")
    if rc == MP_E_VALUE:
        raise ValueError(what or err.msg.decode(errors="replace"))
    raise MemplanError(f"native status {rc}: {err.msg.decode(errors='replace')} {what}")
