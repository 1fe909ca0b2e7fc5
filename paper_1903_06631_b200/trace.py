"""Trace event model, text formats, and the struct-of-arrays ingest form.

Mirrors the reference trace module (pkg/src/memplan/trace.py:1-192): the
same ``EventKind``/``TraceEvent``/``Trace`` types, the JSONL/CSV formats
with identical error lines, and ``validate_trace``.  What is new is
``TraceArrays``: the columnar layout every device kernel consumes
(``kind u8 | var i32 | size i64 | t_us i64``, 21 B/event), built once per
trace and cached on the ``Trace`` object while its events are unchanged.

Variable ids are interned in *lexicographic order of the name strings*, so
an id comparison is a name comparison (Python ``str`` order is code-point
order, equal to UTF-8 byte order).  The UTF-8 name bytes travel with the
arrays so the device can order the rare ``base#alloc`` renames exactly.
"""
from __future__ import annotations

import csv
import io
import itertools
import json
from dataclasses import dataclass, field
from enum import Enum
from typing import Iterable, Iterator, Sequence

import numpy as np

from .errors import InvariantViolation, MalformedRecord

JSONL_KEYS = ("index", "t_us", "kind", "var", "size")
CSV_HEADER = "index,t_us,kind,var,size"

# kind codes shared with include/memplan_b200.h (MP_MALLOC ...)
KIND_CODE = {"malloc": 0, "free": 1, "read": 2, "write": 3}


class EventKind(str, Enum):
    MALLOC = "malloc"
    FREE = "free"
    READ = "read"
    WRITE = "write"


KIND_BY_CODE = (EventKind.MALLOC, EventKind.FREE, EventKind.READ, EventKind.WRITE)
_CODE_OF_KIND = {k: i for i, k in enumerate(KIND_BY_CODE)}


@dataclass(frozen=True)
class TraceEvent:
    index: int
    t_us: int
    kind: EventKind
    var: str
    size: int = 0


@dataclass
class Trace:
    events: list[TraceEvent]
    meta: dict = field(default_factory=dict)

    def __len__(self) -> int:
        return len(self.events)

    def __iter__(self) -> Iterator[TraceEvent]:
        return iter(self.events)

    def __getitem__(self, i):
        return self.events[i]


# ---------------------------------------------------------------------------
# columnar form


class TraceArrays:
    """Struct-of-arrays view of one trace (host numpy, C-contiguous).

    ``names[i]`` is the string of var id ``i``; ids are sorted by name.
    ``index`` is kept only when it differs from the position (unvalidated
    input), so the validator can report the reference's first error.
    """

    __slots__ = ("kind", "var", "size", "t_us", "index", "_names",
                 "name_blob", "name_off", "_meta", "_dev")

    def __init__(self, kind, var, size, t_us, names: Sequence[str],
                 index=None):
        self.kind = np.ascontiguousarray(kind, dtype=np.uint8)
        self.var = np.ascontiguousarray(var, dtype=np.int32)
        self.size = np.ascontiguousarray(size, dtype=np.int64)
        self.t_us = np.ascontiguousarray(t_us, dtype=np.int64)
        self.index = None if index is None else np.ascontiguousarray(index, dtype=np.int64)
        self._names = list(names)
        blobs = [s.encode("utf-8") for s in self._names]
        off = np.zeros(len(blobs) + 1, dtype=np.int64)
        if blobs:
            off[1:] = np.cumsum([len(b) for b in blobs])
        self.name_off = off
        self.name_blob = np.frombuffer(b"".join(blobs) or b"\0", dtype=np.uint8).copy()
        self._meta = None
        self._dev = None

    @classmethod
    def from_blob(cls, kind, var, size, t_us, name_blob, name_off, index=None) -> "TraceArrays":
        """Columns plus names already packed (UTF-8 blob + offsets, sorted);
        the Python strings are decoded only if someone asks for them."""
        self = cls.__new__(cls)
        self.kind = np.ascontiguousarray(kind, dtype=np.uint8)
        self.var = np.ascontiguousarray(var, dtype=np.int32)
        self.size = np.ascontiguousarray(size, dtype=np.int64)
        self.t_us = np.ascontiguousarray(t_us, dtype=np.int64)
        self.index = None if index is None else np.ascontiguousarray(index, dtype=np.int64)
        self._names = None
        self.name_blob = np.ascontiguousarray(name_blob, dtype=np.uint8)
        self.name_off = np.ascontiguousarray(name_off, dtype=np.int64)
        if self.name_blob.size == 0:
            self.name_blob = np.zeros(1, np.uint8)
        self._meta = None
        self._dev = None
        return self

    @property
    def names(self) -> list[str]:
        if self._names is None:
            b, off = self.name_blob.tobytes(), self.name_off.tolist()
            self._names = [b[off[i]:off[i + 1]].decode("utf-8") for i in range(len(off) - 1)]
        return self._names

    def __len__(self) -> int:
        return int(self.kind.shape[0])

    @property
    def nvars(self) -> int:
        return int(self.name_off.shape[0] - 1)

    @classmethod
    def from_columns(cls, kind, var_names, size, t_us, index=None) -> "TraceArrays":
        """Intern an array of var-name strings in lexicographic id order."""
        arr = np.asarray(var_names, dtype=object)
        if arr.size == 0:
            return cls(np.zeros(0, np.uint8), np.zeros(0, np.int32),
                       np.zeros(0, np.int64), np.zeros(0, np.int64), [], index)
        uniq, inv = np.unique(arr.astype(str), return_inverse=True)
        return cls(kind, inv.astype(np.int32), size, t_us, [str(u) for u in uniq], index)

    def to_trace(self) -> Trace:
        names = self.names
        ev = [TraceEvent(index=i, t_us=int(t), kind=KIND_BY_CODE[int(k)],
                         var=names[int(v)], size=int(s))
              for i, (k, v, s, t) in enumerate(zip(self.kind.tolist(), self.var.tolist(),
                                                   self.size.tolist(), self.t_us.tolist()))]
        return Trace(events=ev)


def _events_to_arrays(events: Sequence[TraceEvent]) -> TraceArrays:
    """Columns of a list of event objects: one C pass (csrc/evconv.c) when the
    events are in the plain form, else C-level iteration (attrgetter/map/
    fromiter); names are interned in first-seen order with a dict, then only
    the distinct names are sorted."""
    n = len(events)
    if n == 0:
        return TraceArrays(np.zeros(0, np.uint8), np.zeros(0, np.int32), np.zeros(0, np.int64),
                           np.zeros(0, np.int64), [])
    native = _native_columns(events, n)
    if native is not None:
        kind, size, t_us, index, first, ids = native
    else:
        kind, size, t_us, index, first, ids = _python_columns(events, n)
    # the distinct positions are ranked by name
    uniq = list(ids)
    seen = np.fromiter(ids.values(), np.int64, count=len(uniq))
    order = sorted(range(len(uniq)), key=uniq.__getitem__)
    rank = np.empty(int(seen.max()) + 1, np.int32)
    rank[seen[order]] = np.arange(len(uniq), dtype=np.int32)
    var = rank[first]
    contiguous = bool(np.array_equal(index, np.arange(n, dtype=np.int64)))
    return TraceArrays(kind, var, size, t_us, [uniq[i] for i in order], None if contiguous else index)


def _native_columns(events, n: int):
    """One C pass over a list of events (csrc/evconv.c); None when the
    extension is absent or any event is outside the plain form."""
    if type(events) is not list:
        return None
    try:
        from . import _evconv
    except ImportError:
        return None
    kind = np.empty(n, np.uint8)
    size, t_us, index, first = (np.empty(n, np.int64) for _ in range(4))
    ids: dict[str, int] = {}
    if _evconv.columns(events, KIND_CODE, ids, kind, size, t_us, index, first) is None:
        return None
    return kind, size, t_us, index, first, ids


def _python_columns(events, n: int):
    from operator import attrgetter
    code = KIND_CODE
    kinds = list(map(attrgetter("kind"), events))
    try:
        kind = np.fromiter(map(code.__getitem__, kinds), np.uint8, count=n)
    except KeyError:
        kind = np.fromiter((code[EventKind(k).value] for k in kinds), np.uint8, count=n)
    size = np.fromiter(map(attrgetter("size"), events), np.int64, count=n)
    t_us = np.fromiter(map(attrgetter("t_us"), events), np.int64, count=n)
    index = np.fromiter(map(attrgetter("index"), events), np.int64, count=n)
    ids: dict[str, int] = {}
    # setdefault with the event position: a name keeps the position of its first event
    first = np.fromiter(map(ids.setdefault, map(attrgetter("var"), events), itertools.count()), np.int64, count=n)
    return kind, size, t_us, index, first, ids


def _remember(trace: Trace, arrays: TraceArrays) -> None:
    """Cache the columnar form on a Trace together with a snapshot of its
    event list.  Events are frozen, so the list holding the same event
    objects (or equal ones) in the same order means the same columns."""
    trace.__dict__["_mp_arrays"] = (list(trace.events), arrays)


def as_arrays(trace) -> TraceArrays:
    """Columnar view of a Trace or TraceArrays.

    The reference re-reads ``trace.events`` on every call (trace.py:55-84,
    iteration.py:93-301), so a cached column set is reused only while the
    event list still compares equal to the snapshot taken with it — list
    equality short-circuits on identical elements, so the check is a C-speed
    pointer walk; any in-place edit, append or replacement rebuilds."""
    if isinstance(trace, TraceArrays):
        return trace
    if isinstance(trace, Trace):
        cached = trace.__dict__.get("_mp_arrays")
        events = trace.events
        if cached is not None and type(events) is list and cached[0] == events:
            return cached[1]
        arrays = _events_to_arrays(events)
        if type(events) is list:
            _remember(trace, arrays)
        return arrays
    return _events_to_arrays(list(trace))


def validate_trace(events: Iterable[TraceEvent]) -> None:
    """Check the stream invariants on the device (trace.py:55-84).

    Raises InvariantViolation at the first failing event with the
    reference's reason text.
    """
    from . import _native
    arrays = as_arrays(events if isinstance(events, (Trace, TraceArrays)) else list(events))
    _native.validate(arrays)


# ---------------------------------------------------------------------------
# text formats (host-side plumbing; trace.py:87-192)


def _record(line_no: int, index, t_us, kind, var, size) -> TraceEvent:
    try:
        index, t_us, size = int(index), int(t_us), int(size)
    except (TypeError, ValueError):
        raise MalformedRecord(line_no, "index/t_us/size must be integers")
    try:
        kind = EventKind(kind)
    except ValueError:
        raise MalformedRecord(line_no, f"unknown kind {kind!r}")
    if not isinstance(var, str) or not var:
        raise MalformedRecord(line_no, "var must be a non-empty string")
    return TraceEvent(index=index, t_us=t_us, kind=kind, var=var, size=size)


def _read_jsonl(text: str) -> list[TraceEvent]:
    out = []
    want = set(JSONL_KEYS)
    for line_no, line in enumerate(text.splitlines(), start=1):
        if not line.strip():
            continue
        try:
            rec = json.loads(line)
        except json.JSONDecodeError as exc:
            raise MalformedRecord(line_no, f"bad JSON: {exc.msg}")
        if not isinstance(rec, dict) or set(rec) != want:
            raise MalformedRecord(line_no, f"keys must be exactly {want}")
        out.append(_record(line_no, *(rec[k] for k in JSONL_KEYS)))
    return out


def _read_csv(text: str) -> list[TraceEvent]:
    rows = csv.reader(io.StringIO(text))
    header = next(rows, None)
    if header is None:
        raise MalformedRecord(1, "empty file, header required")
    if header != CSV_HEADER.split(","):
        raise MalformedRecord(1, f"header must be {CSV_HEADER!r}")
    out = []
    for line_no, row in enumerate(rows, start=2):
        if not row:
            continue
        if len(row) != 5:
            raise MalformedRecord(line_no, f"expected 5 fields, got {len(row)}")
        out.append(_record(line_no, *row))
    return out


def _native_reader():
    """The device library's host-side reader entry points (None when the
    library is absent: text decoding is host plumbing, the Python reader is
    the reference semantics)."""
    try:
        from . import _native
        L = _native.lib()
    except Exception:  # noqa: BLE001
        return None
    import ctypes as C
    for name in ("mp_read_trace", "mp_reader_dims", "mp_reader_copy", "mp_reader_free"):
        getattr(L, name).restype = C.c_int
    return L


def _slow_line(fmt: str, line_no: int, line: str):
    """Decode one line with the reference semantics: None for a skipped line,
    else the event; MalformedRecord as the reference raises it."""
    if fmt == "jsonl":
        if not line.strip():
            return None
        return _read_jsonl_line(line_no, line)
    row = next(csv.reader([line]), [])
    if not row:
        return None
    if len(row) != 5:
        raise MalformedRecord(line_no, f"expected 5 fields, got {len(row)}")
    return _record(line_no, *row)


def _read_jsonl_line(line_no: int, line: str) -> TraceEvent:
    try:
        rec = json.loads(line)
    except json.JSONDecodeError as exc:
        raise MalformedRecord(line_no, f"bad JSON: {exc.msg}")
    want = set(JSONL_KEYS)
    if not isinstance(rec, dict) or set(rec) != want:
        raise MalformedRecord(line_no, f"keys must be exactly {want}")
    return _record(line_no, *(rec[k] for k in JSONL_KEYS))


def read_trace_arrays(data: bytes | str, format: str = "jsonl", threads: int = 0) -> TraceArrays:
    """Decode JSONL/CSV text straight into columns, without validation.

    The canonical records (what serialize_trace writes) are decoded by the
    native multi-threaded reader (csrc/reader.cpp); any other line is decoded
    by the reference semantics (trace.py:87-137), so a MalformedRecord carries
    the reference's line and reason.  Var ids are lexicographic name ranks.
    """
    if format not in ("jsonl", "csv"):
        raise ValueError(f"unknown format {format!r}")
    if isinstance(data, str):
        text, raw = data, data.encode("utf-8")
    else:
        raw = bytes(data)
        text = raw.decode("utf-8")  # UnicodeDecodeError exactly as the reference's decode
    L = _native_reader()
    if L is None:
        return as_arrays(_read_jsonl(text) if format == "jsonl" else _read_csv(text))
    import ctypes as C

    from ._abi import MP_E_UNSUPPORTED, MP_OK, MpErr, raise_for
    h = C.c_void_p()
    err = MpErr()
    rc = L.mp_read_trace(C.c_char_p(raw), C.c_int64(len(raw)), C.c_int32(0 if format == "jsonl" else 1),
                         C.c_int32(threads), C.byref(h), C.byref(err))
    if rc == MP_E_UNSUPPORTED:
        return as_arrays(_read_jsonl(text) if format == "jsonl" else _read_csv(text))
    raise_for(rc, err)
    try:
        n, nv, nb, ns = (C.c_int64() for _ in range(4))
        L.mp_reader_dims(h, C.byref(n), C.byref(nv), C.byref(nb), C.byref(ns))
        n, nv, nb, ns = n.value, nv.value, nb.value, ns.value
        kind = np.empty(n, np.uint8)
        var = np.empty(n, np.int32)
        size = np.empty(n, np.int64)
        t_us = np.empty(n, np.int64)
        index = np.empty(n, np.int64)
        line = np.empty(n, np.int64)
        blob = np.empty(max(nb, 1), np.uint8)
        off = np.empty(nv + 1, np.int64)
        slow = np.empty(max(ns, 1), np.int64)
        p = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
        L.mp_reader_copy(h, p(kind), p(var), p(size), p(t_us), p(index), p(line), p(blob), p(off), p(slow))
    finally:
        L.mp_reader_free(h)
    if ns:
        lines = text.split("\n")
        extra = False
        for ln in slow[:ns].tolist():
            s = lines[ln - 1]
            if s.endswith("\r"):
                s = s[:-1]
            if _slow_line(format, ln, s) is not None:
                extra = True  # a valid non-canonical record: decode the file the reference way
        if extra:
            return as_arrays(_read_jsonl(text) if format == "jsonl" else _read_csv(text))
    contiguous = n == 0 or bool(np.array_equal(index, np.arange(n, dtype=np.int64)))
    return TraceArrays.from_blob(kind, var, size, t_us, blob[:max(nb, 1)], off, None if contiguous else index)


def load_trace_arrays(path, format: str | None = None, threads: int = 0) -> TraceArrays:
    """load_trace without materializing events: a file straight to columns."""
    path = str(path)
    with open(path, "rb") as fh:
        return read_trace_arrays(fh.read(), format=_fmt_of(path, format), threads=threads)


def parse_trace(data: bytes | str, format: str = "jsonl") -> Trace:
    """Decode JSONL/CSV text and validate it (trace.py:140-151)."""
    if format not in ("jsonl", "csv"):
        raise ValueError(f"unknown format {format!r}")
    arrays = read_trace_arrays(data, format)
    trace = arrays.to_trace()
    _remember(trace, arrays)
    validate_trace(trace)
    return trace


def serialize_trace(trace: Trace, format: str = "jsonl") -> str:
    """Canonical text form; parse(serialize(t)) round-trips byte-exactly."""
    if format == "jsonl":
        lines = [json.dumps({"index": e.index, "t_us": e.t_us, "kind": e.kind.value,
                             "var": e.var, "size": e.size}, separators=(",", ":"))
                 for e in trace.events]
        return "\n".join(lines) + ("\n" if lines else "")
    if format == "csv":
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(CSV_HEADER.split(","))
        for e in trace.events:
            w.writerow([e.index, e.t_us, e.kind.value, e.var, e.size])
        return buf.getvalue()
    raise ValueError(f"unknown format {format!r}")


def _fmt_of(path: str, format: str | None) -> str:
    if format is not None:
        return format
    return "csv" if path.endswith(".csv") else "jsonl"


def load_trace(path, format: str | None = None) -> Trace:
    path = str(path)
    with open(path, "rb") as fh:
        return parse_trace(fh.read(), format=_fmt_of(path, format))


def save_trace(trace: Trace, path, format: str | None = None) -> None:
    path = str(path)
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(serialize_trace(trace, format=_fmt_of(path, format)))
