"""Native trace reader (csrc/reader.cpp) against the reference-semantics
Python decoder (trace.py:87-137) on CPU: identical columns and names on
canonical and non-canonical input, identical MalformedRecord line/reason."""
import numpy as np
import pytest

from paper_1903_06631_b200 import synth, workloads
from paper_1903_06631_b200 import trace as T
from paper_1903_06631_b200.errors import MalformedRecord


def python_path(text, fmt):
    if isinstance(text, bytes):
        text = text.decode("utf-8")  # parse_trace decodes first (trace.py:143)
    return T.as_arrays(T._read_jsonl(text) if fmt == "jsonl" else T._read_csv(text))


def same(a, b):
    assert a.names == b.names
    for c in ("kind", "var", "size", "t_us"):
        assert np.array_equal(getattr(a, c), getattr(b, c)), c
    assert (a.index is None) == (b.index is None)
    if a.index is not None:
        assert np.array_equal(a.index, b.index)


def outcome(fn):
    try:
        return ("ok", fn())
    except MalformedRecord as e:
        return ("MalformedRecord", e.line, e.reason)
    except Exception as e:  # noqa: BLE001
        return (type(e).__name__, str(e))


def check(text, fmt):
    a, b = outcome(lambda: T.read_trace_arrays(text, fmt)), outcome(lambda: python_path(text, fmt))
    assert a[0] == b[0], (a, b)
    if a[0] == "ok":
        same(a[1], b[1])
    else:
        assert a[1:] == b[1:]
    return a[0]


TRACES = [synth.generate_synthetic_trace(synth.vgg_like(depth=5, scale=0.5, iterations=3, seed=2)),
          workloads.random_periodic_trace(3, slots=24, nvars=8, iterations=4),
          T.Trace(events=[T.TraceEvent(0, 0, T.EventKind.MALLOC, "é名 x", 8),
                          T.TraceEvent(1, 3, T.EventKind.FREE, "é名 x", 0)])]


@pytest.mark.parametrize("fmt", ["jsonl", "csv"])
@pytest.mark.parametrize("ti", range(len(TRACES)))
def test_canonical_round_trip(fmt, ti):
    text = T.serialize_trace(TRACES[ti], fmt)
    assert check(text, fmt) == "ok"
    assert check(text.encode("utf-8"), fmt) == "ok"
    assert check(text.replace("\n", "\r\n"), fmt) == "ok"


JSONL_EDITS = [
    ('{"index": 3, "t_us": 4}', "keys"),
    ('{"index": 3.0, "t_us": 4, "kind": "read", "var": "w0", "size": 0}', "float"),
    ('{"index": true, "t_us": 4, "kind": "read", "var": "w0", "size": 0}', "bool"),
    ('{"index": null, "t_us": 4, "kind": "read", "var": "w0", "size": 0}', "null"),
    ('{"index": 3, "t_us": 4, "kind": "reed", "var": "w0", "size": 0}', "kind"),
    ('{"index": 3, "t_us": 4, "kind": "read", "var": "", "size": 0}', "empty var"),
    ('{"index": 3, "t_us": 4, "kind": "read", "var": 7, "size": 0}', "int var"),
    ('{"index": 3, "t_us": 4, "kind": "read", "var": "w\\u0030", "size": 0}', "escape"),
    ('{"index": 3, "index": 3, "t_us": 4, "kind": "read", "var": "w0", "size": 0}', "dup"),
    ('{"index": 012, "t_us": 4, "kind": "read", "var": "w0", "size": 0}', "leading zero"),
    ('{"index": 99999999999999999999, "t_us": 4, "kind": "read", "var": "w0", "size": 0}', "big"),
    ("   ", "blank"),
    ("not json", "garbage"),
    ('[1, 2]', "list"),
    ('  {"size": 0, "var": "w0", "kind": "read", "t_us": 4, "index": 3}  ', "reordered"),
]


@pytest.mark.parametrize("edit,label", JSONL_EDITS, ids=[e[1] for e in JSONL_EDITS])
def test_jsonl_line_variants(edit, label):
    lines = T.serialize_trace(TRACES[0], "jsonl").split("\n")
    lines[3] = edit
    check("\n".join(lines), "jsonl")


CSV_EDITS = [("3,4,read,w0", "fields"), ("3, 4,read,w0,0", "space int"), ("+3,4,read,w0,0", "plus"),
             ("3,4,read, w0,0", "space var"), ("3,4,reed,w0,0", "kind"), ("3,4,read,,0", "empty var"),
             ("", "empty row"), ("3,4,read,w0,1_0", "underscore"), ('3,4,read,"w0",0', "quoted"),
             ("3,4,read,w0,0,", "six")]


@pytest.mark.parametrize("edit,label", CSV_EDITS, ids=[e[1] for e in CSV_EDITS])
def test_csv_line_variants(edit, label):
    lines = T.serialize_trace(TRACES[0], "csv").split("\n")
    lines[4] = edit
    check("\n".join(lines), "csv")


@pytest.mark.parametrize("text,fmt", [("", "csv"), ("index,t_us,kind,var\n", "csv"), ("", "jsonl"),
                                       ("\n\n", "jsonl"), ('{"a":1}\r{"b":2}', "jsonl"),
                                       ('{"index":0,"t_us":0,"kind":"malloc","var":"a b","size":1}', "jsonl")])
def test_whole_file_cases(text, fmt):
    check(text, fmt)


def test_invalid_utf8_raises_like_the_reference():
    with pytest.raises(UnicodeDecodeError):
        T.read_trace_arrays(b'{"index":0,"t_us":0,"kind":"malloc","var":"\xff","size":1}\n', "jsonl")


def test_threaded_chunks_match_single_thread():
    arrays, _ = workloads.interval_trace(nvars=50000, seed=3, accesses=True)
    text = T.serialize_trace(arrays.to_trace(), "jsonl")
    one = T.read_trace_arrays(text, "jsonl", threads=1)
    many = T.read_trace_arrays(text, "jsonl", threads=8)
    same(one, many)
    same(one, arrays)


def test_parse_and_load_use_the_reader(tmp_path):
    tr = TRACES[0]
    for fmt in ("jsonl", "csv"):
        path = tmp_path / f"t.{fmt}"
        T.save_trace(tr, path)
        same(T.load_trace_arrays(path), T.as_arrays(tr))


def test_native_event_columns_match_python():
    """csrc/evconv.c fills the same columns as the Python conversion, and any
    event outside the plain form hands the whole list to the Python path
    (same values, same errors)."""
    import random
    from paper_1903_06631_b200 import _evconv  # noqa: F401  (built by build())
    rng = random.Random(3)
    kinds = list(T.EventKind)
    ev = [T.TraceEvent(i, rng.randrange(10 ** 6), kinds[rng.randrange(4)], f"v{rng.randrange(300)}",
                       rng.randrange(1 << 40)) for i in range(5000)]
    ev.append(T.TraceEvent(5000, 7, "free", "v1", True))  # plain str kind, bool size
    native = T._native_columns(ev, len(ev))
    assert native is not None
    py = T._python_columns(ev, len(ev))
    for x, y in zip(native[:5], py[:5]):
        assert np.array_equal(x, y)
    assert list(native[5].items()) == list(py[5].items())
    a = T._events_to_arrays(ev)
    odd = list(ev)
    odd[10] = T.TraceEvent(10, odd[10].t_us, odd[10].kind, odd[10].var, np.int64(odd[10].size))
    assert T._native_columns(odd, len(odd)) is None
    b = T._events_to_arrays(odd)
    for f in ("kind", "var", "size", "t_us"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    assert a.names == b.names
    bad = list(ev)
    bad[3] = T.TraceEvent(3, 0, "bogus", "v1", 1)
    with pytest.raises(ValueError):
        T._events_to_arrays(bad)
