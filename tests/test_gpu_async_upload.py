"""The overlapped upload path of plan_arrays (asynchronous per-column upload,
structure validated before extraction, timestamps after the plan) reports
exactly what the reference's validate -> detect -> extract order reports.

The golden scenarios run through plan_arrays(path="grid") on fresh arrays
(so every call uploads asynchronously); injected violations check that a
timestamp violation before a structural one wins, and vice versa.
"""
import numpy as np
import pytest

from golden_util import load, pack, trace_arrays

pytestmark = pytest.mark.gpu

GROUPS = ("hand", "generator", "configs", "periodic", "interval")


def _params():
    for g in GROUPS:
        for sc in load(g):
            yield pytest.param(g, sc["name"], id=f"{g}:{sc['name']}")


def _outcome(arrays):
    from paper_1903_06631_b200.errors import InvariantViolation, PeriodNotFound
    from paper_1903_06631_b200.pipeline import plan_arrays
    try:
        plan = plan_arrays(arrays, path="grid")
    except InvariantViolation as ex:
        return ["InvariantViolation", ex.index, ex.reason]
    except PeriodNotFound:
        return ["PeriodNotFound"]
    return plan


@pytest.mark.parametrize("group,name", list(_params()))
def test_overlapped_plan_matches_reference(group, name):
    sc = next(s for s in load(group) if s["name"] == name)
    got = _outcome(trace_arrays(sc))
    if sc["validate"] is not None:
        assert got == sc["validate"]
        return
    if "detect" in sc and isinstance(sc["detect"][0], str):
        assert got == ["PeriodNotFound"]
        return
    if "detect" not in sc:
        return
    if isinstance(sc["profile"], list):
        assert got == sc["profile"]
        return
    assert not isinstance(got, list), got
    assert [got.period, got.window[0], got.window[1]] == sc["detect"]
    assert pack(got.offsets.tolist()) == sc["plans"]["best_fit"]["offsets"]
    assert got.footprint_bytes == sc["plans"]["best_fit"]["footprint"]


def _valid_trace():
    from paper_1903_06631_b200 import workloads
    arrays, _window = workloads.interval_trace(3000, seed=3)
    return arrays


def _with(arrays, **cols):
    from paper_1903_06631_b200.trace import TraceArrays
    c = {k: np.array(getattr(arrays, k)) for k in ("kind", "var", "size", "t_us")}
    c.update(cols)
    return TraceArrays.from_blob(c["kind"], c["var"], c["size"], c["t_us"], arrays.name_blob, arrays.name_off)


def _first_malloc_after(arrays, pos):
    from paper_1903_06631_b200.trace import KIND_CODE
    k = np.asarray(arrays.kind)
    return int(np.nonzero(k[pos:] == KIND_CODE["malloc"])[0][0]) + pos


def test_valid_trace_plans_through_the_overlapped_path():
    from paper_1903_06631_b200.pipeline import plan_arrays
    a = _valid_trace()
    got = _outcome(a)
    ref = plan_arrays(a, path="grid")  # cached upload, synchronous stages
    assert not isinstance(got, list)
    assert np.array_equal(got.offsets, ref.offsets) and got.footprint_bytes == ref.footprint_bytes


@pytest.mark.parametrize("t_first", [True, False])
def test_first_violation_wins_across_the_split_validation(t_first):
    a = _valid_trace()
    n = len(a)
    t = np.array(a.t_us)
    size = np.array(a.size)
    i_t = n // 3 if t_first else 2 * n // 3
    i_s = _first_malloc_after(a, 2 * n // 3 if t_first else n // 3)
    t[i_t] = t[i_t - 1] - 1        # timestamp decreases (checked before sizes)
    size[i_s] = 0                  # malloc size must be > 0
    got = _outcome(_with(a, t_us=t, size=size))
    assert got[0] == "InvariantViolation"
    assert got[1] == (i_t if t_first else i_s)


def test_timestamp_only_violation_is_reported_after_the_plan():
    a = _valid_trace()
    t = np.array(a.t_us)
    i = len(a) - 5
    t[i] = -1
    got = _outcome(_with(a, t_us=t))
    assert got[0] == "InvariantViolation" and got[1] == i


# ---- period detection: the quick filter's smallest survivor is not a period ----

def _fp_trace(kinds, sizes):
    from paper_1903_06631_b200.trace import TraceArrays
    n = len(kinds)
    return TraceArrays.from_columns(np.array(kinds, np.uint8), [f"v{i % 7}" for i in range(n)],
                                    np.array(sizes, np.int64), np.arange(n, dtype=np.int64))


@pytest.mark.parametrize("shift,reps", [(50, 2), (40, 3), (33, 2), (64, 2)])
def test_detect_when_a_non_period_passes_the_quick_filter(shift, reps):
    """A block whose last 32 events repeat the 32 events `shift` earlier:
    p = shift matches the last 32 pairs (the quick filter's window) but not
    all p of them, so the exact check rejects it and the hash search must
    find the real period (the block length); oracle.detect restates
    iteration.py:93-105."""
    import oracle
    from paper_1903_06631_b200 import _native as N
    from paper_1903_06631_b200.errors import PeriodNotFound
    rng = np.random.default_rng(shift)
    L = 120
    sizes = rng.integers(1, 1 << 40, L)
    sizes[L - 32:] = sizes[L - 32 - shift:L - shift]
    block = [(0, int(x)) for x in sizes]
    ev = block * reps
    arrays = _fp_trace([k for k, _ in ev], [x for _, x in ev])
    rc, want = oracle.detect(arrays)
    assert rc == 0 and want == L
    assert N.detect(arrays) == want
    # and without a real period: the fallback reports none
    arrays = _fp_trace([k for k, _ in block], [x for _, x in block])
    rc, _ = oracle.detect(arrays)
    assert rc != 0
    with pytest.raises(PeriodNotFound):
        N.detect(arrays)
