"""Device pool path vs the reference's golden vectors (bit-exact).

validate_trace -> detect_iteration -> extract_lifetimes -> conflict graph
-> plan_pool (both policies), all through libmemplan_b200.so on the GPU.
"""
import numpy as np
import pytest

from golden_util import canon_adj, canon_profile, load, pack, trace_arrays

pytestmark = pytest.mark.gpu

GROUPS = ("hand", "generator", "configs", "periodic", "interval")


def _params():
    for g in GROUPS:
        for sc in load(g):
            yield pytest.param(g, sc["name"], id=f"{g}:{sc['name']}")


def _get(g, name):
    return next(s for s in load(g) if s["name"] == name)


@pytest.mark.parametrize("group,name", list(_params()))
def test_device_pool_path_matches_reference(group, name):
    from paper_1903_06631_b200 import _native as N
    from paper_1903_06631_b200.errors import InvariantViolation, PeriodNotFound
    sc = _get(group, name)
    arrays = trace_arrays(sc)
    try:
        N.validate(arrays)
        got = None
    except InvariantViolation as ex:
        got = ["InvariantViolation", ex.index, ex.reason]
    assert got == sc["validate"]
    if "detect" not in sc and "window" not in sc:
        return
    if "detect" in sc:
        if isinstance(sc["detect"][0], str):
            with pytest.raises(PeriodNotFound):
                N.detect(arrays)
            return
        p = N.detect(arrays)
        assert [p, len(arrays) - p, len(arrays)] == sc["detect"]
    start, end = sc["window"]
    if isinstance(sc["profile"], list):
        with pytest.raises(InvariantViolation) as ei:
            N.extract(arrays, start, end)
        assert ["InvariantViolation", ei.value.index, ei.value.reason] == sc["profile"]
        return
    dp = N.extract(arrays, start, end)
    fp = N.download_profile(dp, arrays.names, arrays.name_blob, arrays.name_off, (start, end))
    assert canon_profile(fp) == sc["profile"]
    g = N.conflict_from_profile(dp)
    row, col = N.graph_csr(g)
    assert canon_adj(row, col, fp.nvars) == {k: sc["graph"][k] for k in ("edges", "adj")}
    for pol, code in (("best_fit", 1), ("first_fit", 0)):
        offs, foot, _levels = N.plan_pool(g, code, fp.nvars)
        assert pack(offs.tolist()) == sc["plans"][pol]["offsets"], pol
        assert foot == sc["plans"][pol]["footprint"]


@pytest.mark.parametrize("name", [s["name"] for s in load("arcs")])
def test_device_arcs_match_reference(name):
    from paper_1903_06631_b200 import _native as N
    sc = _get("arcs", name)
    arcs = sc["arcs"]
    n = len(arcs)
    # placement tie-break after -size: (alloc, name) rank
    order = sorted(range(n), key=lambda i: (arcs[i][2], arcs[i][0]))
    tie = np.zeros(n, np.int64)
    tie[order] = np.arange(n)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(a[3]) for a in arcs])
    lo = np.array([s[0] for a in arcs for s in a[3]] or [0], np.int32)
    hi = np.array([s[1] for a in arcs for s in a[3]] or [0], np.int32)
    g = N.conflict_from_arcs([a[1] for a in arcs], tie, off, lo, hi)
    row, col = N.graph_csr(g)
    assert canon_adj(row, col, n) == {k: sc["graph"][k] for k in ("edges", "adj")}
    for pol, code in (("best_fit", 1), ("first_fit", 0)):
        offs, foot, _ = N.plan_pool(g, code, n)
        assert pack(offs.tolist()) == sc["plans"][pol]["offsets"], pol
        assert foot == sc["plans"][pol]["footprint"]


@pytest.mark.parametrize("seed", range(6))
def test_plan_arrays_paths_match_oracle(seed):
    """plan_arrays through the one-CTA path (small traces) and the grid path
    give the oracle's plan (pipeline.py)."""
    import oracle as orc
    from paper_1903_06631_b200 import workloads
    from paper_1903_06631_b200.pipeline import plan_arrays
    from paper_1903_06631_b200.trace import as_arrays
    tr = workloads.random_periodic_trace(seed, slots=40, nvars=12, iterations=5)
    arrays = as_arrays(tr)
    for policy, code in (("best_fit", 1), ("first_fit", 0)):
        rc, p = orc.detect(arrays)
        rc, fp = orc.extract(arrays, len(arrays) - p, len(arrays))
        off, lo, hi = orc.profile_segments(fp)
        h, _r, _c = orc.conflict(off, lo, hi)
        rc, offs, foot = orc.plan(h, fp.size, fp.alloc.astype(np.int64), fp.base, fp.name_ralloc(), fp.name_blob,
                                  fp.name_off, code)
        orc.graph_free(h)
        for path in ("cta", "grid"):
            plan = plan_arrays(arrays, policy=policy, path=path)
            assert np.array_equal(plan.offsets, offs), (path, policy)
            assert plan.footprint_bytes == foot and plan.peak_bytes == fp.peak_bytes and plan.period == p


@pytest.mark.parametrize("seed,wide", [(0, False), (1, True), (2, True)])
def test_grid_placement_both_record_layouts(seed, wide):
    """The grid placement gathers predecessors from 16-byte records when every
    size fits 32 bits and from the offset/level/size arrays otherwise
    (placement.cu pred_range); both give the oracle's plan.  `wide` scales
    the sizes past 2^32."""
    import oracle as orc
    from paper_1903_06631_b200 import workloads
    from paper_1903_06631_b200.pipeline import plan_arrays
    from paper_1903_06631_b200.trace import TraceArrays, as_arrays
    a = as_arrays(workloads.random_periodic_trace(seed, slots=40, nvars=12, iterations=5))
    size = np.array(a.size)
    if wide:
        size = size * ((1 << 33) // max(1, int(size.max())) + 1)
        assert size.max() >= 1 << 32
    else:
        assert size.max() < 1 << 32
    arrays = TraceArrays.from_blob(np.array(a.kind), np.array(a.var), size, np.array(a.t_us), a.name_blob, a.name_off)
    rc, p = orc.detect(arrays)
    rc, fp = orc.extract(arrays, len(arrays) - p, len(arrays))
    off, lo, hi = orc.profile_segments(fp)
    h, _r, _c = orc.conflict(off, lo, hi)
    rc, offs, foot = orc.plan(h, fp.size, fp.alloc.astype(np.int64), fp.base, fp.name_ralloc(), fp.name_blob,
                              fp.name_off, 1)
    orc.graph_free(h)
    plan = plan_arrays(arrays, policy="best_fit", path="grid")
    assert np.array_equal(plan.offsets, offs)
    assert plan.footprint_bytes == foot
