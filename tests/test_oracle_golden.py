"""Pin the CPU oracle against the reference's golden vectors (CPU-only).

Every scenario in tests/golden/ was produced by the reference package; the
oracle must reproduce each output bit for bit before it is trusted as the
checker of the device path.
"""
import numpy as np
import pytest

import oracle as orc
from golden_util import (ALT_WEIGHTS, DEFAULT_WEIGHTS, SCORE_CODE, canon_adj, canon_cands,
                         canon_curve, canon_profile, canon_schedule, fhex, load, pack,
                         trace_arrays)
from paper_1903_06631_b200._abi import MP_OK, invariant_reason

TRACE_GROUPS = ("hand", "generator", "configs", "periodic", "interval")


def _scenarios(groups):
    for g in groups:
        for sc in load(g):
            if sc["kind"] == "trace":
                yield pytest.param(g, sc["name"], id=f"{g}:{sc['name']}")


def _get(g, name):
    return next(s for s in load(g) if s["name"] == name)


def err_tuple(rc, err, names):
    if rc == 1:
        return ["InvariantViolation", int(err.index), invariant_reason(err, names)]
    if rc == 2:
        return "PeriodNotFound"
    return rc


def check_swap(fp, blk):
    bw, lat = float.fromhex(blk["bw"]), float.fromhex(blk["lat"])
    c = orc.candidates(fp, blk["threshold"], bw, lat)
    assert canon_cands(c, fp) == blk["candidates"]
    load_ = orc._load(fp)
    names = orc.names_of(fp)
    assert orc.load_min(load_, c) == blk["load_min"]
    cnames = [fp.var_name(v) for v in c.var.tolist()]
    if c.k:
        (doa, aoa, wdoa, sw), order = orc.scores(load_, c, names)
        got = [[fhex(doa[i]), fhex(aoa[i]), fhex(wdoa[i]), fhex(sw[i])] for i in range(c.k)]
        assert got == blk["scores"]
        assert [cnames[i] for i in order] == blk["swdoa_order"]
    for run in blk["runs"]:
        w = ALT_WEIGHTS if run["score"] == "combined_w" else DEFAULT_WEIGHTS
        rc, err, sel = orc.select(load_, c, names, SCORE_CODE[run["score"]], w, run["limit"])
        if rc != MP_OK:
            assert run["selection"] == ["LimitUnreachable", int(err.aux0), int(err.aux1)], run
            continue
        assert [cnames[i] for i in sel] == run["selection"], run
        (so, eo, si, ei), order = orc.schedule(fp, c, names, sel)
        assert canon_schedule(cnames, sel.tolist(), so, eo, si, ei, order.tolist(), c.size,
                              fp.duration_us) == run["schedule"], run
        rc, err, res = orc.simulate(fp, c, names, sel, ((so, eo, si, ei), order), run["limit"])
        if rc == 4:
            reason = "no pending swap-out can free space" if err.aux0 == 0 else \
                f"swap-in of {cnames[int(err.aux1)]!r} cannot start"
            assert run["sim"] == ["SwapDeadlock", int(err.index), reason], run
            continue
        if rc == 5:
            assert run["sim"] == ["IndexError"], run
            continue
        assert rc == MP_OK
        sim = run["sim"]
        assert isinstance(sim, dict), (run, rc)
        d = fp.duration_us
        assert sim["overhead_us"] == fhex(res["delay"])
        assert sim["duration"] == fhex(d + res["delay"])
        assert sim["overhead_pct"] == fhex(res["delay"] / d * 100.0 if d > 0 else 0.0)
        assert sim["rounds"] == res["rounds"]
        assert sim["peak"] == res["ldp"][2]
        assert sim["delayed"] == pack([[int(i), fhex(u)] for i, u in zip(*res["delayed"])])
        assert sim["load_prime"] == canon_curve(*res["lp"])
        assert sim["load_double_prime"] == canon_curve(*res["ldp"])
        assert sim["schedule"] == canon_schedule(cnames, sel.tolist(), res["t_so"], res["t_eo"],
                                                 res["t_si"], res["t_ei"],
                                                 res["event_order"].tolist(), c.size, d)


@pytest.mark.parametrize("group,name", list(_scenarios(TRACE_GROUPS)))
def test_oracle_matches_reference(group, name):
    sc = _get(group, name)
    arrays = trace_arrays(sc)
    rc, err = orc.validate(arrays)
    want = sc["validate"]
    assert (None if rc == MP_OK else err_tuple(rc, err, arrays.names)) == want
    if "detect" not in sc and "window" not in sc:
        return
    if "detect" in sc:
        rc, p = orc.detect(arrays)
        got = [p, len(arrays) - p, len(arrays)] if rc == MP_OK else None
        if isinstance(sc["detect"][0], str):
            assert rc == 2
            return
        assert got == sc["detect"]
        if len(arrays) <= 20000:
            assert orc.detect(arrays, naive=True) == (rc, p)
    start, end = sc["window"]
    rc, fp = orc.extract(arrays, start, end)
    if isinstance(sc["profile"], list):
        assert rc != MP_OK and err_tuple(rc, fp, arrays.names) == sc["profile"]
        return
    assert rc == MP_OK
    assert canon_profile(fp) == sc["profile"]
    off, lo, hi = orc.profile_segments(fp)
    h, row, col = orc.conflict(off, lo, hi)
    assert canon_adj(row, col, fp.nvars) == {k: sc["graph"][k] for k in ("edges", "adj")}
    ralloc = fp.name_ralloc()
    for pol, code in (("best_fit", 1), ("first_fit", 0)):
        rc, offs, foot = orc.plan(h, fp.size, fp.alloc.astype(np.int64), fp.base, ralloc,
                                  fp.name_blob, fp.name_off, code)
        assert rc == MP_OK
        assert pack(offs.tolist()) == sc["plans"][pol]["offsets"]
        assert foot == sc["plans"][pol]["footprint"]
    orc.graph_free(h)
    for blk in sc.get("swap", []):
        check_swap(fp, blk)


@pytest.mark.parametrize("name", [s["name"] for s in load("arcs")])
def test_oracle_arcs(name):
    sc = _get("arcs", name)
    arcs = sc["arcs"]
    names = sorted({a[0] for a in arcs})
    rank = {n: i for i, n in enumerate(names)}
    blob = np.frombuffer("".join(names).encode() or b"\0", np.uint8).copy()
    noff = np.zeros(len(names) + 1, np.int64)
    noff[1:] = np.cumsum([len(n.encode()) for n in names])
    off = np.zeros(len(arcs) + 1, np.int64)
    off[1:] = np.cumsum([len(a[3]) for a in arcs])
    lo = [s[0] for a in arcs for s in a[3]]
    hi = [s[1] for a in arcs for s in a[3]]
    h, row, col = orc.conflict(off, lo, hi)
    assert canon_adj(row, col, len(arcs)) == {k: sc["graph"][k] for k in ("edges", "adj")}
    size = [a[1] for a in arcs]
    alloc = [a[2] for a in arcs]
    nb = [rank[a[0]] for a in arcs]
    for pol, code in (("best_fit", 1), ("first_fit", 0)):
        rc, offs, foot = orc.plan(h, size, alloc, nb, [-1] * len(arcs), blob, noff, code)
        assert pack(offs.tolist()) == sc["plans"][pol]["offsets"]
        assert foot == sc["plans"][pol]["footprint"]
    orc.graph_free(h)


def _synthetic(sc):
    from paper_1903_06631_b200._abi import FlatProfile, MpProfileDims  # noqa: F401
    loads = np.array(sc["loads"], np.int64)
    p = loads.shape[0]
    sp = float.fromhex(sc["spacing"])
    times = np.array([sp * r for r in range(p)], np.float64)
    load_ = orc.Load(p, orc.ptr(loads), orc.ptr(times), sp * p)
    cs = sc["cands"]
    names = sorted({c[0] for c in cs})
    rank = {n: i for i, n in enumerate(names)}
    blob = np.frombuffer("".join(names).encode(), np.uint8).copy()
    noff = np.zeros(len(names) + 1, np.int64)
    noff[1:] = np.cumsum([len(n) for n in names])
    f = lambda j, conv=None: [conv(c[j]) if conv else c[j] for c in cs]  # noqa: E731
    hx = float.fromhex
    ca = orc.CandArrays(len(cs), var=list(range(len(cs))), size=f(1), out_index=f(2),
                        out_t=f(3, hx), out_ready=f(4, hx), in_index=f(5), in_t=f(6, hx),
                        dout=f(7, hx), din=f(8, hx), spans=f(9, int),
                        name_base=[rank[c[0]] for c in cs], name_ralloc=[-1] * len(cs))
    return loads, times, load_, ca, orc.names_of(blob, noff), [c[0] for c in cs]


@pytest.mark.parametrize("name", [s["name"] for s in load("synthetic")])
def test_oracle_synthetic_scores(name):
    sc = _get("synthetic", name)
    loads, times, load_, ca, names, cn = _synthetic(sc)
    (doa, aoa, wdoa, sw), order = orc.scores(load_, ca, names)
    assert [fhex(x) for x in wdoa] == sc["wdoa"]
    assert [fhex(x) for x in doa] == sc["doa"]
    assert [fhex(x) for x in aoa] == sc["aoa"]
    assert [fhex(x) for x in sw] == sc["swdoa"]
    assert orc.load_min(load_, ca) == sc["load_min"]
    for run in sc["runs"]:
        rc, err, sel = orc.select(load_, ca, names, SCORE_CODE[run["score"]], DEFAULT_WEIGHTS,
                                  run["limit"])
        if rc != MP_OK:
            assert run["selection"] == ["LimitUnreachable", int(err.aux0), int(err.aux1)]
        else:
            assert [cn[i] for i in sel] == run["selection"]


def test_standardize_matches_cpython_sum():
    import random
    rng = random.Random(3)
    from paper_1903_06631_b200.errors import MemplanError  # noqa: F401
    for _ in range(3000):
        n = rng.randrange(1, 40)
        xs = [rng.choice((rng.uniform(-1e6, 1e6), rng.randrange(-10**12, 10**12) * 1.0,
                          rng.uniform(-1, 1) * 10 ** rng.randrange(-30, 30))) for _ in range(n)]
        mean = sum(xs) / n
        var = sum((x - mean) ** 2 for x in xs) / n
        want = [0.0] * n if var <= 0 else [(x - mean) / var ** 0.5 for x in xs]
        got = orc.standardize(xs).tolist()
        assert [fhex(a) for a in got] == [fhex(b) for b in want]
