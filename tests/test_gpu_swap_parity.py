"""Device swap path vs the reference's golden vectors (bit-exact).

filter_candidates, the four scores and the SWDOA order, select_by_score for
every score at every limit, build_schedule, simulate (LOAD', LOAD'',
delayed ops, overhead, rounds, final schedule, deadlock / IndexError
parity) and compute_load_min, all through libmemplan_b200.so.
"""
import numpy as np
import pytest

from golden_util import (ALT_WEIGHTS, DEFAULT_WEIGHTS, canon_cands, canon_curve, canon_schedule, fhex, load,
                         pack, trace_arrays)

pytestmark = pytest.mark.gpu

GROUPS = ("hand", "generator", "configs", "periodic", "interval")


def _params():
    for g in GROUPS:
        for sc in load(g):
            if sc.get("swap"):
                yield pytest.param(g, sc["name"], id=f"{g}:{sc['name']}")


def _get(g, name):
    return next(s for s in load(g) if s["name"] == name)


def ranks(names):
    order = sorted(range(len(names)), key=lambda i: names[i])
    r = np.zeros(len(names), np.int32)
    r[order] = np.arange(len(names))
    return r


@pytest.mark.parametrize("group,name", list(_params()))
def test_device_swap_path_matches_reference(group, name):
    from paper_1903_06631_b200 import _native as N
    from paper_1903_06631_b200.errors import LimitUnreachable, SwapDeadlock
    sc = _get(group, name)
    arrays = trace_arrays(sc)
    start, end = sc["window"]
    dp = N.extract(arrays, start, end)
    fp = N.download_profile(dp, arrays.names, arrays.name_blob, arrays.name_off, (start, end))
    vnames = fp.var_names()
    for blk in sc["swap"]:
        bw, lat = float.fromhex(blk["bw"]), float.fromhex(blk["lat"])
        c = N.swap_candidates(dp, fp.nvars, blk["threshold"], bw, lat)
        cnames = [vnames[v] for v in c.var.tolist()]
        c.name_rank = ranks(cnames) if c.k else np.zeros(1, np.int32)
        assert canon_cands(c, fp) == blk["candidates"]
        assert int(N.swap_planned_peak(dp, c)) == blk["load_min"]
        if c.k:
            (doa, aoa, wdoa, sw), order, peaks = N.swap_scores(dp, c)
            got = [[fhex(doa[i]), fhex(aoa[i]), fhex(wdoa[i]), fhex(sw[i])] for i in range(c.k)]
            assert got == blk["scores"]
            assert [cnames[i] for i in order] == blk["swdoa_order"]
            raw = {"doa": doa, "aoa": aoa, "wdoa": wdoa, "swdoa": sw}
        for run in blk["runs"]:
            score, limit = run["score"], run["limit"]
            try:
                if not c.k:
                    sel = np.zeros(0, np.int32)
                    if fp.loads.max() > limit:
                        raise LimitUnreachable(limit, int(fp.loads.max()))
                elif score == "swdoa":
                    # budgeted greedy = prefix of the unbudgeted order
                    j = next((j for j in range(c.k + 1) if peaks[j] <= limit), None)
                    if j is None:
                        raise LimitUnreachable(limit, int(peaks[c.k]))
                    sel = order[:j]
                else:
                    if score in ("combined", "combined_w"):
                        w = ALT_WEIGHTS if score == "combined_w" else DEFAULT_WEIGHTS
                        ranked = np.zeros(c.k)
                        for wi, nm in zip(w, ("aoa", "doa", "wdoa", "swdoa")):
                            ranked = ranked + wi * N.standardize(raw[nm])
                    else:
                        ranked = raw[score]
                    sel = N.swap_select_static(dp, c, ranked, limit)
            except LimitUnreachable as ex:
                assert run["selection"] == ["LimitUnreachable", ex.limit_bytes, ex.achievable_bytes], run
                continue
            assert [cnames[i] for i in sel] == run["selection"], run
            sel = np.asarray(sel, np.int32)
            (so, eo, si, ei), evo = N.swap_schedule(c, sel, c.out_ready[sel], c.in_t[sel])
            assert canon_schedule(cnames, sel.tolist(), so, eo, si, ei, evo.tolist(), c.size,
                                  fp.duration_us) == run["schedule"], run
            try:
                res = N.swap_simulate(dp, fp.period, c, sel, ((so, eo, si, ei), evo), limit,
                                      cand_names=cnames)
            except SwapDeadlock as ex:
                assert run["sim"] == ["SwapDeadlock", ex.index, ex.reason], run
                continue
            except IndexError:
                assert run["sim"] == ["IndexError"], run
                continue
            sim = run["sim"]
            assert isinstance(sim, dict), run
            d = fp.duration_us
            assert sim["overhead_us"] == fhex(res["delay"])
            assert sim["rounds"] == res["rounds"]
            assert sim["peak"] == res["ldp"][2]
            assert sim["delayed"] == pack([[int(i), fhex(u)] for i, u in zip(*res["delayed"])])
            assert sim["load_prime"] == canon_curve(*res["lp"])
            assert sim["load_double_prime"] == canon_curve(*res["ldp"])
            assert sim["schedule"] == canon_schedule(cnames, sel.tolist(), res["t_so"], res["t_eo"], res["t_si"],
                                                     res["t_ei"], res["event_order"].tolist(), c.size, d)
