"""SwapPlanner(score="bo") with the batched device objective
(mp_swap_eval_weights) against the reference's own BO runs
(tests/golden/bo.json.gz): same tuned weights, selection and result."""
import numpy as np
import pytest

from golden_util import fhex, load, trace_arrays
from paper_1903_06631_b200 import SwapPlanner, autoswap, extract_lifetimes, detect_iteration, swapsim
from paper_1903_06631_b200.autoswap import ScoreWeights, TransferModel
from paper_1903_06631_b200.errors import LimitUnreachable, SwapDeadlock

pytestmark = pytest.mark.gpu

SCEN = load("bo")


def profile_of(sc):
    arrays = trace_arrays(sc)
    tr = arrays.to_trace()
    det = detect_iteration(tr)
    return extract_lifetimes(tr, det.window)


@pytest.mark.parametrize("idx", range(len(SCEN)), ids=[s["name"] for s in SCEN])
def test_bo_matches_reference(idx):
    sc = SCEN[idx]
    prof = profile_of(sc)
    for run in sc["runs"]:
        sp = SwapPlanner(limit_bytes=run["limit"], score="bo", threshold_bytes=run["threshold"],
                         bandwidth_bytes_per_s=float.fromhex(run["bw"]), latency_us=float.fromhex(run["lat"]),
                         bo_budget=run["budget"], seed=run["seed"])
        if "error" in run:
            exp = {"LimitUnreachable": LimitUnreachable, "SwapDeadlock": SwapDeadlock}[run["error"][0]]
            with pytest.raises(exp):
                sp.fit(prof)
            continue
        sp.fit(prof)
        assert [fhex(x) for x in sp.weights_.as_tuple()] == run["weights"]
        assert [c.var for c in sp.selection_] == run["selection"]
        assert fhex(sp.overhead_us_) == run["overhead_us"]
        assert sp.achieved_peak_bytes_ == run["achieved"]


def test_batched_objective_equals_the_scalar_path():
    sc = next(s for s in SCEN if s["name"].startswith("vgg_like_d6"))
    prof = profile_of(sc)
    limit = int(prof.load.peak_bytes * 0.88)
    cands = autoswap.filter_candidates(prof, threshold_bytes=1 << 20, transfer=TransferModel(1e9, 5.0))

    def scalar(w):
        sel = autoswap.select_by_score(cands, prof, limit, score="combined", weights=w)
        return swapsim.simulate(swapsim.build_schedule(sel, prof), prof, limit).overhead_us

    ev = autoswap.WeightEvaluator(cands, prof, limit, scalar)
    rng = np.random.default_rng(0)
    ws = [ScoreWeights(*(round(float(v), 9) for v in rng.uniform(-1, 1, 4))) for _ in range(48)]
    ws += [ScoreWeights(1.0, 0.0, 0.0, 0.0), ScoreWeights(0.0, 0.0, 0.0, 1.0)]
    from paper_1903_06631_b200 import _native as N
    from paper_1903_06631_b200.iteration import device_profile
    w = np.array([x.as_tuple() for x in ws])
    st, ov, _ns, _ax = N.swap_eval_weights(device_profile(prof), autoswap._cands(cands), ev.z, w, limit)
    kinds = set()
    for i, wt in enumerate(ws):
        try:
            want = ("ok", fhex(scalar(wt)))
        except (LimitUnreachable, SwapDeadlock, IndexError) as e:
            want = (type(e).__name__,)
        got = ("ok", fhex(ov[i])) if st[i] == 0 else ({3: "LimitUnreachable", 4: "SwapDeadlock", 5: "IndexError"}[int(st[i])],)
        assert got == want, (i, wt, got, want)
        kinds.add(got[0])
    assert "ok" in kinds
    ok = [x for i, x in enumerate(ws) if st[i] == 0]
    assert [fhex(y) for y in ev(ok)] == [fhex(scalar(x)) for x in ok] and ev.launches == 1
