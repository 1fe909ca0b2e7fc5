"""Drop-in semantics the reference gets for free from being plain Python:

* in-place edits of a Trace / IterationProfile / ConflictGraph between calls
  are seen by the next call (tests/golden/edit_programs.py, answers recorded
  from the reference by make_golden_edits.py);
* concurrent calls from several host threads return what a lone call
  returns (the reference's functions are reentrant).
"""
import gzip
import json
import os
import sys
import threading

import pytest

from golden_util import GOLDEN, load, pack

sys.path.insert(0, GOLDEN)
import edit_programs  # noqa: E402

pytestmark = pytest.mark.gpu


def _golden():
    with gzip.open(os.path.join(GOLDEN, "edits.json.gz"), "rt") as fh:
        return json.load(fh)["programs"]


@pytest.mark.parametrize("name", sorted(edit_programs.PROGRAMS))
def test_edit_program_matches_reference(name):
    import paper_1903_06631_b200 as mp
    got = json.loads(json.dumps(edit_programs.PROGRAMS[name](mp)))
    assert got == _golden()[name]


def _api_run(mp, sc):
    """The public-API pipeline of test_gpu_api_golden on one scenario."""
    from test_gpu_api_golden import canon_profile, to_trace
    trace = to_trace(mp, sc)
    prof = mp.extract_lifetimes(trace, tuple(sc["window"]))
    g = mp.build_conflict_graph(prof)
    out = {"profile": canon_profile(prof) == sc["profile"]}
    for pol in ("best_fit", "first_fit"):
        plan = mp.plan_pool(g, pol)
        out[pol] = (pack([plan.offsets[v.var] for v in g.vars]) == sc["plans"][pol]["offsets"]
                    and plan.footprint_bytes == sc["plans"][pol]["footprint"])
    if isinstance(sc.get("detect"), list) and isinstance(sc["detect"][0], int):
        d = mp.detect_iteration(trace)
        out["detect"] = [d.period, *d.window] == sc["detect"]
    return out


def test_threads_plan_goldens_concurrently():
    """8 host threads, each planning a different golden scenario 3 times
    through the public API on the shared device context."""
    import paper_1903_06631_b200 as mp
    scs = [s for g in ("configs", "generator", "periodic", "hand") for s in load(g)
           if isinstance(s.get("profile"), dict) and "plans" in s][:8]
    assert len(scs) == 8
    results, errors = {}, []
    start = threading.Barrier(len(scs))

    def work(k, sc):
        try:
            start.wait()
            results[k] = [_api_run(mp, sc) for _ in range(3)]
        except Exception as ex:  # noqa: BLE001
            errors.append((sc["name"], repr(ex)))

    threads = [threading.Thread(target=work, args=(k, sc)) for k, sc in enumerate(scs)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(600)
    assert not errors, errors
    for k, sc in enumerate(scs):
        for run in results[k]:
            assert all(run.values()), (sc["name"], run)


def test_threads_validate_goldens_concurrently():
    """Concurrent validate/detect on traces with and without violations:
    each thread's error (index, reason) is its own."""
    import paper_1903_06631_b200 as mp
    from test_gpu_api_golden import to_trace
    scs = [s for s in load("hand") if "trace" in s]
    want = {sc["name"]: None if sc["validate"] is None else tuple(sc["validate"][1:]) for sc in scs}
    assert any(w is not None for w in want.values())
    got, errors = {}, []

    def work(sc):
        try:
            for _ in range(5):
                try:
                    mp.validate_trace(to_trace(mp, sc))
                    r = None
                except mp.InvariantViolation as ex:
                    r = (ex.index, ex.reason)
                got.setdefault(sc["name"], []).append(r)
        except Exception as ex:  # noqa: BLE001
            errors.append(repr(ex))

    threads = [threading.Thread(target=work, args=(sc,)) for sc in scs]
    for t in threads:
        t.start()
    for t in threads:
        t.join(600)
    assert not errors, errors
    for name, rs in got.items():
        assert all(r == want[name] for r in rs), (name, rs, want[name])
