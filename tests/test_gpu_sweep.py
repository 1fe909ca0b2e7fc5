"""Device sweep (csrc/sweep.cu, one CTA per trace) against the reference's
golden units and the CPU oracle — bit for bit on every record."""
import numpy as np
import pytest

import oracle as orc
from golden_util import check_sweep_unit, load, sweep_params, trace_arrays
from paper_1903_06631_b200 import sweep, workloads
from paper_1903_06631_b200.errors import LimitUnreachable, SwapDeadlock

pytestmark = pytest.mark.gpu

SCEN = load("sweep")


def _by_params():
    groups = {}
    for sc in SCEN:
        groups.setdefault(sc["params"]["name"], []).append(sc)
    return groups


def compare_with_oracle(batch, res, params):
    recs, brecs, offs, orders = orc.sweep(batch, params)
    bad = []
    for t in range(batch.ntraces):
        same = (res.traces[t].tobytes() == recs[t].tobytes()
                and res.budgets[t].tobytes() == brecs[t].tobytes()
                and np.array_equal(res.offsets_of(t), offs[t])
                and np.array_equal(res.order_of(t), orders[t]))
        if not same:
            bad.append(t)
    assert not bad, f"{len(bad)} units differ, first {bad[:5]}"


@pytest.mark.parametrize("pname", sorted(_by_params()))
def test_sweep_matches_reference_golden(pname):
    scs = _by_params()[pname]
    batch = sweep.SweepBatch.from_traces([trace_arrays(sc) for sc in scs])
    params = sweep_params(scs[0]["params"])
    res = sweep.run_sweep(batch, params)
    for t, sc in enumerate(scs):
        check_sweep_unit(res.traces[t], res.budgets[t], res.offsets_of(t), res.order_of(t), sc["unit"])
    compare_with_oracle(batch, res, params)


@pytest.mark.parametrize("policy,bw", [("best_fit", 12e9), ("first_fit", 1e9)])
def test_sweep_config5_matches_oracle(policy, bw):
    batch = sweep.SweepBatch.from_traces(workloads.sweep_traces())
    params = sweep.SweepParams(budgets=workloads.SWEEP_BUDGETS, policy=policy, bandwidth_bytes_per_s=bw)
    res = sweep.run_sweep(batch, params)
    assert batch.ntraces == 1024 and res.budgets.shape == (1024, 4)
    compare_with_oracle(batch, res, params)


def test_sweep_random_periodic_matches_oracle():
    import random
    traces = []
    for seed in range(160):
        rng = random.Random(seed)
        kw = dict(slots=rng.choice((12, 24, 40, 64)), nvars=rng.randrange(2, 16),
                  iterations=rng.randrange(4, 7), max_wrap=rng.choice((0.9, 1.5, 2.2, 3.0)),
                  n_persistent=rng.randrange(0, 3), n_leak=rng.randrange(0, 2),
                  n_reuse=rng.randrange(0, 3), zero_dt=rng.choice((0.0, 0.2, 0.5)))
        traces.append(workloads.random_periodic_trace(seed, **kw))
    batch = sweep.SweepBatch.from_traces(traces)
    for params in (sweep.SweepParams(budgets=(0.9, 0.75, 0.6), threshold_bytes=1),
                   sweep.SweepParams(budgets=(1.0, 0.8, 0.5, 0.3, 0.1, 0.05, 0.01, 0.0), policy="first_fit",
                                     threshold_bytes=1000, bandwidth_bytes_per_s=1e9, latency_us=1.0)):
        res = sweep.run_sweep(batch, params)
        compare_with_oracle(batch, res, params)


def test_sweep_edges_and_resident_reruns():
    traces = workloads.sweep_traces(n_models=4, n_scales=2)
    batch = sweep.SweepBatch.from_traces(traces)
    # no budgets, unvalidated: pool plans only
    res = sweep.run_sweep(batch, sweep.SweepParams(budgets=(), validate=False))
    assert res.budgets.shape == (8, 0) and (res.traces["status"] == 0).all()
    compare_with_oracle(batch, res, sweep.SweepParams(budgets=(), validate=False))
    # one upload, several parameter sets; repeated runs are identical
    ds = sweep.DeviceSweep(batch)
    outs = []
    for params in (sweep.SweepParams(), sweep.SweepParams(policy="first_fit"), sweep.SweepParams()):
        ds.run(params)
        outs.append(ds.download())
        compare_with_oracle(batch, outs[-1], params)
    assert outs[0].traces.tobytes() == outs[2].traces.tobytes()
    assert outs[0].budgets.tobytes() == outs[2].budgets.tobytes()
    ds.close()
    # an empty batch
    empty = sweep.run_sweep(sweep.SweepBatch.from_traces([]), sweep.SweepParams())
    assert empty.traces.shape == (0,)


def test_sweep_errors_map_to_reference_exceptions():
    scs = _by_params()["slow_link"]
    batch = sweep.SweepBatch.from_traces([trace_arrays(sc) for sc in scs])
    res = sweep.run_sweep(batch, sweep_params(scs[0]["params"]))
    kinds = set()
    for t, sc in enumerate(scs):
        u = sc["unit"]
        if "error" in u:
            with pytest.raises(Exception) as ei:
                res.raise_for(t)
            kinds.add(type(ei.value).__name__)
            continue
        res.raise_for(t)
        for b, g in enumerate(u["budgets"]):
            if "error" not in g:
                res.raise_for(t, b)
                continue
            exp = {"ValueError": ValueError, "LimitUnreachable": LimitUnreachable,
                   "SwapDeadlock": SwapDeadlock, "IndexError": IndexError}[g["error"][0]]
            with pytest.raises(exp) as ei:
                res.raise_for(t, b)
            if exp is LimitUnreachable:
                assert ei.value.limit_bytes == g["error"][1] and ei.value.achievable_bytes == g["error"][2]
            kinds.add(exp.__name__)
    assert {"InvariantViolation", "PeriodNotFound", "LimitUnreachable", "SwapDeadlock"} <= kinds


def test_sweep_sharded_runner_matches_single_device():
    batch = sweep.SweepBatch.from_traces(workloads.sweep_traces(n_models=8, n_scales=3))
    params = sweep.SweepParams()
    whole = sweep.run_sweep(batch, params)
    # every rank's share run on this device, reassembled like rank 0 does
    parts = sweep.shard([batch.events_of(t) for t in range(batch.ntraces)], 4)
    got = sweep.concat_results([(p, sweep.run_sweep(batch.subset(p), params)) for p in parts], batch)
    assert got.traces.tobytes() == whole.traces.tobytes()
    assert got.budgets.tobytes() == whole.budgets.tobytes()
    for t in range(batch.ntraces):
        assert np.array_equal(got.offsets_of(t), whole.offsets_of(t))
        assert np.array_equal(got.order_of(t), whole.order_of(t))


def test_sweep_detect_with_rejected_quick_survivors():
    """Traces whose last 16 fingerprints reappear at several distances: each
    distance passes the sweep's quick filter and fails the exact check (up to
    5 times, past the 4 quick rounds into the warp-per-candidate search);
    the period and every record must equal the oracle's."""
    from paper_1903_06631_b200.trace import TraceArrays
    traces = []
    for ncopies in (0, 1, 3, 5):
        rng = np.random.default_rng(100 + ncopies)
        L = 200
        sizes = rng.integers(1, 1 << 40, L)
        tail = sizes[L - 16:].copy()
        for s in (30, 50, 70, 90, 110)[:ncopies]:
            sizes[L - s - 16:L - s] = tail
        for reps in (2, 3):
            n = L * reps
            kinds = np.zeros(n, np.uint8)       # all mallocs of distinct fresh names
            sz = np.tile(sizes, reps)
            names = [f"x{i}" for i in range(n)]
            # free each variable right after its malloc so the trace is valid
            k2 = np.repeat(kinds, 2)
            k2[1::2] = 1
            s2 = np.repeat(sz, 2)
            s2[1::2] = 0
            n2 = [nm for nm in names for _ in (0, 1)]
            traces.append(TraceArrays.from_columns(k2, n2, s2, np.arange(2 * n, dtype=np.int64)))
    batch = sweep.SweepBatch.from_traces(traces)
    params = sweep.SweepParams(budgets=(0.9, 0.5), threshold_bytes=1)
    res = sweep.run_sweep(batch, params)
    compare_with_oracle(batch, res, params)
    assert all(int(res.traces["period"][t]) == 2 * 200 for t in range(batch.ntraces))
