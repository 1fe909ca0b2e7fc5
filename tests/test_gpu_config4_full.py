"""Config 4 at full size (BASELINE.json configs[3]): the 1,000,001-variable
interval trace (4,000,008 events) planned by the device path, compared with
the C oracle offset for offset, and with the reference's own measurement
(peak 1,876,335,040 B, best-fit footprint 2,015,985,620 B,
31,978,487 conflict edges)."""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF_PEAK = 1_876_335_040
REF_BEST_FIT_FOOTPRINT = 2_015_985_620
REF_EDGES = 31_978_487


@pytest.fixture(scope="module")
def workload():
    from paper_1903_06631_b200 import workloads
    arrays, window = workloads.interval_trace(1_000_000, seed=0)
    return arrays, window


@pytest.fixture(scope="module")
def oracle_profile(workload):
    import oracle as orc
    arrays, window = workload
    rc, fp = orc.extract(arrays, window[0], window[1])
    assert rc == 0
    off, lo, hi = orc.profile_segments(fp)
    h, row, col = orc.conflict(off, lo, hi)
    yield fp, h, row
    orc.graph_free(h)


@pytest.mark.parametrize("policy,code", [("best_fit", 1), ("first_fit", 0)])
def test_config4_full_size_matches_oracle_and_reference(workload, oracle_profile, policy, code):
    import oracle as orc
    from paper_1903_06631_b200.pipeline import plan_arrays
    arrays, window = workload
    fp, h, row = oracle_profile
    plan = plan_arrays(arrays, policy=policy)
    assert plan.period == window[1] - window[0]
    assert plan.nvars == fp.nvars == 1_000_001
    assert plan.peak_bytes == fp.peak_bytes == REF_PEAK
    assert plan.nnz == int(row[-1]) == 2 * REF_EDGES
    rc, offs, foot = orc.plan(h, fp.size, fp.alloc.astype(np.int64), fp.base, fp.name_ralloc(), fp.name_blob,
                              fp.name_off, code)
    assert rc == 0
    assert plan.footprint_bytes == foot
    if policy == "best_fit":
        assert foot == REF_BEST_FIT_FOOTPRINT
    got = np.asarray(plan.offsets)
    assert got.shape == offs.shape
    assert hashlib.sha256(got.tobytes()).hexdigest() == hashlib.sha256(offs.tobytes()).hexdigest()


@pytest.mark.parametrize("accesses,max_size", [(True, 64 << 20), (False, 256 << 20)])
def test_config4_full_size_variants_match_oracle(accesses, max_size):
    """The same 1 M-variable shape with a write after every malloc and a read
    before every free (6 M events: the access-extraction path at full size),
    and with sizes up to 256 MiB (a ~7.5 GB pool: the 64-bit placement
    kernel), offset for offset against the oracle."""
    import oracle as orc
    from paper_1903_06631_b200 import workloads
    from paper_1903_06631_b200.pipeline import plan_arrays
    arrays, window = workloads.interval_trace(1_000_000, seed=1, accesses=accesses, max_size=max_size)
    plan = plan_arrays(arrays, policy="best_fit")
    assert plan.period == window[1] - window[0]
    rc, fp = orc.extract(arrays, window[0], window[1])
    assert rc == 0
    off, lo, hi = orc.profile_segments(fp)
    h, row, _col = orc.conflict(off, lo, hi)
    try:
        assert plan.nvars == fp.nvars and plan.peak_bytes == fp.peak_bytes
        assert plan.nnz == int(row[-1])
        rc, offs, foot = orc.plan(h, fp.size, fp.alloc.astype(np.int64), fp.base, fp.name_ralloc(), fp.name_blob,
                                  fp.name_off, 1)
        assert rc == 0 and plan.footprint_bytes == foot
        if max_size > (64 << 20):
            assert plan.peak_bytes > (1 << 31)
        assert np.array_equal(np.asarray(plan.offsets), offs)
    finally:
        orc.graph_free(h)
