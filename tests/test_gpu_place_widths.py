"""The placement kernel's two widths (placement.cu): the 32-bit hole scan
of the narrow kernel (traced peak under 2^31 bytes), its per-variable
fall-back to the 64-bit scan when a pool that started narrow grows past
2^31, and the 64-bit kernel — each against the C oracle, offset for offset,
for both policies, on interval traces whose sizes put the pool on either
side of 2^31."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NVARS = 60_000


def _oracle(arrays, window, code):
    import oracle as orc
    rc, fp = orc.extract(arrays, window[0], window[1])
    assert rc == 0
    off, lo, hi = orc.profile_segments(fp)
    h, _row, _col = orc.conflict(off, lo, hi)
    try:
        rc, offs, foot = orc.plan(h, fp.size, fp.alloc.astype(np.int64), fp.base, fp.name_ralloc(), fp.name_blob,
                                  fp.name_off, code)
    finally:
        orc.graph_free(h)
    assert rc == 0
    return fp, offs, foot


@pytest.mark.parametrize("max_size,regime", [(48 << 20, "narrow"), (72 << 20, "mixed"), (256 << 20, "wide")])
@pytest.mark.parametrize("policy,code", [("best_fit", 1), ("first_fit", 0)])
def test_placement_widths_match_oracle(max_size, regime, policy, code):
    from paper_1903_06631_b200 import workloads
    from paper_1903_06631_b200.pipeline import plan_arrays
    arrays, window = workloads.interval_trace(NVARS, seed=3, max_size=max_size)
    fp, offs, foot = _oracle(arrays, window, code)
    plan = plan_arrays(arrays, policy=policy)
    assert plan.peak_bytes == fp.peak_bytes
    if regime == "narrow":
        assert foot < 2**31 - 1
    elif regime == "mixed":
        assert fp.peak_bytes < 2**31 - 1 < foot, (fp.peak_bytes, foot)
    else:
        assert fp.peak_bytes >= 2**31
    assert plan.footprint_bytes == foot
    assert np.array_equal(np.asarray(plan.offsets), offs)
