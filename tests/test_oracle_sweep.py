"""Pin the oracle's sweep unit (orc_sweep_unit) against the reference's own
estimators (tests/golden/sweep.json.gz, make_golden_sweep.py); CPU only."""
import pytest

import oracle as orc
from golden_util import check_sweep_unit, load, sweep_params, trace_arrays

SCEN = load("sweep")


@pytest.mark.parametrize("idx", range(len(SCEN)), ids=[s["name"] for s in SCEN])
def test_oracle_sweep_unit(idx):
    sc = SCEN[idx]
    rec, brec, offs, order = orc.sweep_unit(trace_arrays(sc), sweep_params(sc["params"]))
    check_sweep_unit(rec, brec, offs, order, sc["unit"])


def test_golden_covers_every_outcome():
    seen = set()
    for sc in SCEN:
        u = sc["unit"]
        if "error" in u:
            seen.add(u["error"][0])
            continue
        for b in u["budgets"]:
            seen.add(b["error"][0] if "error" in b else "ok")
    assert {"ok", "LimitUnreachable", "ValueError", "SwapDeadlock", "IndexError",
            "InvariantViolation", "PeriodNotFound"} <= seen
