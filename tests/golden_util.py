"""Loading and canonicalizing golden fixtures (tests/golden/*.json.gz).

The fixtures were produced by running the reference package
(tests/golden/make_golden.py).  These helpers turn flat results — from the
CPU oracle or from the device library — into the same canonical JSON so
equality means bit-for-bit parity (floats compare as ``float.hex``).
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os

import numpy as np

from paper_1903_06631_b200._abi import F_PERSISTENT, F_RENAMED, F_WRAPS
from paper_1903_06631_b200.trace import KIND_CODE, TraceArrays

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
INLINE = 400
SCORE_CODE = {"swdoa": 0, "doa": 1, "aoa": 2, "wdoa": 3, "combined": 4, "combined_w": 4}
ALT_WEIGHTS = (0.3, -0.5, 0.2, 0.8)
DEFAULT_WEIGHTS = (0.0, 0.0, 0.0, 1.0)

_cache = {}


def load(group: str) -> list[dict]:
    if group not in _cache:
        with gzip.open(os.path.join(GOLDEN, f"{group}.json.gz"), "rt") as fh:
            _cache[group] = json.load(fh)["scenarios"]
    return _cache[group]


def fhex(x) -> str:
    return float(x).hex()


def pack(lst):
    if len(lst) <= INLINE:
        return lst
    return {"sha256": hashlib.sha256(json.dumps(lst, separators=(",", ":")).encode()).hexdigest(),
            "n": len(lst)}


def trace_arrays(sc: dict) -> TraceArrays:
    tr = sc["trace"]
    code = {"m": KIND_CODE["malloc"], "f": KIND_CODE["free"], "r": KIND_CODE["read"],
            "w": KIND_CODE["write"]}
    kind = np.array([code[c] for c in tr["kind"]], np.uint8)
    index = np.array(tr["index"], np.int64)
    contiguous = np.array_equal(index, np.arange(index.shape[0]))
    return TraceArrays.from_columns(kind, tr["var"], np.array(tr["size"], np.int64),
                                    np.array(tr["t"], np.int64), None if contiguous else index)


def canon_profile(fp) -> dict:
    names = fp.var_names()
    base_names = [fp.names[b] for b in fp.base.tolist()]
    var = []
    ao = fp.acc_off.tolist()
    ai, ak, an = fp.acc_index.tolist(), fp.acc_kind.tolist(), fp.acc_next.tolist()
    times = fp.op_times
    seg = fp.seg.tolist()
    for i in range(fp.nvars):
        accs = [[ai[a], fhex(times[ai[a]]), ak[a], bool(an[a])] for a in range(ao[i], ao[i + 1])]
        ns = int(fp.nseg[i])
        segs = [[seg[4 * i + 2 * s], seg[4 * i + 2 * s + 1]] for s in range(ns)]
        alloc = int(fp.alloc[i])
        free = int(fp.free_[i])
        fl = int(fp.flags[i])
        var.append([names[i], base_names[i], int(fp.size[i]), None if alloc < 0 else alloc,
                    None if free < 0 else free, segs, bool(fl & F_PERSISTENT),
                    bool(fl & F_WRAPS), accs])
    owner = fp.op_owner.tolist()
    return {"period": fp.period, "window": list(fp.window), "vars": pack(var), "nvars": fp.nvars,
            "loads": pack(fp.loads.tolist()), "peak": fp.peak_bytes,
            "peak_index": fp.peak_index, "op_times": pack([fhex(x) for x in times.tolist()]),
            "duration": fhex(fp.duration_us), "op_instance": pack([names[o] for o in owner])}


def canon_adj(row_off, col, nvars) -> dict:
    adj = []
    for i in range(nvars):
        adj.append(sorted(set(col[row_off[i]:row_off[i + 1]].tolist())))
    return {"edges": sum(len(a) for a in adj) // 2, "adj": pack(adj)}


def canon_cands(c, fp) -> list:
    names = fp.var_names()
    return [[names[c.var[i]], int(c.size[i]), int(c.out_index[i]), fhex(c.out_t[i]),
             fhex(c.out_ready[i]), int(c.in_index[i]), fhex(c.in_t[i]), fhex(c.dout[i]),
             fhex(c.din[i]), bool(c.spans[i])] for i in range(c.k)]


def canon_schedule(cnames, sel, t_so, t_eo, t_si, t_ei, event_order, sizes, duration) -> dict:
    ev = []
    for s in event_order:
        ci = sel[s]
        ev.append([cnames[ci], int(sizes[ci]), fhex(t_so[s]), fhex(t_eo[s]), fhex(t_si[s]),
                   fhex(t_ei[s])])
    return {"events": ev, "order": [cnames[ci] for ci in sel], "duration": fhex(duration)}


def canon_curve(t, v, peak, peak_t) -> dict:
    return {"points": pack([[fhex(a), int(b)] for a, b in zip(t.tolist(), v.tolist())]),
            "peak": int(peak), "peak_t": fhex(peak_t)}


# ---------------------------------------------------------------------------
# batched sweep units (tests/golden/sweep.json.gz, make_golden_sweep.py)

V_REASON = {1: "not contiguous", 2: "negative timestamp", 3: "timestamp decreases",
            4: "malloc size must be > 0", 5: "malloc of live id", 6: "size must be 0",
            7: "free of dead id", 8: "use of dead id"}


def sweep_params(prm: dict):
    from paper_1903_06631_b200.sweep import SweepParams
    return SweepParams(budgets=tuple(prm["budgets"]), policy=prm["policy"], threshold_bytes=prm["threshold"],
                       bandwidth_bytes_per_s=prm["bw"], latency_us=prm["lat"], max_rounds=prm["max_rounds"])


def check_sweep_unit(rec, brec, offsets, order, gold: dict) -> None:
    """One unit's flat records (oracle or device) against the reference's."""
    if "error" in gold:
        kind = gold["error"][0]
        if kind == "InvariantViolation":
            assert int(rec["status"]) == 1 and int(rec["err_index"]) == gold["error"][1], (rec, gold)
            assert V_REASON[int(rec["err_code"])] in gold["error"][2], (rec, gold)
        else:
            assert kind == "PeriodNotFound" and int(rec["status"]) == 2, (rec, gold)
        return
    assert int(rec["status"]) == 0, rec
    got = {"period": int(rec["period"]), "nvars": int(rec["nvars"]), "ncarry": int(rec["ncarry"]),
           "naccess": int(rec["naccess"]), "peak": int(rec["peak_bytes"]),
           "peak_index": int(rec["peak_index"]), "duration": fhex(rec["duration_us"]),
           "footprint": int(rec["footprint_bytes"]), "edges": int(rec["edges"]),
           "ncand": int(rec["ncand"]), "load_min": int(rec["load_min"]),
           "offsets": [int(x) for x in offsets]}
    want = {k: gold[k] for k in got}
    assert got == want
    # the greedy prefix the budgets need (the reference's full order cut)
    assert int(rec["norder"]) == len(order) <= len(gold["order"])
    assert [int(x) for x in order] == gold["order"][:len(order)]
    assert len(brec) == len(gold["budgets"])
    code = {"ValueError": 6, "LimitUnreachable": 3, "SwapDeadlock": 4, "IndexError": 5}
    for b, g in zip(brec, gold["budgets"]):
        assert int(b["limit_bytes"]) == g["limit"], (b, g)
        if "error" in g:
            e = g["error"]
            assert int(b["status"]) == code[e[0]], (b, g)
            if e[0] == "LimitUnreachable":
                assert int(b["err_aux"]) == e[2], (b, g)
            if e[0] == "SwapDeadlock":
                assert int(b["err_index"]) == e[1], (b, g)
            continue
        nsel = int(b["nsel"])
        assert nsel <= len(order)
        got_b = {"selection": [int(x) for x in order[:nsel]], "selected_bytes": int(b["selected_bytes"]),
                 "rounds": int(b["rounds"]), "overhead_us": fhex(b["overhead_us"]),
                 "achieved": int(b["achieved_peak_bytes"]), "planned": int(b["planned_peak_bytes"])}
        assert int(b["status"]) == 0 and got_b == {k: g[k] for k in got_b}, (b, g)
