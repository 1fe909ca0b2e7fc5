"""BO objective throughput (SwapPlanner score="bo"): the batched device
evaluator (mp_swap_eval_weights) vs the per-call device path vs the C oracle
(orc_select combined + schedule + simulate, 1 host core), on the config-3
VGG-16 b128 profile.  python tools/bo_bench.py [--m 4096]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import numpy as np  # noqa: E402

import oracle as orc  # noqa: E402
from paper_1903_06631_b200 import _native as N  # noqa: E402
from paper_1903_06631_b200 import autoswap, detect_iteration, extract_lifetimes, swapsim, synth, workloads  # noqa: E402
from paper_1903_06631_b200.autoswap import ScoreWeights, TransferModel  # noqa: E402
from paper_1903_06631_b200.iteration import device_profile  # noqa: E402
from paper_1903_06631_b200.trace import as_arrays  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=4096)
    ap.add_argument("--frac", type=float, default=0.9)
    args = ap.parse_args()
    tr = synth.generate_synthetic_trace(workloads.vgg16_spec(128))
    det = detect_iteration(tr)
    prof = extract_lifetimes(tr, det.window)
    limit = int(prof.load.peak_bytes * args.frac)
    tm = TransferModel(50e9, 10.0)
    cands = autoswap.filter_candidates(prof, threshold_bytes=1 << 20, transfer=tm)

    def scalar(w):
        sel = autoswap.select_by_score(cands, prof, limit, score="combined", weights=w)
        return swapsim.simulate(swapsim.build_schedule(sel, prof), prof, limit).overhead_us

    ev = autoswap.WeightEvaluator(cands, prof, limit, scalar)
    rng = np.random.default_rng(0)
    W = np.round(rng.uniform(-1, 1, (args.m, 4)), 9)
    dp = device_profile(prof)
    cc = autoswap._cands(cands)
    N.swap_eval_weights(dp, cc, ev.z, W[:64], limit)  # warm
    t0 = time.perf_counter()
    st, ov, _ns, _ax = N.swap_eval_weights(dp, cc, ev.z, W, limit)
    tb = time.perf_counter() - t0
    t0 = time.perf_counter()
    for i in range(20):
        N.swap_eval_weights(dp, cc, ev.z, W[i:i + 1], limit)
    t1 = (time.perf_counter() - t0) / 20
    t0 = time.perf_counter()
    okc = 0
    for i in range(20):
        try:
            scalar(ScoreWeights(*W[i]))
            okc += 1
        except Exception:  # noqa: BLE001
            pass
    ts = (time.perf_counter() - t0) / 20
    # the C oracle: select(combined) + schedule + simulate per vector
    a = as_arrays(tr)
    rc, fp = orc.extract(a, det.window[0], det.window[1])
    c = orc.candidates(fp, 1 << 20, 50e9, 10.0)
    names = orc.names_of(fp)
    load = orc._load(fp)
    t0 = time.perf_counter()
    n_or = 200
    for i in range(n_or):
        rc, err, sel = orc.select(load, c, names, 4, W[i], limit)
        if rc == 0:
            sched = orc.schedule(fp, c, names, sel)
            orc.simulate(fp, c, names, sel, sched, limit)
    to = (time.perf_counter() - t0) / n_or
    out = {"profile": "vgg16_b128 (config 3)", "period": prof.period, "candidates": len(cands), "limit_frac": args.frac,
           "batched": {"m": args.m, "seconds": tb, "evals_per_s": args.m / tb,
                       "status": {str(k): int(v) for k, v in zip(*np.unique(st, return_counts=True))}},
           "device_single_launch_s": t1, "device_per_call_path_s": ts, "oracle_c_1core_s": to,
           "batched_vs_oracle_1core": to / (tb / args.m)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
