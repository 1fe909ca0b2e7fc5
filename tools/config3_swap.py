"""Config 3: AutoSwap plans executed on a VGG-16 training iteration.

Run in a fresh process (the allocator must be installed before the first
CUDA allocation):

    python tools/config3_swap.py [--batch 128] [--steps 10] [--fracs 0.9,0.8,0.691,0.6]

1. Records three iterations through the pluggable allocator + dispatch tracer
   (per-op CUDA-event timestamps: the device timeline of an unsynchronised
   run; ``--sync-times`` = the paper's synchronise-per-op profiling).
2. Detects the iteration and extracts lifetimes + access gaps on the device.
3. Measures the host link (pinned D2H / H2D) and uses it as the transfer
   model.
4. For each memory limit (fraction of the traced peak load) and selection
   mode — the reference's SWDOA selection among the executable candidates;
   the same with each swap-in issued at the reference schedule's start
   (``reference_schedule``: the replayed op at ``t_start_in``, no earlier
   than its pool bytes are free); the same restricted to candidates whose
   round trip fits their gap; and
   ``swapexec.select_window_fits`` (ours: copies must fit the executor's
   windows at the measured link rates, optionally with a 4 % stall budget) —
   schedule, simulation (predicted overhead), mapping onto op-granular hook
   points, pool plan on the split lifetimes, and a served + swapped run of
   ``--steps`` iterations.
5. Prints one JSON line: per limit the predicted and measured overhead vs
   the same hooked run without swaps, the pool footprint vs the no-swap pool,
   the bytes moved, and whether the losses equal the unswapped run bit for bit.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("CUBLAS_WORKSPACE_CONFIG", ":4096:8")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def link_bandwidth(nbytes=256 << 20, reps=5):
    """Pinned host <-> device copy bandwidth (bytes/s): D2H, H2D alone and
    both directions at once."""
    import torch
    h1 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d1 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(d2h, h2d):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.cuda.current_stream().synchronize()
        import time
        t = time.perf_counter()
        for _ in range(reps):
            if d2h:
                with torch.cuda.stream(s1):
                    h1.copy_(d1, non_blocking=True)
            if h2d:
                with torch.cuda.stream(s2):
                    d2.copy_(h2, non_blocking=True)
        torch.cuda.synchronize()
        return nbytes * reps / (time.perf_counter() - t)
    run(True, True)
    out = {"d2h": run(True, False), "h2d": run(False, True)}
    both = run(True, True)
    out["duplex_each"] = both
    del h1, h2, d1, d2
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--fracs", default="0.98,0.95,0.93,0.92,0.9,0.88,0.85,0.8,0.7")
    ap.add_argument("--modes", default="reference_selection,transfer_fits_gap,window_fits,window_fits_stall4pct")
    ap.add_argument("--threshold-mib", type=float, default=1.0)
    ap.add_argument("--sync-times", action="store_true",
                    help="time ops with a synchronize each (the paper's profiler) instead of device events")
    a = ap.parse_args()
    from paper_1903_06631_b200 import torchmem, iteration, autoswap, swapsim, smartpool, swapexec
    from paper_1903_06631_b200.errors import LimitUnreachable, SwapDeadlock
    torchmem.install()
    import torch
    from config2_pool import build
    torch.backends.cudnn.benchmark = False
    torch.backends.cudnn.deterministic = True
    torch.use_deterministic_algorithms(True)
    model, opt, step = build(a.batch)
    lossbuf = torch.zeros(max(a.steps, 3), device="cuda")

    def one(i):
        lossbuf[i].copy_(step())

    for i in range(2):
        one(i)
    with torchmem.Tracer(dispatch=True, device_times=not a.sync_times) as tr:
        for i in range(3):
            one(i)
            tr.mark()
    arrays = tr.trace()
    det = iteration.detect_iteration(arrays)
    prof = iteration.extract_lifetimes(arrays, det.window)
    points, base = swapexec.event_points(tr, prof.window)
    last_mark = max(s for s, _t in tr.marks)
    n_ops = last_mark - base - 1
    slot_of = swapexec.window_slots(prof)
    bw = link_bandwidth()
    tm = autoswap.TransferModel(bandwidth_bytes_per_s=min(bw["duplex_each"], bw["d2h"], bw["h2d"]), latency_us=10.0)
    cands = autoswap.filter_candidates(prof, int(a.threshold_mib * (1 << 20)), tm)
    exec_cands = [c for c in cands if not c.spans_iterations and c.var in slot_of]

    params = list(model.parameters())
    snap_m = {k: v.clone() for k, v in model.state_dict().items()}
    snap_mom = [opt.state[p]["momentum_buffer"].clone() for p in params]
    snap_rng = torch.cuda.get_rng_state()

    def restore():
        torch.cuda.set_rng_state(snap_rng)
        with torch.no_grad():
            for k, v in model.state_dict().items():
                v.copy_(snap_m[k])
            for p, mb in zip(params, snap_mom):
                opt.state[p]["momentum_buffer"].copy_(mb)

    def pool_for(actions):
        arcs = swapexec.split_arcs(prof, actions)
        g = smartpool.conflict_graph_from_arcs(prof.period, arcs, prof.peak_bytes)
        plan = min((smartpool.plan_pool(g, pol) for pol in ("best_fit", "first_fit")),
                   key=lambda pl: pl.footprint_bytes)
        # lower bound: the arcs' peak load (no placement can go below it)
        import numpy as np
        delta = np.zeros(prof.period + 1, np.int64)
        for _v, z, _a, segs, _p in arcs:
            for lo, hi in segs:
                delta[lo] += z
                delta[hi] -= z
        plan.arc_peak_bytes = int(np.cumsum(delta).max())
        offs = swapexec.served_offsets(arcs, plan.offsets, actions)
        order = sorted(slot_of, key=slot_of.get)
        sizes = {v.var: v.size for v in prof.variables}
        import numpy as np
        slots = (np.array([offs[v] for v in order], np.int64), np.array([sizes[v] for v in order], np.int64))
        return plan, offs, slots

    def run(actions, hooked=True):
        """Serve (+swap) a.steps iterations from restored state; returns
        (ms per iteration, losses, executor)."""
        plan, offs, slots = pool_for(actions)
        restore()
        torchmem.serve(plan.footprint_bytes, slots)
        ex = swapexec.SwapExecutor(actions, int(torchmem.ctl().mp_alloc_pool_base()), offs, n_ops) if hooked else None
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for i in range(a.steps):
            torchmem.begin_iteration()
            if ex:
                ex.begin()
            try:
                one(i)
            finally:
                if ex:
                    ex.end()
        e.record()
        e.synchronize()
        # the last iteration's gradients live in this pool until the next
        # zero_grad: release them before another plan replaces the pool
        opt.zero_grad(set_to_none=True)
        torch.cuda.synchronize()
        st = torchmem.stats()
        torchmem.passthrough()
        return s.elapsed_time(e) / a.steps, lossbuf[:a.steps].tolist(), ex, plan, st

    ms_plain, losses_plain, _x, plan0, st0 = run([], hooked=False)
    ms_hook, losses_hook, _x, _p, _s = run([], hooked=True)
    ms_hook2, _l, _x, _p, _s = run([], hooked=True)
    fit_cands = [c for c in exec_cands if c.gap_us >= c.delta_out_us + c.delta_in_us]
    rows = []
    pools = {"reference_selection": exec_cands, "reference_schedule": exec_cands, "transfer_fits_gap": fit_cands,
             "window_fits": exec_cands, "window_fits_stall4pct": exec_cands}
    for mode in [m for m in a.modes.split(",") if m]:
        pool = pools[mode]
        for frac in [float(x) for x in a.fracs.split(",") if x]:
            limit = int(prof.peak_bytes * frac)
            row = {"mode": mode, "frac": frac, "limit_bytes": limit}
            try:
                if mode.startswith("window_fits"):
                    budget = 0.04 * prof.period_duration_us if mode.endswith("4pct") else 0.0
                    sel = swapexec.select_window_fits(prof, pool, limit, points, slot_of, bw["d2h"], bw["h2d"],
                                                      stall_budget_us=budget)
                else:
                    sel = autoswap.select_by_score(pool, prof, limit, "swdoa")
            except LimitUnreachable as exc:
                row["error"] = type(exc).__name__
                rows.append(row)
                continue
            sched = swapsim.build_schedule(sel, prof)
            try:
                sim = swapsim.simulate(sched, prof, limit)
            except SwapDeadlock:
                # the reference's replay cannot hold this limit; the executor
                # still runs the selection (its pool layout is the cap)
                row["sim_limit_deadlock"] = True
                sim = swapsim.simulate(sched, prof, None)
            in_ev = swapexec.schedule_in_events(prof, sim) if mode == "reference_schedule" else None
            acts, skipped = swapexec.plan_actions(prof, sel, limit, points, slot_of, in_events=in_ev)
            ms, losses, ex, plan, st = run(acts)
            by = {c.var: c for c in sel}
            # the reference's replay of just the executed subset, no limit:
            # the transfer-bound overhead of the copies that actually run
            exe = [by[x.var] for x in acts]
            sim_x = swapsim.simulate(swapsim.build_schedule(exe, prof), prof, None) if exe else None
            reasons = {}
            for sk in skipped:
                reasons[sk["why"]] = reasons.get(sk["why"], 0) + 1
            row.update({
                "selected": len(sel), "executed": len(acts), "skipped": len(skipped), "skip_reasons": reasons,
                "selected_bytes": int(sum(c.size for c in sel)),
                "executed_planned_peak_bytes": autoswap.planned_peak([by[x.var] for x in acts], prof),
                "swap_bytes_per_iter": int(sum(x.size for x in acts)),
                "predicted_overhead_pct": sim.overhead_pct, "predicted_peak_bytes": sim.achieved_peak_bytes,
                "predicted_executed_overhead_pct": sim_x.overhead_pct if sim_x else 0.0,
                "iter_ms": ms, "measured_overhead_pct": (ms / ms_hook - 1) * 100,
                "pool_footprint_bytes": plan.footprint_bytes, "pool_policy": plan.policy,
                "pool_arc_peak_bytes": plan.arc_peak_bytes,
                "pool_reduction_vs_noswap": 1 - plan.footprint_bytes / plan0.footprint_bytes,
                "losses_equal_unswapped": losses == losses_plain, "allocator": st,
                "link": ex.copy_stats() if acts else None,
            })
            rows.append(row)
    load_min = swapsim.compute_load_min(prof, exec_cands)
    cand_rows = [{"var": c.var, "mib": round(c.size / 2**20, 1), "out": c.out_index, "in": c.in_index,
                  "gap_us": round(c.gap_us, 1), "xfer_us": round(c.delta_out_us, 1)} for c in exec_cands]
    print(json.dumps({
        "config": f"vgg16_b{a.batch}", "load_min_all_candidates_absent": load_min,
        "peak_index": prof.load.peak_index, "candidate_list": cand_rows, "events": len(arrays), "period": prof.period, "window": list(prof.window),
        "ops_per_iter": n_ops, "traced_peak_bytes": prof.peak_bytes, "traced_duration_us": prof.period_duration_us,
        "link_bw_bytes_per_s": bw, "candidates": len(cands), "executable_candidates": len(exec_cands),
        "fit_candidates": len(fit_cands), "load_min_fit_candidates_absent": swapsim.compute_load_min(prof, fit_cands),
        "noswap_pool_bytes": plan0.footprint_bytes, "noswap_pool_arc_peak_bytes": plan0.arc_peak_bytes, "iter_ms_served_plain": ms_plain,
        "iter_ms_served_hooked": ms_hook, "iter_ms_served_hooked_repeat": ms_hook2,
        "hooked_losses_equal_plain": losses_hook == losses_plain, "noswap_allocator": st0,
        "losses": losses_plain[:4], "limits": rows,
        # enough of the profile to replay the selections offline
        "replay": {"loads": [int(x) for x in prof.load.loads], "op_times_us": [float(x) for x in prof.op_times_us],
                   "points": [int(x) for x in points], "slots": sorted(slot_of),
                   "cands": [{"var": c.var, "size": int(c.size), "out_index": int(c.out_index),
                              "in_index": int(c.in_index), "spans_iterations": bool(c.spans_iterations),
                              "gap_us": float(c.gap_us), "delta_out_us": float(c.delta_out_us)} for c in exec_cands]}}))


if __name__ == "__main__":
    main()
