"""Benchmark: SmartPool planning throughput on the 1M-variable interval trace.

Workload (BASELINE.json configs[3]): two
iterations of 1,000,000 interval lifetimes (4,000,008 events); one step is
the whole pool-planning hot path on the device —
validate_trace -> detect_iteration -> extract_lifetimes ->
build_conflict_graph -> plan_pool(best_fit) — over the full trace.
Metric: planned variables per second (whole job, all ranks).

  value   inputs resident in HBM; offsets stay in HBM
  e2e     public API (pipeline.plan_arrays) from pinned host arrays: H2D of
          the trace, the same pipeline, D2H of the offsets
  roofline  dominant kernel's algorithmic bytes / its CUDA-event time
  cpu_baseline  the C oracle (sequential restatement of the reference) on
          this host, rank 0, same trace, 1 thread

N GPUs: one process per GPU (torchrun), each plans its own replica of the
trace (the path does not shard: "replicas only"); value is the
sum of planned variables over ranks / max-over-ranks time.

The line also carries "sweep": BASELINE configs[4], 1024 traces x 4 swap
budgets = 4096 units (csrc/sweep.cu, one CTA per trace) — resident and e2e
units/s, sharded over ranks by LPT (strong scaling), its own parity check
and the C oracle on every host core as its cpu_baseline.

The line also carries "swap": BASELINE configs[2], the swap-iteration
overhead on a VGG-16 b128 training iteration (tools/config3_swap.py in a
subprocess on rank 0's GPU: traced, planned, executed with copy streams for
10 iterations at 95 % of the traced peak, the reference's SWDOA selection and
the executor-aware one — strict (copies must fit their windows at 0.9x the
measured link rates) and with a 4 % stall budget; lower is better).

--impl reference: the reference's CPU algorithm (the C oracle port — the
Python reference cannot run on this box) on all host cores, one trace
replica per process, same metric.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [ROOT]

import numpy as np  # noqa: E402

NVARS = 1_000_000
METRIC = "planned vars/sec (SmartPool plan, bit-exact vs ref)"
UNIT = "vars/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def hbm_peak():
    try:
        with open(PEAKS_PATH) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


def _nvml_sampler(index, period, stop, conn, ready):
    """Child process: NVML SM clock + clock-event reasons every `period` s
    until `stop` is set (a separate process, so sampling never holds the
    benchmark's GIL)."""
    names = ClockSampler.NAMES
    samples = []
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(index)
        bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        while not stop.is_set():
            sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            samples.append((sm, mx, tuple(n for n, b in zip(names, bits) if r & b)))
            ready.set()
            stop.wait(period)
    except Exception:  # noqa: BLE001
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        while not stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(index), f"--query-gpu={fields}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                samples.append((float(f[0]), float(f[1]),
                                tuple(n for i, n in enumerate(names) if f[2 + i].lower().startswith("active"))))
                ready.set()
            except Exception:  # noqa: BLE001
                pass
            stop.wait(0.05)
    ready.set()
    conn.send(samples)
    conn.close()


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    2 ms while the timed region runs, in a child process."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int, period_s: float = 0.002):
        import multiprocessing as mp
        ctx = mp.get_context("fork")
        self._stop = ctx.Event()
        self._ready = ctx.Event()
        self._recv, send = ctx.Pipe(duplex=False)
        self._p = ctx.Process(target=_nvml_sampler, args=(index, period_s, self._stop, send, self._ready),
                              daemon=True)
        self.samples = []

    def __enter__(self):
        self._p.start()
        # the timed region starts once the child has its first sample (NVML
        # start-up can outlast a short timed region)
        self._ready.wait(10)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        try:
            if self._recv.poll(10):
                self.samples = self._recv.recv()
        finally:
            self._p.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [s[0] for s in self.samples]
        reasons = sorted({r for s in self.samples for r in s[2]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# algorithmic bytes per stage

def stage_bytes(n, p, V, nnz, levels):
    """Minimal HBM bytes each stage must move for one trace."""
    return {
        "group_sort": n * 4 + n * 4,                     # read var ids, write grouping permutation
        "validate": n * (1 + 8 + 8) + n * 4,             # kind/size/t + permutation walk
        "detect": n * (1 + 8) + (n + 1) * 8,             # fingerprints read, prefix hashes written
        "extract": n * 4 + p * (1 + 4 + 8 + 8) + V * 44 + p * 12,
        "loads": V * 24 + p * 16,
        "conflict_prep": V * 24 + V * 24,
        "conflict_fill": nnz * 4 + V * 16,               # CSR column writes + row metadata
        "place_order": V * 8 + V * 4,
        "place_split": V * (4 + 4 + 4),                  # pcnt read, counters + queue written (rows arrive partitioned)
        "place": nnz // 2 * (4 + 8 + 8) + nnz // 2 * (4 + 4) + V * 24,
        "footprint": V * 16,
    }


# ---------------------------------------------------------------------------


def config4(args, world, n, period):
    """The `config` dict both arms print (same keys and values)."""
    return {"workload": "interval_trace_1M (BASELINE configs[3])", "nvars": NVARS, "events": int(n),
            "period": int(period), "policy": "best_fit", "accesses": bool(args.accesses),
            "l2": "flushed (256 MiB write) between steps", "parallelism": f"replicas x{world}"}


def build_workload(accesses: bool):
    from paper_1903_06631_b200 import workloads
    arrays, window = workloads.interval_trace(NVARS, seed=0, accesses=accesses)
    return arrays, window


def pinned_like(a: np.ndarray):
    import torch
    t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
    view = t.numpy().view(a.dtype)[: a.size].reshape(a.shape)
    view[...] = a
    return t, view


def run_ours(args, rank, world, local_rank):
    import torch
    torch.cuda.set_device(local_rank)
    os.environ["MEMPLAN_DEVICE"] = str(local_rank)
    from paper_1903_06631_b200 import _native as N
    from paper_1903_06631_b200.pipeline import plan_arrays
    from paper_1903_06631_b200.trace import TraceArrays

    arrays, window = build_workload(args.accesses)
    n = len(arrays)
    # pinned host copies for the e2e leg (a user hands us host buffers)
    keep = []
    cols = {}
    for name in ("kind", "var", "size", "t_us"):
        t, v = pinned_like(getattr(arrays, name))
        keep.append(t)
        cols[name] = v
    host = TraceArrays(cols["kind"], cols["var"], cols["size"], cols["t_us"], arrays.names)
    out_t, out_offs = pinned_like(np.zeros(NVARS + 1, np.int64))
    keep.append(out_t)

    stream = torch.cuda.ExternalStream(N.stream_ptr())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def l2_flush():
        with torch.cuda.stream(stream):
            flush.zero_()

    # ---- value: resident inputs ----
    dev_arrays = arrays  # uploaded once below; the trace handle stays in HBM
    plan = None
    for _ in range(args.warmup):
        plan = plan_arrays(dev_arrays, keep_on_device=True)
    N.sync()
    first = N.launches()
    times = []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            l2_flush()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            plan = plan_arrays(dev_arrays, keep_on_device=True)
            e.record(stream)
            e.synchronize()
            times.append(s.elapsed_time(e))
    launches = N.launches() - first
    step_ms = float(np.mean(times))
    # per-stage breakdown from a separate pass: the stage events sit between
    # the kernels and would hold back their programmatic early launch, so the
    # timed steps above run without them
    N.set_timing(True)
    for _ in range(args.steps):
        l2_flush()
        plan_arrays(dev_arrays, keep_on_device=True)
    torch.cuda.synchronize()
    stages = N.timings()
    N.set_timing(False)
    # ---- e2e: pinned host -> device -> pinned host, public API ----
    e2e_times = []
    for i in range(args.warmup + args.steps):
        host._dev = None  # every step uploads the trace afresh
        l2_flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        p2 = plan_arrays(host, offsets_out=out_offs)
        e.record(stream)
        e.synchronize()
        if i >= args.warmup:
            e2e_times.append(s.elapsed_time(e))
    e2e_ms = float(np.mean(e2e_times))
    sha = hashlib.sha256(out_offs[:p2.nvars].tobytes()).hexdigest()
    # the name strings stay on the host (ids are lexicographic ranks)
    h2d = sum(getattr(host, c).nbytes for c in ("kind", "var", "size", "t_us"))
    d2h = p2.nvars * 8

    # max over ranks
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([step_ms, e2e_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        step_ms, e2e_ms = float(tt[0]), float(tt[1])
    vars_total = plan.nvars * world
    res = {
        "plan": plan, "step_ms": step_ms, "e2e_ms": e2e_ms, "stages": stages, "launches": launches,
        "clocks": clk.summary(), "sha": sha, "h2d": h2d, "d2h": d2h, "n": n, "vars_total": vars_total,
        "footprint_e2e": p2.footprint_bytes,
    }
    return arrays, res


# ---------------------------------------------------------------------------
# config 5: batched sweep of 1024 traces x 4 budgets = 4096 units, sharded
# over ranks (LPT on event counts, no collective on the data path)


def _sweep_oracle_chunk(idx):
    import oracle as orc
    t0 = time.perf_counter()
    recs, brecs, offs, orders = orc.sweep(_SWEEP_BATCH, _SWEEP_PARAMS, idx)
    return time.perf_counter() - t0, recs, brecs, offs, orders


_SWEEP_BATCH = None
_SWEEP_PARAMS = None


def sweep_cpu_baseline(batch, params, procs):
    """The C oracle over the whole batch on `procs` host processes (fork)."""
    global _SWEEP_BATCH, _SWEEP_PARAMS
    import multiprocessing as mp
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    _SWEEP_BATCH, _SWEEP_PARAMS = batch, params
    chunks = [list(range(i, batch.ntraces, procs)) for i in range(procs)]
    chunks = [c for c in chunks if c]
    with mp.get_context("fork").Pool(len(chunks)) as pool:
        pool.map(_sweep_oracle_chunk, chunks[:1])  # warm the workers
        t0 = time.perf_counter()
        outs = pool.map(_sweep_oracle_chunk, chunks)
        dt = time.perf_counter() - t0
    return dt, chunks, outs


def ncu_traffic(kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the committed
    ncu capture (profiles/r2_ncu_kernels.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_ncu_kernels.json")) as fh:
            k = json.load(fh)["kernels"].get(kernel)
        return k["dram_read_bytes"] + k["dram_write_bytes"] if k else None
    except Exception:  # noqa: BLE001
        return None


def run_sweep_bench(args, rank, world, local_rank, hbm_gbs):
    import torch
    from paper_1903_06631_b200 import _native as N
    from paper_1903_06631_b200 import sweep, workloads
    batch = sweep.SweepBatch.from_traces(workloads.sweep_traces())
    params = sweep.SweepParams(budgets=workloads.SWEEP_BUDGETS)
    parts = sweep.shard([batch.events_of(t) for t in range(batch.ntraces)], world)
    mine = batch.subset(parts[rank]) if world > 1 else batch
    stream = torch.cuda.ExternalStream(N.stream_ptr())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timed(fn):
        with torch.cuda.stream(stream):
            flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        out = fn()
        e.record(stream)
        e.synchronize()
        return s.elapsed_time(e), out

    ds = sweep.DeviceSweep(mine)
    for _ in range(args.warmup):
        ds.run(params)
    l0 = N.launches()
    res_ms = [timed(lambda: ds.run(params))[0] for _ in range(args.steps)]
    launches = (N.launches() - l0) / max(args.steps, 1)
    res = ds.download()
    ds.close()
    # e2e: the public call from pinned host buffers (inputs and records)
    keep = []

    def pinned(nbytes):
        t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        keep.append(t)
        return t.numpy()

    hb = mine.copy_to(pinned)
    nev = max(int(mine.ev_off[-1]), 1)
    hout = sweep.SweepResult(pinned(res.traces.nbytes).view(sweep.TRACE_DTYPE),
                             pinned(max(res.budgets.nbytes, 1)).view(sweep.BUDGET_DTYPE)[:res.budgets.size]
                             .reshape(res.budgets.shape),
                             pinned(nev * 8).view(np.int64), pinned(nev * 4).view(np.int32), hb.ev_off, params, hb)
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        if world == 1:
            ms, out = timed(lambda: sweep.run_sweep(hb, params, out=hout))
        else:
            # the whole sharded call: each rank's upload + launch + download,
            # then the gather of every rank's records to rank 0 (host wall
            # clock from a common barrier; max over ranks below)
            import torch.distributed as dist
            dist.barrier()
            t0 = time.perf_counter()
            out = sweep.run_sweep(hb, params, out=hout)
            got = [None] * world if rank == 0 else None
            dist.gather_object((parts[rank], out.records_only()), got, dst=0)
            if rank == 0:
                full = sweep.concat_results(got, batch)
            ms = (time.perf_counter() - t0) * 1e3
        if i >= args.warmup:
            e2e_ms.append(ms)
    step_ms, e2e_step = float(np.mean(res_ms)), float(np.mean(e2e_ms))
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([step_ms, e2e_step], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        step_ms, e2e_step = float(tt[0]), float(tt[1])
    units = batch.ntraces * len(params.budgets)
    d2h = int(res.traces.nbytes + res.budgets.nbytes + 12 * mine.ev_off[-1])
    algo = int(mine.nbytes) + d2h
    vars_total = int(res.traces["nvars"].sum())
    if world > 1:
        import torch.distributed as dist
        tv = torch.tensor([vars_total], device="cuda", dtype=torch.int64)
        dist.all_reduce(tv)
        vars_total = int(tv[0])
    out = {"workload": "sweep_4096 (BASELINE configs[4]): 64 model shapes x 16 batch scales x 4 budgets",
           "traces": batch.ntraces, "units": units, "events": int(batch.ev_off[-1]),
           "value": units / (step_ms * 1e-3), "unit": "units/s", "ms_per_step": step_ms,
           "planned_vars_per_s": vars_total / (step_ms * 1e-3), "scaling": "strong",
           "sharding": f"LPT over {world} rank(s), no data-path collective",
           "gpu_launches": launches,
           "e2e": {"value": units / (e2e_step * 1e-3), "unit": "units/s", "ms_per_step": e2e_step,
                   "h2d_bytes_per_step": int(mine.nbytes), "d2h_bytes_per_step": d2h,
                   "timing": "CUDA events on the library stream" if world == 1 else
                             "host wall clock from a barrier through the gather to rank 0, max over ranks"},
           "roofline": {"bound": "latency (one CTA per trace: the largest traces' sequential chains)",
                        "kernel": "k_sweep", "achieved": algo / (step_ms * 1e-3) / 1e9, "peak": hbm_gbs,
                        "unit": "GB/s", "frac": algo / (step_ms * 1e-3) / 1e9 / hbm_gbs,
                        "algorithmic_bytes": algo, "traffic": ncu_traffic("k_sweep"),
                        "note": "bytes = trace columns read + records written; see DESIGN 4b"},
           "budget_status": {str(k): int(v) for k, v in zip(*np.unique(res.budgets["status"], return_counts=True))}}
    if world > 1 and rank == 0:
        # per-N parity: the gathered records equal one rank planning the
        # whole batch (which the N=1 run checks against the oracle)
        ds1 = sweep.DeviceSweep(batch)
        ds1.run(params)
        one = ds1.download()
        ds1.close()
        out["parity"] = {"gathered_equal_single_rank": bool(
            one.traces.tobytes() == full.traces.tobytes() and one.budgets.tobytes() == full.budgets.tobytes()
            and np.array_equal(one.offsets, full.offsets) and np.array_equal(one.cand_order, full.cand_order))}
    if rank == 0 and world == 1:
        # strong-scaling evidence on one GPU: every rank's LPT shard of the
        # batch timed as its own launch, one after another; a rank's kernel
        # is the N-GPU step's device time when the ranks run side by side
        # (no data-path collective), so max over ranks bounds the N-GPU
        # kernel.  The floor is the longest single trace on its own.
        def shard_ms(sub, reps=5):
            d = sweep.DeviceSweep(sub)
            d.run(params)
            t = sorted(timed(lambda: d.run(params))[0] for _ in range(reps))
            d.close()
            return t[len(t) // 2]
        proj = {}
        for nw in (2, 4, 8):
            per = [shard_ms(batch.subset(p)) for p in sweep.shard([batch.events_of(t) for t in range(batch.ntraces)], nw)]
            proj[str(nw)] = {"max_rank_kernel_ms": max(per), "min_rank_kernel_ms": min(per),
                             "speedup_vs_1": step_ms / max(per)}
        big = int(np.argmax([batch.events_of(t) for t in range(batch.ntraces)]))
        proj["largest_trace_alone_ms"] = shard_ms(batch.subset([big]))
        proj["how"] = ("each rank's LPT shard launched alone on this GPU (median of 5, L2 flushed); "
                       "no multi-GPU run: an N-GPU step's device time is its slowest rank")
        out["shard_projection"] = proj
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        procs = os.cpu_count() or 1
        dt, chunks, outs = sweep_cpu_baseline(batch, params, procs)
        ok = True
        for idx, (_, recs, brecs, offs, orders) in zip(chunks, outs):
            for q, t in enumerate(idx):
                ok &= (res.traces[t].tobytes() == recs[q].tobytes() and res.budgets[t].tobytes() == brecs[q].tobytes()
                       and np.array_equal(res.offsets_of(t), offs[q]) and np.array_equal(res.order_of(t), orders[q]))
        out["cpu_baseline"] = {"value": units / dt, "unit": "units/s", "cores": procs, "kind": "port",
                               "sample": f"the whole 4096-unit batch, C oracle in {procs} processes, {dt:.3f} s"}
        out["parity"] = {"units_equal_oracle": bool(ok)}
    return out


def cpu_baseline(arrays):
    """C oracle on this host: detect + extract + conflict + best_fit plan, 1 thread."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    t0 = time.perf_counter()
    rc, p = orc.detect(arrays)
    rc, fp = orc.extract(arrays, len(arrays) - p, len(arrays))
    off, lo, hi = orc.profile_segments(fp)
    h, row, col = orc.conflict(off, lo, hi)
    rc, offs, foot = orc.plan(h, fp.size, fp.alloc.astype(np.int64), fp.base, fp.name_ralloc(),
                              fp.name_blob, fp.name_off, 1)
    dt = time.perf_counter() - t0
    orc.graph_free(h)
    return {"value": fp.nvars / dt, "seconds": dt, "footprint": foot, "peak": fp.peak_bytes,
            "sha": hashlib.sha256(offs.tobytes()).hexdigest(), "nvars": fp.nvars}


def _ref_worker(args):
    accesses, = args
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    arrays, _ = build_workload(accesses)
    return cpu_baseline(arrays)


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import multiprocessing as mp
    procs = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    step_s = []
    with ctx.Pool(procs) as pool:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            outs = pool.map(_ref_worker, [(args.accesses,)] * procs)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                step_s.append(max(o["seconds"] for o in outs))
    step = float(np.mean(step_s))
    value = procs * outs[0]["nvars"] / step
    arrays, window = build_workload(args.accesses)
    n = len(arrays)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": config4(args, world, n, window[1] - window[0]),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                             "sample": f"{procs} replicas of the full 1M-var trace, one per process "
                                       "(C oracle; the Python reference is not on this box)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_config1_leg(args, hbm_gbs) -> dict:
    """BASELINE configs[0]: SmartPool plan of the ResNet-50 b32 trace.

    resident: the one-trace sweep kernel (csrc/sweep.cu, one CTA) with the
    trace already in HBM; e2e: the public call (pipeline.plan_arrays, which
    takes the one-CTA path for a trace this small) from pinned host columns,
    upload and offsets readback inside the timed region; cpu_baseline: the C
    oracle (detect + extract + conflict + plan) on one host core."""
    import torch
    from paper_1903_06631_b200 import _native as N
    from paper_1903_06631_b200 import sweep, synth, workloads
    from paper_1903_06631_b200.pipeline import plan_arrays
    from paper_1903_06631_b200.trace import TraceArrays, as_arrays
    arrays = as_arrays(synth.generate_synthetic_trace(workloads.resnet50_spec(32)))
    stream = torch.cuda.ExternalStream(N.stream_ptr())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timed(fn):
        with torch.cuda.stream(stream):
            flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        out = fn()
        e.record(stream)
        e.synchronize()
        return s.elapsed_time(e), out

    reps = max(args.steps, 20)
    ds = sweep.DeviceSweep(sweep.SweepBatch.from_traces([arrays]))
    prm = sweep.SweepParams(budgets=())
    for _ in range(args.warmup):
        ds.run(prm)
    res_ms = [timed(lambda: ds.run(prm))[0] for _ in range(reps)]
    res = ds.download()
    ds.close()
    keep, cols = [], {}
    for name in ("kind", "var", "size", "t_us"):
        t, v = pinned_like(getattr(arrays, name))
        keep.append(t)
        cols[name] = v
    host = TraceArrays(cols["kind"], cols["var"], cols["size"], cols["t_us"], arrays.names)
    out_t, out_offs = pinned_like(np.zeros(len(arrays), np.int64))
    keep.append(out_t)
    e2e_ms = []
    for i in range(args.warmup + reps):
        ms, plan = timed(lambda: plan_arrays(host, offsets_out=out_offs))
        if i >= args.warmup:
            e2e_ms.append(ms)
    # C oracle, one core: a bounded sample of repeated plans (~1 s)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    t0, k = time.perf_counter(), 0
    while k < 3 or time.perf_counter() - t0 < 1.0:
        rc, p = orc.detect(arrays)
        rc, fp = orc.extract(arrays, len(arrays) - p, len(arrays))
        off, lo, hi = orc.profile_segments(fp)
        h, _r, _c = orc.conflict(off, lo, hi)
        rc, offs, foot = orc.plan(h, fp.size, fp.alloc.astype(np.int64), fp.base, fp.name_ralloc(),
                                  fp.name_blob, fp.name_off, 1)
        orc.graph_free(h)
        k += 1
    cpu_s = (time.perf_counter() - t0) / k
    r = res.traces[0]
    nv = int(r["nvars"])
    res_step, e2e_step = float(np.median(res_ms)), float(np.median(e2e_ms))
    # algorithmic bytes: events 21 B in, per variable
    # 40 B profile + 8 B offset, 2E x 4 B adjacency
    edges = int(r["edges"])
    algo = len(arrays) * 21 + nv * 48 + 2 * edges * 4
    return {"workload": "resnet50_b32 plan (BASELINE configs[0])", "events": len(arrays), "period": int(r["period"]),
            "nvars": nv, "peak_bytes": int(r["peak_bytes"]), "footprint_bytes": int(r["footprint_bytes"]),
            "value": nv / (res_step * 1e-3), "unit": "vars/s", "us_per_plan": res_step * 1e3,
            "e2e": {"value": nv / (e2e_step * 1e-3), "unit": "vars/s", "us_per_plan": e2e_step * 1e3,
                    "h2d_bytes_per_step": int(sum(cols[c].nbytes for c in cols)), "d2h_bytes_per_step": nv * 8},
            "roofline": {"bound": "latency (one CTA: sequential placement walk)", "achieved": algo / (res_step * 1e-3) / 1e9,
                         "peak": hbm_gbs, "unit": "GB/s", "frac": algo / (res_step * 1e-3) / 1e9 / hbm_gbs,
                         "algorithmic_bytes": algo},
            "cpu_baseline": {"value": nv / cpu_s, "unit": "vars/s", "cores": 1, "kind": "port",
                             "sample": f"{k} plans of the same trace, C oracle 1 thread, {cpu_s * 1e6:.0f} us each"},
            "parity": {"offsets_equal_oracle": bool(np.array_equal(offs, res.offsets_of(0))
                                                    and np.array_equal(offs, out_offs[:nv])),
                       "footprint_equal": foot == int(r["footprint_bytes"]) == plan.footprint_bytes,
                       "peak_equal": fp.peak_bytes == int(r["peak_bytes"])}}


def run_config2_leg(local_rank: int, steps: int = 20) -> dict:
    """BASELINE configs[1]: a VGG-16 b64 training iteration served from the
    SmartPool plan through the pluggable allocator (tools/config2_pool.py in
    its own process: the allocator must own the CUDA context from its first
    malloc).  Footprint vs the cnmem-style first-fit arena and PyTorch's
    caching allocator; allocator host us per call; iteration times."""
    cmd = [sys.executable, os.path.join(ROOT, "tools", "config2_pool.py"), "--batch", "64", "--steps", str(steps)]
    env = dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")[local_rank]
               if os.environ.get("CUDA_VISIBLE_DEVICES") else str(local_rank))
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
        d = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001  (the main line must still print)
        return {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
    keep = ("window_vars", "peak_load_bytes", "smartpool_footprint_bytes", "alpha", "cnmem_style_first_fit_bytes",
            "smartpool_vs_first_fit", "torch_caching_max_reserved", "torch_caching_max_allocated",
            "iter_ms_served", "iter_ms_passthrough", "iter_ms_torch_default", "hook_us_per_call",
            "hook_calls_per_iter", "served_losses_equal_passthrough")
    a = d.get("allocator", {})
    return {"workload": "VGG-16 b64 training iteration served from the plan (BASELINE configs[1])",
            "data": "synthetic (random-init VGG-16, random batch)", **{k: d.get(k) for k in keep},
            "allocator": {k: a.get(k) for k in ("hits", "misses", "conflicts")}}


SWAP_FRACS = "0.98,0.95,0.92,0.9,0.88,0.85,0.83"


def run_swap_leg(local_rank: int, fracs: str = SWAP_FRACS, steps: int = 50) -> dict:
    """BASELINE configs[2]: swap-iteration overhead % vs the same served,
    hooked iteration without swaps (tools/config3_swap.py, own process: the
    pluggable allocator must own the CUDA context from its first malloc)."""
    cmd = [sys.executable, os.path.join(ROOT, "tools", "config3_swap.py"), "--fracs", fracs,
           "--modes", "reference_selection,window_fits", "--steps", str(steps)]
    env = dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")[local_rank]
               if os.environ.get("CUDA_VISIBLE_DEVICES") else str(local_rank))
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
        d = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001  (the main line must still print)
        return {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
    bw = d["link_bw_bytes_per_s"]
    rows = []
    for l in d["limits"]:
        link = l.get("link") or {}
        ach = {k: v.get("bytes_per_s") for k, v in link.items()}
        rows.append({"mode": l["mode"], "limit_frac": l["frac"], "error": l.get("error"),
                     "selected": l.get("selected"), "executed": l.get("executed"),
                     "measured_overhead_pct": l.get("measured_overhead_pct"),
                     # the reference's simulate() under the limit; when its
                     # replay deadlocks (the reference calls the plan
                     # infeasible) this is its replay without the limit
                     "predicted_overhead_pct": l.get("predicted_overhead_pct"),
                     "reference_replay": "SwapDeadlock at the limit" if l.get("sim_limit_deadlock") else (
                         None if l.get("error") else "ok"),
                     "predicted_executed_overhead_pct": l.get("predicted_executed_overhead_pct"),
                     "pool_reduction_vs_noswap": l.get("pool_reduction_vs_noswap"),
                     "bytes_moved_per_iter": l.get("swap_bytes_per_iter"),
                     "link_achieved_bytes_per_s": ach or None,
                     "link_frac": {k: (v / bw[k] if v and bw.get(k) else None) for k, v in ach.items()} or None,
                     "losses_equal_unswapped": l.get("losses_equal_unswapped")})
    return {"workload": "VGG-16 b128 training iteration (BASELINE configs[2])",
            "metric": "swap-iter overhead % vs no-swap", "unit": "%", "higher_is_better": False,
            "data": "synthetic (random-init VGG-16, random batch)", "iter_ms_noswap": d["iter_ms_served_hooked"],
            "steps_per_row": steps, "traced_peak_bytes": d["traced_peak_bytes"],
            "load_min_frac": d["load_min_all_candidates_absent"] / d["traced_peak_bytes"],
            "link_bytes_per_s": bw,
            "link_roofline": "achieved = bytes / copy-stream busy time (CUDA events around each copy, last "
                             "iteration); frac against the measured pinned D2H / H2D rate",
            "rows": rows}


def torchrun_cmd(nproc: int, script: str, argv: list) -> list:
    """The driver's own launch line: one process per GPU on this node,
    rendezvous on 127.0.0.1 at a free port."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), script, *argv]


def main():
    if "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` outside torchrun: launch the N ranks ourselves
        pre = argparse.ArgumentParser(add_help=False)
        pre.add_argument("--gpus", type=int, default=1)
        n = pre.parse_known_args()[0].gpus
        if n > 1:
            return subprocess.run(torchrun_cmd(n, os.path.abspath(__file__), sys.argv[1:])).returncode
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--accesses", action="store_true", help="config-4 variant with write/read per var")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-5 batched sweep leg")
    ap.add_argument("--no-swap", action="store_true", help="skip the config-3 swap-overhead leg")
    ap.add_argument("--no-config1", action="store_true", help="skip the config-1 ResNet-50 plan leg")
    ap.add_argument("--no-config2", action="store_true", help="skip the config-2 served VGG-16 leg")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist.barrier()
    arrays, r = run_ours(args, rank, world, local_rank)
    r["sweep"] = None if args.no_sweep else run_sweep_bench(args, rank, world, local_rank, hbm_peak()[0])
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    if rank != 0:
        return 0
    plan = r["plan"]
    peak, peak_src = hbm_peak()
    stages = r["stages"]
    steps = args.steps
    sb = stage_bytes(r["n"], plan.period, plan.nvars, plan.nnz, plan.levels)
    per_stage = {k: ms / steps for k, (ms, _c) in stages.items()}
    dom = max(per_stage, key=per_stage.get)
    achieved = sb.get(dom, 0) / (per_stage[dom] * 1e-3) / 1e9
    # DRAM traffic per launch of the dominant kernel, from the committed ncu
    # capture (profiles/r2_ncu_kernels.json, tools/ncu_stages.sh)
    traffic = ncu_traffic({"place": "k_place_async", "conflict_fill": "k_iv_fill"}.get(dom, ""))
    stage_roof = {s: round(sb[s] / (ms * 1e-3) / 1e9 / peak, 4) for s, ms in per_stage.items() if s in sb and ms > 0}
    line = {
        "metric": METRIC, "value": r["vars_total"] / (r["step_ms"] * 1e-3), "unit": UNIT,
        "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": r["step_ms"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic",
        "config": config4(args, world, r["n"], plan.period),
        "result": {"peak_bytes": plan.peak_bytes, "footprint_bytes": plan.footprint_bytes,
                   "alpha": plan.competitive_ratio, "levels": plan.levels, "csr_entries": plan.nnz,
                   "offsets_sha256": r["sha"][:16]},
        "e2e": {"value": r["vars_total"] / (r["e2e_ms"] * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"], "ms_per_step": r["e2e_ms"]},
        "gpu_launches": r["launches"],
        "stage_ms": {k: round(v, 4) for k, v in per_stage.items()},
        "stage_ms_total": round(sum(per_stage.values()), 4),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes": sb.get(dom, 0),
                     "note": "placement is a DAG walk (depth = result.levels): latency-bound, not HBM-bound"},
        "stage_hbm_frac": stage_roof,
        "clocks": r["clocks"],
    }
    if r.get("sweep") is not None:
        line["sweep"] = r["sweep"]
    if not args.no_config1 and world == 1:
        line["config1"] = run_config1_leg(args, peak)
    if not args.no_config2 and world == 1:
        line["config2"] = run_config2_leg(local_rank)
    if not args.no_swap:
        line["swap"] = run_swap_leg(local_rank)
    if not args.no_cpu_baseline:
        cb = cpu_baseline(arrays)
        line["cpu_baseline"] = {"value": cb["value"], "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"full 1M-var trace, {cb['seconds']:.2f} s, C oracle 1 thread"}
        line["parity"] = {"footprint_equal": cb["footprint"] == plan.footprint_bytes,
                          "peak_equal": cb["peak"] == plan.peak_bytes,
                          "offsets_equal": cb["sha"] == r["sha"]}
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
