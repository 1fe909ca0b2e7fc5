"""Serve a PyTorch training iteration from a SmartPool plan.

The paper's runtime side ("lookup-table allocation"):
  1. ``install()`` routes every CUDA allocation of the process through
     ``libmemplan_alloc.so`` (``torch.cuda.memory.CUDAPluggableAllocator``);
     call it before the first CUDA allocation.
  2. ``Tracer`` records one or more iterations as a memplan trace: the
     allocator logs malloc/free (sizes rounded to 512 B), a
     ``TorchDispatchMode`` logs each aten op's reads and writes, and ops are
     timestamped after a device synchronize (capture only).
  3. ``plan_iteration`` runs the device pipeline (detect, extract, conflict
     graph, plan_pool) and returns the window's malloc slots.
  4. ``serve(plan)`` makes the k-th allocation of every later iteration
     return pool_base + offset_k; frees are no-ops; a size mismatch falls
     back to cudaMallocAsync and is counted.
"""
from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ALLOC_LIB = os.path.join(HERE, "libmemplan_alloc.so")
MARK_NAME = "~iteration"

_ctl = None


def ctl():
    global _ctl
    if _ctl is None:
        L = C.CDLL(ALLOC_LIB)
        L.mp_alloc_log_size.restype = C.c_int64
        L.mp_alloc_pool_base.restype = C.c_int64
        L.mp_alloc_set_seq.argtypes = [C.c_int64]
        _ctl = L
    return _ctl


def install():
    """Route this process's CUDA allocations through the plan-serving allocator."""
    import torch
    alloc = torch.cuda.memory.CUDAPluggableAllocator(ALLOC_LIB, "mp_torch_alloc", "mp_torch_free")
    torch.cuda.memory.change_current_allocator(alloc)
    ctl()


def stats() -> dict:
    out = (C.c_int64 * 10)()
    ctl().mp_alloc_stats(out)
    return {"hits": out[0], "misses": out[1], "pool_bytes": out[2], "outside_live_bytes": out[3],
            "outside_peak_bytes": out[4], "ordinal": out[5], "conflicts": out[6], "pool_live_blocks": out[7],
            "swap_alias_fallbacks": out[8], "retired_pools_mapped": out[9], **call_stats()}


def call_stats() -> dict:
    """Host cost of the allocator hooks since the last reset: calls and mean
    microseconds per call (lock wait included)."""
    out = (C.c_int64 * 4)()
    ctl().mp_alloc_call_stats(out)
    return {"alloc_calls": out[0], "alloc_ns": out[1], "free_calls": out[2], "free_ns": out[3],
            "alloc_us_per_call": out[1] / out[0] / 1e3 if out[0] else None,
            "free_us_per_call": out[3] / out[2] / 1e3 if out[2] else None}


class Tracer:
    """Record allocations + per-op reads/writes of the code run inside it."""

    def __init__(self, sync_times: bool = True, dispatch: bool = True, device_times: bool = False):
        """dispatch=False records allocations only (no per-op reads/writes,
        timestamps = event order): the program runs exactly as when served,
        so the recorded lifetimes are the served ones (enough for pool
        planning; swap planning needs the accesses and op times).
        device_times=True stamps each op with a CUDA event recorded before
        it instead of synchronising: op times are the device timeline of an
        unsynchronised run (what a swap plan must hide transfers behind)."""
        from torch.utils._python_dispatch import TorchDispatchMode
        tracer = self
        self.sync_times = sync_times and not device_times
        self.device_times = device_times
        self._events = []  # (seq, cuda event) when device_times
        self.dispatch = dispatch
        self.ops = []  # (seq, t_us, [read ptrs], [write ptrs])
        self.spans = {}  # seq -> allocator-log range [lo, hi) recorded inside the op
        self.seq = 0
        self.t0 = None
        self.hook = None  # executor callbacks around each op (swapexec)
        self.record = True

        class Mode(TorchDispatchMode):
            def __torch_dispatch__(self, func, types, args=(), kwargs=None):
                return tracer._dispatch(func, args, kwargs or {})
        self._mode = Mode()

    @staticmethod
    def _ptrs(obj, out):
        import torch
        if isinstance(obj, torch.Tensor):
            if obj.is_cuda:
                try:
                    out.append(obj.untyped_storage().data_ptr())
                except Exception:  # noqa: BLE001
                    pass
        elif isinstance(obj, (list, tuple)):
            for x in obj:
                Tracer._ptrs(x, out)
        elif isinstance(obj, dict):
            for x in obj.values():
                Tracer._ptrs(x, out)

    def _dispatch(self, func, args, kwargs):
        import torch
        self.seq += 1
        ctl().mp_alloc_set_seq(self.seq)
        if self.sync_times:
            torch.cuda.synchronize()
        t = int((time.perf_counter() - self.t0) * 1e6)
        if self.device_times:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self._events.append((self.seq, ev))
        reads = []
        self._ptrs(args, reads)
        self._ptrs(kwargs, reads)
        lo = int(ctl().mp_alloc_log_size())
        if self.hook is not None:
            self.hook.before(self.seq)
        out = func(*args, **kwargs)
        if self.hook is not None:
            self.hook.after(self.seq)
        self.spans[self.seq] = (lo, int(ctl().mp_alloc_log_size()))
        writes = []
        self._ptrs(out, writes)
        # in-place / out= ops write their mutated inputs too
        schema = getattr(func, "_schema", None)
        if schema is not None:
            for i, a in enumerate(schema.arguments):
                if a.alias_info is not None and a.alias_info.is_write and i < len(args):
                    self._ptrs(args[i], writes)
        self.ops.append((self.seq, t, reads, writes))
        return out

    def mark(self):
        """End-of-iteration marker: a synthetic 1-byte malloc/write/read/free
        (like the generator's step tail, synth.py:152-159) so the trace suffix
        never collapses into a short fingerprint period; not a real
        allocation, so it is excluded from the served slots."""
        import torch
        self.seq += 1
        ctl().mp_alloc_set_seq(self.seq)
        if self.sync_times:
            torch.cuda.synchronize()
        t = int((time.perf_counter() - self.t0) * 1e6)
        if self.device_times:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self._events.append((self.seq, ev))
        if not self.dispatch:
            t = self.seq
        self.marks.append((self.seq, t))
        n = int(ctl().mp_alloc_log_size())
        self.spans[self.seq] = (n, n)
        self.ops.append((self.seq, t, [], []))

    def __enter__(self):
        import torch
        self.marks = []
        torch.cuda.synchronize()
        self.t0 = time.perf_counter()
        if self.device_times:
            self._ev0 = torch.cuda.Event(enable_timing=True)
            self._ev0.record()
        self._drain()
        ctl().mp_alloc_set_seq(self.seq)
        ctl().mp_alloc_logging(1)
        if self.dispatch:
            self._mode.__enter__()
        return self

    def __exit__(self, *exc):
        if self.dispatch:
            self._mode.__exit__(*exc)
        import torch
        torch.cuda.synchronize()
        ctl().mp_alloc_logging(0)
        self.alloc_log = self._drain()
        if self.device_times:
            t_of = {s: int(self._ev0.elapsed_time(ev) * 1000.0) for s, ev in self._events}
            self.ops = [(s, t_of.get(s, t), r, w) for s, t, r, w in self.ops]
            self.marks = [(s, t_of.get(s, t)) for s, t in self.marks]
            self._events = []

    @staticmethod
    def _drain():
        n = int(ctl().mp_alloc_log_size())
        cols = [np.zeros(max(n, 1), dt) for dt in (np.int64, np.int32, np.int64, np.int64)]
        ctl().mp_alloc_log_drain(*(c.ctypes.data_as(C.c_void_p) for c in cols))
        return [c[:n] for c in cols]

    def trace(self):
        """Merge allocator and dispatch logs into TraceArrays.  Dispatch
        mode: per op its reads, the allocator records made inside it (log
        order), its writes; ``self.event_seq[i]`` = the op ordinal event i
        belongs to (what a swap executor keys its actions on)."""
        from .trace import KIND_CODE, TraceArrays
        seq, kind, ptr, size = self.alloc_log
        live: dict[int, str] = {}
        counter = 0
        kinds, names, sizes, times = [], [], [], []

        def emit(k, name, z, t):
            kinds.append(KIND_CODE[k])
            names.append(name)
            sizes.append(z)
            times.append(t)
        if not self.dispatch:
            # allocator log order is the ground truth; marks sit between the
            # records of consecutive sequence numbers
            pending = sorted(s for s, _t in self.marks)
            mi = 0
            for s, k, p, z in zip(seq.tolist(), kind.tolist(), ptr.tolist(), size.tolist()):
                while mi < len(pending) and pending[mi] <= s:
                    for kk in ("malloc", "write", "read", "free"):
                        emit(kk, MARK_NAME, 1 if kk == "malloc" else 0, 0)
                    mi += 1
                if k == 0:
                    if p in live:
                        emit("free", live.pop(p), 0, 0)
                    counter += 1
                    live[p] = f"a{counter:07d}"
                    emit("malloc", live[p], z, 0)
                elif p in live:
                    emit("free", live.pop(p), 0, 0)
            for _ in pending[mi:]:
                for kk in ("malloc", "write", "read", "free"):
                    emit(kk, MARK_NAME, 1 if kk == "malloc" else 0, 0)
            return TraceArrays.from_columns(np.array(kinds, np.uint8), names, np.array(sizes, np.int64),
                                            np.arange(len(kinds), dtype=np.int64))
        # dispatch mode: per op, its reads, the allocator records made inside
        # it (log order), its writes; records between ops follow in log order
        nlog = len(seq)
        recs = list(zip(kind.tolist(), ptr.tolist(), size.tolist()))
        mark_seqs = {s for s, _t in self.marks}
        pos = 0
        self.event_seq = []
        self._event_where = []  # 0: at/inside the op, 1: between it and the next

        def run_recs(upto, t, s, where=0):
            nonlocal pos, counter
            while pos < upto:
                k, p, z = recs[pos]
                pos += 1
                if k == 0:
                    if p in live:
                        emit("free", live.pop(p), 0, t)
                        self.event_seq.append(s)
                        self._event_where.append(where)
                    counter += 1
                    live[p] = f"a{counter:07d}"
                    emit("malloc", live[p], z, t)
                    self.event_seq.append(s)
                    self._event_where.append(where)
                elif p in live:
                    emit("free", live.pop(p), 0, t)
                    self.event_seq.append(s)
                    self._event_where.append(where)
        t_prev = 0
        for s, t, reads, writes in self.ops:
            lo, hi = self.spans[s]
            run_recs(lo, t_prev, s - 1, 1)   # records between the previous op and this one
            if s in mark_seqs:
                for k in ("malloc", "write", "read", "free"):
                    emit(k, MARK_NAME, 1 if k == "malloc" else 0, t)
                    self.event_seq.append(s)
                    self._event_where.append(0)
                continue
            for p in dict.fromkeys(reads):
                if p in live:
                    emit("read", live[p], 0, t)
                    self.event_seq.append(s)
                    self._event_where.append(0)
            run_recs(hi, t, s)
            for p in dict.fromkeys(writes):
                if p in live:
                    emit("write", live[p], 0, t)
                    self.event_seq.append(s)
                    self._event_where.append(0)
            t_prev = t
        run_recs(nlog, t_prev, self.seq, 1)
        return TraceArrays.from_columns(np.array(kinds, np.uint8), names, np.array(sizes, np.int64),
                                        np.array(times, np.int64))


def plan_iteration(arrays, policy: str = "best_fit"):
    """Device plan of the last detected iteration; returns (plan, profile, slots).

    slots: (offset, size) per window malloc in allocation order — what the
    allocator serves in that order every iteration.
    """
    from . import iteration, smartpool
    det = iteration.detect_iteration(arrays)
    prof = iteration.extract_lifetimes(arrays, det.window)
    g = smartpool.build_conflict_graph(prof)
    plan = smartpool.plan_pool(g, policy)
    table = smartpool.make_lookup_table(plan, prof)
    items = [it for it in table.items() if not it[1][0].startswith(MARK_NAME)]  # real mallocs, in order
    sizes = plan.sizes
    off = np.array([o for _r, (_v, o) in items], np.int64)
    siz = np.array([sizes[v] for _r, (v, _o) in items], np.int64)
    return plan, prof, (off, siz)


def serve(footprint: int, slots) -> None:
    off, siz = slots
    off = np.ascontiguousarray(off, np.int64)
    siz = np.ascontiguousarray(siz, np.int64)
    rc = ctl().mp_alloc_set_plan(C.c_int64(int(footprint)), C.c_int64(off.shape[0]),
                                 off.ctypes.data_as(C.c_void_p), siz.ctypes.data_as(C.c_void_p))
    if rc:
        raise MemoryError(f"could not reserve a {footprint}-byte pool")
    ctl().mp_alloc_mode(1)


def clash_log(cap: int = 192) -> list:
    """(served iteration, malloc ordinal, other block as iteration<<20|ordinal)
    for the first slot clashes (recorded lifetimes not matching the run)."""
    buf = (C.c_int64 * cap)()
    ctl().mp_alloc_clash_log.restype = C.c_int64
    n = ctl().mp_alloc_clash_log(buf, C.c_int64(cap))
    v = list(buf)[:min(n, cap)]
    return [(v[i], v[i + 1], (v[i + 2] >> 20, v[i + 2] & 0xFFFFF)) for i in range(0, len(v) - 2, 3)]


def begin_iteration() -> None:
    ctl().mp_alloc_begin_iteration()


def passthrough() -> None:
    ctl().mp_alloc_mode(0)


def first_fit_arena_peak(arrays, window) -> int:
    """Footprint an online address-ordered first-fit arena (CnMem-style,
    PAPER.md:58,304) reaches on the window: blocks live at the window start
    are allocated first, then mallocs/frees replay in order.  A comparison
    baseline, not part of the planner."""
    start, end = window
    kind, var, size = arrays.kind, arrays.var, arrays.size
    live_sz = {}
    for i in range(start):
        if kind[i] == 0:
            live_sz[int(var[i])] = int(size[i])
        elif kind[i] == 1:
            live_sz.pop(int(var[i]), None)
    free_list = []  # sorted (offset, length) holes
    top = 0
    where = {}

    def alloc(n):
        nonlocal top
        for idx, (o, ln) in enumerate(free_list):
            if ln >= n:
                if ln == n:
                    free_list.pop(idx)
                else:
                    free_list[idx] = (o + n, ln - n)
                return o
        o = top
        top += n
        return o

    def release(o, n):
        nonlocal top
        free_list.append((o, n))
        free_list.sort()
        merged = []
        for a, ln in free_list:
            if merged and merged[-1][0] + merged[-1][1] == a:
                merged[-1] = (merged[-1][0], merged[-1][1] + ln)
            else:
                merged.append((a, ln))
        if merged and merged[-1][0] + merged[-1][1] == top:
            top = merged[-1][0]
            merged.pop()
        free_list[:] = merged

    peak = 0
    for v, n in live_sz.items():
        where[v] = (alloc(n), n)
    peak = top
    for i in range(start, end):
        k, v = int(kind[i]), int(var[i])
        if k == 0:
            where[v] = (alloc(int(size[i])), int(size[i]))
            peak = max(peak, top)
        elif k == 1 and v in where:
            release(*where.pop(v))
    return peak
