"""Scenario builders shared by the golden generator and the parity tests.

Hand traces restate the reference fixtures' shapes (pkg/tests/conftest.py:
21-82 and the inline traces of test_iteration.py / test_autoswap.py /
test_smartpool.py); the rest are generator, config, randomized-periodic,
interval and raw-arc instances built with this repo's own builders.
"""
from __future__ import annotations

import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from paper_1903_06631_b200 import synth, workloads  # noqa: E402
from paper_1903_06631_b200.trace import EventKind, Trace, TraceEvent  # noqa: E402

MIB = 1 << 20
MB = 10 ** 6


def ops_trace(ops, spacing=10):
    """(kind, var, size) tuples -> Trace with evenly spaced timestamps."""
    return Trace(events=[TraceEvent(i, spacing * i, EventKind(k), v, s)
                         for i, (k, v, s) in enumerate(ops)])


def _congested(iterations=2):
    one = [("malloc", "w1", 25 * MIB), ("write", "w1", 0), ("malloc", "w2", 25 * MIB),
           ("write", "w2", 0), ("malloc", "w3", 25 * MIB), ("write", "w3", 0),
           ("malloc", "a", 45 * MIB), ("write", "a", 0), ("free", "a", 0),
           ("malloc", "b", 20 * MIB), ("write", "b", 0), ("free", "b", 0),
           ("read", "w3", 0), ("free", "w3", 0), ("read", "w2", 0), ("free", "w2", 0),
           ("read", "w1", 0), ("write", "w1", 0), ("free", "w1", 0)]
    return one * iterations


def _three_var(iterations=2):
    one = [("malloc", "v1", 45 * MB), ("write", "v1", 0), ("malloc", "v2", 40 * MB),
           ("write", "v2", 0), ("malloc", "v3", 34 * MB), ("write", "v3", 0),
           ("malloc", "t", 1 * MB), ("free", "t", 0), ("read", "v1", 0), ("free", "v1", 0),
           ("read", "v2", 0), ("free", "v2", 0), ("read", "v3", 0), ("write", "v3", 0),
           ("free", "v3", 0)]
    return one * iterations


def _filter_instance():
    ops = []
    for k in (1, 2):
        ops += [("malloc", f"F{k}", 2 * MIB), ("write", f"F{k}", 0), ("read", f"F{k}", 0),
                ("free", f"F{k}", 0), ("malloc", f"B{k}", 2 * MIB), ("write", f"B{k}", 0),
                ("malloc", f"s{k}", 500_000), ("write", f"s{k}", 0),
                ("malloc", f"T{k}", 3 * MIB), ("free", f"T{k}", 0), ("read", f"s{k}", 0),
                ("free", f"s{k}", 0), ("write", f"B{k}", 0), ("free", f"B{k}", 0)]
    return ops


def _doubled(copies=2):
    return [(k, f"a{c}.{i}", (i + 1) if k == "malloc" else 0)
            for c in range(copies) for i in range(6) for k in ("malloc", "free")]


def _plain_window():
    ops = [("malloc", "w", 5), ("write", "w", 0)]
    for k in (1, 2):
        ops += [("read", "w", 0), ("read", "w", 0), ("malloc", f"x{k}", 10),
                ("write", f"x{k}", 0), ("read", f"x{k}", 0), ("read", "w", 0),
                ("read", "w", 0), ("free", f"x{k}", 0)]
    return ops


def _xy(ysize):
    ops = []
    for k in (1, 2):
        ops += [("malloc", f"x{k}", 10), ("write", f"x{k}", 0), ("read", f"x{k}", 0),
                ("read", f"x{k}", 0), ("free", f"x{k}", 0), ("malloc", f"y{k}", ysize),
                ("write", f"y{k}", 0), ("free", f"y{k}", 0)]
    return ops


def _nest():
    ops = [("malloc", "b0", 8), ("write", "b0", 0)]
    for k in (1, 2, 3):
        ops += [("read", f"b{k-1}", 0), ("free", f"b{k-1}", 0), ("malloc", f"b{k}", 8),
                ("write", f"b{k}", 0), ("malloc", f"s{k}", 1), ("free", f"s{k}", 0)]
    return ops


def _coexist():
    ops = [("malloc", "a0", 8), ("write", "a0", 0)]
    for k in (1, 2, 3):
        ops += [("malloc", f"a{k}", 8), ("write", f"a{k}", 0), ("free", f"a{k-1}", 0)]
    return ops


def _unfreed():
    ops = []
    for k in (1, 2):
        ops += [("malloc", f"keep{k}", 4), ("write", f"keep{k}", 0),
                ("malloc", f"tmp{k}", 9), ("read", f"tmp{k}", 0), ("free", f"tmp{k}", 0)]
    return ops


def _span():
    ops = [("malloc", "w", 2 * MIB), ("write", "w", 0)]
    for k in (1, 2):
        ops += [("malloc", f"a{k}", 5 * MIB), ("write", f"a{k}", 0), ("free", f"a{k}", 0),
                ("read", "w", 0), ("malloc", f"s{k}", 1), ("free", f"s{k}", 0)]
    return ops


def _aperiodic():
    return [(k, f"a{i}", (i + 1) if k == "malloc" else 0) for i in range(25)
            for k in ("malloc", "free")]


def _lookup_a9(n=10000):
    return [(k, f"v{i:05d}", (1024 + i) if k == "malloc" else 0)
            for _ in range(2) for i in range(n) for k in ("malloc", "free")]


DEFAULT_T = (12e9, 10.0, MIB)
FAST_T = (1e12, 0.1, MIB)
SLOW_T = (2e9, 10.0, MIB)
PCIE_T = (50e9, 10.0, MIB)


def hand_group():
    S = []

    def add(name, ops, transfers=(DEFAULT_T,), fracs=(0.9, 0.75, 0.6), **kw):
        S.append(dict(name=name, trace=ops_trace(ops), transfers=transfers, fracs=fracs, **kw))
    add("congested", _congested(), transfers=(DEFAULT_T, FAST_T, (1e18, 0.0, MIB)),
        fracs=(95 / 120, 0.5, 0.45))
    add("congested3", _congested(3))
    add("three_var", _three_var(), transfers=(DEFAULT_T, FAST_T, (1e18, 0.0, MIB),
                                              (float("inf"), 0.0, MIB)),
        fracs=(0.5, 0.375))
    add("filter_instance", _filter_instance(),
        transfers=(DEFAULT_T, FAST_T, (1e9, 3.0, MIB), (12e9, 10.0, 500_000), (12e9, 10.0, 1)),
        fracs=((3 * MIB + 500_000) / (5 * MIB + 500_000 + 3 * MIB), 0.8))
    add("doubled", _doubled())
    add("doubled3", _doubled(3))
    add("plain_window", _plain_window())
    add("disjoint", _xy(10))
    add("step_zero", _xy(3))
    add("nest", _nest(), transfers=((12e9, 10.0, 1),))
    add("coexist", _coexist(), transfers=((12e9, 10.0, 1),))
    add("unfreed", _unfreed(), transfers=((12e9, 10.0, 1),))
    add("span", _span(), transfers=(DEFAULT_T, FAST_T))
    add("aperiodic", _aperiodic())
    add("short", [("malloc", "a", 5), ("write", "a", 0), ("read", "a", 0)])
    add("single", [("malloc", "a", 5)])
    add("a9_lookup", _lookup_a9(), transfers=())
    # invariant violations (validate only; trace.py:55-84 reasons)
    bad = {
        "free_first": [("free", "v1", 0), ("malloc", "v1", 10)],
        "use_after_free": [("malloc", "v1", 10), ("free", "v1", 0), ("read", "v1", 0)],
        "double_free": [("malloc", "v1", 10), ("free", "v1", 0), ("free", "v1", 0)],
        "malloc_live": [("malloc", "v1", 10), ("malloc", "v2", 3), ("malloc", "v1", 4)],
        "zero_malloc": [("malloc", "v1", 0)],
        "sized_read": [("malloc", "v1", 10), ("read", "v1", 7)],
        "sized_free": [("malloc", "v1", 10), ("free", "v1", 10)],
        "neg_malloc": [("malloc", "v1", 10), ("malloc", "v2", -5)],
    }
    for name, ops in bad.items():
        S.append(dict(name="bad_" + name, trace=ops_trace(ops), validate_only=True))
    # timestamp / index faults
    t = ops_trace([("malloc", "a", 4), ("write", "a", 0), ("free", "a", 0)])
    t.events[2] = TraceEvent(2, 5, EventKind.FREE, "a", 0)
    S.append(dict(name="bad_t_decrease", trace=t, validate_only=True))
    t = ops_trace([("malloc", "a", 4), ("write", "a", 0)])
    t.events[0] = TraceEvent(0, -3, EventKind.MALLOC, "a", 4)
    S.append(dict(name="bad_t_negative", trace=t, validate_only=True))
    t = ops_trace([("malloc", "a", 4), ("write", "a", 0), ("free", "a", 0)])
    t.events[1] = TraceEvent(5, 10, EventKind.WRITE, "a", 0)
    S.append(dict(name="bad_index_gap", trace=t, validate_only=True))
    return S


def generator_group():
    S = []
    shapes = [(5, 0.5, 5, 0, 0.5), (5, 0.4, 4, 0, 0.5), (5, 0.4, 4, 4, 0.5), (7, 0.4, 4, 1, 0.5),
              (8, 0.5, 3, 1, 0.0), (6, 1.0, 3, 2, 0.0), (10, 0.25, 4, 3, 0.0),
              (5, 1.0, 4, 4, 0.5), (6, 0.5, 4, 7, 0.5), (4, 0.25, 3, 0, 0.5),
              (12, 4.0, 3, 0, 0.5), (8, 1.0, 3, 0, 0.5), (3, 0.3, 4, 3, 0.9),
              (16, 0.5, 3, 5, 0.5), (9, 0.75, 6, 8, 0.3)]
    for d, sc, it, seed, tr in shapes:
        spec = synth.vgg_like(depth=d, scale=sc, iterations=it, seed=seed, temp_ratio=tr)
        S.append(dict(name=f"vgg_like_d{d}_s{sc}_i{it}_seed{seed}_t{tr}",
                      trace=synth.generate_synthetic_trace(spec),
                      transfers=(DEFAULT_T, SLOW_T, PCIE_T), fracs=(0.95, 0.9, 0.8, 0.75, 0.6, 0.5)))
    return S


def config_group():
    S = []
    for name, spec in (("resnet50_b32", workloads.resnet50_spec(32)),
                       ("vgg16_b64", workloads.vgg16_spec(64)),
                       ("vgg16_b128", workloads.vgg16_spec(128))):
        S.append(dict(name=name, trace=synth.generate_synthetic_trace(spec),
                      transfers=(DEFAULT_T, PCIE_T, (25e9, 10.0, MIB)),
                      fracs=(0.95, 0.9, 0.8, 0.691, 0.6)))
    return S


def random_group(count=40):
    S = []
    for seed in range(count):
        rng = random.Random(1000 + seed)
        kw = dict(slots=rng.choice((12, 24, 40, 64)), nvars=rng.randrange(2, 16),
                  iterations=rng.randrange(4, 7), max_wrap=rng.choice((0.9, 1.5, 2.2, 3.0)),
                  n_persistent=rng.randrange(0, 3), n_leak=rng.randrange(0, 2),
                  n_reuse=rng.randrange(0, 3), zero_dt=rng.choice((0.0, 0.2, 0.5)))
        S.append(dict(name=f"periodic_{seed}", trace=workloads.random_periodic_trace(seed, **kw),
                      transfers=((12e9, 10.0, 1), (1e9, 1.0, 1000)), fracs=(0.9, 0.75, 0.6)))
    return S


def interval_group():
    S = []
    for nv, acc in ((300, False), (300, True), (3000, True)):
        arrays, window = workloads.interval_trace(nvars=nv, seed=nv, accesses=acc,
                                                  max_size=8 << 20)
        S.append(dict(name=f"interval_{nv}_{int(acc)}", trace=arrays.to_trace(),
                      transfers=((50e9, 10.0, 1 << 20),) if acc else (), fracs=(0.9,)))
    return S


def arcs_group():
    S = []
    rng = random.Random(77)
    for case in range(60):
        n = rng.randrange(2, 60 if case < 50 else 400)
        period = rng.choice((10, 100, 1000))
        arcs = []
        for i in range(n):
            nseg = 1 if case < 20 else rng.randrange(1, 4)
            segs = []
            for _ in range(nseg):
                lo = rng.randrange(0, period - 1)
                hi = rng.randrange(lo, period + 1)   # may be empty
                segs.append([lo, hi])
            size = rng.choice((rng.randrange(1, 64), rng.randrange(1024, 1 << 26), 4096))
            alloc = rng.choice((-1, rng.randrange(0, period)))
            arcs.append([f"n{rng.randrange(0, 10 * n):04d}_{i}", size, alloc, segs,
                         rng.random() < 0.05])
        peak = 0
        S.append(dict(kind="arcs", name=f"arcs_{case}", arcs=arcs, period=period, peak=peak))
    return S


def synthetic_group():
    S = []

    def cand(var, gap, d, size, out_index, in_index, out_time, spans=False, d_in=None):
        return [var, size, out_index, float(out_time), float(out_time), in_index,
                float(out_time + gap), float(d), float(d if d_in is None else d_in), spans]
    # divergence fixture shape (test_autoswap.py:145-155)
    S.append(dict(kind="synthetic", name="divergence", loads=[10, 100, 100, 0, 90, 0], spacing=10.0,
                  cands=[cand("A", 30, 1, 60, 0, 3, 0), cand("B", 20, 1, 70, 1, 3, 10),
                         cand("C", 20, 1, 50, 3, 5, 30)], limits=[45, 99, 100, 10]))
    S.append(dict(kind="synthetic", name="rect", loads=[150] * 6, spacing=10.0,
                  cands=[cand("x", 50, 1, 1 << 20, 1, 5, 10), cand("y", 30, 1, 1 << 20, 4, 1, 40, True)],
                  limits=[100, 1]))
    rng = random.Random(21)
    for k in range(40):
        p = rng.choice((12, 30))
        loads = [rng.randrange(0, 1000) for _ in range(p)]
        cs = []
        for i in range(rng.randint(2, 9)):
            lo = rng.randrange(0, p - 2)
            hi = rng.randrange(lo + 1, p)
            sz = rng.randrange(50, 400)
            if rng.random() < 0.3:
                sz = 100  # size ties
            cs.append(cand(f"c{rng.randrange(0, 5)}{i}", 10.0 * (hi - lo), 1.0, sz, lo, hi, 10.0 * lo))
        S.append(dict(kind="synthetic", name=f"greedy_{k}", loads=loads, spacing=rng.choice((10.0, 0.1, 3.3)),
                      cands=cs, limits=[rng.randrange(200, 900), max(loads), 0]))
    return S


def all_groups():
    return {"hand": hand_group(), "generator": generator_group(), "configs": config_group(),
            "periodic": random_group(), "interval": interval_group(), "arcs": arcs_group(),
            "synthetic": synthetic_group()}
