"""Synthetic workloads for the BASELINE.json configs and the parity suite.

* ``resnet50_spec`` / ``vgg16_spec`` — configs 1-3: ``WorkloadSpec`` layer
  tables with the fp32 activation/weight bytes of ResNet-50 and VGG-16 at
  224x224, salted ``+4096*(i+1)`` / ``+1024*(i+1)`` per layer so every
  layer has distinct sizes (the reference's own trick, synth.py:47-49),
  ``temp_ratio=0.5``, 3 iterations, seed 0.
* ``interval_trace`` — config 4: the 1M-variable interval trace of
  SURVEY.md §8(d), emitted straight into ``TraceArrays``.
* ``random_periodic_trace`` — randomized periodic traces with wrapping
  lifetimes, twins that nest or coexist, id reuse inside an iteration,
  carried persistents and never-freed mallocs; these drive the
  build_profile corner cases (iteration.py:189-234).
"""
from __future__ import annotations

import random

import numpy as np

from .synth import WorkloadSpec
from .trace import KIND_CODE, EventKind, Trace, TraceArrays, TraceEvent

F32 = 4


def _salted(acts, weights, name, batch, iterations, seed, temp_ratio):
    a = [x + 4096 * (i + 1) for i, x in enumerate(acts)]
    w = [x + 1024 * (i + 1) for i, x in enumerate(weights)]
    return WorkloadSpec(activation_bytes=a, weight_bytes=w, iterations=iterations,
                        seed=seed, temp_ratio=temp_ratio, name=f"{name}_b{batch}")


def resnet50_layers(batch: int):
    """(activation bytes, weight bytes) per layer: stem conv, 16 bottlenecks
    x 3 convs, fc -> 50 layers."""
    acts, wts = [], []
    acts.append(batch * 64 * 112 * 112 * F32)
    wts.append(7 * 7 * 3 * 64 * F32)
    cin = 64
    for mid, out, blocks, hw in ((64, 256, 3, 56), (128, 512, 4, 28),
                                 (256, 1024, 6, 14), (512, 2048, 3, 7)):
        for _ in range(blocks):
            for k, co, ci in ((1, mid, cin), (3, mid, mid), (1, out, mid)):
                acts.append(batch * co * hw * hw * F32)
                wts.append(k * k * ci * co * F32)
            cin = out
    acts.append(batch * 1000 * F32)
    wts.append(2048 * 1000 * F32)
    return acts, wts


def vgg16_layers(batch: int):
    """13 conv + 5 pool + 3 fc = 21 layers."""
    acts, wts = [], []
    cin, hw = 3, 224
    for block in ((64, 64), (128, 128), (256, 256, 256), (512, 512, 512), (512, 512, 512)):
        for co in block:
            acts.append(batch * co * hw * hw * F32)
            wts.append(3 * 3 * cin * co * F32)
            cin = co
        hw //= 2
        acts.append(batch * cin * hw * hw * F32)   # max-pool output
        wts.append(0)                               # salt only
    for fin, fout in ((512 * 7 * 7, 4096), (4096, 4096), (4096, 1000)):
        acts.append(batch * fout * F32)
        wts.append(fin * fout * F32)
    return acts, wts


def resnet50_spec(batch: int = 32, iterations: int = 3, seed: int = 0,
                  temp_ratio: float = 0.5) -> WorkloadSpec:
    a, w = resnet50_layers(batch)
    return _salted(a, w, "resnet50", batch, iterations, seed, temp_ratio)


def vgg16_spec(batch: int = 64, iterations: int = 3, seed: int = 0,
               temp_ratio: float = 0.5) -> WorkloadSpec:
    a, w = vgg16_layers(batch)
    return _salted(a, w, "vgg16", batch, iterations, seed, temp_ratio)


# ---------------------------------------------------------------------------
# config 4


def interval_trace(nvars: int = 1_000_000, seed: int = 0, accesses: bool = False,
                   max_len: int = 64, max_size: int = 64 << 20) -> tuple[TraceArrays, tuple[int, int]]:
    """Two iterations of ``nvars`` interval lifetimes plus a 4-op tail each.

    Var i of iteration k is malloc'd at slot 2i and freed at slot
    2*min(i+len_i, nvars-1)+1 (ops ordered by slot, then var); with
    ``accesses`` a write follows each malloc and a read precedes each free.
    ``t_us`` is the event index.  Returns the arrays and the window of the
    last iteration (the reference's detect_iteration is O(p^2) here, so the
    window is also what the CPU oracle is handed).
    """
    rng = random.Random(seed)
    sizes = np.array([rng.randrange(512, max_size) for _ in range(nvars)], dtype=np.int64)
    lens = np.array([rng.randrange(1, max_len) for _ in range(nvars)], dtype=np.int64)
    i = np.arange(nvars, dtype=np.int64)
    free_slot = 2 * np.minimum(i + lens, nvars - 1) + 1
    # per iteration: mallocs at even slots, frees at odd slots; order (slot, var)
    slot = np.concatenate([2 * i, free_slot])
    var = np.concatenate([i, i])
    is_free = np.concatenate([np.zeros(nvars, bool), np.ones(nvars, bool)])
    order = np.lexsort((var, slot))
    var, is_free = var[order], is_free[order]
    if accesses:
        # expand: malloc -> (malloc, write); free -> (read, free)
        m = var.shape[0]
        kind = np.empty(2 * m, np.uint8)
        v2 = np.repeat(var, 2)
        kind[0::2] = np.where(is_free, KIND_CODE["read"], KIND_CODE["malloc"])
        kind[1::2] = np.where(is_free, KIND_CODE["free"], KIND_CODE["write"])
        var = v2
    else:
        kind = np.where(is_free, KIND_CODE["free"], KIND_CODE["malloc"]).astype(np.uint8)
    tail_kind = np.array([KIND_CODE[k] for k in ("malloc", "write", "read", "free")], np.uint8)
    per_iter = kind.shape[0] + 4
    # var ids: x<i>.<k> for k in {0,1}, then step0, step1 -> lexicographic ranks
    names = [f"x{j}.{k}" for j in range(nvars) for k in (0, 1)] + ["step0", "step1"]
    sorted_names = sorted(names)
    rank = {nm: r for r, nm in enumerate(sorted_names)}
    xrank = np.array([rank[f"x{j}.{k}"] for j in range(nvars) for k in (0, 1)],
                     dtype=np.int32).reshape(nvars, 2)
    kinds, vids, szs = [], [], []
    for k in (0, 1):
        vid = xrank[var, k]
        sz = np.where(kind == KIND_CODE["malloc"], sizes[var], 0)
        kinds += [kind, tail_kind]
        vids += [vid, np.full(4, rank[f"step{k}"], np.int32)]
        szs += [sz, np.array([1, 0, 0, 0], np.int64)]
    kind_all = np.concatenate(kinds)
    n = kind_all.shape[0]
    arrays = TraceArrays(kind_all, np.concatenate(vids), np.concatenate(szs),
                         np.arange(n, dtype=np.int64), sorted_names)
    return arrays, (n - per_iter, n)


# ---------------------------------------------------------------------------
# randomized periodic traces for the lifetime corner cases


def random_periodic_trace(seed: int, slots: int = 40, nvars: int = 10,
                          iterations: int = 5, max_wrap: float = 2.2,
                          n_persistent: int = 2, n_leak: int = 1,
                          n_reuse: int = 2, zero_dt: float = 0.2) -> Trace:
    """Periodic trace over a random one-iteration template.

    Template vars may outlive the iteration (up to ``max_wrap`` periods),
    which produces carry-ins whose next-iteration twin either nests
    (merge), overlaps (coexist), or lies beyond the previous window (no
    twin).  ``r<j>`` names are reused every iteration and several times
    inside one, so windows hold multiple instances of one base name.
    """
    rng = random.Random(seed)
    S = slots
    ops = []  # (global_pos, order_key, kind, name_fn, size)
    sizes_used = set()

    def fresh_size(lo=1, hi=1 << 20):
        while True:
            s = rng.randrange(lo, hi)
            if s not in sizes_used:
                sizes_used.add(s)
                return s

    template = []  # per var: (malloc slot, lifetime, size, access offsets, kind)
    for j in range(nvars):
        m = rng.randrange(0, S)
        life = rng.randrange(1, max(2, int(max_wrap * S)))
        acc = sorted(rng.sample(range(1, life), min(life - 1, rng.randrange(0, 4)))) if life > 1 else []
        template.append((m, life, fresh_size(), acc))
    reuse = []
    for j in range(n_reuse):
        reps = []
        pos = rng.randrange(0, S // 2)
        for _ in range(rng.randrange(1, 4)):
            if pos + 2 >= S:
                break
            life = rng.randrange(1, max(2, min(8, S - pos - 1)))
            reps.append((pos, life))
            pos += life + rng.randrange(1, 4)
        reuse.append((reps, fresh_size()))
    persist = [(fresh_size(), sorted(rng.sample(range(S), rng.randrange(1, 4))))
               for _ in range(n_persistent)]
    leaks = [(rng.randrange(S), fresh_size()) for _ in range(n_leak)]

    pre = []
    for j, (sz, _) in enumerate(persist):
        pre.append(("malloc", f"p{j}", sz))
        pre.append(("write", f"p{j}", 0))
    base = len(pre)
    total = S * iterations
    for k in range(iterations):
        off = k * S
        for j, (m, life, sz, acc) in enumerate(template):
            name = f"v{j}.{k}"
            ops.append((off + m, 1, j, "malloc", name, sz))
            for a in acc:
                if off + m + a < total:
                    ops.append((off + m + a, 2, j, "read" if a % 2 else "write", name, 0))
            if off + m + life < total:
                ops.append((off + m + life, 0, j, "free", name, 0))
        for j, (reps, sz) in enumerate(reuse):
            for pos, life in reps:
                ops.append((off + pos, 1, 1000 + j, "malloc", f"r{j}", sz))
                ops.append((off + pos + life, 0, 1000 + j, "free", f"r{j}", 0))
        for j, (sz, acc) in enumerate(persist):
            for a in acc:
                ops.append((off + a, 2, 2000 + j, "read", f"p{j}", 0))
        for j, (pos, sz) in enumerate(leaks):
            ops.append((off + pos, 1, 3000 + j, "malloc", f"leak{j}.{k}", sz))
        # aperiodic-suffix guard, like the generator's step tail (synth.py:152-159)
        ops.append((off + S - 1, 9, 0, "malloc", f"end{k}", 3))
        ops.append((off + S - 1, 9, 1, "write", f"end{k}", 0))
        ops.append((off + S - 1, 9, 2, "free", f"end{k}", 0))
    ops.sort(key=lambda o: (o[0], o[1], o[2], o[4]))
    seq = pre + [(o[3], o[4], o[5]) for o in ops]
    events, t = [], 0
    for i, (kind, var, size) in enumerate(seq):
        events.append(TraceEvent(i, t, EventKind(kind), var, size))
        t += 0 if rng.random() < zero_dt else rng.randrange(1, 25)
    return Trace(events=events, meta={"template_period": S})


# ---------------------------------------------------------------------------
# config 5


SWEEP_BUDGETS = (0.9, 0.8, 0.7, 0.6)


def sweep_specs(n_models: int = 64, n_scales: int = 16, iterations: int = 3, seed: int = 0):
    """The (model shape x batch scale) grid of BASELINE configs[4]: model 0
    is VGG-16, model 1 ResNet-50 (batch 8 * (s + 1)), the rest ``vgg_like``
    depths 6-16 with alternating temporaries and their own seeds (activation
    scale (s + 1) / 8).  With 4 budgets per trace, 64 x 16 x 4 = 4096 units."""
    from .synth import vgg_like
    specs = []
    for m in range(n_models):
        for s in range(n_scales):
            sd = seed + 1000 * m + s
            if m == 0:
                specs.append(vgg16_spec(batch=8 * (s + 1), iterations=iterations, seed=sd))
            elif m == 1:
                specs.append(resnet50_spec(batch=8 * (s + 1), iterations=iterations, seed=sd))
            else:
                depth = 6 + (m - 2) % 11
                specs.append(vgg_like(depth=depth, scale=(s + 1) / 8, iterations=iterations, seed=sd,
                                      temp_ratio=0.5 if m % 2 else 0.0))
    return specs


def sweep_traces(n_models: int = 64, n_scales: int = 16, iterations: int = 3, seed: int = 0):
    from .synth import generate_synthetic_trace
    return [generate_synthetic_trace(sp) for sp in sweep_specs(n_models, n_scales, iterations, seed)]
