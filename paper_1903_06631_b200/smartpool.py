"""SmartPool: conflict graph and static pool layout (drop-in for memplan.smartpool).

Reference: pkg/src/memplan/smartpool.py:19-254.  The conflict graph is
built on the device as a CSR (csrc/conflict.cu) and planned there
(csrc/placement.cu); ``ConflictGraph.vars`` / ``.adj`` and
``PoolPlan.offsets`` / ``.sizes`` materialize the reference's Python
containers only when read.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import GraphTooLarge, MemplanError, MissingVariable
from ._abi import F_PERSISTENT
from .iteration import IterationProfile, Segment, device_profile

POLICY_CODE = {"first_fit": 0, "best_fit": 1}


@dataclass
class PoolVar:
    var: str
    size: int
    alloc_index: int
    segments: tuple[Segment, ...]
    persistent: bool


def _freeze_vars(vars_):
    return None if vars_ is None else tuple((pv.var, pv.size, pv.alloc_index) for pv in vars_)


def _freeze_adj(adj):
    return None if adj is None else tuple(frozenset(a) for a in adj)


class ConflictGraph:
    """Weighted interval-conflict graph (smartpool.py:28-33).

    ``vars`` and ``adj`` are plain mutable Python containers, as in the
    reference; the device CSR built from (or uploaded for) them is reused
    only while the values it was built from compare equal, so an in-place
    edit (``g.adj[i].add(j)``, ``g.vars[k].size = ...``) is planned as the
    reference would plan it."""

    def __init__(self, period: int, vars: list[PoolVar] | None = None, adj: list[set[int]] | None = None,
                 peak_load_bytes: int = 0):
        self.period = period
        self.peak_load_bytes = peak_load_bytes
        self._vars = vars
        self._adj = adj
        self._dev = None
        self._sig = {}        # frozen vars/adj the device CSR was built from
        self._vars_fn = None  # builds PoolVar list on demand
        self._nv = len(vars) if vars is not None else 0

    @property
    def vars(self) -> list[PoolVar]:
        if self._vars is None and self._vars_fn is not None:
            self._vars = self._vars_fn()
            if self._dev is not None:
                self._sig["vars"] = _freeze_vars(self._vars)
        return self._vars

    @vars.setter
    def vars(self, value):
        self.adj  # noqa: B018  (materialize the other half before the device copy goes)
        self._vars = value
        self._dev = None

    @property
    def adj(self) -> list[set[int]]:
        if self._adj is None and self._dev is not None:
            row, col = N.graph_csr(self._dev)
            c = col.tolist()
            r = row.tolist()
            self._adj = [set(c[r[i]:r[i + 1]]) for i in range(len(r) - 1)]
            self._sig["adj"] = _freeze_adj(self._adj)
        return self._adj

    @adj.setter
    def adj(self, value):
        self.vars  # noqa: B018
        self._adj = value
        self._dev = None

    def _device_stale(self) -> bool:
        return ((self._adj is not None and "adj" in self._sig and _freeze_adj(self._adj) != self._sig["adj"])
                or (self._vars is not None and "vars" in self._sig
                    and _freeze_vars(self._vars) != self._sig["vars"]))

    @property
    def nvars(self) -> int:
        return len(self._vars) if self._vars is not None else self._nv

    def __repr__(self):
        return f"ConflictGraph(period={self.period}, nvars={self.nvars}, peak={self.peak_load_bytes})"


class PoolPlan:
    """Offsets per variable plus the pool footprint (smartpool.py:36-48)."""

    def __init__(self, policy: str, offsets: dict[str, int] | None = None, sizes: dict[str, int] | None = None,
                 footprint_bytes: int = 0, peak_load_bytes: int = 0):
        self.policy = policy
        self.footprint_bytes = footprint_bytes
        self.peak_load_bytes = peak_load_bytes
        self._offsets = offsets
        self._sizes = sizes
        self._cols = None  # (names, offsets array, sizes array)
        self._fp = None    # the FlatProfile those names came from

    def _build(self):
        names, off, size = self._cols
        if self._offsets is None:
            self._offsets = dict(zip(names, off.tolist()))
        if self._sizes is None:
            self._sizes = dict(zip(names, size.tolist()))

    @property
    def offsets(self) -> dict[str, int]:
        if self._offsets is None:
            self._build()
        return self._offsets

    @offsets.setter
    def offsets(self, value):
        self._offsets = value

    @property
    def sizes(self) -> dict[str, int]:
        if self._sizes is None:
            self._build()
        return self._sizes

    @sizes.setter
    def sizes(self, value):
        self._sizes = value

    @property
    def offset_array(self) -> np.ndarray:
        """Offsets in graph vertex order (no dict materialization)."""
        if self._cols is not None:
            return self._cols[1]
        return np.array(list(self.offsets.values()), np.int64)

    @property
    def competitive_ratio(self) -> float:
        if self.peak_load_bytes <= 0:
            return 1.0
        return self.footprint_bytes / self.peak_load_bytes

    def __eq__(self, other):
        if not isinstance(other, PoolPlan):
            return NotImplemented
        return (self.policy, self.offsets, self.sizes, self.footprint_bytes, self.peak_load_bytes) == \
            (other.policy, other.offsets, other.sizes, other.footprint_bytes, other.peak_load_bytes)

    def __repr__(self):
        return (f"PoolPlan(policy={self.policy!r}, footprint_bytes={self.footprint_bytes}, "
                f"peak_load_bytes={self.peak_load_bytes})")


def _tie_ranks(allocs, names) -> np.ndarray:
    """Rank of (alloc_index, var) per vertex: the placement tie-break after
    -size (smartpool.py:94-98)."""
    order = sorted(range(len(names)), key=lambda i: (allocs[i], names[i]))
    tie = np.zeros(len(names), np.int64)
    tie[order] = np.arange(len(names), dtype=np.int64)
    return tie


def conflict_graph_from_arcs(period: int, arcs, peak_load_bytes: int) -> ConflictGraph:
    """Conflict graph of (var, size, alloc_index, segments, persistent) arcs
    (smartpool.py:51-79); half-open arcs that only touch do not conflict."""
    pool_vars = [PoolVar(*a) for a in arcs]
    n = len(pool_vars)
    seg_off = np.zeros(n + 1, np.int64)
    seg_off[1:] = np.cumsum([len(pv.segments) for pv in pool_vars]) if n else []
    lo = [s[0] for pv in pool_vars for s in pv.segments] or [0]
    hi = [s[1] for pv in pool_vars for s in pv.segments] or [0]
    try:
        lo, hi = np.array(lo, np.int32), np.array(hi, np.int32)
    except OverflowError:
        # the sweep only compares bounds (smartpool.py:57-77): rank them
        pts = sorted(set(lo) | set(hi))
        rank = {x: r for r, x in enumerate(pts)}
        lo = np.array([rank[x] for x in lo], np.int32)
        hi = np.array([rank[x] for x in hi], np.int32)
    tie = _tie_ranks([pv.alloc_index for pv in pool_vars], [pv.var for pv in pool_vars])
    g = ConflictGraph(period=period, vars=pool_vars, adj=None, peak_load_bytes=peak_load_bytes)
    g._dev = N.conflict_from_arcs([pv.size for pv in pool_vars] or [0], tie if n else np.zeros(1, np.int64),
                                  seg_off, lo, hi)
    g._nv = n
    g._sig = {"vars": _freeze_vars(pool_vars)}
    g._names = [pv.var for pv in pool_vars]
    g._sizes = np.array([pv.size for pv in pool_vars], np.int64)
    return g


def build_conflict_graph(profile: IterationProfile) -> ConflictGraph:
    """Conflict graph of a profile's lifetimes (smartpool.py:82-88).

    Like the reference's, the graph is a snapshot: its ``vars`` come from the
    device profile the CSR was built from, not from later edits of
    ``profile``."""
    dp = device_profile(profile)
    g = ConflictGraph(period=profile.period, vars=None, adj=None, peak_load_bytes=profile.peak_bytes)
    g._dev = N.conflict_from_profile(dp)
    g._nv = int(dp.dims().nvars)
    arrays, window = profile._arrays, profile.window
    # a Python-built profile was flattened to upload it; an extracted one
    # downloads its columns from this handle when first needed
    snap = {} if profile._flat is None else {"fp": profile._flat}

    def fp():
        if "fp" not in snap:
            if profile.__dict__.get("_dev") is dp and (profile._flat is not None or profile._arrays is not None):
                snap["fp"] = profile._flat_profile()  # shared with the profile (and its lookup table)
            else:
                snap["fp"] = N.download_profile(dp, arrays.names, arrays.name_blob, arrays.name_off, window)
        return snap["fp"]

    def make_vars():
        f = fp()
        seg, nseg, persistent = f.seg.tolist(), f.nseg.tolist(), (f.flags & F_PERSISTENT).tolist()
        return [PoolVar(name, size, alloc, tuple((seg[4 * i + 2 * k], seg[4 * i + 2 * k + 1])
                                                 for k in range(nseg[i])), bool(persistent[i]))
                for i, (name, size, alloc) in enumerate(zip(f.var_names(), f.size.tolist(), f.alloc.tolist()))]
    g._vars_fn = make_vars
    g._names_fn = lambda: fp().var_names()
    g._fp_fn = fp
    g._sizes_fn = lambda: fp().size
    return g


def _host_csr(vars_, adj):
    """CSR of a Python adjacency as the reference indexes it: rows beyond
    ``len(vars)`` are never read, negative ids index from the end, an id
    outside the list raises IndexError (smartpool.py:131-135).  The library
    mirrors the relation by placement order (mp_graph_from_csr)."""
    n = len(vars_)
    if len(adj) < n:
        raise IndexError("list index out of range")
    rows = [a if isinstance(a, (set, frozenset, list, tuple)) else list(a) for a in adj[:n]]
    row = np.zeros(n + 1, np.int64)
    row[1:] = np.cumsum([len(a) for a in rows]) if n else []
    col = np.fromiter((j for a in rows for j in a), np.int64, count=int(row[-1]))
    if col.size and (col.min() < -n or col.max() >= n):
        raise IndexError("list index out of range")
    col = np.where(col < 0, col + n, col).astype(np.int32)
    return row, (col if col.size else np.zeros(1, np.int32))


def _graph_device(graph: ConflictGraph):
    """Device CSR of a graph: the one built on the device, or an upload of
    the Python containers — redone after any in-place edit."""
    if graph._dev is not None and graph._device_stale():
        graph.vars, graph.adj  # noqa: B018  (both halves on the host)
        graph._dev = None
    if graph._dev is None:
        vars_ = graph.vars
        adj = graph.adj
        n = len(vars_)
        row, col = _host_csr(vars_, adj)
        tie = _tie_ranks([pv.alloc_index for pv in vars_], [pv.var for pv in vars_])
        graph._dev = N.graph_from_csr(row, col, [pv.size for pv in vars_] or [0], tie if n else np.zeros(1, np.int64))
        graph._nv = n
        graph._sig = {"vars": _freeze_vars(vars_), "adj": _freeze_adj(adj)}
    return graph._dev


def _graph_names_sizes(graph: ConflictGraph):
    if getattr(graph, "_names_fn", None) is not None and graph._vars is None:
        return graph._names_fn(), np.asarray(graph._sizes_fn())
    return [pv.var for pv in graph.vars], np.array([pv.size for pv in graph.vars], np.int64)


def plan_pool(graph: ConflictGraph, policy: str = "best_fit") -> PoolPlan:
    """Greedy placement in (-size, alloc, name) order, first/best fit among
    placed neighbours (smartpool.py:122-144), on the device."""
    if policy not in POLICY_CODE:
        raise ValueError(f"unknown policy {policy!r}")
    dg = _graph_device(graph)
    nv = graph.nvars
    offs, footprint, _levels = N.plan_pool(dg, POLICY_CODE[policy], nv)
    plan = PoolPlan(policy=policy, footprint_bytes=footprint if nv else 0,
                    peak_load_bytes=graph.peak_load_bytes)
    names, sizes = _graph_names_sizes(graph)
    plan._cols = (names, offs, sizes)
    plan._fp = graph._fp_fn() if getattr(graph, "_fp_fn", None) is not None and graph._vars is None else None
    plan._levels = _levels
    return plan


def check_plan(plan: PoolPlan, graph: ConflictGraph) -> None:
    """Raise if conflicting variables overlap or the footprint misses one
    (smartpool.py:147-164); a host-side safety checker."""
    offsets = plan.offsets
    for i, pv in enumerate(graph.vars):
        oi = offsets[pv.var]
        if oi < 0:
            raise MemplanError(f"{pv.var} at negative offset")
        if oi + pv.size > plan.footprint_bytes:
            raise MemplanError(f"{pv.var} exceeds footprint")
        for j in graph.adj[i]:
            if j <= i:
                continue
            qv = graph.vars[j]
            oj = offsets[qv.var]
            if oi < oj + qv.size and oj < oi + pv.size:
                raise MemplanError(f"conflicting vars {pv.var} and {qv.var} overlap")


def brute_force_optimal_footprint(graph: ConflictGraph, max_vars: int = 10) -> int:
    """Exact minimum footprint by exhaustive search over subset-sum offsets
    (smartpool.py:167-221); a small-instance test oracle, host-side."""
    n = len(graph.vars)
    if n > max_vars:
        raise GraphTooLarge(f"{n} vars exceeds cap {max_vars}")
    if n == 0:
        return 0
    lower = graph.peak_load_bytes
    best = plan_pool(graph, "best_fit").footprint_bytes
    if best <= lower:
        return best
    vars_, adj = graph.vars, graph.adj
    order = sorted(range(n), key=lambda i: (-vars_[i].size, vars_[i].alloc_index, vars_[i].var))
    sizes = [vars_[i].size for i in order]
    pos = {v: k for k, v in enumerate(order)}
    earlier = [[pos[j] for j in adj[order[k]] if pos[j] < k] for k in range(n)]
    sums = {0}
    for s in sizes:
        sums |= {x + s for x in sums}
    cands = sorted(sums)
    if cands[-1] < (1 << 62) and min(sizes) >= 0:
        # the DFS in host C++ (csrc/brute.cpp), same order and cut-offs
        import ctypes as C
        nb_off = np.zeros(n + 1, np.int64)
        nb_off[1:] = np.cumsum([len(e) for e in earlier])
        nb = np.array([j for e in earlier for j in e] or [0], np.int32)
        sz, cd = np.array(sizes, np.int64), np.array(cands, np.int64)
        out = C.c_int64(best)
        N.lib().mp_brute_force_footprint(C.c_int32(n), N.ptr(sz), N.ptr(nb_off), N.ptr(nb), N.ptr(cd),
                                         C.c_int64(len(cands)), C.c_int64(lower), C.byref(out))
        return int(out.value)
    offs = [0] * n

    def search(k: int, top: int) -> bool:
        nonlocal best
        if k == n:
            best = top
            return best <= lower
        sk = sizes[k]
        for off in cands:
            if off + sk >= best:
                break
            if any(off < offs[j] + sizes[j] and offs[j] < off + sk for j in earlier[k]):
                continue
            offs[k] = off
            if search(k + 1, max(top, off + sk)):
                return True
        return False

    search(0, 0)
    return best


class LookupTable:
    """Window-relative malloc op index -> (var, pool offset) (smartpool.py:224-243).

    Built either from a dict of entries (as the reference) or, by the column
    path of make_lookup_table, from the selected variables' op indices, names
    and offsets (an op -> row index array); the reference's ``_entries`` dict
    is materialized from the columns only if something asks for it."""

    def __init__(self, entries: dict[int, tuple[str, int]] | None = None, _cols=None):
        self._dict = dict(entries) if entries is not None else None
        self._cols = _cols  # (ops int64 array, names list, offsets list, op -> row int64 array)

    @property
    def _entries(self) -> dict[int, tuple[str, int]]:
        if self._dict is None:
            ops, names, offs, _row = self._cols
            self._dict = dict(zip(ops.tolist(), zip(names, offs)))
            self._cols = None
        return self._dict

    def __len__(self) -> int:
        return len(self._dict) if self._dict is not None else len(self._cols[1])

    def _row(self, op_index):
        _ops, _names, _offs, row = self._cols
        try:
            i = int(op_index)
        except (TypeError, ValueError):
            return -1
        if i != op_index or not 0 <= i < row.shape[0]:
            return -1
        return int(row[i])

    def __contains__(self, op_index) -> bool:
        if self._dict is not None:
            return op_index in self._dict
        return self._row(op_index) >= 0

    def offset_for(self, op_index: int) -> int:
        if self._dict is not None:
            return self._dict[op_index][1]
        r = self._row(op_index)
        if r < 0:
            raise KeyError(op_index)
        return self._cols[2][r]

    def var_for(self, op_index: int) -> str:
        if self._dict is not None:
            return self._dict[op_index][0]
        r = self._row(op_index)
        if r < 0:
            raise KeyError(op_index)
        return self._cols[1][r]

    def items(self):
        if self._dict is not None:
            return sorted(self._dict.items())
        ops, names, offs, _row = self._cols
        order = np.argsort(ops, kind="stable").tolist()
        opl = ops.tolist()
        return [(opl[i], (names[i], offs[i])) for i in order]


def make_lookup_table(plan: PoolPlan, profile: IterationProfile) -> LookupTable:
    """Malloc op index -> offset for every window allocation (smartpool.py:246-254)."""
    fast = _lookup_from_columns(plan, profile)
    if fast is not None:
        return fast
    offsets = plan.offsets
    entries = {}
    for v in profile.variables:
        if v.alloc_index is None:
            continue
        if v.var not in offsets:
            raise MissingVariable(v.var)
        entries[v.alloc_index] = (v.var, offsets[v.var])
    return LookupTable(entries)


def _lookup_from_columns(plan: PoolPlan, profile: IterationProfile):
    """The lookup table straight from the columns both sides came from, when
    neither the profile's variables nor the plan's offsets were ever handed
    out as Python containers (so neither can have been edited) and the plan
    names the profile's variables in the profile's order: the same entries
    the per-variable loop builds, without a million VariableLifetime objects.
    Returns None otherwise (the loop runs)."""
    cols = getattr(plan, "_cols", None)
    if cols is None or plan._offsets is not None or "variables" in profile.__dict__:
        return None
    if "variables" not in profile.__dict__.get("_pending", ()) or profile._dev is None:
        return None
    names, offs, _sizes = cols
    fp = profile._flat_profile()
    if getattr(plan, "_fp", None) is not fp:
        # a plan of another snapshot: usable only if it names the same variables in order
        pnames = fp.var_names()
        if len(pnames) != len(names) or pnames != names:
            return None
    alloc = np.asarray(fp.alloc, np.int64)
    sel = np.nonzero(alloc >= 0)[0]
    ops = alloc[sel]
    row = np.full(int(ops.max()) + 1 if ops.size else 0, -1, np.int64)
    row[ops] = np.arange(ops.size, dtype=np.int64)
    if ops.size and np.count_nonzero(row >= 0) != ops.size:
        return None  # repeated op indices: the loop's last-wins dict decides
    offl = np.asarray(offs)[sel].tolist()
    if sel.size == len(names):
        seln = names
    else:
        seln = [names[i] for i in sel.tolist()]
    return LookupTable(_cols=(ops, seln, offl, row))
