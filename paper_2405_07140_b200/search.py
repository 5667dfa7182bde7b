"""DFTSP and brute-force batch search (reference ``dftsp.py``), on the GPU.

Entry points keep the reference signatures and return the reference's
``SearchOutcome`` shape with the caller's own ``Request`` objects:

* ``dftsp``              -> K3 (``eb_dftsp_batch``)
* ``exhaustive_optimal`` -> K4 (``eb_exhaustive_batch``, subsets mode) or K3 in
                            count-vector mode
* ``dfs``                -> one dfs call on the device (``eb_dfs_single``)
* ``partition``          -> device link keys (K1) + host grouping
* ``dftsp_many`` / ``solve_batch`` -> batched throughput API over InstanceBatch
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .feasibility import raise_for_status
from .soa import InstanceBatch, WireBatch, context_record, search_params

__all__ = ["ClassPartition", "SearchOutcome", "SearchTables", "partition", "recover_subset", "dfs", "dftsp",
           "exhaustive_optimal", "dftsp_many", "solve_batch", "BatchResult", "exhaustive_many"]


@dataclass(frozen=True)
class ClassPartition:
    """Pool grouped by output length, cheapest uplink first (dftsp.py:29-39)."""

    lengths: tuple
    classes: tuple
    keys: tuple

    @property
    def sizes(self) -> tuple:
        return tuple(len(c) for c in self.classes)


@dataclass
class SearchOutcome:
    """Search result plus instrumentation (dftsp.py:42-51)."""

    solution: list | None = None
    counts: tuple = ()
    z_found: int = 0
    nodes_visited: int = 0
    nodes_pruned: int = 0
    trajectory: list | None = None


def _ref(s):
    return ctypes.cast(ctypes.pointer(s), ctypes.c_void_p)


def partition(pool, radio, ladder=None) -> ClassPartition:
    """Group a pool by output length (dftsp.py:54-82); keys from the device link kernel."""
    from .radio import _radio_ctx, _raise_link, link_table
    pool = list(pool)
    if ladder is not None:
        allowed = set(ladder)
        for r in pool:
            if r.output_tokens not in allowed:
                raise ValueError(f"request {r.id} output length {r.output_tokens} is not on "
                                 f"the class ladder {sorted(allowed)}")
    if not pool:
        return ClassPartition((), (), ())
    st, out = link_table([r.link.channel_gain for r in pool], [r.link.uplink_power_w for r in pool],
                         [r.prompt_tokens for r in pool], [r.output_tokens for r in pool], _radio_ctx(radio))
    groups: dict = {}
    for j, r in enumerate(pool):
        if st[j] in (_lib.ERR_UPLINK_EFF_ZERO, _lib.ERR_NONPOSITIVE_LINK):
            _raise_link(int(st[j]))
        groups.setdefault(r.output_tokens, []).append((float(out[j, 4]), r.id, j))
    lengths = tuple(sorted(groups))
    classes, keys = [], []
    for n in lengths:
        members = sorted(groups[n], key=lambda t: (t[0], t[1]))
        classes.append(tuple(pool[j] for _, _, j in members))
        keys.append(tuple(k for k, _, _ in members))
    return ClassPartition(lengths, tuple(classes), tuple(keys))


def recover_subset(part: ClassPartition, counts) -> list:
    """Per-class cheapest prefixes named by a count vector (dftsp.py:85-93)."""
    cs = list(counts) + [0] * (len(part.classes) - len(counts))
    out = []
    for k, v in enumerate(cs):
        if not 0 <= v <= len(part.classes[k]):
            raise ValueError(f"count {v} out of range for class {part.lengths[k]}")
        out.extend(part.classes[k][:v])
    return out


class SearchTables:
    """Per-partition prefix tables (dftsp.py:96-132).

    Introspection helper with the reference's layout; the device search builds
    its own tables in shared memory and never reads this object.
    """

    __slots__ = ("sizes", "tail", "lengths", "weights", "up", "dn", "tau_min_prefix")

    def __init__(self, sizes, tail, lengths, weights, up, dn, tau_min_prefix):
        self.sizes, self.tail, self.lengths, self.weights = sizes, tail, lengths, weights
        self.up, self.dn, self.tau_min_prefix = up, dn, tau_min_prefix

    @classmethod
    def build(cls, part: ClassPartition, coeff) -> "SearchTables":
        sizes = list(part.sizes)
        tail = [0] * (len(sizes) + 1)
        for k in reversed(range(len(sizes))):
            tail[k] = tail[k + 1] + sizes[k]
        lengths = list(part.lengths)
        up, dn, taus = [], [], []
        for n, members in zip(lengths, part.classes):
            cu, cd, tm = [0.0], [0.0], [math.inf]
            for r in members:
                cu.append(cu[-1] + coeff.k_up[r.id] * r.prompt_tokens)
                cd.append(cd[-1] + coeff.k_down[r.id] * n)
                tm.append(min(tm[-1], coeff.tau_base(r)))
            up.append(cu)
            dn.append(cd)
            taus.append(tm)
        return cls(sizes, tail, lengths, [coeff.latency_weight(n) for n in lengths], up, dn, taus)


def dfs(z, part, coeff, tau_min=None, *, pruning=True, inclusive_bound=False, exact_tau=False,
        tables=None) -> SearchOutcome:
    """One depth-first search for a feasible batch of exactly z (dftsp.py:135-234), on the GPU."""
    if z < 1:
        raise ValueError("z must be >= 1")
    if tau_min is None and not exact_tau:
        raise ValueError("tau_min is required unless exact_tau is set")
    ctx = coeff.ctx
    ncls = len(part.classes)
    if ncls > _lib.EB_MAX_CLASSES:
        raise ValueError(f"partition has {ncls} classes; the device supports {_lib.EB_MAX_CLASSES}")
    members = [r for c in part.classes for r in c]
    sizes = np.array([len(c) for c in part.classes] or [0], dtype=np.int32)
    lengths = np.array(list(part.lengths) or [0], dtype=np.int32)
    n = max(len(members), 1)
    k_up = np.zeros(n); k_dn = np.zeros(n); prompt = np.zeros(n, dtype=np.int32)
    dl = np.zeros(n); wt = np.zeros(n)
    for j, r in enumerate(members):
        k_up[j] = coeff.k_up[r.id]
        k_dn[j] = coeff.k_down[r.id]
        prompt[j] = r.prompt_tokens
        dl[j] = r.deadline_s
        wt[j] = r.waiting_s
    slot_base = math.nan if ctx.slot_cap_s is None else ctx.slot_cap_s * ctx.node.flops_per_s / ctx.quant.beta
    co = np.array([coeff.k2, coeff.k3, coeff.k4, coeff.k5, slot_base,
                   ctx.radio.uplink_slot_s + ctx.radio.downlink_slot_s, float(ctx.node.flops_per_s),
                   float(ctx.quant.beta)], dtype=np.float64)
    prm = search_params(pruning, inclusive_bound, exact_tau)
    found = ctypes.c_int32(0)
    counts = np.zeros(_lib.EB_MAX_CLASSES, dtype=np.int32)
    vis = ctypes.c_int64(0)
    prn = ctypes.c_int64(0)
    h = _lib.handle()
    _lib.check(h.lib.eb_dfs_single(h.ptr, int(z), ncls, sizes.ctypes.data, lengths.ctypes.data, prompt.ctypes.data,
                                   k_up.ctypes.data, k_dn.ctypes.data, dl.ctypes.data, wt.ctypes.data,
                                   co.ctypes.data, int(coeff.padded_len), int(tau_min is not None),
                                   float(tau_min) if tau_min is not None else 0.0, _ref(prm), ctypes.byref(found),
                                   counts.ctypes.data, ctypes.byref(vis), ctypes.byref(prn)),
               "eb_dfs_single")
    if not found.value:
        return SearchOutcome(nodes_visited=vis.value, nodes_pruned=prn.value)
    cnt = tuple(int(c) for c in counts[:ncls])
    return SearchOutcome(solution=recover_subset(part, cnt), counts=cnt, z_found=z,
                         nodes_visited=vis.value, nodes_pruned=prn.value)


# ---------------------------------------------------------------------------
@dataclass
class BatchResult:
    """Host arrays of an eb_dftsp_batch call (one row per instance)."""

    status: np.ndarray
    error_index: np.ndarray
    z_found: np.ndarray
    nodes_visited: np.ndarray
    nodes_pruned: np.ndarray
    n_classes: np.ndarray
    counts: np.ndarray
    class_lengths: np.ndarray
    solution: np.ndarray
    metrics: np.ndarray
    traj_offsets: np.ndarray | None = None
    traj: np.ndarray | None = None
    traj_len: np.ndarray | None = None
    solution_mask: np.ndarray | None = None    # u64 per instance (K <= 64), bit j = local request j


def solve_batch(batch: InstanceBatch | WireBatch, *, pruning=True, inclusive_bound=False, exact_tau=False,
                collect_trajectory=False, ladder=None, device=None, handle=None, algorithm=0,
                exhaustive_counts=False) -> BatchResult:
    """K3 over a host InstanceBatch: every instance is one dftsp() call.

    ``algorithm``: 0 auto, 1 literal node walk (one dfs call per lane), 2
    leaf-parallel with combinatorial node counts -- identical results."""
    n, nr = batch.n_inst, batch.n_req
    sizes = batch.sizes() if isinstance(batch, WireBatch) else np.diff(batch.offsets)
    res = BatchResult(status=np.zeros(n, np.int32), error_index=np.full(n, -1, np.int32),
                      z_found=np.zeros(n, np.int32), nodes_visited=np.zeros(n, np.int64),
                      nodes_pruned=np.zeros(n, np.int64), n_classes=np.zeros(n, np.int32),
                      counts=np.zeros((n, _lib.EB_MAX_CLASSES), np.int32),
                      class_lengths=np.zeros((n, _lib.EB_MAX_CLASSES), np.int32),
                      solution=np.full(max(nr, 1), -1, np.int32), metrics=np.zeros((n, _lib.EB_N_METRICS)),
                      solution_mask=np.zeros(max(n, 1), np.uint64))
    out = _lib.eb_dftsp_result()
    for name in ("status", "error_index", "z_found", "nodes_visited", "nodes_pruned", "n_classes", "counts",
                 "class_lengths", "solution", "metrics", "solution_mask"):
        setattr(out, name, getattr(res, name).ctypes.data)
    if collect_trajectory:
        rows = sizes * (sizes + 1) // 2
        res.traj_offsets = np.zeros(n + 1, np.int64)
        np.cumsum(rows, out=res.traj_offsets[1:])
        res.traj = np.zeros((max(int(res.traj_offsets[-1]), 1), 4), np.int64)
        res.traj_len = np.zeros(n, np.int32)
        out.traj_offsets = res.traj_offsets.ctypes.data
        out.traj = res.traj.ctypes.data
        out.traj_len = res.traj_len.ctypes.data
    prm = search_params(pruning, inclusive_bound, exact_tau, collect_trajectory, ladder, algorithm,
                        exhaustive_counts)
    h = handle or _lib.handle(device)
    b = batch.struct()
    if isinstance(batch, WireBatch):        # compact wire format (eb_dftsp_batch_packed)
        _lib.check(h.lib.eb_dftsp_batch_packed(h.ptr, batch.contexts.ctypes.data, len(batch.contexts), _ref(prm),
                                               _ref(b), _ref(out), _lib.EB_MEM_HOST), "eb_dftsp_batch_packed")
        return res
    _lib.check(h.lib.eb_dftsp_batch(h.ptr, batch.contexts.ctypes.data, len(batch.contexts), _ref(prm), _ref(b),
                                    _ref(out), _lib.EB_MEM_HOST), "eb_dftsp_batch")
    return res


def _outcome(res: BatchResult, i: int, pool, ctx, ladder, collect) -> SearchOutcome:
    st = int(res.status[i])
    if st != _lib.OK:
        raise_for_status(st, pool, int(res.error_index[i]), ctx, ladder)
    agg = SearchOutcome(trajectory=[] if collect else None)
    agg.nodes_visited = int(res.nodes_visited[i])
    agg.nodes_pruned = int(res.nodes_pruned[i])
    if collect and res.traj_len is not None:
        t0 = int(res.traj_offsets[i])
        agg.trajectory = [tuple(int(v) for v in row) for row in res.traj[t0:t0 + int(res.traj_len[i])]]
    z = int(res.z_found[i])
    if z:
        nc = int(res.n_classes[i])
        agg.counts = tuple(int(c) for c in res.counts[i, :nc])
        agg.z_found = z
    return agg


def dftsp_many(pools, ctx, *, ladder=None, pruning=True, inclusive_bound=False, exact_tau=False,
               collect_trajectory=False, contexts=None, ctx_index=None) -> list:
    """Many independent dftsp() calls in one launch; returns SearchOutcome per pool."""
    pools = [list(p) for p in pools]
    if contexts is None:
        contexts = [ctx]
    recs = np.concatenate([context_record(c) for c in contexts])
    batch = InstanceBatch.from_pools(pools, recs, ctx_index)
    res = solve_batch(batch, pruning=pruning, inclusive_bound=inclusive_bound, exact_tau=exact_tau,
                      collect_trajectory=collect_trajectory, ladder=ladder)
    outs = []
    for i, pool in enumerate(pools):
        c = contexts[0 if ctx_index is None else int(ctx_index[i])]
        agg = _outcome(res, i, pool, c, ladder, collect_trajectory)
        if agg.z_found:
            lo = int(batch.offsets[i])
            agg.solution = [pool[int(j)] for j in res.solution[lo:lo + agg.z_found]]
        outs.append(agg)
    return outs


def dftsp(candidates, ctx, *, ladder=None, pruning=True, inclusive_bound=False, exact_tau=False,
          collect_trajectory=False) -> SearchOutcome:
    """Maximum-cardinality feasible batch (dftsp.py:237-285) on the GPU."""
    pool = list(candidates)
    if not pool:
        return SearchOutcome(trajectory=[] if collect_trajectory else None)
    return dftsp_many([pool], ctx, ladder=ladder, pruning=pruning, inclusive_bound=inclusive_bound,
                      exact_tau=exact_tau, collect_trajectory=collect_trajectory)[0]


# ---------------------------------------------------------------------------
def exhaustive_many(pools, ctx, *, cap=20, contexts=None, ctx_index=None):
    """K4 over many pools: arrays (status, z, lexrank, nodes, mask)."""
    if contexts is None:
        contexts = [ctx]
    recs = np.concatenate([context_record(c) for c in contexts])
    batch = InstanceBatch.from_pools([list(p) for p in pools], recs, ctx_index)
    n = batch.n_inst
    st = np.zeros(n, np.int32); z = np.zeros(n, np.int32); rk = np.zeros(n, np.int64)
    nodes = np.zeros(n, np.int64); mask = np.zeros(n, np.uint64)
    h = _lib.handle()
    b = batch.struct()
    _lib.check(h.lib.eb_exhaustive_batch(h.ptr, recs.ctypes.data, len(recs), _ref(b), int(cap), st.ctypes.data,
                                         z.ctypes.data, rk.ctypes.data, nodes.ctypes.data, mask.ctypes.data,
                                         _lib.EB_MEM_HOST), "eb_exhaustive_batch")
    return st, z, rk, nodes, mask


def exhaustive_optimal(candidates, ctx, *, cap: int = 20, mode: str = "subsets", ladder=None) -> SearchOutcome:
    """Brute-force reference search (dftsp.py:288-332) on the GPU."""
    pool = list(candidates)
    agg = SearchOutcome()
    if not pool:
        return agg
    if len(pool) > cap:
        raise ValueError(f"pool size {len(pool)} exceeds the exhaustive cap {cap}")
    if mode == "subsets":
        if len(pool) > _lib.EB_MAX_K:
            raise ValueError(f"pool of {len(pool)} exceeds the device limit of {_lib.EB_MAX_K}")
        st, z, rk, nodes, mask = exhaustive_many([pool], ctx, cap=cap)
        raise_for_status(int(st[0]), pool, -1, ctx)
        agg.nodes_visited = int(nodes[0])
        if z[0]:
            m = int(mask[0])
            chosen = [r for j, r in enumerate(pool) if (m >> j) & 1]
            agg.solution = sorted(chosen, key=lambda r: r.id)
            agg.z_found = int(z[0])
        return agg
    if mode != "counts":
        raise ValueError(f"unknown exhaustive mode {mode!r}")
    return _exhaustive_counts(pool, ctx, ladder)


def exhaustive_counts_many(pools, ctx, *, ladder=None, contexts=None, ctx_index=None) -> BatchResult:
    """exhaustive_optimal(mode="counts") over many pools in one launch (K3 counts mode)."""
    if contexts is None:
        contexts = [ctx]
    recs = np.concatenate([context_record(c) for c in contexts])
    batch = InstanceBatch.from_pools([list(p) for p in pools], recs, ctx_index)
    return batch, solve_batch(batch, ladder=ladder, exhaustive_counts=True)


def _exhaustive_counts(pool, ctx, ladder) -> SearchOutcome:
    """Count-vector mode (dftsp.py:316-332): K3 in counts mode on the device."""
    batch, res = exhaustive_counts_many([pool], ctx, ladder=ladder)
    st = int(res.status[0])
    if st == _lib.ERR_REVERIFY:
        raise RuntimeError("count-vector solution failed re-verification")
    raise_for_status(st, pool, int(res.error_index[0]), ctx, ladder)
    agg = SearchOutcome(nodes_visited=int(res.nodes_visited[0]))
    z = int(res.z_found[0])
    if z:
        agg.solution = [pool[int(j)] for j in res.solution[:z]]
        agg.z_found = z
    return agg
