"""Benchmark batching schedulers StB and NoB (reference ``baselines.py``), on the GPU.

``static_batch_size`` -> ``eb_static_batch_size_batch``; ``stb_schedule`` ->
``eb_stb_batch``; ``nob_assign`` -> ``eb_nob_batch`` (device per-request cost
and FIFO device assignment; the pool's ``busy_until`` state round-trips).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .feasibility import raise_for_status
from .soa import InstanceBatch, context_record

__all__ = ["GpuPool", "SchedulerDecision", "static_batch_size", "stb_schedule", "nob_assign"]


@dataclass
class GpuPool:
    """Per-device view of the node for NoB (baselines.py:22-39)."""

    device_count: int
    flops_per_device: float
    memory_per_device: float
    busy_until: list = field(default_factory=list)

    def __post_init__(self):
        if self.device_count < 1:
            raise ValueError("device_count must be >= 1")
        if not self.busy_until:
            self.busy_until = [0.0] * self.device_count

    @classmethod
    def from_node(cls, node) -> "GpuPool":
        return cls(node.gpu_count, node.per_gpu_flops, node.per_gpu_memory)


@dataclass
class SchedulerDecision:
    """One epoch's choice (baselines.py:42-48)."""

    scheduled: list = field(default_factory=list)
    search_stats: object = None
    dropped: list = field(default_factory=list)


def _ref(s):
    return ctypes.cast(ctypes.pointer(s), ctypes.c_void_p)


def static_batch_size(spec, quant, node, slot_s: float, s_max: int, n_max: int) -> int:
    """Worst-case overflow-safe batch size (baselines.py:51-65), on the GPU."""
    rec = np.zeros(1, dtype=_lib.CTX_DTYPE)
    for name in ("layers", "hidden_dim", "head_count", "head_dim", "ffn_dim", "bytes_per_param"):
        rec[name] = getattr(spec, name)
    rec["alpha"], rec["beta"] = float(quant.alpha), float(quant.beta)
    rec["flops_per_s"], rec["memory_bytes"] = float(node.flops_per_s), float(node.memory_bytes)
    rec["gpu_count"] = int(node.gpu_count)
    sl = np.array([slot_s], dtype=np.float64)
    sm = np.array([s_max], dtype=np.int64)
    nm = np.array([n_max], dtype=np.int64)
    out = np.zeros(1, dtype=np.int64)
    h = _lib.handle()
    _lib.check(h.lib.eb_static_batch_size_batch(h.ptr, rec.ctypes.data, 1, sl.ctypes.data, sm.ctypes.data,
                                                nm.ctypes.data, out.ctypes.data, _lib.EB_MEM_HOST),
               "eb_static_batch_size_batch")
    return int(out[0])


def stb_schedule(queue, b: int, ctx, delta: float, accuracy_check: bool = True) -> SchedulerDecision:
    """FIFO admission of up to b requests (baselines.py:68-87), on the GPU."""
    q = list(queue)
    if not q:
        return SchedulerDecision()
    rec = context_record(ctx, delta)
    batch = InstanceBatch.from_pools([q], rec)
    bb = np.array([b], dtype=np.int64)
    st = np.zeros(1, np.int32)
    sel = np.zeros(len(q), np.uint8)
    h = _lib.handle()
    bs = batch.struct()
    _lib.check(h.lib.eb_stb_batch(h.ptr, rec.ctypes.data, 1, _ref(bs), bb.ctypes.data, int(bool(accuracy_check)),
                                  st.ctypes.data, sel.ctypes.data, _lib.EB_MEM_HOST), "eb_stb_batch")
    raise_for_status(int(st[0]))
    return SchedulerDecision(scheduled=[r for r, s in zip(q, sel) if s])


def nob_assign(queue, pool: GpuPool, now: float, ctx, delta: float, accuracy_check: bool = True):
    """One request per idle device (baselines.py:90-121), on the GPU; mutates pool.busy_until."""
    q = list(queue)
    decision = SchedulerDecision()
    if not q:
        return decision, []
    rec = context_record(ctx, delta)
    # per-device speed/memory come from the pool (GpuPool.from_node divides the node)
    # the kernel divides by gpu_count; 1 keeps the pool's per-device values exact
    rec["gpu_count"] = 1
    rec["flops_per_s"] = float(pool.flops_per_device)
    rec["memory_bytes"] = float(pool.memory_per_device)
    batch = InstanceBatch.from_pools([q], rec)
    G = pool.device_count
    busy = np.array(pool.busy_until, dtype=np.float64).reshape(1, G)
    now_a = np.array([now], dtype=np.float64)
    st = np.zeros(1, np.int32)
    act = np.zeros(len(q), np.int8)
    comp = np.zeros(len(q), np.float64)
    order = np.zeros(len(q), np.int32)
    nd = np.array([G], dtype=np.int32)
    h = _lib.handle()
    bs = batch.struct()
    _lib.check(h.lib.eb_nob_batch(h.ptr, rec.ctypes.data, 1, _ref(bs), now_a.ctypes.data, int(bool(accuracy_check)),
                                  nd.ctypes.data, G, busy.ctypes.data, st.ctypes.data, act.ctypes.data, comp.ctypes.data,
                                  order.ctypes.data, _lib.EB_MEM_HOST), "eb_nob_batch")
    raise_for_status(int(st[0]))
    pool.busy_until[:] = [float(v) for v in busy[0]]
    completions = []
    for r, a, c in zip(q, act, comp):
        if a == 1:
            decision.scheduled.append(r)
            completions.append(float(c))
        elif a == 2:
            decision.dropped.append((r, "exceeds per-device memory"))
    return decision, completions
