"""Analytical memory/latency model (reference ``costs.py``).

The closed-form integer counts (bytes, FLOPs) are configuration math on
Python ints, exactly as the reference defines them; the device kernels carry
the same formulas in int64 (``csrc/eb_exact.cuh``).  ``batch_cost`` -- the
per-batch memory/latency evaluation on the hot path -- runs on the GPU
(``eb_batch_cost_batch``).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _lib

__all__ = ["NodeCompute", "BatchPlan", "BatchCost", "weight_bytes", "kv_cache_bytes_per_token",
           "kv_bytes_initial", "kv_bytes_autoregressive", "flops_initial", "flops_autoregressive",
           "flops_autoregressive_stepwise", "batch_cost", "batch_cost_many"]


@dataclass(frozen=True)
class NodeCompute:
    """Aggregate compute C (FLOP/s) and memory M (bytes) of the edge node."""

    flops_per_s: float
    memory_bytes: float
    gpu_count: int = 1

    def __post_init__(self):
        if min(self.flops_per_s, self.memory_bytes, self.gpu_count) <= 0:
            raise ValueError("node resources must be strictly positive")

    @property
    def per_gpu_flops(self) -> float:
        return self.flops_per_s / self.gpu_count

    @property
    def per_gpu_memory(self) -> float:
        return self.memory_bytes / self.gpu_count


@dataclass(frozen=True)
class BatchPlan:
    """(prompt, output) entries sharing one padded prompt length."""

    entries: tuple
    padded_len: int

    def __post_init__(self):
        for s, n in self.entries:
            if s > self.padded_len:
                raise ValueError(f"prompt length {s} exceeds padded length {self.padded_len}")
            if n < 1:
                raise ValueError("every output length must be >= 1")

    def __len__(self) -> int:
        return len(self.entries)


class BatchCost(NamedTuple):
    memory_bytes: float
    latency_s: float


def weight_bytes(spec) -> int:
    """L (4 b d d_h n_h + 2 b d f)  (costs.py:62-67)."""
    b, d = spec.bytes_per_param, spec.hidden_dim
    return spec.layers * (4 * b * d * spec.head_dim * spec.head_count + 2 * b * d * spec.ffn_dim)


def kv_cache_bytes_per_token(spec) -> int:
    """2 b L d  (costs.py:70-72)."""
    return 2 * spec.bytes_per_param * spec.layers * spec.hidden_dim


def kv_bytes_initial(spec, padded_len: int, batch: int) -> int:
    if batch < 0:
        raise ValueError("batch must be nonnegative")
    return kv_cache_bytes_per_token(spec) * padded_len * batch


def kv_bytes_autoregressive(spec, output_tokens) -> int:
    return kv_cache_bytes_per_token(spec) * sum(output_tokens)


def flops_initial(spec, padded_len: int) -> int:
    """Prompt pass: L (6 s d^2 + 4 s^2 d + 2 s d^2 + 4 s d f)  (costs.py:87-97)."""
    if padded_len < 1:
        raise ValueError("padded_len must be >= 1")
    s, d, f = padded_len, spec.hidden_dim, spec.ffn_dim
    return spec.layers * (6 * s * d * d + (4 * s * s * d + 2 * s * d * d) + 4 * s * d * f)


def flops_autoregressive(spec, padded_len: int, output_tokens: int) -> int:
    """Generation passes, closed form: L (n-1)(8d^2 + 4 s d + 4 d f + 2 d n)  (costs.py:100-112)."""
    if output_tokens < 1:
        raise ValueError("output_tokens must be >= 1")
    d = spec.hidden_dim
    base = 8 * d * d + 4 * padded_len * d + 4 * d * spec.ffn_dim
    return spec.layers * (output_tokens - 1) * (base + 2 * d * output_tokens)


def flops_autoregressive_stepwise(spec, padded_len: int, output_tokens: int) -> int:
    """Per-step summation cross-check of the closed form (costs.py:115-128)."""
    if output_tokens < 1:
        raise ValueError("output_tokens must be >= 1")
    d = spec.hidden_dim
    base = 8 * d * d + 4 * padded_len * d + 4 * d * spec.ffn_dim
    return spec.layers * sum(base + 4 * d * step for step in range(1, output_tokens))


def _model_ctx(spec, quant, node) -> np.ndarray:
    rec = np.zeros(1, dtype=_lib.CTX_DTYPE)
    rec["layers"] = spec.layers
    rec["hidden_dim"] = spec.hidden_dim
    rec["head_count"] = spec.head_count
    rec["head_dim"] = spec.head_dim
    rec["ffn_dim"] = spec.ffn_dim
    rec["bytes_per_param"] = spec.bytes_per_param
    rec["alpha"] = float(quant.alpha)
    rec["beta"] = float(quant.beta)
    rec["flops_per_s"] = float(node.flops_per_s)
    rec["memory_bytes"] = float(node.memory_bytes)
    rec["gpu_count"] = int(node.gpu_count)
    return rec


def batch_cost_many(plans, contexts: np.ndarray, plan_ctx=None, weight_copies=None, device=None) -> np.ndarray:
    """Batched batch_cost on the GPU: returns [n_plans, 2] (memory_bytes, latency_s)."""
    n = len(plans)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum([len(p.entries) for p in plans], out=off[1:])
    prompt = np.fromiter((s for p in plans for s, _ in p.entries), dtype=np.int32, count=int(off[-1]))
    output = np.fromiter((o for p in plans for _, o in p.entries), dtype=np.int32, count=int(off[-1]))
    padded = np.array([p.padded_len for p in plans], dtype=np.int64)
    wc = None if weight_copies is None else np.ascontiguousarray(weight_copies, dtype=np.int64)
    pc = None if plan_ctx is None else np.ascontiguousarray(plan_ctx, dtype=np.int32)
    out = np.zeros((n, 2), dtype=np.float64)
    h = _lib.handle(device)
    _lib.check(h.lib.eb_batch_cost_batch(h.ptr, contexts.ctypes.data, len(contexts), n, off.ctypes.data,
                                         prompt.ctypes.data, output.ctypes.data, padded.ctypes.data,
                                         _lib.ptr(wc), _lib.ptr(pc), out.ctypes.data, _lib.EB_MEM_HOST),
               "eb_batch_cost_batch")
    return out


def batch_cost(spec, quant, plan, node, weight_copies: int = 1) -> BatchCost:
    """Memory footprint and compute latency of one batch (costs.py:131-148), on the GPU."""
    out = batch_cost_many([plan], _model_ctx(spec, quant, node), weight_copies=[weight_copies])
    return BatchCost(memory_bytes=float(out[0, 0]), latency_s=float(out[0, 1]))
