"""Admission, knapsack coefficients and batch feasibility (reference ``feasibility.py``).

``derive_coefficients`` (K1), ``filter_admissible`` (K1), ``check_knapsack``
and ``check_direct`` (K2) evaluate on the GPU through the C ABI; the
dataclasses and the scalar ``leq`` helper are host-side.  Batched forms
(``check_direct_many`` ...) take many subsets per launch.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .soa import InstanceBatch, context_record, request_columns, requests_struct

__all__ = ["REL_EPS", "leq", "Request", "EdgeContext", "WeightsDoNotFitError", "KnapsackCoefficients",
           "filter_admissible", "derive_coefficients", "check_knapsack", "check_direct", "check_direct_many",
           "admission_mask"]

REL_EPS = 1e-9


def leq(a: float, b: float, eps: float = REL_EPS) -> bool:
    """a <= b up to eps relative to the larger magnitude (feasibility.py:23-30)."""
    return a - b <= eps * max(1.0, abs(a), abs(b))


@dataclass
class Request:
    """An inference request with its link and waiting time (feasibility.py:33-56)."""

    id: int
    prompt_tokens: int
    output_tokens: int
    deadline_s: float
    tolerance: float
    link: object
    arrival_s: float = 0.0
    waiting_s: float = 0.0

    def __post_init__(self):
        checks = ((self.prompt_tokens < 1, "prompt_tokens must be >= 1"),
                  (self.output_tokens < 1, "output_tokens must be >= 1"),
                  (self.deadline_s <= 0, "deadline_s must be strictly positive"),
                  (self.tolerance < 0, "tolerance must be nonnegative"),
                  (self.waiting_s < 0, "waiting_s must be nonnegative"))
        for bad, msg in checks:
            if bad:
                raise ValueError(msg)


@dataclass(frozen=True)
class EdgeContext:
    """Model, quantization, radio and node of the serving edge (feasibility.py:59-71)."""

    llm: object
    quant: object
    radio: object
    node: object
    slot_cap_s: float | None = None


class WeightsDoNotFitError(ValueError):
    """The quantized weights alone exceed node memory."""


@dataclass
class KnapsackCoefficients:
    """Reduced-form coefficients of one pool (feasibility.py:78-125).

    Values are produced on the GPU by ``derive_coefficients``; the small
    scalar methods below restate the reference's affine budgets for callers.
    """

    ctx: object
    padded_len: int
    k_up: dict = field(default_factory=dict)
    k_down: dict = field(default_factory=dict)
    k2: float = 0.0
    k3: float = 0.0
    k4: float = 0.0
    k5: float = 0.0
    _tau: dict = field(default_factory=dict, repr=False)

    def mem_budget(self, z: int) -> float:
        return self.k2 - self.padded_len * z

    def latency_weight(self, n: int) -> float:
        return self.k4 * n + self.k5 * n * n

    def tau_base(self, req) -> float:
        slots = self.ctx.radio.uplink_slot_s + self.ctx.radio.downlink_slot_s
        return (req.deadline_s - req.waiting_s - slots) * self.ctx.node.flops_per_s / self.ctx.quant.beta

    def tau_budget(self, req, z: int) -> float:
        return self.tau_base(req) - self.k3 * z

    def slot_budget(self, z: int) -> float:
        if self.ctx.slot_cap_s is None:
            return math.inf
        return self.ctx.slot_cap_s * self.ctx.node.flops_per_s / self.ctx.quant.beta - self.k3 * z


def _ref(s):
    return ctypes.cast(ctypes.pointer(s), ctypes.c_void_p)


def raise_for_status(status: int, reqs=None, err_index: int = -1, ctx=None, ladder=None) -> None:
    """Map a per-instance eb_status to the reference's exception."""
    if status == _lib.OK:
        return
    r = reqs[err_index] if (reqs is not None and 0 <= err_index < len(reqs)) else None
    if status == _lib.ERR_WEIGHTS_DO_NOT_FIT:
        from .costs import weight_bytes
        m1 = weight_bytes(ctx.llm)
        raise WeightsDoNotFitError(f"weights need {m1} bytes but only "
                                   f"{ctx.node.memory_bytes / ctx.quant.alpha:.4g} scaled bytes are available")
    if status == _lib.ERR_NONPOSITIVE_LINK:
        raise ValueError("power, gain and noise must be strictly positive")
    if status == _lib.ERR_UPLINK_EFF_ZERO:
        raise ValueError("uplink spectral efficiency is zero")
    if status == _lib.ERR_DOWNLINK_EFF_ZERO:
        raise ValueError("downlink spectral efficiency is zero")
    if status == _lib.ERR_OFF_LADDER:
        raise ValueError(f"request {r.id} output length {r.output_tokens} is not on the class ladder "
                         f"{sorted(set(ladder))}")
    if status == _lib.ERR_REVERIFY:
        raise RuntimeError("reduced-form solution failed direct re-verification; "
                           "coefficient derivation is inconsistent")
    if status == _lib.ERR_PADDED_TOO_SMALL:
        raise ValueError("padded_len must cover every candidate prompt")
    if status == _lib.ERR_NAN_INPUT:
        raise ValueError(f"request {r.id if r else '?'} has a NaN deadline, waiting time, gain or power: the "
                         "reference orders such pools by CPython's sort on unordered keys, which the device "
                         "does not reproduce")
    if status == _lib.ERR_DUPLICATE_ID:
        raise ValueError(f"request ids must be unique within a pool (duplicate id {r.id if r else '?'})")
    if status == _lib.ERR_CAP_EXCEEDED:
        raise ValueError("pool size exceeds the exhaustive cap")
    if status in (_lib.ERR_K_TOO_LARGE, _lib.ERR_TOO_MANY_CLASSES, _lib.ERR_OVERFLOW):
        raise ValueError(f"instance outside the device limits: {_lib.status_string(status)}")
    raise _lib.EdgebatchNativeError(_lib.status_string(status))


def filter_admissible(requests, delta: float) -> list:
    """Requests whose tolerance admits degradation delta (feasibility.py:128-130), on the GPU."""
    reqs = list(requests)
    if not reqs:
        return []
    if delta < 0:
        raise ValueError("delta and tolerance must be nonnegative")
    keep = admission_mask([reqs], None, delta, accuracy_check=True, prefilter=False)[0]
    return [r for r, k in zip(reqs, keep) if k]


def admission_mask(pools, ctx, delta: float, accuracy_check=True, prefilter=True, device=None):
    """K1: per-request keep flags of sim._dftsp_candidates (sim.py:264-274) for many pools."""
    if ctx is None:
        rec = np.zeros(1, dtype=_lib.CTX_DTYPE)
    else:
        rec = context_record(ctx)
    rec["delta_ppl"] = float(delta)
    batch = InstanceBatch.from_pools(pools, rec)
    n = batch.n_req
    status = np.zeros(n, dtype=np.int32)
    keep = np.zeros(n, dtype=np.uint8)
    h = _lib.handle(device)
    b = batch.struct()
    _lib.check(h.lib.eb_admission_batch(h.ptr, rec.ctypes.data, 1, _ref(b), int(accuracy_check), int(prefilter),
                                        status.ctypes.data, keep.ctypes.data, _lib.EB_MEM_HOST),
               "eb_admission_batch")
    out = []
    for i, p in enumerate(pools):
        lo, hi = int(batch.offsets[i]), int(batch.offsets[i + 1])
        for j in range(lo, hi):
            if status[j] == _lib.ERR_INVALID_ARG:
                raise ValueError("delta and tolerance must be nonnegative")
            if status[j]:
                raise_for_status(int(status[j]))
        out.append(keep[lo:hi].astype(bool))
    return out


def derive_coefficients(ctx, padded_len: int, requests) -> KnapsackCoefficients:
    """Reduced-form coefficients for a pool (feasibility.py:133-167), computed by the K1 kernel."""
    reqs = list(requests)
    rec = context_record(ctx)
    if reqs:
        batch = InstanceBatch.from_pools([reqs], rec)
    else:
        batch = InstanceBatch.from_pools([[]], rec)
    bad_pad = padded_len < 1
    if bad_pad and reqs:
        raise ValueError("padded_len must cover every candidate prompt")   # every prompt is >= 1
    # padded_len < 1 on an empty pool: the reference still checks the weights
    # first, then flops_initial raises; probe the weights check with padded 1.
    pad = np.array([1 if bad_pad else int(padded_len)], dtype=np.int64)
    status = np.zeros(1, dtype=np.int32)
    err = np.full(1, -1, dtype=np.int32)
    sc = np.zeros(6, dtype=np.float64)
    rq = np.zeros((max(len(reqs), 1), 4), dtype=np.float64)
    h = _lib.handle()
    b = batch.struct()
    _lib.check(h.lib.eb_coefficients_batch(h.ptr, rec.ctypes.data, 1, _ref(b), pad.ctypes.data, status.ctypes.data,
                                           err.ctypes.data, sc.ctypes.data, rq.ctypes.data, _lib.EB_MEM_HOST),
               "eb_coefficients_batch")
    raise_for_status(int(status[0]), reqs, int(err[0]), ctx)
    if bad_pad:
        raise ValueError("padded_len must be >= 1")
    co = KnapsackCoefficients(ctx=ctx, padded_len=int(padded_len), k2=float(sc[0]), k3=float(sc[1]),
                              k4=float(sc[2]), k5=float(sc[3]))
    for j, r in enumerate(reqs):
        co.k_up[r.id] = float(rq[j, 0])
        co.k_down[r.id] = float(rq[j, 1])
    return co


def check_knapsack(subset, coeff: KnapsackCoefficients, z: int, tau_min: float) -> bool:
    """Reduced P2 check (feasibility.py:170-189) on the GPU."""
    sub = list(subset)
    m = len(sub)
    off = np.array([0, m], dtype=np.int64)
    prompt = np.array([r.prompt_tokens for r in sub], dtype=np.int32).reshape(-1)
    output = np.array([r.output_tokens for r in sub], dtype=np.int32).reshape(-1)
    ku = np.array([coeff.k_up[r.id] for r in sub], dtype=np.float64).reshape(-1)
    kd = np.array([coeff.k_down[r.id] for r in sub], dtype=np.float64).reshape(-1)
    ctx = coeff.ctx
    slot_base = math.nan if ctx.slot_cap_s is None else \
        ctx.slot_cap_s * ctx.node.flops_per_s / ctx.quant.beta
    co = np.array([coeff.k2, coeff.k3, coeff.k4, coeff.k5, slot_base, float(coeff.padded_len)], dtype=np.float64)
    zz = np.array([z], dtype=np.int32)
    tm = np.array([tau_min], dtype=np.float64)
    ok = np.zeros(1, dtype=np.uint8)
    h = _lib.handle()
    keep = [prompt, output, ku, kd]
    ptrs = [a.ctypes.data if a.size else None for a in keep]
    _lib.check(h.lib.eb_check_knapsack_batch(h.ptr, 1, off.ctypes.data, *ptrs, co.ctypes.data, zz.ctypes.data,
                                             tm.ctypes.data, ok.ctypes.data, _lib.EB_MEM_HOST),
               "eb_check_knapsack_batch")
    return bool(ok[0])


def check_direct_many(subsets, ctx, padded_lens, device=None):
    """Batched direct P1 check (feasibility.py:192-223): returns (ok[n], metrics[n, 4])."""
    rows = []
    off = np.zeros(len(subsets) + 1, dtype=np.int64)
    for i, s in enumerate(subsets):
        rows.extend(s)
        off[i + 1] = len(rows)
    cols = request_columns(rows) if rows else request_columns([])
    members = np.arange(len(rows), dtype=np.int32)
    rec = context_record(ctx)
    n = len(subsets)
    pad = np.ascontiguousarray(padded_lens, dtype=np.int64)
    status = np.zeros(n, dtype=np.int32)
    ok = np.zeros(n, dtype=np.uint8)
    met = np.zeros((n, 4), dtype=np.float64)
    if not rows:   # keep every pointer valid for the empty case
        cols = {k: np.zeros(1, dtype=v.dtype) for k, v in cols.items()}
        members = np.zeros(1, dtype=np.int32)
    rs = requests_struct(cols)
    h = _lib.handle(device)
    _lib.check(h.lib.eb_check_direct_batch(h.ptr, rec.ctypes.data, 1, _ref(rs), max(len(rows), 1), n,
                                           off.ctypes.data, members.ctypes.data, None, pad.ctypes.data,
                                           status.ctypes.data, ok.ctypes.data, met.ctypes.data, _lib.EB_MEM_HOST),
               "eb_check_direct_batch")
    for s in status:
        if s:
            raise_for_status(int(s))
    return ok.astype(bool), met


def check_direct(subset, ctx, padded_len: int) -> bool:
    """Direct evaluation of the original constraints (feasibility.py:192-223) on the GPU."""
    ok, _ = check_direct_many([list(subset)], ctx, [padded_len])
    return bool(ok[0])
