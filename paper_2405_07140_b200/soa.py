"""Structure-of-arrays packing between reference-style objects and the C ABI.

Host logic only (no arithmetic of the hot path): flattens ``EdgeContext``-like
objects into ``eb_context`` records and ``Request``-like objects into SoA
columns, and wraps batches of instances (CSR offsets) for the batched entry
points.  Objects are duck-typed, so the reference's own ``edgebatch``
dataclasses can be passed unchanged.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import CTX_DTYPE, eb_batch, eb_requests, ptr

REQ_FIELDS = (("id", np.int64), ("prompt_tokens", np.int32), ("output_tokens", np.int32),
              ("deadline_s", np.float64), ("waiting_s", np.float64), ("tolerance", np.float64),
              ("channel_gain", np.float64), ("uplink_power_w", np.float64))
INT32_MAX = 2**31 - 1


def _int_field(value, name: str) -> int:
    iv = int(value)
    if iv != value:
        raise ValueError(f"{name} must be integral for the device cost model, got {value!r}")
    return iv


def context_record(ctx, delta: float = 0.0) -> np.ndarray:
    """One eb_context record from an EdgeContext-like object (feasibility.py:59-71)."""
    rec = np.zeros(1, dtype=CTX_DTYPE)
    llm, quant, radio, node = ctx.llm, ctx.quant, ctx.radio, ctx.node
    rec["layers"] = llm.layers
    rec["hidden_dim"] = llm.hidden_dim
    rec["head_count"] = llm.head_count
    rec["head_dim"] = llm.head_dim
    rec["ffn_dim"] = llm.ffn_dim
    rec["bytes_per_param"] = llm.bytes_per_param
    rec["alpha"] = float(quant.alpha)
    rec["beta"] = float(quant.beta)
    rec["delta_ppl"] = float(delta)
    rec["uplink_band_hz"] = float(radio.uplink_band_hz)
    rec["downlink_band_hz"] = float(radio.downlink_band_hz)
    rec["downlink_power_w"] = float(radio.downlink_power_w)
    rec["noise_density_w_hz"] = float(radio.noise_density_w_hz)
    rec["uplink_slot_s"] = float(radio.uplink_slot_s)
    rec["downlink_slot_s"] = float(radio.downlink_slot_s)
    rec["bits_per_token"] = _int_field(radio.bits_per_token, "bits_per_token")
    rec["flops_per_s"] = float(node.flops_per_s)
    rec["memory_bytes"] = float(node.memory_bytes)
    rec["gpu_count"] = int(node.gpu_count)
    cap = getattr(ctx, "slot_cap_s", None)
    rec["has_slot_cap"] = 0 if cap is None else 1
    rec["slot_cap_s"] = 0.0 if cap is None else float(cap)
    return rec


def request_columns(reqs) -> dict:
    """SoA columns of a list of Request-like objects (order preserved)."""
    n = len(reqs)
    cols = {name: np.empty(n, dtype=dt) for name, dt in REQ_FIELDS}
    for j, r in enumerate(reqs):
        s, o = int(r.prompt_tokens), int(r.output_tokens)
        if not (0 <= s <= INT32_MAX and 0 <= o <= INT32_MAX):
            raise ValueError("prompt/output token counts must fit in int32 for the device path")
        cols["id"][j] = r.id
        cols["prompt_tokens"][j] = s
        cols["output_tokens"][j] = o
        cols["deadline_s"][j] = r.deadline_s
        cols["waiting_s"][j] = r.waiting_s
        cols["tolerance"][j] = r.tolerance
        cols["channel_gain"][j] = r.link.channel_gain
        cols["uplink_power_w"][j] = r.link.uplink_power_w
    return cols


def requests_struct(cols: dict) -> eb_requests:
    s = eb_requests()
    for name, _ in REQ_FIELDS:
        a = cols.get(name)
        setattr(s, name, ptr(a) if a is not None else None)
    s._keep = cols          # the struct holds raw pointers: keep the arrays alive with it
    return s


@dataclass
class InstanceBatch:
    """A batch of independent instances: CSR offsets over SoA request columns.

    Columns are numpy arrays (host) or torch tensors (device, then
    ``on_device`` is True).  ``contexts`` is an array of eb_context records;
    ``ctx_index`` maps each instance to one of them.
    """

    offsets: object
    columns: dict
    contexts: np.ndarray
    ctx_index: object = None
    k_max: int = 0
    on_device: bool = False

    @property
    def n_inst(self) -> int:
        return int(self.offsets.shape[0]) - 1

    @property
    def n_req(self) -> int:
        return int(self.columns["prompt_tokens"].shape[0])

    def struct(self) -> eb_batch:
        b = eb_batch()
        b.n_inst = self.n_inst
        b.n_req = self.n_req
        b.offsets = ptr(self.offsets)
        b.ctx_index = ptr(self.ctx_index)
        b.req = requests_struct(self.columns)
        b.k_max = int(self.k_max)
        b._keep = self          # raw pointers into this batch's arrays
        return b

    def contexts_ptr(self):
        return C.c_void_p(self.contexts.ctypes.data)

    @classmethod
    def from_pools(cls, pools, contexts, ctx_index=None) -> "InstanceBatch":
        """Pack lists of Request-like objects (one list per instance)."""
        sizes = [len(p) for p in pools]
        offsets = np.zeros(len(pools) + 1, dtype=np.int64)
        np.cumsum(sizes, out=offsets[1:])
        flat = [r for p in pools for r in p]
        cols = request_columns(flat)
        if not isinstance(contexts, np.ndarray):
            contexts = np.concatenate([context_record(c) for c in contexts])
        ci = None if ctx_index is None else np.ascontiguousarray(ctx_index, dtype=np.int32)
        return cls(offsets, cols, contexts, ci, max(sizes) if sizes else 1)


# The compact wire format of eb_dftsp_batch_packed (include/edgebatch_b200.h):
# id int32, token counts uint16, uplink power one value when uniform.
WIRE_FIELDS = (("id", np.int32), ("prompt_tokens", np.uint16), ("output_tokens", np.uint16),
               ("deadline_s", np.float64), ("waiting_s", np.float64), ("channel_gain", np.float64))


@dataclass
class WireBatch:
    """An InstanceBatch in the compact wire format (host arrays only).

    ``offsets`` None: every instance has ``k_max`` requests.  ``columns['id']``
    None: ids are the request positions (valid when each instance's ids
    increase along its rows: the search only compares ids within an
    instance, so the results are identical)."""

    offsets: np.ndarray | None
    columns: dict
    uplink_power_w: np.ndarray      # one value (uniform) or one per request
    contexts: np.ndarray
    ctx_index: object = None
    k_max: int = 0
    n_inst_: int = 0
    # dictionary-coded token counts: token_codes (u8) = prompt index | output
    # index << 4 into these tables (None: the u16 columns are shipped)
    token_codes: np.ndarray | None = None
    prompt_dict: np.ndarray | None = None
    output_dict: np.ndarray | None = None

    @property
    def n_inst(self) -> int:
        return int(self.offsets.shape[0]) - 1 if self.offsets is not None else self.n_inst_

    @property
    def n_req(self) -> int:
        return int(self.columns["deadline_s"].shape[0])

    @property
    def uniform_power(self) -> bool:
        return self.uplink_power_w.shape[0] == 1

    def sizes(self) -> np.ndarray:
        if self.offsets is None:
            return np.full(self.n_inst, self.k_max, np.int64)
        return np.diff(self.offsets)

    def nbytes(self) -> int:
        """Bytes one host->device pass of this batch moves."""
        n = sum(int(a.nbytes) for a in self.columns.values() if a is not None) + int(self.uplink_power_w.nbytes)
        if self.token_codes is not None:
            n += int(self.token_codes.nbytes)
        if self.offsets is not None:
            n += int(self.offsets.nbytes)
        if self.ctx_index is not None:
            n += int(self.ctx_index.nbytes)
        return n

    def struct(self) -> "_lib.eb_batch_packed":
        r = _lib.eb_requests_packed()
        for name, _ in WIRE_FIELDS:
            a = self.columns.get(name)
            setattr(r, name, ptr(a) if a is not None else None)
        r.uplink_power_w = ptr(self.uplink_power_w)
        r.uplink_power_uniform = int(self.uniform_power)
        if self.token_codes is not None:
            r.token_codes = ptr(self.token_codes)
            r.n_dict = max(len(self.prompt_dict), len(self.output_dict))
            for i, v in enumerate(self.prompt_dict):
                r.prompt_dict[i] = int(v)
            for i, v in enumerate(self.output_dict):
                r.output_dict[i] = int(v)
        b = _lib.eb_batch_packed()
        b.n_inst = self.n_inst
        b.n_req = self.n_req
        b.offsets = ptr(self.offsets) if self.offsets is not None else None
        b.ctx_index = ptr(self.ctx_index)
        b.req = r
        b.k_max = int(self.k_max)
        b._keep = self
        return b


def pack_wire(batch: InstanceBatch, pin=None, implicit=True) -> WireBatch | None:
    """The wire-format copy of a host batch, or None when a column does not
    narrow losslessly (ids outside int32, token counts outside uint16) or an
    instance is wider than EB_MAX_K.  With ``implicit``, ids that increase
    along every instance's rows and uniform instance sizes are not shipped,
    and token counts with at most 16 distinct values each travel as one
    dictionary byte per request.
    ``pin`` (e.g. ``lambda a: torch.from_numpy(a).pin_memory().numpy()``)
    places the arrays in pinned memory."""
    cols = batch.columns
    sizes = np.diff(batch.offsets)
    if batch.n_inst and int(sizes.max()) > _lib.EB_MAX_K:
        return None
    ids, pt, ot = cols["id"], cols["prompt_tokens"], cols["output_tokens"]
    for a in (pt, ot):
        if a.size and (a.min() < 0 or a.max() > 0xFFFF):
            return None
    out = {name: np.ascontiguousarray(cols[name], dtype=dt) for name, dt in WIRE_FIELDS if name != "id"}
    codes = pdict = odict = None
    if implicit and pt.size:
        pdict, pcode = np.unique(pt, return_inverse=True)
        odict, ocode = np.unique(ot, return_inverse=True)
        if len(pdict) <= 16 and len(odict) <= 16:         # one dictionary byte per request
            codes = (pcode.astype(np.uint8) | (ocode.astype(np.uint8) << 4)).astype(np.uint8)
            out["prompt_tokens"] = out["output_tokens"] = None
        else:
            pdict = odict = None
    rising = False
    if implicit and ids.size:
        step = np.diff(ids) > 0
        first = batch.offsets[1:-1]                   # rows that start an instance (not compared)
        first = first[(first > 0) & (first < ids.size)]
        step[first - 1] = True
        rising = bool(step.all())
    if rising:
        out["id"] = None
    else:
        if ids.size and (ids.min() < -2**31 or ids.max() > INT32_MAX):
            return None
        out["id"] = np.ascontiguousarray(ids, dtype=np.int32)
    pw = np.ascontiguousarray(cols["uplink_power_w"], dtype=np.float64)
    if pw.size and (pw.view(np.int64) == pw[:1].view(np.int64)).all():    # same bits: uniform
        pw = pw[:1].copy()
    k = int(batch.k_max) if batch.k_max else (int(sizes.max()) if batch.n_inst else 1)
    k = max(1, k)
    off = np.ascontiguousarray(batch.offsets, dtype=np.int64)
    if implicit and batch.n_inst and (sizes == k).all():
        off = None
    ci = None if batch.ctx_index is None else np.ascontiguousarray(batch.ctx_index, dtype=np.int32)
    if pin is not None:
        out = {kk: (pin(v) if v is not None else None) for kk, v in out.items()}
        pw = pin(pw)
        off = None if off is None else pin(off)
        ci = None if ci is None else pin(ci)
        codes = None if codes is None else pin(codes)
    return WireBatch(off, out, pw, batch.contexts, ci, k, batch.n_inst, codes, pdict, odict)


def search_params(pruning=True, inclusive_bound=False, exact_tau=False, collect_trajectory=False, ladder=None,
                  algorithm=0, exhaustive_counts=False):
    p = _lib.eb_search_params()
    p.algorithm = int(algorithm)
    p.exhaustive_counts = int(bool(exhaustive_counts))
    p.pruning = int(bool(pruning))
    p.inclusive_bound = int(bool(inclusive_bound))
    p.exact_tau = int(bool(exact_tau))
    p.collect_trajectory = int(bool(collect_trajectory))
    if ladder is None:
        p.ladder_len = 0
    else:
        vals = sorted(set(int(v) for v in ladder))
        if len(vals) > _lib.EB_MAX_CLASSES:
            raise ValueError(f"ladder has {len(vals)} classes; the device supports {_lib.EB_MAX_CLASSES}")
        p.ladder_len = len(vals)
        for i, v in enumerate(vals):
            p.ladder[i] = v
    return p
