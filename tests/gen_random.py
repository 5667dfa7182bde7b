"""Seeded random instance batches for device-vs-oracle parity (numpy only).

Modeled on the reference test strategy (pkg/tests/conftest.py:27-86): small
random models, random ladders and radio/node scaling so that each of the four
budgets (uplink, downlink, memory, deadline) binds on a share of instances.
Everything is vectorised straight into an InstanceBatch; no /root/reference.
"""
from __future__ import annotations

import numpy as np

from paper_2405_07140_b200._lib import CTX_DTYPE
from paper_2405_07140_b200.soa import REQ_FIELDS, InstanceBatch

LADDER_POOL = np.array([16, 32, 64, 128, 256])


def _flops_initial(L, d, f, s):
    return L * (6 * s * d * d + (4 * s * s * d + 2 * s * d * d) + 4 * s * d * f)


def _flops_ar(L, d, f, s, n):
    return L * (n - 1) * (8 * d * d + 4 * s * d + 4 * d * f + 2 * d * n)


def random_batch(seed: int, n_inst: int, k_min: int = 0, k_max: int = 14, max_classes: int = 3,
                 slot_cap_frac: float = 0.3, dup_ladder: bool = True):
    """Returns (InstanceBatch, ladders[n_inst] tuple) with one context per instance."""
    rng = np.random.default_rng(seed)
    ctx = np.zeros(n_inst, dtype=CTX_DTYPE)
    sizes = rng.integers(k_min, k_max + 1, size=n_inst)
    off = np.zeros(n_inst + 1, np.int64)
    np.cumsum(sizes, out=off[1:])
    nr = int(off[-1])
    cols = {name: np.zeros(max(nr, 1), dt) for name, dt in REQ_FIELDS}
    ladders = []
    p_up = 10.0 ** (20.0 / 10.0) / 1000.0
    for i in range(n_inst):
        ncls = int(rng.integers(1, max_classes + 1))
        ladder = tuple(sorted(int(v) for v in rng.choice(LADDER_POOL, size=ncls, replace=False)))
        ladders.append(ladder)
        heads, hd = int(rng.choice([2, 4])), int(rng.choice([8, 16]))
        d = heads * hd
        L = int(rng.integers(1, 5))
        c = ctx[i]
        c["layers"], c["hidden_dim"], c["head_count"], c["head_dim"], c["ffn_dim"], c["bytes_per_param"] = \
            L, d, heads, hd, 4 * d, 2
        c["alpha"] = float(rng.choice([0.25, 0.5, 1.0]))
        c["beta"] = float(rng.choice([0.7, 0.8, 1.0]))
        roomy = rng.random() < 0.3
        lo, hi = int(off[i]), int(off[i + 1])
        k = hi - lo
        s = rng.integers(8, 257, size=k)
        cols["id"][lo:hi] = rng.permutation(1000)[:k] if k else []
        cols["prompt_tokens"][lo:hi] = s
        cols["output_tokens"][lo:hi] = rng.choice(ladder, size=k)
        cols["deadline_s"][lo:hi] = rng.uniform(0.2, 2.5, size=k) * (2.0 if roomy else 1.0)
        cols["tolerance"][lo:hi] = rng.uniform(0.0, 1.0, size=k)
        cols["channel_gain"][lo:hi] = rng.exponential(1e-3, size=k)
        cols["uplink_power_w"][lo:hi] = p_up
        cols["waiting_s"][lo:hi] = rng.uniform(0.0, 0.8, size=k)
        c["uplink_band_hz"] = float(rng.uniform(2e4, 2e6))
        c["downlink_band_hz"] = float(rng.uniform(2e4, 2e6))
        c["downlink_power_w"] = 10.0 ** (43.0 / 10.0) / 1000.0
        c["noise_density_w_hz"] = 10.0 ** (-174.0 / 10.0) / 1000.0
        c["uplink_slot_s"] = float(rng.uniform(0.1, 0.3))
        c["downlink_slot_s"] = float(rng.uniform(0.1, 0.3))
        c["bits_per_token"] = 16
        pad = int(s.max()) if k else 64
        per = _flops_initial(L, d, 4 * d, pad) + _flops_ar(L, d, 4 * d, pad, int(np.median(ladder)))
        z_lat = float(rng.uniform(0.5, 10.0)) * (2.0 if roomy else 1.0)
        c["flops_per_s"] = max(c["beta"] * per * z_lat, 1e6)
        z_mem = float(rng.uniform(0.0, 10.0)) * (2.0 if roomy else 1.0)
        kv = 2 * 2 * L * d * (pad + max(ladder))
        w = L * (4 * 2 * d * hd * heads + 2 * 2 * d * 4 * d)
        c["memory_bytes"] = max(c["alpha"] * (w + z_mem * kv), 1.0)
        c["gpu_count"] = int(rng.integers(1, 5))
        if rng.random() < slot_cap_frac:
            c["has_slot_cap"] = 1
            c["slot_cap_s"] = float(rng.uniform(0.2, 2.0))
    batch = InstanceBatch(off, cols, ctx, np.arange(n_inst, dtype=np.int32), max(int(sizes.max()), 1))
    return batch, ladders


def group_by_ladder(batch: InstanceBatch, ladders):
    """Split into per-ladder sub-batches: {ladder: (idx, sub_batch)}."""
    out = {}
    for i, lad in enumerate(ladders):
        out.setdefault(lad, []).append(i)
    res = {}
    for lad, idx in out.items():
        res[lad] = (idx, take(batch, idx))
    return res


def take(batch: InstanceBatch, idx) -> InstanceBatch:
    off = batch.offsets
    sizes = np.array([off[i + 1] - off[i] for i in idx], np.int64)
    new_off = np.zeros(len(idx) + 1, np.int64)
    np.cumsum(sizes, out=new_off[1:])
    rows = np.concatenate([np.arange(off[i], off[i + 1]) for i in idx]) if len(idx) else np.zeros(0, np.int64)
    cols = {k: np.ascontiguousarray(v[rows]) if len(rows) else np.zeros(1, v.dtype) for k, v in batch.columns.items()}
    ci = np.ascontiguousarray(batch.ctx_index[list(idx)], np.int32)
    return InstanceBatch(new_off, cols, batch.contexts, ci, max(int(sizes.max()) if len(sizes) else 1, 1))
