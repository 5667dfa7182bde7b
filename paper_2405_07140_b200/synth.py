"""Synthetic scheduling instances for the benchmark configs.

Each instance is one ``dftsp(candidates, ctx)`` call on K candidates that
already passed the simulator's admission (``sim._dftsp_candidates``,
sim.py:264-274: accuracy filter + alone-feasible prefilter).  Requests are
drawn with numpy (prompt, output, deadline*scale, tolerance*cap, Rayleigh
gain, waiting ~ U[0, epoch)) in vectorised rounds; admission is decided
exactly on the GPU by the K1 kernel (``eb_admission_batch``) by default; the first K
admitted draws of each instance are kept, ids 0..K-1 in acceptance order.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .catalog import delta_ppl, get_model, get_profile
from .soa import REQ_FIELDS, InstanceBatch


def dbm(x: float) -> float:
    return 10.0 ** (x / 10.0) / 1000.0


@dataclass(frozen=True)
class Workload:
    name: str
    model: str = "bloom-3b"
    profiles: tuple = ("fp16", "w8a16", "w4a16-gptq")
    prompts: tuple = (128, 256, 512)
    outputs: tuple = (128, 256, 512)
    gpu_count: int = 20
    flops_per_gpu: float = 1.33e12
    memory_per_gpu: float = 32e9
    band_hz: float = 20e6
    deadline: tuple = (0.5, 2.0)
    deadline_scale: float = 1.0
    tolerance_cap: float = 1.0
    epoch_s: float = 2.0
    slot_s: float = 0.25
    K: int = 20


CONFIG2 = Workload("config2: Monte Carlo K=20, fp16/w8a16/w4a16-gptq mix, BLOOM-3B, paper defaults")
CONFIG5 = Workload("config5: tight-memory OPT-13B w4a16-gptq, 5 output classes", model="opt-13b",
                   profiles=("w4a16-gptq",), prompts=(512, 1024, 2048), outputs=(64, 128, 256, 512, 1024),
                   gpu_count=1, flops_per_gpu=2.0e15, memory_per_gpu=1.08e10)


def contexts(w: Workload) -> np.ndarray:
    """eb_context records, one per quantization profile of the workload (delta_ppl filled)."""
    llm = get_model(w.model)
    recs = np.zeros(len(w.profiles), dtype=_lib.CTX_DTYPE)
    for i, p in enumerate(w.profiles):
        q = get_profile(p)
        r = recs[i]
        r["layers"], r["hidden_dim"], r["head_count"] = llm.layers, llm.hidden_dim, llm.head_count
        r["head_dim"], r["ffn_dim"], r["bytes_per_param"] = llm.head_dim, llm.ffn_dim, llm.bytes_per_param
        r["alpha"], r["beta"], r["delta_ppl"] = q.alpha, q.beta, delta_ppl(q, llm.name)
        r["uplink_band_hz"] = r["downlink_band_hz"] = w.band_hz
        r["downlink_power_w"] = dbm(43.0)
        r["noise_density_w_hz"] = dbm(-174.0)
        r["uplink_slot_s"] = r["downlink_slot_s"] = w.slot_s
        r["bits_per_token"] = 16
        r["flops_per_s"] = w.gpu_count * w.flops_per_gpu
        r["memory_bytes"] = w.gpu_count * w.memory_per_gpu
        r["gpu_count"] = w.gpu_count
        r["has_slot_cap"] = 1
        r["slot_cap_s"] = w.epoch_s
    return recs


def _draw(rng, n, w: Workload):
    return {
        "prompt_tokens": rng.choice(np.array(w.prompts, np.int32), size=n),
        "output_tokens": rng.choice(np.array(w.outputs, np.int32), size=n),
        "deadline_s": w.deadline_scale * rng.uniform(w.deadline[0], w.deadline[1], size=n),
        "tolerance": w.tolerance_cap * rng.uniform(0.0, 1.0, size=n),
        "channel_gain": rng.exponential(1e-3, size=n),
        "waiting_s": rng.uniform(0.0, w.epoch_s, size=n),
    }


def device_admission(device=None):
    """K1 admission hook on the GPU: (batch, recs) -> (status, keep) per row."""
    h = _lib.handle(device)

    def admit(batch: InstanceBatch, recs):
        nr = batch.n_req
        status = np.zeros(nr, np.int32)
        keep = np.zeros(nr, np.uint8)
        b = batch.struct()
        _lib.check(h.lib.eb_admission_batch(h.ptr, recs.ctypes.data, len(recs),
                                            ctypes.cast(ctypes.pointer(b), ctypes.c_void_p), 1, 1,
                                            status.ctypes.data, keep.ctypes.data, _lib.EB_MEM_HOST),
                   "eb_admission_batch")
        return status, keep

    return admit


def generate(w: Workload, n_inst: int, seed: int = 2405_07140, chunk: int = 100_000, device=None,
             admit=None) -> InstanceBatch:
    """n_inst instances of exactly w.K admitted candidates each (host arrays).

    ``admit(batch, recs) -> (status, keep)`` decides admission per drawn row;
    the default is the device K1 kernel.  Any admission with the reference's
    decisions yields the identical batch (the draws depend only on the seed
    and the keep decisions), which is how the CPU reference arm rebuilds the
    same instances without the CUDA library (bench.py --impl reference)."""
    recs = contexts(w)
    admit = admit or device_admission(device)
    rng = np.random.default_rng(seed)
    prof = rng.integers(0, len(w.profiles), size=n_inst).astype(np.int32)
    K = w.K
    out = {name: np.empty(n_inst * K, dt) for name, dt in REQ_FIELDS}
    p_up = dbm(20.0)
    for c0 in range(0, n_inst, chunk):
        c1 = min(n_inst, c0 + chunk)
        m = c1 - c0
        got = np.zeros(m, np.int64)
        rate = np.full(m, 0.3)
        while True:
            need = K - got
            act = np.nonzero(need > 0)[0]
            if act.size == 0:
                break
            R = np.ceil(need[act] / rate[act] * 1.5).astype(np.int64) + 4
            off = np.zeros(act.size + 1, np.int64)
            np.cumsum(R, out=off[1:])
            nr = int(off[-1])
            cols = _draw(rng, nr, w)
            cols["uplink_power_w"] = np.full(nr, p_up)
            cols["id"] = np.zeros(nr, np.int64)
            ci = prof[c0 + act]
            batch = InstanceBatch(off, {k: np.ascontiguousarray(v) for k, v in cols.items()}, recs,
                                  np.ascontiguousarray(ci), int(R.max()))
            status, keep = admit(batch, recs)
            owner = np.repeat(np.arange(act.size), R)
            kept = keep.astype(bool) & (status == 0)
            # rank of each kept row within its instance (draw order)
            csum = np.cumsum(kept)
            base = np.concatenate([[0], csum[off[1:-1] - 1]]) if act.size > 1 else np.array([0])
            rank = csum - base[owner] - 1
            take = kept & (rank < need[act][owner])
            rows = np.nonzero(take)[0]
            inst = act[owner[rows]]
            slot = got[inst] + rank[rows]
            dest = (c0 + inst) * K + slot
            for name, _ in REQ_FIELDS:
                if name == "id":
                    out["id"][dest] = slot
                else:
                    out[name][dest] = cols[name][rows]
            kept_per = np.bincount(owner[kept], minlength=act.size)
            got[act] += np.minimum(kept_per, need[act])
            rate[act] = np.maximum(kept_per / np.maximum(R, 1), 0.02)
    offsets = np.arange(n_inst + 1, dtype=np.int64) * K
    return InstanceBatch(offsets, out, recs, prof, K)


def brute_family(K: int, n: int, seed: int = 2405_07140, z0: int | None = None, deadline_frac: float = 0.3):
    """Config-4 instances that keep the brute force honest: pools of K users
    whose uplink and downlink fractions are anti-correlated (long prompts with
    short outputs and vice versa, Rayleigh gains), with the uplink and
    downlink slots scaled per pool so that the z0 smallest uplink terms and the
    z0 smallest downlink terms each just fit (z0 = K/2 by default).  The level
    bounds (z smallest terms of each resource apart) then leave every level up
    to z0 live, while the largest jointly feasible batch is smaller: the
    levels in between must be enumerated.  A share `deadline_frac` of the
    users carry deadlines that only fit batches up to a per-user size, so the
    deadline constraint binds on some subsets too.  No slot cap; memory slack.

    Returns [(ctx_rec (1 record), columns)] -- the reference's
    exhaustive_optimal(pool, ctx, cap=K) inputs."""
    from .costs import flops_autoregressive, flops_initial
    rng = np.random.default_rng(seed)
    llm = get_model("bloom-3b")
    q = get_profile("w8a16")
    z0 = z0 or K // 2
    out = []
    for _ in range(n):
        s = rng.integers(32, 2049, size=K).astype(np.int32)
        nout = np.clip(np.rint((2 ** 21) / s * rng.uniform(0.6, 1.4, size=K)), 16, 2048).astype(np.int32)
        gain = rng.exponential(1e-3, size=K)
        p_up = dbm(20.0)
        rec = contexts(Workload("brute", profiles=("w8a16",)))
        r = rec[0]
        noise = r["noise_density_w_hz"] * r["uplink_band_hz"]
        eff_up = np.log2(1.0 + p_up * gain / noise)
        eff_dn = np.log2(1.0 + r["downlink_power_w"] * gain / noise)
        c_up = s * 16.0 / (r["uplink_band_hz"] * eff_up)           # a_i = c_up / T_up
        c_dn = nout * 16.0 / (r["downlink_band_hz"] * eff_dn)
        r["uplink_slot_s"] = np.sort(c_up)[:z0].sum() / 0.999
        r["downlink_slot_s"] = np.sort(c_dn)[:z0].sum() / 0.999
        r["has_slot_cap"] = 0
        r["memory_bytes"] = 1e15
        r["flops_per_s"] = 20 * 1.33e12
        slots = float(r["uplink_slot_s"] + r["downlink_slot_s"])
        waiting = rng.uniform(0.0, 0.5, size=K)
        pad = int(s.max())
        fi = flops_initial(llm, pad)
        med = int(np.median(nout))
        zi = rng.integers(max(1, K // 4), K + 1, size=K)
        comp = np.array([q.beta * (int(z) * fi + int(z) * flops_autoregressive(llm, pad, med)) / r["flops_per_s"]
                         for z in zi])
        tight = rng.random(K) < deadline_frac
        deadline = np.where(tight, waiting + slots + comp, waiting + slots + 1e3)
        cols = {"id": np.arange(K, dtype=np.int64), "prompt_tokens": s, "output_tokens": nout,
                "deadline_s": deadline.astype(np.float64), "waiting_s": waiting, "tolerance": np.ones(K),
                "channel_gain": gain, "uplink_power_w": np.full(K, p_up)}
        out.append((rec, {k: np.ascontiguousarray(v) for k, v in cols.items()}))
    return out
