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
