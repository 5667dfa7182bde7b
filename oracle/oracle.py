"""CPU ORACLE -- test infrastructure only.

ctypes wrapper of ``oracle/liboracle.so`` (the literal C restatement of the
reference hot path in ``oracle/edgebatch_oracle.c``).  Imported only by
tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` arm, always as the checker or the CPU baseline -- never
by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2405_07140_b200 import _lib  # noqa: E402  (struct layouts of the ABI header only)
from paper_2405_07140_b200.soa import InstanceBatch, search_params  # noqa: E402

LIB_PATH = os.path.join(HERE, "liboracle.so")
MAXC = _lib.EB_MAX_CLASSES
MAXK = _lib.EB_MAX_K
_o = None


def load():
    global _o
    if _o is None:
        if not os.path.exists(LIB_PATH):
            from paper_2405_07140_b200._build import build_oracle
            build_oracle()
        lib = C.CDLL(LIB_PATH)
        P, I32, I64, F64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        lib.oracle_dftsp_batch.restype = I32
        lib.oracle_dftsp_batch.argtypes = [P, I32, P, P, P, I32]
        lib.oracle_exhaustive.restype = I32
        lib.oracle_exhaustive.argtypes = [P, I32, P, P, P, P, P, P, P, I32, I32, P, P, P, P]
        lib.oracle_check_direct.restype = I32
        lib.oracle_check_direct.argtypes = [P, I32, P, P, P, P, P, P, I64, P]
        lib.oracle_batch_cost.restype = None
        lib.oracle_batch_cost.argtypes = [P, I32, P, P, I64, I64, P]
        lib.oracle_static_batch_size.restype = I64
        lib.oracle_static_batch_size.argtypes = [P, F64, I64, I64]
        lib.oracle_coefficients.restype = I32
        lib.oracle_coefficients.argtypes = [P, I32, P, P, P, P, P, P, I64, P, P]
        lib.oracle_check_knapsack.restype = I32
        lib.oracle_check_knapsack.argtypes = [P, I32, P, P, P, P, P, P, I32, P, I32, F64]
        lib.oracle_stb.restype = None
        lib.oracle_stb.argtypes = [P, I32, P, P, P, P, P, I64, F64, I32, P]
        lib.oracle_work_reset.restype = None
        lib.oracle_work_reset.argtypes = []
        lib.oracle_work_get.restype = None
        lib.oracle_work_get.argtypes = [P]
        lib.oracle_exhaustive_level.restype = I64
        lib.oracle_exhaustive_level.argtypes = [P, I32, P, P, P, P, P, P, P, I32, I64, I64]
        lib.oracle_exhaustive_counts.restype = I32
        lib.oracle_exhaustive_counts.argtypes = [P, P, I32, P, P, P, P, P, P, P, P, P, P]
        lib.oracle_nob.restype = None
        lib.oracle_nob.argtypes = [P, I32, P, P, P, F64, F64, I32, P, P, P, P]
        lib.oracle_admission_batch.restype = I32
        lib.oracle_exhaustive_mt.restype = I32
        lib.oracle_exhaustive_mt.argtypes = [P, I32, P, P, P, P, P, P, P, I32, I32, P, P, P]
        lib.oracle_admission_batch.argtypes = [P, I32, P, I32, I32, P, P, I32]
        _o = lib
    return _o


def _ref(s):
    return C.cast(C.pointer(s), C.c_void_p)


def dftsp_batch(batch: InstanceBatch, *, pruning=True, inclusive_bound=False, exact_tau=False,
                collect_trajectory=False, ladder=None, threads=1) -> dict:
    """Oracle dftsp over an InstanceBatch; returns the same arrays as search.solve_batch."""
    lib = load()
    n, nr = batch.n_inst, batch.n_req
    sizes = np.diff(batch.offsets)
    res = dict(status=np.zeros(n, np.int32), error_index=np.full(n, -1, np.int32), z_found=np.zeros(n, np.int32),
               nodes_visited=np.zeros(n, np.int64), nodes_pruned=np.zeros(n, np.int64),
               n_classes=np.zeros(n, np.int32), counts=np.zeros((n, MAXC), np.int32),
               class_lengths=np.zeros((n, MAXC), np.int32), solution=np.full(max(nr, 1), -1, np.int32),
               metrics=np.zeros((n, _lib.EB_N_METRICS)))
    out = _lib.eb_dftsp_result()
    for k in ("status", "error_index", "z_found", "nodes_visited", "nodes_pruned", "n_classes", "counts",
              "class_lengths", "solution", "metrics"):
        setattr(out, k, res[k].ctypes.data)
    if collect_trajectory:
        rows = sizes * (sizes + 1) // 2
        res["traj_offsets"] = np.zeros(n + 1, np.int64)
        np.cumsum(rows, out=res["traj_offsets"][1:])
        res["traj"] = np.zeros((max(int(res["traj_offsets"][-1]), 1), 4), np.int64)
        res["traj_len"] = np.zeros(n, np.int32)
        out.traj_offsets = res["traj_offsets"].ctypes.data
        out.traj = res["traj"].ctypes.data
        out.traj_len = res["traj_len"].ctypes.data
    prm = search_params(pruning, inclusive_bound, exact_tau, collect_trajectory, ladder)
    b = batch.struct()
    lib.oracle_dftsp_batch(batch.contexts.ctypes.data, len(batch.contexts), _ref(prm), _ref(b), _ref(out),
                           int(threads))
    return res


def exhaustive(ctx_rec, cols, lo, hi, cap=64, hoist=True):
    """Oracle exhaustive_optimal(mode='subsets') on rows [lo, hi): (status, z, lexrank, nodes, mask)."""
    lib = load()
    n = hi - lo
    z = C.c_int32(0); rk = C.c_int64(0); nodes = C.c_int64(0); mask = C.c_uint64(0)
    a = {k: np.ascontiguousarray(v[lo:hi]) for k, v in cols.items()}
    st = lib.oracle_exhaustive(ctx_rec.ctypes.data, n, a["id"].ctypes.data, a["prompt_tokens"].ctypes.data,
                               a["output_tokens"].ctypes.data, a["deadline_s"].ctypes.data,
                               a["waiting_s"].ctypes.data, a["channel_gain"].ctypes.data,
                               a["uplink_power_w"].ctypes.data, int(cap), int(hoist), C.byref(z), C.byref(rk),
                               C.byref(nodes), C.byref(mask))
    return st, z.value, rk.value, nodes.value, mask.value


def work_counters(batch: InstanceBatch, ladder=None, threads=1, **flags) -> dict:
    """Leaf checks / descends / prune events the reference search performs on `batch`."""
    lib = load()
    lib.oracle_work_reset()
    dftsp_batch(batch, ladder=ladder, threads=threads, **flags)
    w = np.zeros(4, np.int64)
    lib.oracle_work_get(w.ctypes.data)
    return dict(leaf_checks=int(w[0]), descends=int(w[1]), prune_events=int(w[2]))


def level_evaluator(ctx_rec, cols):
    """CPU twin of brute.device_level_range: (z, lo, hi) -> first feasible rank or -1."""
    lib = load()
    a = {k: np.ascontiguousarray(v) for k, v in cols.items()}
    n = int(a["prompt_tokens"].shape[0])

    def level(z, lo, hi):
        r = lib.oracle_exhaustive_level(ctx_rec.ctypes.data, n, a["id"].ctypes.data, a["prompt_tokens"].ctypes.data,
                                        a["output_tokens"].ctypes.data, a["deadline_s"].ctypes.data,
                                        a["waiting_s"].ctypes.data, a["channel_gain"].ctypes.data,
                                        a["uplink_power_w"].ctypes.data, int(z), int(lo), int(hi))
        if r == -2:
            raise ValueError("spectral efficiency is zero")
        return int(r)

    return level


def exhaustive_counts(ctx_rec, cols, lo, hi, ladder=None):
    """Oracle exhaustive_optimal(mode='counts') on rows [lo, hi): (status, z, nodes, solution)."""
    lib = load()
    n = hi - lo
    a = {k: np.ascontiguousarray(v[lo:hi]) for k, v in cols.items()}
    z = C.c_int32(0); nodes = C.c_int64(0)
    sol = np.full(max(n, 1), -1, np.int32)
    prm = search_params(ladder=ladder)
    st = lib.oracle_exhaustive_counts(ctx_rec.ctypes.data, _ref(prm), n, a["id"].ctypes.data,
                                      a["prompt_tokens"].ctypes.data, a["output_tokens"].ctypes.data,
                                      a["deadline_s"].ctypes.data, a["waiting_s"].ctypes.data,
                                      a["channel_gain"].ctypes.data, a["uplink_power_w"].ctypes.data,
                                      C.byref(z), C.byref(nodes), sol.ctypes.data)
    return st, z.value, nodes.value, tuple(int(x) for x in sol[:z.value])


def admission_batch(batch: InstanceBatch, accuracy_check=True, prefilter=True, threads=None):
    """Oracle sim._dftsp_candidates (sim.py:264-274) per row: (status, keep)."""
    lib = load()
    nr = batch.n_req
    status = np.zeros(max(nr, 1), np.int32)
    keep = np.zeros(max(nr, 1), np.uint8)
    b = batch.struct()
    lib.oracle_admission_batch(batch.contexts.ctypes.data, len(batch.contexts), _ref(b), int(accuracy_check),
                               int(prefilter), status.ctypes.data, keep.ctypes.data,
                               int(threads or os.cpu_count() or 1))
    return status[:nr], keep[:nr]


def admit(batch: InstanceBatch, recs):
    """synth.generate's admission hook computed by the oracle (no device)."""
    return admission_batch(batch)


def exhaustive_mt(ctx_rec, cols, threads=None, z_top=0):
    """Literal multi-threaded level scan (no bounds, no pruning) of
    exhaustive_optimal(mode='subsets') on a whole pool: (status, z, lexrank, checked).
    ``z_top`` > 0 starts at that level (the caller proved the ones above infeasible)."""
    lib = load()
    a = {k: np.ascontiguousarray(v) for k, v in cols.items()}
    n = int(a["prompt_tokens"].shape[0])
    z = C.c_int32(0); rk = C.c_int64(0); chk = C.c_int64(0)
    st = lib.oracle_exhaustive_mt(ctx_rec.ctypes.data, n, a["id"].ctypes.data, a["prompt_tokens"].ctypes.data,
                                  a["output_tokens"].ctypes.data, a["deadline_s"].ctypes.data,
                                  a["waiting_s"].ctypes.data, a["channel_gain"].ctypes.data,
                                  a["uplink_power_w"].ctypes.data, int(threads or os.cpu_count() or 1),
                                  int(z_top), C.byref(z), C.byref(rk), C.byref(chk))
    return st, z.value, rk.value, chk.value


def link_fractions(ctx_rec, cols):
    """Per-member (uplink, downlink) fraction terms s*k_up and n*k_down, as
    check_direct forms them (feasibility.py:203-205), from the oracle's libm
    log2 -- for the tests' level-bound proofs."""
    import math
    r = ctx_rec[0]
    nu = float(r["noise_density_w_hz"]) * float(r["uplink_band_hz"])
    nd = float(r["noise_density_w_hz"]) * float(r["downlink_band_hz"])
    up, dn = [], []
    for s, o, g, p in zip(cols["prompt_tokens"].tolist(), cols["output_tokens"].tolist(),
                          cols["channel_gain"].tolist(), cols["uplink_power_w"].tolist()):
        ku = float(r["bits_per_token"]) / (float(r["uplink_slot_s"]) * float(r["uplink_band_hz"]) *
                                          math.log2(1.0 + p * g / nu))
        kd = float(r["bits_per_token"]) / (float(r["downlink_slot_s"]) * float(r["downlink_band_hz"]) *
                                          math.log2(1.0 + float(r["downlink_power_w"]) * g / nd))
        up.append(s * ku)
        dn.append(o * kd)
    return np.array(up), np.array(dn)
