"""K1/K2 kernels and the batching baselines on the GPU against the reference
goldens (units corpus) and the oracle; device log2 bit-exact vs math.log2."""
import math

import numpy as np
import pytest

import oracle
from helpers import load_corpus
from paper_2405_07140_b200 import _lib, radio
from paper_2405_07140_b200.soa import InstanceBatch

pytestmark = pytest.mark.gpu


def _ref(s):
    import ctypes
    return ctypes.cast(ctypes.pointer(s), ctypes.c_void_p)


def test_device_log2_bit_exact_vs_math_log2():
    rng = np.random.default_rng(0)
    n = 1_000_000
    g = rng.exponential(1e-3, n) * 10.0 ** rng.uniform(-9, 6, n)
    p = rng.uniform(1e-3, 10.0, n)
    rec = np.zeros(1, dtype=_lib.CTX_DTYPE)
    rec["uplink_band_hz"] = rec["downlink_band_hz"] = 1.0
    rec["noise_density_w_hz"] = 7.962143e-14
    rec["downlink_power_w"] = 19.95
    rec["uplink_slot_s"] = rec["downlink_slot_s"] = 0.25
    rec["bits_per_token"] = 16
    st, out = radio.link_table(g, p, np.ones(n, np.int32), np.ones(n, np.int32), rec)
    n0 = 7.962143e-14 * 1.0
    exp = np.array([math.log2(1.0 + pi * gi / n0) for pi, gi in zip(p.tolist(), g.tolist())])
    bad = np.nonzero(out[:, 0] != exp)[0]
    assert bad.size == 0, f"{bad.size} mismatches, e.g. x={1.0 + p[bad[0]] * g[bad[0]] / n0!r}"


def _units_batch():
    d = load_corpus("units")
    b = InstanceBatch(d["offsets"], {k[4:]: np.ascontiguousarray(v) for k, v in d.items() if k.startswith("req_")},
                      np.ascontiguousarray(d["ctx"]), np.ascontiguousarray(d["ctx_index"]),
                      int(np.diff(d["offsets"]).max()))
    return d, b


def test_coefficients_match_reference():
    d, b = _units_batch()
    n = b.n_inst
    st = np.zeros(n, np.int32); err = np.zeros(n, np.int32)
    sc = np.zeros((n, 6)); rq = np.zeros((b.n_req, 4))
    h = _lib.handle()
    _lib.check(h.lib.eb_coefficients_batch(h.ptr, b.contexts.ctypes.data, len(b.contexts), _ref(b.struct()), None,
                                           st.ctypes.data, err.ctypes.data, sc.ctypes.data, rq.ctypes.data,
                                           _lib.EB_MEM_HOST), "coeff")
    assert (st == 0).all()
    assert np.array_equal(sc[:, :4], d["coef"])
    assert np.array_equal(rq[:, 0], d["coef_req"][:, 0])   # k_up
    assert np.array_equal(rq[:, 1], d["coef_req"][:, 1])   # k_down
    assert np.array_equal(rq[:, 2], d["coef_req"][:, 2])   # tau_base
    assert np.array_equal(rq[:, 3], d["coef_req"][:, 3])   # min_uplink_fraction


def test_check_direct_and_knapsack_match_reference():
    d, b = _units_batch()
    off = d["offsets"]
    sub_inst, members, sub_off = d["sub_inst"], d["sub_members"], d["sub_off"]
    rows = np.array([off[sub_inst[s]] + members[j] for s in range(len(sub_inst))
                     for j in range(sub_off[s], sub_off[s + 1])], np.int32)
    pad = np.array([int(b.columns["prompt_tokens"][off[i]:off[i + 1]].max()) for i in sub_inst], np.int64)
    ns = len(sub_inst)
    st = np.zeros(ns, np.int32); ok = np.zeros(ns, np.uint8); met = np.zeros((ns, 4))
    sc = np.ascontiguousarray(d["ctx_index"][sub_inst], np.int32)
    h = _lib.handle()
    from paper_2405_07140_b200.soa import requests_struct
    rs = requests_struct(b.columns)
    _lib.check(h.lib.eb_check_direct_batch(h.ptr, b.contexts.ctypes.data, len(b.contexts), _ref(rs), b.n_req, ns,
                                           sub_off.ctypes.data, rows.ctypes.data, sc.ctypes.data, pad.ctypes.data,
                                           st.ctypes.data, ok.ctypes.data, met.ctypes.data, _lib.EB_MEM_HOST), "cd")
    assert (st == 0).all()
    assert np.array_equal(ok, d["sub_direct"])
    # knapsack from device coefficients
    n = b.n_inst
    cst = np.zeros(n, np.int32); cerr = np.zeros(n, np.int32)
    csc = np.zeros((n, 6)); crq = np.zeros((b.n_req, 4))
    _lib.check(h.lib.eb_coefficients_batch(h.ptr, b.contexts.ctypes.data, len(b.contexts), _ref(b.struct()), None,
                                           cst.ctypes.data, cerr.ctypes.data, csc.ctypes.data, crq.ctypes.data,
                                           _lib.EB_MEM_HOST), "coeff")
    co = np.ascontiguousarray(csc[sub_inst])
    z = np.diff(sub_off).astype(np.int32)
    prompt = np.ascontiguousarray(b.columns["prompt_tokens"][rows])
    output = np.ascontiguousarray(b.columns["output_tokens"][rows])
    ku = np.ascontiguousarray(crq[rows, 0]); kd = np.ascontiguousarray(crq[rows, 1])
    tm = np.ascontiguousarray(d["sub_tau_min"])
    ok2 = np.zeros(ns, np.uint8)
    _lib.check(h.lib.eb_check_knapsack_batch(h.ptr, ns, sub_off.ctypes.data, prompt.ctypes.data, output.ctypes.data,
                                             ku.ctypes.data, kd.ctypes.data, co.ctypes.data, z.ctypes.data,
                                             tm.ctypes.data, ok2.ctypes.data, _lib.EB_MEM_HOST), "ks")
    assert np.array_equal(ok2, d["sub_knapsack"])
    assert 0 < ok.sum() < ns


def test_batch_cost_matches_reference():
    d, b = _units_batch()
    off = d["offsets"]
    n = b.n_inst
    pad = np.array([int(b.columns["prompt_tokens"][off[i]:off[i + 1]].max()) for i in range(n)], np.int64)
    out = np.zeros((n, 2))
    h = _lib.handle()
    _lib.check(h.lib.eb_batch_cost_batch(h.ptr, b.contexts.ctypes.data, len(b.contexts), n, off.ctypes.data,
                                         b.columns["prompt_tokens"].ctypes.data,
                                         b.columns["output_tokens"].ctypes.data, pad.ctypes.data, None,
                                         b.ctx_index.ctypes.data, out.ctypes.data, _lib.EB_MEM_HOST), "bc")
    assert np.array_equal(out, d["batch_cost"])


def test_static_batch_size_golden_b13():
    from paper_2405_07140_b200 import NodeCompute, get_model, get_profile, static_batch_size
    b3, w8 = get_model("bloom-3b"), get_profile("w8a16")
    assert static_batch_size(b3, w8, NodeCompute(2.66e13, 640e9, 20), 2.0, 512, 512) == 13   # test_baselines.py:46-52
    # memory-bound closed form (test_baselines.py:35-43)
    node = NodeCompute(1e20, 640e9, 20)
    from paper_2405_07140_b200 import kv_cache_bytes_per_token, weight_bytes
    kv = kv_cache_bytes_per_token(b3) * 1024
    assert static_batch_size(b3, w8, node, 2.0, 512, 512) == int((node.memory_bytes / w8.alpha - weight_bytes(b3)) // kv)
    assert static_batch_size(b3, w8, NodeCompute(2.66e13, w8.alpha * weight_bytes(b3) * 0.9, 20), 2.0, 512, 512) == 0


def test_static_batch_size_vs_oracle_sweep():
    rng = np.random.default_rng(4)
    o = oracle.load()
    n = 400
    recs = np.zeros(n, dtype=_lib.CTX_DTYPE)
    for i in range(n):
        r = recs[i]
        r["layers"], r["hidden_dim"], r["head_count"], r["head_dim"] = 30, 2560, 32, 80
        r["ffn_dim"], r["bytes_per_param"] = 10240, 2
        r["alpha"], r["beta"] = rng.choice([0.25, 0.5, 1.0]), rng.choice([0.7, 0.8, 1.0])
        r["flops_per_s"] = 10 ** rng.uniform(11, 15)
        r["memory_bytes"] = 10 ** rng.uniform(9.3, 12)
        r["gpu_count"] = 1
    slot = rng.uniform(0.1, 4.0, n); sm = rng.integers(16, 2048, n).astype(np.int64)
    nm = rng.integers(16, 1024, n).astype(np.int64)
    out = np.zeros(n, np.int64)
    h = _lib.handle()
    _lib.check(h.lib.eb_static_batch_size_batch(h.ptr, recs.ctypes.data, n, slot.ctypes.data, sm.ctypes.data,
                                                nm.ctypes.data, out.ctypes.data, _lib.EB_MEM_HOST), "sb")
    exp = [o.oracle_static_batch_size(recs[i:i + 1].ctypes.data, float(slot[i]), int(sm[i]), int(nm[i]))
           for i in range(n)]
    assert out.tolist() == exp


def test_stb_and_nob_vs_oracle():
    from gen_random import random_batch
    b, _ = random_batch(21, 200, k_min=0, k_max=20)
    o = oracle.load()
    n = b.n_inst
    recs = b.contexts.copy()
    recs["delta_ppl"] = np.random.default_rng(2).uniform(0, 0.6, len(recs))
    bsz = np.random.default_rng(3).integers(0, 8, n).astype(np.int64)
    st = np.zeros(n, np.int32); sel = np.zeros(b.n_req, np.uint8)
    h = _lib.handle()
    bb = InstanceBatch(b.offsets, b.columns, recs, b.ctx_index, b.k_max)
    _lib.check(h.lib.eb_stb_batch(h.ptr, recs.ctypes.data, len(recs), _ref(bb.struct()), bsz.ctypes.data, 1,
                                  st.ctypes.data, sel.ctypes.data, _lib.EB_MEM_HOST), "stb")
    c = b.columns
    for i in range(n):
        lo, hi = int(b.offsets[i]), int(b.offsets[i + 1])
        exp = np.zeros(hi - lo, np.uint8)
        if hi > lo:
            ci = int(b.ctx_index[i])
            o.oracle_stb(recs[ci:ci + 1].ctypes.data, hi - lo, c["prompt_tokens"][lo:].ctypes.data,
                         c["output_tokens"][lo:].ctypes.data, c["tolerance"][lo:].ctypes.data,
                         c["channel_gain"][lo:].ctypes.data, c["uplink_power_w"][lo:].ctypes.data, int(bsz[i]),
                         float(recs[ci]["delta_ppl"]), 1, exp.ctypes.data)
        assert np.array_equal(sel[lo:hi], exp), i
    # NoB with random busy state
    maxd = 4
    busy = np.random.default_rng(5).uniform(0, 3, (n, maxd))
    now = np.random.default_rng(6).uniform(0, 3, n)
    act = np.zeros(b.n_req, np.int8); comp = np.zeros(b.n_req); order = np.zeros(b.n_req, np.int32)
    busy_dev = busy.copy()
    _lib.check(h.lib.eb_nob_batch(h.ptr, recs.ctypes.data, len(recs), _ref(bb.struct()), now.ctypes.data, 1, None,
                                  maxd, busy_dev.ctypes.data, st.ctypes.data, act.ctypes.data, comp.ctypes.data,
                                  order.ctypes.data, _lib.EB_MEM_HOST), "nob")
    for i in range(n):
        lo, hi = int(b.offsets[i]), int(b.offsets[i + 1])
        ci = int(b.ctx_index[i])
        G = int(recs[ci]["gpu_count"])
        bu = busy[i, :G].copy()
        a2 = np.zeros(max(hi - lo, 1), np.int8); c2 = np.zeros(max(hi - lo, 1)); o2 = np.zeros(max(hi - lo, 1), np.int32)
        if hi > lo:
            o.oracle_nob(recs[ci:ci + 1].ctypes.data, hi - lo, c["prompt_tokens"][lo:].ctypes.data,
                         c["output_tokens"][lo:].ctypes.data, c["tolerance"][lo:].ctypes.data, float(now[i]),
                         float(recs[ci]["delta_ppl"]), 1, bu.ctypes.data, a2.ctypes.data, c2.ctypes.data, o2.ctypes.data)
            assert np.array_equal(act[lo:hi], a2[:hi - lo]), i
            assert np.array_equal(comp[lo:hi], c2[:hi - lo]), i
        assert np.array_equal(busy_dev[i, :G], bu), i
