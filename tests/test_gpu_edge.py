"""Edge inputs the reference accepts (feasibility.py:46-56, radio.py:52-57
reject only nonpositive / negative values), pinned by fixtures generated from
the reference itself (tests/golden/make_edge_golden.py -> edge.npz):

  kind 0  +inf deadlines / waiting times / gains: dftsp reproduced exactly,
          including the reference's RuntimeError (status EB_ERR_REVERIFY)
          where its reduced form and check_direct disagree on infinities;
  kind 1  NaN deadlines / waiting times / gains: the reference then orders the
          pool by CPython's sort on unordered keys; the device returns the
          documented EB_ERR_NAN_INPUT for exactly the pools holding a NaN
          (error_index = the first one), the oracle the same;
  kind 2  duplicate ids: coefficients are keyed by id (feasibility.py:164-166,
          the last duplicate's k_up/k_down win); the device returns the
          documented EB_ERR_DUPLICATE_ID for exactly those pools.
exhaustive_optimal (subsets) has no sort and no id lookup: every kind is
reproduced exactly (NaN members can never be scheduled; the level bounds
treat them as unschedulable)."""
import numpy as np
import pytest

import oracle
from helpers import FLAGS, expected, got, groups, load_corpus, sub_batch
from paper_2405_07140_b200 import _lib, search

pytestmark = pytest.mark.gpu


def _has(d, i, what):
    lo, hi = int(d["offsets"][i]), int(d["offsets"][i + 1])
    if what == "nan":
        return any(np.isnan(d["req_" + k][lo:hi]).any() for k in ("deadline_s", "waiting_s", "channel_gain",
                                                                  "uplink_power_w"))
    ids = d["req_id"][lo:hi]
    return len(set(ids.tolist())) != len(ids)


@pytest.mark.parametrize("tag", ["P", "PE"])
@pytest.mark.parametrize("algo", [1, 2])
def test_dftsp_edge_inputs_vs_reference(tag, algo):
    d = load_corpus("edge")
    kinds = d["kind"]
    n_exact = n_status = 0
    for ladder, idx in groups(d).items():
        b = sub_batch(d, idx)
        res = search.solve_batch(b, ladder=ladder, algorithm=algo, **FLAGS[tag])
        orc = oracle.dftsp_batch(b, ladder=ladder, **FLAGS[tag])
        for j, i in enumerate(idx):
            g = got(res, b, j)
            if kinds[i] == 1 and _has(d, i, "nan"):
                assert g["status"] == _lib.ERR_NAN_INPUT, i
                lo, hi = int(d["offsets"][i]), int(d["offsets"][i + 1])
                first = min(k for k in range(hi - lo) if any(np.isnan(d["req_" + c][lo + k]) for c in
                                                          ("deadline_s", "waiting_s", "channel_gain",
                                                           "uplink_power_w")))
                assert int(res.error_index[j]) == first and int(orc["error_index"][j]) == first
                assert int(orc["status"][j]) == _lib.ERR_NAN_INPUT
                n_status += 1
            elif kinds[i] == 2 and _has(d, i, "dup"):
                assert g["status"] == _lib.ERR_DUPLICATE_ID, i
                n_status += 1
            else:
                e = expected(d, tag, i)
                if e["status"] != 0:
                    assert g["status"] == e["status"], (i, e, g)
                else:
                    assert g == e, (i, e, g)
                n_exact += 1
    assert n_exact >= 80 and n_status >= 60


def test_exhaustive_edge_inputs_vs_reference():
    import ctypes
    d = load_corpus("edge")
    n = len(d["offsets"]) - 1
    b = sub_batch(d, list(range(n)))
    st, z = np.zeros(n, np.int32), np.zeros(n, np.int32)
    rk, nodes, mask = np.zeros(n, np.int64), np.zeros(n, np.int64), np.zeros(n, np.uint64)
    h = _lib.handle()
    bs = b.struct()
    _lib.check(h.lib.eb_exhaustive_batch(h.ptr, b.contexts.ctypes.data, len(b.contexts),
                                         ctypes.cast(ctypes.pointer(bs), ctypes.c_void_p), 16, st.ctypes.data,
                                         z.ctypes.data, rk.ctypes.data, nodes.ctypes.data, mask.ctypes.data,
                                         _lib.EB_MEM_HOST), "eb_exhaustive_batch")
    assert np.array_equal(st, d["ex_status"])
    ok = d["ex_status"] == 0
    assert np.array_equal(z[ok], d["ex_z"][ok])
    assert np.array_equal(nodes[ok], d["ex_nodes"][ok])
    assert np.array_equal(mask[ok], d["ex_mask"][ok])
