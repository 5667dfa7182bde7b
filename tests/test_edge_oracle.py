"""The C oracle on the reference's edge-input fixtures (no GPU): +inf inputs
reproduced exactly, NaN pools -> EB_ERR_NAN_INPUT, duplicate-id pools ->
EB_ERR_DUPLICATE_ID (tests/golden/make_edge_golden.py)."""
import numpy as np
import pytest

import oracle
from helpers import FLAGS, expected, got, groups, load_corpus, sub_batch
from paper_2405_07140_b200 import _lib


@pytest.mark.parametrize("tag", ["P", "PE"])
def test_oracle_edge_inputs(tag):
    d = load_corpus("edge")
    kinds = d["kind"]
    for ladder, idx in groups(d).items():
        b = sub_batch(d, idx)
        orc = oracle.dftsp_batch(b, ladder=ladder, **FLAGS[tag])
        for j, i in enumerate(idx):
            g = got(orc, b, j)
            lo, hi = int(d["offsets"][i]), int(d["offsets"][i + 1])
            nan = any(np.isnan(d["req_" + k][lo:hi]).any() for k in ("deadline_s", "waiting_s", "channel_gain",
                                                                      "uplink_power_w"))
            dup = len(set(d["req_id"][lo:hi].tolist())) != hi - lo
            if nan:
                assert g["status"] == _lib.ERR_NAN_INPUT
            elif dup:
                assert g["status"] == _lib.ERR_DUPLICATE_ID
            else:
                e = expected(d, tag, i)
                assert (g["status"] == e["status"]) if e["status"] else (g == e), (i, e, g)


def test_oracle_exhaustive_edge_inputs():
    d = load_corpus("edge")
    for i in range(len(d["offsets"]) - 1):
        b = sub_batch(d, [i])
        st, z, rk, nodes, mask = oracle.exhaustive(b.contexts[int(b.ctx_index[0]):int(b.ctx_index[0]) + 1],
                                                   b.columns, 0, int(b.offsets[1]), cap=16)
        assert st == d["ex_status"][i]
        if st == 0:
            assert (z, nodes, mask) == (d["ex_z"][i], d["ex_nodes"][i], d["ex_mask"][i]), i
