"""Config 4 at its stated size (BASELINE.json configs[3]): exhaustive_optimal
(mode="subsets", dftsp.py:288-313) at K = 28, 30, 32 on the GPU, single
device and rank-sharded 8 ways, against CPU checks that share none of the
device's shortcuts:

* the adversarial family (synth.brute_family: anti-correlated uplink and
  downlink terms, some binding deadlines, no slot cap) against the oracle's
  literal multi-threaded level scan (oracle_exhaustive_mt: every combination
  of every level checked with check_direct in lexicographic order).  Levels
  above the largest z whose z smallest uplink and z smallest downlink terms
  both fit (a one-line proof computed here from the oracle's link fractions)
  are skipped by the scan; every level from there down to z* is enumerated;
* config-2-style pools (BLOOM-3B mix, K candidates): z* equals the
  reference-pinned DFTSP optimum (so z*+1 is infeasible), the oracle's level
  scan over ranks [0, r*] returns exactly r*, nodes follow the closed form
   and the mask is the r*-th combination.
"""
from math import comb

import numpy as np
import pytest

import oracle
from paper_2405_07140_b200 import brute, search, synth

pytestmark = pytest.mark.gpu


def _proof_top(rec, cols) -> int:
    up, dn = oracle.link_fractions(rec, cols)
    su, sd = np.cumsum(np.sort(up)), np.cumsum(np.sort(dn))
    ok = (su <= 1.0 + 1e-6) & (sd <= 1.0 + 1e-6)
    return int(np.nonzero(ok)[0].max()) + 1 if ok.any() else 1


@pytest.mark.parametrize("K,z0,count", [(28, 14, 8), (30, 15, 8), (32, 16, 4), (32, 12, 4)])
def test_adversarial_family_vs_literal_oracle(K, z0, count):
    fam = synth.brute_family(K, count, seed=K * 100 + z0, z0=z0)
    before = brute.enum_stats()
    for i, (rec, cols) in enumerate(fam):
        top = _proof_top(rec, cols)
        st, z, rk, checked = oracle.exhaustive_mt(rec, cols, z_top=top)
        assert st == 0
        want = (z, rk, brute.nodes_for(K, z, rk), brute.unrank(K, z, rk) if z else 0)
        one = brute.solve_sharded(rec, cols, world=1)
        assert (one.z, one.lexrank, one.nodes_visited, one.mask) == want, (K, i)
        eight = brute.solve_sharded(rec, cols, world=8)
        assert (eight.z, eight.lexrank, eight.nodes_visited, eight.mask) == want, (K, i)
        # adversarial: >= 3 levels above z* survive the device's level bounds
        live = brute.device_level_range(rec, cols).live_mask
        assert bin(live >> z).count("1") >= 3, (K, i, z, bin(live))
        if K == 32 and z0 == 16:
            assert checked >= 1e9, checked          # the literal scan enumerated >= 1e9 subsets
    after = brute.enum_stats()
    assert after[0] > before[0]                     # the device counted its checked combinations


@pytest.mark.parametrize("K", [28, 30, 32])
def test_config2_style_pools_large_k(K):
    w = synth.Workload("config4 config-2-style", K=K)
    b = synth.generate(w, 8, seed=4000 + K)
    d = search.solve_batch(b, ladder=(128, 256, 512))
    assert (d.status == 0).all()
    for i in range(b.n_inst):
        lo, hi = int(b.offsets[i]), int(b.offsets[i + 1])
        ci = int(b.ctx_index[i])
        rec = b.contexts[ci:ci + 1]
        cols = {k: np.ascontiguousarray(v[lo:hi]) for k, v in b.columns.items()}
        got = brute.solve_sharded(rec, cols, world=1)
        assert got.z == int(d.z_found[i]), (K, i)           # DFTSP optimum (reference-pinned)
        assert got.z >= 1
        level = oracle.level_evaluator(rec, cols)
        assert level(got.z, 0, got.lexrank + 1) == got.lexrank, (K, i)   # r* feasible, no lower rank is
        assert got.nodes_visited == sum(comb(K, q) for q in range(got.z + 1, K + 1)) + got.lexrank + 1
        assert got.mask == brute.unrank(K, got.z, got.lexrank)
        eight = brute.solve_sharded(rec, cols, world=8)
        assert (eight.z, eight.lexrank, eight.nodes_visited, eight.mask) == \
            (got.z, got.lexrank, got.nodes_visited, got.mask)
