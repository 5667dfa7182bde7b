"""K1 admission (sim._dftsp_candidates, sim.py:264-274: accuracy filter
catalog.py:146-155 via feasibility.py:128-130, then the alone-feasible
check_direct prefilter) on the GPU against the CPU oracle at volume, and the
benchmark workload rebuilt with either admission (the reference arm's claim
that it times the very instances the GPU solves)."""
import numpy as np
import pytest

import oracle
from paper_2405_07140_b200 import _lib, synth
from paper_2405_07140_b200.soa import InstanceBatch

pytestmark = pytest.mark.gpu


def _rows(seed, n_inst, k, w=synth.CONFIG2, edge=False):
    rng = np.random.default_rng(seed)
    cols = synth._draw(rng, n_inst * k, w)
    nr = n_inst * k
    cols["uplink_power_w"] = np.full(nr, synth.dbm(20.0))
    cols["id"] = np.tile(np.arange(k, dtype=np.int64), n_inst)
    if edge:
        # the reference's raising / degenerate inputs: negative tolerance
        # (accuracy_admissible raises), nonpositive gain or power
        # (spectral_efficiency raises), tiny gains (efficiency rounds to 0),
        # infinite deadline / waiting, exact-boundary tolerances
        m = rng.random(nr)
        cols["tolerance"][m < 0.02] = -0.5
        cols["channel_gain"][(m >= 0.02) & (m < 0.04)] = 0.0
        cols["channel_gain"][(m >= 0.04) & (m < 0.05)] = -1e-3
        cols["uplink_power_w"][(m >= 0.05) & (m < 0.06)] = 0.0
        cols["channel_gain"][(m >= 0.06) & (m < 0.08)] = 1e-30
        cols["deadline_s"][(m >= 0.08) & (m < 0.09)] = np.inf
        cols["waiting_s"][(m >= 0.09) & (m < 0.10)] = np.inf
        recs = synth.contexts(w)
        cols["tolerance"][(m >= 0.10) & (m < 0.13)] = recs["delta_ppl"][rng.integers(0, len(recs), 1)[0]]
    prof = rng.integers(0, len(w.profiles), n_inst).astype(np.int32)
    off = np.arange(n_inst + 1, dtype=np.int64) * k
    return InstanceBatch(off, {kk: np.ascontiguousarray(v) for kk, v in cols.items()}, synth.contexts(w), prof, k)


@pytest.mark.parametrize("edge", [False, True])
def test_admission_kernel_matches_oracle_at_volume(edge):
    b = _rows(11 + edge, 200_000, 20, edge=edge)
    dev = synth.device_admission()(b, b.contexts)
    ora = oracle.admission_batch(b)
    assert np.array_equal(dev[0], ora[0]), np.unique(dev[0][dev[0] != ora[0]])
    assert np.array_equal(dev[1], ora[1])
    kept = ora[1].mean()
    assert 0.05 < kept < 0.95
    if edge:
        assert set(np.unique(ora[0])) >= {0, _lib.ERR_INVALID_ARG, _lib.ERR_NONPOSITIVE_LINK,
                                          _lib.ERR_UPLINK_EFF_ZERO}


def test_admission_config5_matches_oracle():
    b = _rows(5, 100_000, 20, w=synth.CONFIG5)
    dev = synth.device_admission()(b, b.contexts)
    ora = oracle.admission_batch(b)
    assert np.array_equal(dev[0], ora[0]) and np.array_equal(dev[1], ora[1])


def test_bench_workload_identical_under_cpu_admission():
    """10^6 config-2 instances: device-admitted == oracle-admitted, column for column."""
    a = synth.generate(synth.CONFIG2, 1_000_000, seed=2405_07140)
    c = synth.generate(synth.CONFIG2, 1_000_000, seed=2405_07140, admit=oracle.admit)
    assert np.array_equal(a.offsets, c.offsets) and np.array_equal(a.ctx_index, c.ctx_index)
    for k in a.columns:
        assert np.array_equal(a.columns[k], c.columns[k]), k
