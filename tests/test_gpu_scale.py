"""Parity at scale: the device against the CPU oracle on the benchmark
workloads themselves (exact equality of every output field: status, z,
counts, class lengths, nodes_visited, nodes_pruned, solution ids, metrics)."""
import numpy as np
import pytest

import oracle
from paper_2405_07140_b200 import search, synth
from paper_2405_07140_b200.soa import InstanceBatch

pytestmark = pytest.mark.gpu

FIELDS = ("status", "z_found", "nodes_visited", "nodes_pruned", "n_classes", "counts", "class_lengths", "metrics")


def _check(b, ladder, n_check=None, **flags):
    dev = search.solve_batch(b, ladder=ladder, **flags)
    orc = oracle.dftsp_batch(b, ladder=ladder, threads=16, **flags)
    for k in FIELDS:
        a, o = getattr(dev, k), orc[k]
        bad = np.nonzero((a != o).reshape(len(a), -1).any(axis=1))[0]
        assert bad.size == 0, f"{k} differs at {bad[:5]}: gpu={a[bad[0]]} oracle={o[bad[0]]}"
    ok = dev.z_found > 0
    rows = np.concatenate([np.arange(b.offsets[i], b.offsets[i] + dev.z_found[i]) for i in np.nonzero(ok)[0]])
    assert np.array_equal(dev.solution[rows], orc["solution"][rows])
    return dev


def test_config2_200k_instances():
    b = synth.generate(synth.CONFIG2, 200_000, seed=11)
    dev = _check(b, (128, 256, 512))
    assert dev.z_found.mean() > 4


@pytest.mark.parametrize("flags", [dict(pruning=False), dict(inclusive_bound=True), dict(exact_tau=True)])
def test_config2_flag_modes_20k(flags):
    b = synth.generate(synth.CONFIG2, 20_000, seed=12)
    _check(b, (128, 256, 512), **flags)


def test_config5_50k_instances():
    b = synth.generate(synth.CONFIG5, 50_000, seed=13)
    _check(b, synth.CONFIG5.outputs)


@pytest.mark.parametrize("K", [10, 25, 32, 40, 48])
def test_k_sweep(K):
    w = synth.Workload(f"K={K}", profiles=("w8a16",), K=K)
    b = synth.generate(w, 2000 if K <= 32 else 300, seed=14 + K)
    _check(b, (128, 256, 512))


def test_no_ladder_and_v1_agree_on_config2():
    b = synth.generate(synth.CONFIG2, 20_000, seed=15)
    d2 = search.solve_batch(b, ladder=None)
    d1 = search.solve_batch(b, ladder=None, algorithm=1)
    for k in FIELDS:
        assert np.array_equal(getattr(d1, k), getattr(d2, k)), k
