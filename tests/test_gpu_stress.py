"""Randomised parity at volume: every search path (count tables, streamed
three-level counts, unranking tables and count rows for four or more levels,
two requests per lane, the wide pass) against the oracle on fresh seeded
corpora, for all four flag sets.  Bit-exact on every field."""
import numpy as np
import pytest

import oracle
from gen_random import group_by_ladder, random_batch
from helpers import FLAGS
from paper_2405_07140_b200 import search

pytestmark = pytest.mark.gpu

KEYS = ("status", "error_index", "z_found", "nodes_visited", "nodes_pruned", "n_classes", "counts", "class_lengths")


def _same(dev, orc, batch, what):
    for k in KEYS:
        a, b = getattr(dev, k), orc[k]
        if not np.array_equal(a, b):
            i = int(np.nonzero((a != b).reshape(len(a), -1).any(axis=1))[0][0])
            raise AssertionError(f"{what}: {k} differs at instance {i}: gpu={a[i]} oracle={b[i]}")
    ok = dev.status == 0
    z = dev.z_found
    for i in np.nonzero(ok & (z > 0))[0]:
        lo = int(batch.offsets[i])
        assert np.array_equal(dev.solution[lo:lo + z[i]], orc["solution"][lo:lo + z[i]]), f"{what}: solution {i}"
    assert np.array_equal(dev.metrics[ok], orc["metrics"][ok]), f"{what}: metrics"


@pytest.mark.parametrize("tag", ["P", "NP", "PI", "PE"])
@pytest.mark.parametrize("shape", [(1, 32, 3, 24000), (33, 64, 3, 4800), (4, 24, 5, 6000), (20, 64, 5, 1500), (65, 120, 3, 600)])
def test_stress_against_oracle(tag, shape):
    k_min, k_max, max_classes, n = shape
    seed = 7000 + 97 * k_min + 13 * max_classes + sum(map(ord, tag))
    batch, ladders = random_batch(seed, n, k_min=k_min, k_max=k_max, max_classes=max_classes)
    compared = 0
    for lad, (_, sb) in group_by_ladder(batch, ladders).items():
        dev = search.solve_batch(sb, ladder=lad, **FLAGS[tag])
        orc = oracle.dftsp_batch(sb, ladder=lad, threads=16, **FLAGS[tag])
        _same(dev, orc, sb, f"{tag} K={k_min}..{k_max} classes<={max_classes} ladder {lad}")
        compared += sb.n_inst
    assert compared == n
