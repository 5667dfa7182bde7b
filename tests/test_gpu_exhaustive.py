"""K4 brute-force subset search on the GPU: reference goldens, oracle parity,
the node-count closed form, and the rank-range sharding used across GPUs."""
from math import comb

import numpy as np
import pytest

import oracle
from gen_random import random_batch
from helpers import load_corpus
from paper_2405_07140_b200 import _lib, search
from paper_2405_07140_b200.soa import InstanceBatch

pytestmark = pytest.mark.gpu


def _ref(s):
    import ctypes
    return ctypes.cast(ctypes.pointer(s), ctypes.c_void_p)


def _run(b, cap=64):
    n = b.n_inst
    st = np.zeros(n, np.int32); z = np.zeros(n, np.int32); rk = np.zeros(n, np.int64)
    nodes = np.zeros(n, np.int64); mask = np.zeros(n, np.uint64)
    h = _lib.handle()
    _lib.check(h.lib.eb_exhaustive_batch(h.ptr, b.contexts.ctypes.data, len(b.contexts), _ref(b.struct()), cap,
                                         st.ctypes.data, z.ctypes.data, rk.ctypes.data, nodes.ctypes.data,
                                         mask.ctypes.data, _lib.EB_MEM_HOST), "exh")
    return st, z, rk, nodes, mask


@pytest.mark.parametrize("name", ("random_2024", "random_31", "random_1001", "random_77", "scenario"))
def test_exhaustive_matches_reference(name):
    d = load_corpus(name)
    b = InstanceBatch(d["offsets"], {k[4:]: np.ascontiguousarray(v) for k, v in d.items() if k.startswith("req_")},
                      np.ascontiguousarray(d["ctx"]), np.ascontiguousarray(d["ctx_index"]),
                      int(np.diff(d["offsets"]).max()))
    st, z, rk, nodes, mask = _run(b, cap=16)
    okr = d["ex_status"] == 0
    assert np.array_equal(z[okr], d["ex_z"][okr])
    assert np.array_equal(nodes[okr], d["ex_nodes"][okr])
    assert np.array_equal(mask[okr], d["ex_mask"][okr])


def test_exhaustive_vs_oracle_up_to_k18():
    b, _ = random_batch(8, 60, k_min=12, k_max=18)
    st, z, rk, nodes, mask = _run(b)
    for i in range(b.n_inst):
        ci = int(b.ctx_index[i])
        e = oracle.exhaustive(b.contexts[ci:ci + 1], b.columns, int(b.offsets[i]), int(b.offsets[i + 1]))
        assert (int(st[i]), int(z[i]), int(rk[i]), int(nodes[i]), int(mask[i])) == e, i
        n = int(b.offsets[i + 1] - b.offsets[i])
        if z[i]:
            assert nodes[i] == sum(comb(n, q) for q in range(int(z[i]) + 1, n + 1)) + rk[i] + 1


def test_rank_range_sharding_reassembles_the_answer():
    """Splitting each level's ranks into shards (one per GPU) and taking the
    max (z, -rank) key reproduces the single-device answer."""
    from paper_2405_07140_b200.brute import solve_sharded
    b, _ = random_batch(9, 8, k_min=16, k_max=20)
    st, z, rk, nodes, mask = _run(b)
    for i in range(b.n_inst):
        ci = int(b.ctx_index[i])
        lo, hi = int(b.offsets[i]), int(b.offsets[i + 1])
        cols = {k: np.ascontiguousarray(v[lo:hi]) for k, v in b.columns.items()}
        for world in (2, 3, 8):
            got = solve_sharded(b.contexts[ci:ci + 1], cols, world=world)
            assert (got.z, got.lexrank, got.nodes_visited) == (int(z[i]), int(rk[i]), int(nodes[i])), (i, world)


@pytest.mark.parametrize("seed", [21, 22, 23, 24])
def test_branch_and_bound_matches_oracle_many(seed):
    """The prefix bounds of scan_chunk skip only infeasible rank ranges: the
    first feasible rank (and so z, rank, nodes, mask) equals the oracle's plain
    enumeration on many small/medium pools, including tight slot caps."""
    b, _ = random_batch(seed, 250, k_min=1, k_max=15, slot_cap_frac=0.6)
    st, z, rk, nodes, mask = _run(b)
    for i in range(b.n_inst):
        ci = int(b.ctx_index[i])
        e = oracle.exhaustive(b.contexts[ci:ci + 1], b.columns, int(b.offsets[i]), int(b.offsets[i + 1]))
        assert (int(st[i]), int(z[i]), int(rk[i]), int(nodes[i]), int(mask[i])) == e, (seed, i)


@pytest.mark.parametrize("seed", [31, 32])
def test_branch_and_bound_raw_negative_waits(seed):
    """Raw arrays may carry what Request's validation refuses (negative
    waiting_s, feasibility.py:55-56): the division-free deadline refutations
    of scan_chunk apply only where ws >= 0, and the answers still equal the
    oracle's plain enumeration (slot caps and tight deadlines included)."""
    b, _ = random_batch(seed, 200, k_min=1, k_max=14, slot_cap_frac=0.6)
    rng = np.random.default_rng(seed)
    w = b.columns["waiting_s"]
    neg = rng.random(w.shape[0]) < 0.3
    w[neg] = -rng.uniform(0.0, 2.0, int(neg.sum())) * b.columns["deadline_s"][neg]
    st, z, rk, nodes, mask = _run(b)
    for i in range(b.n_inst):
        ci = int(b.ctx_index[i])
        e = oracle.exhaustive(b.contexts[ci:ci + 1], b.columns, int(b.offsets[i]), int(b.offsets[i + 1]))
        assert (int(st[i]), int(z[i]), int(rk[i]), int(nodes[i]), int(mask[i])) == e, (seed, i)


def test_branch_and_bound_config2_pools():
    """Config-2 pools (K=20, BLOOM-3B mix): batch kernel and 5-way rank sharding
    against the oracle's enumeration."""
    from paper_2405_07140_b200 import synth
    from paper_2405_07140_b200.brute import solve_sharded
    b = synth.generate(synth.CONFIG2, 12, seed=77)
    st, z, rk, nodes, mask = _run(b)
    for i in range(b.n_inst):
        ci = int(b.ctx_index[i])
        lo, hi = int(b.offsets[i]), int(b.offsets[i + 1])
        e = oracle.exhaustive(b.contexts[ci:ci + 1], b.columns, lo, hi)
        assert (int(st[i]), int(z[i]), int(rk[i]), int(nodes[i]), int(mask[i])) == e, i
        cols = {k: np.ascontiguousarray(v[lo:hi]) for k, v in b.columns.items()}
        got = solve_sharded(b.contexts[ci:ci + 1], cols, world=5)
        assert (got.z, got.lexrank, got.nodes_visited) == (int(z[i]), int(rk[i]), int(nodes[i])), i


@pytest.mark.parametrize("seed", [31, 32])
def test_live_levels_are_sound(seed):
    """eb_exhaustive_live_levels never refutes a feasible level: every level
    z <= z* (subsets of a feasible set are feasible) stays live."""
    from paper_2405_07140_b200.brute import device_level_range
    b, _ = random_batch(seed, 120, k_min=4, k_max=16, slot_cap_frac=0.6)
    for i in range(b.n_inst):
        ci = int(b.ctx_index[i])
        lo, hi = int(b.offsets[i]), int(b.offsets[i + 1])
        st, z, rk, nodes, mask = oracle.exhaustive(b.contexts[ci:ci + 1], b.columns, lo, hi)
        if st != 0:
            continue
        cols = {k: np.ascontiguousarray(v[lo:hi]) for k, v in b.columns.items()}
        live = device_level_range(b.contexts[ci:ci + 1], cols).live_mask
        assert live & ((1 << z) - 1) == (1 << z) - 1, (i, z, bin(live))
