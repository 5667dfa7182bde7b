"""K3 (instance-parallel DFTSP) parity on the GPU: bit-exact solution ids,
counts, z, nodes_visited and nodes_pruned against (a) golden fixtures from the
reference itself and (b) the C oracle on fresh seeded corpora."""
import os

import numpy as np
import pytest

import oracle
from gen_random import group_by_ladder, random_batch
from helpers import ALL_CORPORA, FLAGS, compare_corpus, corpus_path, groups, load_corpus, sub_batch
from paper_2405_07140_b200 import _lib, search

pytestmark = pytest.mark.gpu

RES_KEYS = ("status", "z_found", "nodes_visited", "nodes_pruned", "n_classes", "counts", "class_lengths")


@pytest.mark.parametrize("algo", [1, 2])
@pytest.mark.parametrize("name", ALL_CORPORA)
def test_gpu_matches_reference_goldens(name, algo):
    if not os.path.exists(corpus_path(name)):
        pytest.skip("corpus missing")
    d = load_corpus(name)
    tags = [t for t in FLAGS if f"{t}_z" in d]

    def _gpu_solve(batch, ladder=None, **flags):
        return search.solve_batch(batch, ladder=ladder, algorithm=algo, **flags)

    for tag in tags:
        bad = compare_corpus(d, tag, _gpu_solve, use_ladder=(tag != "NL"))
        assert not bad, f"{name}/{tag}: {bad[:3]}"


def _assert_same(dev, orc, batch, what):
    for k in RES_KEYS:
        a, b = getattr(dev, k), orc[k]
        if not np.array_equal(a, b):
            i = int(np.nonzero((a != b).reshape(len(a), -1).any(axis=1))[0][0])
            raise AssertionError(f"{what}: {k} differs at instance {i}: gpu={a[i]} oracle={b[i]}")
    ok = dev.status == 0
    for i in np.nonzero(ok)[0]:
        lo = int(batch.offsets[i])
        z = int(dev.z_found[i])
        assert np.array_equal(dev.solution[lo:lo + z], orc["solution"][lo:lo + z]), f"{what}: solution {i}"
        assert np.array_equal(dev.metrics[i], orc["metrics"][i]), f"{what}: metrics {i}"


@pytest.mark.parametrize("algo", [1, 2])
@pytest.mark.parametrize("seed", [11, 12, 13])
@pytest.mark.parametrize("tag", ["P", "NP", "PI", "PE"])
def test_gpu_matches_oracle_fresh_corpora(seed, tag, algo):
    batch, ladders = random_batch(1000 * seed + sum(map(ord, tag)), 600)
    for lad, (idx, sb) in group_by_ladder(batch, ladders).items():
        dev = search.solve_batch(sb, ladder=lad, algorithm=algo, **FLAGS[tag])
        orc = oracle.dftsp_batch(sb, ladder=lad, threads=8, **FLAGS[tag])
        _assert_same(dev, orc, sb, f"seed {seed} {tag} ladder {lad}")


def test_gpu_matches_oracle_no_ladder_many_classes():
    batch, _ = random_batch(77, 400, k_max=20, max_classes=5)
    for algo in (1, 2):
        dev = search.solve_batch(batch, ladder=None, algorithm=algo)
        orc = oracle.dftsp_batch(batch, ladder=None, threads=8)
        _assert_same(dev, orc, batch, f"no ladder, <=5 classes, algo {algo}")


@pytest.mark.parametrize("algo", [1, 2])
@pytest.mark.parametrize("tag", ["P", "NP", "PI"])
def test_gpu_large_k_and_trajectory(algo, tag):
    batch, ladders = random_batch(5, 120, k_min=30, k_max=48, max_classes=4)
    for lad, (idx, sb) in group_by_ladder(batch, ladders).items():
        dev = search.solve_batch(sb, ladder=lad, collect_trajectory=True, algorithm=algo, **FLAGS[tag])
        orc = oracle.dftsp_batch(sb, ladder=lad, collect_trajectory=True, threads=8, **FLAGS[tag])
        _assert_same(dev, orc, sb, f"K 30-48 ladder {lad} {tag} algo {algo}")
        assert np.array_equal(dev.traj_len, orc["traj_len"])
        for j in range(sb.n_inst):
            t0 = int(dev.traj_offsets[j])
            n = int(dev.traj_len[j])
            assert np.array_equal(dev.traj[t0:t0 + n], orc["traj"][t0:t0 + n]), j


@pytest.mark.parametrize("algo", [1, 2])
def test_gpu_trajectory_matches_reference(algo):
    d = load_corpus("random_34")
    lens = d["P_traj_len"]
    starts = np.concatenate([[0], np.cumsum(lens)])
    for ladder, ids in groups(d).items():
        b = sub_batch(d, ids)
        res = search.solve_batch(b, ladder=ladder, collect_trajectory=True, algorithm=algo)
        for j, i in enumerate(ids):
            t0 = int(res.traj_offsets[j])
            got = res.traj[t0:t0 + int(res.traj_len[j])]
            assert np.array_equal(got, d["P_traj"][starts[i]:starts[i + 1]]), i


def test_gpu_k64_and_sixteen_classes():
    """Device limits: 64 candidates over 16 output classes (no ladder).  A
    roomy node makes the top levels feasible so the search (and the oracle)
    terminates; the partition/table machinery still runs at full width."""
    batch, _ = random_batch(99, 6, k_min=64, k_max=64, max_classes=5)
    rng = np.random.default_rng(1)
    batch.columns["output_tokens"][:] = rng.choice(np.arange(1, 17) * 8, size=batch.n_req)
    batch.columns["deadline_s"][:] = 1e6
    batch.columns["channel_gain"][:] = 1.0
    for c in batch.contexts:
        c["memory_bytes"] *= 1e6
        c["flops_per_s"] *= 1e6
        c["uplink_band_hz"] = c["downlink_band_hz"] = 1e9
        c["has_slot_cap"] = 0
    dev = search.solve_batch(batch, ladder=None)
    orc = oracle.dftsp_batch(batch, ladder=None, threads=6)
    _assert_same(dev, orc, batch, "K=64, 16 classes")
    assert (dev.z_found > 40).all()


def test_gpu_k64_three_classes_deep_search():
    """K = 64 with three classes: thousands of dfs calls per instance."""
    batch, ladders = random_batch(98, 8, k_min=60, k_max=64, max_classes=3)
    for lad, (idx, sb) in group_by_ladder(batch, ladders).items():
        for algo in (1, 2):
            dev = search.solve_batch(sb, ladder=lad, algorithm=algo)
            orc = oracle.dftsp_batch(sb, ladder=lad, threads=8)
            _assert_same(dev, orc, sb, f"K=64 ladder {lad} algo {algo}")


def test_gpu_edge_statuses():
    """Empty pools, duplicate ids, off-ladder, weights-do-not-fit: same status
    and offending index as the oracle."""
    batch, ladders = random_batch(3, 64, k_min=0, k_max=6)
    b = batch
    # duplicate ids in instance 5, off-ladder output in instance 7, tiny memory in instance 9
    lo5 = int(b.offsets[5])
    if b.offsets[6] - lo5 >= 2:
        b.columns["id"][lo5 + 1] = b.columns["id"][lo5]
    lo7 = int(b.offsets[7])
    if b.offsets[8] > lo7:
        b.columns["output_tokens"][lo7] = 999
    b.contexts[9]["memory_bytes"] = 1.0
    lad = (16, 32, 64, 128, 256)
    dev = search.solve_batch(b, ladder=lad)
    orc = oracle.dftsp_batch(b, ladder=lad)
    assert np.array_equal(dev.status, orc["status"])
    assert np.array_equal(dev.error_index, orc["error_index"])
    _assert_same(dev, orc, b, "edge statuses")


def test_gpu_duplicate_ids_wide_instances():
    """Instances of 33..64 requests (two per lane): duplicates inside the first
    32, inside the rest, and across the two slices all report the oracle's
    status and offending index (the smallest index with an earlier twin)."""
    batch, ladders = random_batch(41, 40, k_min=40, k_max=64)
    b = batch
    ids = b.columns["id"]
    for inst, (a, c) in {0: (3, 9), 1: (35, 50), 2: (4, 37), 3: (31, 32), 4: (0, 63), 5: (33, 34)}.items():
        lo, hi = int(b.offsets[inst]), int(b.offsets[inst + 1])
        if lo + c < hi:
            ids[lo + c] = ids[lo + a]
    lad = None
    dev = search.solve_batch(b, ladder=lad)
    orc = oracle.dftsp_batch(b, ladder=lad)
    assert np.array_equal(dev.status, orc["status"])
    assert np.array_equal(dev.error_index, orc["error_index"])
    assert (dev.status == _lib.ERR_DUPLICATE_ID).sum() >= 4
    _assert_same(dev, orc, b, "wide duplicates")


def test_gpu_v2_table_overflow_falls_back_exactly():
    """Many classes with many members: u32 leaf counts overflow, the instance
    is re-run by the literal walk and still matches the oracle."""
    batch, _ = random_batch(97, 4, k_min=56, k_max=56, max_classes=5)
    rng = np.random.default_rng(2)
    batch.columns["output_tokens"][:] = rng.choice(np.arange(1, 15) * 8, size=batch.n_req)
    batch.columns["deadline_s"][:] = 1e6
    batch.columns["channel_gain"][:] = 1.0
    for c in batch.contexts:
        c["memory_bytes"] *= 1e6
        c["flops_per_s"] *= 1e6
        c["uplink_band_hz"] = c["downlink_band_hz"] = 1e9
        c["has_slot_cap"] = 0
    dev = search.solve_batch(batch, ladder=None, algorithm=2)
    orc = oracle.dftsp_batch(batch, ladder=None, threads=4)
    _assert_same(dev, orc, batch, "overflow fallback")


@pytest.mark.parametrize("name", ["random_2024", "random_77"])
def test_gpu_exhaustive_counts_mode_matches_reference(name):
    d = load_corpus(name)
    for ladder, ids in groups(d).items():
        b = sub_batch(d, ids)
        res = search.solve_batch(b, ladder=ladder, exhaustive_counts=True)
        for j, i in enumerate(ids):
            assert int(res.status[j]) == int(d["exc_status"][i]), (i, res.status[j])
            if res.status[j] == 0:
                lo = int(b.offsets[j])
                z = int(res.z_found[j])
                assert z == int(d["exc_z"][i]) and int(res.nodes_visited[j]) == int(d["exc_nodes"][i]), i
                lo_d = int(d["offsets"][i])
                assert tuple(res.solution[lo:lo + z]) == tuple(d["exc_solution"][lo_d:lo_d + z]), i


def test_gpu_exhaustive_counts_mode_vs_oracle_fresh():
    batch, ladders = random_batch(123, 300, k_max=12)
    for lad, (idx, sb) in group_by_ladder(batch, ladders).items():
        res = search.solve_batch(sb, ladder=lad, exhaustive_counts=True)
        for j in range(sb.n_inst):
            ci = int(sb.ctx_index[j])
            st, z, nodes, sol = oracle.exhaustive_counts(sb.contexts[ci:ci + 1], sb.columns, int(sb.offsets[j]),
                                                         int(sb.offsets[j + 1]), ladder=lad)
            assert int(res.status[j]) == st, j
            if st == 0:
                lo = int(sb.offsets[j])
                assert (int(res.z_found[j]), int(res.nodes_visited[j])) == (z, nodes), j
                assert tuple(int(x) for x in res.solution[lo:lo + z]) == sol, j


@pytest.mark.parametrize("tag", ["P", "NP", "PE", "PI", "NL"])
def test_gpu_wide_instances_mixed_with_narrow(tag):
    """Instances of 1..160 candidates in one call: the narrow ones take the
    main pass, those over 64 the wide pass; every field equals the oracle."""
    batch, ladders = random_batch(61, 90, k_min=1, k_max=160, max_classes=3)
    assert (np.diff(batch.offsets) > 64).sum() >= 20
    if tag == "NL":
        parts = {None: (None, batch)}
    else:
        parts = group_by_ladder(batch, ladders)
    for lad, (_, sb) in parts.items():
        flags = {} if tag == "NL" else FLAGS[tag]
        dev = search.solve_batch(sb, ladder=lad, **flags)
        orc = oracle.dftsp_batch(sb, ladder=lad, threads=16, **flags)
        _assert_same(dev, orc, sb, f"mixed wide/narrow {tag} ladder {lad}")


@pytest.mark.parametrize("tag", ["P", "NP"])
def test_gpu_widest_instances(tag):
    """Pools of 200..255 candidates (three classes): the leaf-parallel wide
    pass, with count rows past the table range, equals the oracle."""
    batch, ladders = random_batch(67, 12, k_min=200, k_max=255, max_classes=3)
    for lad, (_, sb) in group_by_ladder(batch, ladders).items():
        dev = search.solve_batch(sb, ladder=lad, **FLAGS[tag])
        orc = oracle.dftsp_batch(sb, ladder=lad, threads=16, **FLAGS[tag])
        _assert_same(dev, orc, sb, f"widest {tag} ladder {lad}")


def test_gpu_over_wide_limit_is_k_too_large():
    batch, _ = random_batch(63, 2, k_min=256, k_max=256, max_classes=3)
    dev = search.solve_batch(batch, ladder=None)
    assert (dev.status == _lib.ERR_K_TOO_LARGE).all()


@pytest.mark.parametrize("uniform", [True, False])
def test_gpu_wire_format_matches_wide_call(uniform):
    """eb_dftsp_batch_packed returns exactly what eb_dftsp_batch returns (and
    what the oracle returns) on the same instances."""
    from paper_2405_07140_b200.soa import pack_wire
    batch, ladders = random_batch(4242 + uniform, 3000, k_max=20)
    if not uniform:
        rng = np.random.default_rng(9)
        batch.columns["uplink_power_w"] = batch.columns["uplink_power_w"] * rng.uniform(0.5, 2.0, batch.n_req)
    for lad, (idx, sb) in group_by_ladder(batch, ladders).items():
        w = pack_wire(sb)
        assert w is not None and w.uniform_power == uniform
        dev = search.solve_batch(sb, ladder=lad)
        wire = search.solve_batch(w, ladder=lad)
        for k in RES_KEYS + ("solution", "metrics", "error_index"):
            assert np.array_equal(getattr(dev, k), getattr(wire, k)), (lad, k)
        orc = oracle.dftsp_batch(sb, ladder=lad, threads=8)
        _assert_same(wire, orc, sb, f"wire ladder {lad}")


def test_gpu_wire_format_implicit_ids_and_offsets():
    """Row-position ids and implicit uniform offsets (eb_dftsp_batch_packed with
    id = NULL, offsets = NULL) give exactly the wide call's results when the
    ids rise along each instance's rows."""
    from paper_2405_07140_b200 import synth
    from paper_2405_07140_b200.soa import pack_wire
    b = synth.generate(synth.CONFIG2, 20000, seed=99)           # ids 0..K-1 per instance
    w = pack_wire(b)
    assert w.columns["id"] is None and w.offsets is None
    lad = (128, 256, 512)
    dev = search.solve_batch(b, ladder=lad)
    wire = search.solve_batch(w, ladder=lad)
    for k in RES_KEYS + ("solution", "metrics", "error_index", "solution_mask"):
        assert np.array_equal(getattr(dev, k), getattr(wire, k)), k
    orc = oracle.dftsp_batch(b, ladder=lad, threads=8)
    _assert_same(wire, orc, b, "wire implicit")
    # the selection mask names exactly the solution's local indices
    for i in range(b.n_inst):
        lo, z = int(b.offsets[i]), int(dev.z_found[i])
        want = sum(1 << int(j) for j in dev.solution[lo:lo + z])
        assert int(dev.solution_mask[i]) == want, i
