"""The per-call drop-in API (reference names, Request objects in, SearchOutcome
out) against the CPU oracle on the same pools: dftsp (dftsp.py:237),
dftsp_many, exhaustive_optimal in both modes (dftsp.py:288), check_direct
(feasibility.py:192), recover_subset (dftsp.py:85) and SearchTables.build
(dftsp.py:110).  The solution is the caller's own Request objects, sorted by
id, and the inputs are not mutated (SURVEY.md §8(b) ownership)."""
import numpy as np
import pytest

import oracle
from gen_random import random_batch
from paper_2405_07140_b200 import (EdgeContext, LlmSpec, NodeCompute, QuantProfile, RadioConfig, Request, UserLink,
                                   check_direct, derive_coefficients, dftsp, dftsp_many, exhaustive_optimal,
                                   partition, recover_subset)
from paper_2405_07140_b200.search import SearchTables
from paper_2405_07140_b200.soa import InstanceBatch

pytestmark = pytest.mark.gpu


def ctx_from_record(rec) -> EdgeContext:
    """EdgeContext objects carrying exactly one eb_context record's values."""
    llm = LlmSpec("rnd", int(rec["layers"]), int(rec["hidden_dim"]), int(rec["head_count"]), int(rec["head_dim"]),
                  int(rec["ffn_dim"]), int(rec["bytes_per_param"]))
    quant = QuantProfile("rnd", 16, 16, float(rec["alpha"]), float(rec["beta"]))
    radio = RadioConfig(float(rec["uplink_band_hz"]), float(rec["downlink_band_hz"]), float(rec["downlink_power_w"]),
                        float(rec["noise_density_w_hz"]), float(rec["uplink_slot_s"]), float(rec["downlink_slot_s"]),
                        int(rec["bits_per_token"]))
    node = NodeCompute(float(rec["flops_per_s"]), float(rec["memory_bytes"]), int(rec["gpu_count"]))
    return EdgeContext(llm, quant, radio, node, float(rec["slot_cap_s"]) if rec["has_slot_cap"] else None)


def pools_of(batch):
    out = []
    for i in range(batch.n_inst):
        lo, hi = int(batch.offsets[i]), int(batch.offsets[i + 1])
        c = batch.columns
        out.append([Request(id=int(c["id"][j]), prompt_tokens=int(c["prompt_tokens"][j]),
                            output_tokens=int(c["output_tokens"][j]), deadline_s=float(c["deadline_s"][j]),
                            tolerance=float(c["tolerance"][j]),
                            link=UserLink(float(c["channel_gain"][j]), float(c["uplink_power_w"][j])),
                            waiting_s=float(c["waiting_s"][j])) for j in range(lo, hi)])
    return out


def one(batch, i):
    lo, hi = int(batch.offsets[i]), int(batch.offsets[i + 1])
    ci = int(batch.ctx_index[i])
    cols = {k: np.ascontiguousarray(v[lo:hi]) for k, v in batch.columns.items()}
    return InstanceBatch(np.array([0, hi - lo], np.int64), cols, batch.contexts[ci:ci + 1].copy(),
                         np.zeros(1, np.int32), max(hi - lo, 1))


@pytest.mark.parametrize("seed", [61, 62])
def test_dftsp_per_call_matches_oracle(seed):
    batch, ladders = random_batch(seed, 40, k_min=1, k_max=14)
    pools = pools_of(batch)
    compared = found = 0
    for i, pool in enumerate(pools):
        ctx = ctx_from_record(batch.contexts[int(batch.ctx_index[i])])
        before = [(r.id, r.waiting_s) for r in pool]
        try:
            out = dftsp(pool, ctx, ladder=ladders[i])
        except ValueError:
            continue                                  # reference exceptions: covered by the status tests
        assert [(r.id, r.waiting_s) for r in pool] == before   # inputs untouched
        orc = oracle.dftsp_batch(one(batch, i), ladder=ladders[i])
        compared += 1
        found += out.z_found > 0
        assert out.z_found == int(orc["z_found"][0]), i
        assert out.nodes_visited == int(orc["nodes_visited"][0]) and out.nodes_pruned == int(orc["nodes_pruned"][0])
        if out.z_found:
            ids = [pool[int(j)].id for j in orc["solution"][:out.z_found]]
            assert [r.id for r in out.solution] == ids
            assert all(any(r is p for p in pool) for r in out.solution)      # the caller's objects
            assert [r.id for r in out.solution] == sorted(r.id for r in out.solution)
            assert check_direct(out.solution, ctx, max(r.prompt_tokens for r in pool))
    assert compared >= 30 and found >= 10, (compared, found)


def test_dftsp_many_equals_per_call():
    batch, ladders = random_batch(63, 30, k_min=2, k_max=12, dup_ladder=False)
    pools = pools_of(batch)
    lad = ladders[0]
    keep = [i for i, l in enumerate(ladders) if l == lad]
    ctxs = [ctx_from_record(batch.contexts[int(batch.ctx_index[i])]) for i in keep]
    for i, ctx in zip(keep, ctxs):
        try:
            single = dftsp(pools[i], ctx, ladder=lad)
        except ValueError:
            continue
        many = dftsp_many([pools[i]], ctx, ladder=lad)[0]
        assert (many.z_found, many.nodes_visited, many.nodes_pruned, many.counts) == \
               (single.z_found, single.nodes_visited, single.nodes_pruned, single.counts)


@pytest.mark.parametrize("seed", [64, 65])
def test_exhaustive_optimal_both_modes_match_oracle(seed):
    batch, ladders = random_batch(seed, 40, k_min=1, k_max=12)
    pools = pools_of(batch)
    compared = 0
    for i, pool in enumerate(pools):
        ctx = ctx_from_record(batch.contexts[int(batch.ctx_index[i])])
        ci = int(batch.ctx_index[i])
        lo, hi = int(batch.offsets[i]), int(batch.offsets[i + 1])
        st, z, rk, nodes, mask = oracle.exhaustive(batch.contexts[ci:ci + 1], batch.columns, lo, hi, cap=20)
        if st != 0:
            continue
        out = exhaustive_optimal(pool, ctx, cap=20)
        compared += 1
        assert (out.z_found, out.nodes_visited) == (z, nodes), i
        assert sorted(r.id for r in (out.solution or [])) == sorted(pool[j].id for j in range(len(pool)) if mask >> j & 1)
        stc, zc, nc, _ = oracle.exhaustive_counts(batch.contexts[ci:ci + 1], batch.columns, lo, hi, ladder=ladders[i])
        if stc == 0:
            oc = exhaustive_optimal(pool, ctx, mode="counts", ladder=ladders[i])
            assert (oc.z_found, oc.nodes_visited) == (zc, nc), i
    assert compared >= 30, compared
    with pytest.raises(ValueError):
        exhaustive_optimal(pools[0], ctx_from_record(batch.contexts[0]), mode="bogus")


def test_partition_recover_and_tables():
    batch, ladders = random_batch(66, 10, k_min=6, k_max=12)
    pools = pools_of(batch)
    for i, pool in enumerate(pools):
        ctx = ctx_from_record(batch.contexts[int(batch.ctx_index[i])])
        part = partition(pool, ctx.radio, ladder=ladders[i])
        assert sum(part.sizes) == len(pool) and list(part.lengths) == sorted(part.lengths)
        for keys in part.keys:
            assert list(keys) == sorted(keys)
        counts = tuple(min(1, s) for s in part.sizes)
        sub = recover_subset(part, counts)
        assert [r.id for r in sub] == [c[0].id for c in part.classes if c][:len(sub)]
        co = derive_coefficients(ctx, max(r.prompt_tokens for r in pool), pool)
        t = SearchTables.build(part, co)
        assert t.tail[0] == len(pool) and len(t.up) == len(part.classes)
        for k, members in enumerate(part.classes):
            acc = 0.0
            for x, r in enumerate(members, start=1):
                acc = acc + co.k_up[r.id] * r.prompt_tokens
                assert t.up[k][x] == acc
