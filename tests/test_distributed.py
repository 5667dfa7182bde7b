"""Multi-GPU host logic on CPU with torch.distributed gloo (world size 2):
the brute-force rank-range sharding + all-reduce(MAX) of the packed key, and
the instance sharding of the DFTSP sweep.  The per-rank evaluator is the CPU
oracle (the GPU runs the same driver with device_level_range / K3)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from gen_random import random_batch
from paper_2405_07140_b200 import brute


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _brute_worker(rank, world, port, seed, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, _ = random_batch(seed, 6, k_min=10, k_max=14)
    out = []
    for i in range(b.n_inst):
        lo, hi = int(b.offsets[i]), int(b.offsets[i + 1])
        cols = {k: np.ascontiguousarray(v[lo:hi]) for k, v in b.columns.items()}
        rec = b.contexts[int(b.ctx_index[i]):int(b.ctx_index[i]) + 1]
        res = brute.solve_distributed(rec, cols, level=oracle.level_evaluator(rec, cols))
        out.append((res.z, res.lexrank, res.nodes_visited, res.mask))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("seed", [1, 2])
def test_brute_force_sharded_gloo_world2(seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_brute_worker, args=(r, 2, port, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results[0] == results[1]
    b, _ = random_batch(seed, 6, k_min=10, k_max=14)
    for i, got in enumerate(results[0]):
        rec = b.contexts[int(b.ctx_index[i]):int(b.ctx_index[i]) + 1]
        st, z, rk, nodes, mask = oracle.exhaustive(rec, b.columns, int(b.offsets[i]), int(b.offsets[i + 1]))
        assert got == (z, rk, nodes, mask), i


def test_shard_math_covers_every_rank():
    from math import comb
    for n in (5, 17, 32):
        for z in (1, n // 2, n):
            total = comb(n, z)
            for world in (1, 2, 3, 8):
                pieces = [brute.shard(total, world, g) for g in range(world)]
                assert pieces[0][0] == 0 and pieces[-1][1] == total
                assert all(pieces[g][1] == pieces[g + 1][0] for g in range(world - 1))


def test_key_packing_orders_like_the_reference():
    keys = [(5, 10), (5, 3), (4, 0), (0, -1), (6, 100)]
    packed = sorted(keys, key=lambda k: brute.pack(*k), reverse=True)
    assert packed[0] == (6, 100) and packed[1] == (5, 3)
    for z, r in keys:
        if z:
            assert brute.unpack(brute.pack(z, r)) == (z, r)
    assert brute.combine(keys) == (6, 100)


def test_unrank_matches_itertools():
    from itertools import combinations
    n, z = 9, 4
    for r, combo in enumerate(combinations(range(n), z)):
        assert brute.unrank(n, z, r) == sum(1 << c for c in combo)


def _sweep_worker(rank, world, port, q):
    """Instance sharding: each rank solves its contiguous range; gather == single rank."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from gen_random import take
    b, lad = random_batch(44, 64, k_max=10, max_classes=1)
    n = b.n_inst
    lo, hi = n * rank // world, n * (rank + 1) // world
    idx = list(range(lo, hi))
    sub = take(b, idx)
    res = oracle.dftsp_batch(sub, ladder=None)
    tot = torch.tensor([res["nodes_visited"].sum(), res["z_found"].sum()], dtype=torch.int64)
    dist.all_reduce(tot)
    q.put((rank, tot.tolist()))
    dist.destroy_process_group()


def test_instance_sharding_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sweep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    b, _ = random_batch(44, 64, k_max=10, max_classes=1)
    full = oracle.dftsp_batch(b, ladder=None)
    assert res[0] == res[1] == [int(full["nodes_visited"].sum()), int(full["z_found"].sum())]


def _bench_timing_worker(rank, world, port, q):
    """bench.py's multi-rank plumbing on gloo: the max-over-ranks timing
    reduction and the barrier (NCCL on the GPU box; same calls)."""
    import sys
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    bench.barrier(world)
    t = bench.max_over_ranks(0.25 + rank, world)          # each rank's elapsed seconds
    q.put((rank, t))
    dist.destroy_process_group()


def test_bench_max_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_timing_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert got == {0: 1.25, 1: 1.25}          # every rank reports the slowest rank's time


def test_bench_self_spawns_world2_reference_arm():
    """bench.py --gpus 2 outside torchrun re-launches itself with 2 ranks
    (torch.distributed.run); rank 0 prints one line with n_gpus 2."""
    import json
    import subprocess
    import sys
    from helpers import ROOT
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--n-inst", "3000", "--cpu-sample", "40"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["impl"] == "reference" and j["value"] > 0
    assert j["c_port_agrees_with_reference"] is True
