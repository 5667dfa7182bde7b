"""Brute-force 2^K search sharded across GPUs by subset rank (config 4).

``exhaustive_optimal(mode="subsets")`` (reference dftsp.py:305-313) returns the
first feasible subset in itertools.combinations order, searching sizes from K
down.  Equivalently: z* = the largest size with any
feasible subset and r* = the smallest lexicographic rank among feasible
subsets of size z*; nodes_visited = sum_{z > z*} C(K, z) + r* + 1.

Sharding: every level's rank range [0, C(K, z)) is split into `world`
contiguous pieces; rank g searches its piece of each level from z = K down and
stops at its first level with a hit.  The global answer is the max over ranks
of the key (z, -rank) -- one 8-byte all-reduce(MAX) over NCCL (the only
collective; two tiny ones when K > 56 and the rank no longer fits the key).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from math import comb

import numpy as np

from . import _lib
from .soa import requests_struct

RANK_BITS = 57


@dataclass
class BruteResult:
    z: int
    lexrank: int
    nodes_visited: int
    mask: int


def shard(total: int, world: int, rank: int):
    """Contiguous piece `rank` of [0, total) split `world` ways."""
    return total * rank // world, total * (rank + 1) // world


def pack(z: int, r: int) -> int:
    return (z << RANK_BITS) | ((1 << RANK_BITS) - 1 - r) if z else 0


def unpack(key: int):
    if key == 0:
        return 0, -1
    z = key >> RANK_BITS
    return z, (1 << RANK_BITS) - 1 - (key & ((1 << RANK_BITS) - 1))


def unrank(n: int, z: int, r: int) -> int:
    """Bitmask of the r-th size-z combination of range(n) in lexicographic order."""
    m, v = 0, 0
    for j in range(z):
        while True:
            c = comb(n - v - 1, z - j - 1)
            if r < c:
                m |= 1 << v
                v += 1
                break
            r -= c
            v += 1
    return m


def nodes_for(n: int, z: int, r: int) -> int:
    if z == 0:
        return 2 ** n - 1 if n else 0
    return sum(comb(n, q) for q in range(z + 1, n + 1)) + r + 1


def device_level_range(ctx_rec: np.ndarray, cols: dict, device=None):
    """Level evaluator on this process's GPU: (z, lo, hi) -> first feasible rank or -1."""
    h = _lib.handle(device)
    n = int(cols["prompt_tokens"].shape[0])
    rs = requests_struct(cols)
    ref = ctypes.cast(ctypes.pointer(rs), ctypes.c_void_p)

    def raise_link(code):
        if code == _lib.ERR_NONPOSITIVE_LINK:
            raise ValueError("power, gain and noise must be strictly positive")
        if code in (_lib.ERR_UPLINK_EFF_ZERO, _lib.ERR_DOWNLINK_EFF_ZERO):
            raise ValueError("uplink spectral efficiency is zero" if code == _lib.ERR_UPLINK_EFF_ZERO
                             else "downlink spectral efficiency is zero")

    # levels the sound bounds do not refute (the range search would return -1
    # for the others without enumerating anything)
    live = ctypes.c_uint64(0)
    code = h.lib.eb_exhaustive_live_levels(h.ptr, ctx_rec.ctypes.data, n, ref, ctypes.byref(live))
    raise_link(code)
    _lib.check(code, "eb_exhaustive_live_levels")
    live_mask = int(live.value)

    def level(z: int, lo: int, hi: int) -> int:
        if not (live_mask >> (z - 1)) & 1:
            return -1
        out = ctypes.c_int64(-1)
        code = h.lib.eb_exhaustive_level_range(h.ptr, ctx_rec.ctypes.data, n, ref, z, lo, hi, ctypes.byref(out))
        raise_link(code)
        _lib.check(code, "eb_exhaustive_level_range")
        return int(out.value)

    level.live_mask = live_mask
    return level


def enum_stats(device=None) -> np.ndarray:
    """[combinations checked, prefixes pruned] by this process's brute-force
    kernels on `device` so far (eb_exhaustive_counters)."""
    h = _lib.handle(device)
    out = np.zeros(2, np.int64)
    _lib.check(h.lib.eb_exhaustive_counters(h.ptr, out.ctypes.data), "eb_exhaustive_counters")
    return out


def local_search(n: int, world: int, rank: int, level) -> tuple:
    """This rank's best (z, r) over its shard of every level, searching z = n..1."""
    for z in range(n, 0, -1):
        lo, hi = shard(comb(n, z), world, rank)
        if hi > lo:
            r = level(z, lo, hi)
            if r >= 0:
                return z, r
    return 0, -1


def combine(keys) -> tuple:
    """max over ranks of (z, -r)."""
    best = (0, -1)
    for z, r in keys:
        if z > best[0] or (z == best[0] and z and r < best[1]):
            best = (z, r)
    return best


def finish(n: int, z: int, r: int) -> BruteResult:
    return BruteResult(z, r, nodes_for(n, z, r), unrank(n, z, r) if z else 0)


def solve_sharded(ctx_rec, cols: dict, world: int, level=None, device=None) -> BruteResult:
    """All `world` shards evaluated by this process in turn (single-GPU check of the sharding)."""
    n = int(cols["prompt_tokens"].shape[0])
    level = level or device_level_range(ctx_rec, cols, device)
    return finish(n, *combine(local_search(n, world, g, level) for g in range(world)))


def solve_distributed(ctx_rec, cols: dict, level=None, device=None, group=None) -> BruteResult:
    """One shard of every level per torch.distributed rank, levels z = K..1.

    The levels the sound bounds refute are skipped by every rank alike (the
    live mask is computed from the same data on each rank, no exchange).  On
    each live level every rank scans its contiguous rank range, then one
    8-byte all-reduce(MIN) of the first feasible rank found (or a sentinel)
    decides the level for all ranks together: the first level with any hit is
    z*, the minimum is r*, and no rank descends further alone.
    """
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    n = int(cols["prompt_tokens"].shape[0])
    if device is None and dist.get_backend(group) == "nccl":
        device = torch.cuda.current_device()
    level = level or device_level_range(ctx_rec, cols, device)
    live = getattr(level, "live_mask", (1 << n) - 1)
    on_gpu = dist.get_backend(group) == "nccl"
    tdev = torch.device("cuda", torch.cuda.current_device()) if on_gpu else torch.device("cpu")
    none = 2 ** 63 - 1
    key = torch.empty(1, dtype=torch.int64, device=tdev)
    for z in range(n, 0, -1):
        if not (live >> (z - 1)) & 1:
            continue
        lo, hi = shard(comb(n, z), world, rank)
        r = level(z, lo, hi) if hi > lo else -1
        key.fill_(r if r >= 0 else none)
        dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
        rg = int(key.item())
        if rg != none:
            return finish(n, z, rg)
    return finish(n, 0, -1)
