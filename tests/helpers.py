"""Shared test helpers: golden corpora loading, sub-batching and comparison."""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLDEN = os.path.join(HERE, "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

from paper_2405_07140_b200.soa import REQ_FIELDS, InstanceBatch  # noqa: E402

FLAGS = {
    "P": dict(pruning=True, inclusive_bound=False, exact_tau=False),
    "NP": dict(pruning=False, inclusive_bound=False, exact_tau=False),
    "PI": dict(pruning=True, inclusive_bound=True, exact_tau=False),
    "PE": dict(pruning=True, inclusive_bound=False, exact_tau=True),
    "NL": dict(pruning=True, inclusive_bound=False, exact_tau=False),
}
RANDOM_CORPORA = ("random_2024", "random_31", "random_32", "random_33", "random_34", "random_35",
                  "random_1001", "random_77")
ALL_CORPORA = RANDOM_CORPORA + ("scenario", "config2", "config5", "ksweep", "wide", "wide_np")


def corpus_path(name: str) -> str:
    return os.path.join(GOLDEN, f"{name}.npz")


def load_corpus(name: str) -> dict:
    with np.load(corpus_path(name)) as z:
        d = {k: z[k] for k in z.files}
    meta = os.path.join(GOLDEN, f"{name}.json")
    d["_meta"] = json.load(open(meta)) if os.path.exists(meta) else {}
    return d


def ladder_of(d: dict, i: int):
    row = d["ladder"][i]
    if row[0] < 0:
        return None
    return tuple(int(v) for v in row[1:1 + row[0]])


def groups(d: dict, use_ladder: bool = True) -> dict:
    """Instance indices grouped by ladder (one device call per ladder)."""
    out: dict = {}
    n = len(d["offsets"]) - 1
    for i in range(n):
        key = ladder_of(d, i) if use_ladder else None
        out.setdefault(key, []).append(i)
    return out


def sub_batch(d: dict, idx) -> InstanceBatch:
    """InstanceBatch over the selected instances (rows gathered, CSR rebuilt)."""
    off = d["offsets"]
    sizes = np.array([off[i + 1] - off[i] for i in idx], np.int64)
    new_off = np.zeros(len(idx) + 1, np.int64)
    np.cumsum(sizes, out=new_off[1:])
    rows = np.concatenate([np.arange(off[i], off[i + 1]) for i in idx]) if len(idx) else np.zeros(0, np.int64)
    cols = {name: np.ascontiguousarray(d["req_" + name][rows].astype(dt)) for name, dt in REQ_FIELDS}
    if len(rows) == 0:
        cols = {name: np.zeros(1, dt) for name, dt in REQ_FIELDS}
    ci = np.ascontiguousarray(d["ctx_index"][list(idx)], np.int32)
    kmax = int(sizes.max()) if len(sizes) else 1
    return InstanceBatch(new_off, cols, np.ascontiguousarray(d["ctx"]), ci, max(kmax, 1))


def expected(d: dict, tag: str, i: int) -> dict:
    off = d["offsets"]
    lo = int(off[i])
    z = int(d[f"{tag}_z"][i])
    return dict(status=int(d[f"{tag}_status"][i]), z=z, visited=int(d[f"{tag}_visited"][i]),
                pruned=int(d[f"{tag}_pruned"][i]), counts=tuple(int(c) for c in d[f"{tag}_counts"][i, :d[f"{tag}_ncls"][i]]),
                solution=tuple(int(s) for s in d[f"{tag}_solution"][lo:lo + z]))


def got(res, batch: InstanceBatch, j: int) -> dict:
    """Same view of a solve_batch/oracle result row j."""
    g = (lambda k: getattr(res, k)) if not isinstance(res, dict) else (lambda k: res[k])
    lo = int(batch.offsets[j])
    z = int(g("z_found")[j])
    status = int(g("status")[j])
    nc = int(g("n_classes")[j])
    return dict(status=status, z=z if status == 0 else 0,
                visited=int(g("nodes_visited")[j]) if status == 0 else 0,
                pruned=int(g("nodes_pruned")[j]) if status == 0 else 0,
                counts=tuple(int(c) for c in g("counts")[j, :nc]) if status == 0 else (),
                solution=tuple(int(s) for s in g("solution")[lo:lo + z]) if status == 0 else ())


def compare_corpus(d: dict, tag: str, solve, use_ladder: bool = True, max_report: int = 5):
    """Run `solve(batch, ladder=..., **flags)` per ladder group; return list of mismatches."""
    bad = []
    for ladder, idx in groups(d, use_ladder).items():
        b = sub_batch(d, idx)
        res = solve(b, ladder=ladder, **FLAGS[tag])
        for j, i in enumerate(idx):
            e, g = expected(d, tag, i), got(res, b, j)
            if e["status"] != 0:
                ok = g["status"] == e["status"]
            else:
                ok = e == g
            if not ok:
                bad.append((i, e, g))
                if len(bad) >= max_report:
                    return bad
    return bad
