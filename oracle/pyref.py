"""THE UNMODIFIED PYTHON REFERENCE as a CPU baseline -- test infrastructure only.

Imports the reference package `edgebatch` from oracle/_ref/ (staged verbatim
from /root/reference/pkg/src by oracle/make_ref.py; it travels to the GPU box
with the repo snapshot) and times its own public entry point
``edgebatch.dftsp(candidates, ctx, ladder=...)`` (dftsp.py:237) on instances of
the benchmark workload, the way BASELINE.md §3 asks:

  * the instances are the device's InstanceBatch rows turned into the
    reference's own ``Request`` / ``UserLink`` / ``EdgeContext`` objects
    (feasibility.py:33-71, radio.py:46-57) before the timer starts;
  * ``concurrent.futures.ProcessPoolExecutor(nproc)`` over contiguous
    chunks, the reference's own sweep parallelism (cli.py:262-264);
  * the step time is the span from the first worker's first dftsp call to the
    last worker's last return (object construction excluded).

Used only by bench.py (--impl reference, and the cpu_baseline leg) and tests;
never by the product package.
"""
from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def available() -> bool:
    return os.path.isfile(os.path.join(REF_DIR, "edgebatch", "dftsp.py"))


def import_reference():
    if not available():
        raise RuntimeError("oracle/_ref/edgebatch is missing: run oracle/make_ref.py in the build container")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import edgebatch
    assert os.path.dirname(os.path.abspath(edgebatch.__file__)) == os.path.join(REF_DIR, "edgebatch"), \
        "a different edgebatch shadows oracle/_ref"
    return edgebatch


def context_of(rec):
    """eb_context record -> the reference EdgeContext (catalog.py, radio.py, costs.py)."""
    eb = import_reference()
    llm = eb.LlmSpec("bench-model", int(rec["layers"]), int(rec["hidden_dim"]), int(rec["head_count"]),
                     int(rec["head_dim"]), int(rec["ffn_dim"]), int(rec["bytes_per_param"]))
    quant = eb.QuantProfile("bench-q", 16, 16, alpha=float(rec["alpha"]), beta=float(rec["beta"]),
                            delta_ppl_by_model={"bench-model": float(rec["delta_ppl"])})
    radio = eb.RadioConfig(uplink_band_hz=float(rec["uplink_band_hz"]), downlink_band_hz=float(rec["downlink_band_hz"]),
                           downlink_power_w=float(rec["downlink_power_w"]),
                           noise_density_w_hz=float(rec["noise_density_w_hz"]),
                           uplink_slot_s=float(rec["uplink_slot_s"]), downlink_slot_s=float(rec["downlink_slot_s"]),
                           bits_per_token=int(rec["bits_per_token"]))
    node = eb.NodeCompute(float(rec["flops_per_s"]), float(rec["memory_bytes"]), int(rec["gpu_count"]))
    cap = float(rec["slot_cap_s"]) if int(rec["has_slot_cap"]) else None
    return eb.EdgeContext(llm, quant, radio, node, slot_cap_s=cap)


def requests_of(cols: dict, lo: int, hi: int) -> list:
    eb = import_reference()
    out = []
    for j in range(lo, hi):
        out.append(eb.Request(id=int(cols["id"][j]), prompt_tokens=int(cols["prompt_tokens"][j]),
                              output_tokens=int(cols["output_tokens"][j]), deadline_s=float(cols["deadline_s"][j]),
                              tolerance=float(cols["tolerance"][j]),
                              link=eb.UserLink(float(cols["channel_gain"][j]), float(cols["uplink_power_w"][j])),
                              waiting_s=float(cols["waiting_s"][j])))
    return out


def _chunk_job(job):
    """Worker: build the reference objects for a chunk, then time dftsp over it."""
    recs, offsets, ctx_index, cols, ladder, flags = job
    eb = import_reference()
    ctxs = [context_of(recs[i]) for i in range(len(recs))]
    pools = [(ctxs[int(ctx_index[i])], requests_of(cols, int(offsets[i]), int(offsets[i + 1])))
             for i in range(len(offsets) - 1)]
    z = np.zeros(len(pools), np.int32)
    vis = np.zeros(len(pools), np.int64)
    prn = np.zeros(len(pools), np.int64)
    t0 = time.time()
    for i, (ctx, reqs) in enumerate(pools):
        o = eb.dftsp(reqs, ctx, ladder=ladder, **flags)
        z[i], vis[i], prn[i] = o.z_found, o.nodes_visited, o.nodes_pruned
    t1 = time.time()
    return t0, t1, z, vis, prn


class ReferencePool:
    """A persistent ProcessPoolExecutor(procs) running the reference's dftsp."""

    def __init__(self, procs: int | None = None):
        import multiprocessing as mp
        self.procs = procs or os.cpu_count() or 1
        import_reference()
        # spawn: the parent may hold a CUDA context (fork after CUDA init is unsafe)
        self.ex = ProcessPoolExecutor(self.procs, mp_context=mp.get_context("spawn"))
        list(self.ex.map(_noop, range(self.procs)))   # start every worker before any timing

    def run(self, batch, lo: int, hi: int, ladder=None, **flags):
        """dftsp on instances [lo, hi) of `batch`: (span_s, z, visited, pruned)."""
        n = hi - lo
        cuts = [lo + n * t // self.procs for t in range(self.procs + 1)]
        jobs = []
        for a, b in zip(cuts[:-1], cuts[1:]):
            if b <= a:
                continue
            r0, r1 = int(batch.offsets[a]), int(batch.offsets[b])
            cols = {k: np.ascontiguousarray(v[r0:r1]) for k, v in batch.columns.items()}
            jobs.append((batch.contexts, batch.offsets[a:b + 1] - r0, batch.ctx_index[a:b], cols,
                         tuple(ladder) if ladder else None, flags))
        res = list(self.ex.map(_chunk_job, jobs))
        span = max(r[1] for r in res) - min(r[0] for r in res)
        return (span, np.concatenate([r[2] for r in res]), np.concatenate([r[3] for r in res]),
                np.concatenate([r[4] for r in res]))

    def close(self):
        self.ex.shutdown(wait=True, cancel_futures=True)


def _noop(_):
    import_reference()
    return os.getpid()
