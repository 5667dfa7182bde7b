#!/usr/bin/env python3
"""Benchmark the non-headline BASELINE.json configs on one B200 (JSON line each).

  config1  per-epoch candidate pools the reference simulator hands to dftsp on
           pkg/scenarios (captured by tests/golden/make_golden.py): DFTSP and
           brute force, parity vs the reference's recorded outputs
  config3  K = 10..40 sweep x deadline scale x tolerance cap (w8a16): DFTSP
           instances/s per K and mean z, beside the StB / NoB batching baselines
           on the same queues (mean scheduled and on-time requests)
  config4  brute force 2^K, K = 28..32: level-by-level rank-range search
           (brute.solve_sharded, world 1 on this GPU; the same driver shards by
           rank over NCCL), z cross-checked against DFTSP (optimality)
  config5  tight-memory OPT-13B edge (5 output classes): DFTSP instances/s

kernel_inst_per_s: inputs resident in HBM (eb_dftsp_batch, EB_MEM_DEVICE);
wire_e2e_inst_per_s: pinned host buffers through eb_dftsp_batch_packed (copies
included); api_inst_per_s: search.solve_batch on pageable numpy arrays (the
Python convenience API, allocation and pageable copies included).
CPU columns time the C oracle port on a bounded sample with all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

from paper_2405_07140_b200 import _lib, brute, search, synth  # noqa: E402
from paper_2405_07140_b200.soa import InstanceBatch  # noqa: E402


def ev_time(fn, reps=3):
    import torch
    fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    return min(t)


def device_rates(batch, ladder, reps=3):
    """(kernel inst/s with inputs resident in HBM, end-to-end inst/s through
    eb_dftsp_batch_packed with pinned host buffers) -- bench.py's two legs."""
    import ctypes
    import torch
    from paper_2405_07140_b200.soa import pack_wire, search_params
    dev = torch.device("cuda", 0)
    h = _lib.handle(0)
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    n, nr = batch.n_inst, batch.n_req

    def td(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    used = [k for k in batch.columns if k != "tolerance"]
    db = InstanceBatch(td(batch.offsets), {k: td(batch.columns[k]) for k in used}, batch.contexts,
                       td(batch.ctx_index), batch.k_max, on_device=True).struct()
    d_ctx = td(batch.contexts.view(np.uint8))
    outs = {"status": (n, torch.int32), "z_found": (n, torch.int32), "nodes_visited": (n, torch.int64),
            "nodes_pruned": (n, torch.int64), "solution": (nr, torch.int32)}
    dres, hres = _lib.eb_dftsp_result(), _lib.eb_dftsp_result()
    keep = []
    for k, (m, dt) in outs.items():
        a = torch.zeros(m, dtype=dt, device=dev)
        b = torch.zeros(m, dtype=dt).pin_memory()
        keep += [a, b]
        setattr(dres, k, a.data_ptr())
        setattr(hres, k, b.data_ptr())
    prm = search_params(ladder=ladder)
    ref = lambda x: ctypes.cast(ctypes.pointer(x), ctypes.c_void_p)  # noqa: E731
    wb = pack_wire(batch, pin=lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy())
    wbs = wb.struct() if wb is not None else None        # the wire format stops at EB_MAX_K

    def k_dev():
        _lib.check(h.lib.eb_dftsp_batch(h.ptr, d_ctx.data_ptr(), len(batch.contexts), ref(prm), ref(db), ref(dres),
                                        _lib.EB_MEM_DEVICE), "device")

    def k_wire():
        _lib.check(h.lib.eb_dftsp_batch_packed(h.ptr, batch.contexts.ctypes.data, len(batch.contexts), ref(prm),
                                               ref(wbs), ref(hres), _lib.EB_MEM_HOST), "wire")

    def timed(fn):
        with torch.cuda.stream(st):
            fn()
            st.synchronize()
            best = float("inf")
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fn()
                e1.record(st)
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1) / 1e3)
        return n / best
    return timed(k_dev), (timed(k_wire) if wbs is not None else float("nan"))


def cpu_rate(batch, ladder, sample, threads):
    import oracle
    n = min(sample, batch.n_inst)
    sub = InstanceBatch(batch.offsets[:n + 1].copy(), {k: v[:int(batch.offsets[n])] for k, v in batch.columns.items()},
                        batch.contexts, batch.ctx_index[:n].copy(), batch.k_max)
    t0 = time.perf_counter()
    res = oracle.dftsp_batch(sub, ladder=ladder, threads=threads)
    return n / (time.perf_counter() - t0), res


def config1(threads):
    from helpers import groups, load_corpus, sub_batch, expected, got
    d = load_corpus("scenario")
    n = len(d["offsets"]) - 1
    bad = 0
    tot = 0.0
    for ladder, ids in groups(d).items():
        b = sub_batch(d, ids)
        tot += ev_time(lambda: search.solve_batch(b, ladder=ladder), reps=3)
        res = search.solve_batch(b, ladder=ladder)
        bad += sum(expected(d, "P", i) != got(res, b, j) for j, i in enumerate(ids))
    # brute force on the pools the reference's own oracle cap (16) admits
    from helpers import sub_batch as sb
    small = [i for i in range(n) if d["offsets"][i + 1] - d["offsets"][i] <= 12 and d["ex_status"][i] == 0]
    b = sb(d, small)
    from test_gpu_exhaustive import _run  # noqa
    t_ex = ev_time(lambda: _run(b, cap=16), reps=3)
    st, z, rk, nodes, mask = _run(b, cap=16)
    bad_ex = int(np.sum(z != d["ex_z"][small]) + np.sum(nodes != d["ex_nodes"][small]))
    return {"config": "config1: scenario epochs (pkg/scenarios default/throughput, rates 2-50)", "instances": n,
            "dftsp_inst_per_s": round(n / tot, 1), "mismatches_vs_reference": int(bad),
            "brute_instances": len(small), "brute_inst_per_s": round(len(small) / t_ex, 1),
            "brute_mismatches_vs_reference": bad_ex}


def batching_baselines(b, w):
    """StB and NoB on the same queues (the instances' candidates, FIFO in row
    order), on the device: mean on-time requests per instance.  StB: b =
    static_batch_size (baselines.py:51-65), FIFO admission (eb_stb_batch),
    then the batch's own cost (eb_batch_cost_batch); a member is on time when
    waiting + slots + latency <= deadline (sim.py:369-385).  NoB: every device
    idle, one request per device (eb_nob_batch), on time when waiting +
    completion <= deadline."""
    import ctypes
    h = _lib.handle(0)
    ref = lambda x: ctypes.cast(ctypes.pointer(x), ctypes.c_void_p)  # noqa: E731
    n, nr = b.n_inst, b.n_req
    ctx = b.contexts
    slots = float(ctx["uplink_slot_s"][0] + ctx["downlink_slot_s"][0])
    sl = np.full(len(ctx), w.epoch_s)
    smax = np.full(len(ctx), max(w.prompts), np.int64)
    nmax = np.full(len(ctx), max(w.outputs), np.int64)
    bsz = np.zeros(len(ctx), np.int64)
    _lib.check(h.lib.eb_static_batch_size_batch(h.ptr, ctx.ctypes.data, len(ctx), sl.ctypes.data, smax.ctypes.data,
                                                nmax.ctypes.data, bsz.ctypes.data, _lib.EB_MEM_HOST), "static_b")
    bb = np.ascontiguousarray(bsz[b.ctx_index])
    st = np.zeros(n, np.int32)
    sel = np.zeros(nr, np.uint8)
    bs = b.struct()
    _lib.check(h.lib.eb_stb_batch(h.ptr, ctx.ctypes.data, len(ctx), ref(bs), bb.ctypes.data, 1, st.ctypes.data,
                                  sel.ctypes.data, _lib.EB_MEM_HOST), "stb")
    rows = np.nonzero(sel)[0]
    owner = np.searchsorted(b.offsets, rows, side="right") - 1
    plan_off = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(owner, minlength=n), out=plan_off[1:])
    pr = np.ascontiguousarray(b.columns["prompt_tokens"][rows])
    ou = np.ascontiguousarray(b.columns["output_tokens"][rows])
    padded = np.zeros(n, np.int64)
    np.maximum.at(padded, owner, pr.astype(np.int64))
    cost = np.zeros((n, 2))
    pc = np.ascontiguousarray(b.ctx_index)
    _lib.check(h.lib.eb_batch_cost_batch(h.ptr, ctx.ctypes.data, len(ctx), n, plan_off.ctypes.data, pr.ctypes.data,
                                         ou.ctypes.data, padded.ctypes.data, None, pc.ctypes.data, cost.ctypes.data,
                                         _lib.EB_MEM_HOST), "batch_cost")
    lat = cost[owner, 1]
    w_s, dl = b.columns["waiting_s"][rows], b.columns["deadline_s"][rows]
    stb_on = np.bincount(owner[(w_s + slots + lat) - dl <= 1e-9 * np.maximum(1.0, np.abs(dl))], minlength=n)
    now = np.zeros(n)
    G = int(ctx["gpu_count"].max())
    busy = np.zeros((n, G))
    st2 = np.zeros(n, np.int32)
    act = np.zeros(nr, np.int8)
    comp = np.zeros(nr)
    order = np.zeros(nr, np.int32)
    _lib.check(h.lib.eb_nob_batch(h.ptr, ctx.ctypes.data, len(ctx), ref(bs), now.ctypes.data, 1, None, G,
                                  busy.ctypes.data, st2.ctypes.data, act.ctypes.data, comp.ctypes.data,
                                  order.ctypes.data, _lib.EB_MEM_HOST), "nob")
    r2 = np.nonzero(act == 1)[0]
    o2 = np.searchsorted(b.offsets, r2, side="right") - 1
    tot = b.columns["waiting_s"][r2] + comp[r2]
    d2 = b.columns["deadline_s"][r2]
    nob_on = np.bincount(o2[tot - d2 <= 1e-9 * np.maximum(1.0, np.abs(d2))], minlength=n)
    return {"stb_b": int(bsz[0]), "stb_scheduled_mean": float(sel.sum() / n), "stb_on_time_mean": float(stb_on.mean()),
            "nob_scheduled_mean": float((act == 1).sum() / n), "nob_on_time_mean": float(nob_on.mean())}


def config3(threads, n_per_k):
    out = []
    for K in (10, 15, 20, 25, 30, 35, 40):
        for ds, tc in ((0.5, 0.25), (1.0, 1.0), (2.0, 0.5)):
            w = synth.Workload(f"config3 K={K} ds={ds} tc={tc}", profiles=("w8a16",), K=K, deadline_scale=ds,
                               tolerance_cap=tc)
            n = n_per_k if K <= 20 else max(n_per_k // 4, 1000)
            b = synth.generate(w, n, seed=2405_0714 + K)
            dt = ev_time(lambda: search.solve_batch(b, ladder=(128, 256, 512)), reps=2)
            res = search.solve_batch(b, ladder=(128, 256, 512))
            kr, er = device_rates(b, (128, 256, 512))
            cr, orc = cpu_rate(b, (128, 256, 512), 2000 if K <= 25 else 300, threads)
            ok = bool(np.array_equal(orc["nodes_visited"], res.nodes_visited[:len(orc["nodes_visited"])]))
            base = batching_baselines(b, w)
            out.append({"K": K, "deadline_scale": ds, "tolerance_cap": tc, "instances": n, **base,
                        "kernel_inst_per_s": round(kr, 1), "wire_e2e_inst_per_s": round(er, 1),
                        "api_inst_per_s": round(n / dt, 1), "mean_z": float(res.z_found.mean()),
                        "mean_nodes_visited": float(res.nodes_visited.mean()), "cpu_port_inst_per_s": round(cr, 1),
                        "parity_sample_ok": ok})
    return {"config": "config3: K sweep x deadline x tolerance (w8a16)", "rows": out}


def config4(ks, per_k):
    """Brute force (exhaustive_optimal subsets mode) at K = 28..32 on the
    adversarial family (synth.brute_family) and on config-2-style pools.
    Rates are instances/s and the device's checked combinations/s
    (brute.enum_stats); reference-accounted nodes are reported separately and
    are not an enumeration rate."""
    import torch
    out = []
    for K in ks:
        fams = [("adversarial", synth.brute_family(K, per_k, seed=2405_0714 + K))]
        w = synth.Workload(f"config4 K={K}", K=K)
        b = synth.generate(w, per_k, seed=2405_0715 + K)
        dres = search.solve_batch(b, ladder=(128, 256, 512))
        pools = []
        for i in range(per_k):
            lo, hi = int(b.offsets[i]), int(b.offsets[i + 1])
            cols = {k: np.ascontiguousarray(v[lo:hi]) for k, v in b.columns.items()}
            pools.append((b.contexts[int(b.ctx_index[i]):int(b.ctx_index[i]) + 1].copy(), cols))
        fams.append(("config2-style", pools))
        for name, insts in fams:
            for j, (rec, cols) in enumerate(insts):
                torch.cuda.synchronize()
                s0 = brute.enum_stats()
                t0 = time.perf_counter()
                r = brute.solve_sharded(rec, cols, world=1)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
                chk = brute.enum_stats() - s0
                row = {"K": K, "family": name, "z": r.z, "lexrank": r.lexrank, "seconds": round(dt, 5),
                       "checked_subsets": int(chk[0]), "pruned_prefixes": int(chk[1]),
                       "checked_subsets_per_s": round(int(chk[0]) / dt, 1),
                       "reference_nodes_visited": r.nodes_visited,
                       "reference_extrapolated_s_1core": round(r.nodes_visited / 6.0e4, 1)}
                if name == "config2-style":
                    row["dftsp_z"] = int(dres.z_found[j])
                    row["optimality_ok"] = r.z == int(dres.z_found[j])
                out.append(row)
    return {"config": "config4: brute force 2^K (subsets mode), rank-range level search", "rows": out}


def config5(threads, n):
    b = synth.generate(synth.CONFIG5, n, seed=2405_0716)
    lad = synth.CONFIG5.outputs
    dt = ev_time(lambda: search.solve_batch(b, ladder=lad), reps=2)
    res = search.solve_batch(b, ladder=lad)
    kr, er = device_rates(b, lad)
    cr, orc = cpu_rate(b, lad, 3000, threads)
    ok = bool(np.array_equal(orc["nodes_visited"], res.nodes_visited[:len(orc["nodes_visited"])]))
    return {"config": synth.CONFIG5.name, "instances": n, "kernel_inst_per_s": round(kr, 1),
            "wire_e2e_inst_per_s": round(er, 1), "api_inst_per_s": round(n / dt, 1),
            "mean_z": float(res.z_found.mean()), "mean_nodes_visited": float(res.nodes_visited.mean()),
            "cpu_port_inst_per_s": round(cr, 1), "cpu_threads": threads, "parity_sample_ok": ok}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="1,3,4,5")
    ap.add_argument("--n3", type=int, default=100_000)
    ap.add_argument("--n5", type=int, default=1_000_000)
    ap.add_argument("--k4", default="28,29,30,31,32")
    ap.add_argument("--per-k4", type=int, default=2)
    args = ap.parse_args()
    threads = os.cpu_count() or 1
    which = set(args.which.split(","))
    if "1" in which:
        print(json.dumps(config1(threads)), flush=True)
    if "5" in which:
        print(json.dumps(config5(threads, args.n5)), flush=True)
    if "3" in which:
        print(json.dumps(config3(threads, args.n3)), flush=True)
    if "4" in which:
        print(json.dumps(config4([int(k) for k in args.k4.split(",")], args.per_k4)), flush=True)


if __name__ == "__main__":
    main()
