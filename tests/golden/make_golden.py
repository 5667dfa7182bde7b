#!/usr/bin/env python3
"""Generate golden fixtures by running the REFERENCE implementation itself.

Runs only in the build container, where the read-only reference lives at
/root/reference (pure Python package `edgebatch`, imported from
pkg/src; its own test helper `conftest.random_instance` from pkg/tests).
The fixtures (small .npz files next to this script) travel with the repo;
the GPU box never reads /root/reference.

Corpora (one .npz each):
  random_<seed>   conftest.random_instance corpora with the reference test
                  suite's seeds (2024, 31, 32, 33, 34, 35 slot-cap, 1001, 77);
                  flag sets P / NP / PI / PE / NL; exhaustive subsets mode
  scenario        per-epoch candidate pools captured from edgebatch.sim.run on
                  pkg/scenarios/*.yaml at several arrival rates / seeds
  config2         SURVEY Appendix D generator, K=20, fp16/w8a16/w4a16 mix
  config5         tight-memory OPT-13B edge, 5 output classes, K=20
  ksweep          K in {10, 25, 30, 40}, varied deadline/tolerance scales
  units           check_direct / check_knapsack / coefficients / batch_cost /
                  static_batch_size / stb / nob / link-math goldens

Usage:  python tests/golden/make_golden.py [--quick]
"""
from __future__ import annotations

import dataclasses
import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [REF_SRC, REF_TESTS, ROOT]

import edgebatch as eb  # noqa: E402  (the reference)
from conftest import random_instance, random_subset  # noqa: E402  (reference test helper)

from paper_2405_07140_b200._lib import CTX_DTYPE  # noqa: E402  (record layout only)

MAXC = 16
FLAGSETS = {
    "P": dict(pruning=True),
    "NP": dict(pruning=False),
    "PI": dict(pruning=True, inclusive_bound=True),
    "PE": dict(pruning=True, exact_tau=True),
}


def ctx_rec(ctx, delta=0.0):
    rec = np.zeros(1, dtype=CTX_DTYPE)
    l, q, r, n = ctx.llm, ctx.quant, ctx.radio, ctx.node
    for k in ("layers", "hidden_dim", "head_count", "head_dim", "ffn_dim", "bytes_per_param"):
        rec[k] = getattr(l, k)
    rec["alpha"], rec["beta"], rec["delta_ppl"] = q.alpha, q.beta, delta
    for k in ("uplink_band_hz", "downlink_band_hz", "downlink_power_w", "noise_density_w_hz", "uplink_slot_s",
              "downlink_slot_s"):
        rec[k] = getattr(r, k)
    rec["bits_per_token"] = r.bits_per_token
    rec["flops_per_s"], rec["memory_bytes"], rec["gpu_count"] = n.flops_per_s, n.memory_bytes, n.gpu_count
    rec["has_slot_cap"] = ctx.slot_cap_s is not None
    rec["slot_cap_s"] = ctx.slot_cap_s or 0.0
    return rec


COLS = (("id", np.int64), ("prompt_tokens", np.int32), ("output_tokens", np.int32), ("deadline_s", np.float64),
        ("waiting_s", np.float64), ("tolerance", np.float64), ("channel_gain", np.float64),
        ("uplink_power_w", np.float64))


def pack(instances):
    """instances: list of (ctx, ladder|None, requests).  Returns dict of arrays."""
    ctxs, ctx_index, offsets, ladders, rows = [], [], [0], [], []
    ctx_ids = {}
    for ctx, ladder, reqs in instances:
        key = id(ctx)
        if key not in ctx_ids:
            ctx_ids[key] = len(ctxs)
            ctxs.append(ctx_rec(ctx))
        ctx_index.append(ctx_ids[key])
        rows.extend(reqs)
        offsets.append(len(rows))
        lad = np.zeros(MAXC + 1, np.int32)
        if ladder is not None:
            vals = sorted(set(ladder))
            lad[0] = len(vals)
            lad[1:1 + len(vals)] = vals
        else:
            lad[0] = -1
        ladders.append(lad)
    out = {"ctx": np.concatenate(ctxs) if ctxs else np.zeros(0, CTX_DTYPE),
           "ctx_index": np.array(ctx_index, np.int32), "offsets": np.array(offsets, np.int64),
           "ladder": np.array(ladders, np.int32).reshape(-1, MAXC + 1)}
    for name, dt in COLS:
        if name == "channel_gain":
            vals = [r.link.channel_gain for r in rows]
        elif name == "uplink_power_w":
            vals = [r.link.uplink_power_w for r in rows]
        else:
            vals = [getattr(r, name) for r in rows]
        out["req_" + name] = np.array(vals, dtype=dt)
    return out


STATUS = {"ok": 0, "weights": 10, "uplink": 11, "downlink": 12, "ladder": 13, "reverify": 14}


def run_dftsp(instances, tag, flags, use_ladder=True, traj=False):
    """Reference dftsp on each instance: arrays prefixed with tag."""
    n = len(instances)
    nreq = sum(len(r) for _, _, r in instances)
    st = np.zeros(n, np.int32); z = np.zeros(n, np.int32); vis = np.zeros(n, np.int64)
    prn = np.zeros(n, np.int64); ncl = np.zeros(n, np.int32); cnt = np.zeros((n, MAXC), np.int32)
    sol = np.full(max(nreq, 1), -1, np.int32)
    trajs = []
    row = 0
    for i, (ctx, ladder, reqs) in enumerate(instances):
        try:
            out = eb.dftsp(reqs, ctx, ladder=ladder if use_ladder else None, collect_trajectory=traj, **flags)
        except eb.WeightsDoNotFitError:
            st[i] = STATUS["weights"]
        except RuntimeError:
            st[i] = STATUS["reverify"]
        except ValueError as exc:
            msg = str(exc)
            st[i] = STATUS["ladder"] if "ladder" in msg else STATUS["uplink"] if "uplink" in msg else \
                STATUS["downlink"] if "downlink" in msg else 99
        else:
            z[i], vis[i], prn[i] = out.z_found, out.nodes_visited, out.nodes_pruned
            ncl[i] = len(out.counts)
            cnt[i, :len(out.counts)] = out.counts
            if out.solution:
                idx = {id(r): j for j, r in enumerate(reqs)}
                sol[row:row + len(out.solution)] = [idx[id(r)] for r in out.solution]
            if traj:
                trajs.append(np.array(out.trajectory, np.int64).reshape(-1, 4))
        row += len(reqs)
    res = {f"{tag}_status": st, f"{tag}_z": z, f"{tag}_visited": vis, f"{tag}_pruned": prn,
           f"{tag}_ncls": ncl, f"{tag}_counts": cnt, f"{tag}_solution": sol}
    if traj:
        lens = np.array([len(t) for t in trajs], np.int64)
        res[f"{tag}_traj_len"] = lens
        res[f"{tag}_traj"] = np.concatenate(trajs) if trajs else np.zeros((0, 4), np.int64)
    return res


def run_exhaustive(instances, cap=16):
    n = len(instances)
    z = np.zeros(n, np.int32); nodes = np.zeros(n, np.int64); mask = np.zeros(n, np.uint64)
    st = np.zeros(n, np.int32)
    for i, (ctx, _, reqs) in enumerate(instances):
        if len(reqs) > cap:
            st[i] = 16
            continue
        try:
            out = eb.exhaustive_optimal(reqs, ctx, cap=cap)
        except ValueError as exc:
            st[i] = STATUS["uplink"] if "uplink" in str(exc) else STATUS["downlink"] if "downlink" in str(exc) else 99
            continue
        z[i], nodes[i] = out.z_found, out.nodes_visited
        if out.solution:
            idx = {id(r): j for j, r in enumerate(reqs)}
            m = 0
            for r in out.solution:
                m |= 1 << idx[id(r)]
            mask[i] = m
    return {"ex_status": st, "ex_z": z, "ex_nodes": nodes, "ex_mask": mask}


def run_exhaustive_counts(instances, cap=64):
    """Reference exhaustive_optimal(mode="counts") (dftsp.py:316-332)."""
    n = len(instances)
    nreq = sum(len(r) for _, _, r in instances)
    st = np.zeros(n, np.int32); z = np.zeros(n, np.int32); nodes = np.zeros(n, np.int64)
    sol = np.full(max(nreq, 1), -1, np.int32)
    row = 0
    for i, (ctx, ladder, reqs) in enumerate(instances):
        try:
            out = eb.exhaustive_optimal(reqs, ctx, cap=cap, mode="counts", ladder=ladder)
        except RuntimeError:
            st[i] = STATUS["reverify"]
        except ValueError as exc:
            msg = str(exc)
            st[i] = STATUS["ladder"] if "ladder" in msg else STATUS["uplink"] if "uplink" in msg else \
                STATUS["downlink"] if "downlink" in msg else 99
        else:
            z[i], nodes[i] = out.z_found, out.nodes_visited
            if out.solution:
                idx = {id(r): j for j, r in enumerate(reqs)}
                sol[row:row + len(out.solution)] = [idx[id(r)] for r in out.solution]
        row += len(reqs)
    return {"exc_status": st, "exc_z": z, "exc_nodes": nodes, "exc_solution": sol}


def save(name, data, meta):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **data)
    meta_path = os.path.join(HERE, f"{name}.json")
    with open(meta_path, "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(f"  {name}: {os.path.getsize(path) / 1024:.1f} KiB, {meta.get('n_inst')} instances")


# --------------------------------------------------------------------------
def corpus_random(seed, count, flagsets=("P", "NP", "PI", "PE", "NL"), exhaustive=True, traj=False, counts=False,
                  **kw):
    rng = np.random.default_rng(seed)
    inst = [random_instance(rng, **kw) for _ in range(count)]
    inst = [(ctx, ladder, reqs) for ladder, ctx, reqs in inst]
    data = pack(inst)
    for tag in flagsets:
        if tag == "NL":
            data.update(run_dftsp(inst, "NL", FLAGSETS["P"], use_ladder=False, traj=traj))
        else:
            data.update(run_dftsp(inst, tag, FLAGSETS[tag], traj=traj and tag == "P"))
    if exhaustive:
        data.update(run_exhaustive(inst))
    if counts:
        data.update(run_exhaustive_counts(inst))
    save(f"random_{seed}", data, {"n_inst": len(inst), "seed": seed, "generator": "conftest.random_instance",
                                  "kwargs": kw, "flagsets": list(flagsets)})


def corpus_scenarios(quick):
    from edgebatch import cli, sim
    captured = []
    orig = sim.dftsp

    def hook(cands, ctx, **kw):
        captured.append((ctx, kw.get("ladder"), list(cands), dict(kw)))
        return orig(cands, ctx, **kw)

    sim.dftsp = hook
    try:
        files = ["default.yaml", "throughput.yaml"]
        rates = [2, 5, 8, 10, 15, 20, 50] if not quick else [5, 20]
        for f in files:
            base = cli.parse_scenario(os.path.join("/root/reference/pkg/scenarios", f))
            for rate in rates:
                for seed in (0, 1):
                    sc = dataclasses.replace(base, arrival_rate=float(rate), seed=seed,
                                             duration=min(base.duration, 12.0), compare_pruning=False)
                    sim.run(sc)
    finally:
        sim.dftsp = orig
    # keep pools of moderate size (the golden must stay small); dedupe empties
    inst = [(c, lad, reqs) for c, lad, reqs, _ in captured if 0 < len(reqs) <= 48][:400]
    data = pack(inst)
    data.update(run_dftsp(inst, "P", FLAGSETS["P"]))
    data.update(run_exhaustive(inst, cap=12))
    save("scenario", data, {"n_inst": len(inst), "source": "edgebatch.sim.run on pkg/scenarios default/throughput",
                            "rates": rates})


def appendix_d(rng_seed, count, K, model="bloom-3b", profiles=("fp16", "w8a16", "w4a16-gptq"),
               prompts=(128, 256, 512), outputs=(128, 256, 512), gpu_count=20, flops_per_gpu=1.33e12,
               mem_per_gpu=32e9, deadline=(0.5, 2.0), deadline_scale=1.0, tol_cap=1.0, epoch=2.0):
    """SURVEY Appendix D generator: draw until K requests pass sim._dftsp_candidates."""
    llm = eb.get_model(model)
    radio = eb.RadioConfig(20e6, 20e6, eb.dbm_to_watts(43.0), eb.dbm_to_watts(-174.0), 0.25, 0.25)
    node = eb.NodeCompute(gpu_count * flops_per_gpu, gpu_count * mem_per_gpu, gpu_count)
    ctxs = {p: eb.EdgeContext(llm, eb.get_profile(p), radio, node, slot_cap_s=epoch) for p in profiles}
    p_up = eb.dbm_to_watts(20.0)
    out = []
    for i in range(count):
        rng = np.random.default_rng([rng_seed, i])
        prof = profiles[int(rng.integers(len(profiles)))]
        ctx = ctxs[prof]
        delta = eb.delta_ppl(ctx.quant, llm.name)
        reqs = []
        j = 0
        while len(reqs) < K:
            r = eb.Request(id=len(reqs), prompt_tokens=int(rng.choice(prompts)), output_tokens=int(rng.choice(outputs)),
                           deadline_s=deadline_scale * float(rng.uniform(*deadline)),
                           tolerance=tol_cap * float(rng.uniform(0.0, 1.0)),
                           link=eb.UserLink(float(rng.exponential(1e-3)), p_up),
                           waiting_s=float(rng.uniform(0.0, epoch)))
            j += 1
            if delta <= r.tolerance and eb.check_direct((r,), ctx, r.prompt_tokens):
                reqs.append(r)
            if j > 100000:
                break
        out.append((ctx, tuple(outputs), reqs))
    return out


def corpus_config2(count):
    inst = appendix_d(2405_07140, count, 20)
    data = pack(inst)
    t = time.time()
    data.update(run_dftsp(inst, "P", FLAGSETS["P"]))
    print(f"    reference dftsp: {(time.time() - t) / count * 1e3:.2f} ms/instance")
    save("config2", data, {"n_inst": len(inst), "K": 20, "generator": "SURVEY Appendix D, seed 2405_07140"})


def corpus_config5(count):
    inst = appendix_d(2405_07141, count, 20, model="opt-13b", profiles=("w4a16-gptq",), prompts=(512, 1024, 2048),
                      outputs=(64, 128, 256, 512, 1024), gpu_count=1, flops_per_gpu=2.0e15, mem_per_gpu=1.08e10)
    data = pack(inst)
    data.update(run_dftsp(inst, "P", FLAGSETS["P"]))
    save("config5", data, {"n_inst": len(inst), "K": 20, "generator": "Appendix D, OPT-13B tight memory"})


def corpus_ksweep(per_k):
    inst = []
    for K in (10, 25, 30, 40):
        for ds, tc in ((0.5, 0.25), (1.0, 1.0), (2.0, 0.5)):
            inst += appendix_d(2405_07142 + K, per_k, K, profiles=("w8a16",), deadline_scale=ds, tol_cap=tc)
    data = pack(inst)
    data.update(run_dftsp(inst, "P", FLAGSETS["P"]))
    save("ksweep", data, {"n_inst": len(inst), "K": [10, 25, 30, 40]})


def _wide_instances():
    inst = []
    for K in (65, 96, 128):
        for ds, tc in ((0.5, 0.25), (1.0, 1.0), (2.0, 0.5)):
            inst += appendix_d(2405_07150 + K, 2, K, profiles=("w8a16", "fp16"), deadline_scale=ds, tol_cap=tc)
    inst += appendix_d(2405_07151, 1, 200, profiles=("w8a16",), deadline_scale=0.5, tol_cap=1.0)
    inst += appendix_d(2405_07152, 1, 255, profiles=("w8a16",), deadline_scale=0.3, tol_cap=1.0)
    return inst


def corpus_wide(parts=("wide", "wide_np")):
    """Instances wider than EB_MAX_K (64): the device's wide pass, up to EB_MAX_K_DFTSP (255).
    ``wide``: P/PI/PE on K = 65..255; ``wide_np``: the unpruned search on the K = 65 ones."""
    inst = _wide_instances()
    t = time.time()
    if "wide" in parts:
        data = pack(inst)
        for tag in ("P", "PI", "PE"):
            data.update(run_dftsp(inst, tag, FLAGSETS[tag]))
        save("wide", data, {"n_inst": len(inst), "K": [65, 96, 128, 200, 255], "generator": "Appendix D, K > 64"})
    if "wide_np" in parts:
        small = [x for x in inst if len(x[2]) <= 65]
        data = pack(small)
        data.update(run_dftsp(small, "NP", FLAGSETS["NP"]))
        save("wide_np", data, {"n_inst": len(small), "K": [65], "generator": "Appendix D, K = 65, unpruned"})
    print(f"    wide corpora: {time.time() - t:.0f} s")


def corpus_units():
    """Subset-level goldens: check_direct/check_knapsack/coefficients/batch_cost on random instances."""
    rng = np.random.default_rng(42)
    subsets = []   # (instance idx, member local indices, z, tau_min)
    inst = []
    for _ in range(120):
        ladder, ctx, reqs = random_instance(rng, slot_cap_s=1.0 if rng.random() < 0.3 else None)
        if not reqs:
            continue
        inst.append((ctx, ladder, reqs))
        i = len(inst) - 1
        pad = max(r.prompt_tokens for r in reqs)
        co = eb.derive_coefficients(ctx, pad, reqs)
        for _ in range(8):
            sub = random_subset(rng, reqs)
            z = len(sub)
            if z == 0:
                continue
            tau_min = min(co.tau_budget(r, z) for r in sub)
            idx = {id(r): j for j, r in enumerate(reqs)}
            subsets.append((i, [idx[id(r)] for r in sub], z, tau_min,
                            eb.check_direct(sub, ctx, pad), eb.check_knapsack(sub, co, z, tau_min)))
    data = pack(inst)
    sub_off = np.zeros(len(subsets) + 1, np.int64)
    np.cumsum([len(s[1]) for s in subsets], out=sub_off[1:])
    data["sub_inst"] = np.array([s[0] for s in subsets], np.int32)
    data["sub_members"] = np.array([m for s in subsets for m in s[1]], np.int32)
    data["sub_off"] = sub_off
    data["sub_tau_min"] = np.array([s[3] for s in subsets], np.float64)
    data["sub_direct"] = np.array([s[4] for s in subsets], np.uint8)
    data["sub_knapsack"] = np.array([s[5] for s in subsets], np.uint8)
    # coefficients per instance at pool padding
    coef = np.zeros((len(inst), 4)); kreq = []
    lat = []
    for i, (ctx, _, reqs) in enumerate(inst):
        pad = max(r.prompt_tokens for r in reqs)
        co = eb.derive_coefficients(ctx, pad, reqs)
        coef[i] = (co.k2, co.k3, co.k4, co.k5)
        for r in reqs:
            kreq.append((co.k_up[r.id], co.k_down[r.id], co.tau_base(r),
                         eb.min_uplink_fraction(r.prompt_tokens, r.link, ctx.radio),
                         eb.spectral_efficiency(r.link.uplink_power_w, r.link.channel_gain, ctx.radio.uplink_noise_w)))
        plan = eb.BatchPlan(tuple((r.prompt_tokens, r.output_tokens) for r in reqs), pad)
        c = eb.batch_cost(ctx.llm, ctx.quant, plan, ctx.node)
        lat.append((c.memory_bytes, c.latency_s))
    data["coef"] = coef
    data["coef_req"] = np.array(kreq, np.float64)
    data["batch_cost"] = np.array(lat, np.float64)
    save("units", data, {"n_inst": len(inst), "n_sub": len(subsets), "seed": 42})


SIM_CASES = [
    ("default.yaml", dict(seed=0, arrival_rate=50.0, duration=12.0)),
    ("default.yaml", dict(seed=1, arrival_rate=10.0, duration=12.0, compare_pruning=True)),
    ("throughput.yaml", dict(duration=10.0)),
    ("default.yaml", dict(seed=2, arrival_rate=30.0, duration=12.0, scheduler="stb", deadline_scale=3.0)),
    ("default.yaml", dict(seed=3, arrival_rate=30.0, duration=12.0, scheduler="nob", deadline_scale=3.0)),
    ("default.yaml", dict(seed=4, arrival_rate=5.0, duration=12.0, scheduler="brute")),
    ("default.yaml", dict(seed=5, arrival_rate=20.0, duration=12.0, verify_oracle=True)),
    ("default.yaml", dict(seed=6, arrival_rate=40.0, duration=12.0, exact_tau=True, inclusive_prune_bound=True)),
    ("default.yaml", dict(seed=7, arrival_rate=40.0, duration=12.0, channel_mode="shared")),
    ("default.yaml", dict(seed=8, arrival_rate=50.0, duration=12.0, quant_profile="w4a16-gptq", tolerance_cap=1.0)),
    ("default.yaml", dict(seed=9, arrival_rate=30.0, duration=12.0, model="opt-13b", deadline_scale=2.0)),
    ("default.yaml", dict(seed=10, arrival_rate=60.0, duration=8.0, admission_prefilter=False, accuracy_check=False)),
]


def corpus_sim():
    """Reference simulator runs (edgebatch.sim.run) for the lock-step batched runner's parity."""
    from edgebatch import cli, sim
    out = []
    for fname, over in SIM_CASES:
        base = cli.parse_scenario(os.path.join("/root/reference/pkg/scenarios", fname))
        sc = dataclasses.replace(base, **over)
        m = sim.run(sc)
        metrics = {f.name: getattr(m, f.name) for f in dataclasses.fields(m) if f.name != "trace"}
        trace = [dataclasses.asdict(t) for t in m.trace]
        scd = dataclasses.asdict(sc)
        out.append({"scenario": scd, "metrics": metrics, "trace": trace})
    with open(os.path.join(HERE, "sim_runs.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
    print(f"  sim_runs: {len(out)} runs")


SWEEP_CASES = [
    (dict(duration=8.0, epoch_s=0.5, uplink_slot_s=0.1, downlink_slot_s=0.1), ("arrival_rate", (5, 20, 40), 2)),
    (dict(duration=8.0, epoch_s=0.5, uplink_slot_s=0.1, downlink_slot_s=0.1, arrival_rate=6.0, seed=3),
     ("scheduler", ("dftsp", "stb", "nob", "brute"), 2)),
    (dict(duration=10.0, arrival_rate=20.0, compare_pruning=True, seed=7),
     ("quant_profile", ("fp16", "w8a16", "w4a16-gptq"), 1)),
    (dict(duration=10.0, arrival_rate=30.0, seed=11), ("deadline_scale", (0.5, 1.0, 2.0), 2)),
    (dict(duration=10.0, arrival_rate=15.0, seed=2), ("model", ("bloom-3b", "opt-13b", "nope-1b"), 1)),
]


def corpus_sweeps():
    """Reference cli.run_sweep tables + emitted bytes, for sweep.run_sweep / emit parity."""
    import dataclasses
    import tempfile
    from edgebatch import cli, sim
    out = []
    for over, (axis, values, reps) in SWEEP_CASES:
        sc = dataclasses.replace(sim.Scenario(), **over)
        table = cli.run_sweep(sc, cli.SweepSpec(axis, tuple(values), reps))
        with tempfile.TemporaryDirectory() as d:
            cli.emit(table, "csv", f"{d}/t.csv")
            cli.emit(table, "json", f"{d}/t.json")
            csv_text = open(f"{d}/t.csv").read()
            json_text = open(f"{d}/t.json").read()
        out.append({"scenario": sim.resolved_mapping(sc), "axis": axis, "values": list(values), "repetitions": reps,
                    "rows": table, "csv": csv_text, "json": json_text})
    sc = dataclasses.replace(sim.Scenario(), duration=8.0, arrival_rate=25.0, compare_pruning=True, seed=4)
    m = sim.run(sc)
    with tempfile.TemporaryDirectory() as d:
        cli.emit_trace(m, f"{d}/trace.csv")
        trace_text = open(f"{d}/trace.csv").read()
    with open(os.path.join(HERE, "sim_sweeps.json"), "w") as fh:
        json.dump({"sweeps": out, "trace_run": {"scenario": sim.resolved_mapping(sc), "csv": trace_text}}, fh,
                  indent=0, sort_keys=True)
    print(f"  sim_sweeps: {len(out)} sweeps")


def main():
    quick = "--quick" in sys.argv
    if "--sim-only" in sys.argv:
        corpus_sim()
        corpus_sweeps()
        return
    if "--wide-only" in sys.argv:
        corpus_wide(tuple(a for a in sys.argv[2:] if not a.startswith("--")) or ("wide", "wide_np"))
        return
    t0 = time.time()
    corpus_random(2024, 200, counts=True)
    corpus_random(31, 120)
    corpus_random(32, 80, max_requests=12)
    corpus_random(33, 80, max_requests=12)
    corpus_random(34, 20, min_requests=6, max_requests=12, traj=True, flagsets=("P", "NL"))
    corpus_random(35, 100, slot_cap_s=1.0)
    corpus_random(1001, 200)
    corpus_random(77, 60, max_requests=9, counts=True)
    corpus_units()
    corpus_scenarios(quick)
    corpus_config2(60 if quick else 300)
    corpus_config5(20 if quick else 60)
    corpus_ksweep(2 if quick else 4)
    corpus_wide()
    corpus_sim()
    corpus_sweeps()
    print(f"done in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
