"""The paper's simulator sweeps (reference acceptance criteria 4-6,
pkg/tests/test_acceptance.py:96-170), all scenarios in one lock-step run.

Criterion 4: DFTSP node-count reduction vs arrival rate (compare_pruning).
Criterion 5: DFTSP >= StB >= NoB throughput and BLOOM-3B >= BLOOM-7.1B over
             an arrival-rate sweep, with saturation at the top rates.
Criterion 6: quantization trends -- w4 >= w8 with accuracy ignored;
             throughput monotone in the tolerance cap, GPTQ >= ZQ-local.

``evaluate()`` builds exactly the reference's scenarios, runs them with
``sweep.run_many`` and applies the reference's assertions; it returns the
verdicts and the raw numbers.
"""
from __future__ import annotations

import time

from .sweep import Scenario, complexity_reduction, run_many

FAST = dict(epoch_s=0.5, uplink_slot_s=0.1, downlink_slot_s=0.1)


def scenarios() -> dict:
    """name -> Scenario for every run the three criteria make."""
    out = {}
    for rate in (10, 50, 100, 200):                                   # criterion 4
        out[("c4", rate)] = Scenario(arrival_rate=rate, duration=12.0, seed=0, compare_pruning=True)
    base = dict(duration=30.0, seed=5, **FAST)
    for model in ("bloom-3b", "bloom-7.1b"):                           # criterion 5
        for sched in ("dftsp", "stb", "nob"):
            for rate in (5, 10, 20, 40, 50, 60, 80):
                out[("c5", model, sched, rate)] = Scenario(model=model, scheduler=sched, arrival_rate=rate, **base)
    sat = dict(duration=30.0, seed=5, arrival_rate=40.0, accuracy_check=False, **FAST)
    for model in ("bloom-3b", "bloom-7.1b", "opt-13b"):               # criterion 6a
        for prof in ("w4a16-gptq", "w8a16"):
            out[("c6a", model, prof)] = Scenario(model=model, quant_profile=prof, **sat)
    for model, rate in (("bloom-3b", 20.0), ("opt-13b", 2.0)):        # criterion 6b
        for prof in ("w4a16-gptq", "w4a16-zq-local"):
            for cap in (0.0, 0.5, 0.8, 0.9, 1.0):
                out[("c6b", model, prof, cap)] = Scenario(model=model, quant_profile=prof, tolerance_cap=cap,
                                                         arrival_rate=rate, duration=40.0, seed=5, **FAST)
    return out


def evaluate(device=None) -> dict:
    scs = scenarios()
    keys = list(scs)
    t0 = time.perf_counter()
    res = run_many([scs[k] for k in keys], device=device)
    dt = time.perf_counter() - t0
    m = dict(zip(keys, res))
    errors = {str(k): v.error for k, v in m.items() if v.error}
    # criterion 4 (test_acceptance.py:96-111)
    reds = [complexity_reduction(m[("c4", r)].cmp_nodes_with_pruning, m[("c4", r)].cmp_nodes_without_pruning)
            for r in (10, 50, 100, 200)]
    c4 = all(a < b for a, b in zip(reds, reds[1:])) and reds[0] >= 30.0 and reds[-1] >= 80.0
    # criterion 5 (:114-135)
    rates = (5, 10, 20, 40, 50, 60, 80)
    thr = {k[1:]: v.throughput for k, v in m.items() if k[0] == "c5"}
    models = ("bloom-3b", "bloom-7.1b")
    sched_ok = all(thr[(mo, "dftsp", r)] >= thr[(mo, "stb", r)] >= thr[(mo, "nob", r)] for mo in models for r in rates)
    model_ok = all(thr[("bloom-3b", s, r)] >= thr[("bloom-7.1b", s, r)] for s in ("dftsp", "stb", "nob") for r in rates)
    top = [thr[("bloom-3b", "dftsp", r)] for r in rates[-3:]]
    sat_ok = all(abs(b - a) / max(a, b) < 0.05 for a, b in zip(top, top[1:]))
    c5 = sched_ok and model_ok and sat_ok
    # criterion 6 (:138-170)
    beta_ok = all(m[("c6a", mo, "w4a16-gptq")].throughput >= m[("c6a", mo, "w8a16")].throughput
                  for mo in ("bloom-3b", "bloom-7.1b", "opt-13b"))
    caps = (0.0, 0.5, 0.8, 0.9, 1.0)
    mono_ok = dom_ok = True
    curves = {}
    for mo in ("bloom-3b", "opt-13b"):
        for prof in ("w4a16-gptq", "w4a16-zq-local"):
            c = [m[("c6b", mo, prof, cap)].throughput for cap in caps]
            curves[f"{mo}/{prof}"] = c
            mono_ok = mono_ok and all(a <= b + 1e-12 for a, b in zip(c, c[1:]))
        dom_ok = dom_ok and all(z <= g + 1e-12 for g, z in zip(curves[f"{mo}/w4a16-gptq"],
                                                                 curves[f"{mo}/w4a16-zq-local"]))
    c6 = beta_ok and mono_ok and dom_ok
    return dict(seconds=dt, runs=len(keys), errors=errors, criterion_4=c4, criterion_5=c5, criterion_6=c6,
                reductions_pct=reds, top3=top, sched_ok=sched_ok, model_ok=model_ok, sat_ok=sat_ok,
                beta_ok=beta_ok, mono_ok=mono_ok, dom_ok=dom_ok, curves=curves,
                epochs=sum(len(v.trace) for v in res),
                nodes_visited=sum(v.nodes_visited_total for v in res),
                nodes_unpruned=sum(v.cmp_nodes_without_pruning or 0 for v in res))
