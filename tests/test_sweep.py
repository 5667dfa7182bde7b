"""Lock-step batched simulator (paper_2405_07140_b200.sweep) against runs of
the reference simulator (tests/golden/sim_runs.json, recorded from
edgebatch.sim.run by tests/golden/make_golden.py --sim-only).  CPU: the
device entry points are served by the oracle (tests/sweep_oracle.py), which
checks the simulator's host bookkeeping -- workload draws, expiry, waiting
times, completions, traces -- independently of the kernels."""
import dataclasses
import json
import os

import pytest

import sweep_oracle
from paper_2405_07140_b200 import sweep

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "sim_runs.json")


def load_runs():
    with open(GOLDEN) as fh:
        return json.load(fh)


def compare(got, exp):
    assert got.error is None, got.error
    for k, v in exp["metrics"].items():
        assert getattr(got, k) == v, f"metric {k}: {getattr(got, k)} != {v}"
    assert len(got.trace) == len(exp["trace"])
    for row_g, row_e in zip(got.trace, exp["trace"]):
        assert dataclasses.asdict(row_g) == row_e, f"epoch {row_e['epoch']}: {row_g} != {row_e}"


def test_workload_draws_match_reference():
    for run in load_runs():
        sc = sweep.Scenario.from_mapping(run["scenario"])
        import numpy as np
        w = sweep.generate_workload(sc, np.random.default_rng([sc.seed, 11]))
        assert len(w) == run["metrics"]["generated"]


def test_workload_fast_draws_equal_numpy_calls():
    """generate_workload's cheaper calls consume the PCG64 stream exactly as
    the reference's rng.choice / rng.uniform do (sim.py:248-252)."""
    import numpy as np
    sc = sweep.Scenario(seed=3, duration=30.0, prompt_choices=(7, 100, 2000, 9), output_classes=(1, 5, 64))
    fast = sweep.generate_workload(sc, np.random.default_rng([3, 11]))
    rng = np.random.default_rng([3, 11])
    t, ref = 0.0, []
    while True:
        t += rng.exponential(1.0 / sc.arrival_rate)
        if t >= sc.duration:
            break
        ref.append((t, int(rng.choice(sc.prompt_choices)), int(rng.choice(sc.output_classes)),
                    sc.deadline_scale * float(rng.uniform(*sc.deadline_range_s)),
                    sc.tolerance_cap * float(rng.uniform(0.0, 1.0)), float(rng.exponential(sc.mean_channel_gain))))
    got = [(r.arrival_s, r.prompt_tokens, r.output_tokens, r.deadline_s, r.tolerance, r.link.channel_gain) for r in fast]
    assert got == ref


def test_sweep_host_logic_matches_reference_runs(monkeypatch):
    sweep_oracle.install(monkeypatch)
    runs = load_runs()
    got = sweep.run_many([r["scenario"] for r in runs])
    for g, e in zip(got, runs):
        compare(g, e)


def test_sweep_runs_are_independent(monkeypatch):
    """A run's result does not depend on which other runs share its lock-step."""
    sweep_oracle.install(monkeypatch)
    runs = load_runs()
    alone = sweep.run_many([runs[5]["scenario"]])[0]
    compare(alone, runs[5])


def test_sweep_errors_stay_per_run(monkeypatch):
    sweep_oracle.install(monkeypatch)
    runs = load_runs()
    bad = dict(runs[5]["scenario"], oracle_cap=2)            # brute refuses > 2 candidates
    invalid = dict(runs[0]["scenario"], epoch_s=0.1)         # slots do not fit the epoch
    got = sweep.run_many([bad, runs[1]["scenario"], invalid])
    assert got[0].error.startswith("ConfigError: scheduler: brute refuses")
    assert isinstance(got[0].exception, sweep.ConfigError)
    assert got[2].error == "ConfigError: epoch_s: must fit the uplink and downlink slots"
    compare(got[1], runs[1])


def test_scenario_validation_messages():
    with pytest.raises(sweep.ConfigError, match="scheduler: must be one of"):
        sweep.Scenario(scheduler="fifo").validate()
    with pytest.raises(sweep.ConfigError, match="model/quant_profile"):
        sweep.Scenario(model="nope").validate()
    with pytest.raises(sweep.ConfigError, match="deadline_range_s"):
        sweep.Scenario(deadline_range_s=(2.0, 1.0)).validate()


SWEEPS = os.path.join(os.path.dirname(__file__), "golden", "sim_sweeps.json")


def load_sweeps():
    with open(SWEEPS) as fh:
        return json.load(fh)


def check_sweeps(tmp_path):
    """sweep.run_sweep + emit against the reference's cli.run_sweep tables and bytes."""
    d = load_sweeps()
    for k, case in enumerate(d["sweeps"]):
        sc = sweep.Scenario.from_mapping(case["scenario"])
        table = sweep.run_sweep(sc, sweep.SweepSpec(case["axis"], tuple(case["values"]), case["repetitions"]))
        assert len(table) == len(case["rows"])
        for got, exp in zip(table, case["rows"]):
            assert got == exp, f"sweep {k}: {got} != {exp}"
        sweep.emit(table, "csv", tmp_path / f"{k}.csv")
        sweep.emit(table, "json", tmp_path / f"{k}.json")
        assert (tmp_path / f"{k}.csv").read_text() == case["csv"]
        assert (tmp_path / f"{k}.json").read_text() == case["json"]
    tr = d["trace_run"]
    m = sweep.run(sweep.Scenario.from_mapping(tr["scenario"]))
    sweep.emit_trace(m, tmp_path / "trace.csv")
    assert (tmp_path / "trace.csv").read_text() == tr["csv"]


def test_sweep_tables_and_emission_match_reference(monkeypatch, tmp_path):
    sweep_oracle.install(monkeypatch)
    check_sweeps(tmp_path)


def test_config_hash_matches_reference():
    for case in load_sweeps()["sweeps"]:
        sc = sweep.Scenario.from_mapping(case["scenario"])
        data_rows = [r for r in case["rows"] if r["kind"] == "data"]
        assert any(sweep.config_hash(sweep.apply_axis(sc, case["axis"], r["value"])) == r["config_hash"]
                   for r in data_rows)
