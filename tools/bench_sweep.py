"""Throughput of the lock-step batched simulator (paper_2405_07140_b200.sweep).

    python tools/bench_sweep.py --runs 256            # device path (B200)
    python tools/bench_sweep.py --reference --runs 4  # reference sim.run, this container only

Workload: ``--runs`` seeds of one scenario (paper defaults: BLOOM-3B / W8A16,
50 req/s, 20 s, 2 s epochs, DFTSP) -- the seed sweep behind the paper's
throughput figures.  The device number is wall clock around run_many (the
simulator is host-driven: per epoch, host bookkeeping + one batched launch
per entry point), so it includes every host cost.  The reference number is
edgebatch.sim.run on one core, per run.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def scenarios(n, **over):
    base = dict(seed=0)
    base.update(over)
    return [dict(base, seed=s) for s in range(n)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=256)
    ap.add_argument("--duration", type=float, default=20.0)
    ap.add_argument("--rate", type=float, default=50.0)
    ap.add_argument("--scheduler", default="dftsp")
    ap.add_argument("--set", action="append", default=[], help="extra scenario field, key=value (JSON value)")
    ap.add_argument("--reference", action="store_true")
    a = ap.parse_args()
    extra = {k: json.loads(v) for k, v in (kv.split("=", 1) for kv in a.set)}
    scs = scenarios(a.runs, duration=a.duration, arrival_rate=a.rate, scheduler=a.scheduler, **extra)
    if a.reference:
        sys.path.insert(0, "/root/reference/pkg/src")
        from edgebatch import sim
        t = time.perf_counter()
        done = 0
        for s in scs:
            sim.run(sim.Scenario(**s))
            done += 1
        dt = time.perf_counter() - t
        print(json.dumps(dict(impl="reference sim.run (1 core)", runs=done, seconds=round(dt, 3),
                              runs_per_s=done / dt, scenario=scs[0])))
        return
    from paper_2405_07140_b200 import _lib, sweep
    h = _lib.handle()
    sweep.run_many(scs[:2])                                    # warm-up: library load, first launches
    l0 = h.launches()
    t = time.perf_counter()
    prof = {}
    out = sweep.run_many(scs, profile=prof)
    dt = time.perf_counter() - t
    errs = sum(o.error is not None for o in out)
    epochs = sum(len(o.trace) for o in out)
    print(json.dumps(dict(impl="sweep.run_many (lock-step, device)", runs=len(out), errors=errs,
                          seconds=round(dt, 3), runs_per_s=len(out) / dt, epochs=epochs,
                          dftsp_instances=epochs,
                          launches=h.launches() - l0,
                          completed_mean=sum(o.completed_total for o in out) / max(len(out), 1),
                          phases_s={k: round(v, 3) for k, v in sorted(prof.items())},
                          scenario=scs[0])))


if __name__ == "__main__":
    main()
