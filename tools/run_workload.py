#!/usr/bin/env python3
"""Solve one synthetic workload on the device (for ncu captures of non-headline
configs).  python tools/run_workload.py --K 40 --n 100000 [--config5]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]
from bench_configs import device_rates  # noqa: E402
from paper_2405_07140_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=40)
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--config5", action="store_true")
a = ap.parse_args()
if a.config5:
    w, lad = synth.CONFIG5, synth.CONFIG5.outputs
else:
    w, lad = synth.Workload(f"K={a.K}", profiles=("w8a16",), K=a.K), (128, 256, 512)
b = synth.generate(w, a.n, seed=11)
k, e = device_rates(b, lad, reps=2)
print(f"{w.name}: kernel {k / 1e6:.2f} M inst/s, wire e2e {e / 1e6:.2f} M inst/s")
