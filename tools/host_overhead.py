#!/usr/bin/env python3
"""Per-call and per-chunk host overhead of the host-memory DFTSP pipeline:
wall time of eb_dftsp_batch_packed (pinned buffers) vs the device-resident
kernel on config-2 batches of growing size."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]
from bench_configs import device_rates  # noqa: E402
from paper_2405_07140_b200 import synth  # noqa: E402

for n in (2048, 8192, 16384, 32768, 100000, 400000):
    b = synth.generate(synth.CONFIG2, n, seed=3)
    k, e = device_rates(b, (128, 256, 512), reps=5)
    print(f"n={n:7d} kernel {n / k * 1e3:8.3f} ms   wire e2e {n / e * 1e3:8.3f} ms   "
          f"overhead {(n / e - n / k) * 1e3:7.3f} ms", flush=True)
