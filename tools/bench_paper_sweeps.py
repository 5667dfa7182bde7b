"""Reference acceptance criteria 4-6 (the paper's simulator sweeps) in one
lock-step run on the device; prints one JSON line with verdicts and time.

    python tools/bench_paper_sweeps.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2405_07140_b200 import _lib, paper_sweeps  # noqa: E402

if __name__ == "__main__":
    h = _lib.handle()
    l0 = h.launches()
    r = paper_sweeps.evaluate()
    r["launches"] = h.launches() - l0
    print(json.dumps(r))
