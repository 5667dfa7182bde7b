#!/usr/bin/env python3
"""Stage the unmodified Python reference into oracle/_ref/ (test infrastructure).

The reference (`edgebatch`, pure Python) cannot be compiled; its hot path is
the Python code itself.  This recipe copies the package sources verbatim from
/root/reference/pkg/src/edgebatch into oracle/_ref/edgebatch -- git-ignored
(never part of the repo's history) but NOT gpurun-ignored, so the copy travels
to the GPU box, where /root/reference does not exist.  There it is imported by
oracle/pyref.py as the reference CPU baseline (bench.py --impl reference and
the cpu_baseline leg) and by tests/test_gpu_compat.py to run the reference
simulator with and without the device drop-in.  A MANIFEST with each file's
sha256 records exactly what was staged.

Runs in the build container only (build() calls it when /root/reference is
present); on the GPU box the staged copy is used as is.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import sys

SRC = "/root/reference/pkg/src/edgebatch"
SCEN = "/root/reference/pkg/scenarios"
HERE = os.path.dirname(os.path.abspath(__file__))
DST = os.path.join(HERE, "_ref")


def stage(force: bool = False) -> str | None:
    if not os.path.isdir(SRC):
        return DST if os.path.isdir(os.path.join(DST, "edgebatch")) else None
    files = sorted(f for f in os.listdir(SRC) if f.endswith(".py"))
    manifest = []
    for f in files:
        with open(os.path.join(SRC, f), "rb") as fh:
            manifest.append(f"{hashlib.sha256(fh.read()).hexdigest()}  edgebatch/{f}")
    mpath = os.path.join(DST, "MANIFEST")
    text = "\n".join(manifest) + "\n"
    if not force and os.path.exists(mpath) and open(mpath).read() == text:
        return DST
    shutil.rmtree(DST, ignore_errors=True)
    os.makedirs(os.path.join(DST, "edgebatch"))
    for f in files:
        shutil.copy2(os.path.join(SRC, f), os.path.join(DST, "edgebatch", f))
    if os.path.isdir(SCEN):
        shutil.copytree(SCEN, os.path.join(DST, "scenarios"))
    with open(mpath, "w") as fh:
        fh.write(text)
    return DST


if __name__ == "__main__":
    print(stage(force="--force" in sys.argv))
