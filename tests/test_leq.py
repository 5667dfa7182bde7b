"""The device leq (csrc/eb_exact.cuh: integer max(1, |a|, |b|) scale) equals
the reference's leq (feasibility.py:28-30) on every input, NaN/inf/signed
zero/subnormal included, and so does the margin form the search bounds use.
CPU: the same header compiled for the host."""
import os
import shutil
import subprocess

import pytest

from helpers import ROOT

CSRC = os.path.join(ROOT, "paper_2405_07140_b200", "csrc")


def test_leq_scale_matches_python_max(tmp_path):
    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("g++ not available")
    exe = str(tmp_path / "leq_check")
    subprocess.run([gxx, "-O2", "-ffp-contract=off", "-x", "c++", "-I", CSRC,
                    os.path.join(ROOT, "tests", "native", "leq_check.cpp"), "-o", exe, "-lm"], check=True)
    out = subprocess.run([exe, "20000000", "3"], capture_output=True, text=True, check=True)
    assert out.stdout.strip() == "0", out.stderr[:2000]
