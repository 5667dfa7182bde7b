"""The device log2 port (csrc/eb_exact.cuh) is bit-identical to the glibc log2
that CPython's math.log2 calls (reference radio.py:68).  CPU: the same source
compiled for the host against this libm; GPU twin in test_gpu_units.py."""
import ctypes
import math
import os
import random
import shutil
import subprocess

import pytest

from helpers import ROOT

CSRC = os.path.join(ROOT, "paper_2405_07140_b200", "csrc")


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("g++ not available")
    exe = str(tmp_path_factory.mktemp("log2") / "log2_check")
    subprocess.run([gxx, "-O2", "-ffp-contract=off", "-x", "c++", "-I", CSRC,
                    os.path.join(ROOT, "tests", "native", "log2_check.cpp"), "-o", exe, "-lm"], check=True)
    return exe


def test_port_bit_exact_vs_libm_10M(checker):
    out = subprocess.run([checker, "10000000", "7"], capture_output=True, text=True, check=True)
    assert out.stdout.strip() == "0", out.stderr[:2000]


def test_libm_is_what_cpython_calls():
    m = ctypes.CDLL("libm.so.6")
    m.log2.restype = ctypes.c_double
    m.log2.argtypes = [ctypes.c_double]
    rng = random.Random(5)
    for _ in range(20000):
        x = 1.0 + rng.expovariate(1.0) * 10 ** rng.uniform(-8, 14)
        assert m.log2(x) == math.log2(x)


def test_table_header_matches_this_libm(tmp_path):
    """The committed table is the one in this container's libm (regenerate + compare)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen", os.path.join(ROOT, "tools", "gen_log2_table.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    gen.OUT = str(tmp_path / "t.h")
    try:
        gen.main()
    except SystemExit as exc:
        pytest.skip(f"libm layout differs here: {exc}")
    committed = open(os.path.join(CSRC, "log2_glibc_table.h")).read().splitlines()[5:]
    fresh = open(gen.OUT).read().splitlines()[5:]
    assert committed == fresh
