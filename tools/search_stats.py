#!/usr/bin/env python3
"""Search statistics of the leaf-parallel DFTSP kernel on a workload (debug
build with -DEB_STATS; not the product library).  Builds
build/stats/libedgebatch_b200.so, runs N config-2 instances and prints per
instance: windows, windows with live leaves, leaf batches, leaves, U-table
builds, live calls, calls in sequence up to the winner.
  python tools/search_stats.py [--build-only] [--exact] [--config5] [N]"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "stats", "libedgebatch_b200.so")


def build():
    from paper_2405_07140_b200 import _build
    import glob
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(_build.CSRC, "*.cu")))
    cmd = [_build._nvcc(), *_build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-shared", "-DEB_STATS",
           "-Xcompiler", "-fPIC,-ffp-contract=off", "-I", os.path.join(ROOT, "include"), "-o", OUT, *srcs]
    subprocess.run(cmd, check=True)


def main():
    if "--build-only" in sys.argv:
        build()
        return
    n = int(sys.argv[-1]) if sys.argv[-1].isdigit() else 100_000
    from paper_2405_07140_b200 import _lib, search, synth
    _lib.LIB_PATH = OUT
    lib = _lib.load()
    lib.eb_debug_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
    w = synth.CONFIG5 if "--config5" in sys.argv else synth.CONFIG2
    b = synth.generate(w, n, seed=5)
    st = (ctypes.c_ulonglong * 16)()
    lib.eb_debug_stats(st, 1)
    res = search.solve_batch(b, ladder=tuple(w.outputs), exact_tau="--exact" in sys.argv)
    lib.eb_debug_stats(st, 0)
    names = ["instances", "windows", "windows_T>0", "leaf_batches", "leaves", "u_builds", "live_calls",
             "calls_to_winner"]
    inst = st[0]
    for i, nm in enumerate(names):
        print(f"{nm:16s} {st[i]:14d}  per-instance {st[i] / max(inst, 1):9.2f}")
    print("mean z", res.z_found.mean())


if __name__ == "__main__":
    main()
