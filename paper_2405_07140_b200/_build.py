"""Build the in-tree CUDA library (sm_100a) and the test-only CPU oracle.

``build_library()`` compiles ``csrc/*.cu`` into ``libedgebatch_b200.so`` next
to this file (git-ignored, travels to the GPU box with the repo snapshot).
Flags that matter for bit-exactness: ``-fmad=false`` (no FMA contraction in
device code; the kernels additionally use explicit ``__dadd_rn``-style
intrinsics) and ``-ffp-contract=off`` for host code.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libedgebatch_b200.so")
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_LIB = os.path.join(ORACLE_DIR, "liboracle.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_library(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(ROOT, "include", "edgebatch_b200.h")]
    if not force and not _stale(LIB, deps):
        return LIB
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
             "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-v" if verbose else "-O3",
             "-I", os.path.join(ROOT, "include")]
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)

    headers = [d for d in deps if not d.endswith(".cu")]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        if not force and not _stale(obj, [src, *headers]):
            return obj, subprocess.CompletedProcess([], 0, "", "")
        return obj, subprocess.run([_nvcc(), *flags, "-c", "-o", obj, src], capture_output=True, text=True)

    # one nvcc per translation unit, in parallel (eb_dftsp.cu dominates)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        results = list(ex.map(compile_one, srcs))
    for _, res in results:
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed building libedgebatch_b200.so")
        if verbose:
            sys.stderr.write(res.stderr)
    res = subprocess.run([_nvcc(), *ARCH, "-shared", "-o", LIB + ".tmp", *[o for o, _ in results]],
                         capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libedgebatch_b200.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


def source_hash() -> str:
    """sha256 (16 hex) over the CUDA sources and the ABI header: ties a
    committed ncu capture to the kernels it measured (bench.py flags
    captures of other sources as stale)."""
    import hashlib
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                   glob.glob(os.path.join(CSRC, "*.h"))) + [os.path.join(ROOT, "include", "edgebatch_b200.h")]
    for f in files:
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def stage_reference() -> str | None:
    """Test-only: stage the unmodified Python reference into oracle/_ref
    (oracle/make_ref.py; a no-op where /root/reference is absent)."""
    sys.path.insert(0, ORACLE_DIR)
    try:
        import make_ref
        return make_ref.stage()
    finally:
        sys.path.remove(ORACLE_DIR)


def build_oracle(force: bool = False) -> str:
    """Test-only: compile the CPU oracle (oracle/edgebatch_oracle.c)."""
    src = os.path.join(ORACLE_DIR, "edgebatch_oracle.c")
    deps = [src, os.path.join(ROOT, "include", "edgebatch_b200.h")]
    if not force and not _stale(ORACLE_LIB, deps):
        return ORACLE_LIB
    cc = shutil.which("gcc") or "cc"
    cmd = [cc, "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math", "-std=gnu11",
           "-o", ORACLE_LIB + ".tmp", src, "-lm", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("gcc failed building the oracle")
    os.replace(ORACLE_LIB + ".tmp", ORACLE_LIB)
    return ORACLE_LIB


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose="-v" in sys.argv))
    print(build_oracle(force="--force" in sys.argv))
