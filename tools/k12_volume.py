#!/usr/bin/env python3
"""K1/K2 kernels at volume on one GPU (device-resident inputs, EB_MEM_DEVICE):
eb_link_batch, eb_admission_batch, eb_coefficients_batch,
eb_check_direct_batch and eb_check_knapsack_batch over the config-2 workload
(10^6 instances x 20 requests = 2e7 rows; check_direct / check_knapsack on
the 2e6 candidate batches of the first 10^5 instances' DFTSP solutions' sizes
... simplified here to each instance's 6 first rows).  Prints one JSON line
per kernel: launch time (CUDA events, best of 5) and algorithmic HBM bytes /
time against MEASURED_PEAKS.json.  Run under ncu for the counters:
  ncu --set full -k regex:"link_kernel|admission_kernel|coeff_kernel|check_direct_kernel|check_knapsack_kernel" \\
      python tools/k12_volume.py --reps 1
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2405_07140_b200 import _lib, synth  # noqa: E402
from paper_2405_07140_b200.soa import InstanceBatch, requests_struct  # noqa: E402


def ref(s):
    return ctypes.cast(ctypes.pointer(s), ctypes.c_void_p)


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-inst", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    h = _lib.handle(0)
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    rng = np.random.default_rng(1)
    n, K = args.n_inst, 20
    w = synth.CONFIG2
    cols = synth._draw(rng, n * K, w)
    cols["uplink_power_w"] = np.full(n * K, synth.dbm(20.0))
    cols["id"] = np.tile(np.arange(K, dtype=np.int64), n)
    recs = synth.contexts(w)
    prof = rng.integers(0, len(recs), n).astype(np.int32)
    off = np.arange(n + 1, dtype=np.int64) * K
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    d_cols = {k: T(v) for k, v in cols.items()}
    d_off, d_ci, d_ctx = T(off), T(prof), T(recs.view(np.uint8))
    b = InstanceBatch(d_off, d_cols, recs, d_ci, K, on_device=True)
    bs = b.struct()
    rs = requests_struct(d_cols)
    nr = n * K
    req_ctx = T(np.repeat(prof, K))
    out = {}

    def timed(name, fn, bytes_alg):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        out[name] = {"ms": round(best * 1e3, 4), "alg_bytes": bytes_alg, "gb_s": round(bytes_alg / best / 1e9, 1)}

    status = torch.zeros(nr, dtype=torch.int32, device=dev)
    link = torch.zeros(nr * 6, dtype=torch.float64, device=dev)
    timed("link_kernel", lambda: _lib.check(h.lib.eb_link_batch(h.ptr, d_ctx.data_ptr(), len(recs), ref(rs), nr,
                                                                   req_ctx.data_ptr(), status.data_ptr(),
                                                                   link.data_ptr(), _lib.EB_MEM_DEVICE), "link"),
          nr * (8 + 8 + 4 + 4 + 4) + nr * (4 + 48))
    keep = torch.zeros(nr, dtype=torch.uint8, device=dev)
    timed("admission_kernel", lambda: _lib.check(h.lib.eb_admission_batch(
        h.ptr, d_ctx.data_ptr(), len(recs), ref(bs), 1, 1, status.data_ptr(), keep.data_ptr(),
        _lib.EB_MEM_DEVICE), "admission"), nr * (8 * 5 + 4 + 4) + nr * 5)
    ist = torch.zeros(n, dtype=torch.int32, device=dev)
    ierr = torch.zeros(n, dtype=torch.int32, device=dev)
    sc = torch.zeros(n * 6, dtype=torch.float64, device=dev)
    rq = torch.zeros(nr * 4, dtype=torch.float64, device=dev)
    timed("coeff_kernel", lambda: _lib.check(h.lib.eb_coefficients_batch(
        h.ptr, d_ctx.data_ptr(), len(recs), ref(bs), None, ist.data_ptr(), ierr.data_ptr(), sc.data_ptr(),
        rq.data_ptr(), _lib.EB_MEM_DEVICE), "coeff"), nr * (8 * 4 + 4) + n * (48 + 8) + nr * 32)
    # one candidate batch per instance: its first 6 rows
    z = 6
    sub_off = T(np.arange(n + 1, dtype=np.int64) * z)
    members = T((np.arange(n)[:, None] * K + np.arange(z)[None, :]).reshape(-1).astype(np.int32))
    pad = T(np.full(n, 512, np.int64))
    ok = torch.zeros(n, dtype=torch.uint8, device=dev)
    met = torch.zeros(n * 4, dtype=torch.float64, device=dev)
    timed("check_direct_kernel", lambda: _lib.check(h.lib.eb_check_direct_batch(
        h.ptr, d_ctx.data_ptr(), len(recs), ref(rs), nr, n, sub_off.data_ptr(), members.data_ptr(),
        d_ci.data_ptr(), pad.data_ptr(), ist.data_ptr(), ok.data_ptr(), met.data_ptr(), _lib.EB_MEM_DEVICE),
        "check_direct"), n * z * (4 + 8 * 4 + 8) + n * (8 + 8 + 4 + 4 + 1 + 32))
    ku, kd = rq[0::4].contiguous(), rq[1::4].contiguous()
    zz = T(np.full(n, z, np.int32))
    taum = T(np.full(n, 1e30))
    prm_p = T(cols["prompt_tokens"].reshape(n, K)[:, :z].reshape(-1))
    prm_o = T(cols["output_tokens"].reshape(n, K)[:, :z].reshape(-1))
    ku6 = ku.view(n, K)[:, :z].contiguous().view(-1)
    kd6 = kd.view(n, K)[:, :z].contiguous().view(-1)
    timed("check_knapsack_kernel", lambda: _lib.check(h.lib.eb_check_knapsack_batch(
        h.ptr, n, sub_off.data_ptr(), prm_p.data_ptr(), prm_o.data_ptr(), ku6.data_ptr(), kd6.data_ptr(),
        sc.data_ptr(), zz.data_ptr(), taum.data_ptr(), ok.data_ptr(), _lib.EB_MEM_DEVICE), "knapsack"),
        n * z * (4 + 4 + 8 + 8) + n * (8 + 48 + 4 + 8 + 1))
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except (OSError, ValueError):
        pass
    for k, v in out.items():
        hbm = peaks.get("hbm_gbs")
        print(json.dumps({"kernel": k, **v, "rows": nr, "instances": n, "hbm_peak_gb_s": hbm,
                          "hbm_frac": round(v["gb_s"] / hbm, 4) if hbm else None}))


if __name__ == "__main__":
    main()
