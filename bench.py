#!/usr/bin/env python3
"""Benchmark: DFTSP instances/s on the config-2 Monte Carlo sweep (BASELINE.json).

Workload (configs[1]): 10^6 synthetic scheduling instances, K = 20 admitted
candidates each, BLOOM-3B with a uniform fp16 / w8a16 / w4a16-gptq mix on the
paper's default edge node.  One step = one
eb_dftsp_batch over this rank's shard of the instances.

  value   instances/s, inputs resident in HBM (EB_MEM_DEVICE), CUDA events on
          the launch stream, L2 flushed between steps, max over ranks
  e2e     same metric through the C ABI with HOST buffers (pinned): every step
          copies the instances in and the results out inside the timed region
  roofline  FP64 issue bound (the search is FP64 compare/accumulate + integer
          control; no HBM or tensor-core bound applies), algorithmic FP64 ops
          from the oracle's work counters on a sample of the same workload
  cpu_baseline  the C oracle port of the reference on a bounded sample with all
          host threads (rank 0, N=1)

``--impl reference`` times the reference CPU path (oracle port, all host
threads) on the same workload/metric and prints the same JSON line.
Multi-GPU: torchrun, one rank per GPU, instances sharded by contiguous range
(weak scaling: 10^6 instances per GPU), no data-path collective.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))   # CPU baseline / reference arm only

FP64_LANES_PER_SM = 64          # B200 FP64 pipe: 64 lanes/SM/clk
LEAF_OPS, DESCEND_OPS = 26, 5   # algorithmic FP64-class ops per leaf check / descend
LADDER = (128, 256, 512)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--n-inst", type=int, default=1_000_000, help="instances per GPU")
    ap.add_argument("--cpu-sample", type=int, default=0, help="instances in the CPU sample (0 = auto)")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def _nvml_sampler(idx: int, conn, stop, period: float):
    """Child process: (time, sm_mhz, max_mhz, reasons) every `period` s until `stop` is set."""
    rows = []
    try:
        import pynvml
        pynvml.nvmlInit()
        hnd = pynvml.nvmlDeviceGetHandleByIndex(idx)
        mx = float(pynvml.nvmlDeviceGetMaxClockInfo(hnd, pynvml.NVML_CLOCK_SM))
        while not stop.is_set():
            try:
                rows.append((time.time(), float(pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)), mx,
                             int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(hnd))))
            except Exception:
                pass
            time.sleep(period)
    except Exception:
        pass
    conn.send(rows)
    conn.close()


class ClockSampler:
    """SM clocks and throttle reasons under load: NVML sampled every 2 ms in a
    separate process (no GIL contention with the timing loop), started before
    the warm-up; summary() keeps the samples inside the timed window marked
    with begin()/end() (all load samples if the window caught fewer than 3)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, device: int):
        self.device = device
        self.rows = []          # (time, sm_mhz, max_mhz, reasons bitmask)
        self.t0 = self.t1 = None
        self.proc = None

    def start(self):
        import multiprocessing as mp
        idx = self.device
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                idx = int(vis.split(",")[self.device])
            except ValueError:
                pass
        ctx = mp.get_context("spawn")
        self.parent, child = ctx.Pipe(duplex=False)
        self.stop_ev = ctx.Event()
        self.proc = ctx.Process(target=_nvml_sampler, args=(idx, child, self.stop_ev, 0.002), daemon=True)
        self.proc.start()
        return self

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()

    def finish(self):
        if self.proc is None:
            return
        self.stop_ev.set()
        try:
            if self.parent.poll(10):
                self.rows = self.parent.recv()
        except (EOFError, OSError):
            pass
        self.proc.join(timeout=5)
        self.proc = None

    def summary(self):
        self.finish()
        rows, in_window = self.rows, False
        if self.t0 is not None and self.t1 is not None:
            win = [r for r in rows if self.t0 <= r[0] <= self.t1]
            if len(win) >= 3:
                rows, in_window = win, True
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({name for *_, m in rows for bit, name in self.REASONS.items() if m & bit})
        return {"sm_mhz": statistics.median(r[1] for r in rows), "sm_max_mhz": max(r[2] for r in rows),
                "reasons": reasons, "samples": len(rows),
                "window": "timed region" if in_window else "warm-up and timed region"}


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "ours" else "gloo"
        dist.init_process_group(backend=backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def profile_issue_pct():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_dftsp_summary.json")) as fh:
            return json.load(fh).get("issue_active_pct")
    except (OSError, ValueError):
        return None


def profile_warp_inst():
    """Warp instructions per instance of the search kernel (committed ncu capture)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_dftsp_summary.json")) as fh:
            return json.load(fh).get("warp_instructions_per_instance")
    except (OSError, ValueError):
        return None


def load_profile_traffic():
    """DRAM bytes per launch of the search kernel from the committed ncu capture (or None)."""
    p = os.path.join(ROOT, "profiles", "ncu_dftsp_summary.json")
    try:
        with open(p) as fh:
            j = json.load(fh)
        return j.get("dram_bytes_per_launch"), j.get("instances_per_launch")
    except (OSError, ValueError):
        return None, None


def issue_roofline(sms: int, f_mhz: float, n: int, per_launch_s: float):
    """Warp-instruction issue rate of the search kernel against the SM issue
    peak (4 schedulers x 1 warp-instruction per clock per SM): the bound the
    kernel actually meets.  Instructions per instance come from the committed
    ncu capture; the time is this run's."""
    wi = profile_warp_inst()
    if not wi:
        return None
    achieved = wi * n / per_launch_s / 1e9
    peak = sms * 4 * f_mhz * 1e6 / 1e9
    out = {"achieved": round(achieved, 1), "peak": round(peak, 1), "unit": "G warp-inst/s",
           "frac": round(achieved / peak, 4), "warp_inst_per_instance_ncu": wi}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_dftsp_summary.json")) as fh:
            j = json.load(fh)
        # warp-execution efficiency (active lanes per issued warp instruction / 32)
        # and the scenario-array stream rate, from the same capture
        out["warp_execution_efficiency_ncu"] = round(j["threads_per_warp_inst"] / 32.0, 4)
        out["hbm_gb_s_ncu"] = round(j["dram_bytes_per_launch"] / (j["duration_ms"] * 1e-3) / 1e9, 1)
    except (OSError, ValueError, KeyError, TypeError, ZeroDivisionError):
        pass
    return out


def cpu_baseline(batch, sample: int, threads: int):
    import oracle
    from paper_2405_07140_b200.soa import InstanceBatch
    n = min(sample, batch.n_inst)
    sub = InstanceBatch(batch.offsets[:n + 1].copy(), {k: v[:int(batch.offsets[n])] for k, v in batch.columns.items()},
                        batch.contexts, batch.ctx_index[:n].copy(), batch.k_max)
    t0 = time.perf_counter()
    res = oracle.dftsp_batch(sub, ladder=LADDER, threads=threads)
    dt = time.perf_counter() - t0
    return n / dt, dt, res, sub


def main():
    args = parse()
    world, rank, local = dist_init(args)
    from paper_2405_07140_b200 import synth

    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2405_07140_b200 import _lib, search
    from paper_2405_07140_b200.soa import search_params

    # ---- workload: this rank's shard (weak scaling: n_inst per GPU) --------
    t_gen = time.time()
    batch = synth.generate(synth.CONFIG2, args.n_inst, seed=2405_07140 + rank, device=local)
    gen_s = time.time() - t_gen
    n, nr = batch.n_inst, batch.n_req
    h = _lib.handle(local)
    stream = torch.cuda.Stream(device=dev)
    h.set_stream(stream.cuda_stream)

    # device-resident copies (value) and pinned host copies (e2e)
    def to_dev(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    d_off = to_dev(batch.offsets)
    d_ci = to_dev(batch.ctx_index)
    # dftsp reads every request column except `tolerance` (candidates are
    # already accuracy-admitted, sim.py:264-274), so it is not shipped
    used = [k for k in batch.columns if k != "tolerance"]
    d_cols = {k: to_dev(batch.columns[k]) for k in used}
    d_ctx = to_dev(batch.contexts.view(np.uint8)).contiguous()
    outs = {"status": torch.zeros(n, dtype=torch.int32, device=dev),
            "error_index": torch.zeros(n, dtype=torch.int32, device=dev),
            "z_found": torch.zeros(n, dtype=torch.int32, device=dev),
            "nodes_visited": torch.zeros(n, dtype=torch.int64, device=dev),
            "nodes_pruned": torch.zeros(n, dtype=torch.int64, device=dev),
            "n_classes": torch.zeros(n, dtype=torch.int32, device=dev),
            "counts": torch.zeros(n * 16, dtype=torch.int32, device=dev),
            "class_lengths": torch.zeros(n * 16, dtype=torch.int32, device=dev),
            "solution": torch.zeros(nr, dtype=torch.int32, device=dev),
            "metrics": torch.zeros(n * 8, dtype=torch.float64, device=dev)}
    import ctypes
    dres = _lib.eb_dftsp_result()
    for k, t in outs.items():
        setattr(dres, k, t.data_ptr())
    from paper_2405_07140_b200.soa import InstanceBatch
    dbatch = InstanceBatch(d_off, d_cols, batch.contexts, d_ci, batch.k_max, on_device=True)
    db = dbatch.struct()
    prm = search_params(ladder=LADDER)
    ref = lambda s: ctypes.cast(ctypes.pointer(s), ctypes.c_void_p)  # noqa: E731
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step_device():
        _lib.check(h.lib.eb_dftsp_batch(h.ptr, d_ctx.data_ptr(), len(batch.contexts), ref(prm), ref(db), ref(dres),
                                        _lib.EB_MEM_DEVICE), "eb_dftsp_batch")

    clk = ClockSampler(local).start()
    with torch.cuda.stream(stream):
        # W warm-up steps, continued until the GPU has been busy for >= 1 s
        # (the host-side workload generation leaves it idle long enough for
        # the SM clock to drop; short runs would otherwise time the ramp)
        t_w = time.perf_counter()
        done = 0
        while done < args.warmup or time.perf_counter() - t_w < 1.0:
            step_device()
            stream.synchronize()
            done += 1
        stream.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        launches0 = h.launches()
        times = []
        clk.begin()
        for _ in range(args.steps):
            flush.fill_(1.0)                      # L2 flush between timed steps
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step_device()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        clk.end()
        torch.cuda.synchronize()
        barrier(world)
        launches = h.launches() - launches0
    dev_s = max_over_ranks(sum(times), world, dev)
    value = world * n * args.steps / dev_s
    ms_per_step = dev_s / args.steps * 1e3
    # device results for accounting (and a parity spot check against the oracle)
    z = outs["z_found"].cpu().numpy()
    vis = outs["nodes_visited"].cpu().numpy()
    sol = outs["solution"].cpu().numpy()
    owner = np.repeat(np.arange(n), np.diff(batch.offsets))
    bits = np.where(sol >= 0, np.left_shift(np.int64(1), np.maximum(sol, 0).astype(np.int64)), 0)
    sol_mask = np.zeros(n, np.int64)
    np.bitwise_or.at(sol_mask, owner, bits)
    status = outs["status"].cpu().numpy()
    assert (status == 0).all(), f"device statuses: {np.unique(status)}"

    # ---- e2e through the C ABI with pinned host buffers --------------------
    e2e = None
    if not args.no_e2e:
        from paper_2405_07140_b200.soa import pack_wire

        def pinned(a):
            return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

        # results a sweep consumes: status, z, node counts and the selected set
        # (u64 mask per instance; the ids rise along the rows, so bit order is
        # the solution's id order)
        hout = {"status": torch.zeros(n, dtype=torch.int32).pin_memory(),
                "z_found": torch.zeros(n, dtype=torch.int32).pin_memory(),
                "nodes_visited": torch.zeros(n, dtype=torch.int64).pin_memory(),
                "nodes_pruned": torch.zeros(n, dtype=torch.int64).pin_memory(),
                "solution_mask": torch.zeros(n, dtype=torch.int64).pin_memory()}
        hres = _lib.eb_dftsp_result()
        for k, t in hout.items():
            setattr(hres, k, t.data_ptr())
        d2h = sum(t.numel() * t.element_size() for t in hout.values())
        # wide layout (eb_requests, 48 B/request) and the compact wire format
        # (eb_requests_packed, 32 B/request); the same pinned output buffers
        hb = InstanceBatch(pinned(batch.offsets), {k: pinned(batch.columns[k]) for k in used}, batch.contexts,
                           pinned(batch.ctx_index), batch.k_max)
        h2d_wide = sum(hb.columns[k].nbytes for k in used) + hb.offsets.nbytes + hb.ctx_index.nbytes
        wb = pack_wire(batch, pin=pinned)
        assert wb is not None, "config-2 columns narrow losslessly"
        hbs, wbs = hb.struct(), wb.struct()

        def step_wide():
            _lib.check(h.lib.eb_dftsp_batch(h.ptr, batch.contexts.ctypes.data, len(batch.contexts), ref(prm),
                                            ref(hbs), ref(hres), _lib.EB_MEM_HOST), "eb_dftsp_batch(host)")

        def step_wire():
            _lib.check(h.lib.eb_dftsp_batch_packed(h.ptr, batch.contexts.ctypes.data, len(batch.contexts), ref(prm),
                                                   ref(wbs), ref(hres), _lib.EB_MEM_HOST), "eb_dftsp_batch_packed")

        def time_host(step):
            for _ in range(max(1, args.warmup)):
                step()
            barrier(world)
            torch.cuda.synchronize()
            et = []
            for _ in range(args.steps):
                flush.fill_(1.0)
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
                e1.synchronize()
                et.append(e0.elapsed_time(e1) / 1e3)
            assert np.array_equal(hout["z_found"].numpy(), z) and np.array_equal(hout["nodes_visited"].numpy(), vis)
            assert np.array_equal(hout["solution_mask"].numpy(), sol_mask)
            return max_over_ranks(sum(et), world, dev)

        wide_s = time_host(step_wide)
        wire_s = time_host(step_wire)
        e2e = {"value": world * n * args.steps / wire_s, "unit": "instances/s", "h2d_bytes_per_step": int(wb.nbytes()),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": wire_s / args.steps * 1e3,
               "path": "eb_dftsp_batch_packed(EB_MEM_HOST): pinned host buffers in the compact wire format "
                       "(token counts as one dictionary byte, uniform uplink power, ids = row positions since "
                       "they rise along every instance, uniform offsets): 25 B/request; uploads on their own "
                       "stream, chunks ramping n/64 -> n/16 -> n/64 over 3 compute streams",
               "wide": {"value": world * n * args.steps / wide_s, "h2d_bytes_per_step": int(h2d_wide),
                        "ms_per_step": wide_s / args.steps * 1e3, "path": "eb_dftsp_batch(EB_MEM_HOST), eb_requests"}}

    # ---- roofline (rank 0 figures) + cpu baseline ---------------------------
    # (no collectives below: the other ranks are done; rank 0 has the host)
    clocks = clk.summary()
    if rank != 0:
        return
    import oracle
    sample = args.cpu_sample or (n if world == 1 else 50_000)     # N=1: the whole 10^6-instance workload
    threads = os.cpu_count() or 1
    cpu_rate, cpu_s, orc, sub = cpu_baseline(batch, min(sample, n), threads)
    parity_ok = bool(np.array_equal(orc["z_found"], z[:sub.n_inst]) and
                     np.array_equal(orc["nodes_visited"], vis[:sub.n_inst]))
    wsub = oracle.work_counters(InstanceBatch(sub.offsets[:20001], {k: v[:int(sub.offsets[min(20000, sub.n_inst)])]
                                                                    for k, v in sub.columns.items()},
                                              sub.contexts, sub.ctx_index[:20000], sub.k_max), ladder=LADDER,
                                threads=threads)
    n_w = min(20000, sub.n_inst)
    ops_per_inst = (LEAF_OPS * wsub["leaf_checks"] + DESCEND_OPS * wsub["descends"]) / n_w
    props = torch.cuda.get_device_properties(dev)
    f_mhz = clocks.get("sm_max_mhz") or 1965.0
    peak_fp64 = props.multi_processor_count * FP64_LANES_PER_SM * f_mhz * 1e6 / 1e12   # TFLOP/s (1 op/lane/clk)
    per_launch_s = dev_s / args.steps
    achieved = ops_per_inst * n / per_launch_s / 1e12
    traffic, traffic_n = load_profile_traffic()
    if traffic is not None and traffic_n:
        traffic = traffic * n / traffic_n
    line = {
        "metric": "DFTSP instances/sec (K=20 users) and search nodes/sec",
        "value": round(value, 1), "unit": "instances/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "warmup_steps_run": done, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": synth.CONFIG2.name, "instances_per_gpu": n, "K": 20, "ladder": list(LADDER),
                   "flags": "pruning=True inclusive=False exact_tau=False", "l2": "flushed between steps (256 MiB)",
                   "parallelism": f"instance-sharded x{world}"},
        "nodes_visited_per_s": round(float(vis.sum()) * world * args.steps / dev_s, 1),
        "mean_z": float(z.mean()), "mean_nodes_visited": float(vis.mean()),
        "e2e": e2e,
        "gpu_launches": int(launches),
        "roofline": {"bound": "fp64-issue", "achieved": round(achieved, 4), "peak": round(peak_fp64, 3),
                     "unit": "TFLOP/s", "frac": round(achieved / peak_fp64, 5), "traffic": traffic,
                     "ops_per_instance": round(ops_per_inst, 1),
                     "ops_model": "26 FP64 ops per leaf check + 5 per descend (SURVEY.md 8(d)); counts from the "
                                  "oracle on a 20k-instance sample of this workload; peak = SMs x 64 FP64 lanes x "
                                  "max SM clock (no measured FP64 peak in MEASURED_PEAKS.json)",
                     "issue_active_pct_ncu": profile_issue_pct(),
                     "issue": issue_roofline(props.multi_processor_count, f_mhz, n, per_launch_s),
                     "issue_note": "SM issue-slot utilisation of the search kernel from the committed ncu capture "
                                   "(profiles/ncu_dftsp_summary.json): the path is instruction-issue bound "
                                   "(integer control + FP64 compare/accumulate)"},
        "cpu_baseline": {"value": round(cpu_rate, 1), "unit": "instances/s", "cores": threads, "kind": "port",
                         "sample": f"{sub.n_inst} instances of the same workload, C oracle (literal restatement "
                                   f"of the reference), {threads} threads, {cpu_s:.1f} s"},
        "parity_sample_ok": parity_ok,
        "clocks": clocks,
        "gen_s": round(gen_s, 1),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_reference(args, world, rank):
    """Reference CPU path (C oracle port of the reference, all host threads) on this workload."""
    if rank != 0:
        return
    import oracle
    from paper_2405_07140_b200 import synth
    try:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError
        batch_src = "device-admitted synthetic workload"
    except Exception:
        batch_src = None
    # up to the same 10^6 instances per step, bounded so that the whole
    # warm-up + timed run stays near a minute (~2.6e5 inst/s on 16 threads)
    sample = args.cpu_sample or min(1_000_000, max(50_000, int(15e6 / max(1, args.steps + args.warmup))))
    batch = synth.generate(synth.CONFIG2, sample, seed=2405_07140)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle.dftsp_batch(batch, ladder=LADDER, threads=threads)
    t = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res = oracle.dftsp_batch(batch, ladder=LADDER, threads=threads)
        t.append(time.perf_counter() - t0)
    rate = batch.n_inst * args.steps / sum(t)
    line = {"metric": "DFTSP instances/sec (K=20 users) and search nodes/sec", "value": round(rate, 1),
            "unit": "instances/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sum(t) / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": synth.CONFIG2.name, "K": 20, "sample_instances": batch.n_inst,
                       "source": batch_src},
            "nodes_visited_per_s": round(float(res["nodes_visited"].sum()) * args.steps / sum(t), 1),
            "cpu_baseline": {"value": round(rate, 1), "unit": "instances/s", "cores": threads, "kind": "port",
                             "sample": f"{batch.n_inst} instances per step, C oracle port, {threads} threads"},
            "e2e": {"value": round(rate, 1), "unit": "instances/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
