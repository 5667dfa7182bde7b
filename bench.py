#!/usr/bin/env python3
"""Benchmark: DFTSP instances/s on the config-2 Monte Carlo sweep (BASELINE.json).

Workload (configs[1]): 10^6 synthetic scheduling instances per GPU, K = 20
admitted candidates each, BLOOM-3B with a uniform fp16 / w8a16 / w4a16-gptq
mix on the paper's default edge node.  One step
= one eb_dftsp_batch over this rank's instances.

  value     instances/s, inputs resident in HBM (EB_MEM_DEVICE), CUDA events on
            the launch stream, L2 flushed between steps, max over ranks
  e2e       the same metric through the C ABI with HOST buffers (pinned), the
            general request layout (eb_requests, what a caller hands over) and
            the whole SearchOutcome read back (dftsp.py:42-51: status, z,
            nodes visited/pruned, class counts, solution ids); every step's
            copies are inside the timed region.  `e2e.wire` is the compact
            wire format (eb_dftsp_batch_packed) with its host packing cost
  roofline  FP64/issue bound of the search kernel: algorithmic FP64 ops per
            instance (oracle work counters) over the kernel time, against the
            FP64 add rate and the warp-instruction issue rate MEASURED in this
            run by eb_probe_peaks; ncu-only counters come from the committed
            capture and are flagged stale when the CUDA sources changed
  cpu_baseline  the unmodified Python reference (oracle/_ref, its own
            dftsp() with ProcessPoolExecutor(nproc), cli.py:262-264) on a
            bounded sample of the same instances (rank 0, N=1); the C port of
            it is reported beside (cpu_port) and checks the device on ALL
            instances, every output field

``--impl reference`` times that Python reference on the same workload/metric
and prints the same JSON line (rank 0 only; other ranks exit 0).  It rebuilds
the identical 10^6 instances with the CPU admission oracle, so the CUDA
library is never loaded on that arm.
``--gpus N`` without torchrun re-launches itself under torch.distributed.run
with N ranks (one per GPU, NCCL); instances are sharded by rank (weak scaling,
10^6 per GPU), no data-path collective.
``--config 5`` runs the tight-memory edge workload (configs[4]) instead;
``--config 4`` the brute-force K=32 search sharded by subset rank over the
ranks (configs[3], brute.solve_distributed).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))   # CPU baselines / checker only

LEAF_OPS, DESCEND_OPS = 26, 5   # algorithmic FP64-class ops per leaf check / descend
METRIC = "DFTSP instances/sec (K=20 users) and search nodes/sec"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", type=int, default=2, choices=(2, 4, 5))
    ap.add_argument("--n-inst", type=int, default=1_000_000, help="instances per GPU")
    ap.add_argument("--cpu-sample", type=int, default=0, help="instances per reference step (0 = auto)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baselines (profiling runs)")
    ap.add_argument("--brute-k", type=int, default=32)
    ap.add_argument("--brute-n", type=int, default=8, help="config 4: instances per step")
    return ap.parse_args()


# ---------------------------------------------------------------- plumbing --
def self_spawn(args) -> int:
    """--gpus N > 1 outside torchrun: re-launch under torch.distributed.run."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "WARN")
    return subprocess.call(cmd, env=env)


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if args.impl == "ours":
            import torch
            torch.cuda.set_device(local)
            dist.init_process_group(backend="nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend="gloo")
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} rank(s)", file=sys.stderr)
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


def ranks_info(world, dev):
    """(distinct GPUs across ranks, NCCL communicator size) -- the scaling run's evidence."""
    import torch
    uuid = str(torch.cuda.get_device_properties(dev).uuid)
    if world == 1:
        return 1, 1
    import torch.distributed as dist
    got = [None] * world
    dist.all_gather_object(got, uuid)
    return len(set(got)), dist.get_world_size()


def _nvml_sampler(idx: int, conn, stop, period: float, ready=None):
    """Child process: (time, sm_mhz, max_mhz, reasons) every `period` s until `stop` is set."""
    rows = []
    try:
        import pynvml
        pynvml.nvmlInit()
        hnd = pynvml.nvmlDeviceGetHandleByIndex(idx)
        mx = float(pynvml.nvmlDeviceGetMaxClockInfo(hnd, pynvml.NVML_CLOCK_SM))
        if ready is not None:
            ready.set()
        while not stop.is_set():
            try:
                rows.append((time.time(), float(pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)), mx,
                             int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(hnd))))
            except Exception:
                pass
            time.sleep(period)
    except Exception:
        pass
    if ready is not None:
        ready.set()             # NVML unavailable: do not hold the caller
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
        self.rows = []
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
        ready = ctx.Event()
        self.proc = ctx.Process(target=_nvml_sampler, args=(idx, child, self.stop_ev, 0.002, ready), daemon=True)
        self.proc.start()
        ready.wait(30)          # sampling before the warm-up starts (short runs: config 4)
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


def ncu_profile(config: int = 2):
    """The committed ncu capture of this config's search kernel, and whether it was taken on these sources."""
    name = "ncu_config5_summary.json" if config == 5 else "ncu_dftsp_summary.json"
    try:
        with open(os.path.join(ROOT, "profiles", name)) as fh:
            j = json.load(fh)
    except (OSError, ValueError):
        return None, False
    from paper_2405_07140_b200._build import source_hash
    return j, j.get("source_hash") == source_hash()


def workload(config: int):
    from paper_2405_07140_b200 import synth
    if config == 5:
        return synth.CONFIG5, (64, 128, 256, 512, 1024)
    return synth.CONFIG2, (128, 256, 512)


def config_dict(w, ladder, n, world):
    return {"workload": w.name, "instances_per_gpu": n, "K": w.K, "ladder": list(ladder),
            "flags": "pruning=True inclusive=False exact_tau=False",
            "l2": "flushed between steps (256 MiB write)", "parallelism": f"instance-sharded x{world}"}


# ------------------------------------------------------------ reference arm --
def reference_rate(batch, ladder, per_step: int, steps: int, warmup: int, procs: int):
    """The Python reference's dftsp over consecutive slices of `batch`
    (ProcessPoolExecutor(procs)); returns rate, spans, and agreement with the C
    port on the instances it solved."""
    import oracle
    import pyref
    pool = pyref.ReferencePool(procs)
    n = batch.n_inst
    spans, vis_sum, done, agree = [], 0, 0, True
    try:
        for k in range(warmup + steps):
            lo = (k * per_step) % max(1, n - per_step + 1)
            span, z, vis, prn = pool.run(batch, lo, lo + per_step, ladder=ladder)
            if k >= warmup:
                spans.append(span)
                vis_sum += int(vis.sum())
                done += per_step
                if len(spans) <= 2:     # the C port reproduces the reference on what it solved
                    sub = slice_batch(batch, lo, lo + per_step)
                    o = oracle.dftsp_batch(sub, ladder=ladder, threads=procs)
                    agree &= bool(np.array_equal(o["z_found"], z) and np.array_equal(o["nodes_visited"], vis)
                                  and np.array_equal(o["nodes_pruned"], prn))
    finally:
        pool.close()
    t = sum(spans)
    return done / t, vis_sum / t, t, agree


def slice_batch(batch, lo, hi):
    from paper_2405_07140_b200.soa import InstanceBatch
    r0, r1 = int(batch.offsets[lo]), int(batch.offsets[hi])
    return InstanceBatch(batch.offsets[lo:hi + 1] - r0, {k: v[r0:r1] for k, v in batch.columns.items()},
                         batch.contexts, batch.ctx_index[lo:hi].copy(), batch.k_max)


def run_reference(args, world, rank):
    """Reference CPU path: the unmodified Python reference (oracle/_ref) with
    all host cores, on the same 10^6 instances (rebuilt with the CPU admission
    oracle, so libedgebatch_b200.so is never loaded here)."""
    if rank != 0:
        return 0
    import oracle
    import pyref
    from paper_2405_07140_b200 import synth
    w, ladder = workload(args.config)
    procs = os.cpu_count() or 1
    base = {"metric": METRIC, "unit": "instances/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference"}
    if args.config == 4:
        base["unavailable"] = ("brute force K=28-32 is not timeable on the CPU reference (~20 h per instance "
                               "per core, BASELINE.md §2c); the config-4 arm reports its extrapolation")
        print(json.dumps(base), flush=True)
        return 0
    if not pyref.available():
        base["unavailable"] = "oracle/_ref (the staged Python reference) is missing"
        print(json.dumps(base), flush=True)
        return 0
    t0 = time.time()
    batch = synth.generate(w, args.n_inst, seed=2405_07140, admit=oracle.admit)
    gen_s = time.time() - t0
    per_step = args.cpu_sample or procs * 60
    rate, vis_rate, t, agree = reference_rate(batch, ladder, per_step, args.steps, args.warmup, procs)
    line = dict(base)
    line.update({
        "value": round(rate, 2), "ms_per_step": round(t / args.steps * 1e3, 3),
        "config": config_dict(w, ladder, args.n_inst, world),
        "nodes_visited_per_s": round(vis_rate, 1),
        "cpu_baseline": {"value": round(rate, 2), "unit": "instances/s", "cores": procs, "kind": "reference",
                         "sample": f"{per_step} consecutive instances of the same {args.n_inst}-instance set per step, "
                                   f"unmodified Python reference edgebatch.dftsp (oracle/_ref) in "
                                   f"ProcessPoolExecutor({procs}); object construction untimed"},
        "e2e": {"value": round(rate, 2), "unit": "instances/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "c_port_agrees_with_reference": agree,
        "same_instances": "synth.generate(seed=2405_07140) with the CPU admission oracle (device-identical)",
        "gen_s": round(gen_s, 1),
    })
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm --
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_spawn(args)
    world, rank, local = dist_init(args)
    if args.impl == "reference":
        return run_reference(args, world, rank)
    if args.config == 4:
        return run_config4(args, world, rank, local)
    return run_dftsp(args, world, rank, local)


def run_dftsp(args, world, rank, local):
    import ctypes

    import torch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2405_07140_b200 import _lib, synth
    from paper_2405_07140_b200.soa import InstanceBatch, pack_wire, search_params

    w, ladder = workload(args.config)
    t_gen = time.time()
    batch = synth.generate(w, args.n_inst, seed=2405_07140 + rank, device=local)
    gen_s = time.time() - t_gen
    n, nr = batch.n_inst, batch.n_req
    h = _lib.handle(local)
    stream = torch.cuda.Stream(device=dev)
    h.set_stream(stream.cuda_stream)

    def to_dev(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    # dftsp reads every request column except `tolerance` (candidates are
    # already accuracy-admitted, sim.py:264-274), so it is not shipped
    used = [k for k in batch.columns if k != "tolerance"]
    d_off, d_ci = to_dev(batch.offsets), to_dev(batch.ctx_index)
    d_cols = {k: to_dev(batch.columns[k]) for k in used}
    d_ctx = to_dev(batch.contexts.view(np.uint8)).contiguous()
    shapes = {"status": (n, torch.int32), "error_index": (n, torch.int32), "z_found": (n, torch.int32),
              "nodes_visited": (n, torch.int64), "nodes_pruned": (n, torch.int64), "n_classes": (n, torch.int32),
              "counts": (n * 16, torch.int32), "class_lengths": (n * 16, torch.int32),
              "solution": (nr, torch.int32), "metrics": (n * 8, torch.float64)}
    outs = {k: torch.zeros(m, dtype=t, device=dev) for k, (m, t) in shapes.items()}
    dres = _lib.eb_dftsp_result()
    for k, t in outs.items():
        setattr(dres, k, t.data_ptr())
    dbatch = InstanceBatch(d_off, d_cols, batch.contexts, d_ci, batch.k_max, on_device=True)
    db = dbatch.struct()
    prm = search_params(ladder=ladder)
    ref = lambda s: ctypes.cast(ctypes.pointer(s), ctypes.c_void_p)  # noqa: E731
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step_device():
        _lib.check(h.lib.eb_dftsp_batch(h.ptr, d_ctx.data_ptr(), len(batch.contexts), ref(prm), ref(db), ref(dres),
                                        _lib.EB_MEM_DEVICE), "eb_dftsp_batch")

    # live roofline denominators (before the sampler: the probe is short)
    fp64_peak = ctypes.c_double(0.0)
    issue_peak = ctypes.c_double(0.0)
    with torch.cuda.stream(stream):
        _lib.check(h.lib.eb_probe_peaks(h.ptr, ctypes.byref(fp64_peak), ctypes.byref(issue_peak)), "eb_probe_peaks")

    clk = ClockSampler(local).start()
    with torch.cuda.stream(stream):
        # W warm-up steps, continued until the GPU has been busy for >= 1 s
        # (host-side generation leaves it idle long enough for the SM clock to drop)
        t_w = time.perf_counter()
        done = 0
        while done < args.warmup or time.perf_counter() - t_w < 1.0:
            step_device()
            stream.synchronize()
            done += 1
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
    res = {k: t.cpu().numpy() for k, t in outs.items()}
    assert (res["status"] == 0).all(), f"device statuses: {np.unique(res['status'])}"

    # ---- e2e through the C ABI with pinned host buffers --------------------
    e2e = None
    if not args.no_e2e:
        def pinned(a):
            return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

        # what SearchOutcome carries (dftsp.py:42-51): status, z, node counts,
        # the class counts and the solution ids
        hout = {"status": (n, torch.int32), "z_found": (n, torch.int32), "nodes_visited": (n, torch.int64),
                "nodes_pruned": (n, torch.int64), "n_classes": (n, torch.int32), "counts": (n * 16, torch.int32),
                "solution": (nr, torch.int32)}
        hout = {k: torch.zeros(m, dtype=t).pin_memory() for k, (m, t) in hout.items()}
        hres = _lib.eb_dftsp_result()
        for k, t in hout.items():
            setattr(hres, k, t.data_ptr())
        d2h = sum(t.numel() * t.element_size() for t in hout.values())
        hb = InstanceBatch(pinned(batch.offsets), {k: pinned(batch.columns[k]) for k in used}, batch.contexts,
                           pinned(batch.ctx_index), batch.k_max)
        h2d = sum(hb.columns[k].nbytes for k in used) + hb.offsets.nbytes + hb.ctx_index.nbytes
        hbs = hb.struct()
        # wire variant: smaller output (mask) and a host packing cost, timed once
        mout = {"status": torch.zeros(n, dtype=torch.int32).pin_memory(),
                "z_found": torch.zeros(n, dtype=torch.int32).pin_memory(),
                "nodes_visited": torch.zeros(n, dtype=torch.int64).pin_memory(),
                "nodes_pruned": torch.zeros(n, dtype=torch.int64).pin_memory(),
                "solution_mask": torch.zeros(n, dtype=torch.int64).pin_memory()}
        mres = _lib.eb_dftsp_result()
        for k, t in mout.items():
            setattr(mres, k, t.data_ptr())
        t_pack = time.perf_counter()
        wb = pack_wire(batch, pin=pinned)
        pack_s = time.perf_counter() - t_pack
        wbs = wb.struct() if wb is not None else None

        def step_general():
            _lib.check(h.lib.eb_dftsp_batch(h.ptr, batch.contexts.ctypes.data, len(batch.contexts), ref(prm),
                                            ref(hbs), ref(hres), _lib.EB_MEM_HOST), "eb_dftsp_batch(host)")

        def step_wire():
            _lib.check(h.lib.eb_dftsp_batch_packed(h.ptr, batch.contexts.ctypes.data, len(batch.contexts), ref(prm),
                                                   ref(wbs), ref(mres), _lib.EB_MEM_HOST), "eb_dftsp_batch_packed")

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
            return max_over_ranks(sum(et), world, dev)

        gen_s_e2e = time_host(step_general)
        for k in hout:
            assert np.array_equal(hout[k].numpy(), res[k]), f"e2e readback differs from the device run: {k}"
        e2e = {"value": world * n * args.steps / gen_s_e2e, "unit": "instances/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": gen_s_e2e / args.steps * 1e3,
               "path": "eb_dftsp_batch(EB_MEM_HOST): pinned host buffers in the general request layout "
                       "(eb_requests columns the caller fills, 48 B/request) in; status, z, nodes visited/pruned, "
                       "n_classes, counts[16] and the solution ids out; uploads on their own stream, chunks "
                       "pipelined over 3 compute streams"}
        if wbs is not None:
            wire_s = time_host(step_wire)
            owner = np.repeat(np.arange(n), np.diff(batch.offsets))
            sol = res["solution"]
            bits = np.where(sol >= 0, np.left_shift(np.int64(1), np.maximum(sol, 0).astype(np.int64)), 0)
            sol_mask = np.zeros(n, np.int64)
            np.bitwise_or.at(sol_mask, owner, bits)
            assert np.array_equal(mout["solution_mask"].numpy(), sol_mask)
            e2e["wire"] = {"value": world * n * args.steps / wire_s, "h2d_bytes_per_step": int(wb.nbytes()),
                           "d2h_bytes_per_step": int(sum(t.numel() * t.element_size() for t in mout.values())),
                           "ms_per_step": wire_s / args.steps * 1e3, "host_pack_s": round(pack_s, 3),
                           "path": "eb_dftsp_batch_packed(EB_MEM_HOST): the compact wire format (token counts as "
                                   "one dictionary byte, uniform uplink power, ids = row positions), valid only "
                                   "for columns that narrow losslessly; solution as a u64 mask. host_pack_s "
                                   "(soa.pack_wire, numpy) is NOT in the timed region"}

    clocks = clk.summary()
    gpus_active, comm = ranks_info(world, dev)
    if rank != 0:
        return 0

    # ---- parity of every output field on ALL instances (C port, all threads)
    import oracle
    threads = os.cpu_count() or 1
    parity_ok, cpu_port = None, None
    if not args.no_cpu:
        t0 = time.perf_counter()
        orc = oracle.dftsp_batch(batch, ladder=ladder, threads=threads)
        port_s = time.perf_counter() - t0
        cpu_port = {"value": round(n / port_s, 1), "unit": "instances/s", "cores": threads, "kind": "port",
                    "sample": f"all {n} instances, C restatement of the reference (oracle/), {threads} threads"}
        fields = ("status", "z_found", "nodes_visited", "nodes_pruned", "n_classes", "counts", "class_lengths",
                  "solution", "metrics")
        bad = [k for k in fields if not np.array_equal(np.asarray(orc[k]).reshape(-1), res[k].reshape(-1))]
        parity_ok = not bad

    # ---- roofline ----------------------------------------------------------
    props = torch.cuda.get_device_properties(dev)
    f_mhz = clocks.get("sm_max_mhz") or 1965.0
    nw = min(20000, n)
    wsub = oracle.work_counters(slice_batch(batch, 0, nw), ladder=ladder, threads=threads)
    ops_per_inst = (LEAF_OPS * wsub["leaf_checks"] + DESCEND_OPS * wsub["descends"]) / nw
    per_launch_s = dev_s / args.steps
    achieved = ops_per_inst * n / per_launch_s / 1e12
    peak = fp64_peak.value / 1e12
    prof, current = ncu_profile(args.config)
    issue = {"peak_measured": round(issue_peak.value / 1e9, 1),
             "peak_nominal": round(props.multi_processor_count * 4 * f_mhz * 1e6 / 1e9, 1), "unit": "G warp-inst/s"}
    traffic = None
    if prof:
        wi = prof.get("warp_instructions_per_instance")
        if wi:
            issue["achieved"] = round(wi * n / per_launch_s / 1e9, 1)
            issue["frac"] = round(issue["achieved"] / issue["peak_measured"], 4)
        issue["warp_inst_per_instance_ncu"] = wi
        issue["warp_execution_efficiency_ncu"] = round(prof.get("threads_per_warp_inst", 0) / 32.0, 4)
        issue["issue_active_pct_ncu"] = prof.get("issue_active_pct")
        issue["ncu_capture_current"] = current
        if prof.get("dram_bytes_per_launch") and prof.get("instances_per_launch"):
            traffic = prof["dram_bytes_per_launch"] * n / prof["instances_per_launch"]

    # ---- the reference CPU path (north-star denominator) -------------------
    cpu = None
    if not args.no_cpu and world == 1:
        import pyref
        if pyref.available():
            per = args.cpu_sample or threads * 250      # ~1 s of the 16-core box per step, ~10 s in all
            reps = 10
            rate, _, t, agree = reference_rate(batch, ladder, per, reps, 1, threads)
            cpu = {"value": round(rate, 2), "unit": "instances/s", "cores": threads, "kind": "reference",
                   "sample": f"{reps} x {per} instances of this workload, unmodified Python reference edgebatch.dftsp "
                             f"(oracle/_ref) in ProcessPoolExecutor({threads}), {t:.1f} s",
                   "c_port_agrees_with_reference": agree}
        else:
            cpu = cpu_port
    line = {
        "metric": METRIC, "value": round(value, 1) if parity_ok is not False else None, "unit": "instances/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "warmup_steps_run": done,
        "ms_per_step": round(dev_s / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(w, ladder, n, world),
        "nodes_visited_per_s": round(float(res["nodes_visited"].sum()) * world * args.steps / dev_s, 1),
        "mean_z": float(res["z_found"].mean()), "mean_nodes_visited": float(res["nodes_visited"].mean()),
        "e2e": e2e,
        "gpu_launches": int(launches),
        "roofline": {"bound": "fp64-issue", "achieved": round(achieved, 4), "peak": round(peak, 3),
                     "unit": "TFLOP/s", "frac": round(achieved / peak, 5), "traffic": traffic,
                     "ops_per_instance": round(ops_per_inst, 1),
                     "ops_model": "26 FP64 ops per leaf check + 5 per descend of the REFERENCE algorithm (SURVEY.md "
                                  "8(d)), counted by the oracle on 20k instances of this workload; the device "
                                  "skips provably failing calls, so this is a reference-equivalent rate; peak = "
                                  "FP64 add rate measured in this run (eb_probe_peaks)",
                     "issue": issue},
        "cpu_baseline": cpu, "cpu_port": cpu_port,
        "parity": {"ok": parity_ok, "instances": n if parity_ok is not None else 0,
                   "fields": "status z nodes_visited nodes_pruned n_classes counts class_lengths solution metrics"},
        "gpus_active": gpus_active, "comm_nranks": comm,
        "clocks": clocks,
        "gen_s": round(gen_s, 1),
    }
    if parity_ok is False:
        line["parity"]["mismatched"] = bad
    print(json.dumps(line), flush=True)
    return 0 if parity_ok is not False else 1


def run_config4(args, world, rank, local):
    """Brute force (exhaustive_optimal subsets mode, dftsp.py:288-313) at K =
    --brute-k over the adversarial family, every level's rank range sharded
    over the ranks; one 8-byte all-reduce(MIN) per live level."""
    import torch
    torch.cuda.set_device(local)
    from paper_2405_07140_b200 import brute, synth
    K = args.brute_k
    insts = synth.brute_family(K, args.brute_n, seed=2405_07140)
    clk = ClockSampler(local).start()
    for rec, cols in insts[:min(len(insts), max(1, args.warmup))]:
        brute.solve_distributed(rec, cols) if world > 1 else brute.solve_sharded(rec, cols, 1, device=local)
    barrier(world)
    torch.cuda.synchronize()
    clk.begin()
    stats0 = brute.enum_stats(local)
    t0 = time.perf_counter()
    out = []
    for _ in range(args.steps):
        for rec, cols in insts:
            r = brute.solve_distributed(rec, cols) if world > 1 else brute.solve_sharded(rec, cols, 1, device=local)
            out.append((r.z, r.lexrank, r.nodes_visited, r.mask))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    clk.end()
    stats = brute.enum_stats(local) - stats0
    wall = max_over_ranks(wall, world, torch.device("cuda", local))
    checked = torch.tensor([float(stats[0]), float(stats[1])], dtype=torch.float64, device=torch.device("cuda", local))
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(checked)
    clocks = clk.summary()
    gpus_active, comm = ranks_info(world, torch.device("cuda", local))
    if rank != 0:
        return 0
    # parity sample against the literal C scan (oracle/, test-only checker):
    # the answer's rank is feasible at its level, and the 2^16 ranks before it
    # are not (tests/test_gpu_brute_large.py checks whole levels)
    parity = None
    if not args.no_cpu:
        import oracle
        bad, cpu_n, cpu_s = [], 0, 0.0
        for i, ((rec, cols), o) in enumerate(zip(insts, out[:len(insts)])):
            z, r = int(o[0]), int(o[1])
            if z == 0:
                continue
            level = oracle.level_evaluator(rec, cols)
            t1 = time.perf_counter()
            below = level(z, max(0, r - (1 << 16)), r)
            cpu_s += time.perf_counter() - t1
            cpu_n += r - max(0, r - (1 << 16))
            if level(z, r, r + 1) != r or below != -1:
                bad.append(i)
        parity = {"ok": not bad, "instances": len(insts),
                  "check": "C restatement (oracle/): rank r* feasible at level z*, ranks [r*-2^16, r*) infeasible"}
        if bad:
            parity["mismatched"] = bad
        cpu4 = {"value": round(cpu_n / cpu_s, 1) if cpu_s > 0 else None, "unit": "checked subsets/s", "cores": 1,
                "kind": "port", "sample": f"{cpu_n} ranks just below each answer (the parity sample), literal "
                                          "check_direct scan of the C restatement (oracle/), one thread"}
    n_solved = args.steps * len(insts)
    line = {"metric": "brute-force exhaustive_optimal instances/sec (K=%d) and checked subsets/sec" % K,
            "value": round(n_solved / wall, 4), "unit": "instances/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(wall / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config4: brute force 2^K, K={K}, adversarial family (synth.brute_family)",
                       "instances_per_step": len(insts), "parallelism": f"subset-rank-sharded x{world}"},
            "checked_subsets_per_s": round(float(checked[0].item()) / wall, 1),
            "pruned_prefixes_per_s": round(float(checked[1].item()) / wall, 1),
            "reference_nodes_per_s": round(sum(o[2] for o in out[:len(insts)]) * args.steps / wall, 1),
            "results": [list(o) for o in out[:len(insts)]], "parity": parity,
            "cpu_baseline": cpu4 if parity is not None else None,
            "gpus_active": gpus_active, "comm_nranks": comm, "clocks": clocks}
    if parity is not None and not parity["ok"]:
        line["value"] = None
    print(json.dumps(line), flush=True)
    return 0 if parity is None or parity["ok"] else 1


if __name__ == "__main__":
    sys.exit(main())
