"""Lock-step batched simulator: many (scenario, seed) runs, one device launch per epoch step.

The reference simulator (``sim.run``, reference sim.py:277-412) is the hot
path's real caller: every epoch it filters the queue (sim.py:264-274), calls
``dftsp`` / ``exhaustive_optimal`` / ``stb_schedule`` / ``nob_assign``, then
charges ``batch_cost`` and checks completions.  Epoch e+1 depends on epoch
e's decision, so one run is sequential -- but independent runs (sweep points,
seeds) are not.  ``run_many`` advances all runs in lock-step and, at each
epoch, issues each device entry point once for every run that needs it
(admission, DFTSP with its compare-pruning twin, brute force / verify-oracle,
StB, NoB, batch cost, the debug re-check).  Host code only does the
reference's bookkeeping (arrivals, expiry, waiting times, completion
accounting) with the same float expressions, so metrics and traces equal the
reference's exactly (tests/test_gpu_sweep.py against sim runs recorded from
the reference).

Workloads are generated on the host with the reference's numpy PCG64 streams
(``default_rng([seed, 11])`` / ``[seed, 22]``, sim.py:231-261, 283-284).
"""
from __future__ import annotations

import ctypes
import math
import time
from collections import deque
from dataclasses import dataclass, field, fields

import numpy as np

from . import _lib
from .baselines import static_batch_size
from .catalog import delta_ppl, get_model, get_profile, load_catalog
from .costs import NodeCompute
from .feasibility import EdgeContext, Request, leq, raise_for_status
from .radio import RadioConfig, UserLink, dbm_to_watts
from .soa import InstanceBatch, context_record, request_columns, requests_struct
from .search import solve_batch

SCHEDULERS = ("dftsp", "stb", "nob", "brute")
CHANNEL_MODES = ("per_user", "shared")


class ConfigError(ValueError):
    """A scenario field failed validation (reference sim.py:30-31)."""


@dataclass
class Scenario:
    """Resolved description of one simulation run (reference sim.py:35-80)."""

    model: str = "bloom-3b"
    quant_profile: str = "w8a16"
    scheduler: str = "dftsp"
    seed: int = 0
    arrival_rate: float = 50.0
    duration: float = 20.0
    epoch_s: float = 2.0
    uplink_bandwidth_hz: float = 20e6
    downlink_bandwidth_hz: float = 20e6
    uplink_power_dbm: float = 20.0
    downlink_power_dbm: float = 43.0
    noise_density_dbm_hz: float = -174.0
    uplink_slot_s: float = 0.25
    downlink_slot_s: float = 0.25
    bits_per_token: int = 16
    mean_channel_gain: float = 1e-3
    channel_mode: str = "per_user"
    gpu_count: int = 20
    flops_per_gpu: float = 1.33e12
    memory_per_gpu_bytes: float = 32e9
    output_classes: tuple = (128, 256, 512)
    prompt_choices: tuple = (128, 256, 512)
    deadline_range_s: tuple = (0.5, 2.0)
    deadline_scale: float = 1.0
    tolerance_cap: float = 1.0
    pruning: bool = True
    inclusive_prune_bound: bool = False
    exact_tau: bool = False
    accuracy_check: bool = True
    admission_prefilter: bool = True
    compute_slot_cap: bool = True
    compare_pruning: bool = False
    compare_stride: int = 1
    verify_oracle: bool = False
    oracle_cap: int = 16
    debug_checks: bool = True
    catalog_config: dict = field(default_factory=dict)

    @classmethod
    def from_mapping(cls, m: dict) -> "Scenario":
        names = {f.name for f in fields(cls)}
        kw = {k: (tuple(v) if isinstance(v, list) else v) for k, v in m.items() if k in names}
        return cls(**kw)

    def validate(self) -> None:
        """Field checks of the reference (sim.py:82-125), same messages."""
        def need(ok, name, msg):
            if not ok:
                raise ConfigError(f"{name}: {msg}")
        need(self.arrival_rate >= 0, "arrival_rate", "must be >= 0")
        need(self.duration > 0, "duration", "must be > 0")
        need(self.epoch_s > 0, "epoch_s", "must be > 0")
        need(self.uplink_slot_s > 0, "uplink_slot_s", "must be > 0")
        need(self.downlink_slot_s > 0, "downlink_slot_s", "must be > 0")
        need(self.epoch_s >= self.uplink_slot_s + self.downlink_slot_s, "epoch_s",
             "must fit the uplink and downlink slots")
        need(self.uplink_bandwidth_hz > 0, "uplink_bandwidth_hz", "must be > 0")
        need(self.downlink_bandwidth_hz > 0, "downlink_bandwidth_hz", "must be > 0")
        need(self.bits_per_token >= 1, "bits_per_token", "must be >= 1")
        need(self.mean_channel_gain > 0, "mean_channel_gain", "must be > 0")
        need(self.channel_mode in CHANNEL_MODES, "channel_mode", f"must be one of {CHANNEL_MODES}")
        need(self.gpu_count >= 1, "gpu_count", "must be >= 1")
        need(self.flops_per_gpu > 0, "flops_per_gpu", "must be > 0")
        need(self.memory_per_gpu_bytes > 0, "memory_per_gpu_bytes", "must be > 0")
        need(len(self.output_classes) > 0, "output_classes", "must be nonempty")
        need(all(n >= 1 for n in self.output_classes), "output_classes", "entries must be >= 1")
        need(list(self.output_classes) == sorted(set(self.output_classes)), "output_classes",
             "must be strictly increasing")
        need(len(self.prompt_choices) > 0, "prompt_choices", "must be nonempty")
        need(all(s >= 1 for s in self.prompt_choices), "prompt_choices", "entries must be >= 1")
        lo, hi = self.deadline_range_s
        need(0 < lo <= hi, "deadline_range_s", "must satisfy 0 < low <= high")
        need(self.deadline_scale > 0, "deadline_scale", "must be > 0")
        need(self.tolerance_cap >= 0, "tolerance_cap", "must be >= 0")
        need(self.scheduler in SCHEDULERS, "scheduler", f"must be one of {SCHEDULERS}")
        need(self.compare_stride >= 1, "compare_stride", "must be >= 1")
        need(self.oracle_cap >= 1, "oracle_cap", "must be >= 1")
        try:
            llm, quant = self.resolve_catalog()
        except (KeyError, ValueError) as exc:
            raise ConfigError(f"model/quant_profile: {exc}") from exc
        try:
            delta_ppl(quant, llm.name)
        except KeyError as exc:
            raise ConfigError(f"quant_profile: {exc}") from exc

    def resolve_catalog(self):
        """Model and quantization profile with catalog overrides (sim.py:128-133)."""
        extra_m, extra_p = load_catalog(self.catalog_config or {})
        return get_model(self.model, extra_m), get_profile(self.quant_profile, extra_p)


@dataclass
class EpochTrace:
    """Per-epoch instrumentation row (sim.py:178-195)."""

    epoch: int
    t_s: float
    queue_len: int
    candidates: int
    batch: int
    nodes_visited: int
    nodes_pruned: int
    nodes_visited_noprune: int | None
    memory_bytes: float
    latency_s: float
    completed: int
    missed_expired: int
    missed_late: int


@dataclass
class SimMetrics:
    """Counters and per-epoch trace of one run (sim.py:197-222), plus the
    run's failure (``error``/``exception``; None when it completed)."""

    duration_s: float = 0.0
    epochs: int = 0
    generated: int = 0
    scheduled_total: int = 0
    completed_total: int = 0
    missed_expired: int = 0
    missed_late: int = 0
    dropped_total: int = 0
    still_queued: int = 0
    throughput: float = 0.0
    nodes_visited_total: int = 0
    nodes_pruned_total: int = 0
    cmp_nodes_with_pruning: int | None = None
    cmp_nodes_without_pruning: int | None = None
    oracle_checks: int = 0
    oracle_mismatches: int = 0
    trace: list = field(default_factory=list)
    error: str | None = field(default=None, compare=False)
    exception: BaseException | None = field(default=None, compare=False, repr=False)

    @property
    def missed_total(self) -> int:
        return self.missed_expired + self.missed_late


def generate_workload(sc: Scenario, rng) -> list:
    """Time-ordered request stream, the reference's draw order (sim.py:231-261)."""
    out = []
    if sc.arrival_rate <= 0:
        return out
    p_up = dbm_to_watts(sc.uplink_power_dbm)
    lo, hi = sc.deadline_range_s
    # Same PCG64 draws, cheaper calls: Generator.choice(seq) draws
    # integers(0, len(seq)), and uniform(lo, hi) is lo + (hi - lo) * random()
    # (numpy random_uniform); both checked stream-for-stream in tests/test_sweep.py.
    prompts, outputs = tuple(sc.prompt_choices), tuple(sc.output_classes)
    npr, nout = len(prompts), len(outputs)
    span = hi - lo
    scale = 1.0 / sc.arrival_rate
    exp, integers, rand = rng.exponential, rng.integers, rng.random
    t = 0.0
    i = 0
    while True:
        t += exp(scale)
        if t >= sc.duration:
            break
        prompt = int(prompts[integers(0, npr)])
        output = int(outputs[integers(0, nout)])
        deadline = sc.deadline_scale * float(lo + span * rand())
        tolerance = sc.tolerance_cap * float(0.0 + (1.0 - 0.0) * rand())
        gain = float(exp(sc.mean_channel_gain))
        out.append(Request(id=i, prompt_tokens=prompt, output_tokens=output, deadline_s=deadline,
                           tolerance=tolerance, link=UserLink(gain, p_up), arrival_s=t))
        i += 1
    return out


@dataclass
class _Run:
    sc: Scenario
    ctx: EdgeContext
    delta: float
    rec: np.ndarray
    pending: deque
    chan_rng: object
    p_up: float
    ladder: tuple
    nepochs: int
    oracle_stride: int
    stb_b: int = 0
    busy: list | None = None
    queue: list = field(default_factory=list)
    metrics: dict = field(default_factory=dict)
    trace: list = field(default_factory=list)
    error: str | None = None
    exc: BaseException | None = None


def _start(sc: Scenario) -> _Run:
    sc.validate()
    llm, quant = sc.resolve_catalog()
    radio = RadioConfig(uplink_band_hz=sc.uplink_bandwidth_hz, downlink_band_hz=sc.downlink_bandwidth_hz,
                        downlink_power_w=dbm_to_watts(sc.downlink_power_dbm),
                        noise_density_w_hz=dbm_to_watts(sc.noise_density_dbm_hz),
                        uplink_slot_s=sc.uplink_slot_s, downlink_slot_s=sc.downlink_slot_s,
                        bits_per_token=sc.bits_per_token)
    node = NodeCompute(flops_per_s=sc.gpu_count * sc.flops_per_gpu,
                       memory_bytes=sc.gpu_count * sc.memory_per_gpu_bytes, gpu_count=sc.gpu_count)
    ctx = EdgeContext(llm=llm, quant=quant, radio=radio, node=node,
                      slot_cap_s=sc.epoch_s if sc.compute_slot_cap else None)
    delta = delta_ppl(quant, llm.name)
    workload = generate_workload(sc, np.random.default_rng([sc.seed, 11]))
    nepochs = max(1, math.ceil(sc.duration / sc.epoch_s))
    run = _Run(sc=sc, ctx=ctx, delta=delta, rec=context_record(ctx, delta), pending=deque(workload),
               chan_rng=np.random.default_rng([sc.seed, 22]), p_up=dbm_to_watts(sc.uplink_power_dbm),
               ladder=tuple(sc.output_classes), nepochs=nepochs, oracle_stride=max(1, nepochs // 4))
    run.metrics = dict(duration_s=sc.duration, epochs=nepochs, generated=len(workload), scheduled_total=0,
                       completed_total=0, missed_expired=0, missed_late=0, dropped_total=0, still_queued=0,
                       throughput=0.0, nodes_visited_total=0, nodes_pruned_total=0,
                       cmp_nodes_with_pruning=0 if (sc.compare_pruning and sc.scheduler == "dftsp") else None,
                       cmp_nodes_without_pruning=0 if (sc.compare_pruning and sc.scheduler == "dftsp") else None,
                       oracle_checks=0, oracle_mismatches=0)
    if sc.scheduler == "stb":
        run.stb_b = static_batch_size(llm, quant, node, sc.epoch_s, max(sc.prompt_choices), max(sc.output_classes))
    if sc.scheduler == "nob":
        run.busy = [0.0] * sc.gpu_count
    return run


def _ref(s):
    return ctypes.cast(ctypes.pointer(s), ctypes.c_void_p)


def _pack(pools, runs):
    """InstanceBatch over pools (lists of Requests), one context per run."""
    recs = np.concatenate([r.rec for r in runs])
    return InstanceBatch.from_pools(pools, recs, np.arange(len(runs), dtype=np.int32))


def _fail(run, exc) -> None:
    """The reference's run() would raise here: the run stops, the others go on."""
    if run.error is None:
        run.error = f"{type(exc).__name__}: {exc}"
        run.exc = exc


def _raise_status(run, status, pool=None, err_index=-1, ladder=None) -> bool:
    if not status:
        return False
    try:
        if status == _lib.ERR_INVALID_ARG:
            raise ValueError("delta and tolerance must be nonnegative")
        raise_for_status(int(status), pool, int(err_index), run.ctx, ladder)
    except (ValueError, RuntimeError) as exc:
        _fail(run, exc)
        return True
    return False


def _admission(runs, queues, acc, pre, h):
    """_dftsp_candidates (sim.py:264-274) for runs sharing (accuracy_check, admission_prefilter)."""
    b = _pack(queues, runs)
    st = np.zeros(max(b.n_req, 1), np.int32)
    keep = np.zeros(max(b.n_req, 1), np.uint8)
    if b.n_req:
        _lib.check(h.lib.eb_admission_batch(h.ptr, b.contexts.ctypes.data, len(b.contexts), _ref(b.struct()),
                                            int(acc), int(pre), st.ctypes.data, keep.ctypes.data,
                                            _lib.EB_MEM_HOST), "eb_admission_batch")
    out = []
    for i, (r, q) in enumerate(zip(runs, queues)):
        lo = int(b.offsets[i])
        bad = next((int(v) for v in st[lo:lo + len(q)] if v), 0)
        if _raise_status(r, bad):
            out.append(None)
            continue
        out.append([x for x, k in zip(q, keep[lo:lo + len(q)]) if k])
    return out


def _dftsp(runs, pools, pruning, h):
    """dftsp(cands, ctx, ladder, pruning, ...) (dftsp.py:204-285): one eb_dftsp_batch per
    (ladder, inclusive_bound, exact_tau) group; per run (solution, z, nodes_visited, nodes_pruned)."""
    res = [None] * len(runs)
    groups: dict = {}
    for i, r in enumerate(runs):
        groups.setdefault((r.ladder, r.sc.inclusive_prune_bound, r.sc.exact_tau), []).append(i)
    for (ladder, incl, exact), idx in groups.items():
        b = _pack([pools[i] for i in idx], [runs[i] for i in idx])
        out = solve_batch(b, pruning=pruning, inclusive_bound=incl, exact_tau=exact, ladder=ladder, handle=h)
        for j, i in enumerate(idx):
            if _raise_status(runs[i], int(out.status[j]), pools[i], int(out.error_index[j]), ladder):
                continue
            z = int(out.z_found[j])
            lo = int(b.offsets[j])
            sol = [pools[i][int(k)] for k in out.solution[lo:lo + z]] if z else []
            res[i] = (sol, z, int(out.nodes_visited[j]), int(out.nodes_pruned[j]))
    return res


def _exhaustive(runs, pools, h):
    """exhaustive_optimal(cands, ctx, cap) (dftsp.py:288-332) per run; an empty pool visits nothing."""
    out = [([], 0, 0, 0)] * len(pools)
    idx = [i for i, p in enumerate(pools) if p]
    if not idx:
        return out
    b = _pack([pools[i] for i in idx], [runs[i] for i in idx])
    n = b.n_inst
    st = np.zeros(n, np.int32); z = np.zeros(n, np.int32); rk = np.zeros(n, np.int64)
    nodes = np.zeros(n, np.int64); mask = np.zeros(n, np.uint64)
    _lib.check(h.lib.eb_exhaustive_batch(h.ptr, b.contexts.ctypes.data, len(b.contexts), _ref(b.struct()),
                                         _lib.EB_MAX_K, st.ctypes.data, z.ctypes.data, rk.ctypes.data,
                                         nodes.ctypes.data, mask.ctypes.data, _lib.EB_MEM_HOST),
               "eb_exhaustive_batch")
    for j, i in enumerate(idx):
        p = pools[i]
        if _raise_status(runs[i], int(st[j]), p):
            out[i] = None
            continue
        m = int(mask[j])
        chosen = sorted((x for k, x in enumerate(p) if (m >> k) & 1), key=lambda x: x.id) if z[j] else []
        out[i] = (chosen, int(z[j]), int(nodes[j]), 0)
    return out


def _stb(runs, queues, h):
    """stb_schedule(queue, b, ctx, delta, accuracy_check) (baselines.py:68-87) per run."""
    out = [None] * len(runs)
    for acc in (True, False):
        idx = [i for i, r in enumerate(runs) if bool(r.sc.accuracy_check) == acc]
        if not idx:
            continue
        b = _pack([queues[i] for i in idx], [runs[i] for i in idx])
        bb = np.array([runs[i].stb_b for i in idx], np.int64)
        st = np.zeros(len(idx), np.int32)
        sel = np.zeros(max(b.n_req, 1), np.uint8)
        _lib.check(h.lib.eb_stb_batch(h.ptr, b.contexts.ctypes.data, len(b.contexts), _ref(b.struct()),
                                      bb.ctypes.data, int(acc), st.ctypes.data, sel.ctypes.data, _lib.EB_MEM_HOST),
                   "eb_stb_batch")
        for j, i in enumerate(idx):
            if _raise_status(runs[i], int(st[j])):
                continue
            lo = int(b.offsets[j])
            out[i] = [x for x, s in zip(queues[i], sel[lo:lo + len(queues[i])]) if s]
    return out


def _nob(runs, queues, now, h):
    """nob_assign(queue, pool, t_e, ctx, delta, accuracy_check) (baselines.py:90-121) per run;
    each run's GpuPool.busy_until lives in ``run.busy``."""
    out = [None] * len(runs)
    for acc in (True, False):
        idx = [i for i, r in enumerate(runs) if bool(r.sc.accuracy_check) == acc]
        if not idx:
            continue
        b = _pack([queues[i] for i in idx], [runs[i] for i in idx])
        maxd = max(runs[i].sc.gpu_count for i in idx)
        busy = np.zeros((len(idx), maxd))
        for j, i in enumerate(idx):
            busy[j, :len(runs[i].busy)] = runs[i].busy
        nw = np.array([now[i] for i in idx], np.float64)
        st = np.zeros(len(idx), np.int32)
        nr = max(b.n_req, 1)
        act = np.zeros(nr, np.int8); comp = np.zeros(nr); order = np.zeros(nr, np.int32)
        _lib.check(h.lib.eb_nob_batch(h.ptr, b.contexts.ctypes.data, len(b.contexts), _ref(b.struct()),
                                      nw.ctypes.data, int(acc), None, maxd, busy.ctypes.data, st.ctypes.data,
                                      act.ctypes.data, comp.ctypes.data, order.ctypes.data, _lib.EB_MEM_HOST),
                   "eb_nob_batch")
        for j, i in enumerate(idx):
            r = runs[i]
            if _raise_status(r, int(st[j])):
                continue
            r.busy = [float(v) for v in busy[j, :len(r.busy)]]
            lo = int(b.offsets[j])
            sched, comps, dropped = [], [], []
            for k, req in enumerate(queues[i]):
                a = act[lo + k]
                if a == 1:
                    sched.append(req)
                    comps.append(float(comp[lo + k]))
                elif a == 2:
                    dropped.append((req, "exceeds per-device memory"))
            out[i] = (sched, comps, dropped)
    return out


def _costs_and_checks(runs, batches, debug_flags, h):
    """batch_cost at the batch's own padding (sim.py:363-371) and the debug
    check_direct re-verification (sim.py:372-374), one launch each."""
    n = len(batches)
    recs = np.concatenate([r.rec for r in runs])
    off = np.zeros(n + 1, np.int64)
    np.cumsum([len(bt) for bt in batches], out=off[1:])
    pa = np.array([x.prompt_tokens for bt in batches for x in bt], np.int32)
    oa = np.array([x.output_tokens for bt in batches for x in bt], np.int32)
    pad = np.array([max(x.prompt_tokens for x in bt) for bt in batches], np.int64)
    pc = np.arange(n, dtype=np.int32)
    cost = np.zeros((n, 2))
    _lib.check(h.lib.eb_batch_cost_batch(h.ptr, recs.ctypes.data, n, n, off.ctypes.data, pa.ctypes.data,
                                         oa.ctypes.data, pad.ctypes.data, None, pc.ctypes.data, cost.ctypes.data,
                                         _lib.EB_MEM_HOST), "eb_batch_cost_batch")
    ok = np.ones(n, bool)
    st = np.zeros(n, np.int32)
    chk = [i for i in range(n) if debug_flags[i]]
    if chk:
        rows = [x for i in chk for x in batches[i]]
        soff = np.zeros(len(chk) + 1, np.int64)
        np.cumsum([len(batches[i]) for i in chk], out=soff[1:])
        members = np.arange(len(rows), dtype=np.int32)
        sc = np.array(chk, np.int32)
        spad = pad[chk]
        cst = np.zeros(len(chk), np.int32)
        okc = np.zeros(len(chk), np.uint8)
        cols = request_columns(rows)
        _lib.check(h.lib.eb_check_direct_batch(h.ptr, recs.ctypes.data, n, _ref(requests_struct(cols)),
                                               len(rows), len(chk), soff.ctypes.data, members.ctypes.data,
                                               sc.ctypes.data, spad.ctypes.data, cst.ctypes.data, okc.ctypes.data,
                                               None, _lib.EB_MEM_HOST), "eb_check_direct_batch")
        for j, i in enumerate(chk):
            ok[i], st[i] = bool(okc[j]), cst[j]
    return cost, ok, st


def _handle(device):
    return _lib.handle(device)


_PROFILE: dict | None = None


def _tick(name, t0):
    if _PROFILE is not None:
        _PROFILE[name] = _PROFILE.get(name, 0.0) + time.perf_counter() - t0


def _t(name, fn):
    """fn, timed into the run_many(profile=...) dict (wall seconds, host packing + device call)."""
    if _PROFILE is None:
        return fn

    def timed(*a):
        t0 = time.perf_counter()
        try:
            return fn(*a)
        finally:
            _tick(name, t0)
    return timed


def run_many(scenarios, device=None, profile: dict | None = None) -> list:
    """Simulate every scenario in lock-step (each one exactly as sim.run, sim.py:277-412).

    Returns one dict per scenario: the SimMetrics fields (sim.py:206-222),
    ``trace`` (EpochTrace rows, sim.py:190-203, as dicts) and ``error``:
    None, or the exception the reference's ``run`` raises for that scenario
    (ConfigError, a search/link ValueError, the compare-pruning or
    debug-check RuntimeError) -- the other runs continue.  ``profile``: a
    dict that receives wall seconds per phase."""
    global _PROFILE
    _PROFILE = profile
    try:
        return _run_many(scenarios, device)
    finally:
        _PROFILE = None


def _run_many(scenarios, device):
    h = _handle(device)
    runs, failed = [], {}
    for k, sc in enumerate(scenarios):
        sc = Scenario.from_mapping(sc) if isinstance(sc, dict) else sc
        try:
            runs.append(_start(sc))
        except ValueError as exc:                     # ConfigError and friends; device errors propagate
            failed[k] = exc
            runs.append(None)
    live_runs = [r for r in runs if r is not None]
    max_epochs = max((r.nepochs for r in live_runs), default=0)
    for e in range(1, max_epochs + 1):
        live = [r for r in live_runs if e <= r.nepochs and r.error is None]
        if not live:
            break
        t0 = time.perf_counter()
        step = {id(r): _arrivals(r, e) for r in live}
        _tick("host_arrivals", t0)
        _epoch(live, step, e, h)
        t0 = time.perf_counter()
        for r in live:
            if r.error is None:
                _account(r, step[id(r)], e)
        _tick("host_accounting", t0)
    out = []
    for k, r in enumerate(runs):
        if r is None:
            exc = failed[k]
            out.append(SimMetrics(error=f"{type(exc).__name__}: {exc}", exception=exc))
            continue
        m = SimMetrics(**r.metrics, trace=[EpochTrace(**row) for row in r.trace], error=r.error, exception=r.exc)
        m.still_queued = len(r.queue) + len(r.pending)
        m.throughput = m.completed_total / r.sc.duration
        out.append(m)
    return out


def run(sc) -> "SimMetrics":
    """One scenario, exactly as the reference's ``run`` (sim.py:277-412): its
    metrics, or the exception it raises."""
    m = run_many([sc])[0]
    if m.exception is not None:
        raise m.exception
    return m


def complexity_reduction(with_pruning, without_pruning):
    """Node-count reduction in percent; None when no comparison is available (sim.py:224-228)."""
    if with_pruning is None or without_pruning is None or without_pruning <= 0:
        return None
    return 100.0 * (1.0 - with_pruning / without_pruning)


def _arrivals(r, e) -> dict:
    """Arrivals, expiry, shared-channel redraw and waiting times (sim.py:303-321)."""
    sc = r.sc
    t_e = e * sc.epoch_s
    while r.pending and r.pending[0].arrival_s < t_e:
        r.queue.append(r.pending.popleft())
    alive, expired = [], 0
    for q in r.queue:
        if q.arrival_s + q.deadline_s <= t_e:
            expired += 1
        else:
            alive.append(q)
    r.queue = alive
    r.metrics["missed_expired"] += expired
    if sc.channel_mode == "shared":
        gain = float(r.chan_rng.exponential(sc.mean_channel_gain))
        for q in r.queue:
            q.link = UserLink(gain, r.p_up)
    for q in r.queue:
        q.waiting_s = t_e - q.arrival_s
    return dict(t_e=t_e, expired=expired, queue_len=len(r.queue), batch=[], completions=[], dropped=[],
                stats=None, cands=r.queue, trace_np=None)


def _epoch(live, step, e, h):
    """One scheduling decision for every live run (sim.py:323-378), batched per entry point."""
    ok = lambda rs: [r for r in rs if r.error is None]      # noqa: E731
    by = {s: [r for r in live if r.sc.scheduler == s] for s in SCHEDULERS}
    groups: dict = {}
    for r in by["dftsp"] + by["brute"]:
        groups.setdefault((bool(r.sc.accuracy_check), bool(r.sc.admission_prefilter)), []).append(r)
    for (acc, pre), rs in groups.items():
        cands = _t("admission", _admission)(rs, [r.queue for r in rs], acc, pre, h) if (acc or pre) else [list(r.queue) for r in rs]
        for r, c in zip(rs, cands):
            if c is not None:
                step[id(r)]["cands"] = c

    rs = ok(by["dftsp"])
    for pruning in (True, False):
        grp = [r for r in rs if bool(r.sc.pruning) == pruning]
        if grp:
            for r, o in zip(grp, _t("dftsp", _dftsp)(grp, [step[id(r)]["cands"] for r in grp], pruning, h)):
                if o is not None:
                    step[id(r)]["stats"], step[id(r)]["batch"] = o, o[0]
    rs = ok(rs)
    cmp = [r for r in rs if r.sc.compare_pruning and (e - 1) % r.sc.compare_stride == 0]
    if cmp:
        for r, o in zip(cmp, _t("dftsp_compare", _dftsp)(cmp, [step[id(r)]["cands"] for r in cmp], False, h)):
            if o is None:
                continue
            st = step[id(r)]
            if o[1] != st["stats"][1]:
                _fail(r, RuntimeError("pruned and unpruned searches disagree on batch size"))
                continue
            st["cmp"] = (st["stats"][2], o[2])
            st["trace_np"] = o[2]
    orc = [r for r in ok(rs) if r.sc.verify_oracle and (e - 1) % r.oracle_stride == 0
           and len(step[id(r)]["cands"]) <= r.sc.oracle_cap]
    if orc:
        for r, o in zip(orc, _t("verify_oracle", _exhaustive)(orc, [step[id(r)]["cands"] for r in orc], h)):
            if o is not None:
                step[id(r)]["oracle"] = o[1]

    rs = []
    for r in ok(by["brute"]):
        n = len(step[id(r)]["cands"])
        if n > r.sc.oracle_cap:
            _fail(r, ConfigError(f"scheduler: brute refuses {n} candidates (cap {r.sc.oracle_cap})"))
        else:
            rs.append(r)
    if rs:
        for r, o in zip(rs, _t("brute", _exhaustive)(rs, [step[id(r)]["cands"] for r in rs], h)):
            if o is not None:
                step[id(r)]["stats"], step[id(r)]["batch"] = o, o[0]

    rs = by["stb"]
    if rs:
        for r, sel in zip(rs, _t("stb", _stb)(rs, [r.queue for r in rs], h)):
            if sel is not None:
                step[id(r)]["batch"] = sel
    rs = by["nob"]
    if rs:
        for r, o in zip(rs, _t("nob", _nob)(rs, [r.queue for r in rs], [step[id(r)]["t_e"] for r in rs], h)):
            if o is not None:
                st = step[id(r)]
                st["batch"], st["completions"], st["dropped"] = o

    costed = [r for r in ok(live) if step[id(r)]["batch"] and r.sc.scheduler != "nob"]
    if costed:
        cost, good, status = _t("cost_check", _costs_and_checks)(
            costed, [step[id(r)]["batch"] for r in costed],
            [r.sc.debug_checks and r.sc.scheduler in ("dftsp", "brute") for r in costed], h)
        for i, r in enumerate(costed):
            if _raise_status(r, int(status[i]), step[id(r)]["batch"]):
                continue
            if not good[i]:
                _fail(r, RuntimeError("scheduled batch violates the direct check"))
                continue
            st = step[id(r)]
            st["mem"], st["lat"] = float(cost[i, 0]), float(cost[i, 1])
            radio = r.ctx.radio
            done = st["t_e"] + radio.uplink_slot_s + st["lat"] + radio.downlink_slot_s
            st["completions"] = [done] * len(st["batch"])


def _account(r, st, e):
    """Completion accounting and the EpochTrace row (sim.py:376-408)."""
    m = r.metrics
    batch = st["batch"]
    completed = late = 0
    for q, done in zip(batch, st["completions"]):
        if leq(done - q.arrival_s, q.deadline_s):
            completed += 1
        else:
            late += 1
    m["scheduled_total"] += len(batch)
    m["completed_total"] += completed
    m["missed_late"] += late
    m["dropped_total"] += len(st["dropped"])
    gone = {id(q) for q in batch}
    gone.update(id(q) for q, _ in st["dropped"])
    r.queue = [q for q in r.queue if id(q) not in gone]
    stats = st["stats"]
    if "cmp" in st:
        m["cmp_nodes_with_pruning"] += st["cmp"][0]
        m["cmp_nodes_without_pruning"] += st["cmp"][1]
    if "oracle" in st:
        m["oracle_checks"] += 1
        if st["oracle"] != stats[1]:
            m["oracle_mismatches"] += 1
    nv = stats[2] if stats else 0
    npr = stats[3] if stats else 0
    m["nodes_visited_total"] += nv
    m["nodes_pruned_total"] += npr
    r.trace.append(dict(epoch=e, t_s=st["t_e"], queue_len=st["queue_len"],
                        candidates=len(st["cands"]) if r.sc.scheduler in ("dftsp", "brute") else st["queue_len"],
                        batch=len(batch), nodes_visited=nv, nodes_pruned=npr, nodes_visited_noprune=st["trace_np"],
                        memory_bytes=st.get("mem", 0.0), latency_s=st.get("lat", 0.0), completed=completed,
                        missed_expired=st["expired"], missed_late=late))


# ---- parameter sweeps and emission (reference cli.py:27-322) -------------
# The reference's run_sweep runs every (value, seed) point through sim.run,
# one process per point; here every point is one run of a single lock-step
# run_many, so each epoch's searches of all points share one launch.

SWEEP_AXES = ("arrival_rate", "deadline_scale", "tolerance_cap", "quant_profile", "model", "scheduler")
_NUMERIC_AXES = {"arrival_rate", "deadline_scale", "tolerance_cap"}
COLUMNS = (
    "kind", "axis", "value", "seed", "scheduler", "model", "quant_profile",
    "throughput", "completed", "scheduled", "missed", "dropped", "still_queued",
    "generated", "nodes_visited", "nodes_pruned", "cmp_nodes_with",
    "cmp_nodes_without", "reduction_pct", "oracle_checks", "oracle_mismatches",
    "error", "config_hash",
)
_AGGREGATE_FIELDS = (
    "throughput", "completed", "scheduled", "missed", "dropped", "still_queued",
    "generated", "nodes_visited", "nodes_pruned", "cmp_nodes_with",
    "cmp_nodes_without", "reduction_pct",
)


@dataclass(frozen=True)
class SweepSpec:
    """One swept axis: scenario knob, its values, seeds per value (cli.py:46-60)."""

    axis: str
    values: tuple
    repetitions: int = 1

    def __post_init__(self):
        if self.axis not in SWEEP_AXES:
            raise ConfigError(f"sweep.axis: must be one of {SWEEP_AXES}")
        if not self.values:
            raise ConfigError("sweep.values: must be nonempty")
        if self.repetitions < 1:
            raise ConfigError("sweep.repetitions: must be >= 1")


def resolved_mapping(sc: Scenario) -> dict:
    """Every resolved scenario field, tuples as lists (sim.py:166-175)."""
    out = {}
    for f in fields(Scenario):
        v = getattr(sc, f.name)
        out[f.name] = list(v) if isinstance(v, tuple) else v
    return out


def config_hash(sc: Scenario) -> str:
    """Stable short hash of the resolved scenario, seed excluded (cli.py:189-194)."""
    import hashlib
    import json
    payload = resolved_mapping(sc)
    payload.pop("seed", None)
    blob = json.dumps(payload, sort_keys=True, separators=(",", ":"))
    return hashlib.sha256(blob.encode()).hexdigest()[:12]


def _fmt6(x):
    if x is None:
        return None
    if isinstance(x, (bool, int)):
        return x
    return float(f"{float(x):.6g}")


def apply_axis(sc: Scenario, axis: str, value) -> Scenario:
    """Scenario with one sweep axis overridden (cli.py:230-236)."""
    from dataclasses import replace
    return replace(sc, **{axis: float(value) if axis in _NUMERIC_AXES else str(value)})


def metrics_row(axis, value, sc: Scenario, m: "SimMetrics | None", error: str = "") -> dict:
    """One data row (cli.py:205-227)."""
    row = {name: None for name in COLUMNS}
    row.update(kind="data", axis=axis, value=value, seed=sc.seed, scheduler=sc.scheduler, model=sc.model,
               quant_profile=sc.quant_profile, error=error, config_hash=config_hash(sc))
    if m is not None:
        red = complexity_reduction(m.cmp_nodes_with_pruning, m.cmp_nodes_without_pruning)
        row.update(throughput=_fmt6(m.throughput), completed=m.completed_total, scheduled=m.scheduled_total,
                   missed=m.missed_total, dropped=m.dropped_total, still_queued=m.still_queued,
                   generated=m.generated, nodes_visited=m.nodes_visited_total, nodes_pruned=m.nodes_pruned_total,
                   cmp_nodes_with=m.cmp_nodes_with_pruning, cmp_nodes_without=m.cmp_nodes_without_pruning,
                   reduction_pct=_fmt6(red), oracle_checks=m.oracle_checks, oracle_mismatches=m.oracle_mismatches)
    return row


def run_sweep(sc: Scenario, spec: SweepSpec, device=None) -> list:
    """Every (value, seed) point plus per-value mean/std rows, as cli.run_sweep
    (cli.py:248-285), with all points simulated in one lock-step run_many."""
    from dataclasses import replace
    from statistics import mean, stdev
    points = []
    for value in spec.values:
        varied = apply_axis(sc, spec.axis, value)
        for rep in range(spec.repetitions):
            points.append((spec.axis, value, replace(varied, seed=sc.seed + rep)))
    results = run_many([p[2] for p in points], device=device)
    rows = []
    for (axis, value, psc), m in zip(points, results):
        if m.exception is not None:                  # per-row failure: recorded, sweep continues
            rows.append(metrics_row(axis, value, psc, None, error=str(m.exception)))
        else:
            rows.append(metrics_row(axis, value, psc, m))
    rows.sort(key=lambda r: (str(r["axis"]), str(r["value"]), r["seed"]))
    out = []
    for value in spec.values:
        group = [r for r in rows if r["value"] == value]
        out.extend(group)
        good = [r for r in group if not r["error"]]
        for kind, fn in (("mean", mean), ("std", lambda v: stdev(v) if len(v) > 1 else 0.0)):
            agg = {name: None for name in COLUMNS}
            agg.update(kind=kind, axis=spec.axis, value=value, seed=None,
                       scheduler=sc.scheduler if spec.axis != "scheduler" else value,
                       model=sc.model if spec.axis != "model" else value,
                       quant_profile=sc.quant_profile if spec.axis != "quant_profile" else value,
                       error="", config_hash=group[0]["config_hash"] if group else "")
            for name in _AGGREGATE_FIELDS:
                vals = [r[name] for r in good if r[name] is not None]
                agg[name] = _fmt6(fn(vals)) if vals else None
            out.append(agg)
    return out


def _cell(value) -> str:
    if value is None:
        return ""
    if isinstance(value, float):
        return f"{value:.6g}"
    return str(value)


def emit(table: list, fmt: str, path) -> None:
    """Result table as CSV or JSON with stable bytes (cli.py:297-312)."""
    import json
    from pathlib import Path
    if not table:
        raise ValueError("refusing to emit an empty table")
    if fmt not in ("csv", "json"):
        raise ValueError(f"unknown format {fmt!r}")
    path = Path(path)
    if fmt == "csv":
        lines = [",".join(COLUMNS)] + [",".join(_cell(row[n]) for n in COLUMNS) for row in table]
        path.write_text("\n".join(lines) + "\n")
    else:
        payload = {"columns": list(COLUMNS), "rows": [{n: row[n] for n in COLUMNS} for row in table]}
        path.write_text(json.dumps(payload, indent=2, sort_keys=True) + "\n")


def emit_trace(m: "SimMetrics", path) -> None:
    """Per-epoch trace of one run as CSV (cli.py:315-322)."""
    from pathlib import Path
    cols = tuple(f.name for f in fields(EpochTrace))
    lines = [",".join(cols)] + [",".join(_cell(_fmt6(getattr(row, c))) for c in cols) for row in m.trace]
    Path(path).write_text("\n".join(lines) + "\n")
