"""Test infrastructure: serve sweep.run_many's device entry points from the
CPU oracle, so the simulator's host bookkeeping can be checked against the
reference's recorded runs without a GPU (tests/test_sweep.py).  The GPU test
(tests/test_gpu_sweep.py) runs the real device path against the same runs."""
import numpy as np

import oracle
from paper_2405_07140_b200 import sweep
from paper_2405_07140_b200.feasibility import raise_for_status
from paper_2405_07140_b200.soa import request_columns

def _cols(reqs):
    return request_columns(reqs) if reqs else None


def _p(a):
    return a.ctypes.data


def _fail_status(run, st, pool=None):
    try:
        raise_for_status(int(st), pool, -1, run.ctx)
    except (ValueError, RuntimeError) as exc:
        sweep._fail(run, exc)


def _check_direct(run, reqs, padded):
    c = _cols(reqs)
    met = np.zeros(16)
    return oracle.load().oracle_check_direct(_p(run.rec), len(reqs), _p(c["prompt_tokens"]), _p(c["output_tokens"]),
                                             _p(c["deadline_s"]), _p(c["waiting_s"]), _p(c["channel_gain"]),
                                             _p(c["uplink_power_w"]), int(padded), _p(met))


def admission(runs, queues, acc, pre, h):
    out = []
    for r, q in zip(runs, queues):
        c = [x for x in q if r.delta <= x.tolerance] if acc else list(q)
        if pre:
            keep = []
            for x in c:
                v = _check_direct(r, [x], x.prompt_tokens)
                if v < 0:
                    _fail_status(r, -v, [x])
                    keep = None
                    break
                if v == 1:
                    keep.append(x)
            c = keep
        out.append(c)
    return out


def dftsp(runs, pools, pruning, h):
    out = []
    for r, p in zip(runs, pools):
        b = sweep._pack([p], [r])
        res = oracle.dftsp_batch(b, pruning=pruning, inclusive_bound=r.sc.inclusive_prune_bound,
                                 exact_tau=r.sc.exact_tau, ladder=r.ladder)
        st = int(res["status"][0])
        if st:
            _fail_status(r, st, p)
            out.append(None)
            continue
        z = int(res["z_found"][0])
        out.append(([p[int(k)] for k in res["solution"][:z]], z, int(res["nodes_visited"][0]),
                    int(res["nodes_pruned"][0])))
    return out


def exhaustive(runs, pools, h):
    out = []
    for r, p in zip(runs, pools):
        if not p:
            out.append(([], 0, 0, 0))
            continue
        cols = request_columns(p)
        st, z, rk, nodes, mask = oracle.exhaustive(r.rec, cols, 0, len(p), cap=64)
        if st:
            _fail_status(r, st, p)
            out.append(None)
            continue
        chosen = sorted((x for k, x in enumerate(p) if (mask >> k) & 1), key=lambda x: x.id) if z else []
        out.append((chosen, z, nodes, 0))
    return out


def stb(runs, queues, h):
    out = []
    for r, q in zip(runs, queues):
        if not q:
            out.append([])
            continue
        c = request_columns(q)
        sel = np.zeros(len(q), np.uint8)
        oracle.load().oracle_stb(_p(r.rec), len(q), _p(c["prompt_tokens"]), _p(c["output_tokens"]),
                                 _p(c["tolerance"]), _p(c["channel_gain"]), _p(c["uplink_power_w"]), int(r.stb_b),
                                 float(r.delta), int(bool(r.sc.accuracy_check)), _p(sel))
        out.append([x for x, s in zip(q, sel) if s])
    return out


def nob(runs, queues, now, h):
    out = []
    for r, q, t in zip(runs, queues, now):
        if not q:
            out.append(([], [], []))
            continue
        c = request_columns(q)
        busy = np.array(r.busy, np.float64)
        act = np.zeros(len(q), np.int8); comp = np.zeros(len(q)); order = np.zeros(len(q), np.int32)
        oracle.load().oracle_nob(_p(r.rec), len(q), _p(c["prompt_tokens"]), _p(c["output_tokens"]),
                                 _p(c["tolerance"]), float(t), float(r.delta), int(bool(r.sc.accuracy_check)),
                                 _p(busy), _p(act), _p(comp), _p(order))
        r.busy = [float(v) for v in busy]
        sched = [x for x, a in zip(q, act) if a == 1]
        comps = [float(v) for v, a in zip(comp, act) if a == 1]
        dropped = [(x, "exceeds per-device memory") for x, a in zip(q, act) if a == 2]
        out.append((sched, comps, dropped))
    return out


def costs_and_checks(runs, batches, debug_flags, h):
    n = len(batches)
    cost = np.zeros((n, 2))
    ok = np.ones(n, bool)
    st = np.zeros(n, np.int32)
    for i, (r, bt, dbg) in enumerate(zip(runs, batches, debug_flags)):
        pad = max(x.prompt_tokens for x in bt)
        s = np.array([x.prompt_tokens for x in bt], np.int32)
        o = np.array([x.output_tokens for x in bt], np.int32)
        out = np.zeros(2)
        oracle.load().oracle_batch_cost(_p(r.rec), len(bt), _p(s), _p(o), int(pad), 1, _p(out))
        cost[i] = out
        if dbg:
            v = _check_direct(r, bt, pad)
            if v < 0:
                st[i] = -v
            else:
                ok[i] = v == 1
    return cost, ok, st


def static_batch_size(spec, quant, node, slot_s, s_max, n_max):
    from paper_2405_07140_b200 import _lib
    rec = np.zeros(1, dtype=_lib.CTX_DTYPE)
    for name in ("layers", "hidden_dim", "head_count", "head_dim", "ffn_dim", "bytes_per_param"):
        rec[name] = getattr(spec, name)
    rec["alpha"], rec["beta"] = float(quant.alpha), float(quant.beta)
    rec["flops_per_s"], rec["memory_bytes"], rec["gpu_count"] = float(node.flops_per_s), float(node.memory_bytes), node.gpu_count
    return int(oracle.load().oracle_static_batch_size(_p(rec), float(slot_s), int(s_max), int(n_max)))


def install(monkeypatch):
    monkeypatch.setattr(sweep, "static_batch_size", static_batch_size)
    monkeypatch.setattr(sweep, "_handle", lambda device: None)
    monkeypatch.setattr(sweep, "_admission", admission)
    monkeypatch.setattr(sweep, "_dftsp", dftsp)
    monkeypatch.setattr(sweep, "_exhaustive", exhaustive)
    monkeypatch.setattr(sweep, "_stb", stb)
    monkeypatch.setattr(sweep, "_nob", nob)
    monkeypatch.setattr(sweep, "_costs_and_checks", costs_and_checks)
