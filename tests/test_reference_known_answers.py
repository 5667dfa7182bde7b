"""Known-answer tests of the reference's own suite, restated
against this package's drop-in API.  Each case names the reference test it
follows (pkg/tests/<file>:<line>).  The exact integer cost model is host
Python (CPU tests); link math, coefficients, batch cost and the dfs walk run
on the device (GPU tests)."""
import math

import pytest

from paper_2405_07140_b200 import (BatchPlan, EdgeContext, LlmSpec, NodeCompute, RadioConfig, Request, UserLink,
                                   batch_cost, dbm_to_watts, derive_coefficients, dfs, flops_autoregressive,
                                   flops_autoregressive_stepwise, flops_initial, get_model, get_profile,
                                   kv_bytes_autoregressive, kv_bytes_initial, min_downlink_fraction,
                                   min_uplink_fraction, partition, spectral_efficiency, uplink_fraction_per_token,
                                   downlink_fraction_per_token, weight_bytes)

B3 = get_model("bloom-3b")
OPT = get_model("opt-13b")
FP16 = get_profile("fp16")
NODE = NodeCompute(flops_per_s=2.66e13, memory_bytes=640e9, gpu_count=20)


def radio(**kw):
    """Paper radio (reference test_radio.py:15-22): 20 MHz bands, 43 dBm
    downlink, -174 dBm/Hz noise, 0.25 s slots."""
    base = dict(uplink_band_hz=20e6, downlink_band_hz=20e6, downlink_power_w=dbm_to_watts(43.0),
                noise_density_w_hz=dbm_to_watts(-174.0), uplink_slot_s=0.25, downlink_slot_s=0.25)
    base.update(kw)
    return RadioConfig(**base)


# ---- cost model (host, exact integers) ----------------------------------
def test_weight_bytes_exact():                       # test_costs.py:17-20
    assert weight_bytes(B3) == 4_718_592_000
    assert weight_bytes(OPT) == 25_165_824_000
    assert weight_bytes(get_model("bloom-7.1b")) == 12_079_595_520
    assert weight_bytes(LlmSpec("none", 0, 2560, 32, 80, 10240)) == 0          # :23-25


def test_kv_bytes():                                 # test_costs.py:28-41
    assert kv_bytes_initial(B3, 512, 4) == 629_145_600
    assert kv_bytes_initial(B3, 512, 0) == 0
    assert kv_bytes_autoregressive(B3, [128]) == 39_321_600
    assert kv_bytes_autoregressive(B3, []) == 0
    lens = [128, 256, 512]
    assert kv_bytes_autoregressive(B3, lens) == sum(kv_bytes_autoregressive(B3, [n]) for n in lens)


def test_flops_exact():                              # test_costs.py:44-66
    assert flops_initial(B3, 512) == 2_496_449_740_800
    assert flops_initial(LlmSpec("unit", 7, 1, 1, 1, 1), 1) == 16 * 7
    s, d, f, L = 64, B3.hidden_dim, B3.ffn_dim, B3.layers
    linear, quad = L * (6 * d * d + 2 * d * d + 4 * d * f), L * 4 * d
    assert flops_initial(B3, 2 * s) == linear * 2 * s + quad * 4 * s * s
    assert flops_autoregressive(B3, 512, 128) == 621_733_478_400 == 127 * 30 * 163_184_640
    assert flops_autoregressive(B3, 512, 1) == 0 == flops_autoregressive_stepwise(B3, 512, 1)


def test_flops_autoregressive_matches_stepwise():   # test_costs.py:69-78
    import numpy as np
    rng = np.random.default_rng(5)
    specs = [B3, OPT, LlmSpec("toy", 3, 32, 4, 8, 128)]
    for _ in range(200):
        spec = specs[int(rng.integers(len(specs)))]
        s, n = int(rng.integers(1, 700)), int(rng.integers(1, 700))
        assert flops_autoregressive(spec, s, n) == flops_autoregressive_stepwise(spec, s, n)


# ---- device: link math, coefficients, batch cost, dfs walks --------------
@pytest.mark.gpu
def test_batch_cost_single_request():               # test_costs.py:96-107
    cost = batch_cost(B3, FP16, BatchPlan(((512, 128),), 512), NODE)
    assert cost.latency_s == pytest.approx((2_496_449_740_800 + 621_733_478_400) / 2.66e13)
    assert cost.latency_s == pytest.approx(0.0939 + 0.0234, abs=2e-4)
    assert cost.memory_bytes == weight_bytes(B3) + kv_bytes_initial(B3, 512, 1) + kv_bytes_autoregressive(B3, [128])
    empty = batch_cost(B3, FP16, BatchPlan((), 0), NODE)                       # :89-93
    assert empty.memory_bytes == weight_bytes(B3) and empty.latency_s == 0.0


@pytest.mark.gpu
def test_spectral_efficiency_values():               # test_radio.py:32-41
    cfg = radio()
    assert cfg.uplink_noise_w == pytest.approx(7.962143e-14, rel=1e-6)
    up = spectral_efficiency(0.1, 1e-3, cfg.uplink_noise_w)
    assert up == math.log2(1 + 0.1e-3 / cfg.uplink_noise_w)                    # bit-exact: glibc log2 port
    assert up == pytest.approx(30.226, rel=1e-4)
    assert spectral_efficiency(cfg.downlink_power_w, 1e-3, cfg.downlink_noise_w) == pytest.approx(37.867, rel=1e-4)
    assert spectral_efficiency(1.0, 1.0, 1.0) == pytest.approx(1.0)            # :28-29
    for args in ((0.0, 1.0, 1.0), (1.0, -1.0, 1.0), (1.0, 1.0, 0.0)):          # :44-47
        with pytest.raises(ValueError):
            spectral_efficiency(*args)


@pytest.mark.gpu
def test_link_fractions():                           # test_radio.py:50-75
    cfg = radio()
    link = UserLink(channel_gain=1e-3, uplink_power_w=0.1)
    assert min_uplink_fraction(0, link, cfg) == 0.0
    frac = min_uplink_fraction(512, link, cfg)
    eff = spectral_efficiency(0.1, 1e-3, cfg.uplink_noise_w)
    assert frac == pytest.approx(512 * 16 / (0.25 * 20e6 * eff))
    assert frac == pytest.approx(5.4205e-5, rel=1e-3)
    assert min_uplink_fraction(1024, link, cfg) == 2 * frac
    assert frac == 512 * uplink_fraction_per_token(link, cfg)
    per_token = downlink_fraction_per_token(link, cfg)
    assert per_token == pytest.approx(8.4507e-8, rel=1e-3)
    assert min_downlink_fraction(7, link, cfg) == 7 * per_token
    assert min_uplink_fraction(512, UserLink(1e-12, 0.1), radio(uplink_band_hz=2e3)) > 1.0     # :85-88


def _request(i=0, s=256, n=128, tau=1.5, wait=0.1, gain=1e-3, p=0.1, tol=1.0):
    return Request(id=i, prompt_tokens=s, output_tokens=n, deadline_s=tau, tolerance=tol, link=UserLink(gain, p),
                   waiting_s=wait)


def _ctx():
    return EdgeContext(llm=B3, quant=FP16, radio=radio(), node=NODE)


@pytest.mark.gpu
def test_coefficient_values_bloom3b():               # test_feasibility.py:37-45
    co = derive_coefficients(_ctx(), 512, [_request()])
    assert co.k5 == 2 * 30 * 2560 == 153_600
    assert co.k2 == pytest.approx((640e9 - 4_718_592_000) / (4 * 30 * 2560))
    assert co.k2 == pytest.approx(2.068e6, rel=1e-3)
    gen_base = 8 * 2560 ** 2 + 4 * 512 * 2560 + 4 * 2560 * 10240
    assert co.k4 == 30 * (gen_base - 2 * 2560)
    assert co.k3 == 2_496_449_740_800 - 30 * gen_base


@pytest.mark.gpu
def test_uplink_coefficient_matches_min_fraction_exactly():     # test_feasibility.py:48-57
    import numpy as np
    rng = np.random.default_rng(3)
    cfg = radio()
    reqs = [_request(i, s=int(rng.integers(1, 600)), gain=float(rng.exponential(1e-3))) for i in range(20)]
    co = derive_coefficients(_ctx(), 600, reqs)
    for r in reqs:
        assert co.k_up[r.id] * r.prompt_tokens == min_uplink_fraction(r.prompt_tokens, r.link, cfg)


def _pool(class_sizes, ladder=(128, 256, 512)):
    """Pool with the given per-class sizes, uplink cost rising with id
    (test_dftsp.py:17-29)."""
    reqs, i = [], 0
    for k, size in enumerate(class_sizes):
        for _ in range(size):
            reqs.append(Request(id=i, prompt_tokens=64 + i, output_tokens=ladder[k], deadline_s=1.5, tolerance=1.0,
                                link=UserLink(1e-3 / (1.0 + 0.1 * i), 0.1), waiting_s=0.0))
            i += 1
    return reqs


@pytest.mark.gpu
def test_dfs_exact_walks():                          # test_dftsp.py:98-142
    ctx = _ctx()
    pool = _pool((4, 4, 2))
    co = derive_coefficients(ctx, 512, pool)
    part = partition(pool, ctx.radio)
    assert part.lengths == (128, 256, 512) and part.sizes == (4, 4, 2)       # :37-45
    first = dfs(6, part, co, tau_min=1e30)
    assert first.counts == (4, 2, 0) and first.nodes_visited == 3 and first.nodes_pruned == 0
    on = dfs(7, part, co, tau_min=1e30, pruning=True)
    off = dfs(7, part, co, tau_min=1e30, pruning=False)
    assert on.counts == off.counts == (4, 3, 0) and on.nodes_visited <= off.nodes_visited
    small = _pool((2, 2))
    co2 = derive_coefficients(ctx, 512, small)
    part2 = partition(small, ctx.radio)
    cut = dfs(5, part2, co2, tau_min=1e30, pruning=True)
    assert cut.solution is None and cut.nodes_visited == 0 and cut.nodes_pruned == 1
    assert dfs(5, part2, co2, tau_min=1e30, pruning=False).nodes_visited > 0


@pytest.mark.gpu
def test_partition_single_class_ties():              # test_dftsp.py:48-54
    pool = [Request(id=i, prompt_tokens=100, output_tokens=128, deadline_s=1.0, tolerance=1.0,
                    link=UserLink(1e-3, 0.1)) for i in (4, 1, 3)]
    part = partition(pool, radio())
    assert part.sizes == (3,)
    assert [r.id for r in part.classes[0]] == [1, 3, 4]
