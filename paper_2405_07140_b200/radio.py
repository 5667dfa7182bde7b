"""OFDMA link model (reference ``radio.py``), evaluated on the GPU.

``spectral_efficiency`` / ``*_fraction_per_token`` / ``min_*_fraction`` call
the K1 link kernel (``eb_link_batch``) through the C ABI; the device log2 is
a bit-exact port of the glibc ``log2`` CPython's ``math.log2`` uses.  Config
records (``RadioConfig``, ``UserLink``, ``dbm_to_watts``) and the host RNG
sampler stay on the host.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["RadioConfig", "UserLink", "dbm_to_watts", "spectral_efficiency", "uplink_fraction_per_token",
           "downlink_fraction_per_token", "min_uplink_fraction", "min_downlink_fraction",
           "sample_channel_power", "link_table"]


@dataclass(frozen=True)
class RadioConfig:
    """Shared radio parameters (reference radio.py:16-43); SI units."""

    uplink_band_hz: float
    downlink_band_hz: float
    downlink_power_w: float
    noise_density_w_hz: float
    uplink_slot_s: float
    downlink_slot_s: float
    bits_per_token: int = 16

    def __post_init__(self):
        for attr in ("uplink_band_hz", "downlink_band_hz", "downlink_power_w", "noise_density_w_hz",
                     "uplink_slot_s", "downlink_slot_s", "bits_per_token"):
            if getattr(self, attr) <= 0:
                raise ValueError(f"radio.{attr} must be strictly positive")

    @property
    def uplink_noise_w(self) -> float:
        return self.noise_density_w_hz * self.uplink_band_hz

    @property
    def downlink_noise_w(self) -> float:
        return self.noise_density_w_hz * self.downlink_band_hz


@dataclass(frozen=True)
class UserLink:
    """Per-user channel power gain |h|^2 and uplink transmit power (radio.py:46-57)."""

    channel_gain: float
    uplink_power_w: float

    def __post_init__(self):
        if self.channel_gain <= 0:
            raise ValueError("channel_gain must be strictly positive")
        if self.uplink_power_w <= 0:
            raise ValueError("uplink_power_w must be strictly positive")


def dbm_to_watts(dbm: float) -> float:
    """Config-time unit conversion (radio.py:60-61)."""
    return 10.0 ** (dbm / 10.0) / 1000.0


def _radio_ctx(cfg, *, up_band=None, up_density=None, dn_power=None, dn_band=None, dn_density=None):
    rec = np.zeros(1, dtype=_lib.CTX_DTYPE)
    rec["uplink_band_hz"] = float(cfg.uplink_band_hz if up_band is None else up_band)
    rec["downlink_band_hz"] = float(cfg.downlink_band_hz if dn_band is None else dn_band)
    rec["downlink_power_w"] = float(cfg.downlink_power_w if dn_power is None else dn_power)
    rec["noise_density_w_hz"] = float(cfg.noise_density_w_hz if up_density is None else up_density)
    rec["uplink_slot_s"] = float(cfg.uplink_slot_s)
    rec["downlink_slot_s"] = float(cfg.downlink_slot_s)
    rec["bits_per_token"] = int(cfg.bits_per_token)
    return rec


def link_table(gains, uplink_powers, prompts, outputs, contexts, req_ctx=None, device=None):
    """Batched K1 link math: columns (eta_up, eta_dn, k_up, k_down, rho_up_min, rho_dn_min).

    Returns (status[n], out[n, 6]); status != 0 where the reference raises.
    """
    from .soa import requests_struct
    cols = {"channel_gain": np.ascontiguousarray(gains, dtype=np.float64),
            "uplink_power_w": np.ascontiguousarray(uplink_powers, dtype=np.float64),
            "prompt_tokens": np.ascontiguousarray(prompts, dtype=np.int32),
            "output_tokens": np.ascontiguousarray(outputs, dtype=np.int32)}
    n = cols["channel_gain"].shape[0]
    status = np.zeros(n, dtype=np.int32)
    out = np.zeros((n, 6), dtype=np.float64)
    rc = None if req_ctx is None else np.ascontiguousarray(req_ctx, dtype=np.int32)
    h = _lib.handle(device)
    _lib.check(h.lib.eb_link_batch(h.ptr, contexts.ctypes.data, len(contexts), _as_ref(requests_struct(cols)),
                                   n, _lib.ptr(rc), status.ctypes.data, out.ctypes.data, _lib.EB_MEM_HOST),
               "eb_link_batch")
    return status, out


def _as_ref(struct):
    import ctypes
    return ctypes.cast(ctypes.pointer(struct), ctypes.c_void_p)


def _raise_link(status: int) -> None:
    if status == _lib.ERR_NONPOSITIVE_LINK:
        raise ValueError("power, gain and noise must be strictly positive")
    if status == _lib.ERR_UPLINK_EFF_ZERO:
        raise ValueError("uplink spectral efficiency is zero")
    if status == _lib.ERR_DOWNLINK_EFF_ZERO:
        raise ValueError("downlink spectral efficiency is zero")
    if status:
        raise _lib.EdgebatchNativeError(_lib.status_string(status))


def _one(link, cfg, prompt=0, output=0):
    st, out = link_table([link.channel_gain], [link.uplink_power_w], [prompt], [output], _radio_ctx(cfg))
    return int(st[0]), out[0]


def spectral_efficiency(power_w: float, channel_gain: float, noise_w: float) -> float:
    """log2(1 + P |h|^2 / N0) (radio.py:64-68), computed by the device log2 port."""
    if power_w <= 0 or channel_gain <= 0 or noise_w <= 0:
        raise ValueError("power, gain and noise must be strictly positive")
    # uplink column with band 1 Hz and density = noise_w gives N0 = noise_w * 1.0 exactly
    rec = np.zeros(1, dtype=_lib.CTX_DTYPE)
    rec["uplink_band_hz"] = 1.0
    rec["downlink_band_hz"] = 1.0
    rec["noise_density_w_hz"] = float(noise_w)
    rec["downlink_power_w"] = 1.0
    rec["uplink_slot_s"] = rec["downlink_slot_s"] = 1.0
    rec["bits_per_token"] = 1
    _, out = link_table([channel_gain], [power_w], [0], [0], rec)
    return float(out[0, 0])


def _check_up(link, cfg) -> None:
    if link.uplink_power_w <= 0 or link.channel_gain <= 0 or cfg.uplink_noise_w <= 0:
        _raise_link(_lib.ERR_NONPOSITIVE_LINK)        # radio.py:63-64


def _check_dn(link, cfg) -> None:
    if cfg.downlink_power_w <= 0 or link.channel_gain <= 0 or cfg.downlink_noise_w <= 0:
        _raise_link(_lib.ERR_NONPOSITIVE_LINK)


def uplink_fraction_per_token(link, cfg) -> float:
    _check_up(link, cfg)
    st, out = _one(link, cfg)
    if st == _lib.ERR_UPLINK_EFF_ZERO:
        _raise_link(st)
    return float(out[2])


def downlink_fraction_per_token(link, cfg) -> float:
    _check_dn(link, cfg)
    st, out = _one(link, cfg)
    if out[1] <= 0.0:
        _raise_link(_lib.ERR_DOWNLINK_EFF_ZERO)
    return float(out[3])


def min_uplink_fraction(prompt_tokens: int, link, cfg) -> float:
    if prompt_tokens < 0:
        raise ValueError("prompt_tokens must be nonnegative")
    _check_up(link, cfg)
    st, out = _one(link, cfg, prompt=prompt_tokens)
    if st == _lib.ERR_UPLINK_EFF_ZERO:
        _raise_link(st)
    return float(out[4])


def min_downlink_fraction(output_tokens: int, link, cfg) -> float:
    if output_tokens < 0:
        raise ValueError("output_tokens must be nonnegative")
    _check_dn(link, cfg)
    st, out = _one(link, cfg, output=output_tokens)
    if out[1] <= 0.0:
        _raise_link(_lib.ERR_DOWNLINK_EFF_ZERO)
    return float(out[5])


def sample_channel_power(rng, mean_gain: float) -> float:
    """Rayleigh fading power draw (radio.py:104-112), host RNG."""
    if mean_gain <= 0:
        raise ValueError("mean_gain must be strictly positive")
    return float(rng.exponential(mean_gain))
