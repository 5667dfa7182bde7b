"""Swap the GPU implementations into an installed reference ``edgebatch``.

``install_into_edgebatch()`` rebinds the hot-path names in every place the
reference resolves them, so the reference's own simulator / CLI run their
scheduling searches on the B200 without other changes:

* the package namespace (``edgebatch.dftsp`` ..., reference __init__.py:4-23);
* the defining modules (``sys.modules['edgebatch.dftsp']`` -- note that the
  attribute ``edgebatch.dftsp`` is the *function*, so the module must be taken
  from ``sys.modules``; ``edgebatch.feasibility``, ``edgebatch.baselines``,
  ``edgebatch.costs``, ``edgebatch.radio``);
* ``edgebatch.sim``, which binds ``dftsp``, ``exhaustive_optimal``,
  ``check_direct``, ``batch_cost``, ``stb_schedule``, ``nob_assign``,
  ``static_batch_size`` and ``filter_admissible`` at import time
  (reference sim.py:19-24).

Request / EdgeContext objects stay the reference's own dataclasses: the GPU
functions are duck-typed over their attributes and return the caller's
objects.  ``uninstall()`` restores the originals.
"""
from __future__ import annotations

import importlib
import sys

from . import baselines, costs, feasibility, radio, search

# name -> replacement; only functions on the hot path (records stay the reference's)
REPLACEMENTS = {
    "dftsp": search.dftsp,
    "exhaustive_optimal": search.exhaustive_optimal,
    "dfs": search.dfs,
    "partition": search.partition,
    "check_direct": feasibility.check_direct,
    "check_knapsack": feasibility.check_knapsack,
    "derive_coefficients": feasibility.derive_coefficients,
    "filter_admissible": feasibility.filter_admissible,
    "batch_cost": costs.batch_cost,
    "static_batch_size": baselines.static_batch_size,
    "stb_schedule": baselines.stb_schedule,
    "nob_assign": baselines.nob_assign,
    "spectral_efficiency": radio.spectral_efficiency,
    "uplink_fraction_per_token": radio.uplink_fraction_per_token,
    "downlink_fraction_per_token": radio.downlink_fraction_per_token,
    "min_uplink_fraction": radio.min_uplink_fraction,
    "min_downlink_fraction": radio.min_downlink_fraction,
}
MODULES = ("edgebatch", "edgebatch.dftsp", "edgebatch.feasibility", "edgebatch.baselines", "edgebatch.costs",
           "edgebatch.radio", "edgebatch.sim", "edgebatch.cli")
_saved: list = []


def install_into_edgebatch() -> list:
    """Patch every module of an importable ``edgebatch``; returns the patched (module, name) pairs."""
    importlib.import_module("edgebatch")
    patched = []
    for modname in MODULES:
        try:
            importlib.import_module(modname)
        except ImportError:
            continue
        mod = sys.modules[modname]
        for name, fn in REPLACEMENTS.items():
            if name in vars(mod) and callable(vars(mod)[name]) and vars(mod)[name] is not fn:
                _saved.append((mod, name, vars(mod)[name]))
                setattr(mod, name, fn)
                patched.append((modname, name))
    return patched


def uninstall() -> None:
    while _saved:
        mod, name, orig = _saved.pop()
        setattr(mod, name, orig)
