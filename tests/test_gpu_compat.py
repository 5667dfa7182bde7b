"""The reference-side binding on hardware: the UNMODIFIED
reference simulator (oracle/_ref, staged verbatim from /root/reference by
oracle/make_ref.py) run on its own scenario files once as is and once with
compat.install_into_edgebatch() routing every hot-path call (dftsp,
exhaustive_optimal, check_direct, filter_admissible, batch_cost, the StB /
NoB baselines ...) through the CUDA library.  Every SimMetrics field and
every per-epoch trace row must be identical."""
import dataclasses
import os

import pytest

import pyref

pytestmark = pytest.mark.gpu

SCENARIOS = ("default.yaml", "pruning_comparison.yaml", "throughput.yaml")


def _run(path, **changes):
    eb = pyref.import_reference()
    from edgebatch import cli, sim
    sc = cli.parse_scenario(path)
    if changes:
        sc = dataclasses.replace(sc, **changes)
    return sim.run(sc)


def _fields(m):
    return {f.name: getattr(m, f.name) for f in dataclasses.fields(m)}


@pytest.mark.skipif(not pyref.available(), reason="oracle/_ref not staged")
@pytest.mark.parametrize("scenario,changes", [
    ("default.yaml", {}),
    ("default.yaml", {"scheduler": "stb"}),
    ("default.yaml", {"scheduler": "nob"}),
    ("pruning_comparison.yaml", {"duration": 6.0}),
    ("throughput.yaml", {"duration": 10.0}),
    ("default.yaml", {"verify_oracle": True, "duration": 6.0}),
])
def test_reference_simulator_through_the_device(scenario, changes):
    path = os.path.join(pyref.REF_DIR, "scenarios", scenario)
    pyref.import_reference()
    from paper_2405_07140_b200 import _lib, compat
    want = _run(path, **changes)
    h = _lib.handle()
    before = h.launches()
    patched = compat.install_into_edgebatch()
    try:
        assert ("edgebatch.sim", "dftsp") in patched
        got = _run(path, **changes)
    finally:
        compat.uninstall()
    assert h.launches() > before, "the patched run launched no device kernels"
    a, b = _fields(want), _fields(got)
    assert a.keys() == b.keys()
    for k in a:
        assert a[k] == b[k], (scenario, changes, k)
