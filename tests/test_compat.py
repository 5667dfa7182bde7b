"""install_into_edgebatch() rebinds every hot-path name the reference resolves
(package, defining modules, and sim.py's import-time bindings).  Runs on the
unmodified reference staged in oracle/_ref (oracle/make_ref.py)."""
import sys

import pytest

import pyref


@pytest.mark.skipif(not pyref.available(), reason="oracle/_ref not staged")
def test_install_patches_sim_and_modules():
    edgebatch = pyref.import_reference()
    import edgebatch.sim as sim
    from paper_2405_07140_b200 import baselines, compat, feasibility, search
    patched = compat.install_into_edgebatch()
    try:
        assert sim.dftsp is search.dftsp
        assert sim.exhaustive_optimal is search.exhaustive_optimal
        assert sim.check_direct is feasibility.check_direct
        assert sim.stb_schedule is baselines.stb_schedule
        assert edgebatch.dftsp is search.dftsp
        assert sys.modules["edgebatch.dftsp"].dftsp is search.dftsp
        assert ("edgebatch.sim", "nob_assign") in patched
    finally:
        compat.uninstall()
    assert sim.dftsp is not search.dftsp
