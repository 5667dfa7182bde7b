"""install_into_edgebatch() rebinds every hot-path name the reference resolves
(package, defining modules, and sim.py's import-time bindings).  Runs only
where the reference package is importable (the build container)."""
import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
def test_install_patches_sim_and_modules():
    sys.path.insert(0, REF)
    try:
        import edgebatch
        import edgebatch.sim as sim
        from paper_2405_07140_b200 import compat, search, feasibility, baselines
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
    finally:
        sys.path.remove(REF)
