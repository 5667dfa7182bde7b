"""CPU checks of the admission oracle (sim.py:264-274) against the reference's
own recorded per-epoch candidate counts, and of the workload generator's
admission hook (no GPU)."""
import numpy as np

import oracle
from paper_2405_07140_b200 import synth


def test_oracle_admission_generates_exact_k():
    b = synth.generate(synth.CONFIG2, 2000, seed=3, admit=oracle.admit)
    assert b.n_inst == 2000 and (np.diff(b.offsets) == 20).all()
    st, keep = oracle.admission_batch(b)
    assert (st == 0).all() and keep.all()      # every kept candidate passes admission again


def test_oracle_admission_matches_python_reference():
    """The C admission against the unmodified reference's filter_admissible +
    check_direct((r,), ctx, r.prompt_tokens) on raw draws."""
    import pytest
    import pyref
    if not pyref.available():
        pytest.skip("oracle/_ref not staged")
    eb = pyref.import_reference()
    import test_gpu_admission as t
    b = t._rows(21, 300, 20)
    st, keep = oracle.admission_batch(b)
    ctxs = [pyref.context_of(b.contexts[i]) for i in range(len(b.contexts))]
    for i in range(b.n_inst):
        ctx = ctxs[int(b.ctx_index[i])]
        delta = float(b.contexts[int(b.ctx_index[i])]["delta_ppl"])
        reqs = pyref.requests_of(b.columns, int(b.offsets[i]), int(b.offsets[i + 1]))
        adm = eb.filter_admissible(reqs, delta)
        ok = {r.id for r in adm if eb.check_direct((r,), ctx, r.prompt_tokens)}
        for j, r in enumerate(reqs):
            assert bool(keep[int(b.offsets[i]) + j]) == (r.id in ok), (i, j)
