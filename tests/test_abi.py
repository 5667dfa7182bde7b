"""The C-ABI library builds, loads without a GPU and exports exactly the
entry points include/edgebatch_b200.h declares; ctypes layouts match C."""
import ctypes
import os
import re
import shutil
import subprocess

import pytest

from helpers import ROOT
from paper_2405_07140_b200 import _lib
from paper_2405_07140_b200._build import build_library

HEADER = os.path.join(ROOT, "include", "edgebatch_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int32_t|int64_t|const char \*)\s*(eb_[a-z_0-9]+)\s*\(", text, re.M)))


def test_library_builds_and_loads():
    path = build_library()
    assert os.path.exists(path)
    lib = _lib.load()
    assert lib.eb_abi_version() == _lib.ABI_VERSION == 2
    assert lib.eb_status_string(0) == b"ok"


def test_every_declared_symbol_is_exported():
    syms = declared_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(build_library())
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED_SYMBOLS), set(syms) ^ set(_lib.EXPORTED_SYMBOLS)


def test_cubin_targets_sm100a():
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump missing")
    out = subprocess.run([cuobjdump, "--list-elf", build_library()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_c(tmp_path):
    gcc = shutil.which("gcc")
    if not gcc:
        pytest.skip("gcc missing")
    src = tmp_path / "lay.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "edgebatch_b200.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(eb_context), sizeof(eb_requests),'
                   ' sizeof(eb_batch), sizeof(eb_search_params), sizeof(eb_dftsp_result),'
                   ' offsetof(eb_batch, k_max));return 0;}\n')
    exe = tmp_path / "lay"
    subprocess.run([gcc, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    want = [ctypes.sizeof(_lib.eb_context), ctypes.sizeof(_lib.eb_requests), ctypes.sizeof(_lib.eb_batch),
            ctypes.sizeof(_lib.eb_search_params), ctypes.sizeof(_lib.eb_dftsp_result),
            _lib.eb_batch.k_max.offset]
    assert got == want


def test_packed_struct_layouts_match_c(tmp_path):
    gcc = shutil.which("gcc")
    if not gcc:
        pytest.skip("gcc missing")
    src = tmp_path / "lay2.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "edgebatch_b200.h"\n'
                   'int main(){printf("%zu %zu %zu %zu\\n", sizeof(eb_requests_packed), sizeof(eb_batch_packed),'
                   ' offsetof(eb_requests_packed, uplink_power_uniform), offsetof(eb_batch_packed, k_max));'
                   'return 0;}\n')
    exe = tmp_path / "lay2"
    subprocess.run([gcc, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    want = [ctypes.sizeof(_lib.eb_requests_packed), ctypes.sizeof(_lib.eb_batch_packed),
            _lib.eb_requests_packed.uplink_power_uniform.offset, _lib.eb_batch_packed.k_max.offset]
    assert got == want


def test_pack_wire_is_lossless_or_refuses():
    """Host logic of the wire format: values round-trip exactly; columns that
    do not narrow losslessly make pack_wire refuse (the caller keeps the wide call)."""
    import numpy as np
    from gen_random import random_batch
    from paper_2405_07140_b200.soa import pack_wire
    batch, _ = random_batch(5, 200)
    w = pack_wire(batch)
    assert w is not None and w.uniform_power
    assert w.columns["id"] is not None          # random ids do not rise along the rows: shipped
    assert w.offsets is not None                # ragged sizes: shipped
    for name in ("id", "prompt_tokens", "output_tokens"):
        assert np.array_equal(w.columns[name].astype(np.int64), batch.columns[name].astype(np.int64))
    for name in ("deadline_s", "waiting_s", "channel_gain"):
        assert w.columns[name].tobytes() == batch.columns[name].tobytes()
    assert w.nbytes() < sum(batch.columns[k].nbytes for k in batch.columns if k != "tolerance")
    cols = dict(batch.columns)
    cols["uplink_power_w"] = cols["uplink_power_w"].copy()
    cols["uplink_power_w"][3] *= 2
    b2 = type(batch)(batch.offsets, cols, batch.contexts, batch.ctx_index, batch.k_max)
    w2 = pack_wire(b2)
    assert not w2.uniform_power and w2.uplink_power_w.tobytes() == cols["uplink_power_w"].tobytes()
    for name, bad in (("id", 2**31), ("prompt_tokens", 70000), ("output_tokens", -1)):
        c3 = dict(batch.columns)
        c3[name] = c3[name].copy()
        c3[name][0] = bad
        assert pack_wire(type(batch)(batch.offsets, c3, batch.contexts, batch.ctx_index, batch.k_max)) is None


def test_pack_wire_implicit_ids_and_offsets():
    """Ids rising along each instance's rows and uniform sizes are not shipped
    (positions reproduce every id comparison); anything else is."""
    import numpy as np
    from paper_2405_07140_b200.soa import InstanceBatch, pack_wire
    from gen_random import random_batch
    batch, _ = random_batch(6, 50, k_min=7, k_max=7)
    cols = dict(batch.columns)
    ids = np.concatenate([np.sort(cols["id"][batch.offsets[i]:batch.offsets[i + 1]]) for i in range(batch.n_inst)])
    cols["id"] = ids
    b = InstanceBatch(batch.offsets, cols, batch.contexts, batch.ctx_index, 7)
    w = pack_wire(b)
    assert w.columns["id"] is None and w.offsets is None and w.n_inst == 50 and w.k_max == 7
    assert np.array_equal(w.sizes(), np.full(50, 7))
    full = pack_wire(b, implicit=False)
    assert w.nbytes() == full.nbytes() - 4 * b.n_req - 8 * (b.n_inst + 1)
    cols2 = dict(cols)
    cols2["id"] = ids.copy()
    cols2["id"][3], cols2["id"][4] = ids[4], ids[3]          # one descent inside instance 0
    assert pack_wire(InstanceBatch(batch.offsets, cols2, batch.contexts, batch.ctx_index, 7)).columns["id"] is not None


def test_pack_wire_token_dictionary():
    """Token counts with <= 16 distinct values travel as one code byte whose
    tables decode every row exactly; more distinct values keep the u16 columns."""
    import numpy as np
    from paper_2405_07140_b200 import synth
    from paper_2405_07140_b200.soa import pack_wire
    rng = np.random.default_rng(0)
    n = 500
    from paper_2405_07140_b200.soa import REQ_FIELDS, InstanceBatch
    cols = {name: np.zeros(n, dt) for name, dt in REQ_FIELDS}
    cols["prompt_tokens"][:] = rng.choice([128, 256, 512], n)
    cols["output_tokens"][:] = rng.choice([64, 128, 256, 512, 1024], n)
    cols["id"][:] = np.tile(np.arange(20), n // 20)
    cols["deadline_s"][:] = rng.uniform(0.5, 2, n)
    off = np.arange(0, n + 1, 20, dtype=np.int64)
    batch = InstanceBatch(off, cols, synth.contexts(synth.CONFIG2), np.zeros(n // 20, np.int32), 20)
    w = pack_wire(batch)
    assert w.token_codes is not None and w.columns["prompt_tokens"] is None
    assert np.array_equal(w.prompt_dict[w.token_codes & 15], cols["prompt_tokens"])
    assert np.array_equal(w.output_dict[w.token_codes >> 4], cols["output_tokens"])
    s = w.struct()
    assert s.req.n_dict == 5 and s.req.token_codes
    cols["prompt_tokens"][:] = np.arange(n) % 40 + 1                  # 40 distinct prompts
    w2 = pack_wire(InstanceBatch(off, cols, batch.contexts, batch.ctx_index, 20))
    assert w2.token_codes is None and w2.columns["prompt_tokens"] is not None


def test_no_gpu_means_loud_failure():
    """Without a device the product raises -- there is no CPU fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.EdgebatchNativeError):
        _lib.Handle(0)
