"""NCCL on the GPU: brute.solve_distributed (config 4's rank-range sharding,
one all-reduce(MIN) per live level) and the instance-sharded sweep of
bench.py, launched by torch.distributed.run with one rank per visible GPU
(1 on the test box; the logic for 2 ranks is covered with gloo in
test_distributed.py).  Results must equal the literal CPU oracle."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from helpers import ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_brute_and_instance_sharding(tmp_path):
    import torch
    import oracle
    from paper_2405_07140_b200 import brute, synth

    world = max(1, min(torch.cuda.device_count(), 2))
    out = str(tmp_path / "res")
    env = dict(os.environ, NCCL_DEBUG="WARN")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "tests", "nccl_worker.py"), out]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    res = [json.loads(open(f"{out}.{r}").read()) for r in range(world)]
    assert all(r["backend"] == "nccl" and r["world"] == world for r in res)
    # brute force: every rank holds the combined answer; it equals the literal level scan
    for i, (rec, cols) in enumerate(synth.brute_family(24, 2, seed=5)):
        st, z, rk, _ = oracle.exhaustive_mt(rec, cols)
        assert st == 0
        want = [z, rk, brute.nodes_for(24, z, rk), brute.unrank(24, z, rk) if z else 0]
        for r in res:
            assert r["brute"][i] == want, (i, r["rank"])
    # instance sharding: the all-reduced totals equal the oracle over all instances
    b = synth.generate(synth.CONFIG2, 4096, seed=11)
    o = oracle.dftsp_batch(b, ladder=(128, 256, 512))
    assert res[0]["z_sum"] == int(np.asarray(o["z_found"]).sum())
    assert res[0]["nodes_sum"] == int(np.asarray(o["nodes_visited"]).sum())
    got = np.concatenate([np.asarray(r["local_z"]) for r in sorted(res, key=lambda r: r["rank"])])
    assert np.array_equal(got, np.asarray(o["z_found"]))
