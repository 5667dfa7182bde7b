"""Worker for tests/test_gpu_nccl.py, launched by torch.distributed.run: the
config-4 brute force through brute.solve_distributed over a real NCCL
communicator (one all-reduce(MIN) per live level on the GPU), and the
instance-sharded DFTSP of bench.py's weak-scaling path, on this rank's GPU.
Writes one JSON line per rank to the file named by argv[1]."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(out_path):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2405_07140_b200 import brute, search, synth

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group(backend="nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    res = {"rank": rank, "world": world, "backend": dist.get_backend(), "device": torch.cuda.current_device()}
    brutes = []
    for rec, cols in synth.brute_family(24, 2, seed=5):
        r = brute.solve_distributed(rec, cols)
        brutes.append([int(r.z), int(r.lexrank), int(r.nodes_visited), int(r.mask)])
    res["brute"] = brutes
    # instance sharding: this rank's contiguous share of 4096 config-2 instances
    n = 4096
    lo, hi = rank * n // world, (rank + 1) * n // world
    b = synth.generate(synth.CONFIG2, n, seed=11)
    sub = synth.slice_batch(b, lo, hi) if hasattr(synth, "slice_batch") else None
    if sub is None:
        from paper_2405_07140_b200.soa import InstanceBatch
        r0, r1 = int(b.offsets[lo]), int(b.offsets[hi])
        sub = InstanceBatch(b.offsets[lo:hi + 1] - r0, {k: v[r0:r1] for k, v in b.columns.items()},
                            b.contexts, b.ctx_index[lo:hi].copy(), b.k_max)
    out = search.solve_batch(sub, ladder=(128, 256, 512))
    tot = torch.tensor([int(out.z_found.sum()), int(out.nodes_visited.sum())], dtype=torch.int64, device="cuda")
    dist.all_reduce(tot)
    res["z_sum"], res["nodes_sum"] = int(tot[0]), int(tot[1])
    res["local_z"] = [int(x) for x in np.asarray(out.z_found)]
    with open(f"{out_path}.{rank}", "w") as fh:
        fh.write(json.dumps(res))
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
