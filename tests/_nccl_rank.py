"""One rank of the real-NCCL row-slab test (tests/test_gpu_nccl.py), launched by torch.distributed.run:
rank r drives cuda:r, gets the NCCL id through torch.distributed (nccl backend), runs a row-slab
solve of the case in argv[1] (the product library: real NCCL, packed halo exchange, interior /
boundary split, CUDA-graph replay) and saves its slab's fields, labels and records to argv[2]_r.npz."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2510_16154_b200 as msa  # noqa: E402
from _loopback_case import FIELDS, image  # noqa: E402


def main():
    spec = json.loads(sys.argv[1])
    out = sys.argv[2]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    B, H, W, C = spec["shape"]
    I = image(np.random.default_rng(spec["seed"]), B, H, W, C)
    nid = [msa.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(nid, src=0)
    p = msa.Params(batch=B, height=H, width=W, channels=C, shard=msa.SHARD_ROWS, rank=rank, world=world, device=rank,
                   nccl_id=nid[0], **spec["params"])
    res = {}
    with msa.Solver(p, I) as s:
        st = s.solve()
        st += s.solve()  # a second solve from the new state replays / re-captures the graph
        s.set_timing(True)
        s.step(p.iters_per_round)
        info = s.query()
        for k, w in FIELDS:
            res[k] = s.get_field(w)
        lab, cnt, pal = s.labels(0.1, 64)
    res.update(lab=lab, cnt=cnt, pal=pal, row0=info.row0, nrows=info.nrows, halo_ms=info.halo_ms,
               halo_exchanges=info.halo_exchanges, e_tv=np.array([r["e_tv"] for r in st]))
    np.savez(f"{out}_{rank}.npz", **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
