"""NCCL worker for tests/test_slabs_gpu.py: one process per GPU (here world 1
on the test box: the transposes run through ncclAlltoAll to the rank itself).
Writes the run_loading_path records of a small path to argv[1] (rank 0)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_04391_b200 import distributed as D, homogenize as H  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig  # noqa: E402


def main():
    dist.init_process_group("gloo")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    from paper_2006_04391_b200 import _lib

    _lib.check(_lib.load().am_set_device(local))
    comm = D.comm_from_torch(transport=sys.argv[2] if len(sys.argv) > 2 else "p2p")
    cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
    grid = H.toy_mmc_grid(16)
    hom = H.Homogenizer(grid, cfg, comm=comm)
    path = H.LoadingPath(steps=20)
    t = path.times()
    ex = path.eps_xx(t)
    out = []
    for k in (1, 2, 3):
        eb = np.zeros(6)
        eb[0] = ex[k]
        eps, sig, info = hom.solve_step(eb, t[k] - t[k - 1], free_mask=np.array([False] + [True] * 5))
        out.append({"iterations": info.iterations, "history": info.history,
                    "eps_slab_sum": float(np.sum(eps)), "sig_slab": sig.tolist() if k == 3 else None})
        hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
    if comm.rank == 0:
        json.dump(out, open(sys.argv[1], "w"))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
