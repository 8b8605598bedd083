"""gloo worker for tests/test_distributed_cpu.py (world size 2)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import slab_model as M  # noqa: E402
from paper_2006_04391_b200 import distributed as D  # noqa: E402


def main():
    dist.init_process_group("gloo")
    r, k = dist.get_rank(), dist.get_world_size()
    # 1. NCCL id hand-off through the torch group
    c = D.comm_from_torch()
    ids = [None] * k
    dist.all_gather_object(ids, c.uid)
    assert c.rank == r and c.world == k and len(c.uid) == 128 and all(u == ids[0] for u in ids)
    # 2. slab decomposition of the transforms vs the global numpy rfftn
    for nx, ny, nz in ((8, 6, 5), (4, 4, 8), (16, 8, 7)):
        rng = np.random.default_rng(7)
        g = rng.normal(size=(6, nx, ny, nz))
        x0, x1 = D.slab_range(nx, k, r)
        S = M.forward(g[:, x0:x1], nx)
        ref = np.fft.rfftn(g, axes=(1, 2, 3))  # (6, nx, ny, nzh)
        nyl = ny // k
        want = ref[:, :, r * nyl:(r + 1) * nyl, :].transpose(1, 0, 2, 3)
        assert np.max(np.abs(S - want)) <= 1e-12 * np.max(np.abs(ref)), "forward transpose"
        back = M.inverse(S, ny, nz) / (nx * ny * nz)
        assert np.max(np.abs(back - g[:, x0:x1])) <= 1e-12, "inverse transpose"
        # 3. reduction slots: disjoint per rank, their sum in index order is independent of k
        part = M.plane_partials(S, r * nyl, ny, nz // 2 + 1)
        t = torch.from_numpy(part)
        dist.all_reduce(t)
        whole = M.plane_partials(ref.transpose(1, 0, 2, 3), 0, ny, nz // 2 + 1)
        assert np.array_equal(t.numpy(), whole), "reduction slots depend on the slab count"
        # 4. plane-ordered field means (eps.mean(), sigma_bar) and C_bar records
        # (solver.cu field_means / k_refstats_planes): each rank fills the
        # records of its own x planes, zeros elsewhere; the all-reduce is
        # exact and the plane-ordered sum equals the one-rank result bitwise
        pl = np.zeros((nx, 6))
        pl[x0:x1] = g[:, x0:x1].sum(axis=(2, 3)).T
        t = torch.from_numpy(pl)
        dist.all_reduce(t)
        assert np.array_equal(t.numpy(), g.sum(axis=(2, 3)).T), "plane records depend on the slab count"
    dist.barrier()
    if r == 0:
        print("WORKER-OK", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
