"""Parity at sizes the oracle cannot run end to end:
per-voxel parity of sampled voxels of a converged 128^3 load step against
the C oracle, and one field step (Green operator, residual) of that grid
against the numpy oracle."""

import numpy as np
import pytest

from oracle import homogenize as OH
from oracle import material as OM

pytestmark = pytest.mark.gpu


def rel(x, y):
    x, y = np.asarray(x, float), np.asarray(y, float)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300))


def test_sampled_voxels_128():
    from paper_2006_04391_b200 import homogenize as H
    from paper_2006_04391_b200.evaluator import StrategyConfig

    cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
    grid = H.toy_mmc_grid(128)
    hom = H.Homogenizer(grid, cfg)
    path = H.LoadingPath(steps=20)
    t = path.times()
    eb = np.zeros(6)
    eb[0] = path.eps_xx(t)[2]  # a step deep enough to be plastic almost everywhere
    dt = t[1] - t[0]
    eps, sig, info = hom.solve_step(eb, dt, free_mask=np.array([False] + [True] * 5))
    assert info.iterations > 10
    pend = np.empty((len(grid.voxel_index[0]), 7))
    hom._pull_state([pend, np.empty((len(grid.voxel_index[1]), 0))], pending=True)
    rng = np.random.default_rng(0)
    pick = np.sort(rng.choice(len(grid.voxel_index[0]), 4096, replace=False))
    vox = grid.voxel_index[0][pick]
    e = eps.reshape(6, -1)[:, vox].T
    r = OM.evaluate(OM.ALUMINUM, np.zeros_like(e), np.zeros((len(vox), 7)), e, np.full(len(vox), dt), False,
                    threads=8)
    assert np.all(r["status"] == 0)
    assert rel(sig.reshape(6, -1)[:, vox].T, r["sigma"]) < 1e-10
    assert rel(pend[pick], r["a"]) < 1e-10
    # one field step of the converged grid against the numpy oracle
    lam, mu = hom.reference.lam, hom.reference.mu
    tau = sig - OH.iso(lam, mu, eps)
    assert rel(H.GreenOperator(grid.dims, hom.reference).apply(tau), OH.green_apply(tau, lam, mu)) < 1e-12
    assert abs(H.equilibrium_residual(sig) / OH.residual(sig) - 1) < 1e-10
    assert abs(info.residual / OH.residual(sig) - 1) < 1e-8
