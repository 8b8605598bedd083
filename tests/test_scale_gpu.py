"""Parity at the benchmarked sizes, where the oracle cannot run a load step
end to end:

* per-voxel parity of >= 2^16 sampled EVP voxels at the converged iteration
  of load step 1 of config 4 (256^3) and config 5 (512^3, fibre E = 3000
  GPa): the voxels' (eps_n, a_n, eps, dt) are dumped from the device and
  re-evaluated by the C oracle (per-voxel results do not depend on the
  batch); stress and internal state within 1e-10, the consistent tangent
  within 1e-8, each voxel scaled by its own magnitude;
* one full-grid basic-scheme field step (homogenize.py:445-465: residual,
  mixed-BC update, Green operator) against the numpy oracle: the device's
  iterate k+1 from its (eps_k, sigma_k); at 512^3 with the Green table
  built kx-slab by kx-slab.

Iteration counts at these sizes cannot be checked against a reference run
(weeks of CPU); they are checked against the slab-decomposed solver
(tests/test_slabs_gpu.py) and, at 16^3-128^3, against the reference's
fixtures (tests/test_homogenize_gpu.py).
"""

import os

import numpy as np
import pytest

from _util import rowwise_relerr
from oracle import homogenize as OH
from oracle import material as OM

pytestmark = pytest.mark.gpu

FREE = np.array([False] + [True] * 5)


def rel(x, y):
    x, y = np.asarray(x, float), np.asarray(y, float)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300))


@pytest.fixture(scope="module")
def mods():
    from paper_2006_04391_b200 import gsm
    from paper_2006_04391_b200 import homogenize as H
    from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays

    return gsm, H, StrategyConfig(strategy="automatic", integrator="implicit-euler"), evaluate_arrays


def _grid(mods, n, fibre_E):
    gsm, H, _, _ = mods
    fibre = gsm.LinearElastic(fibre_E, 0.25) if fibre_E else None
    return H.toy_mmc_grid(n, fiber_law=fibre)


def _step1(H):
    path = H.LoadingPath(steps=20)
    t = path.times()
    eb = np.zeros(6)
    eb[0] = path.eps_xx(t)[1]
    return eb, t[1] - t[0]


def _sampled_voxels(mods, grid, hom, eps, sig, dt, nsample, parity_log, tag, C_field=None):
    """(eps_n = 0, a_n = 0, eps) of sampled EVP voxels of load step 1 through
    the C oracle: sigma and the pending state (the converged evaluation's)
    within 1e-10; C within 1e-8, from the solver's own tangent sweep when
    C_field is given, else from the material-point entry on the same inputs."""
    _, _, cfg, evaluate_arrays = mods
    idx0 = grid.voxel_index[0]
    pend = np.empty((len(idx0), 7))
    hom._pull_state([pend] + [np.empty((len(i), 0)) for i in grid.voxel_index[1:]], pending=1)
    rng = np.random.default_rng(0)
    pick = np.sort(rng.choice(len(idx0), nsample, replace=False))
    vox = idx0[pick]
    e = np.ascontiguousarray(eps.reshape(6, -1)[:, vox].T)
    z6, z7 = np.zeros_like(e), np.zeros((len(vox), 7))
    r = OM.evaluate(OM.ALUMINUM, z6, z7, e, np.full(len(vox), dt), True, threads=os.cpu_count() or 8)
    assert np.all(r["status"] == 0)
    errs = {
        "voxels": int(len(vox)),
        "plastic_frac": float(np.mean(r["iters"] > 1)),
        "sigma": float(rowwise_relerr(sig.reshape(6, -1)[:, vox].T, r["sigma"]).max()),
        "a": float(rowwise_relerr(pend[pick], r["a"]).max()),
    }
    if C_field is not None:
        errs["C_solver_sweep"] = float(rowwise_relerr(C_field[vox], r["C"]).max())
    g = evaluate_arrays(grid.materials[0], cfg, z6, z7, e, np.full(len(vox), dt), want_tangent=True)
    errs["C_eval_arrays"] = float(rowwise_relerr(g.C, r["C"]).max())
    errs["newton_counts_equal"] = bool(np.array_equal(g.newton_iters, r["iters"]))
    parity_log(tag, **errs)
    assert errs["sigma"] <= 1e-10 and errs["a"] <= 1e-10, errs
    assert errs["C_eval_arrays"] <= 1e-8 and errs.get("C_solver_sweep", 0.0) <= 1e-8, errs
    assert errs["newton_counts_equal"]
    return errs


def _field_step(mods, grid, dt, eb, k, parity_log, tag, slabwise=False):
    """Device iterate k+1 of load step 1 vs the numpy oracle applied to the
    device's (eps_k, sigma_k): eps_{k+1} = ebar_{k+1} + fluct with the
    mixed-BC update of the free mean strains (homogenize.py:459-465)."""
    gsm, H, cfg, _ = mods
    hom = H.Homogenizer(grid, cfg, max_iterations=k - 1)
    with pytest.raises(H.SolverError):
        hom.solve_step(eb, dt, free_mask=FREE)
    eps_k = hom._get(0)
    hom.max_iterations = k
    with pytest.raises(H.SolverError) as ei:
        hom.solve_step(eb, dt, free_mask=FREE)
    eps_k1, sig_k = hom._get(0), hom._get(2)
    lam, mu = hom.reference.lam, hom.reference.mu
    hist = ei.value.history
    del hom
    sbar = sig_k.mean(axis=(1, 2, 3))
    res = OH.residual(sig_k)
    scale = np.sqrt(np.sum(sbar * OH.DUP * sbar))
    res_bc = np.linalg.norm(sbar[FREE]) / scale
    ebar = eps_k.mean(axis=(1, 2, 3))
    ebar[FREE] += np.linalg.solve(OH.iso_matrix(lam, mu)[np.ix_(FREE, FREE)], -sbar[FREE])
    tau = sig_k - OH.iso(lam, mu, eps_k)
    del eps_k
    fl = OH.green_apply_slabwise(tau, lam, mu) if slabwise else OH.green_apply(tau, lam, mu)
    del tau
    for c in range(6):
        fl[c] += ebar[c]
    errs = {"iteration": k, "eps_next": rel(eps_k1, fl), "residual": abs(hist[-1] / max(res, res_bc) - 1)}
    parity_log(tag, **errs)
    assert errs["eps_next"] <= 1e-10 and errs["residual"] <= 1e-10, errs


def test_config4_256_step1(mods, parity_log):
    """Config 4 grid, load step 1: 2^16 sampled voxels (C from the solver's
    tangent sweep itself) and the field step at iteration 20."""
    _, H, cfg, _ = mods
    grid = _grid(mods, 256, None)
    eb, dt = _step1(H)
    hom = H.Homogenizer(grid, cfg)
    eps, sig, info = hom.solve_step(eb, dt, free_mask=FREE)
    assert info.iterations > 10
    _, C, _, _ = hom.evaluate_field(eps, dt, want_tangent=True)
    _sampled_voxels(mods, grid, hom, eps, sig, dt, 1 << 16, parity_log, "config4_256_sampled", C_field=C)
    parity_log("config4_256_iterations", iterations=info.iterations)
    del C, hom
    _field_step(mods, grid, dt, eb, 20, parity_log, "config4_256_field_step")


def test_config5_512_step1(mods, parity_log):
    """Config 5 grid (fibre E = 3000 GPa, ~55x contrast), load step 1 on one
    GPU: 2^16 sampled voxels at the converged iteration and the field step
    at iteration 20 with the slab-wise Green table."""
    _, H, cfg, _ = mods
    grid = _grid(mods, 512, 3000e9)
    eb, dt = _step1(H)
    hom = H.Homogenizer(grid, cfg)
    eps, sig, info = hom.solve_step(eb, dt, free_mask=FREE)
    parity_log("config5_512_iterations", iterations=info.iterations)
    _sampled_voxels(mods, grid, hom, eps, sig, dt, 1 << 16, parity_log, "config5_512_sampled")
    del hom, eps, sig
    _field_step(mods, grid, dt, eb, 20, parity_log, "config5_512_field_step", slabwise=True)


def test_config4_256_slab_algorithm(mods, parity_log):
    """The multi-GPU algorithm (x slabs, 2-D FFTs, transposes, 1-D FFTs over
    x) at the config-4 size, on 2 / 4 / 8 slabs of one GPU: the single-slab
    run's iteration count, fields within 1e-10, and bitwise equal results
    for every slab count (the NCCL mode runs the same kernels per rank)."""
    _, H, cfg, _ = mods
    grid = _grid(mods, 256, None)
    eb, dt = _step1(H)
    hom = H.Homogenizer(H.VoxelGrid(grid.material_ids, grid.materials), cfg)
    eps0, sig0, info0 = hom.solve_step(eb, dt, free_mask=FREE)
    del hom
    ref = None
    errs = {}
    for k in (2, 4, 8):
        hom = H.Homogenizer(H.VoxelGrid(grid.material_ids, grid.materials), cfg, slabs=k)
        eps, sig, info = hom.solve_step(eb, dt, free_mask=FREE)
        del hom
        assert info.iterations == info0.iterations
        errs[f"slabs{k}_sigma"] = rel(sig, sig0)
        errs[f"slabs{k}_eps"] = rel(eps, eps0)
        assert errs[f"slabs{k}_sigma"] <= 1e-10 and errs[f"slabs{k}_eps"] <= 1e-10
        if ref is None:
            ref = (eps, sig, info.history)
        else:
            errs[f"slabs{k}_bitwise_equal_to_2"] = bool(np.array_equal(eps, ref[0]) and np.array_equal(sig, ref[1])
                                                        and info.history == ref[2])
            assert errs[f"slabs{k}_bitwise_equal_to_2"]
    parity_log("config4_256_slab_algorithm", iterations=info0.iterations, **errs)
