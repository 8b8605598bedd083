"""GPU basic scheme (csrc/solver.cu through paper_2006_04391_b200.homogenize) vs
the reference fixtures and the numpy oracle.

Bars (BASELINE.json north star): identical basic-scheme iteration counts,
fields / homogenized stress within 1e-10 relative, tangent-derived
quantities within 1e-8 relative.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import homogenize as OH
from oracle import material as OM

pytestmark = pytest.mark.gpu

TOL = 1e-10


def rel(x, y):
    x, y = np.asarray(x, float), np.asarray(y, float)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300))


@pytest.fixture(scope="module")
def H():
    from paper_2006_04391_b200 import homogenize

    return homogenize


@pytest.fixture(scope="module")
def AUTO():
    from paper_2006_04391_b200.evaluator import StrategyConfig

    return StrategyConfig(strategy="automatic", integrator="implicit-euler")


def test_fourier_operators_golden(H):
    g = golden("fourier.npz")
    ref = H.ReferenceMaterial(*g["ref"])
    for k in range(int(g["ndims"])):
        t = f"d{k}_"
        assert rel(H.GreenOperator(g[t + "dims"], ref).apply(g[t + "tau"]), g[t + "green"]) < 1e-13
        assert abs(H.equilibrium_residual(g[t + "sig"]) / float(g[t + "residual"]) - 1) < 1e-12
        assert rel(H.apply_isotropic(ref, g[t + "eps"]), g[t + "iso"]) < 1e-15
    for k in range(3):
        r = H.reference_update(g[f"ru{k}_C"])
        assert rel([r.lam, r.mu], g[f"ru{k}_lam_mu"]) < 1e-13


@pytest.mark.parametrize("dims", [(64, 64, 64), (9, 8, 7), (16, 12, 10), (2, 3, 4), (1, 1, 6)])
def test_fourier_operators_random(H, dims):
    rng = np.random.default_rng(sum(dims))
    tau = rng.normal(0, 1e8, (6,) + dims)
    lam, mu = 8e10, 7e10
    assert rel(H.green_apply(tau, H.ReferenceMaterial(lam, mu)), OH.green_apply(tau, lam, mu)) < 1e-13
    sig = tau + np.array([3e8, 1e8, -2e8, 1e7, 0, 5e6])[:, None, None, None]
    assert abs(H.equilibrium_residual(sig) / OH.residual(sig) - 1) < 1e-12
    # constant tau -> zero correction
    const = np.broadcast_to(np.arange(1.0, 7.0)[:, None, None, None], (6,) + dims).copy()
    assert np.max(np.abs(H.green_apply(const, H.ReferenceMaterial(lam, mu)))) < 1e-12 * 6 / mu


def test_reference_update_errors(H):
    C = np.broadcast_to(np.eye(6) * 1e10, (4, 6, 6)).copy()
    C[2, 1, 1] = np.nan
    with pytest.raises(ValueError):
        H.reference_update(C)


@pytest.mark.parametrize("tag", ["strain", "mixed"])
def test_config1(H, AUTO, tag):
    from paper_2006_04391_b200 import gsm

    g = golden("config1.npz")
    grid = H.VoxelGrid(g["ids"], [gsm.LinearElastic(55e9, 0.33), gsm.LinearElastic(300e9, 0.25)])
    hom = H.Homogenizer(grid, AUTO)
    assert rel([hom.reference.lam, hom.reference.mu], g[f"{tag}_ref"]) < 1e-14
    eb = np.zeros(6)
    eb[0] = 1e-3
    free = np.zeros(6, bool) if tag == "strain" else np.array([False] + [True] * 5)
    eps, sig, info = hom.solve_step(eb, 1.0, free_mask=free)
    assert info.iterations == int(g[f"{tag}_iters"])
    assert len(info.history) == info.iterations
    assert rel(info.history, g[f"{tag}_history"]) < 1e-8
    sub = g["sub"]
    assert rel(sig.reshape(6, -1)[:, sub], g[f"{tag}_sig_sub"]) < TOL
    assert rel(eps.reshape(6, -1)[:, sub], g[f"{tag}_eps_sub"]) < TOL
    assert rel(sig.mean(axis=(1, 2, 3))[:3], g[f"{tag}_sig_bar"][:3]) < TOL


def test_config1_solver_error(H, AUTO):
    from paper_2006_04391_b200 import gsm

    g = golden("config1.npz")
    grid = H.VoxelGrid(g["ids"], [gsm.LinearElastic(55e9, 0.33), gsm.LinearElastic(300e9, 0.25)])
    hom = H.Homogenizer(grid, AUTO, max_iterations=4)
    eb = np.zeros(6)
    eb[0] = 1e-3
    with pytest.raises(H.SolverError) as ei:
        hom.solve_step(eb, 1.0)
    assert rel(ei.value.history, g["cap_history"]) < 1e-8


def test_path8_manual_loop(H, AUTO):
    """The reference's per-step sequence through the public Homogenizer API (8^3, 6 steps)."""
    g = golden("path8_auto.npz")
    grid = H.toy_mmc_grid(8)
    assert np.array_equal(grid.material_ids, g["ids"])
    hom = H.Homogenizer(grid, AUTO)
    path = H.LoadingPath(steps=20)
    times = path.times()
    targets = path.eps_xx(times)
    free = np.array([False, True, True, True, True, True])
    for k in range(1, 7):
        dt = times[k] - times[k - 1]
        eb = np.zeros(6)
        eb[0] = targets[k]
        eps, sigma, info = hom.solve_step(eb, dt, free_mask=free)
        assert info.iterations == g["iterations"][k - 1]
        assert rel(sigma.mean(axis=(1, 2, 3)), g["sig"][k - 1]) < TOL
        ebar = eps.mean(axis=(1, 2, 3))
        _, C_vox, _, _ = hom.evaluate_field(eps, dt, want_tangent=True)
        assert rel(C_vox.mean(axis=0), g["Cbar"][k - 1]) < 1e-8
        hom.commit_step(eps, ebar)
        hom.set_reference(H.reference_update(C_vox))
        assert rel([hom.reference.lam, hom.reference.mu], g["refs"][k]) < 1e-8
    assert rel(hom.eps_n, g["eps_n"]) < TOL
    assert rel(grid.state[0], g["state0"]) < TOL


@pytest.mark.parametrize("warm", [False, True])
def test_run_loading_path_16(H, AUTO, warm):
    """Full 20-step path at 16^3: identical iteration counts
    (also with the Newton warm start, which changes per-voxel Newton counts only)."""
    g = golden("path16_conv.npz")
    grid = H.toy_mmc_grid(16)
    assert np.array_equal(grid.material_ids, g["ids"])
    recs = H.run_loading_path(grid, H.LoadingPath(steps=20), AUTO, newton_warm_start=warm)
    assert [r["iterations"] for r in recs] == g["iterations"].tolist()
    sig = np.stack([r["sig"] for r in recs])
    assert rel(sig[:, 0], g["sig"][:, 0]) < 1e-9
    assert rel([r["C11"] for r in recs], g["C11"]) < 1e-8
    assert rel([r["C12"] for r in recs], g["C12"]) < 1e-8
    assert rel([r["eps_xx"] for r in recs], g["eps_xx"]) < 1e-9
    assert all(r["mean_substeps"] == 1.0 for r in recs)


@pytest.mark.parametrize("slabs", [1, 2])
def test_warm_start_matches_cold(H, AUTO, slabs):
    """Newton warm start: same basic-scheme iterations, fields equal to round-off (32^3, 3 steps)."""
    out = []
    for warm in (False, True):
        hom = H.Homogenizer(H.toy_mmc_grid(32), AUTO, newton_warm_start=warm, slabs=slabs)
        path = H.LoadingPath(steps=20)
        t = path.times()
        res = []
        for k in range(1, 4):
            eb = np.zeros(6)
            eb[0] = path.eps_xx(t[k])
            eps, sigma, info = hom.solve_step(eb, t[k] - t[k - 1], free_mask=np.array([False] + [True] * 5))
            res.append((info.iterations, eps, sigma))
            hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
        out.append((res, hom.grid.state[0]))
    (cold, s_cold), (warm, s_warm) = out
    for (ic, ec, sc), (iw, ew, sw) in zip(cold, warm):
        assert ic == iw
        assert rel(ew, ec) < 1e-12 and rel(sw, sc) < 1e-12
    assert rel(s_warm, s_cold) < 1e-12


def test_odd_grid_vs_oracle(H, AUTO):
    """Odd, anisotropic 9x8x7 two-phase EVP grid, two loading steps vs the oracle."""
    from paper_2006_04391_b200 import gsm

    rng = np.random.default_rng(4)
    ids = (rng.random((9, 8, 7)) < 0.25).astype(np.uint8)
    grid = H.VoxelGrid(ids, [gsm.MichelSuquet(), gsm.LinearElastic(300e9, 0.25)])
    hom = H.Homogenizer(grid, AUTO)
    ob = OH.Basic(ids, [OM.ALUMINUM, OM.law_params(0, 300e9, 0.25)])
    t, ex = OH.loading_times(20)
    free = np.array([False, True, True, True, True, True])
    for k in (1, 2):
        dt = t[k] - t[k - 1]
        eb = np.zeros(6)
        eb[0] = ex[k]
        eps, sig, info = hom.solve_step(eb, dt, free_mask=free)
        oe, osig, oit, _ = ob.solve_step(eb, dt, free)
        assert info.iterations == oit
        assert rel(sig, osig) < TOL and rel(eps, oe) < TOL
        ebar = eps.mean(axis=(1, 2, 3))
        _, C, _, _ = hom.evaluate_field(eps, dt, want_tangent=True)
        _, oC, _ = ob.evaluate(oe, dt, True)
        assert rel(C, oC) < 1e-8
        hom.commit_step(eps, ebar)
        ob.commit(oe, oe.mean(axis=(1, 2, 3)))
        hom.set_reference(H.reference_update(C))
        ob.lam, ob.mu = OH.reference_update(oC)
        assert rel([hom.reference.lam, hom.reference.mu], [ob.lam, ob.mu]) < 1e-8
    assert rel(grid.state[0], ob.state[0]) < TOL


def test_empty_phase_and_evaluate_field(H, AUTO):
    """An unused material id, evaluate_field without tangent, free_mask None."""
    from paper_2006_04391_b200 import gsm

    ids = np.zeros((8, 6, 4), dtype=np.uint8)
    ids[2:4] = 2
    laws = [gsm.MichelSuquet(), gsm.LinearElastic(300e9, 0.25), gsm.LinearElastic(70e9, 0.3)]
    grid = H.VoxelGrid(ids, laws)
    hom = H.Homogenizer(grid, AUTO)
    ob = OH.Basic(ids, [OM.ALUMINUM, OM.law_params(0, 300e9, 0.25), OM.law_params(0, 70e9, 0.3)])
    assert rel([hom.reference.lam, hom.reference.mu], [ob.lam, ob.mu]) < 1e-14
    eb = np.array([2e-3, 0, 0, 0, 0, 5e-4])
    eps, sig, info = hom.solve_step(eb, 0.1)
    oe, osig, oit, _ = ob.solve_step(eb, 0.1)
    assert info.iterations == oit and rel(sig, osig) < TOL
    s2, C, state, mean_sub = hom.evaluate_field(eps, 0.1)
    assert C is None and mean_sub == 1.0 and rel(s2, sig) < 1e-15
    assert state[1].shape == (0, 0) and state[0].shape == (len(grid.voxel_index[0]), 7)
    hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
    assert rel(grid.state[0], ob.pending[0] if ob.pending is not None else ob.evaluate(oe, 0.1)[2][0]) < TOL


def test_slab_count_must_divide(H, AUTO):
    from paper_2006_04391_b200 import gsm

    grid = H.VoxelGrid(np.zeros((6, 6, 4), dtype=np.uint8), [gsm.LinearElastic(1e9, 0.3)])
    with pytest.raises(ValueError):
        H.Homogenizer(grid, AUTO, slabs=4)
