"""GPU basic scheme (csrc/solver.cu through paper_2006_04391_b200.homogenize) vs
the reference fixtures and the numpy oracle.

Bars (BASELINE.json north star): identical basic-scheme iteration counts,
fields / homogenized stress within 1e-10 relative, tangent-derived
quantities within 1e-8 relative.
"""

import numpy as np
import pytest

from _util import check_path_records, rowwise_relerr
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


def _path_fixture(n):
    import os

    from conftest import GOLDEN

    f = os.path.join(GOLDEN, f"path{n}_conv.npz")
    if not os.path.exists(f):
        pytest.skip(f"no reference fixture for the {n}^3 path")
    return np.load(f)


@pytest.mark.parametrize("warm", [False, True])
@pytest.mark.parametrize("n", [16, 32, 64, 128])
def test_run_loading_path(H, AUTO, n, warm, parity_log):
    """Full 20-step path at n^3 vs the reference (per-law conventional route,
    SURVEY §8c / App. A.2b; identical counts to the automatic route at 16^3):
    identical iteration counts, also with the Newton warm start (which
    changes per-voxel Newton counts only)."""
    g = _path_fixture(n)
    grid = H.toy_mmc_grid(n)
    assert np.array_equal(grid.material_ids, g["ids"])
    recs = H.run_loading_path(grid, H.LoadingPath(steps=20), AUTO, newton_warm_start=warm)
    check_path_records(recs, g, f"path{n}{'_warm' if warm else ''}", parity_log)
    if len(g["iterations"]) == 20 and not warm:
        # committed state and strain of the last step at the sampled voxels
        sub = g["sub"]
        st = np.zeros((n**3, 7))
        st[grid.voxel_index[0]] = grid.state[0]
        e_state = float(rowwise_relerr(st[sub], g["state_sub"].T).max())
        parity_log(f"path{n}_final_state", state=e_state)
        assert e_state <= TOL


def test_path_manual_loop_32(H, AUTO, parity_log):
    """The reference's per-step sequence through the public Homogenizer API
    at 32^3 (first 4 steps): per-step histories, full C_bar, reference
    materials and eps.mean() as the committed mean strain."""
    g = _path_fixture(32)
    grid = H.toy_mmc_grid(32)
    hom = H.Homogenizer(grid, AUTO)
    path = H.LoadingPath(steps=20)
    times = path.times()
    targets = path.eps_xx(times)
    free = np.array([False, True, True, True, True, True])
    hist = np.split(g["history_flat"], np.cumsum(g["iterations"])[:-1])
    worst = dict(hist=0.0, ebar=0.0, Cbar=0.0, ref=0.0)
    for k in range(1, 5):
        dt = times[k] - times[k - 1]
        eb = np.zeros(6)
        eb[0] = targets[k]
        eps, sigma, info = hom.solve_step(eb, dt, free_mask=free)
        assert info.iterations == g["iterations"][k - 1]
        worst["hist"] = max(worst["hist"], rel(info.history, hist[k - 1]))
        ebar = eps.mean(axis=(1, 2, 3))
        worst["ebar"] = max(worst["ebar"], rel(ebar, g["ebar"][k - 1]))
        _, C_vox, _, _ = hom.evaluate_field(eps, dt, want_tangent=True)
        worst["Cbar"] = max(worst["Cbar"], rel(C_vox.mean(axis=0), g["Cbar"][k - 1]))
        hom.commit_step(eps, ebar)
        hom.set_reference(H.reference_update(C_vox))
        worst["ref"] = max(worst["ref"], rel([hom.reference.lam, hom.reference.mu], g["refs"][k]))
    parity_log("path32_manual", **worst)
    assert worst["hist"] < 1e-8 and worst["ebar"] < TOL and worst["Cbar"] < 1e-8 and worst["ref"] < 1e-8, worst


def test_commit_keeps_solve_step_state(H, AUTO):
    """commit_step commits the state of the last converged solve_step, not
    that of a later evaluate_field at another strain (homogenize.py:455-457,
    474-480); without a solve_step nothing is committed."""
    grid = H.toy_mmc_grid(8)
    hom = H.Homogenizer(grid, AUTO)
    free = np.array([False] + [True] * 5)
    eb = np.array([2e-3, 0, 0, 0, 0, 0])
    eps, sigma, info = hom.solve_step(eb, 0.4, free_mask=free)
    _, _, state_conv, _ = hom.evaluate_field(eps, 0.4)
    s2, C2, state_pert, _ = hom.evaluate_field(1.5 * eps, 0.4, want_tangent=True)
    assert rel(state_pert[0], state_conv[0]) > 1e-3  # the perturbed evaluation differs
    hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
    assert rel(grid.state[0], state_conv[0]) == 0.0
    assert rel(hom.eps_n, eps) == 0.0
    # evaluate_field alone, then commit: the committed state stays
    before = grid.state[0].copy()
    hom.evaluate_field(2.0 * eps, 0.4)
    hom.commit_step(2.0 * eps, 2.0 * eps.mean(axis=(1, 2, 3)))
    assert rel(grid.state[0], before) == 0.0
    assert rel(hom.eps_n, 2.0 * eps) == 0.0


def test_path8_default_cfg_ode23(H):
    """First 3 steps of the 8^3 path with the default StrategyConfig()
    (automatic, ode23) against the reference: the per-step tangent sweep is
    a coupled adaptive integration with its own step sequence, and the
    committed state must still be solve_step's (homogenize.py:508-512)."""
    import os

    from conftest import GOLDEN
    from paper_2006_04391_b200.evaluator import StrategyConfig

    f = os.path.join(GOLDEN, "path8_ode23.npz")
    if not os.path.exists(f):
        pytest.skip("no ode23 path fixture")
    g = np.load(f)
    grid = H.toy_mmc_grid(8)
    hom = H.Homogenizer(grid, StrategyConfig())
    path = H.LoadingPath()  # 80 steps (homogenize.py:52-77)
    times = path.times()
    free = np.array([False] + [True] * 5)
    for k in range(1, 4):
        dt = times[k] - times[k - 1]
        eb = np.zeros(6)
        eb[0] = path.eps_xx(times[k])
        eps, sigma, info = hom.solve_step(eb, dt, free_mask=free)
        assert info.iterations == g["iterations"][k - 1]
        assert info.mean_substeps == pytest.approx(g["mean_substeps"][k - 1], rel=1e-12)
        assert rel(sigma.mean(axis=(1, 2, 3)), g["sig"][k - 1]) < TOL
        ebar = eps.mean(axis=(1, 2, 3))
        _, C_vox, _, _ = hom.evaluate_field(eps, dt, want_tangent=True)
        assert rel(C_vox.mean(axis=0), g["Cbar"][k - 1]) < 1e-8
        hom.commit_step(eps, ebar)
        hom.set_reference(H.reference_update(C_vox))
        assert rel([hom.reference.lam, hom.reference.mu], g["refs"][k]) < 1e-8
    st = np.zeros((512, 7))
    st[grid.voxel_index[0]] = grid.state[0]
    assert float(rowwise_relerr(st[g["sub"]], g["state_sub"].T).max()) <= TOL


def test_path8_default_cfg_ode23_solver_error(H, parity_log):
    """LoadingPath(steps=20) with the default StrategyConfig(): the reference
    converges step 1 and raises SolverError in step 2 after 5000 iterations
    (ode23's error control keeps the residual above tol); so must this."""
    from paper_2006_04391_b200.evaluator import StrategyConfig

    g = golden("path8_ode23_fail.npz")
    grid = H.toy_mmc_grid(8)
    hom = H.Homogenizer(grid, StrategyConfig())
    path = H.LoadingPath(steps=20)
    t = path.times()
    free = np.array([False] + [True] * 5)
    eb = np.zeros(6)
    eb[0] = path.eps_xx(t[1])
    eps, sigma, info = hom.solve_step(eb, t[1], free_mask=free)
    assert info.iterations == int(g["step1_iters"])
    assert rel(sigma.mean(axis=(1, 2, 3)), g["step1_sig"]) < TOL
    _, C_vox, _, _ = hom.evaluate_field(eps, t[1], want_tangent=True)
    hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
    hom.set_reference(H.reference_update(C_vox))
    eb[0] = path.eps_xx(t[2])
    with pytest.raises(H.SolverError) as ei:
        hom.solve_step(eb, t[2] - t[1], free_mask=free)
    hist, ref = np.array(ei.value.history), g["fail_history"]
    assert len(hist) == len(ref) == 5000
    # the residual sequence follows the reference's until the adaptive step
    # controller's discrete decisions amplify round-off
    agree = int(np.argmax(np.abs(hist - ref) > 1e-6 * np.abs(ref))) or len(ref)
    parity_log("path8_ode23_fail", history_agree=agree, last=float(hist[-1]), ref_last=float(ref[-1]))
    assert agree >= 20


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


def test_grid_keeps_committed_state(H, AUTO):
    """The grid carries the committed state like the reference's in-place
    commits: after run_loading_path (whose solver is released) grid.state is
    the final state, and a new Homogenizer on the grid starts from it."""
    g8 = H.toy_mmc_grid(8)
    recs = H.run_loading_path(g8, H.LoadingPath(steps=20), AUTO)
    final = [a.copy() for a in g8.state]
    assert np.max(np.abs(final[0])) > 0.0
    hom = H.Homogenizer(g8, AUTO)
    assert rel(g8.state[0], final[0]) == 0.0
    eb = np.zeros(6)
    eb[0] = recs[-1]["eps_xx"]
    eps, sig, info = hom.solve_step(eb, 0.1, free_mask=np.array([False] + [True] * 5))
    hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
    committed = [a.copy() for a in g8.state]
    del hom  # released: the grid keeps what was committed
    assert rel(g8.state[0], committed[0]) == 0.0


def test_graph_replay_bitwise_equal_to_eager(H, AUTO):
    """The per-step CUDA graph replays the eager iteration's kernels in the
    same order: fields and histories are bitwise identical (AM_NO_GRAPHS=1
    selects the eager path at solver creation)."""
    import os

    out = []
    for off in ("1", "0"):
        os.environ["AM_NO_GRAPHS"] = off
        try:
            hom = H.Homogenizer(H.toy_mmc_grid(16), AUTO)
        finally:
            os.environ.pop("AM_NO_GRAPHS", None)
        path = H.LoadingPath(steps=20)
        t = path.times()
        res = []
        for k in (1, 2):
            eb = np.zeros(6)
            eb[0] = path.eps_xx(t[k])
            eps, sig, info = hom.solve_step(eb, t[k] - t[k - 1], free_mask=np.array([False] + [True] * 5))
            res.append((eps, sig, info.history))
            hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
        out.append(res)
    for (e0, s0, h0), (e1, s1, h1) in zip(*out):
        assert np.array_equal(e0, e1) and np.array_equal(s0, s1) and h0 == h1


@pytest.mark.parametrize("graphs,slabs", [("0", 1), ("1", 1), ("0", 4)])
def test_fft_callback_bitwise_equal_to_copy(H, AUTO, graphs, slabs):
    """The inverse transform reading ehat'/N through a cuFFT load callback
    (fft_cb.cu; AM_FFT_CALLBACK=1 forces it below 128^3) gives bitwise the
    fields and histories of the path where k_fourier writes the scaled copy:
    one slab eager and as graph replays, and the x-slab algorithm (each
    slab's inverse x transform, and the transposes riding on the 2-D
    transforms' store / load callbacks instead of k_pack_peer /
    k_unpack_peer), mixed BC."""
    import ctypes
    import os

    from paper_2006_04391_b200 import _lib

    out = []
    for cb in ("0", "1"):
        os.environ["AM_FFT_CALLBACK"] = cb
        os.environ["AM_NO_GRAPHS"] = "0" if graphs == "1" else "1"
        try:
            hom = H.Homogenizer(H.toy_mmc_grid(16), AUTO, slabs=slabs)
        finally:
            os.environ.pop("AM_FFT_CALLBACK", None)
            os.environ.pop("AM_NO_GRAPHS", None)
        on = ctypes.c_int(-1)
        _lib.check(hom._lib.am_solver_fft_callback(hom._h, ctypes.byref(on)))
        assert (on.value & 1) == int(cb), "the cuFFT load callback did not link in this process"
        if slabs > 1:  # bit 1: sigma's transposes on the 2-D transforms' callbacks
            assert (on.value >> 1) == int(cb)
        path = H.LoadingPath(steps=20)
        t = path.times()
        res = []
        for k in (1, 2, 3):
            eb = np.zeros(6)
            eb[0] = path.eps_xx(t[k])
            eps, sig, info = hom.solve_step(eb, t[k] - t[k - 1], free_mask=np.array([False] + [True] * 5))
            res.append((eps, sig, info.history))
            hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
        out.append(res)
    for (e0, s0, h0), (e1, s1, h1) in zip(*out):
        assert np.array_equal(e0, e1) and np.array_equal(s0, s1) and h0 == h1


def test_fft_callback_default_from_128(H, AUTO):
    """Power-of-two grids from 128^3 on take the callback path by default;
    other voxel counts never do (the origin's N ebar / N must be exact)."""
    import ctypes

    hom = H.Homogenizer(H.toy_mmc_grid(128), AUTO)
    on = ctypes.c_int(-1)
    hom._lib.am_solver_fft_callback(hom._h, ctypes.byref(on))
    assert on.value == 1
    small = H.Homogenizer(H.toy_mmc_grid(16), AUTO)
    small._lib.am_solver_fft_callback(small._h, ctypes.byref(on))
    assert on.value == 0
    import os

    os.environ["AM_FFT_CALLBACK"] = "1"
    try:
        odd = H.Homogenizer(H.toy_mmc_grid(12), AUTO)
    finally:
        os.environ.pop("AM_FFT_CALLBACK", None)
    odd._lib.am_solver_fft_callback(odd._h, ctypes.byref(on))
    assert on.value == 0
