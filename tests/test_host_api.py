"""Host-side parts of the drop-in API that need no GPU: geometry generation,
loading path, geometry I/O, config validation, parameter files."""

import numpy as np
import pytest

from conftest import golden


def test_toy_mmc_grid_matches_reference_ids():
    from paper_2006_04391_b200 import homogenize as H

    assert np.array_equal(H.toy_mmc_grid(8).material_ids, golden("path8_auto.npz")["ids"])
    assert np.array_equal(H.toy_mmc_grid(16).material_ids, golden("path16_conv.npz")["ids"])


def test_sphere_ids_match_config1():
    from paper_2006_04391_b200.workloads import sphere_ids

    assert np.array_equal(sphere_ids(32), golden("config1.npz")["ids"])


def test_loading_path_times_match_reference():
    from paper_2006_04391_b200 import homogenize as H

    g = golden("path16_conv.npz")
    path = H.LoadingPath(steps=20)
    t = path.times()
    np.testing.assert_array_equal(t[1:], g["time"])
    assert abs(path.total_time - 7.609635714285714) < 1e-12  # (2 eps_max - eps_min) / rate
    assert path.eps_xx(t)[-1] == pytest.approx(-3.48441e-3)


def test_voxel_grid_validation():
    from paper_2006_04391_b200 import gsm, homogenize as H

    with pytest.raises(ValueError):
        H.VoxelGrid(np.zeros((4, 4)), [gsm.LinearElastic(1e9, 0.3)])
    with pytest.raises(ValueError):
        H.VoxelGrid(np.full((2, 2, 2), 3), [gsm.LinearElastic(1e9, 0.3)])
    g = H.VoxelGrid(np.zeros((2, 3, 4), dtype=np.uint8), [gsm.MichelSuquet(), gsm.LinearElastic(1e9, 0.3)])
    assert g.n_voxels == 24 and [len(i) for i in g.voxel_index] == [24, 0]
    assert g.state[0].shape == (24, 7) and g.state[1].shape == (0, 0)


def test_geometry_roundtrip(tmp_path):
    from paper_2006_04391_b200 import homogenize as H

    ids = H.toy_mmc_grid(8).material_ids
    H.save_geometry(tmp_path / "g.raw", ids, ["matrix", "fiber"])
    back, names = H.load_geometry(tmp_path / "g.raw")
    assert np.array_equal(back, ids) and names == ["matrix", "fiber"]
    big = np.full((2, 2, 2), 300)
    H.save_geometry(tmp_path / "h.raw", big, ["x"] * 301)
    assert H.load_geometry(tmp_path / "h.raw")[0].dtype == np.dtype("<u2")


def test_strategy_config_validation():
    from paper_2006_04391_b200.evaluator import ConfigError, StrategyConfig

    assert StrategyConfig().integrator == "ode23"
    assert StrategyConfig(error_measure="stress").resolved_newton_mode == "stress"
    for bad in (dict(error_measure="x"), dict(newton_mode="y"), dict(integrator="rk4"),
                dict(strategy="semi-automatic", integrator="ode23s", newton_mode="bad")):
        with pytest.raises(ConfigError):
            StrategyConfig(**bad)


def test_michel_suquet_params_file(tmp_path):
    from paper_2006_04391_b200 import gsm

    p = tmp_path / "al.txt"
    p.write_text("# aluminium\nE = 55e9\nnu = 0.33\nsigma_Y = 25e6\nH = 1.8e9\neps0_dot = 1\nsigma_d = 130e6\nn = 3.6\n")
    assert gsm.load_michel_suquet_params(p) == gsm.ALUMINUM_MATRIX
    p.write_text("E = 1\nbogus = 2\n")
    with pytest.raises(ValueError):
        gsm.load_michel_suquet_params(p)
    with pytest.raises(ValueError):
        gsm.MichelSuquetParams(E=1, nu=0.6, sigma_Y=1, H=1, eps0_dot=1, sigma_d=1, n=1)


def test_reference_material_matrix():
    from oracle import homogenize as OH
    from paper_2006_04391_b200 import homogenize as H

    np.testing.assert_array_equal(H.ReferenceMaterial(3.0, 2.0).matrix(), OH.iso_matrix(3.0, 2.0))


def test_lawops_strategy_validation():
    """LawOps / module functions reject strategies like gsm.py:420-427 before touching the device."""
    from paper_2006_04391_b200 import gsm

    law = gsm.MichelSuquet()
    with pytest.raises(ValueError):
        gsm.LawOps(law, "numeric")
    with pytest.raises(ValueError):
        gsm.LawOps(law, "conventional")  # the class takes automatic / semi-automatic only

    class NoHand(gsm.GsmDefinition):
        m = 0

    with pytest.raises(ValueError):
        gsm.LawOps(NoHand(), "semi-automatic")
    with pytest.raises(ValueError):
        gsm.stress(NoHand(), np.zeros(6), np.zeros(0), strategy="conventional")  # conventional -> semi
    with pytest.raises(ValueError):
        gsm.evolution_rhs(law, np.zeros(6), np.zeros(7), strategy="numeric")
    with pytest.raises(ValueError):
        gsm.conventional_evaluate(gsm.LinearElastic(1e9, 0.3), np.zeros(6), np.zeros(0), np.zeros(6), 0.1)


def test_law_subclass_has_no_device_potentials():
    """A subclass may override the potentials: it must not run on the built-in
    device laws (ConfigError, no CPU fallback)."""
    from paper_2006_04391_b200 import _lib, gsm
    from paper_2006_04391_b200.evaluator import ConfigError

    class Stiffer(gsm.LinearElastic):
        def omega(self, eps, a):  # pragma: no cover - never evaluated
            return 2.0 * super().omega(eps, a)

    assert _lib.make_law(gsm.LinearElastic(1e9, 0.3)).kind == _lib.AM_LAW_LINEAR_ELASTIC
    assert _lib.make_law(gsm.MichelSuquet()).kind == _lib.AM_LAW_MICHEL_SUQUET
    with pytest.raises(ConfigError):
        _lib.make_law(Stiffer(1e9, 0.3))


def test_loading_path_fixtures_are_consistent():
    """The n^3 path fixtures (reference, per-law conventional route) share the
    loading times and geometry generator with this package."""
    import os

    from conftest import GOLDEN
    from paper_2006_04391_b200 import homogenize as H

    t = H.LoadingPath(steps=20).times()
    for n in (16, 32, 64, 128):
        f = os.path.join(GOLDEN, f"path{n}_conv.npz")
        if not os.path.exists(f):
            continue
        g = np.load(f)
        k = len(g["iterations"])
        np.testing.assert_array_equal(t[1:k + 1], g["time"])
        assert np.array_equal(H.toy_mmc_grid(n).material_ids, g["ids"])


def test_python_potentials_match_device_formulas():
    """The Python potentials (gsm.py:100-256, written over generic scalars
    like the reference's) are the formulas the device compiles: complex-step
    derivatives of omega give the oracle's sigma and A = -domega/da, a
    4th-order difference of psi gives the oracle's f = dpsi/dA."""
    from oracle import material as OM
    from paper_2006_04391_b200 import gsm

    rng = np.random.default_rng(3)
    law = gsm.MichelSuquet()
    h = 1e-30
    for _ in range(12):
        eps = rng.normal(0, 2e-3, 6)
        a = np.concatenate([rng.normal(0, 5e-4, 6), [abs(rng.normal(0, 1e-3))]])
        sig, A, f, _, _ = OM.constitutive(OM.ALUMINUM, eps, a)
        d_eps = [law.omega([complex(x) + (1j * h if i == k else 0) for i, x in enumerate(eps)], list(a)).imag / h
                 for k in range(6)]
        d_a = [law.omega(list(eps), [complex(x) + (1j * h if i == k else 0) for i, x in enumerate(a)]).imag / h
               for k in range(7)]
        assert np.max(np.abs(np.array(d_eps) - sig)) <= 1e-13 * np.max(np.abs(sig))
        assert np.max(np.abs(-np.array(d_a) - A)) <= 1e-13 * np.max(np.abs(A))
        if law.psi(list(A)) <= 0.0:
            continue  # elastic: f = 0
        g = []
        for k in range(7):
            dk = 1e-4 * max(abs(A[k]), 1e5)

            def ps(t, k=k):
                x = list(A)
                x[k] = A[k] + t
                return law.psi(x)

            g.append((8 * (ps(dk) - ps(-dk)) - (ps(2 * dk) - ps(-2 * dk))) / (12 * dk))
        assert np.max(np.abs(np.array(g) - f)) <= 1e-7 * np.max(np.abs(f))
    le = gsm.LinearElastic(300e9, 0.25)
    eps = rng.normal(0, 1e-3, 6)
    d = [le.omega([complex(x) + (1j * h if i == k else 0) for i, x in enumerate(eps)], []).imag / h for k in range(6)]
    assert np.max(np.abs(np.array(d) - le.Ce @ eps)) <= 1e-13 * np.max(np.abs(le.Ce @ eps))
    assert np.max(np.abs(gsm.DEV6 @ np.arange(6.0) - np.array(gsm.dev_components(list(np.arange(6.0)))))) <= 1e-15
