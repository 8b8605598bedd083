"""Semi-automatic strategy on the GPU vs the reference's semi-automatic
results (tests/golden/material_semi.npz), and the basic scheme with it
(identical 16^3 path iteration counts)."""

import numpy as np
import pytest

from conftest import golden
from _util import TOL_STATE, TOL_TANGENT, assert_close, check_path_records

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2006_04391_b200 import gsm
    from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays

    return gsm, StrategyConfig, evaluate_arrays


@pytest.mark.parametrize("tang", [False, True])
def test_semi_implicit_euler(api, tang):
    gsm, SC, ev = api
    g = golden("material_semi.npz")
    tag = f"ie_{'t' if tang else 'n'}"
    cfg = SC(strategy="semi-automatic", integrator="implicit-euler")
    r = ev(gsm.MichelSuquet(), cfg, g["eps_n"], g["a_n"], g["eps_np1"], g["dt"], want_tangent=tang)
    assert np.array_equal(r.newton_iters, g[tag + "_iters"])
    assert_close(r.sigma, g[tag + "_sigma"], TOL_STATE, "sigma")
    assert_close(r.a, g[tag + "_a"], TOL_STATE, "a")
    if tang:
        assert_close(r.C, g[tag + "_C"], TOL_TANGENT, "C")


@pytest.mark.parametrize("integ", ["ode12", "ode23", "ode23s", "ode23s_stress"])
@pytest.mark.parametrize("tang", [False, True])
def test_semi_adaptive(api, integ, tang):
    gsm, SC, ev = api
    g = golden("material_semi.npz")
    tag = f"{integ}_{'t' if tang else 'n'}"
    meas = "stress" if integ.endswith("stress") else "internal"
    cfg = SC(strategy="semi-automatic", integrator=integ.replace("_stress", ""), error_measure=meas)
    r = ev(gsm.MichelSuquet(), cfg, g["eps_n"], g["a_n"], g["eps_np1"], g["dt"], want_tangent=tang)
    assert np.array_equal(r.substeps, g[tag + "_substeps"])
    assert np.array_equal(r.rejected, g[tag + "_rejected"])
    assert_close(r.sigma, g[tag + "_sigma"], TOL_STATE, "sigma")
    assert_close(r.a, g[tag + "_a"], TOL_STATE, "a")
    if tang:
        assert_close(r.C, g[tag + "_C"], TOL_TANGENT, "C")


def test_semi_linear_elastic(api):
    gsm, SC, ev = api
    g = golden("material_semi.npz")
    cfg = SC(strategy="semi-automatic", integrator="implicit-euler")
    r = ev(gsm.LinearElastic(300e9, 0.25), cfg, g["eps_n"], np.zeros((256, 0)), g["eps_np1"], g["dt"], True)
    assert_close(r.sigma, g["le_sigma"], 1e-15)
    assert_close(r.C, g["le_C"], 1e-15)


def test_semi_path16(api):
    gsm, SC, _ = api
    from paper_2006_04391_b200 import homogenize as H

    g = golden("path16_conv.npz")
    cfg = SC(strategy="semi-automatic", integrator="implicit-euler")
    recs = H.run_loading_path(H.toy_mmc_grid(16), H.LoadingPath(steps=20), cfg)
    check_path_records(recs, g, "path16_semi")


@pytest.mark.parametrize("tang", [False, True])
def test_conventional(api, tang):
    """strategy='conventional': radial return kernel vs the reference."""
    gsm, SC, ev = api
    g = golden("material_semi.npz")
    tag = f"conv_{'t' if tang else 'n'}"
    cfg = SC(strategy="conventional", integrator="implicit-euler")
    r = ev(gsm.MichelSuquet(), cfg, g["eps_n"], g["a_n"], g["eps_np1"], g["dt"], want_tangent=tang)
    assert_close(r.sigma, g[tag + "_sigma"], TOL_STATE, "sigma")
    assert_close(r.a, g[tag + "_a"], TOL_STATE, "a")
    if tang:
        assert_close(r.C, g[tag + "_C"], TOL_TANGENT, "C")


def test_conventional_rejects_linear_elastic(api):
    gsm, SC, ev = api
    from paper_2006_04391_b200.evaluator import ConfigError

    cfg = SC(strategy="conventional", integrator="implicit-euler")
    with pytest.raises(ConfigError):
        ev(gsm.LinearElastic(1e9, 0.3), cfg, np.zeros((2, 6)), np.zeros((2, 0)), np.zeros((2, 6)), 0.1)


def test_radial_return_stall_raises_everywhere():
    """A stalled radial return (gsm.py:377-378) raises gsm.NewtonError from
    conventional_evaluate, evaluate_arrays(strategy="conventional") and the
    basic scheme's solve_step, like the reference (fixture radial_stall.npz);
    a smaller strain of the same law matches the reference."""
    from paper_2006_04391_b200 import gsm
    from paper_2006_04391_b200 import homogenize as H
    from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays

    g = golden("radial_stall.npz")
    for k in ("conventional_evaluate", "evaluate_arrays", "solve_step"):
        assert str(g[f"raised_{k}"]) == "NewtonError"
    law = gsm.MichelSuquet(gsm.MichelSuquetParams(*g["params"]))
    conv = StrategyConfig(strategy="conventional", integrator="implicit-euler")
    ep, dt = g["eps_np1"], float(g["dt"])
    z6, z7 = np.zeros((1, 6)), np.zeros((1, 7))
    with pytest.raises(gsm.NewtonError):
        gsm.conventional_evaluate(law, z6, z7, ep[None], dt)
    with pytest.raises(gsm.NewtonError):
        evaluate_arrays(law, conv, z6, z7, ep[None], dt)
    hom = H.Homogenizer(H.VoxelGrid(np.zeros((2, 2, 2), np.uint8), [law]), conv)
    with pytest.raises(gsm.NewtonError):
        hom.solve_step(ep, dt, free_mask=np.zeros(6, bool))
    sig, a, C = gsm.conventional_evaluate(law, z6, z7, g["ok_eps"][None], dt, want_tangent=True)
    assert_close(sig[0], g["ok_sigma"], TOL_STATE, "sigma")
    assert_close(a[0], g["ok_a"], TOL_STATE, "a")
    assert_close(C[0], g["ok_C"], TOL_TANGENT, "C")
