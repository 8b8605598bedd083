"""Adaptive ode12 / ode23 on the GPU (k_adaptive through evaluate_arrays) vs
the reference's results (tests/golden/adaptive.npz): identical accepted and
rejected substep counts, sigma / a within 1e-10, C within 1e-8."""

import numpy as np
import pytest

from conftest import golden
from _util import TOL_STATE, TOL_TANGENT, assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2006_04391_b200 import gsm
    from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays

    return gsm, StrategyConfig, evaluate_arrays


@pytest.mark.parametrize("integ", ["ode12", "ode23"])
@pytest.mark.parametrize("meas", ["internal", "stress"])
@pytest.mark.parametrize("tang", [False, True])
def test_adaptive_vs_reference(api, integ, meas, tang):
    gsm, SC, ev = api
    g = golden("adaptive.npz")
    tag = f"{integ}_{meas}_{'t' if tang else 'n'}"
    cfg = SC(strategy="automatic", integrator=integ, error_measure=meas)
    r = ev(gsm.MichelSuquet(), cfg, g["eps_n"], g["a_n"], g["eps_np1"], g["dt"], want_tangent=tang)
    assert np.array_equal(r.substeps, g[tag + "_substeps"])
    assert np.array_equal(r.rejected, g[tag + "_rejected"])
    assert_close(r.sigma, g[tag + "_sigma"], TOL_STATE, "sigma")
    assert_close(r.a, g[tag + "_a"], TOL_STATE, "a")
    if tang:
        assert_close(r.C, g[tag + "_C"], TOL_TANGENT, "C")


def test_default_config_is_ode23(api):
    gsm, SC, ev = api
    g = golden("adaptive.npz")
    r = ev(gsm.MichelSuquet(), SC(), g["eps_n"], g["a_n"], g["eps_np1"], g["dt"], want_tangent=True)
    assert np.array_equal(r.substeps, g["ode23_internal_t_substeps"])


def test_integration_error(api):
    gsm, SC, ev = api
    from paper_2006_04391_b200.odeint import IntegrationError

    g = golden("adaptive.npz")
    cfg = SC(strategy="automatic", integrator="ode23", max_substeps=3)
    with pytest.raises(IntegrationError):
        ev(gsm.MichelSuquet(), cfg, np.zeros((4, 6)), np.zeros((4, 7)), g["cap_eps_np1"], 1.0, want_tangent=True)


def test_record_steps(api):
    """EvalResult.steps of the adaptive integrator: every attempt's step size
    (to round-off) and acceptance (exactly), frozen points [(0.0, True)]."""
    gsm, SC, ev = api
    g = golden("adaptive.npz")
    cfg = SC(integrator="ode23", record_steps=True)
    r = ev(gsm.MichelSuquet(), cfg, g["eps_n"][120:152], g["a_n"][120:152], g["eps_np1"][120:152], g["dt"][120:152],
           want_tangent=True)
    flat = [(b, h, acc) for b, lst in enumerate(r.steps) for (h, acc) in lst]
    assert [f[0] for f in flat] == g["rec_b"].tolist()
    assert [f[2] for f in flat] == g["rec_acc"].tolist()
    np.testing.assert_allclose([f[1] for f in flat], g["rec_h"], rtol=1e-10, atol=0)


def test_basic_scheme_with_ode23(api):
    """The basic scheme with the default StrategyConfig() (ode23) on the 8^3
    toy grid: load step 1 as the reference (iterations, mean substeps,
    history, mean stress); load step 2 stagnates near 5e-4 and raises
    SolverError, as in the reference."""
    gsm, SC, _ = api
    from paper_2006_04391_b200 import homogenize as H

    g = golden("adaptive.npz")
    hom = H.Homogenizer(H.toy_mmc_grid(8), SC(), max_iterations=400)
    path = H.LoadingPath(steps=20)
    t, ex = path.times(), path.eps_xx(path.times())
    free = np.array([False] + [True] * 5)
    eb = np.zeros(6)
    eb[0] = ex[1]
    eps, sig, info = hom.solve_step(eb, t[1] - t[0], free_mask=free)
    assert info.iterations == int(g["path8_ode23_iters"])
    assert info.mean_substeps == float(g["path8_ode23_mean_substeps"])
    assert np.max(np.abs(np.array(info.history) / g["path8_ode23_history"] - 1)) < 1e-6
    assert_close(sig.mean(axis=(1, 2, 3)), g["path8_ode23_sig_bar"], 1e-8)
    hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
    eb[0] = ex[2]
    assert str(g["path8_ode23_step2_err"]) == "SolverError"
    with pytest.raises(H.SolverError):
        hom.solve_step(eb, t[2] - t[1], free_mask=free)
