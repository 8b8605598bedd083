"""Semi-automatic strategy (csrc/semi.cuh, hand partials of gsm.py:258-328
and the nested Jacobians of gsm.py:463-481) compiled for the host vs the
reference's semi-automatic results (tests/golden/material_semi.npz)."""

import numpy as np
import pytest

import _hostcheck as HC
from conftest import golden
from oracle import material as OM
from _util import TOL_STATE, TOL_TANGENT, assert_close


@pytest.mark.parametrize("tang", [False, True])
def test_semi_implicit_euler(tang):
    g = golden("material_semi.npz")
    tag = f"ie_{'t' if tang else 'n'}"
    r = HC.evaluate(OM.ALUMINUM, g["eps_n"], g["a_n"], g["eps_np1"], g["dt"], tang, semi=True)
    assert r["code"] == 0
    assert np.array_equal(r["iters"], g[tag + "_iters"])
    assert_close(r["sigma"], g[tag + "_sigma"], TOL_STATE, "sigma")
    assert_close(r["a"], g[tag + "_a"], TOL_STATE, "a")
    if tang:
        assert_close(r["C"], g[tag + "_C"], TOL_TANGENT, "C")


SCHEME = {"ode12": 12, "ode23": 23, "ode23s": 32, "ode23s_stress": 32}


@pytest.mark.parametrize("integ", ["ode12", "ode23", "ode23s", "ode23s_stress"])
@pytest.mark.parametrize("tang", [False, True])
def test_semi_adaptive(integ, tang):
    g = golden("material_semi.npz")
    tag = f"{integ}_{'t' if tang else 'n'}"
    meas = "stress" if integ.endswith("stress") else "internal"
    r = HC.adaptive(OM.ALUMINUM, SCHEME[integ], tang, meas, g["eps_n"], g["a_n"], g["eps_np1"], g["dt"], semi=True)
    assert r["code"] == 0
    assert np.array_equal(r["substeps"], g[tag + "_substeps"])
    assert np.array_equal(r["rejected"], g[tag + "_rejected"])
    assert_close(r["sigma"], g[tag + "_sigma"], TOL_STATE, "sigma")
    assert_close(r["a"], g[tag + "_a"], TOL_STATE, "a")
    if tang:
        assert_close(r["C"], g[tag + "_C"], TOL_TANGENT, "C")


def test_semi_linear_elastic():
    g = golden("material_semi.npz")
    r = HC.evaluate(OM.law_params(0, 300e9, 0.25), g["eps_n"], None, g["eps_np1"], g["dt"], True, semi=True)
    assert_close(r["sigma"], g["le_sigma"], 1e-15)
    assert_close(r["C"], g["le_C"], 1e-15)


@pytest.mark.parametrize("tang", [False, True])
def test_conventional(tang):
    g = golden("material_semi.npz")
    tag = f"conv_{'t' if tang else 'n'}"
    r = HC.conventional(OM.ALUMINUM, g["eps_np1"], g["a_n"], g["dt"], tang)
    assert r["code"] == 0
    assert_close(r["sigma"], g[tag + "_sigma"], TOL_STATE, "sigma")
    assert_close(r["a"], g[tag + "_a"], TOL_STATE, "a")
    if tang:
        assert_close(r["C"], g[tag + "_C"], TOL_TANGENT, "C")
