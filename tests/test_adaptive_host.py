"""Adaptive ode12 / ode23 (csrc/adaptive.cuh) compiled for the host vs the
reference's own results (tests/golden/adaptive.npz, made by gsmkit's
adaptive_integrate through evaluate_arrays).  Same bars as the GPU tests:
identical accepted / rejected substep counts, state and stress within
1e-10, tangent within 1e-8."""

import numpy as np
import pytest

import _hostcheck as HC
from conftest import golden
from oracle import material as OM
from _util import TOL_STATE, TOL_TANGENT, assert_close


@pytest.mark.parametrize("integ", ["ode12", "ode23"])
@pytest.mark.parametrize("meas", ["internal", "stress"])
@pytest.mark.parametrize("tang", [False, True])
def test_adaptive_vs_reference(integ, meas, tang):
    g = golden("adaptive.npz")
    tag = f"{integ}_{meas}_{'t' if tang else 'n'}"
    r = HC.adaptive(OM.ALUMINUM, 23 if integ == "ode23" else 12, tang, meas, g["eps_n"], g["a_n"], g["eps_np1"],
                    g["dt"])
    assert r["code"] == 0
    assert np.array_equal(r["substeps"], g[tag + "_substeps"])
    assert np.array_equal(r["rejected"], g[tag + "_rejected"])
    assert_close(r["sigma"], g[tag + "_sigma"], TOL_STATE, "sigma")
    assert_close(r["a"], g[tag + "_a"], TOL_STATE, "a")
    if tang:
        assert_close(r["C"], g[tag + "_C"], TOL_TANGENT, "C")


def test_substep_cap_raises():
    g = golden("adaptive.npz")
    assert str(g["cap_err"]) == "IntegrationError"
    r = HC.adaptive(OM.ALUMINUM, 23, True, "internal", np.zeros((4, 6)), np.zeros((4, 7)), g["cap_eps_np1"], 1.0,
                    max_substeps=3)
    assert r["code"] & 8
