"""GPU parity of gsm.LawOps (gsm.py:412-566) under both strategies, the
module-level strategy switch (gsm.py:574-602, conventional -> semi) and
conventional_evaluate (gsm.py:605-609), against fixtures made by running the
reference (tests/golden/make_golden.py, job "lawops")."""

import numpy as np
import pytest

from conftest import golden
from _util import TOL_STATE, TOL_TANGENT, assert_close, rowwise_relerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gsm():
    from paper_2006_04391_b200 import _lib, gsm

    _lib.load()
    return gsm


@pytest.mark.parametrize("tag,strategy", [("auto", "automatic"), ("semi", "semi-automatic")])
def test_lawops_golden(gsm, tag, strategy):
    g = golden("lawops.npz")
    ops = gsm.LawOps(gsm.MichelSuquet(), strategy)
    eps, a, da = g["eps"], g["a"], g["da"]
    assert_close(ops.stress(eps, a), g[tag + "_stress"], 1e-14, "stress")
    # the reference only evaluates gen_stress point by point; the device batches it
    assert_close(ops.gen_stress(eps, a), g[tag + "_gen_stress"], 1e-14, "gen_stress")
    f, J, Je = ops.rhs_and_jacobians(eps, a)
    assert_close(f, g[tag + "_rhs"], 1e-12, "rhs")
    assert_close(J, g[tag + "_dfda"], 1e-12, "dfda")
    assert_close(Je, g[tag + "_dfde"], 1e-12, "dfde")
    sig, C = ops.stress_and_tangent(eps, a, da)
    assert_close(sig, g[tag + "_st_sigma"], 1e-14, "sigma")
    assert rowwise_relerr(C, g[tag + "_st_C"]).max() <= TOL_TANGENT
    assert_close(ops.elastic_tangent(eps, a), g[tag + "_elastic_C"], 1e-14, "elastic C")
    le = gsm.LawOps(gsm.LinearElastic(300e9, 0.25), strategy)
    z = np.zeros((len(eps), 0))
    assert_close(le.stress(eps, z), g["le_" + tag + "_stress"], 1e-14)
    assert_close(le.stress_and_tangent(eps, z, np.zeros((len(eps), 0, 6)))[1], g["le_" + tag + "_C"], 1e-14)


def test_lawops_batch_shapes(gsm):
    """Arbitrary leading batch axes (gsm.py:412-418), single points included."""
    g = golden("lawops.npz")
    ops = gsm.LawOps(gsm.MichelSuquet(), "automatic")
    eps = g["eps"][:24].reshape(2, 3, 4, 6)
    a = g["a"][:24].reshape(2, 3, 4, 7)
    f, J, Je = ops.rhs_and_jacobians(eps, a)
    assert f.shape == (2, 3, 4, 7) and J.shape == (2, 3, 4, 7, 7) and Je.shape == (2, 3, 4, 7, 6)
    assert np.array_equal(J.reshape(24, 7, 7), ops.rhs_and_jacobians(g["eps"][:24], g["a"][:24])[1])
    s1 = ops.stress(g["eps"][10], g["a"][10])
    assert s1.shape == (6,) and np.array_equal(s1, ops.stress(g["eps"], g["a"])[10])


def test_module_strategy_switch(gsm):
    g = golden("lawops.npz")
    law = gsm.MichelSuquet()
    for strat in ("semi-automatic", "conventional"):
        assert_close(gsm.evolution_rhs(law, g["eps"], g["a"], strategy=strat), g["semi_rhs"], 1e-12)
        assert_close(gsm.rhs_jacobian(law, g["eps"], g["a"], strategy=strat), g["semi_dfda"], 1e-12)
    with pytest.raises(ValueError):
        gsm.stress(law, g["eps"], g["a"], strategy="numeric")

    class NoHand(gsm.GsmDefinition):
        m = 0

    with pytest.raises(ValueError):
        gsm.LawOps(NoHand(), "semi-automatic")


def test_conventional_evaluate(gsm):
    g = golden("lawops.npz")
    law = gsm.MichelSuquet()
    sig, a_new, C = gsm.conventional_evaluate(law, g["eps"], g["a"], g["conv_eps_np1"], g["conv_h"],
                                              want_tangent=True)
    assert rowwise_relerr(sig, g["conv_sigma"]).max() <= TOL_STATE
    assert rowwise_relerr(a_new, g["conv_a"]).max() <= TOL_STATE
    assert rowwise_relerr(C, g["conv_C"]).max() <= TOL_TANGENT
    s1, a1, C1 = gsm.conventional_evaluate(law, g["eps"][5], g["a"][5], g["conv_eps_np1"][5], 0.05)
    assert s1.shape == (6,) and a1.shape == (7,) and C1 is None
    with pytest.raises(ValueError):
        gsm.conventional_evaluate(gsm.LinearElastic(1e9, 0.3), g["eps"], np.zeros((128, 0)), g["eps"], 0.1)
