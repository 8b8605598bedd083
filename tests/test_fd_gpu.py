"""Device derivatives against central finite differences of the device's own
primal maps (SPEC.md acceptance criterion 1, and criterion 4 for the
step-size-free implicit Euler route), on 1000 random config-2 states:

* dF/da and dF/deps of the evolution right-hand side (gsm.LawOps,
  reverse-mode AD under both strategies) vs central differences of F,
  relative error < 1e-6;
* the consistent tangent of evaluate_arrays (implicit Euler, automatic,
  semi-automatic and conventional) vs central differences of
  sigma_{n+1}(eps_{n+1}), relative error < 1e-5 (the Newton's converged tolerance bounds the
  differences' noise).
The AD itself is pinned bitwise to the reference's (tests/test_oracle.py);
these check the derivatives mean what they claim on the device.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def batch():
    from paper_2006_04391_b200.workloads import config2_batch

    return config2_batch(1000, seed=11)


def _fd_relerr(fd, exact):
    """Per point: max |fd - exact| over the matrix / max |exact|."""
    num = np.abs(fd - exact).reshape(len(fd), -1).max(axis=1)
    return num / np.maximum(np.abs(exact).reshape(len(fd), -1).max(axis=1), 1e-300)


@pytest.mark.parametrize("strategy", ["automatic", "semi-automatic"])
def test_rhs_jacobians_vs_fd(batch, strategy):
    from paper_2006_04391_b200 import gsm

    eps_n, a_n, eps, _ = batch
    ops = gsm.LawOps(gsm.MichelSuquet(), strategy)
    _, J, Je = ops.rhs_and_jacobians(eps, a_n)
    for x, exact, which in ((a_n, J, "a"), (eps, Je, "eps")):
        cols = []
        for j in range(x.shape[1]):
            h = 1e-5 * np.maximum(np.abs(x).max(axis=1), 1e-6)
            xp, xm = x.copy(), x.copy()
            xp[:, j] += h
            xm[:, j] -= h
            fp = ops.rhs(eps, xp) if which == "a" else ops.rhs(xp, a_n)
            fm = ops.rhs(eps, xm) if which == "a" else ops.rhs(xm, a_n)
            cols.append((fp - fm) / (2.0 * h[:, None]))
        fd = np.stack(cols, axis=-1)
        err = _fd_relerr(fd, exact)
        assert np.median(err) < 1e-8 and err.max() < 1e-6, (which, float(err.max()))


@pytest.mark.parametrize("strategy", ["automatic", "semi-automatic", "conventional"])
def test_implicit_euler_tangent_vs_fd(batch, strategy):
    from paper_2006_04391_b200 import gsm
    from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays

    eps_n, a_n, eps, dt = batch
    law = gsm.MichelSuquet()
    cfg = StrategyConfig(strategy=strategy, integrator="implicit-euler")
    C = evaluate_arrays(law, cfg, eps_n, a_n, eps, dt, want_tangent=True).C
    h = 1e-6 * np.abs(eps).max(axis=1)
    cols = []
    for j in range(6):
        ep, em = eps.copy(), eps.copy()
        ep[:, j] += h
        em[:, j] -= h
        sp = evaluate_arrays(law, cfg, eps_n, a_n, ep, dt).sigma
        sm = evaluate_arrays(law, cfg, eps_n, a_n, em, dt).sigma
        cols.append((sp - sm) / (2.0 * h[:, None]))
    err = _fd_relerr(np.stack(cols, axis=-1), C)
    assert err.max() < 1e-5, float(err.max())
