"""The numpy basic-scheme oracle (oracle/homogenize.py) against the reference's fixtures.

tests/golden/{fourier,config1,path8_auto}.npz were produced by
tests/golden/make_golden.py running gsmkit itself; these tests pin the
oracle before the GPU tests use it as the checker.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import homogenize as OH
from oracle import material as OM

LE_MATRIX = OM.law_params(0, 55e9, 0.33)
LE_FIBER = OM.law_params(0, 300e9, 0.25)


def test_fourier_operators():
    g = golden("fourier.npz")
    lam, mu = g["ref"]
    for k in range(int(g["ndims"])):
        t = f"d{k}_"
        np.testing.assert_allclose(OH.green_apply(g[t + "tau"], lam, mu), g[t + "green"], rtol=0, atol=1e-15 *
                                   np.abs(g[t + "green"]).max())
        assert abs(OH.residual(g[t + "sig"]) / float(g[t + "residual"]) - 1.0) < 1e-13
        np.testing.assert_array_equal(OH.iso(lam, mu, g[t + "eps"]), g[t + "iso"])
    for k in range(3):
        lm = OH.reference_update(g[f"ru{k}_C"])
        np.testing.assert_allclose(lm, g[f"ru{k}_lam_mu"], rtol=1e-14)


@pytest.mark.parametrize("tag", ["strain", "mixed"])
def test_config1(tag):
    g = golden("config1.npz")
    b = OH.Basic(g["ids"], [LE_MATRIX, LE_FIBER])
    np.testing.assert_allclose([b.lam, b.mu], g[f"{tag}_ref"], rtol=1e-15)
    eb = np.zeros(6)
    eb[0] = 1e-3
    free = np.zeros(6, bool) if tag == "strain" else np.array([False] + [True] * 5)
    eps, sig, it, hist = b.solve_step(eb, 1.0, free)
    assert it == int(g[f"{tag}_iters"])
    np.testing.assert_allclose(hist, g[f"{tag}_history"], rtol=1e-12)
    sub = g["sub"]
    np.testing.assert_allclose(sig.reshape(6, -1)[:, sub], g[f"{tag}_sig_sub"], rtol=0,
                               atol=1e-13 * np.abs(g[f"{tag}_sig_sub"]).max())
    np.testing.assert_allclose(eps.reshape(6, -1)[:, sub], g[f"{tag}_eps_sub"], rtol=0,
                               atol=1e-13 * np.abs(g[f"{tag}_eps_sub"]).max())


def test_config1_iteration_cap():
    g = golden("config1.npz")
    b = OH.Basic(g["ids"], [LE_MATRIX, LE_FIBER], max_iterations=4)
    eb = np.zeros(6)
    eb[0] = 1e-3
    with pytest.raises(OH.NotConverged) as ei:
        b.solve_step(eb, 1.0)
    np.testing.assert_allclose(ei.value.history, g["cap_history"], rtol=1e-12)


def test_path8_first_steps():
    """8^3 fibre composite, automatic route, 6 of 20 steps: counts exact."""
    g = golden("path8_auto.npz")
    recs, b = OH.loading_path(g["ids"], [OM.ALUMINUM, LE_FIBER], 20, n_steps=6)
    assert [r["iterations"] for r in recs] == g["iterations"].tolist()
    for k, r in enumerate(recs):
        np.testing.assert_allclose(r["sig"], g["sig"][k], rtol=0, atol=1e-12 * np.abs(g["sig"][k]).max())
        assert abs(r["C11"] / g["C11"][k] - 1) < 1e-13 and abs(r["C12"] / g["C12"][k] - 1) < 1e-13
        np.testing.assert_allclose([r["lam"], r["mu"]], g["refs"][k + 1], rtol=1e-13)
    np.testing.assert_allclose(b.eps_n, g["eps_n"], rtol=0, atol=1e-12 * np.abs(g["eps_n"]).max())
    np.testing.assert_allclose(b.state[0], g["state0"], rtol=0, atol=1e-12 * np.abs(g["state0"]).max())


def test_green_apply_slabwise_matches_table():
    """The slab-wise Green application (512^3 checks) is the table version."""
    rng = np.random.default_rng(5)
    for dims in [(16, 12, 10), (9, 8, 7), (8, 6, 5)]:
        tau = rng.normal(0, 1e8, (6,) + dims)
        a = OH.green_apply(tau, 8e10, 7e10)
        b = OH.green_apply_slabwise(tau, 8e10, 7e10, kx_chunk=3)
        assert np.max(np.abs(a - b)) <= 1e-14 * np.max(np.abs(a))
