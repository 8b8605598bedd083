"""Single-GPU basic scheme with the x transforms fused into the Fourier
update (csrc/xfused.cuh; nx = 256, opt-in with AM_XFUSED=1): parity with the
numpy oracle and with the default 3-D cuFFT path."""

import os

import numpy as np
import pytest

from oracle import homogenize as OH
from oracle import material as OM

pytestmark = pytest.mark.gpu

TOL = 1e-10


def rel(x, y):
    x, y = np.asarray(x, dtype=float), np.asarray(y, dtype=float)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300))


@pytest.fixture(scope="module")
def H():
    from paper_2006_04391_b200 import _lib, homogenize

    _lib.load()
    return homogenize


@pytest.fixture(scope="module")
def AUTO():
    from paper_2006_04391_b200.evaluator import StrategyConfig

    return StrategyConfig(strategy="automatic", integrator="implicit-euler")


def _grid(H, shape, seed, frac=0.25):
    from paper_2006_04391_b200 import gsm

    ids = (np.random.default_rng(seed).random(shape) < frac).astype(np.uint8)
    return ids, H.VoxelGrid(ids, [gsm.MichelSuquet(), gsm.LinearElastic(300e9, 0.25)])


def _fused(H, grid, cfg, on):
    os.environ["AM_XFUSED"] = "1" if on else "0"
    try:
        return H.Homogenizer(grid, cfg)
    finally:
        os.environ.pop("AM_XFUSED", None)


def test_xfused_vs_oracle(H, AUTO):
    """256 x 4 x 6 two-phase EVP grid, two mixed-BC loading steps with reference updates."""
    ids, grid = _grid(H, (256, 4, 6), 7)
    hom = _fused(H, grid, AUTO, True)
    ob = OH.Basic(ids, [OM.ALUMINUM, OM.law_params(0, 300e9, 0.25)])
    t, ex = OH.loading_times(20)
    free = np.array([False, True, True, True, True, True])
    for k in (1, 2):
        dt = t[k] - t[k - 1]
        eb = np.zeros(6)
        eb[0] = ex[k]
        eps, sig, info = hom.solve_step(eb, dt, free_mask=free)
        oe, osig, oit, ohist = ob.solve_step(eb, dt, free)
        assert info.iterations == oit
        assert rel(info.history, ohist) < 1e-8
        assert rel(sig, osig) < TOL and rel(eps, oe) < TOL
        _, C, _, _ = hom.evaluate_field(eps, dt, want_tangent=True)
        _, oC, _ = ob.evaluate(oe, dt, True)
        hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
        ob.commit(oe, oe.mean(axis=(1, 2, 3)))
        hom.set_reference(H.reference_update(C))
        ob.lam, ob.mu = OH.reference_update(oC)
    assert rel(grid.state[0], ob.state[0]) < TOL


@pytest.mark.parametrize("shape,bc", [((256, 16, 12), "mixed"), ((256, 8, 9), "strain")])
def test_xfused_vs_3d_cufft(H, AUTO, shape, bc):
    """Same loading steps through the fused path and the 3-D cuFFT path:
    identical iteration counts, fields equal to round-off (odd nz included)."""
    out = []
    for on in (True, False):
        _, grid = _grid(H, shape, 11)
        hom = _fused(H, grid, AUTO, on)
        path = H.LoadingPath(steps=20)
        t = path.times()
        free = np.array([False] + [True] * 5) if bc == "mixed" else None
        res = []
        for k in (1, 2, 3):
            eb = np.zeros(6)
            eb[0] = path.eps_xx(t[k])
            if bc == "strain":
                eb[1] = -0.3 * eb[0]
                eb[5] = 0.2 * eb[0]
            eps, sig, info = hom.solve_step(eb, t[k] - t[k - 1], free_mask=free)
            res.append((info.iterations, np.array(info.history), eps, sig))
            hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
        out.append(res)
    for (i0, h0, e0, s0), (i1, h1, e1, s1) in zip(*out):
        assert i0 == i1
        assert rel(h0, h1) < 1e-10
        assert rel(e0, e1) < 1e-12 and rel(s0, s1) < 1e-12
