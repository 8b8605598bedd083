"""The reference-side binding of INTEGRATION.md §3, run inside the pristine
reference: gsmkit (installed unmodified into baseline/_ref by
__graft_entry__.build()) gets the documented ctypes block exec'd into its
evaluator module and the documented two-line hook in evaluate_arrays; then
the reference's OWN Homogenizer / solve_step / evaluate_field / commit_step
run config 1, the first steps of the 8^3 path and its run_loading_path the
full 16^3 20-step path with every material evaluation on libautomat.so,
against the fixtures the unmodified reference produced (tests/golden)."""

import os
import re
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref")


def rel(x, y):
    x, y = np.asarray(x, float), np.asarray(y, float)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300))


@pytest.fixture(scope="module")
def gsmkit():
    if not os.path.isfile(os.path.join(REF, "gsmkit", "evaluator.py")):
        pytest.skip("baseline/_ref has no gsmkit (run __graft_entry__.build() where /root/reference exists)")
    sys.path.insert(0, REF)
    try:
        import gsmkit.evaluator as ev
        import gsmkit.gsm as gsm
        import gsmkit.homogenize as H
    finally:
        sys.path.remove(REF)
    assert os.path.dirname(ev.__file__).startswith(REF)
    md = open(os.path.join(ROOT, "INTEGRATION.md"), encoding="utf-8").read()
    block = re.search(r"<!-- gsmkit-binding:begin -->\s*```python\n(.*?)```\s*<!-- gsmkit-binding:end -->", md, re.S)
    assert block, "INTEGRATION.md §3 binding block not found"
    exec(compile(block.group(1), "INTEGRATION.md#3", "exec"), ev.__dict__)  # noqa: S102
    orig = ev.evaluate_arrays
    calls = {"gpu": 0, "cpu": 0}

    def evaluate_arrays(law, cfg, eps_n, a_n, eps_np1, dt, want_tangent=False, threads=1):
        ev._validate_for_law(law, cfg)
        if ev._gpu_route(law, cfg):  # the documented hook
            calls["gpu"] += 1
            return ev._evaluate_arrays_gpu(law, cfg, eps_n, a_n, eps_np1, dt, want_tangent)
        calls["cpu"] += 1
        return orig(law, cfg, eps_n, a_n, eps_np1, dt, want_tangent, threads)

    os.environ["AUTOMAT_LIB"] = os.path.join(ROOT, "paper_2006_04391_b200", "libautomat.so")
    ev.evaluate_arrays = H.evaluate_arrays = evaluate_arrays
    yield ev, gsm, H, calls
    ev.evaluate_arrays = H.evaluate_arrays = orig
    os.environ.pop("AUTOMAT_LIB", None)


def test_reference_homogenizer_config1_on_gpu(gsmkit):
    ev, gsm, H, calls = gsmkit
    g = golden("config1.npz")
    cfg = ev.StrategyConfig(strategy="automatic", integrator="implicit-euler")
    for tag, free in (("strain", np.zeros(6, bool)), ("mixed", np.array([False] + [True] * 5))):
        grid = H.VoxelGrid(g["ids"], [gsm.LinearElastic(55e9, 0.33), gsm.LinearElastic(300e9, 0.25)])
        hom = H.Homogenizer(grid, cfg)
        eb = np.zeros(6)
        eb[0] = 1e-3
        before = calls["gpu"]
        eps, sig, info = hom.solve_step(eb, 1.0, free_mask=free)
        assert calls["gpu"] - before == 2 * info.iterations  # two phases per iteration, all on the device
        assert info.iterations == int(g[f"{tag}_iters"])
        assert rel(info.history, g[f"{tag}_history"]) < 1e-8
        assert rel(sig.reshape(6, -1)[:, g["sub"]], g[f"{tag}_sig_sub"]) < 1e-10
        assert rel(eps.reshape(6, -1)[:, g["sub"]], g[f"{tag}_eps_sub"]) < 1e-10
    assert calls["cpu"] == 0


def test_reference_homogenizer_path8_on_gpu(gsmkit):
    """The reference's per-step loop (homogenize.py:485-528) at 8^3, 6 steps:
    EVP matrix + elastic fibre, tangent sweeps and reference updates."""
    ev, gsm, H, calls = gsmkit
    g = golden("path8_auto.npz")
    cfg = ev.StrategyConfig(strategy="automatic", integrator="implicit-euler")
    grid = H.toy_mmc_grid(8)
    assert np.array_equal(grid.material_ids, g["ids"])
    hom = H.Homogenizer(grid, cfg)
    path = H.LoadingPath(steps=20)
    times = path.times()
    targets = path.eps_xx(times)
    free = np.array([False, True, True, True, True, True])
    cpu0 = calls["cpu"]
    for k in range(1, 7):
        dt = times[k] - times[k - 1]
        eb = np.zeros(6)
        eb[0] = targets[k]
        eps, sigma, info = hom.solve_step(eb, dt, free_mask=free)
        assert info.iterations == g["iterations"][k - 1]
        assert rel(sigma.mean(axis=(1, 2, 3)), g["sig"][k - 1]) < 1e-10
        ebar = eps.mean(axis=(1, 2, 3))
        _, C_vox, _, _ = hom.evaluate_field(eps, dt, want_tangent=True)
        assert rel(C_vox.mean(axis=0), g["Cbar"][k - 1]) < 1e-8
        hom.commit_step(eps, ebar)
        hom.set_reference(H.reference_update(C_vox))
        assert rel([hom.reference.lam, hom.reference.mu], g["refs"][k]) < 1e-8
    assert rel(hom.eps_n, g["eps_n"]) < 1e-10
    assert rel(grid.state[0], g["state0"]) < 1e-10
    assert calls["cpu"] == cpu0


def test_reference_run_loading_path16_on_gpu(gsmkit):
    """The reference's own run_loading_path (homogenize.py:485-528) at 16^3,
    20 steps, every material evaluation (iterations and tangent sweeps) on
    libautomat through the binding: the reference fixture's iteration counts
    and records (path16_conv.npz)."""
    ev, gsm, H, calls = gsmkit
    g = golden("path16_conv.npz")
    cfg = ev.StrategyConfig(strategy="automatic", integrator="implicit-euler")
    cpu0, gpu0 = calls["cpu"], calls["gpu"]
    recs = H.run_loading_path(H.toy_mmc_grid(16), H.LoadingPath(steps=20), cfg)
    assert calls["cpu"] == cpu0 and calls["gpu"] - gpu0 >= 2 * int(g["iterations"].sum())
    assert [r["iterations"] for r in recs] == g["iterations"].tolist()
    sig = np.stack([r["sig"] for r in recs])
    assert float(np.max(np.abs(sig - g["sig"]).max(axis=1) / np.abs(g["sig"]).max(axis=1))) <= 1e-10
    assert rel([r["C11"] for r in recs], g["C11"]) <= 1e-8
    assert rel([r["eps_xx"] for r in recs], g["eps_xx"]) <= 1e-10


def test_reference_evaluate_arrays_every_route_on_gpu(gsmkit):
    """Through the binding, every strategy x integrator the reference accepts
    runs on libautomat and matches the reference's own CPU route (the
    original evaluate_arrays on the same inputs)."""
    ev, gsm, H, calls = gsmkit
    from paper_2006_04391_b200.workloads import config2_batch

    en, an, ep, dt = config2_batch(64, seed=4)
    law = gsm.MichelSuquet()
    for strat, integ in (("automatic", "implicit-euler"), ("semi-automatic", "implicit-euler"),
                         ("conventional", "implicit-euler"), ("automatic", "ode23"), ("semi-automatic", "ode23s")):
        cfg = ev.StrategyConfig(strategy=strat, integrator=integ)
        g0 = calls["gpu"]
        r = ev.evaluate_arrays(law, cfg, en, an, ep, dt, want_tangent=True)
        assert calls["gpu"] == g0 + 1, (strat, integ)
        ref = ev._evaluate_chunk(law, cfg, en, an, ep, np.broadcast_to(dt, (len(dt),)).copy(), True)
        assert rel(r.sigma, ref.sigma) <= 1e-10 and rel(r.a, ref.a) <= 1e-10, (strat, integ)
        assert rel(r.C, ref.C) <= 1e-8, (strat, integ)
        assert np.array_equal(r.substeps, ref.substeps) and np.array_equal(r.rejected, ref.rejected), (strat, integ)
