"""GPU parity of the material kernel (K1) against the reference fixtures and the oracle.

Tolerances are the north star's: stress and internal variables within 1e-10
relative, tangent within 1e-8 relative, identical per-voxel Newton counts.
"""

import ctypes

import numpy as np
import pytest

from conftest import golden
from oracle import material as OM
from _util import TOL_STATE, TOL_TANGENT, assert_close, rowwise_relerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2006_04391_b200 import _lib, gsm
    from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays

    _lib.load()
    cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
    return gsm, cfg, evaluate_arrays


@pytest.mark.parametrize("tangent", [False, True])
def test_config2_golden(api, tangent):
    gsm, cfg, ev = api
    g = golden("material_evp.npz")
    r = ev(gsm.MichelSuquet(), cfg, g["eps_n"], g["a_n"], g["eps_np1"], g["dt"], want_tangent=tangent)
    assert np.array_equal(r.newton_iters, g["iters"])
    assert_close(r.sigma, g["sigma"], TOL_STATE, "sigma")
    assert_close(r.a, g["a"], TOL_STATE, "a")
    assert np.max(rowwise_relerr(r.sigma, g["sigma"])) <= TOL_STATE
    if tangent:
        assert_close(r.C, g["C"], TOL_TANGENT, "C")
        assert np.max(rowwise_relerr(r.C, g["C"])) <= TOL_TANGENT
    else:
        assert r.C is None
    assert np.all(r.substeps == 1) and np.all(r.rejected == 0)


def test_stress_newton_mode(api):
    gsm, _, ev = api
    from paper_2006_04391_b200.evaluator import StrategyConfig

    g = golden("material_evp.npz")
    cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler", error_measure="stress")
    r = ev(gsm.MichelSuquet(), cfg, g["eps_n"], g["a_n"], g["eps_np1"], g["dt"])
    assert np.array_equal(r.newton_iters, g["iters_stress"])
    assert_close(r.sigma, g["sigma_stress"], TOL_STATE)
    assert_close(r.a, g["a_stress"], TOL_STATE)


@pytest.mark.parametrize("case", [str(c) for c in golden("material_edge.npz")["cases"]])
@pytest.mark.parametrize("t", ["n", "t"])
def test_edge_cases(api, case, t):
    gsm, cfg, ev = api
    from paper_2006_04391_b200.odeint import NewtonDivergenceError

    g = golden("material_edge.npz")
    tag = f"{case}_{t}"
    args = (gsm.MichelSuquet(), cfg, g[tag + "_eps_n"], g[tag + "_a_n"], g[tag + "_eps_np1"], g[tag + "_dt"])
    if str(g[tag + "_err"]) == "NewtonDivergenceError":
        with pytest.raises(NewtonDivergenceError):
            ev(*args, want_tangent=(t == "t"))
        return
    r = ev(*args, want_tangent=(t == "t"))
    assert np.array_equal(r.newton_iters, g[tag + "_iters"])
    assert_close(r.sigma, g[tag + "_sigma"], TOL_STATE, "sigma")
    assert_close(r.a, g[tag + "_a"], TOL_STATE, "a")
    if t == "t":
        assert_close(r.C, g[tag + "_C"], TOL_TANGENT, "C")


@pytest.mark.parametrize("name,E,nu", [("le_matrix", 55e9, 0.33), ("le_fiber", 300e9, 0.25)])
def test_linear_elastic(api, name, E, nu):
    gsm, cfg, ev = api
    g = golden("material_edge.npz")
    B = g[name + "_eps_n"].shape[0]
    r = ev(gsm.LinearElastic(E, nu), cfg, g[name + "_eps_n"], np.zeros((B, 0)), g[name + "_eps_np1"], 0.05, True)
    assert_close(r.sigma, g[name + "_sigma"], TOL_STATE)
    assert_close(r.C, g[name + "_C"], TOL_TANGENT)
    assert r.a.shape == (B, 0)


def test_config2_vs_oracle_65536(api):
    """2^16 config-2 voxels: the scale the survey's parity gate names."""
    gsm, cfg, ev = api
    from paper_2006_04391_b200.workloads import config2_batch

    en, an, ep, dt = config2_batch(1 << 16, seed=0)
    r = ev(gsm.MichelSuquet(), cfg, en, an, ep, dt, want_tangent=True)
    o = OM.evaluate(OM.ALUMINUM, en, an, ep, dt, True, threads=8)
    assert np.array_equal(r.newton_iters, o["iters"])
    assert np.max(rowwise_relerr(r.sigma, o["sigma"])) <= TOL_STATE
    assert np.max(rowwise_relerr(r.a, o["a"])) <= TOL_STATE
    assert np.max(rowwise_relerr(r.C, o["C"])) <= TOL_TANGENT


def test_device_soa_entry_matches_host_entry(api):
    """am_eval_batch (device SoA pointers, caller's stream) == am_eval_batch_host, bitwise."""
    import torch

    gsm, cfg, ev = api
    from paper_2006_04391_b200 import _lib
    from paper_2006_04391_b200.workloads import config2_batch

    B = 3000
    en, an, ep, dt = config2_batch(B, seed=5)
    ref = ev(gsm.MichelSuquet(), cfg, en, an, ep, dt, want_tangent=True)
    dev = torch.device("cuda:0")
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x.T)).to(dev)  # noqa: E731  AoS -> SoA
    d_en, d_an, d_ep = t(en), t(an), t(ep)
    d_sig = torch.empty((6, B), dtype=torch.float64, device=dev)
    d_a = torch.empty((7, B), dtype=torch.float64, device=dev)
    d_C = torch.empty((36, B), dtype=torch.float64, device=dev)
    d_it = torch.empty(B, dtype=torch.int32, device=dev)
    d_st = torch.empty(B, dtype=torch.uint8, device=dev)
    d_fl = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _lib.load()
    rc = lib.am_eval_batch(
        _lib.make_law(gsm.MichelSuquet()), _lib.make_cfg(cfg), B, d_en.data_ptr(), d_an.data_ptr(), d_ep.data_ptr(),
        None, 0.05, 1, d_sig.data_ptr(), d_a.data_ptr(), d_C.data_ptr(), d_it.data_ptr(), None, d_st.data_ptr(),
        d_fl.data_ptr(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    _lib.check(rc)
    torch.cuda.synchronize()
    assert np.array_equal(d_sig.cpu().numpy().T, ref.sigma)
    assert np.array_equal(d_a.cpu().numpy().T, ref.a)
    assert np.array_equal(d_C.cpu().numpy().T.reshape(B, 6, 6), ref.C)
    assert np.array_equal(d_it.cpu().numpy(), ref.newton_iters)
    assert int(d_fl.item()) == 0


def test_results_independent_of_batching(api):
    """Per-voxel results do not depend on batch composition (evaluator.py:1-10)."""
    gsm, cfg, ev = api
    from paper_2006_04391_b200.workloads import config2_batch

    en, an, ep, dt = config2_batch(700, seed=9)
    full = ev(gsm.MichelSuquet(), cfg, en, an, ep, dt, want_tangent=True)
    part = ev(gsm.MichelSuquet(), cfg, en[100:133], an[100:133], ep[100:133], dt[100:133], want_tangent=True)
    assert np.array_equal(part.sigma, full.sigma[100:133])
    assert np.array_equal(part.C, full.C[100:133])


def test_constitutive_ops(api):
    gsm, _, _ = api
    g = golden("constitutive.npz")
    law = gsm.MichelSuquet()
    assert_close(gsm.stress(law, g["eps"], g["a"]), g["stress"], 1e-14)
    assert_close(gsm.generalized_stress(law, g["eps"], g["a"]), g["gen_stress"], 1e-14)
    assert_close(gsm.evolution_rhs(law, g["eps"], g["a"]), g["rhs"], 1e-12)
    assert_close(gsm.rhs_jacobian(law, g["eps"], g["a"]), g["dfda"], 1e-12)
    assert_close(gsm.rhs_strain_jacobian(law, g["eps"], g["a"]), g["dfde"], 1e-12)
    assert_close(gsm.stress(gsm.LinearElastic(300e9, 0.25), g["eps"], np.zeros((len(g["eps"]), 0))),
                 g["le_stress"], 1e-14)


def test_python_law_rejected(api):
    gsm, cfg, ev = api
    from paper_2006_04391_b200.evaluator import ConfigError

    class MyLaw(gsm.GsmDefinition):
        m = 1

    with pytest.raises(ConfigError):
        ev(MyLaw(), cfg, np.zeros((2, 6)), np.zeros((2, 1)), np.zeros((2, 6)), 0.1)


def test_evaluate_batch_isolates_failures(api):
    gsm, cfg, _ = api
    from paper_2006_04391_b200.evaluator import EvalRequest, evaluate_batch

    g = golden("material_edge.npz")
    reqs = [EvalRequest(g["large_n_eps_n"][i], g["large_n_a_n"][i], g["large_n_eps_np1"][i], 1.0) for i in range(3)]
    reqs.append(EvalRequest(np.zeros(6), np.zeros(7), g["newton_fail_n_eps_np1"][0], 1e6))
    res, errs = evaluate_batch(gsm.MichelSuquet(), cfg, reqs)
    assert list(errs) == [3] and errs[3].startswith("NewtonDivergenceError")
    for i in range(3):
        assert_close(res[i].sigma, g["large_n_sigma"][i], TOL_STATE)


def test_evaluate_batch_groups_and_config_errors(api):
    """material_ids grouping, a law without device potentials reported per
    request, and batch results equal to single-request results."""
    gsm, cfg, ev = api
    from paper_2006_04391_b200.evaluator import EvalRequest, evaluate, evaluate_batch
    from paper_2006_04391_b200.workloads import config2_batch

    class PyLaw(gsm.GsmDefinition):
        m = 0

    en, an, ep, dt = config2_batch(6, seed=3)
    reqs = [EvalRequest(en[i], an[i] if i % 3 else np.zeros(0), ep[i], 0.05, want_tangent=True) for i in range(6)]
    ids = [1 if i % 3 else 0 for i in range(6)]
    laws = {0: PyLaw(), 1: gsm.MichelSuquet()}
    res, errs = evaluate_batch(laws, cfg, reqs, material_ids=ids)
    assert sorted(errs) == [0, 3] and all(e.startswith("ConfigError") for e in errs.values())
    for i in (1, 2, 4, 5):
        one = evaluate(gsm.MichelSuquet(), cfg, reqs[i])
        assert np.array_equal(res[i].sigma, one.sigma) and np.array_equal(res[i].C, one.C)


def test_host_entry_pageable_vs_pinned(api):
    """am_eval_batch_host stages pageable arrays through pinned slots (3-slot
    pipeline, chunk ramp 2^12 .. 2^17): results equal the pinned-array path
    bit for bit, for a batch spanning many chunks, every output array
    pageable or pinned in any mix."""
    import torch

    gsm, cfg, ev = api
    from paper_2006_04391_b200 import _lib
    from paper_2006_04391_b200.workloads import config2_batch

    B = 300_001
    en, an, ep, dt = config2_batch(B, seed=17)
    lib = _lib.load()
    law, c = _lib.make_law(gsm.MichelSuquet()), _lib.make_cfg(cfg)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731

    def run(inputs, pinned_out):
        alloc = (lambda s, d=np.float64: torch.empty(s, dtype=getattr(torch, np.dtype(d).name)).pin_memory().numpy()) \
            if pinned_out else (lambda s, d=np.float64: np.full(s, 7, dtype=d))
        sig, a, C = alloc((B, 6)), alloc((B, 7)), alloc((B, 6, 6))
        it, st = alloc((B,), np.int32), alloc((B,), np.uint8)
        _lib.check(lib.am_eval_batch_host(law, c, B, *[_lib.ptr(x) for x in inputs], 1, _lib.ptr(sig), _lib.ptr(a),
                                          _lib.ptr(C), _lib.ptr(it, _lib._i32p), None, _lib.ptr(st, _lib._u8p)))
        return sig, a, C, it, st

    pageable = (en, an, ep, dt)
    pinned = tuple(pin(x) for x in pageable)
    mixed = (en, pinned[1], ep, pinned[3])
    base = run(pinned, True)
    for inputs, po in ((pageable, False), (pageable, True), (pinned, False), (mixed, False)):
        got = run(inputs, po)
        for x, y in zip(got, base):
            assert np.array_equal(x, y)
    assert np.all(base[4] == 0)


def test_evaluate_arrays_results_from_pool(api):
    """evaluate_arrays returns its results in recycled page-locked blocks:
    every element is rewritten (garbage planted in the pool never shows)."""
    gsm, cfg, ev = api
    from paper_2006_04391_b200 import _lib
    from paper_2006_04391_b200.workloads import config2_batch

    B = 50_000
    en, an, ep, dt = config2_batch(B, seed=3)
    ref = ev(gsm.MichelSuquet(), cfg, en, an, ep, dt, want_tangent=True)
    ref = (ref.sigma.copy(), ref.a.copy(), ref.C.copy(), ref.newton_iters.copy())
    for law, m in ((gsm.MichelSuquet(), 7), (gsm.LinearElastic(300e9, 0.25), 0)):
        junk = [_lib.pinned_empty(s) for s in ((B, 6), (B, 7), (B, 6, 6), (B, 2))]
        for j in junk:
            j.fill(np.nan)
        del junk, j  # back to the pool
        r = ev(law, cfg, en, an[:, :m], ep, dt, want_tangent=True)
        assert np.all(np.isfinite(r.sigma)) and np.all(np.isfinite(r.C)) and np.all(np.isfinite(r.a))
        assert np.all(r.substeps == 1) and np.all(r.rejected == 0)
        if m:
            assert np.array_equal(r.sigma, ref[0]) and np.array_equal(r.C, ref[2])
            assert np.array_equal(r.newton_iters, ref[3])
        else:
            assert np.all(r.newton_iters == 0)
