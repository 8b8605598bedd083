"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container only (the reference tree does not exist on the
GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--skip-slow]

Every fixture is produced by importing ``gsmkit`` from
/root/reference/pkg/src and calling its public API unchanged, with
``StrategyConfig(strategy="automatic", integrator="implicit-euler")``
unless stated. Per-voxel Newton iteration counts are taken with a wrapper
around ``MaterialStepProblem.rhs_and_jac`` that counts the compacted
indices the Newton loop passes (odeint.py:376-377); the tangent
post-process calls it with idx=None (odeint.py:421) and is not counted.
"""

import argparse
import importlib.util
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from gsmkit import gsm, linalg, odeint  # noqa: E402
from gsmkit import homogenize as H  # noqa: E402
from gsmkit.evaluator import StrategyConfig, evaluate_arrays  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.environ.get("GOLD_OUT", HERE)  # long runs write elsewhere first
_spec = importlib.util.spec_from_file_location(
    "workloads", os.path.join(HERE, "..", "..", "paper_2006_04391_b200", "workloads.py")
)
W = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(W)

AUTO = StrategyConfig(strategy="automatic", integrator="implicit-euler")
AUTO_STRESS = StrategyConfig(strategy="automatic", integrator="implicit-euler", error_measure="stress")
CONV = StrategyConfig(strategy="conventional", integrator="implicit-euler")

# ---------------------------------------------------------------- counters
_COUNT = {"arr": None}
_orig_rhs_and_jac = odeint.MaterialStepProblem.rhs_and_jac


def _counting_rhs_and_jac(self, t, y, idx=None):
    if idx is not None and _COUNT["arr"] is not None:
        np.add.at(_COUNT["arr"], idx, 1)
    return _orig_rhs_and_jac(self, t, y, idx)


odeint.MaterialStepProblem.rhs_and_jac = _counting_rhs_and_jac


def eval_counted(law, cfg, eps_n, a_n, eps_np1, dt, want_tangent):
    """evaluate_arrays with per-voxel Newton counts (single chunk)."""
    B = eps_np1.shape[0]
    cfg = StrategyConfig(
        strategy=cfg.strategy,
        integrator=cfg.integrator,
        error_measure=cfg.error_measure,
        chunk_size=max(B, 1),
    )
    _COUNT["arr"] = np.zeros(B, dtype=np.int64)
    try:
        r = evaluate_arrays(law, cfg, eps_n, a_n, eps_np1, dt, want_tangent=want_tangent)
        err = ""
    except Exception as exc:  # noqa: BLE001
        r = None
        err = type(exc).__name__
    cnt = _COUNT["arr"]
    _COUNT["arr"] = None
    frozen = np.broadcast_to(np.asarray(dt, dtype=float), (B,)) == 0.0
    if frozen.any() and not frozen.all():
        # the mixed split (evaluator.py:151-156) re-enters _evaluate_chunk on
        # the dt > 0 subset, so the Newton indices are local to that subset
        ipos = np.flatnonzero(~frozen)
        full = np.zeros(B, dtype=np.int64)
        full[ipos] = cnt[: len(ipos)]
        cnt = full
    return r, cnt, err


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name} ({os.path.getsize(path) / 1024:.1f} KiB)")


# ---------------------------------------------------------------- material
def make_material():
    law = gsm.MichelSuquet()
    eps_n, a_n, eps_np1, dt = W.config2_batch(1024, seed=0)
    r, cnt, err = eval_counted(law, AUTO, eps_n, a_n, eps_np1, dt, True)
    assert not err
    rs, cnts, errs = eval_counted(law, AUTO_STRESS, eps_n, a_n, eps_np1, dt, False)
    assert not errs
    save(
        "material_evp.npz",
        eps_n=eps_n, a_n=a_n, eps_np1=eps_np1, dt=dt,
        sigma=r.sigma, a=r.a, C=r.C, iters=cnt,
        sigma_stress=rs.sigma, a_stress=rs.a, iters_stress=cnts,
    )

    # edge cases, one law call per case (the reference raises per call)
    rng = np.random.default_rng(7)
    cases = {}

    # elastic voxels: tiny strains, zero state -> one Newton iteration each
    B = 64
    en = rng.normal(0, 1e-6, (B, 6)); ep = en + rng.normal(0, 1e-6, (B, 6)); an = np.zeros((B, 7))
    cases["elastic"] = (en, an, ep, np.full(B, 0.05))

    # frozen mix: every third voxel has dt == 0 (evaluator.py:142-170)
    en, an, ep, dtv = W.config2_batch(48, seed=11)
    dtv[::3] = 0.0
    cases["frozen_mix"] = (en, an, ep, dtv)

    # all frozen
    en, an, ep, dtv = W.config2_batch(16, seed=12)
    cases["frozen_all"] = (en, an, ep, np.zeros(16))

    # negative alpha on input: clamp_state (gsm.py:252-256) after integration
    en, an, ep, dtv = W.config2_batch(32, seed=13)
    an[:, 6] = -np.abs(an[:, 6])
    ep[:16] = en[:16] + 1e-7  # elastic half keeps a_n, clamp shows
    cases["clamp"] = (en, an, ep, dtv)

    # large increments, long steps: many Newton iterations
    en = np.zeros((64, 6)); ep = rng.normal(0, 1.0, (64, 6)); an = np.zeros((64, 7))
    cases["large"] = (en, an, ep, np.full(64, 1.0))

    # varied dt per voxel
    en, an, ep, dtv = W.config2_batch(64, seed=14)
    dtv = 10.0 ** rng.uniform(-4, 2, 64)
    cases["dt_sweep"] = (en, an, ep, dtv)

    # Newton failure: singular iteration matrix at huge h (odeint.py:380-381)
    en = np.zeros((4, 6)); ep = np.random.default_rng(1).normal(0, 1.0, (4, 6)); an = np.zeros((4, 7))
    cases["newton_fail"] = (en, an, ep, np.full(4, 1e6))

    out = {}
    for name, (en, an, ep, dtv) in cases.items():
        for tang in (False, True):
            r, cnt, err = eval_counted(law, AUTO, en, an, ep, dtv, tang)
            tag = f"{name}_{'t' if tang else 'n'}"
            out[f"{tag}_eps_n"] = en
            out[f"{tag}_a_n"] = an
            out[f"{tag}_eps_np1"] = ep
            out[f"{tag}_dt"] = dtv
            out[f"{tag}_err"] = np.array(err)
            out[f"{tag}_iters"] = cnt
            if r is not None:
                out[f"{tag}_sigma"] = r.sigma
                out[f"{tag}_a"] = r.a
                if tang:
                    out[f"{tag}_C"] = r.C
    out["cases"] = np.array(sorted(cases))

    # linear elastic laws (m == 0 path, evaluator.py:134-140)
    for lname, law_le in (("le_matrix", gsm.LinearElastic(55e9, 0.33)), ("le_fiber", gsm.LinearElastic(300e9, 0.25))):
        B = 64
        en = rng.normal(0, 1e-3, (B, 6)); ep = en + rng.normal(0, 1e-3, (B, 6))
        an = np.zeros((B, 0))
        r, _, err = eval_counted(law_le, AUTO, en, an, ep, np.full(B, 0.05), True)
        assert not err
        out[f"{lname}_eps_n"] = en
        out[f"{lname}_eps_np1"] = ep
        out[f"{lname}_sigma"] = r.sigma
        out[f"{lname}_C"] = r.C
    save("material_edge.npz", **out)


# ---------------------------------------------------------------- adaptive integrators
def make_adaptive():
    """ode12 / ode23 (automatic strategy), internal and stress error measures,
    with and without the coupled tangent: sigma, a, C, substeps, rejected."""
    law = gsm.MichelSuquet()
    out = {}
    en, an, ep, dt = W.config2_batch(192, seed=21)
    dt = dt.copy()
    dt[64:128] = 10.0 ** np.random.default_rng(22).uniform(-3, 1, 64)  # varied step lengths
    dt[128:136] = 0.0  # frozen points inside an adaptive batch
    out.update(eps_n=en, a_n=an, eps_np1=ep, dt=dt)
    for integ in ("ode12", "ode23"):
        for meas in ("internal", "stress"):
            cfg = StrategyConfig(strategy="automatic", integrator=integ, error_measure=meas)
            for tang in (False, True):
                t0 = time.time()
                r = evaluate_arrays(law, cfg, en, an, ep, dt, want_tangent=tang)
                tag = f"{integ}_{meas}_{'t' if tang else 'n'}"
                out[tag + "_sigma"] = r.sigma
                out[tag + "_a"] = r.a
                out[tag + "_substeps"] = r.substeps
                out[tag + "_rejected"] = r.rejected
                if tang:
                    out[tag + "_C"] = r.C
                print(f"adaptive {tag}: {time.time() - t0:.1f}s, substeps {r.substeps.sum()}, rejected {r.rejected.sum()}")
    # record_steps: every attempt's (h, accepted), including frozen points
    cfg = StrategyConfig(strategy="automatic", integrator="ode23", record_steps=True)
    r = evaluate_arrays(law, cfg, en[120:152], an[120:152], ep[120:152], dt[120:152], want_tangent=True)
    flat = [(b, h, acc) for b, lst in enumerate(r.steps) for (h, acc) in lst]
    out.update(rec_b=np.array([f[0] for f in flat]), rec_h=np.array([f[1] for f in flat]),
               rec_acc=np.array([f[2] for f in flat]))
    # IntegrationError: substep cap on large increments
    cfg = StrategyConfig(strategy="automatic", integrator="ode23", max_substeps=3)
    e2 = np.zeros((4, 6))
    p2 = np.random.default_rng(23).normal(0, 1e-2, (4, 6))
    try:
        evaluate_arrays(law, cfg, e2, np.zeros((4, 7)), p2, np.full(4, 1.0), want_tangent=True)
        err = ""
    except Exception as exc:  # noqa: BLE001
        err = type(exc).__name__
    out.update(cap_eps_np1=p2, cap_err=np.array(err))
    print("cap case:", err)
    # basic scheme with the default StrategyConfig() (ode23): 8^3 toy grid,
    # load step 1 converges; step 2 stagnates near 5e-4 (the adaptive step
    # selection makes sigma(eps) non-smooth) and raises SolverError
    grid = H.toy_mmc_grid(8)
    hom = H.Homogenizer(grid, StrategyConfig(), max_iterations=400)
    path = H.LoadingPath(steps=20)
    tt = path.times()
    ex = path.eps_xx(tt)
    free = np.array([False] + [True] * 5)
    eb = np.zeros(6)
    eb[0] = ex[1]
    eps, sig, info = hom.solve_step(eb, tt[1] - tt[0], free_mask=free)
    out.update(path8_ode23_iters=np.array(info.iterations), path8_ode23_mean_substeps=np.array(info.mean_substeps),
               path8_ode23_history=np.array(info.history), path8_ode23_sig_bar=sig.mean(axis=(1, 2, 3)))
    hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
    eb[0] = ex[2]
    try:
        hom.solve_step(eb, tt[2] - tt[1], free_mask=free)
        err = ""
    except H.SolverError:
        err = "SolverError"
    out.update(path8_ode23_step2_err=np.array(err))
    print("path8 ode23:", info.iterations, info.mean_substeps, err)
    save("adaptive.npz", **out)


# ---------------------------------------------------------------- semi-automatic strategy
def make_semi():
    """strategy='semi-automatic' (hand partials, gsm.py:258-328, 463-481):
    implicit Euler with Newton counts, and ode23 / ode12, with and without tangent."""
    law = gsm.MichelSuquet()
    out = {}
    en, an, ep, dt = W.config2_batch(256, seed=31)
    dt = dt.copy()
    dt[200:232] = 10.0 ** np.random.default_rng(32).uniform(-3, 1, 32)
    dt[232:240] = 0.0
    out.update(eps_n=en, a_n=an, eps_np1=ep, dt=dt)
    SEMI = StrategyConfig(strategy="semi-automatic", integrator="implicit-euler")
    for tang in (False, True):
        r, cnt, err = eval_counted(law, SEMI, en, an, ep, dt, tang)
        assert not err
        tag = f"ie_{'t' if tang else 'n'}"
        out[tag + "_sigma"], out[tag + "_a"], out[tag + "_iters"] = r.sigma, r.a, cnt
        if tang:
            out[tag + "_C"] = r.C
    for integ in ("ode12", "ode23", "ode23s"):
        cfg = StrategyConfig(strategy="semi-automatic", integrator=integ)
        for tang in (False, True):
            r = evaluate_arrays(law, cfg, en, an, ep, dt, want_tangent=tang)
            tag = f"{integ}_{'t' if tang else 'n'}"
            out[tag + "_sigma"], out[tag + "_a"] = r.sigma, r.a
            out[tag + "_substeps"], out[tag + "_rejected"] = r.substeps, r.rejected
            if tang:
                out[tag + "_C"] = r.C
    cfg = StrategyConfig(strategy="semi-automatic", integrator="ode23s", error_measure="stress")
    for tang in (False, True):
        r = evaluate_arrays(law, cfg, en, an, ep, dt, want_tangent=tang)
        tag = f"ode23s_stress_{'t' if tang else 'n'}"
        out[tag + "_sigma"], out[tag + "_a"] = r.sigma, r.a
        out[tag + "_substeps"], out[tag + "_rejected"] = r.substeps, r.rejected
        if tang:
            out[tag + "_C"] = r.C
    le = gsm.LinearElastic(300e9, 0.25)
    r = evaluate_arrays(le, SEMI, en, np.zeros((256, 0)), ep, dt, want_tangent=True)
    out.update(le_sigma=r.sigma, le_C=r.C)
    # conventional radial return (gsm.py:332-404, evaluator.py:172-174)
    for tang in (False, True):
        r = evaluate_arrays(law, CONV, en, an, ep, dt, want_tangent=tang)
        tag = f"conv_{'t' if tang else 'n'}"
        out[tag + "_sigma"], out[tag + "_a"] = r.sigma, r.a
        if tang:
            out[tag + "_C"] = r.C
    save("material_semi.npz", **out)


# ---------------------------------------------------------------- constitutive
def make_constitutive():
    law = gsm.MichelSuquet()
    rng = np.random.default_rng(3)
    B = 256
    eps = rng.normal(0, 2e-3, (B, 6))
    a = np.zeros((B, 7))
    a[:, :6] = rng.normal(0, 5e-4, (B, 6))
    a[:, 6] = np.abs(rng.normal(0, 1e-3, B))
    a[:8] = 0.0
    eps[:4] = 0.0  # elastic states -> zero flow, zero Jacobians
    # The reference's batched generalized_stress fails to stack the scalar
    # A_alpha = -sigma_Y (gsm.py:50, 441-449); evaluate point by point.
    def per_point(fn):
        return np.stack([np.asarray(fn(law, eps[i], a[i]), dtype=float) for i in range(B)])

    save(
        "constitutive.npz",
        eps=eps, a=a,
        stress=per_point(gsm.stress),
        gen_stress=per_point(gsm.generalized_stress),
        rhs=per_point(gsm.evolution_rhs),
        dfda=per_point(gsm.rhs_jacobian),
        dfde=per_point(gsm.rhs_strain_jacobian),
        le_stress=gsm.stress(gsm.LinearElastic(300e9, 0.25), eps, np.zeros((B, 0))),
    )


# ---------------------------------------------------------------- lawops
def make_lawops():
    """LawOps under both strategies (gsm.py:412-566) and conventional_evaluate (gsm.py:605-609)."""
    law = gsm.MichelSuquet()
    rng = np.random.default_rng(4)
    B = 128
    eps = rng.normal(0, 2e-3, (B, 6))
    a = np.zeros((B, 7))
    a[:, :6] = rng.normal(0, 5e-4, (B, 6))
    a[:, 6] = np.abs(rng.normal(0, 1e-3, B))
    a[:8] = 0.0
    eps[:4] = 0.0
    da = rng.normal(0, 1.0, (B, 7, 6))
    out = {"eps": eps, "a": a, "da": da}
    for tag, strat in (("auto", "automatic"), ("semi", "semi-automatic")):
        ops = gsm.LawOps(law, strat)
        out[tag + "_stress"] = ops.stress(eps, a)
        out[tag + "_gen_stress"] = np.stack([np.asarray(ops.gen_stress(eps[i], a[i]), dtype=float)
                                             for i in range(B)])
        f, J, Je = ops.rhs_and_jacobians(eps, a)
        out[tag + "_rhs"], out[tag + "_dfda"], out[tag + "_dfde"] = f, J, Je
        sig, C = ops.stress_and_tangent(eps, a, da)
        out[tag + "_st_sigma"], out[tag + "_st_C"] = sig, C
        out[tag + "_elastic_C"] = ops.elastic_tangent(eps, a)
    le = gsm.LinearElastic(300e9, 0.25)
    for tag, strat in (("auto", "automatic"), ("semi", "semi-automatic")):
        ops = gsm.LawOps(le, strat)
        out["le_" + tag + "_stress"] = ops.stress(eps, np.zeros((B, 0)))
        out["le_" + tag + "_C"] = ops.stress_and_tangent(eps, np.zeros((B, 0)), np.zeros((B, 0, 6)))[1]
    # conventional radial return: a loading step from the states above
    eps_np1 = eps + rng.normal(0, 3e-3, (B, 6))
    h = np.full(B, 0.05)
    h[:3] = 0.0
    sig, a_new, C = gsm.conventional_evaluate(law, eps, a, eps_np1, h, want_tangent=True)
    out.update(conv_eps_np1=eps_np1, conv_h=h, conv_sigma=sig, conv_a=a_new, conv_C=C)
    save("lawops.npz", **out)


# ---------------------------------------------------------------- fourier
def make_fourier():
    rng = np.random.default_rng(5)
    out = {}
    dims_list = [(8, 8, 8), (16, 12, 10), (9, 8, 7), (4, 6, 5), (1, 8, 6)]
    ref = H.ReferenceMaterial(lam=80068553737.28441, mu=70338345864.66165)
    for k, dims in enumerate(dims_list):
        tau = rng.normal(0, 1e8, (6,) + dims)
        sig = rng.normal(0, 1e8, (6,) + dims) + np.array([3e8, 1e8, -2e8, 1e7, 0, 5e6])[:, None, None, None]
        eps = rng.normal(0, 1e-3, (6,) + dims)
        out[f"d{k}_dims"] = np.array(dims)
        out[f"d{k}_tau"] = tau
        out[f"d{k}_green"] = H.GreenOperator(dims, ref).apply(tau)
        out[f"d{k}_sig"] = sig
        out[f"d{k}_residual"] = np.array(H.equilibrium_residual(sig))
        out[f"d{k}_eps"] = eps
        out[f"d{k}_iso"] = H.apply_isotropic(ref, eps)
    out["ndims"] = np.array(len(dims_list))
    out["ref"] = np.array([ref.lam, ref.mu])

    # reference_update on random tangent fields (homogenize.py:307-329)
    for k in range(3):
        N = 300
        law = gsm.MichelSuquet()
        C = np.broadcast_to(law.Ce, (N, 6, 6)).copy()
        C += rng.normal(0, 5e9, (N, 6, 6))
        out[f"ru{k}_C"] = C
        r = H.reference_update(C)
        out[f"ru{k}_lam_mu"] = np.array([r.lam, r.mu])
    save("fourier.npz", **out)


# ---------------------------------------------------------------- config 1
def make_config1():
    n = 32
    ids = W.sphere_ids(n)
    out = {"ids": ids}
    sub = np.arange(0, n**3, 37)
    out["sub"] = sub
    for tag, free in (("strain", np.zeros(6, dtype=bool)), ("mixed", np.array([False] + [True] * 5))):
        grid = H.VoxelGrid(ids, [gsm.LinearElastic(55e9, 0.33), gsm.LinearElastic(300e9, 0.25)])
        hom = H.Homogenizer(grid, AUTO)
        eb = np.zeros(6); eb[0] = 1e-3
        t0 = time.time()
        eps, sig, info = hom.solve_step(eb, 1.0, free_mask=free)
        print(f"config1 {tag}: {info.iterations} it, {time.time() - t0:.2f}s")
        out[f"{tag}_iters"] = np.array(info.iterations)
        out[f"{tag}_history"] = np.array(info.history)
        out[f"{tag}_sig_bar"] = sig.mean(axis=(1, 2, 3))
        out[f"{tag}_eps_bar"] = eps.mean(axis=(1, 2, 3))
        out[f"{tag}_sig_sub"] = sig.reshape(6, -1)[:, sub]
        out[f"{tag}_eps_sub"] = eps.reshape(6, -1)[:, sub]
        out[f"{tag}_ref"] = np.array([hom.reference.lam, hom.reference.mu])
    # SolverError: iteration cap with history (homogenize.py:466-471)
    grid = H.VoxelGrid(ids, [gsm.LinearElastic(55e9, 0.33), gsm.LinearElastic(300e9, 0.25)])
    hom = H.Homogenizer(grid, AUTO, max_iterations=4)
    eb = np.zeros(6); eb[0] = 1e-3
    try:
        hom.solve_step(eb, 1.0)
        raise AssertionError("expected SolverError")
    except H.SolverError as exc:
        out["cap_history"] = np.array(exc.history)
    save("config1.npz", **out)


# ---------------------------------------------------------------- loading paths
def _records_to_arrays(recs):
    return dict(
        step=np.array([r["step"] for r in recs]),
        time=np.array([r["time"] for r in recs]),
        eps_xx=np.array([r["eps_xx"] for r in recs]),
        sig=np.stack([r["sig"] for r in recs]),
        C11=np.array([r["C11"] for r in recs]),
        C12=np.array([r["C12"] for r in recs]),
        iterations=np.array([r["iterations"] for r in recs]),
        mean_substeps=np.array([r["mean_substeps"] for r in recs]),
    )


def make_path8():
    """8^3 toy MMC, 6 of 20 steps, fully automatic route, plus final state."""
    grid = H.toy_mmc_grid(8)
    path = H.LoadingPath(steps=20)
    t0 = time.time()
    # run the loop by hand to stop after 6 steps and keep the state
    hom = H.Homogenizer(grid, AUTO)
    times = path.times()
    targets = path.eps_xx(times)
    free = np.array([False, True, True, True, True, True])
    recs = []
    refs = [(hom.reference.lam, hom.reference.mu)]
    for k in range(1, 7):
        dt = times[k] - times[k - 1]
        eb = np.zeros(6); eb[0] = targets[k]
        eps, sigma, info = hom.solve_step(eb, dt, free_mask=free)
        ebar = eps.mean(axis=(1, 2, 3))
        _, C_vox, _, _ = hom.evaluate_field(eps, dt, want_tangent=True)
        C_bar = C_vox.mean(axis=0)
        hom.commit_step(eps, ebar)
        hom.set_reference(H.reference_update(C_vox))
        refs.append((hom.reference.lam, hom.reference.mu))
        recs.append({"step": k, "time": float(times[k]), "eps_xx": float(ebar[0]), "sig": sigma.mean(axis=(1, 2, 3)),
                     "C11": float(C_bar[0, 0]), "C12": float(C_bar[0, 1]), "iterations": info.iterations,
                     "mean_substeps": info.mean_substeps, "Cbar": C_bar, "history": info.history})
        print(f"path8 step {k}: {info.iterations} it ({time.time() - t0:.1f}s)")
    arr = _records_to_arrays(recs)
    arr["Cbar"] = np.stack([r["Cbar"] for r in recs])
    hist = [np.array(r["history"]) for r in recs]
    arr["history_flat"] = np.concatenate(hist)
    arr["refs"] = np.array(refs)
    arr["ids"] = grid.material_ids
    arr["eps_n"] = hom.eps_n
    arr["state0"] = grid.state[0]
    save("path8_auto.npz", **arr)


def make_path16_conv():
    """16^3 toy MMC, 20 steps, per-law conventional oracle."""
    _ea = H.evaluate_arrays

    def _per_law(law, cfg, *a, **k):
        if cfg.strategy == "conventional" and not law.has_conventional:
            cfg = AUTO
        return _ea(law, cfg, *a, **k)

    H.evaluate_arrays = _per_law
    try:
        t0 = time.time()
        grid = H.toy_mmc_grid(16)
        recs = H.run_loading_path(grid, H.LoadingPath(steps=20), CONV)
        print(f"path16 conventional: {time.time() - t0:.1f}s")
    finally:
        H.evaluate_arrays = _ea
    arr = _records_to_arrays(recs)
    arr["ids"] = grid.material_ids
    save("path16_conv.npz", **arr)


def make_path_conv(n, steps=20):
    """n^3 toy MMC, LoadingPath(steps), per-law conventional oracle (SURVEY
    §8c, App. C): the same call sequence as the reference's run_loading_path
    (homogenize.py:485-528), written out so the Homogenizer stays reachable
    for per-step histories, reference materials and final field samples.
    The fixture is rewritten after every step, so a long run (128^3: hours)
    pins every step it has finished."""
    _ea = H.evaluate_arrays

    def _per_law(law, cfg, *a, **k):
        if cfg.strategy == "conventional" and not law.has_conventional:
            cfg = AUTO
        return _ea(law, cfg, *a, **k)

    H.evaluate_arrays = _per_law
    try:
        _path_by_hand(n, CONV, f"path{n}_conv.npz", steps)
    finally:
        H.evaluate_arrays = _ea


def make_path8_ode23():
    """8^3 toy MMC, first 3 of the default LoadingPath()'s 80 steps with the
    DEFAULT StrategyConfig()
    (automatic, ode23): the tangent sweep of run_loading_path is a coupled
    adaptive integration with its own step sequence, and the state committed
    must be solve_step's (homogenize.py:508-512)."""
    _path_by_hand(8, StrategyConfig(), "path8_ode23.npz", 80, last=3)


def make_path8_ode23_fail():
    """The same with LoadingPath(steps=20): step 1 converges, step 2 raises
    SolverError after 5000 iterations (the adaptive integrator's tolerance
    keeps the residual above 1e-5); fixture = step-1 records + the history."""
    grid = H.toy_mmc_grid(8)
    hom = H.Homogenizer(grid, StrategyConfig())
    path = H.LoadingPath(steps=20)
    t = path.times()
    free = np.array([False, True, True, True, True, True])
    out = {}
    for k in (1, 2):
        eb = np.zeros(6)
        eb[0] = path.eps_xx(t[k])
        try:
            eps, sigma, info = hom.solve_step(eb, t[k] - t[k - 1], free_mask=free)
        except H.SolverError as exc:
            out["fail_step"] = np.array(k)
            out["fail_history"] = np.array(exc.history)
            break
        out[f"step{k}_iters"] = np.array(info.iterations)
        out[f"step{k}_sig"] = sigma.mean(axis=(1, 2, 3))
        _, C_vox, _, _ = hom.evaluate_field(eps, t[k] - t[k - 1], want_tangent=True)
        hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
        hom.set_reference(H.reference_update(C_vox))
    save("path8_ode23_fail.npz", **out)


def make_tangent_singular():
    """The tangent post-process's check_singular LU (odeint.py:417-426,
    linalg.py:103-104) at given states: M = I - h df/da(eps(t1), a) for
    plastic states and h over 1e-2 .. 1e16, with the reference's verdict
    (SingularMatrixError or not).  In a full evaluation the Newton fails
    first (same criterion on the iterates' M); this pins the tangent's own
    route."""
    law = gsm.MichelSuquet()
    ops = gsm.LawOps(law, "automatic")
    rng = np.random.default_rng(31)
    B = 96
    eps_n = rng.normal(0, 1e-3, (B, 6))
    eps_np1 = eps_n + rng.normal(0, 1.0, (B, 6)) * 10.0 ** rng.uniform(-3, 0, (B, 1))
    a = np.zeros((B, 7))
    a[:, :6] = rng.normal(0, 5e-4, (B, 6))
    a[:, 6] = np.abs(rng.normal(0, 1e-3, B))
    dt = 10.0 ** np.linspace(-2, 16, B)
    e1 = eps_n + 1.0 * (eps_np1 - eps_n)  # odeint.py:256-264 at t1 = h
    _, J, _ = ops.rhs_and_jacobians(e1, a)
    singular = np.zeros(B, dtype=bool)
    ratio = np.zeros(B)  # min |pivot| / max|M| of the reference's LU (threshold 1e-14)
    for b in range(B):
        M = np.eye(7) - dt[b] * J[b]
        lu, _, _ = linalg.lu_factor(M, check_singular=False)
        ratio[b] = np.min(np.abs(np.diag(lu))) / np.max(np.abs(M))
        try:
            linalg.lu_factor(M, check_singular=True)
        except linalg.SingularMatrixError:
            singular[b] = True
    print("tangent singular cases:", int(singular.sum()), "of", B)
    save("tangent_singular.npz", eps_n=eps_n, eps_np1=eps_np1, a=a, dt=dt, singular=singular, ratio=ratio)


def make_radial_stall():
    """A Michel-Suquet parameter set (n = 10, small sigma_d) whose radial
    return stalls (gsm.py:377-378 NewtonError) at eps_n = 0, a_n = 0: the
    reference raises from conventional_evaluate, from evaluate_arrays with
    strategy="conventional" and from Homogenizer.solve_step on a homogeneous
    grid (first evaluation at eps = ebar); other points of the same batch
    evaluate fine."""
    p = gsm.MichelSuquetParams(E=55e9, nu=0.33, sigma_Y=25e6, H=11999049.779393503,
                               eps0_dot=0.001761331668073649, sigma_d=116442.23751767876, n=10.0)
    law = gsm.MichelSuquet(p)
    ep = np.array([0.00086759, 0.00034892, -0.00137607, 0.00095601, 0.00047135, -0.000567])
    dt = 0.43330783852286625
    out = dict(params=np.array([p.E, p.nu, p.sigma_Y, p.H, p.eps0_dot, p.sigma_d, p.n]), eps_np1=ep, dt=np.array(dt))
    raised = {}
    try:
        gsm.conventional_evaluate(law, np.zeros((1, 6)), np.zeros((1, 7)), ep[None], dt)
        raised["conventional_evaluate"] = ""
    except gsm.NewtonError as exc:
        raised["conventional_evaluate"] = type(exc).__name__
    try:
        evaluate_arrays(law, CONV, np.zeros((1, 6)), np.zeros((1, 7)), ep[None], dt)
        raised["evaluate_arrays"] = ""
    except gsm.NewtonError as exc:
        raised["evaluate_arrays"] = type(exc).__name__
    hom = H.Homogenizer(H.VoxelGrid(np.zeros((2, 2, 2), np.uint8), [law]), CONV)
    try:
        hom.solve_step(ep, dt, free_mask=np.zeros(6, bool))
        raised["solve_step"] = ""
    except gsm.NewtonError as exc:
        raised["solve_step"] = type(exc).__name__
    # a smaller strain of the same law evaluates fine
    ok = 0.01 * ep
    sig, a_new, C = gsm.conventional_evaluate(law, np.zeros((1, 6)), np.zeros((1, 7)), ok[None], dt,
                                              want_tangent=True)
    out.update(ok_eps=ok, ok_sigma=sig[0], ok_a=a_new[0], ok_C=C[0])
    for k, v in raised.items():
        out[f"raised_{k}"] = np.array(v)
    print("radial stall:", raised)
    save("radial_stall.npz", **out)


def _path_by_hand(n, cfg, name, steps, last=None):
    """The reference's run_loading_path sequence (homogenize.py:485-528) by hand."""
    t0 = time.time()
    grid = H.toy_mmc_grid(n)
    path = H.LoadingPath(steps=steps)
    hom = H.Homogenizer(grid, cfg)
    times = path.times()
    targets = path.eps_xx(times)
    free = np.array([False, True, True, True, True, True]) if path.mixed_bc else np.zeros(6, dtype=bool)
    recs, hist, refs = [], [], [(hom.reference.lam, hom.reference.mu)]
    rng = np.random.default_rng(7)
    sub = np.sort(rng.choice(n**3, size=min(4096, n**3), replace=False))
    for k in range(1, (last or steps) + 1):
        dt = times[k] - times[k - 1]
        eb = np.zeros(6)
        eb[0] = targets[k]
        eps, sigma, info = hom.solve_step(eb, dt, free_mask=free)
        ebar = eps.mean(axis=(1, 2, 3))
        sig_bar = sigma.mean(axis=(1, 2, 3))
        _, C_vox, _, _ = hom.evaluate_field(eps, dt, want_tangent=True)
        C_bar = C_vox.mean(axis=0)
        hom.commit_step(eps, ebar)
        hom.set_reference(H.reference_update(C_vox))
        refs.append((hom.reference.lam, hom.reference.mu))
        recs.append({"step": k, "time": float(times[k]), "eps_xx": float(ebar[0]), "sig": sig_bar.copy(),
                     "C11": float(C_bar[0, 0]), "C12": float(C_bar[0, 1]), "iterations": info.iterations,
                     "mean_substeps": info.mean_substeps, "Cbar": C_bar, "ebar": ebar})
        hist.append(np.array(info.history))
        del C_vox
        arr = _records_to_arrays(recs)
        arr["Cbar"] = np.stack([r["Cbar"] for r in recs])
        arr["ebar"] = np.stack([r["ebar"] for r in recs])
        arr["history_flat"] = np.concatenate(hist)
        arr["refs"] = np.array(refs)
        arr["ids"] = grid.material_ids
        arr["sub"] = sub
        # converged fields of the last finished step, sampled
        arr["eps_sub"] = eps.reshape(6, -1)[:, sub]
        arr["sig_sub"] = sigma.reshape(6, -1)[:, sub]
        # committed matrix state (material 0, m = 7) at the sampled voxels
        st = np.zeros((n**3, grid.materials[0].m))
        st[grid.voxel_index[0]] = grid.state[0]
        arr["state_sub"] = st[sub].T.copy()
        arr["seconds"] = np.array(time.time() - t0)
        save(name, **arr)
        print(f"{name} step {k}: {info.iterations} it ({time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-slow", action="store_true")
    ap.add_argument("--only", default="")
    ap.add_argument("--path-n", type=int, default=0, help="run make_path_conv(n) only")
    args = ap.parse_args()
    if args.path_n:
        make_path_conv(args.path_n)
        sys.exit(0)
    jobs = {
        "material": make_material,
        "adaptive": make_adaptive,
        "semi": make_semi,
        "constitutive": make_constitutive,
        "lawops": make_lawops,
        "fourier": make_fourier,
        "config1": make_config1,
        "path16": make_path16_conv,
        "path8": make_path8,
        "path8_ode23": make_path8_ode23,
        "path8_ode23_fail": make_path8_ode23_fail,
        "radial": make_radial_stall,
        "tangent_singular": make_tangent_singular,
        "path32": lambda: make_path_conv(32),
        "path64": lambda: make_path_conv(64),
    }
    for name, fn in jobs.items():
        if args.only and name not in args.only.split(","):
            continue
        if args.skip_slow and name in ("path8", "path8_ode23", "path8_ode23_fail", "path32", "path64"):
            continue
        t0 = time.time()
        fn()
        print(f"[{name}] {time.time() - t0:.1f}s")
