"""The multi-GPU slab algorithm of the basic scheme on one B200.

* local mode: k x-slabs driven from one process (2-D FFTs, all-to-all
  transposes as device copies, 1-D FFTs over x) must reproduce the
  single-slab solver: identical iteration counts, fields to round-off;
* nccl mode: the same algorithm with ncclAlltoAll / ncclAllReduce over a
  communicator (world size 1 here: the rank exchanges with itself).
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from _util import check_path_records
from conftest import ROOT, golden

pytestmark = pytest.mark.gpu


def rel(x, y):
    x, y = np.asarray(x, float), np.asarray(y, float)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300))


@pytest.fixture(scope="module")
def mods():
    from paper_2006_04391_b200 import gsm, homogenize
    from paper_2006_04391_b200.evaluator import StrategyConfig

    return gsm, homogenize, StrategyConfig(strategy="automatic", integrator="implicit-euler")


@pytest.mark.parametrize("slabs", [2, 4, 8])
def test_config1_slabs(mods, slabs):
    gsm, H, cfg = mods
    g = golden("config1.npz")
    laws = [gsm.LinearElastic(55e9, 0.33), gsm.LinearElastic(300e9, 0.25)]
    eb = np.zeros(6)
    eb[0] = 1e-3
    free = np.array([False] + [True] * 5)
    eps, sig, info = H.Homogenizer(H.VoxelGrid(g["ids"], laws), cfg, slabs=slabs).solve_step(eb, 1.0, free)
    assert info.iterations == int(g["mixed_iters"])
    assert rel(info.history, g["mixed_history"]) < 1e-8
    sub = g["sub"]
    assert rel(sig.reshape(6, -1)[:, sub], g["mixed_sig_sub"]) < 1e-10
    assert rel(eps.reshape(6, -1)[:, sub], g["mixed_eps_sub"]) < 1e-10


@pytest.mark.parametrize("slabs", [2, 4])
def test_path16_slabs(mods, slabs):
    gsm, H, cfg = mods
    g = golden("path16_conv.npz")
    recs = H.run_loading_path(H.toy_mmc_grid(16), H.LoadingPath(steps=20), cfg, slabs=slabs)
    check_path_records(recs, g, f"path16_slabs{slabs}")


def test_slabs_match_single_fields(mods):
    """Odd nz, two phases with EVP: slab runs agree with the single-slab run."""
    gsm, H, cfg = mods
    rng = np.random.default_rng(3)
    ids = (rng.random((16, 8, 7)) < 0.3).astype(np.uint8)
    laws = [gsm.MichelSuquet(), gsm.LinearElastic(300e9, 0.25)]
    res = {}
    for k in (1, 2, 4, 8):
        grid = H.VoxelGrid(ids, laws)
        hom = H.Homogenizer(grid, cfg, slabs=k)
        path = H.LoadingPath(steps=20)
        t, ex = path.times(), path.eps_xx(path.times())
        out = []
        for s in (1, 2):
            eb = np.zeros(6)
            eb[0] = ex[s]
            eps, sig, info = hom.solve_step(eb, t[s] - t[s - 1], np.array([False] + [True] * 5))
            _, C, _, _ = hom.evaluate_field(eps, t[s] - t[s - 1], want_tangent=True)
            hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
            hom.set_reference(H.reference_update(C))
            out.append((info.iterations, eps, sig, C))
        res[k] = (out, [a.copy() for a in grid.state])
    base, st0 = res[1]
    for k in (2, 4, 8):
        out, st = res[k]
        for (i0, e0, s0, c0), (i1, e1, s1, c1) in zip(base, out):
            assert i0 == i1
            assert rel(e1, e0) < 1e-12 and rel(s1, s0) < 1e-12 and rel(c1, c0) < 1e-11
        assert rel(st[0], st0[0]) < 1e-12


@pytest.mark.parametrize("transport,cb", [("p2p", "0"), ("nccl", "0"), ("p2p", "1"), ("nccl", "1")])
def test_nccl_single_rank(mods, tmp_path, transport, cb):
    """One slab per process (world 1 here): fused P2P transposes or
    ncclAlltoAll, with ncclAllReduce reductions, vs the local single-slab
    solver; cb = 1: the inverse x transform reads ehat'/N through the load
    callback (AM_FFT_CALLBACK=1)."""
    gsm, H, cfg = mods
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "recs.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "dist", "worker_gpu.py"),
           str(out), transport]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=dict(os.environ, AM_FFT_CALLBACK=cb))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    got = json.load(open(out))
    hom = H.Homogenizer(H.toy_mmc_grid(16), cfg)
    path = H.LoadingPath(steps=20)
    t, ex = path.times(), path.eps_xx(path.times())
    for k, rec in zip((1, 2, 3), got):
        eb = np.zeros(6)
        eb[0] = ex[k]
        eps, sig, info = hom.solve_step(eb, t[k] - t[k - 1], np.array([False] + [True] * 5))
        assert rec["iterations"] == info.iterations
        assert rel(rec["history"], info.history) < 1e-8
        assert abs(rec["eps_slab_sum"] - float(np.sum(eps))) <= 1e-10 * np.sum(np.abs(eps))
        if rec["sig_slab"] is not None:
            assert rel(rec["sig_slab"], sig) < 1e-10
        hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))


def test_slab_count_independent_bits(mods, parity_log):
    """With the transpose algorithm (2, 4, 8 slabs; the NCCL mode at 2, 4, 8
    GPUs runs the same kernels per slab) every reduction is fixed-order by
    global plane: records are bitwise identical across slab counts."""
    gsm, H, cfg = mods
    recs = {}
    for k in (2, 4, 8):
        r = H.run_loading_path(H.toy_mmc_grid(16), H.LoadingPath(steps=3), cfg, slabs=k)
        recs[k] = [(x["iterations"], x["eps_xx"], tuple(x["sig"]), x["C11"], x["C12"]) for x in r]
    same = {k: recs[k] == recs[2] for k in (4, 8)}
    parity_log("slab_bits", **{f"slabs{k}_equal_to_2": v for k, v in same.items()})
    assert all(same.values()), recs


@pytest.mark.parametrize("cb", ["0", "1"])
@pytest.mark.parametrize("slabs", [2, 4])
def test_local_alltoall_transport_bitwise(mods, slabs, cb):
    """The NCCL transport's data layout with more than one slab, on one GPU:
    AM_LOCAL_ALLTOALL=1 sends the local slabs' transposes through the
    all-to-all buffers (device copies in place of ncclAlltoAll; with
    AM_FFT_CALLBACK=1 the 2-D transforms' callbacks write / read those
    buffers).  Fields and histories are bitwise those of the sibling-P2P
    transposes (pure data movement)."""
    gsm, H, cfg = mods
    out = []
    for lt in ("0", "1"):
        os.environ["AM_LOCAL_ALLTOALL"] = lt
        os.environ["AM_FFT_CALLBACK"] = cb
        try:
            hom = H.Homogenizer(H.toy_mmc_grid(16), cfg, slabs=slabs)
        finally:
            os.environ.pop("AM_LOCAL_ALLTOALL", None)
            os.environ.pop("AM_FFT_CALLBACK", None)
        path = H.LoadingPath(steps=20)
        t = path.times()
        res = []
        for k in (1, 2):
            eb = np.zeros(6)
            eb[0] = path.eps_xx(t[k])
            eps, sig, info = hom.solve_step(eb, t[k] - t[k - 1], free_mask=np.array([False] + [True] * 5))
            res.append((eps, sig, info.history))
            hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
        out.append(res)
    for (e0, s0, h0), (e1, s1, h1) in zip(*out):
        assert np.array_equal(e0, e1) and np.array_equal(s0, s1) and h0 == h1


def test_callbacks_bitwise_at_256(mods):
    """Config-4 grid on 8 slabs, the first 6 iterations of load step 1 with
    the cuFFT callbacks (default at 256^3: inverse x transform loading
    ehat'/N, sigma's transposes inside the 2-D transforms) and without
    (AM_FFT_CALLBACK=0: scaled copy, pack / unpack kernels): residual
    histories, strain and stress fields bitwise equal."""
    import ctypes

    gsm, H, cfg = mods
    grid = H.toy_mmc_grid(256)
    path = H.LoadingPath(steps=20)
    t = path.times()
    eb = np.zeros(6)
    eb[0] = path.eps_xx(t[1])
    out = []
    for cb in ("0", "1"):
        os.environ["AM_FFT_CALLBACK"] = cb
        try:
            hom = H.Homogenizer(grid, cfg, slabs=8, max_iterations=6)
        finally:
            os.environ.pop("AM_FFT_CALLBACK", None)
        on = ctypes.c_int(-1)
        hom._lib.am_solver_fft_callback(hom._h, ctypes.byref(on))
        assert on.value == (3 if cb == "1" else 0)
        with pytest.raises(H.SolverError) as exc:
            hom._solve(eb, t[1] - t[0], np.array([False] + [True] * 5))
        out.append((exc.value.history, hom._get(0), hom._get(2)))
        del hom
    (h0, e0, s0), (h1, e1, s1) = out
    assert h0 == h1 and np.array_equal(e0, e1) and np.array_equal(s0, s1)
