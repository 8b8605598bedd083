"""Config-3 loading path at n^3: per-step wall time of the basic scheme, the
tangent sweep (+ reference update) and the commit, and the solver's phase
times, to locate the time outside the basic-scheme iterations.

usage: python tools/path_probe.py [n] [warm]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04391_b200 import _lib, homogenize as H  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
warm = len(sys.argv) > 2 and sys.argv[2] == "warm"
cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
hom = H.Homogenizer(H.toy_mmc_grid(n), cfg, newton_warm_start=warm)
lib = hom._lib
path = H.LoadingPath(steps=20)
times = path.times()
targets = path.eps_xx(times)
free = np.array([False] + [True] * 5)
Cbar, lam_mu = np.zeros(36), np.zeros(2)
tot = {"solve": 0.0, "sweep": 0.0, "commit": 0.0}
its = 0
lib.am_solver_timing(hom._h, 1, None)
for k in range(1, len(times)):
    dt = times[k] - times[k - 1]
    tgt = np.zeros(6)
    tgt[0] = targets[k]
    t0 = time.perf_counter()
    info, _ = hom._solve(tgt, dt, free)
    t1 = time.perf_counter()
    _lib.check(lib.am_solver_tangent_sweep(hom._h, float(dt), _lib.ptr(Cbar), _lib.ptr(lam_mu), None))
    t2 = time.perf_counter()
    ebar = np.array(info.ebar[:])
    _lib.check(lib.am_solver_commit(hom._h, _lib.ptr(ebar)))
    hom.set_reference(H.ReferenceMaterial(lam=float(lam_mu[0]), mu=float(lam_mu[1])))
    t3 = time.perf_counter()
    tot["solve"] += t1 - t0
    tot["sweep"] += t2 - t1
    tot["commit"] += t3 - t2
    its += info.iterations
    print(k, info.iterations, f"solve {1e3 * (t1 - t0):.1f} ms ({1e3 * (t1 - t0) / info.iterations:.3f}/it) "
          f"sweep {1e3 * (t2 - t1):.1f} ms commit+ref {1e3 * (t3 - t2):.1f} ms", flush=True)
ph = np.zeros(5)
lib.am_solver_timing(hom._h, -1, _lib.ptr(ph))
print("total", its, {k: round(v, 3) for k, v in tot.items()},
      "phase ms/it", [round(x / ph[4], 3) for x in ph[:4]])
