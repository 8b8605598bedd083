"""Per-iteration phase times vs wall time of load step 1 at 128^3 / 256^3, cold and warm Newton start."""
import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2006_04391_b200 import _lib, homogenize as H
from paper_2006_04391_b200.evaluator import StrategyConfig
cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
lib = _lib.load()
for n in (128, 256):
  for warm in (False, True):
    hom = H.Homogenizer(H.toy_mmc_grid(n), cfg, newton_warm_start=warm)
    path = H.LoadingPath(steps=20); t = path.times()
    eb = np.zeros(6); eb[0] = path.eps_xx(t)[1]
    lib.am_solver_timing(hom._h, 1, None)
    t0 = time.perf_counter()
    info, _ = hom._solve(eb, t[1] - t[0], np.array([False] + [True] * 5))
    wall = time.perf_counter() - t0
    tm = np.zeros(5); lib.am_solver_timing(hom._h, -1, _lib.ptr(tm))
    k = tm[4]
    print(n, warm, info.iterations, f"wall/it {wall/info.iterations*1e3:.3f} ms", {"mat": round(tm[0]/k,3), "fwd": round(tm[1]/k,3), "four": round(tm[2]/k,3), "inv": round(tm[3]/(k-1),3), "sum": round((tm[0]+tm[1]+tm[2])/k + tm[3]/(k-1),3)})
