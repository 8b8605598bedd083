"""Config 5 on one GPU: 512^3 high-contrast composite (fibre E = 3000 GPa,
SURVEY.md §8d), load step 1 of LoadingPath(steps=20), device memory and
basic-scheme iterations/s.  usage: python tools/config5_probe.py [n] [warm|cold] [max_iterations]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2006_04391_b200 import _lib, gsm, homogenize as H  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
warm = len(sys.argv) > 2 and sys.argv[2] == "warm"
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 5000
t0 = time.perf_counter()
grid = H.toy_mmc_grid(n, fiber_law=gsm.LinearElastic(3000e9, 0.25))
t_geo = time.perf_counter() - t0
free0, total = torch.cuda.mem_get_info()
hom = H.Homogenizer(grid, StrategyConfig(strategy="automatic", integrator="implicit-euler"), newton_warm_start=warm,
                    max_iterations=cap)
free1, _ = torch.cuda.mem_get_info()
lib = _lib.load()
_lib.check(lib.am_solver_timing(hom._h, 1, None))
path = H.LoadingPath(steps=20)
t = path.times()
eb = np.zeros(6)
eb[0] = path.eps_xx(t)[1]
torch.cuda.synchronize()
t0 = time.perf_counter()
try:
    info, hist = hom._solve(eb, t[1] - t[0], np.array([False] + [True] * 5))
    its, res, sbar = info.iterations, info.residual, list(info.sig_bar)
except H.SolverError as exc:  # max_iterations cap: a per-iteration rate
    its, res, sbar = len(exc.history), exc.history[-1], None
torch.cuda.synchronize()
wall = time.perf_counter() - t0
ph = np.zeros(5)
_lib.check(lib.am_solver_timing(hom._h, -1, _lib.ptr(ph)))
k = ph[4]
print(json.dumps({
    "grid": n, "voxels": n ** 3, "newton_warm_start": warm, "fibre": "LinearElastic(3000e9, 0.25)", "geometry_s": round(t_geo, 2),
    "device_bytes_solver": int(free0 - free1), "device_total": int(total),
    "iterations": its, "capped": its >= cap, "seconds": wall, "it_per_s": its / wall,
    "phase_ms_per_iteration": {"material": ph[0] / k, "d2z": ph[1] / k, "fourier": ph[2] / k,
                               "z2d": ph[3] / max(k - 1, 1)},
    "sig_bar": sbar, "residual": res,
}))
