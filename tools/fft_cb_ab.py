"""A/B of the inverse transform's load callback (AM_FFT_CALLBACK=0 / 1) on
the config-4 grid, load step 1: graph-replayed iterations/s (alternating
runs) and the eager phase split.  usage: python tools/fft_cb_ab.py [n] [reps]"""
import ctypes
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2006_04391_b200 import _lib, homogenize as H  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
path = H.LoadingPath(steps=20)
t = path.times()
eb = np.zeros(6)
eb[0] = path.eps_xx(t[1])
free = np.array([False] + [True] * 5)
lib = _lib.load()
out = {"n": n}
for rep in range(reps):
    for cb in ("0", "1"):
        os.environ["AM_FFT_CALLBACK"] = cb
        hom = H.Homogenizer(H.toy_mmc_grid(n), cfg)
        on = ctypes.c_int(-1)
        lib.am_solver_fft_callback(hom._h, ctypes.byref(on))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        info, _ = hom._solve(eb, t[1] - t[0], free)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        out.setdefault(f"cb{cb}", []).append({"on": on.value, "iterations": info.iterations,
                                              "ms_per_it": 1e3 * wall / info.iterations})
        if rep == 0:  # eager phase split
            _lib.check(lib.am_solver_timing(hom._h, 1, None))
            hom2 = hom
            info, _ = hom2._solve(eb, t[1] - t[0], free)
            ph = np.zeros(5)
            _lib.check(lib.am_solver_timing(hom._h, -1, _lib.ptr(ph)))
            k = ph[4]
            out[f"cb{cb}_phases_ms"] = {"material": ph[0] / k, "d2z": ph[1] / k, "fourier": ph[2] / k,
                                        "z2d": ph[3] / max(k - 1, 1)}
        del hom
print(json.dumps(out))
