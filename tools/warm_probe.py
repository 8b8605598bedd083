"""Newton warm start inside the basic scheme (am_solver_set_warm_start):
iteration counts, macroscopic results and time, cold vs warm.

usage: python tools/warm_probe.py [n_path] [n_step1]
  config-3-like loading path at n_path^3 (20 steps, reference update), then
  load step 1 at n_step1^3 with per-phase timing.
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04391_b200 import _lib, homogenize as H  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig  # noqa: E402

n_path = int(sys.argv[1]) if len(sys.argv) > 1 else 128
n_step = int(sys.argv[2]) if len(sys.argv) > 2 else 256
cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
lib = _lib.load()
out = {}
for warm in (False, True):
    tag = "warm" if warm else "cold"
    r = {}
    if n_path:
        H.run_loading_path(H.toy_mmc_grid(32), H.LoadingPath(steps=2), cfg, newton_warm_start=warm)  # warm-up
        grid = H.toy_mmc_grid(n_path)
        t0 = time.perf_counter()
        recs = H.run_loading_path(grid, H.LoadingPath(steps=20), cfg, newton_warm_start=warm)
        r["path_seconds"] = time.perf_counter() - t0
        r["path_iterations"] = [int(x["iterations"]) for x in recs]
        r["path_sig_xx"] = [float(x["sig"][0]) for x in recs]
        r["path_C11"] = [float(x["C11"]) for x in recs]
        print(tag, "path", sum(r["path_iterations"]), f"{r['path_seconds']:.3f}s", flush=True)
    if n_step:
        hom = H.Homogenizer(H.toy_mmc_grid(n_step), cfg, newton_warm_start=warm)
        path = H.LoadingPath(steps=20)
        t = path.times()
        eb = np.zeros(6)
        eb[0] = path.eps_xx(t)[1]
        lib.am_solver_timing(hom._h, 1, None)
        eps, sig, info = hom.solve_step(eb, t[1] - t[0], free_mask=np.array([False] + [True] * 5))
        tm = np.zeros(5)
        lib.am_solver_timing(hom._h, -1, _lib.ptr(tm))
        r["step1_iterations"] = int(info.iterations)
        r["step1_ms_per_it"] = {"material": tm[0] / tm[4], "d2z": tm[1] / tm[4], "fourier": tm[2] / tm[4],
                                "z2d": tm[3] / tm[4]}
        r["step1_sig_bar"] = [float(x) for x in sig.reshape(6, -1).mean(axis=1)]
        np.save(f"/tmp/warm_sig_{tag}.npy", sig[:, ::4, ::4, ::4])
        print(tag, "step1", info.iterations, r["step1_ms_per_it"], flush=True)
        del hom
    out[tag] = r
c, w = out["cold"], out["warm"]
if n_path:
    print("path iterations identical:", c["path_iterations"] == w["path_iterations"])
    print("path max rel sig_xx diff:", max(abs(a - b) / abs(a) for a, b in zip(c["path_sig_xx"], w["path_sig_xx"])))
    print("path max rel C11 diff:", max(abs(a - b) / abs(a) for a, b in zip(c["path_C11"], w["path_C11"])))
if n_step:
    sc, sw = np.load("/tmp/warm_sig_cold.npy"), np.load("/tmp/warm_sig_warm.npy")
    print("step1 iterations", c["step1_iterations"], w["step1_iterations"],
          "sigma field rel diff", float(np.abs(sc - sw).max() / np.abs(sc).max()))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/warm_probe.json", "w"), indent=1)
