"""Dump run_loading_path records (toy_mmc_grid(n), 20 steps, automatic
implicit Euler) for comparison with the reference's per-law conventional
fixtures (tests/golden/path{n}_conv.npz).

usage: python tools/path_records.py out.npz n [n ...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04391_b200 import homogenize as H  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig  # noqa: E402

out = {}
cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
for n in map(int, sys.argv[2:]):
    t0 = time.perf_counter()
    recs = H.run_loading_path(H.toy_mmc_grid(n), H.LoadingPath(steps=20), cfg)
    out[f"n{n}_iterations"] = np.array([r["iterations"] for r in recs])
    out[f"n{n}_sig"] = np.stack([r["sig"] for r in recs])
    out[f"n{n}_eps_xx"] = np.array([r["eps_xx"] for r in recs])
    out[f"n{n}_C11"] = np.array([r["C11"] for r in recs])
    out[f"n{n}_C12"] = np.array([r["C12"] for r in recs])
    print(n, f"{time.perf_counter() - t0:.1f}s", out[f"n{n}_iterations"].tolist(), flush=True)
    np.savez(sys.argv[1], **out)
