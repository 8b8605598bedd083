"""Scaled-down Fig. 7 / Fig. 8 of the paper (SPEC.md acceptance criteria 6
and 7) on the device: the 16^3 toy MMC loading path with implicit Euler,
ode12, ode23 and ode23s (semi-automatic), at several step counts; prints
per-run iterations, wall time and the sigma_bar_xx series as JSON lines.
usage: python tools/spec_fig7_probe.py [n] [steps,...] [error_measure]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04391_b200 import homogenize as H  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
steps = [int(s) for s in sys.argv[2].split(",")] if len(sys.argv) > 2 else [20, 80]
measure = sys.argv[3] if len(sys.argv) > 3 else "internal"
routes = [("automatic", "implicit-euler"), ("automatic", "ode12"), ("automatic", "ode23"), ("semi-automatic", "ode23s")]
for st in steps:
    for strat, integ in routes:
        cfg = StrategyConfig(strategy=strat, integrator=integ, error_measure=measure)
        t0 = time.perf_counter()
        try:
            recs = H.run_loading_path(H.toy_mmc_grid(n), H.LoadingPath(steps=st), cfg)
            out = {"iterations": [r["iterations"] for r in recs], "sig_xx": [float(r["sig"][0]) for r in recs],
                   "mean_substeps": [r["mean_substeps"] for r in recs]}
        except Exception as exc:  # noqa: BLE001
            out = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
        print(json.dumps({"n": n, "steps": st, "integrator": integ, "strategy": strat, "measure": measure,
                          "seconds": round(time.perf_counter() - t0, 2), **out}), flush=True)
