"""A few basic-scheme iterations at n^3 for ncu (launch list / full capture).

usage: python tools/basic_profile.py [n] [iterations] [warm|cold] [slabs]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04391_b200 import homogenize as H  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
its = int(sys.argv[2]) if len(sys.argv) > 2 else 3
warm = len(sys.argv) > 3 and sys.argv[3] == "warm"
slabs = int(sys.argv[4]) if len(sys.argv) > 4 else 1
hom = H.Homogenizer(H.toy_mmc_grid(n), StrategyConfig(strategy="automatic", integrator="implicit-euler"),
                    max_iterations=its, newton_warm_start=warm, slabs=slabs)
path = H.LoadingPath(steps=20)
t = path.times()
eb = np.zeros(6)
eb[0] = path.eps_xx(t)[1]
try:
    hom.solve_step(eb, t[1] - t[0], free_mask=np.array([False] + [True] * 5))
except H.SolverError as e:
    print("stopped after", len(e.history), "iterations:", e.history)
