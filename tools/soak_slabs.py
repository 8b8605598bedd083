"""8-slab solvers at 256^3 (callback plans, shared cuFFT work area) created
and released three times: device memory returns to its baseline.
usage: python tools/soak_slabs.py"""
import sys; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np, torch
from paper_2006_04391_b200 import homogenize as H
from paper_2006_04391_b200.evaluator import StrategyConfig
cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
def mem(): f, t = torch.cuda.mem_get_info(); return (t - f) / 2**30
print("start", round(mem(), 2))
g = H.toy_mmc_grid(256)
for k in range(3):
    hom = H.Homogenizer(g, cfg, slabs=8, max_iterations=10)
    print("created", k, round(mem(), 2), flush=True)
    try:
        hom.solve_step(np.array([1e-4, 0, 0, 0, 0, 0]), 1.0)
    except H.SolverError:
        pass
    del hom
    print("freed", k, round(mem(), 2), flush=True)
