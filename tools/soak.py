import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2006_04391_b200 import gsm, homogenize as H
from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays
from paper_2006_04391_b200.workloads import config2_batch
cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
def mem(): f, t = torch.cuda.mem_get_info(); return (t - f) / 2**30
print("start", round(mem(), 2))
for k in range(3):
    recs = H.run_loading_path(H.toy_mmc_grid(128), H.LoadingPath(steps=20), cfg)
    print("path", k, sum(r["iterations"] for r in recs), round(mem(), 2), flush=True)
en, an, ep, dt = config2_batch(1 << 20)
for k in range(10):
    r = evaluate_arrays(gsm.MichelSuquet(), cfg, en, an, ep, dt, want_tangent=True)
print("eval", round(mem(), 2))
import psutil; print("host rss GB", round(psutil.Process().memory_info().rss / 2**30, 2))
