"""Per-step basic-scheme iterations of the n^3 loading path, cold vs Newton warm start.
usage: python tools/warm_path.py n"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04391_b200 import homogenize as H  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
for warm in (False, True):
    recs = H.run_loading_path(H.toy_mmc_grid(n), H.LoadingPath(steps=20), cfg, newton_warm_start=warm)
    print("warm" if warm else "cold", [r["iterations"] for r in recs], sum(r["iterations"] for r in recs), flush=True)
