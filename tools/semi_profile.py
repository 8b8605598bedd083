"""One semi-automatic implicit-Euler evaluation of 2^18 config-2 points (stress + tangent) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04391_b200 import gsm  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays  # noqa: E402
from paper_2006_04391_b200.workloads import config2_batch  # noqa: E402

strategy = sys.argv[1] if len(sys.argv) > 1 else "semi-automatic"
en, an, ep, dt = config2_batch(1 << 18)
cfg = StrategyConfig(strategy=strategy, integrator="implicit-euler")
for _ in range(2):
    evaluate_arrays(gsm.MichelSuquet(), cfg, en, an, ep, dt, want_tangent=True)
