"""Two evaluations of 2^18 config-2 points (stress + tangent) for ncu.

usage: python tools/semi_profile.py [strategy] [integrator]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04391_b200 import gsm  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays  # noqa: E402
from paper_2006_04391_b200.workloads import config2_batch  # noqa: E402

strategy = sys.argv[1] if len(sys.argv) > 1 else "semi-automatic"
en, an, ep, dt = config2_batch(1 << 18)
integrator = sys.argv[2] if len(sys.argv) > 2 else "implicit-euler"
cfg = StrategyConfig(strategy=strategy, integrator=integrator)
for _ in range(2):
    evaluate_arrays(gsm.MichelSuquet(), cfg, en, an, ep, dt, want_tangent=True)
