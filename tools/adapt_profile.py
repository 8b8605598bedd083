"""Coupled adaptive route on the config-2 batch (default StrategyConfig():
automatic ode23, stress + tangent), for ncu captures of k_adaptive*.
usage: python tools/adapt_profile.py [B] [integrator]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04391_b200 import gsm  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays  # noqa: E402
from paper_2006_04391_b200.workloads import config2_batch  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 17
integ = sys.argv[2] if len(sys.argv) > 2 else "ode23"
en, an, ep, dt = config2_batch(B)
r = evaluate_arrays(gsm.MichelSuquet(), StrategyConfig(integrator=integ), en, an, ep, dt, want_tangent=True)
print(integ, "mean substeps", float(r.substeps.mean()), "rejected", float(r.rejected.mean()))
