"""Host-entry paths for compute-sanitizer: pageable / pinned inputs and
outputs through am_eval_batch_host (several chunks), evaluate_arrays with
pooled results, every strategy / integrator on a small batch.
usage: compute-sanitizer --tool memcheck python tools/sanitize_host.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04391_b200 import gsm  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays  # noqa: E402
from paper_2006_04391_b200.workloads import config2_batch  # noqa: E402

en, an, ep, dt = config2_batch(20000, seed=2)
law = gsm.MichelSuquet()
for strat, integ in (("automatic", "implicit-euler"), ("semi-automatic", "implicit-euler"),
                     ("conventional", "implicit-euler"), ("automatic", "ode23"), ("automatic", "ode12"),
                     ("semi-automatic", "ode23s")):
    n = 20000 if integ == "implicit-euler" else 500
    for tang in (False, True):
        r = evaluate_arrays(law, StrategyConfig(strategy=strat, integrator=integ), en[:n], an[:n], ep[:n], dt[:n],
                            want_tangent=tang)
        assert np.all(np.isfinite(r.sigma))
r = evaluate_arrays(gsm.LinearElastic(300e9, 0.25), StrategyConfig(), en, np.zeros((len(en), 0)), ep, dt, True)
print("SANITIZE_HOST_OK")
