"""Small slab-decomposed run for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): 2, 4 and 8 local slabs exercise the fused P2P
pack / unpack transposes (k_pack_peer / k_unpack_peer), the slab reductions
and the plane-ordered tangent statistics; 1 slab the 3-D cuFFT path.

usage: compute-sanitizer --tool memcheck python tools/sanitize_slabs.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04391_b200 import homogenize as H  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig  # noqa: E402

cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
for slabs in (1, 2, 4, 8):
    hom = H.Homogenizer(H.toy_mmc_grid(16), cfg, slabs=slabs)
    path = H.LoadingPath(steps=20)
    t = path.times()
    for k in range(1, int(os.environ.get("AM_SAN_STEPS", "1")) + 1):
        eb = np.zeros(6)
        eb[0] = path.eps_xx(t[k])
        eps, sig, info = hom.solve_step(eb, t[k] - t[k - 1], free_mask=np.array([False] + [True] * 5))
        _, C, _, _ = hom.evaluate_field(eps, t[k] - t[k - 1], want_tangent=True)
        hom.commit_step(eps, eps.mean(axis=(1, 2, 3)))
        hom.set_reference(H.reference_update(C))
        print(f"slabs {slabs} step {k}: {info.iterations} iterations", flush=True)
    del hom
print("SANITIZE_RUN_OK")
