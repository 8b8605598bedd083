"""Uncoupled (no tangent) and coupled ode23 / implicit Euler on the config-2
batch, device-resident: the default StrategyConfig() inside the basic scheme
evaluates without tangent.  usage: python tools/ode23_probe.py [B]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2006_04391_b200 import _lib, gsm  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig  # noqa: E402
from paper_2006_04391_b200.workloads import config2_batch  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
lib = _lib.load()
law = _lib.make_law(gsm.MichelSuquet())
en, an, ep, dt = config2_batch(B)
dev = torch.device("cuda:0")
t = lambda x: torch.from_numpy(np.ascontiguousarray(x.T)).to(dev)  # noqa: E731
d_en, d_an, d_ep = t(en), t(an), t(ep)
d_sig = torch.empty((6, B), dtype=torch.float64, device=dev)
d_a = torch.empty((7, B), dtype=torch.float64, device=dev)
d_C = torch.empty((36, B), dtype=torch.float64, device=dev)
d_it = torch.empty(B, dtype=torch.int32, device=dev)
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for integ in ("implicit-euler", "ode23", "ode12"):
    for tang in (0, 1):
        cfg = _lib.make_cfg(StrategyConfig(integrator=integ))

        def run():
            _lib.check(lib.am_eval_batch(law, cfg, B, d_en.data_ptr(), d_an.data_ptr(), d_ep.data_ptr(), None, 0.05,
                                         tang, d_sig.data_ptr(), d_a.data_ptr(), d_C.data_ptr(), d_it.data_ptr(),
                                         None, None, None, sp))

        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{integ:15s} tangent={tang}: {B / ms / 1e3:.3g} M evals/s ({ms:.2f} ms)", flush=True)
