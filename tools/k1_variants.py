"""Time K1 variants (tools/variants/*/libautomat.so) on the config-2 batch.

usage (GPU box): python tools/k1_variants.py [B]
Prints evals/s with and without tangent per variant, device-resident inputs.
"""
import ctypes
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    os.environ["AM_LIB"] = sys.argv[2]
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    from paper_2006_04391_b200 import _lib, gsm
    from paper_2006_04391_b200.evaluator import StrategyConfig
    from paper_2006_04391_b200.workloads import config2_batch

    B = int(sys.argv[3])
    lib = _lib.load()
    law = _lib.make_law(gsm.MichelSuquet())
    out = {}
    for mode in ("internal", "stress"):
        cfg = _lib.make_cfg(StrategyConfig(strategy="automatic", integrator="implicit-euler", error_measure=mode))
        en, an, ep, dt = config2_batch(B, seed=0)
        dev = torch.device("cuda:0")
        soa = lambda x: torch.from_numpy(np.ascontiguousarray(x.T)).to(dev)  # noqa: E731
        d_en, d_an, d_ep = soa(en), soa(an), soa(ep)
        d_sig = torch.empty((6, B), dtype=torch.float64, device=dev)
        d_a = torch.empty((7, B), dtype=torch.float64, device=dev)
        d_C = torch.empty((36, B), dtype=torch.float64, device=dev)
        d_it = torch.empty(B, dtype=torch.int32, device=dev)
        for tang in ((0, 1) if mode == "internal" else (0,)):
            def step():
                _lib.check(lib.am_eval_batch(law, cfg, B, d_en.data_ptr(), d_an.data_ptr(), d_ep.data_ptr(), None,
                                             0.05, tang, d_sig.data_ptr(), d_a.data_ptr(),
                                             d_C.data_ptr() if tang else None, d_it.data_ptr(), None, None, None, None))
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                step()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            out[f"{mode}{'+C' if tang else ''}"] = f"{B / ms / 1e6:.1f} M/s ({ms:.3f} ms)"
    print(os.path.basename(os.path.dirname(sys.argv[2])), out, flush=True)
else:
    B = sys.argv[1] if len(sys.argv) > 1 else str(1 << 20)
    libs = sorted(glob.glob(os.path.join(ROOT, "tools", "variants", "*", "libautomat.so")))
    libs.insert(0, os.path.join(ROOT, "paper_2006_04391_b200", "libautomat.so"))
    for lib in libs:
        subprocess.run([sys.executable, __file__, "--one", lib, B], check=False)
