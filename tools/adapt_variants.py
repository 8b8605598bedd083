"""Device-resident timing of the coupled adaptive routes (config-2 batch,
stress + tangent) for libautomat variants (tools/variants/*/libautomat.so).
usage (GPU box): python tools/adapt_variants.py [B]"""
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
    en, an, ep, dt = config2_batch(B, seed=0)
    dev = torch.device("cuda:0")
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x.T)).to(dev)  # noqa: E731
    d_en, d_an, d_ep = t(en), t(an), t(ep)
    d_sig = torch.empty((6, B), dtype=torch.float64, device=dev)
    d_a = torch.empty((7, B), dtype=torch.float64, device=dev)
    d_C = torch.empty((36, B), dtype=torch.float64, device=dev)
    d_it = torch.empty(B, dtype=torch.int32, device=dev)
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    out = {}
    for integ, meas, strat in (("ode23", "internal", "automatic"), ("ode12", "internal", "automatic"),
                               ("ode23", "stress", "automatic"), ("ode23s", "internal", "semi-automatic"),
                               ("ode23s", "stress", "semi-automatic")):
        cfg = _lib.make_cfg(StrategyConfig(strategy=strat, integrator=integ, error_measure=meas))

        def run():
            _lib.check(lib.am_eval_batch(law, cfg, B, d_en.data_ptr(), d_an.data_ptr(), d_ep.data_ptr(), None, 0.05, 1,
                                         d_sig.data_ptr(), d_a.data_ptr(), d_C.data_ptr(), d_it.data_ptr(), None, None,
                                         None, sp))

        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        out[f"{strat[:4]}/{integ}/{meas}"] = f"{B / ms / 1e3:.3g} M/s ({ms:.2f} ms, substeps {d_it.double().mean().item():.2f})"
    print(os.path.basename(os.path.dirname(sys.argv[2])), out, flush=True)
else:
    B = sys.argv[1] if len(sys.argv) > 1 else str(1 << 18)
    libs = [os.path.join(ROOT, "paper_2006_04391_b200", "libautomat.so")]
    libs += sorted(glob.glob(os.path.join(ROOT, "tools", "variants", "*", "libautomat.so")))
    for lib in libs:
        subprocess.run([sys.executable, __file__, "--one", lib, B], check=False)
