"""e2e (host AoS arrays through am_eval_batch_host) timing of libautomat variants.
usage (GPU box): python tools/e2e_variants.py"""
import glob
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    os.environ["AM_LIB"] = sys.argv[2]
    sys.path.insert(0, ROOT)
    import torch

    from paper_2006_04391_b200 import _lib, gsm
    from paper_2006_04391_b200.evaluator import StrategyConfig
    from paper_2006_04391_b200.workloads import config2_batch

    B = 1 << 20
    lib = _lib.load()
    law = _lib.make_law(gsm.MichelSuquet())
    cfg = _lib.make_cfg(StrategyConfig(strategy="automatic", integrator="implicit-euler"))
    en, an, ep, dt = config2_batch(B)
    pin = lambda shape, dtype=torch.float64: torch.empty(shape, dtype=dtype, pin_memory=True).numpy()  # noqa: E731
    h = [pin((B, 6)), pin((B, 7)), pin((B, 6)), pin((B,))]
    h[0][:], h[1][:], h[2][:], h[3][:] = en, an, ep, dt
    o = [pin((B, 6)), pin((B, 7)), pin((B, 6, 6)), pin((B,), torch.int32)]

    def step():
        _lib.check(lib.am_eval_batch_host(law, cfg, B, *[_lib.ptr(x) for x in h], 1, _lib.ptr(o[0]), _lib.ptr(o[1]),
                                          _lib.ptr(o[2]), _lib.ptr(o[3], _lib._i32p), None, None))

    for _ in range(2):
        step()
    t0 = time.perf_counter()
    for _ in range(5):
        step()
    ms = (time.perf_counter() - t0) / 5 * 1e3
    print(os.path.basename(os.path.dirname(sys.argv[2])), f"{ms:.3f} ms, {B / ms / 1e3:.3e} evals/s", flush=True)
elif len(sys.argv) > 1 and sys.argv[1] == "--bw":
    # raw pinned-host <-> device copy bandwidth: the ceiling of the e2e path
    import torch

    B = 1 << 20
    hin = torch.empty(B * 20, dtype=torch.float64, pin_memory=True)
    hout = torch.empty(B * 50, dtype=torch.float64, pin_memory=True)
    din = torch.empty_like(hin, device="cuda")
    dout = torch.empty_like(hout, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name, fn in (("h2d 168 MB", lambda: din.copy_(hin, non_blocking=True)),
                     ("d2h 419 MB", lambda: hout.copy_(dout, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        nb = (hin if name.startswith("h2d") else hout).numel() * 8
        print(name, f"{nb / dt / 1e9:.1f} GB/s", flush=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1):
            din.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(dout, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"concurrent h2d+d2h: {dt * 1e3:.2f} ms per (168 + 419) MB -> e2e ceiling {B / dt:.3e} evals/s", flush=True)
else:
    libs = [os.path.join(ROOT, "paper_2006_04391_b200", "libautomat.so")]
    libs += sorted(glob.glob(os.path.join(ROOT, "tools", "variants", "*", "libautomat.so")))
    for lib in libs:
        subprocess.run([sys.executable, __file__, "--one", lib], check=False)
