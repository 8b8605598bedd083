"""Where the end-to-end time of the host entry goes (config 2, 2^20 points):
evaluate_arrays vs am_eval_batch_host with pinned / pageable inputs and
outputs, plain host memcpy rates, and the pinned pool's behaviour.

usage: python tools/e2e_probe.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2006_04391_b200 import _lib, gsm  # noqa: E402
from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays  # noqa: E402
from paper_2006_04391_b200.workloads import config2_batch  # noqa: E402

B = 1 << 20
lib = _lib.load()
law, cfg = gsm.MichelSuquet(), StrategyConfig(strategy="automatic", integrator="implicit-euler")
sl, sc = _lib.make_law(law), _lib.make_cfg(cfg)
en, an, ep, dt = config2_batch(B)


def timeit(fn, n=5):
    fn()
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e3


pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
pinned_in = tuple(pin(x) for x in (en, an, ep, dt))
outs_pin = [torch.empty(s, dtype=torch.float64).pin_memory().numpy() for s in ((B, 6), (B, 7), (B, 6, 6))]
it_pin = torch.empty(B, dtype=torch.int32).pin_memory().numpy()
outs_pg = [np.empty(s) for s in ((B, 6), (B, 7), (B, 6, 6))]
it_pg = np.empty(B, dtype=np.int32)
for o in outs_pg:
    o.fill(0)


def abi(inputs, outs, it):
    _lib.check(lib.am_eval_batch_host(sl, sc, B, *[_lib.ptr(x) for x in inputs], 1, *[_lib.ptr(o) for o in outs],
                                      _lib.ptr(it, _lib._i32p), None, None))


res = {}
res["abi pinned in / pinned out"] = timeit(lambda: abi(pinned_in, outs_pin, it_pin))
res["abi pageable in / pinned out"] = timeit(lambda: abi((en, an, ep, dt), outs_pin, it_pin))
res["abi pinned in / pageable out"] = timeit(lambda: abi(pinned_in, outs_pg, it_pg))
res["abi pageable in / pageable out"] = timeit(lambda: abi((en, an, ep, dt), outs_pg, it_pg))
res["evaluate_arrays"] = timeit(lambda: evaluate_arrays(law, cfg, en, an, ep, dt, want_tangent=True))
r = None


def ev_keep():
    global r
    r = evaluate_arrays(law, cfg, en, an, ep, dt, want_tangent=True)


res["evaluate_arrays (result kept across calls)"] = timeit(ev_keep)
# host memcpy rates (single thread, numpy) pageable -> pinned
dst = torch.empty(B * 20, dtype=torch.float64).pin_memory().numpy()
src = np.random.default_rng(0).random(B * 20)
res["numpy copy 160 MiB pageable->pinned (1 thread)"] = timeit(lambda: np.copyto(dst, src))
res["pinned_empty 4 arrays"] = timeit(lambda: [_lib.pinned_empty(s) for s in ((B, 6), (B, 7), (B, 6, 6), (B,))])
for k, v in res.items():
    print(f"{k:55s} {v:8.2f} ms  ({B / v / 1e3:.3g} evals/s)")
print("cpu count", os.cpu_count())
