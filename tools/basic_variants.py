"""Per-phase basic-scheme timing (load step 1, toy_mmc_grid(n)) for libautomat variants.

usage (GPU box): python tools/basic_variants.py [n] [max_iterations] [cold|warm]
Also prints the Newton-iteration histogram of the converged sweep.
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    os.environ["AM_LIB"] = sys.argv[2]
    n, its = int(sys.argv[3]), int(sys.argv[4])
    warm = len(sys.argv) > 5 and sys.argv[5] == "warm"
    sys.path.insert(0, ROOT)
    import numpy as np

    from paper_2006_04391_b200 import _lib, homogenize as H
    from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays

    cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
    grid = H.toy_mmc_grid(n)
    hom = H.Homogenizer(grid, cfg, max_iterations=its, newton_warm_start=warm)
    lib = _lib.load()
    _lib.check(lib.am_solver_timing(hom._h, 1, None))
    path = H.LoadingPath(steps=20)
    t = path.times()
    eb = np.zeros(6)
    eb[0] = path.eps_xx(t)[1]
    try:
        info, hist = hom._solve(eb, t[1] - t[0], np.array([False] + [True] * 5))
        it = info.iterations
    except H.SolverError as e:
        it = len(e.history)
    ph = np.zeros(5)
    _lib.check(lib.am_solver_timing(hom._h, -1, _lib.ptr(ph)))
    k = max(ph[4], 1)
    out = {"iterations": it, "material": ph[0] / k, "fwd": ph[1] / k, "fourier": ph[2] / k, "inv": ph[3] / max(k - 1, 1)}
    # Newton counts of the last sweep on a sample of the matrix voxels
    eps = hom._get(0).reshape(6, -1)
    idx = grid.voxel_index[0][:: max(1, len(grid.voxel_index[0]) // 200000)]
    r = evaluate_arrays(grid.materials[0], cfg, np.zeros((len(idx), 6)), np.zeros((len(idx), 7)), eps[:, idx].T,
                        t[1] - t[0])
    h = np.bincount(r.newton_iters)
    print(os.path.basename(os.path.dirname(sys.argv[2])), {k: round(v, 3) if isinstance(v, float) else v
                                                           for k, v in out.items()},
          "newton hist", h.tolist(), "mean", round(float(r.newton_iters.mean()), 3), flush=True)
else:
    n = sys.argv[1] if len(sys.argv) > 1 else "256"
    its = sys.argv[2] if len(sys.argv) > 2 else "5000"
    mode = sys.argv[3] if len(sys.argv) > 3 else "cold"
    libs = [os.path.join(ROOT, "paper_2006_04391_b200", "libautomat.so")]
    libs += sorted(glob.glob(os.path.join(ROOT, "tools", "variants", "*", "libautomat.so")))
    for lib in libs:
        subprocess.run([sys.executable, __file__, "--one", lib, n, its, mode], check=False)
