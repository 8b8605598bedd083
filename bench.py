"""Benchmark: voxel stress + AD-tangent evaluations per second (fp64) on B200.

Workload (BASELINE.json configs[1]): 2^20 independent elasto-viscoplastic
(Michel-Suquet, Table-1) material points per GPU, random strain increments
(SURVEY.md §8d generator), automatic strategy, implicit Euler, stress +
second-order AD consistent tangent.  One step = one material evaluation of
the whole batch.  Multi-GPU: one process per GPU, each rank evaluates its own
2^20 points (weak scaling, no data-path collective -- the material points are
independent); the step time is the max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--impl reference`` times the reference algorithm's CPU implementation
(the C restatement in oracle/, all host threads) on a bounded sample of the
same workload.
"""

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "voxel stress+tangent evals/sec (fp64) and basic-scheme iterations/sec at 256³"
UNIT = "evals/s"
B_DEFAULT = 1 << 20


def flops_per_eval(iters, tangent=True):
    """Algorithmic fp64 flops of one evaluation: 1072 per Newton
    iteration + 2273 for the tangent post-process, stress and tangent
    (+38 without tangent)."""
    return 1072.0 * iters + (2273.0 if tangent else 38.0)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_rate(B, threads, seed=0):
    """evals/s of the C oracle (reference algorithm) on a B-point sample."""
    from oracle import material as OM
    from paper_2006_04391_b200.workloads import config2_batch

    en, an, ep, dt = config2_batch(B, seed=seed)
    t0 = time.perf_counter()
    OM.evaluate(OM.ALUMINUM, en, an, ep, dt, True, threads=threads)
    return B / (time.perf_counter() - t0)


def cpu_baseline(target_s=12.0):
    threads = os.cpu_count() or 1
    probe = oracle_rate(max(256, 64 * threads), threads, seed=7)
    B = int(min(1 << 17, max(1024, probe * target_s)))
    rate = oracle_rate(B, threads, seed=0)
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{B} config-2 points (first {B} of the seeded generator, seed 0), "
                      f"C restatement of gsmkit automatic implicit-Euler + tangent, {threads} threads, {cpu_model()}"}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, flag in zip(names, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": smax, "reasons": sorted(reasons)}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def gsmkit_rates():
    """The reference package itself (gsmkit, installed unmodified in
    baseline/_ref by __graft_entry__.build()) on small config-2 samples:
    evaluate_arrays on the automatic route (threads = 1 and all host
    threads; GIL-bound) and the conventional radial return, the reference's
    fastest CPU route.  Informational keys of the
    reference line; None when baseline/_ref is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isfile(os.path.join(ref, "gsmkit", "evaluator.py")):
        return None
    sys.path.insert(0, ref)
    try:
        from gsmkit import gsm as rg
        from gsmkit.evaluator import StrategyConfig as RSC, evaluate_arrays as rev
    finally:
        sys.path.remove(ref)
    from paper_2006_04391_b200.workloads import config2_batch

    out = {}
    threads = os.cpu_count() or 1
    for key, strat, n, thr in (("automatic_1_thread", "automatic", 1 << 12, 1),
                               (f"automatic_{threads}_threads", "automatic", 1 << 13, threads),
                               ("conventional_1_thread", "conventional", 1 << 16, 1)):
        en, an, ep, dt = config2_batch(n, seed=0)
        cfg = RSC(strategy=strat, integrator="implicit-euler")
        t0 = time.perf_counter()
        rev(rg.MichelSuquet(), cfg, en, an, ep, dt, want_tangent=True, threads=thr)
        out[key] = {"evals_per_s": n / (time.perf_counter() - t0), "points": n}
    out["note"] = ("gsmkit (the unmodified reference, Python + numpy) from baseline/_ref, stress + tangent, "
                   "config-2 sample; the reference arm's value is the C restatement of the automatic route "
                   "(kind: port, all host threads), the faster of the two implementations of this path")
    return out


def run_reference(args, rank):
    """--impl reference: the reference algorithm on the host cores (rank 0 only)."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    probe = oracle_rate(max(256, 32 * threads), threads, seed=7)
    B = int(min(1 << 16, max(512, probe * 2.0)))  # ~2 s of CPU work per step
    for _ in range(args.warmup):
        oracle_rate(B, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle_rate(B, threads)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = B / (ms * 1e-3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config 2 sample: {B} of 2^20 EVP material points, stress + AD tangent",
                   "law": "MichelSuquet(ALUMINUM_MATRIX)", "strategy": "automatic", "integrator": "implicit-euler"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{B} points per step, C restatement of gsmkit (oracle/material_oracle.c), "
                                   f"{threads} threads, {cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        line["gsmkit"] = gsmkit_rates()
    except Exception as exc:  # noqa: BLE001 - informational only
        line["gsmkit"] = {"error": f"{type(exc).__name__}: {exc}"}
    print(json.dumps(line), flush=True)


FREE = np.array([False, True, True, True, True, True])


def _solver_stream(hom, dev):
    import torch

    from paper_2006_04391_b200 import _lib

    sp = ctypes.c_void_p()
    _lib.check(hom._lib.am_solver_stream(hom._h, ctypes.byref(sp)))
    return torch.cuda.ExternalStream(sp.value, device=dev)


def _max_over_ranks(dist, dev, x):
    if dist is None:
        return float(x)
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def basic_step(grid, n, dev, dist=None, comm=None, warm=False, max_iterations=5000, label=""):
    """Basic-scheme iterations/s of load step 1 of LoadingPath(steps=20)
    (mixed BC, tol 1e-5) on `grid`, device time (CUDA events on the solver
    stream, max over ranks); per-phase times from am_solver_timing.  With
    `comm` the grid is x-slab decomposed over the ranks (strong scaling).
    max_iterations < the step's count times that many iterations (the
    SolverError is expected and caught)."""
    import torch

    from paper_2006_04391_b200 import _lib, homogenize as H
    from paper_2006_04391_b200.evaluator import StrategyConfig

    cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
    hom = H.Homogenizer(grid, cfg, comm=comm, newton_warm_start=warm, max_iterations=max_iterations)
    lib = hom._lib
    stream = _solver_stream(hom, dev)
    path = H.LoadingPath(steps=20)
    times = path.times()
    target = np.zeros(6)
    target[0] = path.eps_xx(times)[1]
    _lib.check(lib.am_solver_timing(hom._h, 1, None))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    capped = False
    with Clocks(torch.cuda.current_device()) as clk:
        e0.record(stream)
        try:
            info, _ = hom._solve(target, times[1] - times[0], FREE)
            iters = info.iterations
        except H.SolverError as exc:
            if max_iterations >= 5000:
                raise
            iters, capped = len(exc.history), True
        e1.record(stream)
        torch.cuda.synchronize()
    ms = _max_over_ranks(dist, dev, e0.elapsed_time(e1))
    ph = np.zeros(5)
    _lib.check(lib.am_solver_timing(hom._h, -1, _lib.ptr(ph)))
    world = comm.world if comm is not None else 1
    Nh = n * n * (n // 2 + 1) // world  # rfft bins per rank
    it_t = ph[4] or 1.0
    fourier_ms = ph[2] / it_t
    zcb = ctypes.c_int(0)
    _lib.check(lib.am_solver_fft_callback(hom._h, ctypes.byref(zcb)))
    # read shat, ehat; write ehat (complex128 x 6), and without the inverse
    # transform's load callback also the scaled copy ehat'/N into shat
    fourier_bytes = (3 if zcb.value else 4) * 96.0 * Nh
    out = {
        "value": iters / (ms * 1e-3), "unit": "it/s", "iterations": iters, "ms_total": ms,
        "ms_per_iteration": ms / iters,
        "phase_ms_per_iteration": {"material": ph[0] / it_t, "forward_fft": ph[1] / it_t,
                                   "fourier+reduce": fourier_ms, "origin+inverse_fft": ph[3] / max(it_t - 1, 1)},
        "fourier_roofline": {"bound": "hbm", "achieved": fourier_bytes / (fourier_ms * 1e-3) / 1e9,
                             "peak": hbm_peak(), "unit": "GB/s",
                             "frac": fourier_bytes / (fourier_ms * 1e-3) / 1e9 / hbm_peak(),
                             "traffic_per_launch_algorithmic": fourier_bytes},
        "fft_load_callback": bool(zcb.value),
        "clocks": clk.summary(),
    }
    if capped:
        out["note"] = f"first {iters} iterations of load step 1 (max_iterations cap; per-iteration rate)"
    del hom
    return out


def loading_path_run(grid, dev, dist=None, comm=None, steps=20, warm=False):
    """The public run_loading_path (tension-compression, mixed BC, reference
    update per step) on `grid`: wall time of the whole call with device
    synchronisation on both sides (host-driven loop: convergence tests and
    tangent sweeps included), max over ranks."""
    import torch

    from paper_2006_04391_b200 import homogenize as H
    from paper_2006_04391_b200.evaluator import StrategyConfig

    cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    recs = H.run_loading_path(grid, H.LoadingPath(steps=steps), cfg, comm=comm, newton_warm_start=warm)
    torch.cuda.synchronize()
    wall = _max_over_ranks(dist, dev, time.perf_counter() - t0)
    its = int(sum(r["iterations"] for r in recs))
    return {"value": its / wall, "unit": "it/s", "seconds": wall, "iterations_total": its,
            "iterations_per_step": [r["iterations"] for r in recs],
            "sig_xx_final": float(recs[-1]["sig"][0]), "C11_final": recs[-1]["C11"]}


def oracle_basic_seconds_per_iteration(n, k=2):
    """CPU reference arm of the basic scheme: the oracle's
    (C restatement of the automatic route + numpy field step, all host
    threads) seconds per iteration of load step 1 at n^3, k iterations."""
    from oracle import homogenize as OH
    from oracle import material as OM
    from paper_2006_04391_b200 import homogenize as H

    ids = H.toy_mmc_grid(n).material_ids
    b = OH.Basic(ids, [OM.ALUMINUM, OM.law_params(0, 300e9, 0.25)], max_iterations=k,
                 threads=os.cpu_count() or 1)
    t, ex = OH.loading_times(20)
    eb = np.zeros(6)
    eb[0] = ex[1]
    t0 = time.perf_counter()
    try:
        b.solve_step(eb, t[1], FREE)
    except OH.NotConverged:
        pass
    return (time.perf_counter() - t0) / k


def config1_run(dev):
    """Config 1: 32^3 two-phase elastic sphere, one load step (strain BC and
    mixed BC), Homogenizer.solve_step device time; the numpy oracle (CPU)
    timed on the same step."""
    import torch

    from oracle import homogenize as OH
    from oracle import material as OM
    from paper_2006_04391_b200 import gsm, homogenize as H
    from paper_2006_04391_b200.evaluator import StrategyConfig
    from paper_2006_04391_b200.workloads import sphere_ids

    cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
    ids = sphere_ids(32)
    eb = np.zeros(6)
    eb[0] = 1e-3
    out = {"config": {"workload": "config 1: 32^3 two-phase elastic sphere (VF 0.2), one load step, tol 1e-5"}}
    for tag, free in (("strain_bc", np.zeros(6, bool)), ("mixed_bc", FREE)):
        best = None
        for _ in range(3):
            hom = H.Homogenizer(H.VoxelGrid(ids, [gsm.LinearElastic(55e9, 0.33), gsm.LinearElastic(300e9, 0.25)]),
                                cfg)
            stream = _solver_stream(hom, dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            info, _ = hom._solve(eb, 1.0, free)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
            del hom
        ob = OH.Basic(ids, [OM.law_params(0, 55e9, 0.33), OM.law_params(0, 300e9, 0.25)])
        t0 = time.perf_counter()
        _, _, oit, _ = ob.solve_step(eb, 1.0, free)
        cpu_s = time.perf_counter() - t0
        out[tag] = {"iterations": info.iterations, "ms": best, "value": info.iterations / (best * 1e-3),
                    "unit": "it/s", "oracle_iterations": oit,
                    "cpu_baseline": {"seconds": cpu_s, "value": oit / cpu_s, "unit": "it/s", "cores": 1,
                                     "kind": "port", "sample": "the same load step, numpy restatement (oracle/)"}}
    return out


def agree(dist, dev, ok):
    """All ranks proceed only if every rank's setup succeeded (no rank is left
    waiting in a collective the others skipped)."""
    if dist is None:
        return bool(ok)
    import torch

    t = torch.tensor([int(ok)], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0  # B200_PROFILING.md fallback


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=B_DEFAULT)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--basic", type=int, default=256, help="config-4 grid size n (0: skip the basic scheme)")
    ap.add_argument("--path", type=int, default=128, help="config-3 grid size n (0: skip)")
    ap.add_argument("--big", type=int, default=512, help="config-5 grid size n (0: skip)")
    ap.add_argument("--big-iterations", type=int, default=0,
                    help="config-5 iterations timed on one GPU (0: 300; the full load step on >1 GPU)")
    ap.add_argument("--no-strategies", action="store_true")
    ap.add_argument("--watchdog", type=float, default=1500.0,
                    help="seconds allowed for the basic-scheme runs before the line is printed with an error")
    ap.add_argument("--p2p", action="store_true",
                    help="at >1 GPU also time config 4 with the fused P2P (CUDA IPC) transposes")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    if world > 1:
        # communicator evidence in the driver's log (NCCL INIT lines), for
        # torch's communicator and libautomat's slab communicator alike
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")

    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)

    from paper_2006_04391_b200 import _lib, gsm
    from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays
    from paper_2006_04391_b200.workloads import config2_batch

    lib = _lib.load()
    _lib.check(lib.am_set_device(local))
    law = gsm.MichelSuquet()
    cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
    s_law, s_cfg = _lib.make_law(law), _lib.make_cfg(cfg)
    B = args.batch

    en, an, ep, dt = config2_batch(B, seed=rank)
    soa = lambda x: torch.from_numpy(np.ascontiguousarray(x.T)).to(dev)  # noqa: E731
    d_en, d_an, d_ep = soa(en), soa(an), soa(ep)
    d_dt = torch.from_numpy(dt).to(dev)
    d_sig = torch.empty((6, B), dtype=torch.float64, device=dev)
    d_a = torch.empty((7, B), dtype=torch.float64, device=dev)
    d_C = torch.empty((36, B), dtype=torch.float64, device=dev)
    d_it = torch.empty(B, dtype=torch.int32, device=dev)
    d_fl = torch.zeros(1, dtype=torch.int32, device=dev)
    d_st = torch.empty(B, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)

    def step():
        rc = lib.am_eval_batch(s_law, s_cfg, B, d_en.data_ptr(), d_an.data_ptr(), d_ep.data_ptr(), d_dt.data_ptr(),
                               0.0, 1, d_sig.data_ptr(), d_a.data_ptr(), d_C.data_ptr(), d_it.data_ptr(), None,
                               d_st.data_ptr(), d_fl.data_ptr(), sp)
        if rc:
            _lib.check(rc)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if int(d_fl.item()) != 0:
        raise RuntimeError(f"material kernel reported status flags {int(d_fl.item())}")

    # ---- config 2, device-resident (inputs in HBM; 552 MiB of I/O per step > 126 MB L2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    ms_max = _max_over_ranks(dist, dev, ms)
    value = world * B / (ms_max * 1e-3)
    clocks = clk.summary()

    iters = d_it.cpu().numpy()
    fl = float(np.sum(flops_per_eval(iters.astype(np.float64))))
    achieved = fl / (ms * 1e-3) / 1e12
    traffic = traffic_newton = traffic_tangent = None
    try:  # DRAM bytes per point of the two K1 kernels from the committed ncu capture
        tj = json.load(open(os.path.join(ROOT, "profiles", "r02", "traffic.json")))
        traffic_newton = B * tj["k_material_newton_raw_bytes_per_point"]
        traffic_tangent = B * tj["k_tangent_bytes_per_point"]
        traffic = traffic_newton + traffic_tangent
    except (OSError, KeyError, ValueError):
        pass
    peak = ctypes.c_double(0.0)
    _lib.check(lib.am_probe_fp64_tflops(5, ctypes.byref(peak)))
    # per-kernel device times of the same launches (CUDA events around the
    # Newton and the tangent kernel on this stream; a separate pass, since
    # the events synchronise after every launch)
    kt = np.zeros(3)
    _lib.check(lib.am_k1_timing(1, None))
    for _ in range(max(3, args.steps)):
        step()
    torch.cuda.synchronize()
    _lib.check(lib.am_k1_timing(-1, _lib.ptr(kt)))
    _lib.check(lib.am_k1_timing(0, None))
    t_newton, t_tangent = kt[0] / kt[2], kt[1] / kt[2]
    fl_newton = float(np.sum(1072.0 * iters.astype(np.float64) + 18.0))  # raw Newton: + delta eps, eps(t1)
    fl_tangent = 2255.0 * B  # tangent post-process 1695 + stress 20 + C 540

    # ---- the paper's strategy comparison on the same batch (stress + tangent,
    # device-resident): every strategy x integrator route the reference offers
    strategies = {}
    for strat, integ in (() if args.no_strategies else (
            ("automatic", "implicit-euler"), ("semi-automatic", "implicit-euler"),
            ("conventional", "implicit-euler"), ("automatic", "ode12"), ("automatic", "ode23"),
            ("semi-automatic", "ode23"), ("semi-automatic", "ode23s"))):
        c2 = _lib.make_cfg(StrategyConfig(strategy=strat, integrator=integ))

        def run(c2=c2):
            rc = lib.am_eval_batch(s_law, c2, B, d_en.data_ptr(), d_an.data_ptr(), d_ep.data_ptr(), d_dt.data_ptr(),
                                   0.0, 1, d_sig.data_ptr(), d_a.data_ptr(), d_C.data_ptr(), d_it.data_ptr(), None,
                                   d_st.data_ptr(), d_fl.data_ptr(), sp)
            if rc:
                _lib.check(rc)

        run()
        run()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(5):
            run()
        f1.record(stream)
        torch.cuda.synchronize()
        t_ms = f0.elapsed_time(f1) / 5
        strategies[f"{strat}/{integ}"] = {
            "evals_per_s": B / (t_ms * 1e-3), "ms": t_ms,
            ("mean_newton_iters" if integ == "implicit-euler" else "mean_substeps"): float(d_it.double().mean().item())}
    step()  # leave the headline route's outputs in the buffers
    torch.cuda.synchronize()

    # ---- end to end, headline: the reference's own call, evaluate_arrays,
    # with the caller's plain (pageable) numpy arrays; results come back as
    # numpy arrays.  Host->device and device->host copies inside the timed region.
    def e2e_py():
        return evaluate_arrays(law, cfg, en, an, ep, dt, want_tangent=True)

    for _ in range(2):
        r = e2e_py()
    del r
    e2e_steps = max(3, min(args.steps, 10))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        r = e2e_py()
    e2e_s = _max_over_ranks(dist, dev, (time.perf_counter() - t0) / e2e_steps)
    assert np.array_equal(r.newton_iters, iters), "evaluate_arrays disagrees with the device path"
    del r
    e2e_value = world * B / e2e_s

    # the same through the C ABI with pinned host buffers (the copy ceiling of the path)
    pin = lambda shape, dtype=torch.float64: torch.empty(shape, dtype=dtype, pin_memory=True).numpy()  # noqa: E731
    h_en, h_an, h_ep, h_dt = pin((B, 6)), pin((B, 7)), pin((B, 6)), pin((B,))
    h_en[:], h_an[:], h_ep[:], h_dt[:] = en, an, ep, dt
    h_sig, h_a, h_C, h_it = pin((B, 6)), pin((B, 7)), pin((B, 6, 6)), pin((B,), torch.int32)

    def e2e_abi():
        _lib.check(lib.am_eval_batch_host(s_law, s_cfg, B, _lib.ptr(h_en), _lib.ptr(h_an), _lib.ptr(h_ep),
                                          _lib.ptr(h_dt), 1, _lib.ptr(h_sig), _lib.ptr(h_a), _lib.ptr(h_C),
                                          _lib.ptr(h_it, _lib._i32p), None, None))

    for _ in range(2):
        e2e_abi()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_abi()
    abi_value = world * B / _max_over_ranks(dist, dev, (time.perf_counter() - t0) / e2e_steps)
    assert np.array_equal(h_it, iters), "e2e path disagrees with the device path"
    # PCIe ceiling: the same bytes as plain concurrent pinned copies (H2D on
    # one stream, D2H on another), no kernels
    h2d = B * (6 + 7 + 6 + 1) * 8
    d2h = B * (6 + 7 + 36) * 8 + B * (4 + 4 + 1)  # + Newton counts, rejected, status
    hin = torch.empty(h2d // 8, dtype=torch.float64, pin_memory=True)
    hout = torch.empty(d2h // 8, dtype=torch.float64, pin_memory=True)
    din, dout = torch.empty_like(hin, device=dev), torch.empty_like(hout, device=dev)
    s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

    def copies():
        with torch.cuda.stream(s_in):
            din.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s_out):
            hout.copy_(dout, non_blocking=True)

    copies()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        copies()
    torch.cuda.synchronize()
    pcie_ceiling = B / ((time.perf_counter() - t0) / 3)
    del hin, hout, din, dout, h_en, h_an, h_ep, h_dt, h_sig, h_a, h_C, h_it
    del d_en, d_an, d_ep, d_dt, d_sig, d_a, d_C, d_it, d_st
    torch.cuda.empty_cache()

    basic, errors = {}, []
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config 2: {B} EVP material points per GPU, stress + second-order AD tangent",
                   "law": "MichelSuquet(ALUMINUM_MATRIX)", "strategy": "automatic", "integrator": "implicit-euler",
                   "batch_per_gpu": B, "parallelism": f"dp{world} (independent points, no collective)",
                   "l2": "inputs+outputs 552 MiB per step > 126 MB L2 (no flush needed)",
                   "mean_newton_iters": float(iters.mean())},
        "roofline": {"bound": "fp64", "kernel": "k_material<MichelSuquetLaw> (Newton, the dominant kernel)",
                     "achieved": fl_newton / (t_newton * 1e-3) / 1e12, "peak": peak.value, "unit": "TFLOP/s",
                     "frac": fl_newton / (t_newton * 1e-3) / 1e12 / peak.value if peak.value else None,
                     "traffic": traffic_newton,
                     "traffic_source": "ncu dram__bytes_read + dram__bytes_write of this kernel per point "
                                       "(profiles/r02/traffic.json) x points per launch",
                     "peak_source": "measured: am_probe_fp64_tflops DFMA microbenchmark on this GPU "
                                    "(MEASURED_PEAKS.json has no fp64 entry)",
                     "work_per_launch": f"{fl_newton:.4g} algorithmic fp64 flops per launch (1072 per Newton "
                                        "iteration of each point + 18, SURVEY §8d)",
                     "launch_ms": t_newton, "share_of_step": t_newton / (t_newton + t_tangent),
                     "timing": "CUDA events around each kernel on the launching stream (am_k1_timing), "
                               f"{int(kt[2])} launches",
                     "tangent_kernel": {"kernel": "k_tangent<MichelSuquetLaw>", "launch_ms": t_tangent,
                                        "achieved": fl_tangent / (t_tangent * 1e-3) / 1e12,
                                        "frac": fl_tangent / (t_tangent * 1e-3) / 1e12 / peak.value,
                                        "work_per_launch": f"{fl_tangent:.4g} flops (2255 per point)",
                                        "traffic": traffic_tangent},
                     "step": {"achieved": achieved, "frac": achieved / peak.value if peak.value else None,
                              "traffic": traffic,
                              "work_per_step": f"{fl:.4g} flops (1072*N_it + 2273 per eval); one step = the "
                                               "Newton kernel + the tangent kernel"}},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "evaluator.evaluate_arrays (the reference's drop-in call) with the caller's pageable numpy "
                        "arrays -> am_eval_batch_host: pinned staging of the inputs by a host copy pool, results "
                        "returned in pooled page-locked numpy arrays, 3-stream chunked H2D|kernels|D2H",
                "c_abi_pinned": {"value": abi_value, "unit": UNIT,
                                 "path": "am_eval_batch_host (C ABI) with caller-pinned host AoS buffers"},
                "pcie_ceiling": pcie_ceiling, "frac_of_pcie_ceiling": e2e_value / world / pcie_ceiling,
                "pcie_ceiling_note": "same bytes as concurrent pinned H2D + D2H copies without kernels (per GPU)"},
        "gpu_launches": 2 * args.steps,
        "gpu_launches_note": "K1 launches (Newton + tangent kernel) of the config-2 timed region",
        "clocks": clocks,
        "basic_scheme": basic,
    }
    if strategies:
        line["strategies"] = strategies
        line["strategies_note"] = ("config-2 batch, stress + tangent, device-resident, 5 launches each after 2 "
                                   "warm-up; conventional = the paper's hand-derived radial return baseline")
    # a hang in a collective must not swallow the headline: past the budget
    # rank 0 prints the line with an error key and every rank exits non-zero
    import threading

    current = {"key": None}

    def watchdog():
        if rank == 0:
            line["error"] = (f"watchdog: basic-scheme runs exceeded {args.watchdog} s "
                             f"(in {current['key']})")
            print(json.dumps(line), flush=True)
        os._exit(3)

    dog = threading.Timer(args.watchdog, watchdog)
    dog.daemon = True
    dog.start()

    # ---- basic scheme (configs 1, 3, 4, 5): first-class keys; a failure
    # fails the bench (non-zero exit after the line)
    from paper_2006_04391_b200 import distributed as D, homogenize as H

    comm_of = (lambda transport: D.comm_from_torch(transport=transport)) if dist is not None else (lambda t: None)
    par = (lambda t: "single GPU (3-D cuFFT)" if world == 1 else
           f"x-slabs over {world} GPUs, 2-D cuFFT + {'ncclAlltoAll' if t == 'nccl' else 'fused P2P pack/unpack over NVLink'}"
           " transposes + 1-D cuFFT over x (strong scaling)")
    warm_note = ("Homogenizer(newton_warm_start=True): each voxel's Newton starts at its previous basic-scheme "
                 "iterate instead of a_n (opt-in, not in the reference; same equations and tolerance, identical "
                 "basic-scheme iterations)")

    def guarded(key, fn):
        current["key"] = key
        try:
            basic[key] = fn()
        except Exception as exc:  # noqa: BLE001 - reported, then the bench exits non-zero
            basic[key] = {"error": f"{type(exc).__name__}: {exc}"}
            errors.append(key)

    # a VoxelGrid carries its committed internal state (the reference commits
    # into grid.state), so every run gets a fresh grid of the same geometry
    def fresh(g):
        return H.VoxelGrid(g.material_ids, g.materials)

    if args.basic:
        n = args.basic
        grid4 = H.toy_mmc_grid(n)
        wl4 = (f"config 4: toy_mmc_grid({n}) (EVP matrix, VF 0.10 elastic fibre), LoadingPath(steps=20), mixed BC, "
               f"tol 1e-5, {world} GPU(s)")

        def c4_step():
            r = basic_step(fresh(grid4), n, dev, dist, comm_of("nccl"))
            r["config"] = {"workload": wl4 + ", load step 1", "parallelism": par("nccl"), "voxels": n**3,
                           "evp_voxels": int(len(grid4.voxel_index[0]))}
            rw = basic_step(fresh(grid4), n, dev, dist, comm_of("nccl"), warm=True)
            r["newton_warm_start"] = {k: rw[k] for k in ("value", "unit", "iterations", "ms_per_iteration",
                                                         "phase_ms_per_iteration")}
            r["newton_warm_start"]["note"] = warm_note
            if world > 1 and args.p2p:
                rp = basic_step(fresh(grid4), n, dev, dist, comm_of("p2p"))
                r["p2p_transport"] = {k: rp[k] for k in ("value", "unit", "iterations", "ms_per_iteration",
                                                         "phase_ms_per_iteration")}
            return r

        def c4_path():
            r = loading_path_run(fresh(grid4), dev, dist, comm_of("nccl"))
            r["config"] = {"workload": wl4 + ", all 20 load steps through run_loading_path (reference update per "
                                             "step, tangent sweeps included)", "parallelism": par("nccl")}
            r["note"] = "20-step average: iterations of all steps / wall time of run_loading_path"
            return r

        guarded("config4_step1", c4_step)
        guarded("config4_20_steps", c4_path)
    if args.path:
        grid3 = H.toy_mmc_grid(args.path)

        def c3():
            r = loading_path_run(fresh(grid3), dev, dist, comm_of("nccl"))
            r["config"] = {"workload": f"config 3: toy_mmc_grid({args.path}), LoadingPath(steps=20), mixed BC, "
                                       "reference update per step, run_loading_path", "parallelism": par("nccl")}
            rw = loading_path_run(fresh(grid3), dev, dist, comm_of("nccl"), warm=True)
            r["newton_warm_start"] = {k: rw[k] for k in ("value", "unit", "seconds", "iterations_total",
                                                         "sig_xx_final", "C11_final")}
            r["newton_warm_start"]["note"] = warm_note
            return r

        guarded("config3_path", c3)
    if args.big:
        n = args.big
        grid5 = H.toy_mmc_grid(n, fiber_law=gsm.LinearElastic(3000e9, 0.25))
        cap = 5000 if world > 1 else (args.big_iterations or 300)

        def c5():
            r = basic_step(fresh(grid5), n, dev, dist, comm_of("nccl"), max_iterations=cap)
            r["config"] = {"workload": f"config 5: toy_mmc_grid({n}, fiber_law=LinearElastic(3000e9, 0.25)) "
                                       f"(~55x contrast), load step 1 of LoadingPath(steps=20), mixed BC, tol 1e-5",
                           "parallelism": par("nccl"), "voxels": n**3}
            return r

        guarded("config5_step1", c5)
    if world == 1 and args.basic:
        guarded("config1", lambda: config1_run(dev))

        def slab_alg():
            # the multi-GPU algorithm (2-D FFTs, 8 x-slab transposes as device
            # copies, 1-D FFTs over x) on this one GPU: same iterations, and the
            # per-iteration cost of the decomposition itself
            hom = H.Homogenizer(fresh(grid4), cfg, slabs=8)
            stream = _solver_stream(hom, dev)
            path = H.LoadingPath(steps=20)
            t = path.times()
            target = np.zeros(6)
            target[0] = path.eps_xx(t)[1]
            _lib.check(hom._lib.am_solver_timing(hom._h, 1, None))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            info, _ = hom._solve(target, t[1] - t[0], FREE)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            ph = np.zeros(5)
            _lib.check(hom._lib.am_solver_timing(hom._h, -1, _lib.ptr(ph)))
            k = ph[4] or 1.0
            cbits = ctypes.c_int(0)
            _lib.check(hom._lib.am_solver_fft_callback(hom._h, ctypes.byref(cbits)))
            return {"value": info.iterations / (ms * 1e-3), "unit": "it/s", "iterations": info.iterations,
                    "ms_per_iteration": ms / info.iterations,
                    "fft_load_callback": bool(cbits.value & 1), "transposes_in_fft_callbacks": bool(cbits.value & 2),
                    "phase_ms_per_iteration": {"material": ph[0] / k, "forward_fft+transpose": ph[1] / k,
                                               "fourier+reduce": ph[2] / k,
                                               "origin+inverse_fft+transpose": ph[3] / max(k - 1, 1)},
                    "config": {"workload": "config 4 grid, load step 1, 8 x-slabs of one GPU (am_solver_create_slabs: "
                                           "the multi-GPU algorithm, transposes through the sibling slabs' spectra)"}}

        guarded("config4_step1_slab_algorithm", slab_alg)

    dog.cancel()
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        if errors:
            sys.exit(1)
        return

    if not args.no_cpu_baseline and world == 1:  # the CPU arm is timed at N = 1 only
        line["cpu_baseline"] = cpu_baseline()
        if args.basic or args.path:
            threads = os.cpu_count() or 1
            s64 = oracle_basic_seconds_per_iteration(64)
            ref = {"seconds_per_iteration_64": s64, "cores": threads, "kind": "port",
                   "sample": "2 iterations of load step 1 at 64^3 (C restatement of the automatic route, all host "
                             "threads, + numpy field step), N-scaled to the config's grid"}
            for key, n in (("config4_step1", args.basic), ("config3_path", args.path)):
                if n and key in basic and "error" not in basic[key]:
                    s = s64 * (n / 64) ** 3
                    basic[key]["cpu_baseline"] = dict(ref, value=1.0 / s, unit="it/s",
                                                      seconds_per_iteration_scaled=s)
    if errors:
        line["error"] = f"basic-scheme runs failed: {', '.join(errors)}"
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    if errors:
        sys.exit(1)


if __name__ == "__main__":
    main()
