"""ctypes front end of the C material oracle (test infrastructure only).

Mirrors ``gsmkit.evaluator.evaluate_arrays`` (evaluator.py:206-248) for the
automatic implicit-Euler route, plus the per-voxel Newton counts the
reference only exposes through a wrapper.
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_dp = ctypes.POINTER(ctypes.c_double)


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle_material.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.oracle_eval_batch.restype = ctypes.c_int
        L.oracle_eval_batch.argtypes = [
            ctypes.c_int, _dp, ctypes.c_int, ctypes.c_double, ctypes.c_int64,
            _dp, _dp, _dp, _dp, ctypes.c_int, _dp, _dp, _dp,
            ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_uint8), ctypes.c_int,
        ]
        L.oracle_constitutive.restype = None
        L.oracle_constitutive.argtypes = [ctypes.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.oracle_grad.restype = None
        L.oracle_grad.argtypes = [ctypes.c_int, _dp, ctypes.c_int, _dp, _dp]
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(_dp) if a is not None else None


ST_NEWTON, ST_SINGULAR, ST_NONFINITE = 1, 2, 4


def law_params(kind, E, nu, sigma_Y=1.0, H=1.0, eps0_dot=1.0, sigma_d=1.0, n=1.0):
    return kind, np.array([E, nu, sigma_Y, H, eps0_dot, sigma_d, n], dtype=float)


ALUMINUM = law_params(1, 55e9, 0.33, 25e6, 1.8e9, 1.0, 130e6, 3.6)


def evaluate(law, eps_n, a_n, eps_np1, dt, want_tangent=False, newton_mode="internal",
             newton_tol=1e-10, threads=1):
    """Returns dict(sigma, a, C, iters, status, code).

    ``law`` is ``(kind, params)`` (see ``law_params``); arrays are AoS like
    the reference's evaluate_arrays.
    """
    kind, prm = law
    m = 7 if kind == 1 else 0
    eps_n = np.ascontiguousarray(eps_n, dtype=float)
    eps_np1 = np.ascontiguousarray(eps_np1, dtype=float)
    B = eps_np1.shape[0]
    a_n = np.ascontiguousarray(a_n, dtype=float).reshape(B, m) if m else np.zeros((B, 0))
    dt = np.ascontiguousarray(np.broadcast_to(np.asarray(dt, dtype=float), (B,)))
    sig = np.zeros((B, 6))
    a = np.zeros((B, m))
    C = np.zeros((B, 6, 6)) if want_tangent else None
    iters = np.zeros(B, dtype=np.int32)
    status = np.zeros(B, dtype=np.uint8)
    code = lib().oracle_eval_batch(
        kind, _p(prm), 1 if newton_mode == "stress" else 0, newton_tol, B,
        _p(eps_n), _p(a_n) if m else None, _p(eps_np1), _p(dt), int(bool(want_tangent)),
        _p(sig), _p(a) if m else None, _p(C),
        iters.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
        status.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), int(threads),
    )
    if m == 0:
        a = a_n.copy()
    return dict(sigma=sig, a=a, C=C, iters=iters, status=status, code=code)


def constitutive(law, eps, a):
    """stress, generalized stress, rhs, d rhs/da, d rhs/deps at one point (gsm.py:574-602)."""
    kind, prm = law
    eps = np.ascontiguousarray(eps, dtype=float)
    a = np.ascontiguousarray(a, dtype=float) if kind == 1 else np.zeros(7)
    sig = np.zeros(6); A = np.zeros(7); f = np.zeros(7); J = np.zeros((7, 7)); dfde = np.zeros((7, 6))
    lib().oracle_constitutive(kind, _p(prm), _p(eps), _p(a), _p(sig), _p(A), _p(f), _p(J), _p(dfde))
    return sig, A, f, J, dfde


def grad(law, which, x):
    kind, prm = law
    x = np.ascontiguousarray(x, dtype=float)
    g = np.zeros(13 if which == 0 else 7)
    lib().oracle_grad(kind, _p(prm), which, _p(x), _p(g))
    return g
