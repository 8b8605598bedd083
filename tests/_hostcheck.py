"""ctypes front end of tests/hostcheck: the device material code built with g++.

Test infrastructure only -- lets the CPU suite exercise csrc/material.cuh
(AD, Newton, LU, tangent) against the oracle and the reference fixtures
without a GPU.  The product package never loads it.
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "hostcheck")
_L = None
_dp = ctypes.POINTER(ctypes.c_double)


def lib():
    global _L
    if _L is None:
        subprocess.run(["make", "-s", "-C", HERE], check=True)
        _L = ctypes.CDLL(os.path.join(HERE, "libhostcheck.so"))
        _L.hostcheck_eval.restype = ctypes.c_int
    return _L


def _p(a):
    return a.ctypes.data_as(_dp)


def evaluate(law, eps_n, a_n, eps_np1, dt, want_tangent, newton_mode=0, tol=1e-10):
    kind, prm = law
    m = 7 if kind == 1 else 0
    eps_n = np.ascontiguousarray(eps_n, dtype=float)
    eps_np1 = np.ascontiguousarray(eps_np1, dtype=float)
    B = eps_np1.shape[0]
    an = np.ascontiguousarray(a_n, dtype=float) if m else np.zeros((B, 1))
    dt = np.ascontiguousarray(np.broadcast_to(np.asarray(dt, dtype=float), (B,)))
    sig = np.zeros((B, 6)); a = np.zeros((B, max(m, 1))); C = np.zeros((B, 6, 6))
    it = np.zeros(B, np.int32); st = np.zeros(B, np.uint8)
    code = lib().hostcheck_eval(
        kind, _p(prm), int(newton_mode), ctypes.c_double(tol), ctypes.c_int64(B), _p(eps_n), _p(an), _p(eps_np1),
        _p(dt), int(bool(want_tangent)), _p(sig), _p(a), _p(C),
        it.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
    return dict(sigma=sig, a=a[:, :m], C=C if want_tangent else None, iters=it, status=st, code=code)
