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


def evaluate(law, eps_n, a_n, eps_np1, dt, want_tangent, newton_mode=0, tol=1e-10, semi=False):
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
        it.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
        int(bool(semi)))
    return dict(sigma=sig, a=a[:, :m], C=C if want_tangent else None, iters=it, status=st, code=code)


def adaptive(law, scheme, coupled, measure, eps_n, a_n, eps_np1, dt, atol=1e-6, rtol=1e-3, max_substeps=10000,
             semi=False):
    """Host build of the adaptive kernel (ode12 / ode23, automatic strategy)."""
    kind, prm = law
    eps_n = np.ascontiguousarray(eps_n, dtype=float)
    eps_np1 = np.ascontiguousarray(eps_np1, dtype=float)
    B = eps_np1.shape[0]
    an = np.ascontiguousarray(a_n, dtype=float)
    dt = np.ascontiguousarray(np.broadcast_to(np.asarray(dt, dtype=float), (B,)))
    sig = np.zeros((B, 6)); a = np.zeros((B, 7)); C = np.zeros((B, 6, 6))
    sub = np.zeros(B, np.int32); rej = np.zeros(B, np.int32); st = np.zeros(B, np.uint8)
    i32 = ctypes.POINTER(ctypes.c_int32)
    code = lib().hostcheck_adaptive(
        _p(prm), int(scheme), int(bool(coupled)), 1 if measure == "stress" else 0, ctypes.c_double(atol),
        ctypes.c_double(rtol), int(max_substeps), ctypes.c_int64(B), _p(eps_n), _p(an), _p(eps_np1), _p(dt),
        _p(sig), _p(a), _p(C), sub.ctypes.data_as(i32), rej.ctypes.data_as(i32),
        st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), int(bool(semi)))
    return dict(sigma=sig, a=a, C=C if coupled else None, substeps=sub, rejected=rej, status=st, code=code)


def conventional(law, eps_np1, a_n, dt, want_tangent):
    """Host build of the radial-return kernel (strategy='conventional')."""
    kind, prm = law
    eps_np1 = np.ascontiguousarray(eps_np1, dtype=float)
    B = eps_np1.shape[0]
    an = np.ascontiguousarray(a_n, dtype=float)
    dt = np.ascontiguousarray(np.broadcast_to(np.asarray(dt, dtype=float), (B,)))
    sig = np.zeros((B, 6)); a = np.zeros((B, 7)); C = np.zeros((B, 6, 6))
    code = lib().hostcheck_conventional(_p(prm), ctypes.c_int64(B), _p(eps_np1), _p(an), _p(dt), int(bool(want_tangent)),
                                        _p(sig), _p(a), _p(C))
    return dict(sigma=sig, a=a, C=C if want_tangent else None, code=code)


def tangent_point(law, eps_n, a, eps_np1, dt):
    """Host build of the tangent post-process at a given state (no Newton)."""
    _, prm = law
    eps_n = np.ascontiguousarray(eps_n, dtype=float)
    eps_np1 = np.ascontiguousarray(eps_np1, dtype=float)
    a = np.ascontiguousarray(a, dtype=float)
    B = eps_np1.shape[0]
    dt = np.ascontiguousarray(np.broadcast_to(np.asarray(dt, dtype=float), (B,)))
    sig = np.zeros((B, 6)); C = np.zeros((B, 6, 6)); st = np.zeros(B, np.uint8)
    lib().hostcheck_tangent_point(_p(prm), ctypes.c_int64(B), _p(eps_n), _p(a), _p(eps_np1), _p(dt), _p(sig), _p(C),
                                  st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
    return dict(sigma=sig, C=C, status=st)
