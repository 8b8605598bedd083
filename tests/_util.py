"""Shared comparison helpers for the parity tests."""

import numpy as np

# north-star tolerances (BASELINE.json north_star)
TOL_STATE = 1e-10   # per-voxel stress and internal variables, relative
TOL_TANGENT = 1e-8  # consistent tangent, relative


def relerr(x, y):
    """Normwise relative error max|x-y| / max|y| (0 when both vanish)."""
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    den = np.max(np.abs(y)) if y.size else 0.0
    num = np.max(np.abs(x - y)) if y.size else 0.0
    if den == 0.0:
        return num
    return num / den


def rowwise_relerr(x, y):
    """Per-row normwise relative error (each voxel scaled by its own magnitude)."""
    x = np.asarray(x, dtype=float).reshape(len(x), -1)
    y = np.asarray(y, dtype=float).reshape(len(y), -1)
    den = np.maximum(np.max(np.abs(y), axis=1), 1e-300)
    return np.max(np.abs(x - y), axis=1) / den


def assert_close(x, y, tol, what=""):
    e = relerr(x, y)
    assert e <= tol, f"{what}: relative error {e:.3e} > {tol:.1e}"
