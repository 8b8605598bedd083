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
    """Normwise AND per-row relative error within tol.  Per row (voxel /
    point: the leading axis) the scale is the row's own magnitude, floored at
    1e-6 of the batch magnitude so that rows that vanish in the reference
    (e.g. the state of a frozen elastic point) compare absolutely."""
    e = relerr(x, y)
    assert e <= tol, f"{what}: relative error {e:.3e} > {tol:.1e}"
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    if y.ndim >= 2 and y.size:
        xr, yr = x.reshape(len(x), -1), y.reshape(len(y), -1)
        big = np.max(np.abs(yr))
        den = np.maximum(np.max(np.abs(yr), axis=1), 1e-6 * big)
        den = np.where(den > 0.0, den, 1.0)
        er = float(np.max(np.max(np.abs(xr - yr), axis=1) / den))
        assert er <= tol, f"{what}: per-row relative error {er:.3e} > {tol:.1e}"


def check_path_records(recs, g, what, parity_log=None):
    """Loading-path records against a reference fixture: identical
    iteration counts, sigma_bar / eps_bar within 1e-10 (per step, each
    record scaled by its own magnitude), C_bar / reference materials within
    TOL_TANGENT.  Returns the measured errors."""
    k = len(g["iterations"])
    recs = recs[:k]
    assert [r["iterations"] for r in recs] == g["iterations"].tolist(), what
    sig = np.stack([r["sig"] for r in recs])
    errs = {
        "steps": k,
        "sig_bar": float(rowwise_relerr(sig, g["sig"]).max()),
        "sig_xx": float(np.max(np.abs(sig[:, 0] - g["sig"][:, 0]) / np.abs(g["sig"][:, 0]))),
        "eps_xx": float(np.max(np.abs(np.array([r["eps_xx"] for r in recs]) - g["eps_xx"]) / np.abs(g["eps_xx"]))),
        "C11": float(np.max(np.abs(np.array([r["C11"] for r in recs]) - g["C11"]) / np.abs(g["C11"]))),
        "C12": float(np.max(np.abs(np.array([r["C12"] for r in recs]) - g["C12"]) / np.abs(g["C12"]))),
    }
    if parity_log is not None:
        parity_log(what, **errs)
    assert errs["sig_bar"] <= TOL_STATE and errs["sig_xx"] <= TOL_STATE and errs["eps_xx"] <= TOL_STATE, (what, errs)
    assert errs["C11"] <= TOL_TANGENT and errs["C12"] <= TOL_TANGENT, (what, errs)
    assert all(r["mean_substeps"] == 1.0 for r in recs)
    return errs
