"""Voigt conventions and small host-side tensor constants (gsmkit/linalg.py).

Voigt order (xx, yy, zz, yz, xz, xy); strains carry engineering shear,
stresses tensor shear (linalg.py:1-10).  The batched LU of the reference
(linalg.py:75-143) lives inside the device material kernel
(csrc/material.cuh lu_factor / lu_solve); only the exception types and the
constant builders are needed on the host.
"""

import numpy as np

VOIGT_COMPONENTS = ("xx", "yy", "zz", "yz", "xz", "xy")

# duplication weights of the shear entries in a stress-like contraction (linalg.py:17)
SHEAR_DUP = np.array([1.0, 1.0, 1.0, 2.0, 2.0, 2.0])


class SingularMatrixError(np.linalg.LinAlgError):
    """Raised when an LU pivot falls below the singularity threshold (linalg.py:20)."""


class EigenvalueError(np.linalg.LinAlgError):
    """Eigenvalue iteration failure (linalg.py:24)."""


def lame_parameters(E, nu):
    """Lame pair (lambda, mu) from Young's modulus and Poisson's ratio (linalg.py:49-53)."""
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = E / (2.0 * (1.0 + nu))
    return lam, mu


def isotropic_stiffness(E, nu):
    """6x6 isotropic stiffness for engineering-shear strains (linalg.py:56-63)."""
    lam, mu = lame_parameters(E, nu)
    C = np.zeros((6, 6))
    C[:3, :3] = lam
    C[0, 0] = C[1, 1] = C[2, 2] = lam + 2.0 * mu
    C[3, 3] = C[4, 4] = C[5, 5] = mu
    return C
