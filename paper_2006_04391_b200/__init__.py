"""AutoMat on B200: generalized standard materials from two potentials.

Drop-in surface of the reference package ``gsmkit`` (modules ``gsm``,
``evaluator``, ``homogenize``, ``linalg``, ``odeint``) whose hot path --
per-voxel automatic-differentiation material evaluation with an
implicit-Euler Newton and consistent tangent, and the Moulinec-Suquet basic
scheme around it -- runs as hand-written sm_100a CUDA kernels in
``libautomat.so`` (C ABI: include/automat.h), bound with ctypes.
"""

from . import gsm, linalg, odeint  # noqa: F401

__all__ = ["gsm", "linalg", "odeint", "evaluator", "homogenize", "workloads"]
