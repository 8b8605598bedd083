"""Integration error types of the reference (gsmkit/odeint.py:30-35).

The implicit-Euler Newton (odeint.py:357-426) runs inside the device
material kernel (csrc/material.cuh newton_ie / eval_voxel); these are the
exception classes the host shim raises from its status codes.
"""


class IntegrationError(RuntimeError):
    """Substep count cap exceeded, step size underflow, or similar."""


class NewtonDivergenceError(IntegrationError):
    """Newton iteration on an implicit step failed to converge."""
