"""Seeded synthetic inputs for the configurations named in BASELINE.json.

Shared by the golden-fixture script, the tests and ``bench.py``; plain numpy,
no device code. Each generator follows the recipe recorded in SURVEY.md §8(d)
so that fixtures made from the reference and runs of this package see the
same inputs.
"""

import numpy as np


def config2_batch(B, seed=0, dt=0.05):
    """Config 2: independent elasto-viscoplastic material points.

    eps_n ~ N(0, 1e-3^2), eps_np1 = eps_n + N(0, 1e-3^2); a_n[:, :6] ~
    N(0, (2e-4)^2) made deviatoric, a_n[:, 6] = |N(0, 1e-3^2)|; dt = 0.05.
    Arrays are AoS (B, 6) / (B, 7) like the reference's evaluate_arrays
    arguments (evaluator.py:206).
    """
    rng = np.random.default_rng(seed)
    eps_n = rng.normal(0.0, 1e-3, (B, 6))
    eps_np1 = eps_n + rng.normal(0.0, 1e-3, (B, 6))
    a_n = np.zeros((B, 7))
    ev = rng.normal(0.0, 2e-4, (B, 6))
    ev[:, :3] -= ev[:, :3].mean(axis=1, keepdims=True)
    a_n[:, :6] = ev
    a_n[:, 6] = np.abs(rng.normal(0.0, 1e-3, B))
    dtv = np.full(B, float(dt))
    return eps_n, a_n, eps_np1, dtv


def sphere_ids(n, volume_fraction=0.2):
    """Config 1 geometry: centred sphere on an n^3 grid (voxel-centre coords)."""
    c = np.arange(n) + 0.5
    X, Y, Z = np.meshgrid(c, c, c, indexing="ij")
    R = (3.0 * volume_fraction * n**3 / (4.0 * np.pi)) ** (1.0 / 3.0)
    d = np.sqrt((X - n / 2) ** 2 + (Y - n / 2) ** 2 + (Z - n / 2) ** 2)
    return (d <= R).astype(np.uint8)
