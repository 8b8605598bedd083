"""Closed-form effective stiffness of a two-phase isotropic elastic laminate,
the homogenizer known answer of SPEC.md acceptance criterion 9.

Phases vary along axis ``d`` only, so the exact fields are piecewise
constant: every phase carries eps_bar + sym(n (x) v_i) with sum f_i v_i = 0
(compatibility) and the traction C_i eps_i n is the same in every phase
(equilibrium).  With K_i = n.C_i.n the acoustic tensor and b_i = C_i eps_bar n,
t = (sum f_i K_i^-1)^-1 sum f_i K_i^-1 b_i and v_i = K_i^-1 (t - b_i).
Voigt order (xx, yy, zz, yz, xz, xy), strains with engineering shear
(paper_2006_04391_b200/linalg.py)."""

import numpy as np

VOIGT = ((0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1))


def lame(E, nu):
    return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))


def iso_tensor(lam, mu):
    d = np.eye(3)
    return (lam * np.einsum("ij,kl->ijkl", d, d)
            + mu * (np.einsum("ik,jl->ijkl", d, d) + np.einsum("il,jk->ijkl", d, d)))


def strain_tensor(e):
    t = np.zeros((3, 3))
    for p, (i, j) in enumerate(VOIGT):
        t[i, j] = t[j, i] = e[p] if p < 3 else 0.5 * e[p]
    return t


def laminate_stress(phases, fractions, axis, ebar):
    """Mean Voigt stress of the laminate under the macroscopic strain ``ebar``
    (Voigt); ``phases`` are (E, nu) pairs, ``fractions`` their volume fractions."""
    n = np.eye(3)[axis]
    E = strain_tensor(ebar)
    Cs = [iso_tensor(*lame(*p)) for p in phases]
    Ks = [np.einsum("j,ijkl,l->ik", n, C, n) for C in Cs]
    bs = [np.einsum("ijkl,kl,j->i", C, E, n) for C in Cs]
    Kinv = [np.linalg.inv(K) for K in Ks]
    t = np.linalg.solve(sum(f * Ki for f, Ki in zip(fractions, Kinv)),
                        sum(f * Ki @ b for f, Ki, b in zip(fractions, Kinv, bs)))
    sig = np.zeros((3, 3))
    for f, C, Ki, b in zip(fractions, Cs, Kinv, bs):
        v = Ki @ (t - b)
        sig += f * np.einsum("ijkl,kl->ij", C, E + 0.5 * (np.outer(n, v) + np.outer(v, n)))
    return np.array([sig[i, j] for i, j in VOIGT])


def laminate_stiffness(phases, fractions, axis):
    """6x6 Voigt effective stiffness (columns: unit engineering strains)."""
    return np.stack([laminate_stress(phases, fractions, axis, np.eye(6)[j]) for j in range(6)], axis=1)


def laminate_ids(n, axis, layer):
    """(n, n, n) material ids: phase 1 on the first ``layer`` planes along ``axis``."""
    ids = np.zeros((n, n, n), dtype=np.uint8)
    sl = [slice(None)] * 3
    sl[axis] = slice(0, layer)
    ids[tuple(sl)] = 1
    return ids
