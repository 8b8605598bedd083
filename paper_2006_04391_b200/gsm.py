"""Generalized standard materials defined by two potentials (gsmkit/gsm.py).

A law is a free energy omega(eps, a) plus a force potential psi(A) over the
generalized stresses A = -domega/da.  In this package the potentials of the
shipped laws are compiled into the device material kernel
(csrc/laws.cuh) and every derived quantity -- sigma, A, f = dpsi/dA, the
Jacobians and the consistent tangent -- comes from the device AD
(csrc/ad.cuh).  The Python classes carry the parameters, the constant
matrices the solver needs on the host (elastic stiffness for the initial
reference material), and the potentials written over generic scalars (the
same formulas the device code compiles, usable for inspection on plain
floats).

Module-level operations (``stress`` ... ``rhs_strain_jacobian``,
gsm.py:574-602) run on the GPU through ``am_constitutive_host``.
"""

from dataclasses import dataclass

import numpy as np

from . import _lib
from .linalg import SHEAR_DUP, isotropic_stiffness, lame_parameters

# deviatoric projector on stress-like Voigt vectors (gsm.py:36-37)
DEV6 = np.eye(6)
DEV6[:3, :3] -= 1.0 / 3.0


class NewtonError(RuntimeError):
    """Scalar return-mapping Newton failed to converge (gsm.py:40)."""


def _sqrt(x):
    return x.sqrt() if hasattr(x, "sqrt") else np.sqrt(x)


def _pos(x):
    return x.pos() if hasattr(x, "pos") else np.maximum(x, 0.0)


def dev_components(s):
    """Deviator of a Voigt 6-list of scalar-likes (gsm.py:62-65)."""
    p = (s[0] + s[1] + s[2]) * (1.0 / 3.0)
    return [s[0] - p, s[1] - p, s[2] - p, s[3], s[4], s[5]]


def mises_components(s):
    """Guarded von Mises norm of the deviator (gsm.py:68-79): (norm, deviator)."""
    d = dev_components(s)
    q = 1.5 * (d[0] * d[0] + d[1] * d[1] + d[2] * d[2] + 2.0 * (d[3] * d[3] + d[4] * d[4] + d[5] * d[5]))
    qv = getattr(q, "val", q)
    mask = np.where(np.asarray(qv) > 0.0, 1.0, 0.0)
    return _sqrt(q + (1.0 - mask)) * mask, d


class GsmDefinition:
    """Base class: a material is two potentials over generic scalars (gsm.py:82-97).

    Only laws with device potentials (LinearElastic, MichelSuquet) can be
    evaluated; other subclasses raise ConfigError at evaluation time.
    """

    m = 0
    has_hand_partials = False
    has_conventional = False

    def omega(self, eps, a):
        raise NotImplementedError

    def psi(self, A):
        raise NotImplementedError

    def clamp_state(self, a):
        return a


class LinearElastic(GsmDefinition):
    """Isotropic linear elasticity; no internal variables (gsm.py:100-153)."""

    m = 0
    has_hand_partials = True

    def __init__(self, E, nu):
        self.E = float(E)
        self.nu = float(nu)
        self.lam, self.mu = lame_parameters(self.E, self.nu)
        self.Ce = isotropic_stiffness(self.E, self.nu)

    def omega(self, eps, a):
        tr = eps[0] + eps[1] + eps[2]
        w = 0.5 * self.lam * tr * tr
        w = w + self.mu * (eps[0] * eps[0] + eps[1] * eps[1] + eps[2] * eps[2])
        return w + 0.5 * self.mu * (eps[3] * eps[3] + eps[4] * eps[4] + eps[5] * eps[5])

    def psi(self, A):
        return 0.0

    @property
    def d2w_ee(self):
        return self.Ce

    @property
    def d2w_ae(self):
        return np.zeros((0, 6))

    @property
    def d2w_aa(self):
        return np.zeros((0, 0))


@dataclass(frozen=True)
class MichelSuquetParams:
    """Material constants, SI units (gsm.py:156-174)."""

    E: float
    nu: float
    sigma_Y: float
    H: float
    eps0_dot: float
    sigma_d: float
    n: float

    def __post_init__(self):
        for name in ("E", "nu", "sigma_Y", "H", "eps0_dot", "sigma_d", "n"):
            if getattr(self, name) <= 0.0:
                raise ValueError(f"{name} must be positive")
        if self.nu >= 0.5:
            raise ValueError("nu must be < 0.5")


#: calibration of the aluminum matrix (gsm.py:177-179, PAPER Table 1)
ALUMINUM_MATRIX = MichelSuquetParams(E=55e9, nu=0.33, sigma_Y=25e6, H=1.8e9, eps0_dot=1.0, sigma_d=130e6, n=3.6)

#: linear elastic fiber material paired with the aluminum matrix (gsm.py:182)
ALUMINA_FIBER = dict(E=300e9, nu=0.25)


def load_michel_suquet_params(path):
    """Read ``key = value`` constants; unknown keys rejected (gsm.py:185-207)."""
    fields = MichelSuquetParams.__dataclass_fields__
    values = {}
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw_line in enumerate(fh, 1):
            line = raw_line.split("#", 1)[0].strip()
            if not line:
                continue
            key, sep, raw = line.partition("=")
            if not sep:
                raise ValueError(f"{path}:{lineno}: expected 'key = value'")
            key = key.strip()
            if key not in fields:
                raise ValueError(f"{path}:{lineno}: unknown key {key!r}")
            values[key] = float(raw.strip())
    missing = set(fields) - set(values)
    if missing:
        raise ValueError(f"{path}: missing keys {sorted(missing)}")
    return MichelSuquetParams(**values)


class MichelSuquet(GsmDefinition):
    """Elasto-viscoplastic law, kinematic hardening, Norton flow (gsm.py:210-256).

    State a = (eps_vp[0:6], alpha).
    """

    m = 7
    has_hand_partials = True
    has_conventional = True

    def __init__(self, params=ALUMINUM_MATRIX):
        self.params = params
        self.lam, self.mu = lame_parameters(params.E, params.nu)
        self.Ce = isotropic_stiffness(params.E, params.nu)
        self.Hmat = np.diag([params.H] * 3 + [params.H / 2.0] * 3)
        self._d2w_aa = np.zeros((7, 7))
        self._d2w_aa[:6, :6] = self.Ce + (2.0 / 3.0) * self.Hmat
        self._d2w_ae = np.zeros((7, 6))
        self._d2w_ae[:6, :] = -self.Ce

    def omega(self, eps, a):
        p = self.params
        ee = [eps[i] - a[i] for i in range(6)]
        tr = ee[0] + ee[1] + ee[2]
        w = 0.5 * self.lam * tr * tr
        w = w + self.mu * (ee[0] * ee[0] + ee[1] * ee[1] + ee[2] * ee[2])
        w = w + 0.5 * self.mu * (ee[3] * ee[3] + ee[4] * ee[4] + ee[5] * ee[5])
        w = w + (p.H / 3.0) * (a[0] * a[0] + a[1] * a[1] + a[2] * a[2])
        w = w + (p.H / 6.0) * (a[3] * a[3] + a[4] * a[4] + a[5] * a[5])
        return w + p.sigma_Y * a[6]

    def psi(self, A):
        p = self.params
        norm, _ = mises_components(A[:6])
        y = norm + A[6]
        return (p.sigma_d * p.eps0_dot / (p.n + 1.0)) * _pos(y * (1.0 / p.sigma_d)) ** (p.n + 1.0)

    def clamp_state(self, a):
        """alpha >= 0 (gsm.py:252-256)."""
        out = np.array(a, dtype=float, copy=True)
        out[..., 6] = np.maximum(out[..., 6], 0.0)
        return out

    @property
    def d2w_ee(self):
        return self.Ce

    @property
    def d2w_ae(self):
        return self._d2w_ae

    @property
    def d2w_aa(self):
        return self._d2w_aa


# ---------------------------------------------------------------------------
# module-level constitutive operations (gsm.py:574-602), on the device
# ---------------------------------------------------------------------------

_STRATEGIES = ("automatic", "semi-automatic", "conventional")


def _constitutive(law, eps, a, strategy):
    if strategy not in _STRATEGIES:
        raise ValueError(f"unsupported strategy {strategy!r}")
    lib = _lib.load()
    s_law = _lib.make_law(law)
    m = law.m
    eps = np.asarray(eps, dtype=float)
    batch = eps.shape[:-1]
    B = int(np.prod(batch, dtype=np.int64))
    e = _lib.f64(eps, (B, 6))
    av = _lib.f64(np.broadcast_to(np.asarray(a, dtype=float), batch + (m,)), (B, m)) if m else np.zeros((B, 1))
    sig = np.zeros((B, 6))
    A = np.zeros((B, max(m, 1)))
    f = np.zeros((B, max(m, 1)))
    J = np.zeros((B, max(m, 1), max(m, 1)))
    Je = np.zeros((B, max(m, 1), 6))
    rc = lib.am_constitutive_host(s_law, B, _lib.ptr(e), _lib.ptr(av), _lib.ptr(sig), _lib.ptr(A), _lib.ptr(f),
                                  _lib.ptr(J), _lib.ptr(Je))
    _lib.check(rc, "constitutive")
    return (sig.reshape(batch + (6,)), A[:, :m].reshape(batch + (m,)), f[:, :m].reshape(batch + (m,)),
            J[:, :m, :m].reshape(batch + (m, m)), Je[:, :m].reshape(batch + (m, 6)))


def stress(law, eps, a, strategy="automatic"):
    """Stress sigma = domega/deps at (eps, a)."""
    return _constitutive(law, eps, a, strategy)[0]


def generalized_stress(law, eps, a, strategy="automatic"):
    """Generalized stresses A = -domega/da at (eps, a)."""
    return _constitutive(law, eps, a, strategy)[1]


def evolution_rhs(law, eps, a, strategy="automatic"):
    """Evolution right-hand side f(eps, a) = dpsi/dA(-domega/da)."""
    return _constitutive(law, eps, a, strategy)[2]


def rhs_jacobian(law, eps, a, strategy="automatic"):
    """Jacobian df/da of the evolution right-hand side."""
    return _constitutive(law, eps, a, strategy)[3]


def rhs_strain_jacobian(law, eps, a, strategy="automatic"):
    """Jacobian df/deps of the evolution right-hand side."""
    return _constitutive(law, eps, a, strategy)[4]
