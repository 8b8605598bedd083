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
gsm.py:574-602) and ``LawOps`` (gsm.py:412-566) run on the GPU through
``am_lawops_host``; ``conventional_evaluate`` through the conventional route
of ``am_eval_batch_host``.
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

    def conventional_step(self, eps_n, a_n, eps_np1, h, want_tangent):
        """Backward-Euler radial return, ``(sigma, a_new, C)`` (gsm.py:332-404), on the device."""
        return _conventional_step(self, eps_n, a_n, eps_np1, h, want_tangent)

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

_STRATEGY_CODES = {"automatic": 1, "semi-automatic": 2, "conventional": 0}


def _lawops(law, strategy, eps, a, da=None, want=("sigma", "A", "f", "dfda", "dfde"), C=False):
    """One device call of LawOps at arbitrary leading batch shape (gsm.py:412-418)."""
    if strategy not in _STRATEGY_CODES:
        raise ValueError(f"unsupported strategy {strategy!r}")
    if strategy in ("semi-automatic", "conventional") and not law.has_hand_partials:
        raise ValueError("law does not ship hand-coded partials")  # _ops_for maps conventional to semi (gsm.py:574-577)
    lib = _lib.load()
    s_law = _lib.make_law(law)
    m = law.m
    eps = np.asarray(eps, dtype=float)
    batch = eps.shape[:-1]
    B = int(np.prod(batch, dtype=np.int64))
    e = _lib.f64(eps, (B, 6))
    av = _lib.f64(np.broadcast_to(np.asarray(a, dtype=float), batch + (m,)), (B, m)) if m else np.zeros((B, 1))
    dav = _lib.f64(np.broadcast_to(np.asarray(da, dtype=float), batch + (m, 6)), (B, m, 6)) if (da is not None and m) \
        else None
    mm = max(m, 1)
    out = {"sigma": np.zeros((B, 6)), "A": np.zeros((B, mm)), "f": np.zeros((B, mm)), "dfda": np.zeros((B, mm, mm)),
           "dfde": np.zeros((B, mm, 6))}
    Cv = np.zeros((B, 6, 6)) if C else None
    ptr = {k: (_lib.ptr(v) if k in want else None) for k, v in out.items()}
    rc = lib.am_lawops_host(s_law, _STRATEGY_CODES[strategy], B, _lib.ptr(e), _lib.ptr(av), _lib.ptr(dav),
                            ptr["sigma"], ptr["A"], ptr["f"], ptr["dfda"], ptr["dfde"], _lib.ptr(Cv))
    _lib.check(rc, "LawOps")
    res = {"sigma": out["sigma"].reshape(batch + (6,)), "A": out["A"][:, :m].reshape(batch + (m,)),
           "f": out["f"][:, :m].reshape(batch + (m,)), "dfda": out["dfda"][:, :m, :m].reshape(batch + (m, m)),
           "dfde": out["dfde"][:, :m].reshape(batch + (m, 6))}
    if C:
        res["C"] = Cv.reshape(batch + (6, 6))
    return res


class LawOps:
    """Uniform evaluation surface of a law under a strategy (gsm.py:412-566), on the device.

    Array operations only: the ``*_generic`` methods of the reference run
    Python payloads through Python potentials, which have no device
    counterpart.
    """

    def __init__(self, law, strategy):
        if strategy not in ("automatic", "semi-automatic"):
            raise ValueError(f"unsupported strategy {strategy!r}")
        if strategy == "semi-automatic" and not law.has_hand_partials:
            raise ValueError("law does not ship hand-coded partials")
        _lib.make_law(law)  # ConfigError for laws without device potentials
        self.law = law
        self.strategy = strategy
        self.m = law.m

    def stress(self, eps, a):
        return _lawops(self.law, self.strategy, eps, a, want=("sigma",))["sigma"]

    def gen_stress(self, eps, a):
        return _lawops(self.law, self.strategy, eps, a, want=("A",))["A"]

    def rhs(self, eps, a):
        return _lawops(self.law, self.strategy, eps, a, want=("f",))["f"]

    def rhs_and_jacobians(self, eps, a):
        """RHS with d f/d a and d f/d eps, shape (..., m, m) and (..., m, 6)."""
        r = _lawops(self.law, self.strategy, eps, a, want=("f", "dfda", "dfde"))
        return r["f"], r["dfda"], r["dfde"]

    def stress_and_tangent(self, eps, a, da_deps):
        """Stress and consistent tangent C = d2w/de2 + d2w/dade . da/de."""
        r = _lawops(self.law, self.strategy, eps, a, da=da_deps, want=("sigma",), C=True)
        return r["sigma"], r["C"]

    def elastic_tangent(self, eps, a):
        """Second strain derivative of omega (exact tangent when a is frozen)."""
        return _lawops(self.law, self.strategy, eps, a, want=(), C=True)["C"]


def stress(law, eps, a, strategy="automatic"):
    """Stress sigma = domega/deps at (eps, a)."""
    return _lawops(law, strategy, eps, a, want=("sigma",))["sigma"]


def generalized_stress(law, eps, a, strategy="automatic"):
    """Generalized stresses A = -domega/da at (eps, a)."""
    return _lawops(law, strategy, eps, a, want=("A",))["A"]


def evolution_rhs(law, eps, a, strategy="automatic"):
    """Evolution right-hand side f(eps, a) = dpsi/dA(-domega/da)."""
    return _lawops(law, strategy, eps, a, want=("f",))["f"]


def rhs_jacobian(law, eps, a, strategy="automatic"):
    """Jacobian df/da of the evolution right-hand side."""
    return _lawops(law, strategy, eps, a, want=("dfda",))["dfda"]


def rhs_strain_jacobian(law, eps, a, strategy="automatic"):
    """Jacobian df/deps of the evolution right-hand side."""
    return _lawops(law, strategy, eps, a, want=("dfde",))["dfde"]


def conventional_evaluate(law, eps_n, a_n, eps_np1, h, want_tangent=False):
    """Material-specific single-step evaluation (radial return, gsm.py:605-609).

    Runs the device radial return (csrc/conventional.cuh); a stalled scalar
    Newton raises ``NewtonError`` like gsm.py:377-378.
    """
    if not law.has_conventional:
        raise ValueError("law has no conventional evaluation routine")
    return law.conventional_step(eps_n, a_n, eps_np1, h, want_tangent)


def _conventional_step(law, eps_n, a_n, eps_np1, h, want_tangent):
    """MichelSuquet.conventional_step (gsm.py:332-404) on the device."""
    from .evaluator import StrategyConfig, _evaluate_arrays_status

    eps_np1 = np.asarray(eps_np1, dtype=float)
    a_n = np.asarray(a_n, dtype=float)
    squeeze = eps_np1.ndim == 1
    if squeeze:
        eps_np1 = eps_np1[None]
        a_n = np.broadcast_to(a_n, (1, law.m))
    batch = eps_np1.shape[:-1]
    B = int(np.prod(batch, dtype=np.int64))
    hv = np.broadcast_to(np.asarray(h, dtype=float), batch).reshape(B)
    a2 = np.broadcast_to(a_n, batch + (law.m,)).reshape(B, law.m)
    e2 = eps_np1.reshape(B, 6)
    cfg = StrategyConfig(strategy="conventional", integrator="implicit-euler")
    r, rc, _ = _evaluate_arrays_status(law, cfg, e2, a2, e2, hv, want_tangent)
    _lib.check(rc, "conventional_step")
    sigma = r.sigma.reshape(batch + (6,))
    a_new = r.a.reshape(batch + (law.m,))
    C = None if r.C is None else r.C.reshape(batch + (6, 6))
    if squeeze:
        sigma, a_new = sigma[0], a_new[0]
        C = None if C is None else C[0]
    return sigma, a_new, C
