"""ctypes binding of libautomat.so (include/automat.h).

The library is the only compute path of this package: if it is missing or
no CUDA device is visible, every entry point raises -- there is no CPU
fallback.
"""

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# AM_LIB overrides the library path (kernel-variant experiments under tools/)
LIB_PATH = os.environ.get("AM_LIB") or os.path.join(HERE, "libautomat.so")

AM_OK = 0
AM_ERR_CONFIG = 1
AM_ERR_NEWTON = 2
AM_ERR_SINGULAR = 3
AM_ERR_NOT_CONVERGED = 4
AM_ERR_CUDA = 5
AM_ERR_NCCL = 6
AM_ERR_ARG = 7
AM_ERR_NONFINITE = 8
AM_ERR_INTEGRATION = 9
AM_ERR_RADIAL = 10

AM_LAW_LINEAR_ELASTIC = 0
AM_LAW_MICHEL_SUQUET = 1
STRATEGY_CODES = {"conventional": 0, "automatic": 1, "semi-automatic": 2}
INTEGRATOR_CODES = {"implicit-euler": 0, "ode12": 1, "ode23": 2, "ode23s": 3}
NEWTON_CODES = {"internal": 0, "stress": 1}

VOXEL_NEWTON_FAILED = 1
VOXEL_SINGULAR = 2
VOXEL_NONFINITE = 4
VOXEL_INTEGRATION = 8
VOXEL_RADIAL = 16
ERROR_MEASURE_CODES = {"internal": 0, "stress": 1}


class am_law(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("reserved", ctypes.c_int32),
        ("E", ctypes.c_double), ("nu", ctypes.c_double),
        ("sigma_Y", ctypes.c_double), ("H", ctypes.c_double), ("eps0_dot", ctypes.c_double),
        ("sigma_d", ctypes.c_double), ("n", ctypes.c_double),
    ]


class am_cfg(ctypes.Structure):
    _fields_ = [
        ("strategy", ctypes.c_int32), ("integrator", ctypes.c_int32),
        ("newton_mode", ctypes.c_int32), ("max_newton", ctypes.c_int32),
        ("newton_tol", ctypes.c_double),
        ("error_measure", ctypes.c_int32), ("max_substeps", ctypes.c_int32),
        ("atol", ctypes.c_double), ("rtol", ctypes.c_double),
    ]


class am_stepinfo(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
        ("residual", ctypes.c_double), ("mean_substeps", ctypes.c_double),
        ("ebar", ctypes.c_double * 6), ("sig_bar", ctypes.c_double * 6),
    ]


_dp = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p

# symbol -> (restype, argtypes); the list is also what the CPU test-suite
# checks against include/automat.h
SIGNATURES = {
    "am_last_error": (ctypes.c_char_p, []),
    "am_version": (ctypes.c_char_p, []),
    "am_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "am_set_device": (ctypes.c_int, [ctypes.c_int]),
    "am_eval_batch": (ctypes.c_int, [
        ctypes.POINTER(am_law), ctypes.POINTER(am_cfg), ctypes.c_int64,
        _vp, _vp, _vp, _vp, ctypes.c_double, ctypes.c_int,
        _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
    ]),
    "am_eval_batch_host": (ctypes.c_int, [
        ctypes.POINTER(am_law), ctypes.POINTER(am_cfg), ctypes.c_int64,
        _dp, _dp, _dp, _dp, ctypes.c_int, _dp, _dp, _dp, _i32p, _i32p, _u8p,
    ]),
    "am_eval_batch_record_host": (ctypes.c_int, [
        ctypes.POINTER(am_law), ctypes.POINTER(am_cfg), ctypes.c_int64,
        _dp, _dp, _dp, _dp, ctypes.c_int, _dp, _dp, _dp, _i32p, _i32p, _i64p, _dp, _u8p,
    ]),
    "am_probe_fp64_tflops": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
    "am_host_alloc": (ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(_vp)]),
    "am_k1_timing": (ctypes.c_int, [ctypes.c_int, _dp]),
    "am_host_free": (ctypes.c_int, [_vp]),
    "am_lawops_host": (ctypes.c_int, [
        ctypes.POINTER(am_law), ctypes.c_int, ctypes.c_int64, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
    ]),
    "am_constitutive_host": (ctypes.c_int, [
        ctypes.POINTER(am_law), ctypes.c_int64, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
    ]),
    # basic scheme (solver.cu)
    "am_solver_create": (ctypes.c_int, [
        ctypes.c_int, ctypes.c_int, ctypes.c_int, _u8p, ctypes.c_int, ctypes.POINTER(am_law), ctypes.POINTER(am_cfg),
        ctypes.POINTER(_vp),
    ]),
    "am_solver_create_slabs": (ctypes.c_int, [
        ctypes.c_int, ctypes.c_int, ctypes.c_int, _u8p, ctypes.c_int, ctypes.POINTER(am_law), ctypes.POINTER(am_cfg),
        ctypes.c_int, ctypes.POINTER(_vp),
    ]),
    "am_nccl_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "am_solver_create_nccl": (ctypes.c_int, [
        ctypes.c_int, ctypes.c_int, ctypes.c_int, _u8p, ctypes.c_int, ctypes.POINTER(am_law), ctypes.POINTER(am_cfg),
        ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp),
    ]),
    "am_solver_ipc_export": (ctypes.c_int, [_vp, ctypes.c_char_p]),
    "am_solver_ipc_import": (ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_int]),
    "am_solver_layout": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(ctypes.c_int)]),
    "am_solver_destroy": (ctypes.c_int, [_vp]),
    "am_solver_set_reference": (ctypes.c_int, [_vp, ctypes.c_double, ctypes.c_double]),
    "am_solver_get_reference": (ctypes.c_int, [_vp, _dp, _dp]),
    "am_solver_set_mean": (ctypes.c_int, [_vp, _dp]),
    "am_solver_solve_step": (ctypes.c_int, [
        _vp, _dp, ctypes.c_double, _u8p, ctypes.c_double, ctypes.c_int, ctypes.POINTER(am_stepinfo), _dp, ctypes.c_int,
    ]),
    "am_solver_commit": (ctypes.c_int, [_vp, _dp]),
    "am_solver_set_warm_start": (ctypes.c_int, [_vp, ctypes.c_int]),
    "am_solver_fft_callback": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int)]),
    "am_solver_evaluate": (ctypes.c_int, [_vp, ctypes.c_double]),
    "am_solver_tangent_sweep": (ctypes.c_int, [_vp, ctypes.c_double, _dp, _dp, _dp]),
    "am_solver_get_field": (ctypes.c_int, [_vp, ctypes.c_int, _dp]),
    "am_solver_set_field": (ctypes.c_int, [_vp, ctypes.c_int, _dp]),
    "am_solver_get_state": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _dp]),
    "am_solver_set_state": (ctypes.c_int, [_vp, ctypes.c_int, _dp]),
    "am_solver_phase_count": (ctypes.c_int, [_vp, ctypes.c_int, _i64p]),
    "am_solver_synchronize": (ctypes.c_int, [_vp]),
    "am_solver_timing": (ctypes.c_int, [_vp, ctypes.c_int, _dp]),
    "am_solver_stream": (ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    "am_green_apply_host": (ctypes.c_int, [
        ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, _dp, _dp,
    ]),
    "am_equilibrium_residual_host": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp]),
    "am_apply_isotropic_host": (ctypes.c_int, [ctypes.c_int64, ctypes.c_double, ctypes.c_double, _dp, _dp]),
    "am_reference_update_host": (ctypes.c_int, [ctypes.c_int64, _dp, _dp, _dp]),
}

_LIB = None


def load(require_device=True):
    """Load libautomat.so (raises if it is absent: no CPU fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the package has no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    if require_device:
        n = ctypes.c_int(0)
        rc = _LIB.am_device_count(ctypes.byref(n))
        if rc != AM_OK or n.value < 1:
            raise RuntimeError(
                "libautomat: no CUDA device available (" + last_error() + "); this package has no CPU fallback"
            )
    return _LIB


def last_error():
    if _LIB is None:
        return ""
    msg = _LIB.am_last_error()
    return msg.decode() if msg else ""


def ptr(a, kind=_dp):
    if a is None:
        return None
    return a.ctypes.data_as(kind)


def make_law(law):
    """am_law for a gsm law object; ConfigError for laws without device potentials."""
    from .evaluator import ConfigError
    from .gsm import LinearElastic, MichelSuquet

    s = am_law()
    # exact types: a subclass may override omega / psi / clamp_state, which the
    # device potentials would silently ignore
    if type(law) is MichelSuquet:
        p = law.params
        s.kind = AM_LAW_MICHEL_SUQUET
        s.E, s.nu, s.sigma_Y, s.H = p.E, p.nu, p.sigma_Y, p.H
        s.eps0_dot, s.sigma_d, s.n = p.eps0_dot, p.sigma_d, p.n
    elif type(law) is LinearElastic:
        s.kind = AM_LAW_LINEAR_ELASTIC
        s.E, s.nu = law.E, law.nu
    else:
        raise ConfigError(
            f"law {type(law).__name__} has no device potentials; this build ships LinearElastic and "
            "MichelSuquet as sm_100a potentials (no CPU evaluation path)"
        )
    return s


def make_cfg(cfg):
    s = am_cfg()
    s.strategy = STRATEGY_CODES[cfg.strategy]
    s.integrator = INTEGRATOR_CODES[cfg.integrator]
    s.newton_mode = NEWTON_CODES[cfg.resolved_newton_mode]
    s.max_newton = 50
    s.newton_tol = 1e-10
    s.error_measure = ERROR_MEASURE_CODES[cfg.error_measure]
    s.max_substeps = int(cfg.max_substeps)
    s.atol = float(cfg.atol)
    s.rtol = float(cfg.rtol)
    return s


def check(rc, where=""):
    """Map an am_status to the reference's exception classes."""
    if rc == AM_OK:
        return
    msg = last_error()
    if where:
        msg = f"{where}: {msg}"
    from .evaluator import ConfigError
    from .linalg import SingularMatrixError
    from .odeint import IntegrationError, NewtonDivergenceError

    if rc == AM_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == AM_ERR_NEWTON:
        raise NewtonDivergenceError(msg)
    if rc == AM_ERR_INTEGRATION:
        raise IntegrationError(msg)
    if rc == AM_ERR_RADIAL:
        from .gsm import NewtonError

        raise NewtonError(msg)
    if rc == AM_ERR_SINGULAR:
        raise SingularMatrixError(msg)
    if rc == AM_ERR_NOT_CONVERGED:
        from .homogenize import SolverError

        raise SolverError(msg)
    if rc in (AM_ERR_ARG, AM_ERR_NONFINITE):
        raise ValueError(msg)
    raise RuntimeError(f"libautomat error {rc}: {msg}")


def f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


class _PinnedBlock:
    """A page-locked host block from the library's pool (am_host_alloc),
    returned to the pool when the last array viewing it is released."""

    __slots__ = ("ptr",)

    def __init__(self, nbytes):
        p = ctypes.c_void_p()
        check(load().am_host_alloc(int(nbytes), ctypes.byref(p)), "pinned host allocation")
        self.ptr = p.value

    def __del__(self):
        if self.ptr and _LIB is not None:
            _LIB.am_host_free(ctypes.c_void_p(self.ptr))
            self.ptr = None


def pinned_empty(shape, dtype=np.float64):
    """Uninitialised numpy array in page-locked host memory (result arrays of
    the host entry points: the device copies land in them directly)."""
    dtype = np.dtype(dtype)
    count = int(np.prod(shape))
    nbytes = max(count * dtype.itemsize, 1)
    blk = _PinnedBlock(nbytes)
    buf = (ctypes.c_char * nbytes).from_address(blk.ptr)
    buf._block = blk  # the block lives as long as any view of buf
    return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)
