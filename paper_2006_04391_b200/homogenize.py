"""FFT-based homogenization with the Moulinec-Suquet basic scheme (gsmkit/homogenize.py).

Same public surface as the reference module -- ``VoxelGrid``,
``toy_mmc_grid``, ``GreenOperator``, ``green_apply``,
``equilibrium_residual``, ``apply_isotropic``, ``reference_update``,
``Homogenizer``, ``run_loading_path``, ``LoadingPath``, ``StepInfo``,
``SolverError``, ``save_geometry`` / ``load_geometry`` -- with the numerical
work on the GPU (csrc/solver.cu):

* ``Homogenizer`` owns a device solver handle: strain, stress and committed
  fields, per-phase internal states, cuFFT plans.  One basic-scheme
  iteration is the material kernel over every phase, one batched D2Z of
  the stress, the fused Fourier kernel (residual + Green update) and one
  batched Z2D; the host only sees eight doubles per iteration.
* ``run_loading_path`` keeps everything on the device: the per-step tangent
  sweep is fused with ``reference_update`` and the tangent field is never
  materialised.

Field layout is component-first: (6, Nx, Ny, Nz), Voigt (xx, yy, zz, yz, xz, xy).
Geometry construction (``toy_mmc_grid``) and file I/O are host-side input
handling, as in the reference.
"""

import ctypes
import json
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .linalg import SHEAR_DUP  # noqa: F401  (re-exported like the reference)


class SolverError(RuntimeError):
    """Basic scheme failed to converge; carries the residual history (homogenize.py:29-34)."""

    def __init__(self, message, history=None):
        super().__init__(message)
        self.history = history or []


@dataclass(frozen=True)
class ReferenceMaterial:
    """Isotropic reference stiffness defining the preconditioner (homogenize.py:37-49)."""

    lam: float
    mu: float

    def matrix(self):
        C = np.zeros((6, 6))
        C[:3, :3] = self.lam
        C[0, 0] = C[1, 1] = C[2, 2] = self.lam + 2.0 * self.mu
        C[3, 3] = C[4, 4] = C[5, 5] = self.mu
        return C


@dataclass
class LoadingPath:
    """Piecewise-linear uniaxial tension-compression history (homogenize.py:52-77)."""

    rate: float = 1.4e-3
    eps_max: float = 3.58454e-3
    eps_min: float = -3.48441e-3
    steps: int = 80
    mixed_bc: bool = True

    @property
    def total_time(self):
        return (self.eps_max + (self.eps_max - self.eps_min)) / self.rate

    def times(self):
        return np.linspace(0.0, self.total_time, self.steps + 1)

    def eps_xx(self, t):
        t = np.asarray(t, dtype=float)
        t_turn = self.eps_max / self.rate
        return np.where(t <= t_turn, self.rate * t, self.eps_max - self.rate * (t - t_turn))


# ---------------------------------------------------------------------------
# grids and geometry (host-side input handling)
# ---------------------------------------------------------------------------


class VoxelGrid:
    """Periodic voxel grid with per-voxel material ids and internal state (homogenize.py:85-107).

    While a ``Homogenizer`` is bound to the grid the authoritative internal
    state lives on the device; ``state`` is fetched from there on access
    (and copied back when the solver is released), so the grid carries the
    committed state like the reference's in-place commits (homogenize.py:474-480).
    The grid references its solver weakly: releasing the Homogenizer frees
    its device memory.
    """

    def __init__(self, material_ids, materials):
        self.material_ids = np.asarray(material_ids)
        self.dims = self.material_ids.shape
        if len(self.dims) != 3:
            raise ValueError("material_ids must be a 3d array")
        self.materials = list(materials)
        ids_flat = self.material_ids.reshape(-1)
        present = np.unique(ids_flat)
        if present.max() >= len(self.materials):
            raise ValueError("material id exceeds material table")
        self.voxel_index = [np.flatnonzero(ids_flat == mid) for mid in range(len(self.materials))]
        self._state = [np.zeros((len(idx), law.m)) for idx, law in zip(self.voxel_index, self.materials)]
        self._solver = None  # weakref to the Homogenizer whose device state is authoritative

    @property
    def state(self):
        solver = self._solver() if self._solver is not None else None
        if solver is not None and solver._state_dirty:
            solver._pull_state(self._state)
            solver._state_dirty = False
        return self._state

    @property
    def n_voxels(self):
        return self.material_ids.size

    def reset_state(self):
        for arr in self._state:
            arr[:] = 0.0
        solver = self._solver() if self._solver is not None else None
        if solver is not None:
            solver._push_state(self._state)


def toy_mmc_grid(n=16, matrix_law=None, fiber_law=None, volume_fraction=0.10, seed=2024):
    """One tilted spherocylindrical fibre in a matrix (homogenize.py:110-141).

    Axis and position from the seeded RNG; the radius is bisected (60 steps)
    until the voxelised volume fraction reaches the requested value.
    """
    from .gsm import ALUMINA_FIBER, LinearElastic, MichelSuquet

    rng = np.random.default_rng(seed)
    center = 0.5 * n + rng.uniform(-0.05 * n, 0.05 * n, size=3)
    axis = np.array([1.0, 0.0, 0.0]) + rng.uniform(-0.3, 0.3, size=3)
    axis /= np.linalg.norm(axis)
    half_len = 0.34 * n
    c = np.arange(n) + 0.5
    coords = np.stack(np.meshgrid(c, c, c, indexing="ij"), axis=-1)
    rel = coords - center
    s = np.clip(rel @ axis, -half_len, half_len)
    dist = np.linalg.norm(rel - s[..., None] * axis, axis=-1)
    target = volume_fraction * n**3
    lo, hi = 0.5, 0.5 * n
    for _ in range(60):
        r = 0.5 * (lo + hi)
        if np.count_nonzero(dist <= r) < target:
            lo = r
        else:
            hi = r
    ids = (dist <= 0.5 * (lo + hi)).astype(np.uint8)
    return VoxelGrid(ids, [matrix_law or MichelSuquet(), fiber_law or LinearElastic(**ALUMINA_FIBER)])


def save_geometry(path, material_ids, material_names):
    """Raw little-endian voxel ids plus a JSON sidecar (homogenize.py:144-156)."""
    ids = np.asarray(material_ids)
    dtype = "u1" if ids.max() < 256 else "u2"
    ids.astype("<" + dtype).tofile(path)
    meta = {"dims": list(ids.shape), "dtype": dtype, "byte_order": "little", "materials": list(material_names)}
    with open(str(path) + ".json", "w", encoding="utf-8") as fh:
        json.dump(meta, fh, indent=2)


def load_geometry(path):
    """Inverse of save_geometry; returns (ids, names) (homogenize.py:159-166)."""
    with open(str(path) + ".json", "r", encoding="utf-8") as fh:
        meta = json.load(fh)
    ids = np.fromfile(path, dtype="<" + meta["dtype"]).reshape(tuple(meta["dims"]))
    return ids, meta["materials"]


# ---------------------------------------------------------------------------
# field operators (device)
# ---------------------------------------------------------------------------


def _field(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 4 or a.shape[0] != 6:
        raise ValueError("expected a (6, Nx, Ny, Nz) field")
    return a


class GreenOperator:
    """Periodic Green operator of an isotropic reference (homogenize.py:174-233).

    ``apply(tau)`` returns -Gamma0 tau: cuFFT D2Z, the per-frequency operator
    evaluated on the fly (no 36-entry table per frequency), Z2D.
    """

    def __init__(self, dims, ref):
        self.dims = tuple(int(x) for x in dims)
        self.ref = ref

    def apply(self, tau):
        tau = _field(tau)
        if tau.shape[1:] != self.dims:
            raise ValueError(f"field dims {tau.shape[1:]} != operator dims {self.dims}")
        out = np.empty_like(tau)
        lib = _lib.load()
        _lib.check(lib.am_green_apply_host(*self.dims, float(self.ref.lam), float(self.ref.mu), _lib.ptr(tau),
                                           _lib.ptr(out)), "GreenOperator.apply")
        return out


def green_apply(tau, ref):
    """One-shot Green operator application (homogenize.py:236-238)."""
    return GreenOperator(np.shape(tau)[1:], ref).apply(tau)


def equilibrium_residual(sig_field):
    """RMS of the Fourier traction misfit over the mean-stress norm (homogenize.py:241-267)."""
    sig = _field(sig_field)
    res = ctypes.c_double(0.0)
    lib = _lib.load()
    _lib.check(lib.am_equilibrium_residual_host(*sig.shape[1:], _lib.ptr(sig), ctypes.byref(res)),
               "equilibrium_residual")
    return float(res.value)


def apply_isotropic(ref, eps_field):
    """C_ref : eps for a (6, ...) engineering-strain field (homogenize.py:270-281)."""
    eps = np.ascontiguousarray(eps_field, dtype=np.float64)
    out = np.empty_like(eps)
    n = eps.size // 6
    lib = _lib.load()
    _lib.check(lib.am_apply_isotropic_host(n, float(ref.lam), float(ref.mu), _lib.ptr(eps), _lib.ptr(out)),
               "apply_isotropic")
    return out


def reference_update(C_field):
    """Isotropic reference bracketing the tangent field's spectra (homogenize.py:307-329).

    Raises ValueError on non-finite tangents, like the reference.
    """
    C = np.ascontiguousarray(C_field, dtype=np.float64).reshape(-1, 6, 6)
    lam, mu = ctypes.c_double(0.0), ctypes.c_double(0.0)
    lib = _lib.load()
    _lib.check(lib.am_reference_update_host(C.shape[0], _lib.ptr(C), ctypes.byref(lam), ctypes.byref(mu)),
               "reference_update")
    return ReferenceMaterial(lam=float(lam.value), mu=float(mu.value))


# ---------------------------------------------------------------------------
# the solver
# ---------------------------------------------------------------------------


@dataclass
class StepInfo:
    iterations: int
    residual: float
    mean_substeps: float
    history: list


class Homogenizer:
    """Basic-scheme solver owning the grid state over a loading history (homogenize.py:345-480).

    Fields and internal states live on the GPU; ``eps_n``, ``grid.state``
    and the arrays returned by ``solve_step`` / ``evaluate_field`` are host
    copies.
    """

    def __init__(self, grid, cfg, threads=1, tol=1e-5, max_iterations=5000, slabs=1, comm=None,
                 newton_warm_start=False):
        """``newton_warm_start`` (implicit Euler; not in the reference) starts
        each voxel's Newton at its previous basic-scheme iterate instead of
        a_n from the second iteration of a step on: same equations and
        tolerance, fewer Newton iterations, results equal to round-off.
        ``slabs`` > 1 runs the multi-GPU slab algorithm from this process on
        one device (x-slabs, all-to-all transposes as device copies); ``comm``
        (distributed.Comm) makes this process one rank of an NCCL-connected
        slab decomposition, in which case host fields are the rank's x-slab
        (6, nx / world, ny, nz) and ``grid.state`` is not synchronised."""
        from .evaluator import _validate_for_law

        self.grid = grid
        self.comm = comm
        self.cfg = cfg
        self.threads = threads
        self.tol = tol
        self.max_iterations = max_iterations
        for law in grid.materials:
            _validate_for_law(law, cfg)
        self._lib = _lib.load()
        laws = (_lib.am_law * len(grid.materials))(*[_lib.make_law(law) for law in grid.materials])
        self._cfg = _lib.make_cfg(cfg)
        ids = np.ascontiguousarray(grid.material_ids, dtype=np.uint8)
        h = ctypes.c_void_p()
        args = (*grid.dims, _lib.ptr(ids, _lib._u8p), len(grid.materials), laws, ctypes.byref(self._cfg))
        if comm is not None:
            rc = self._lib.am_solver_create_nccl(*args, comm.uid, comm.rank, comm.world, ctypes.byref(h))
            self._local_dims = (grid.dims[0] // comm.world,) + tuple(grid.dims[1:])
        elif slabs > 1:
            rc = self._lib.am_solver_create_slabs(*args, int(slabs), ctypes.byref(h))
            self._local_dims = tuple(grid.dims)
        else:
            rc = self._lib.am_solver_create(*args, ctypes.byref(h))
            self._local_dims = tuple(grid.dims)
        _lib.check(rc, "Homogenizer")
        self._h = h
        if newton_warm_start:
            _lib.check(self._lib.am_solver_set_warm_start(h, 1), "newton_warm_start")
        if comm is not None and comm.allgather is not None and comm.transport == "p2p":
            # fused transposes over NVLink: swap the spectrum buffers' IPC handles
            mine = ctypes.create_string_buffer(128)
            _lib.check(self._lib.am_solver_ipc_export(h, mine), "ipc export")
            every = comm.allgather(mine.raw)
            _lib.check(self._lib.am_solver_ipc_import(h, b"".join(every), comm.world), "ipc import")
        self._ebar_n = np.zeros(6)
        self._last = None  # (eps, ebar) host arrays of the last converged step
        self._state_dirty = False  # committed device state newer than grid._state
        if comm is None:
            self._push_state(grid._state)
            grid._solver = weakref.ref(self)
        else:
            self._push_state(self._local_states(grid._state))
        self.reference = None
        self.set_reference(self.elastic_reference())

    def __del__(self):
        h = getattr(self, "_h", None)
        lib = getattr(_lib, "_LIB", None) if _lib is not None else None  # module globals go away at shutdown
        if h is not None and h.value and lib is not None:
            grid = getattr(self, "grid", None)
            ref = grid._solver if grid is not None else None
            if ref is not None and self.comm is None and ref() in (None, self) and getattr(self, "_state_dirty", False):
                try:  # the grid keeps the committed state (the solver is going away)
                    self._pull_state(grid._state)
                except Exception:  # noqa: BLE001 - best effort during teardown
                    pass
            lib.am_solver_destroy(h)
            self._h = None

    # -- state transfer --------------------------------------------------------

    def _local_states(self, states):
        """This rank's part of per-phase global states (the voxels of its x-slab)."""
        from .distributed import slab_range

        x0, x1 = slab_range(self.grid.dims[0], self.comm.world, self.comm.rank)
        plane = int(np.prod(self.grid.dims[1:]))
        out = []
        for arr, idx in zip(states, self.grid.voxel_index):
            sel = (idx >= x0 * plane) & (idx < x1 * plane)
            out.append(np.asarray(arr)[sel])
        return out

    def _push_state(self, states):
        for i, (arr, law) in enumerate(zip(states, self.grid.materials)):
            if law.m and len(arr):
                a = np.ascontiguousarray(arr, dtype=np.float64)
                _lib.check(self._lib.am_solver_set_state(self._h, i, _lib.ptr(a)))

    def _pull_state(self, states, pending=False):
        for i, (arr, law) in enumerate(zip(states, self.grid.materials)):
            if law.m and len(arr):
                buf = np.empty((len(arr), law.m))
                _lib.check(self._lib.am_solver_get_state(self._h, i, int(pending), _lib.ptr(buf)))
                arr[:] = buf

    def _get(self, which):
        out = np.empty((6,) + self._local_dims)
        _lib.check(self._lib.am_solver_get_field(self._h, which, _lib.ptr(out)))
        return out

    def _set(self, which, field):
        f = _field(field)
        if f.shape[1:] != self._local_dims:
            raise ValueError(f"field dims {f.shape[1:]} != {self._local_dims}")
        _lib.check(self._lib.am_solver_set_field(self._h, which, _lib.ptr(f)))

    @property
    def eps_n(self):
        return self._get(1)

    @eps_n.setter
    def eps_n(self, value):
        self._set(1, value)

    @property
    def ebar_n(self):
        return self._ebar_n.copy()

    @ebar_n.setter
    def ebar_n(self, value):
        self._ebar_n = np.array(value, dtype=float)
        _lib.check(self._lib.am_solver_set_mean(self._h, _lib.ptr(self._ebar_n)))

    # -- reference handling --------------------------------------------------

    def elastic_tangent_field(self):
        """Per-voxel elastic stiffness (homogenize.py:362-373)."""
        C = np.zeros((self.grid.n_voxels, 6, 6))
        for law, idx in zip(self.grid.materials, self.grid.voxel_index):
            if len(idx):
                C[idx] = law.d2w_ee
        return C

    def elastic_reference(self):
        """reference_update of the elastic tangent field (homogenize.py:375-376).

        Every voxel of a phase has the same stiffness and reference_update
        keeps only extremes, so the phases' stiffnesses suffice.
        """
        Cs = [law.d2w_ee for law, idx in zip(self.grid.materials, self.grid.voxel_index) if len(idx)]
        return reference_update(np.stack(Cs))

    def set_reference(self, ref):
        self.reference = ref
        _lib.check(self._lib.am_solver_set_reference(self._h, float(ref.lam), float(ref.mu)))

    # -- material sweeps ------------------------------------------------------

    def evaluate_field(self, eps_np1_field, dt, want_tangent=False):
        """One material evaluation per voxel from the committed state (homogenize.py:389-421).

        Returns (sigma_field, C (N, 6, 6) or None, state list, mean substeps).
        The evaluation's state goes to a device scratch slot: the pending
        state of the last solve_step, which commit_step commits, is untouched
        (homogenize.py:399-421, 474-480).
        """
        self._set(0, eps_np1_field)
        self._last = None
        C = None
        if want_tangent:
            C = np.empty((self.grid.n_voxels, 6, 6))
            _lib.check(self._lib.am_solver_tangent_sweep(self._h, float(dt), None, None, _lib.ptr(C)), "evaluate_field")
        else:
            _lib.check(self._lib.am_solver_evaluate(self._h, float(dt)), "evaluate_field")
        sigma = self._get(2)
        state = [np.empty((len(i), law.m)) for i, law in zip(self.grid.voxel_index, self.grid.materials)]
        self._pull_state(state, pending=2)
        return sigma, C, state, 1.0

    # -- one loading step ------------------------------------------------------

    def _solve(self, ebar_target, dt, free_mask):
        free = np.zeros(6, dtype=np.uint8) if free_mask is None else np.asarray(free_mask, dtype=bool).astype(np.uint8)
        target = np.ascontiguousarray(ebar_target, dtype=float)
        info = _lib.am_stepinfo()
        hist = np.zeros(max(1, self.max_iterations))
        rc = self._lib.am_solver_solve_step(self._h, _lib.ptr(target), float(dt), _lib.ptr(free, _lib._u8p),
                                            float(self.tol), int(self.max_iterations), ctypes.byref(info),
                                            _lib.ptr(hist), len(hist))
        history = hist[: info.iterations].tolist()
        if rc == _lib.AM_ERR_NOT_CONVERGED:
            raise SolverError(
                f"basic scheme did not converge in {self.max_iterations} iterations (last residual {history[-1]:.3e})",
                history,
            )
        _lib.check(rc, "solve_step")
        return info, history

    def solve_step(self, ebar_target, dt, free_mask=None):
        """Converge the strain field for one loading step (homogenize.py:425-472)."""
        info, history = self._solve(ebar_target, dt, free_mask)
        eps, sigma = self._get(0), self._get(2)
        self._last = (eps, np.array(info.ebar[:]))
        return eps, sigma, StepInfo(iterations=info.iterations, residual=history[-1], mean_substeps=info.mean_substeps,
                                    history=history)

    def commit_step(self, eps, ebar):
        """eps_n <- eps, ebar_n <- ebar, internal state <- the state of the last
        converged solve_step, if any (homogenize.py:474-480)."""
        if self._last is None or eps is not self._last[0]:
            self._set(0, eps)
        self._ebar_n = np.array(ebar, dtype=float)
        _lib.check(self._lib.am_solver_commit(self._h, _lib.ptr(self._ebar_n)))
        self._state_dirty = True
        self._last = None


def run_loading_path(grid, path, cfg, update_reference=True, threads=1, tol=1e-5, max_iterations=5000, slabs=1,
                     comm=None, newton_warm_start=False):
    """March the loading path; one record dict per step (homogenize.py:485-528).

    Device-resident: per step the basic scheme, then (update_reference) the
    tangent sweep fused with reference_update, commit, new reference.
    ``slabs`` / ``comm`` / ``newton_warm_start``: see Homogenizer (every rank
    returns the same records).
    """
    hom = Homogenizer(grid, cfg, threads=threads, tol=tol, max_iterations=max_iterations, slabs=slabs, comm=comm,
                      newton_warm_start=newton_warm_start)
    lib = hom._lib
    times = path.times()
    eps_targets = path.eps_xx(times)
    free = np.array([False, True, True, True, True, True]) if path.mixed_bc else np.zeros(6, dtype=bool)
    records = []
    Cbar = np.zeros(36)
    lam_mu = np.zeros(2)
    for k in range(1, len(times)):
        dt = times[k] - times[k - 1]
        target = np.zeros(6)
        target[0] = eps_targets[k]
        info, _ = hom._solve(target, dt, free)
        ebar = np.array(info.ebar[:])
        sig_bar = np.array(info.sig_bar[:])
        C11 = C12 = float("nan")
        if update_reference:
            _lib.check(lib.am_solver_tangent_sweep(hom._h, float(dt), _lib.ptr(Cbar), _lib.ptr(lam_mu), None),
                       "tangent sweep")
            C11, C12 = float(Cbar[0]), float(Cbar[1])
            hom._ebar_n = ebar
            _lib.check(lib.am_solver_commit(hom._h, _lib.ptr(ebar)))
            hom.set_reference(ReferenceMaterial(lam=float(lam_mu[0]), mu=float(lam_mu[1])))
        else:
            hom._ebar_n = ebar
            _lib.check(lib.am_solver_commit(hom._h, _lib.ptr(ebar)))
        hom._state_dirty = True
        if k == len(times) - 1 and comm is None:
            hom.grid.state  # noqa: B018  (refresh the host copy of the final state)
        records.append({
            "step": k, "time": float(times[k]), "eps_xx": float(ebar[0]), "sig": sig_bar.copy(),
            "C11": C11, "C12": C12, "iterations": info.iterations, "mean_substeps": info.mean_substeps,
        })
    return records
