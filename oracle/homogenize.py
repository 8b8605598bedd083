"""numpy restatement of the Moulinec-Suquet basic scheme -- TEST INFRASTRUCTURE ONLY.

CPU checker for the GPU solver (paper_2006_04391_b200/csrc/solver.cu); only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline arm may use it.
It restates gsmkit/homogenize.py step by step:

* ``green_matrix``        GreenOperator._assemble + Nyquist/origin rules (homogenize.py:184-227)
* ``green_apply``         GreenOperator.apply (homogenize.py:229-233)
* ``green_apply_slabwise`` the same with the table built per kx slab (512^3 checks)
* ``residual``            equilibrium_residual (homogenize.py:241-267)
* ``iso``                 apply_isotropic (homogenize.py:270-281)
* ``reference_update``    reference_update with the Mandel / deviatoric basis (homogenize.py:288-329)
* ``Basic``               Homogenizer.solve_step / commit_step / evaluate_field (homogenize.py:345-480)
* ``loading_path``        run_loading_path (homogenize.py:485-528)

The per-voxel material laws are evaluated by the C oracle (oracle/material.py),
so the whole chain is independent of the product code.  Pinned against the
fixtures the reference produced (tests/golden, tests/test_oracle_homogenize.py).
"""

import numpy as np

from . import material as OM

VOIGT = ((0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1))
DUP = np.array([1.0, 1.0, 1.0, 2.0, 2.0, 2.0])


def iso_matrix(lam, mu):
    C = np.zeros((6, 6))
    C[:3, :3] = lam
    C[[0, 1, 2], [0, 1, 2]] = lam + 2.0 * mu
    C[[3, 4, 5], [3, 4, 5]] = mu
    return C


def _freqs(dims):
    nx, ny, nz = dims
    return np.fft.fftfreq(nx, 1.0 / nx), np.fft.fftfreq(ny, 1.0 / ny), np.fft.rfftfreq(nz, 1.0 / nz)


def _unit(dims):
    fx, fy, fz = _freqs(dims)
    xi = np.stack(np.meshgrid(fx, fy, fz, indexing="ij"))
    nrm = np.sqrt((xi**2).sum(axis=0))
    nrm[0, 0, 0] = 1.0
    return xi / nrm, (fx, fy, fz)


def green_matrix(dims, lam, mu):
    """(6, 6, nx, ny, nz//2+1) table of the isotropic Green operator."""
    n, (fx, fy, fz) = _unit(dims)
    c1 = 1.0 / (4.0 * mu)
    c2 = (lam + mu) / (mu * (lam + 2.0 * mu))
    G = np.empty((6, 6) + n.shape[1:])
    for p, (k, h) in enumerate(VOIGT):
        for q, (i, j) in enumerate(VOIGT):
            t = c1 * ((k == i) * n[h] * n[j] + (h == i) * n[k] * n[j] + (k == j) * n[h] * n[i] + (h == j) * n[k] * n[i])
            G[p, q] = (2.0 if p > 2 else 1.0) * (2.0 if q > 2 else 1.0) * (t - c2 * n[i] * n[j] * n[k] * n[h])
    nx, ny, nz = dims
    nyq = ((np.abs(np.abs(fx) - nx / 2.0) < 1e-9)[:, None, None]
           | (np.abs(np.abs(fy) - ny / 2.0) < 1e-9)[None, :, None]
           | (np.abs(np.abs(fz) - nz / 2.0) < 1e-9)[None, None, :])
    if nyq.any():
        G[:, :, nyq] = np.linalg.inv(iso_matrix(lam, mu))[:, :, None]
    G[:, :, 0, 0, 0] = 0.0
    return G


def green_apply(tau, lam, mu, G=None):
    dims = tau.shape[1:]
    G = green_matrix(dims, lam, mu) if G is None else G
    th = np.fft.rfftn(tau, axes=(1, 2, 3))
    return np.fft.irfftn(-np.einsum("pqxyz,qxyz->pxyz", G, th), s=dims, axes=(1, 2, 3))


def green_apply_slabwise(tau, lam, mu, kx_chunk=16):
    """green_apply with the Green table built kx-slab by kx-slab (the full
    (6, 6, nx, ny, nz/2+1) table is 18 GiB at 512^3); same formulas and
    Nyquist / origin rules as green_matrix (homogenize.py:184-233)."""
    dims = tau.shape[1:]
    nx, ny, nz = dims
    fx, fy, fz = _freqs(dims)
    c1 = 1.0 / (4.0 * mu)
    c2 = (lam + mu) / (mu * (lam + 2.0 * mu))
    Cinv = np.linalg.inv(iso_matrix(lam, mu))
    nyq_y = np.abs(np.abs(fy) - ny / 2.0) < 1e-9
    nyq_z = np.abs(np.abs(fz) - nz / 2.0) < 1e-9
    th = np.fft.rfftn(tau, axes=(1, 2, 3))
    for x0 in range(0, nx, kx_chunk):
        x1 = min(nx, x0 + kx_chunk)
        xi = np.stack(np.meshgrid(fx[x0:x1], fy, fz, indexing="ij"))
        nrm = np.sqrt((xi**2).sum(axis=0))
        if x0 == 0:
            nrm[0, 0, 0] = 1.0
        n = xi / nrm
        out = np.zeros((6,) + n.shape[1:], dtype=complex)
        nyq = ((np.abs(np.abs(fx[x0:x1]) - nx / 2.0) < 1e-9)[:, None, None] | nyq_y[None, :, None]
               | nyq_z[None, None, :])
        for p, (k, h) in enumerate(VOIGT):
            for q, (i, j) in enumerate(VOIGT):
                t = c1 * ((k == i) * n[h] * n[j] + (h == i) * n[k] * n[j] + (k == j) * n[h] * n[i]
                          + (h == j) * n[k] * n[i])
                G = (2.0 if p > 2 else 1.0) * (2.0 if q > 2 else 1.0) * (t - c2 * n[i] * n[j] * n[k] * n[h])
                G[nyq] = Cinv[p, q]
                if x0 == 0:
                    G[0, 0, 0] = 0.0
                out[p] -= G * th[q, x0:x1]
        th[:, x0:x1] = out
    return np.fft.irfftn(th, s=dims, axes=(1, 2, 3))


def residual(sig):
    dims = sig.shape[1:]
    n, _ = _unit(dims)
    sh = np.fft.rfftn(sig, axes=(1, 2, 3))
    t0 = n[0] * sh[0] + n[1] * sh[5] + n[2] * sh[4]
    t1 = n[0] * sh[5] + n[1] * sh[1] + n[2] * sh[3]
    t2 = n[0] * sh[4] + n[1] * sh[3] + n[2] * sh[2]
    sq = np.abs(t0) ** 2 + np.abs(t1) ** 2 + np.abs(t2) ** 2
    sq[0, 0, 0] = 0.0
    w = np.full(sq.shape, 2.0)
    w[..., 0] = 1.0
    if dims[2] % 2 == 0:
        w[..., -1] = 1.0
    N = np.prod(dims)
    sbar = sig.mean(axis=(1, 2, 3))
    return np.sqrt((w * sq).sum() / N**2) / max(np.sqrt(np.sum(sbar * DUP * sbar)), 1e-300)


def iso(lam, mu, e):
    tr = e[0] + e[1] + e[2]
    out = np.empty_like(e)
    for i in range(3):
        out[i] = lam * tr + 2.0 * mu * e[i]
        out[3 + i] = mu * e[3 + i]
    return out


def _dev_basis():
    vol = np.array([1.0, 1.0, 1.0, 0.0, 0.0, 0.0]) / np.sqrt(3.0)
    out = []
    for e in np.eye(6):
        v = e - (e @ vol) * vol
        for b in out:
            v = v - (v @ b) * b
        if np.linalg.norm(v) > 1e-12:
            out.append(v / np.linalg.norm(v))
    return vol, np.stack(out[:5], axis=1)


def reference_update(C):
    C = np.asarray(C, dtype=float).reshape(-1, 6, 6)
    if not np.all(np.isfinite(C)):
        raise ValueError("tangent field contains non-finite entries")
    vol, B = _dev_basis()
    M = np.diag([1.0, 1.0, 1.0, np.sqrt(2.0), np.sqrt(2.0), np.sqrt(2.0)])
    S = 0.5 * (C + np.swapaxes(C, 1, 2))
    H = M @ S @ M
    kappa = np.einsum("i,bij,j->b", vol, H, vol) / 3.0
    ev = np.linalg.eigvalsh(np.einsum("ip,bij,jq->bpq", B, H, B))
    mu = 0.5 * (ev[:, 0].min() / 2.0 + ev[:, -1].max() / 2.0)
    kap = 0.5 * (kappa.min() + kappa.max())
    return kap - 2.0 * mu / 3.0, mu


class NotConverged(RuntimeError):
    def __init__(self, history):
        super().__init__("basic scheme did not converge")
        self.history = history


class Basic:
    """Homogenizer restated; ``laws`` are oracle.material law tuples per material id."""

    def __init__(self, ids, laws, tol=1e-5, max_iterations=5000, threads=8):
        self.ids = np.asarray(ids)
        self.dims = self.ids.shape
        self.laws = laws
        self.tol = tol
        self.max_iterations = max_iterations
        self.threads = threads
        flat = self.ids.reshape(-1)
        self.index = [np.flatnonzero(flat == k) for k in range(len(laws))]
        self.state = [np.zeros((len(i), 7 if law[0] == 1 else 0)) for i, law in zip(self.index, laws)]
        self.eps_n = np.zeros((6,) + self.dims)
        self.ebar_n = np.zeros(6)
        self.pending = None
        Ce = [iso_matrix(*_lame(law)) for law, i in zip(laws, self.index) if len(i)]
        self.lam, self.mu = reference_update(np.stack(Ce))

    def evaluate(self, eps, dt, tangent=False):
        N = int(np.prod(self.dims))
        sig = np.zeros((6, N))
        C = np.zeros((N, 6, 6)) if tangent else None
        en, ep = self.eps_n.reshape(6, -1), eps.reshape(6, -1)
        new = []
        for law, idx, a in zip(self.laws, self.index, self.state):
            if not len(idx):
                new.append(a.copy())
                continue
            r = OM.evaluate(law, en[:, idx].T, a, ep[:, idx].T, np.full(len(idx), dt), tangent, threads=self.threads)
            if np.any(r["status"] & OM.ST_NEWTON):
                raise RuntimeError("NewtonDivergenceError")
            sig[:, idx] = r["sigma"].T
            if tangent:
                C[idx] = r["C"]
            new.append(r["a"])
        return sig.reshape((6,) + self.dims), C, new

    def solve_step(self, ebar_target, dt, free=None):
        free = np.zeros(6, dtype=bool) if free is None else np.asarray(free, dtype=bool)
        ebar = np.array(ebar_target, dtype=float)
        ebar[free] = self.ebar_n[free]
        eps = self.eps_n + (ebar - self.ebar_n)[:, None, None, None]
        G = green_matrix(self.dims, self.lam, self.mu)
        Cff = iso_matrix(self.lam, self.mu)[np.ix_(free, free)]
        hist = []
        for it in range(1, self.max_iterations + 1):
            sig, _, st = self.evaluate(eps, dt)
            sbar = sig.mean(axis=(1, 2, 3))
            res = residual(sig)
            scale = max(np.sqrt(np.sum(sbar * DUP * sbar)), 1e-300)
            rbc = np.linalg.norm(sbar[free]) / scale if free.any() else 0.0
            hist.append(max(res, rbc))
            if res < self.tol and rbc < self.tol:
                self.pending = st
                return eps, sig, it, hist
            fl = green_apply(sig - iso(self.lam, self.mu, eps), self.lam, self.mu, G)
            if free.any():
                ebar[free] += np.linalg.solve(Cff, -sbar[free])
            eps = ebar[:, None, None, None] + fl
        raise NotConverged(hist)

    def commit(self, eps, ebar):
        self.eps_n = eps
        self.ebar_n = np.array(ebar, dtype=float)
        if self.pending is not None:
            self.state = self.pending
            self.pending = None


def _lame(law):
    E, nu = law[1][0], law[1][1]
    return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))


def loading_times(steps, rate=1.4e-3, eps_max=3.58454e-3, eps_min=-3.48441e-3):
    """LoadingPath.times / eps_xx (homogenize.py:52-77)."""
    T = (eps_max + (eps_max - eps_min)) / rate
    t = np.linspace(0.0, T, steps + 1)
    turn = eps_max / rate
    return t, np.where(t <= turn, rate * t, eps_max - rate * (t - turn))


def loading_path(ids, laws, steps, n_steps=None, threads=8, tol=1e-5):
    """run_loading_path with mixed BCs and reference updates; first n_steps steps."""
    b = Basic(ids, laws, tol=tol, threads=threads)
    t, ex = loading_times(steps)
    free = np.array([False, True, True, True, True, True])
    recs = []
    for k in range(1, (n_steps or steps) + 1):
        dt = t[k] - t[k - 1]
        target = np.zeros(6)
        target[0] = ex[k]
        eps, sig, it, hist = b.solve_step(target, dt, free)
        ebar = eps.mean(axis=(1, 2, 3))
        _, C, _ = b.evaluate(eps, dt, True)
        Cb = C.mean(axis=0)
        b.commit(eps, ebar)
        b.lam, b.mu = reference_update(C)
        recs.append(dict(step=k, eps_xx=ebar[0], sig=sig.mean(axis=(1, 2, 3)), C11=Cb[0, 0], C12=Cb[0, 1],
                         iterations=it, lam=b.lam, mu=b.mu))
    return recs, b
