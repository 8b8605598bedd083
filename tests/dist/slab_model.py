"""numpy + torch.distributed model of the basic scheme's slab decomposition.

Restates, for CPU tests over gloo, the data movement of csrc/solver.cu's
multi-slab algorithm: x-slabs (6, nx/k, ny, nz) in real space; forward =
2-D rfft over (y, z) -> k_pack to blocks [dest][xl][c][ky_local][kz] ->
all-to-all -> 1-D fft over x, giving the ky-slab layout [kx][c][ky_local][kz];
inverse mirrors it (1-D ifft over x -> all-to-all -> k_unpack -> 2-D irfft).
Test infrastructure only.
"""

import numpy as np
import torch
import torch.distributed as dist


def pack(P, k):
    """k_pack: P (6, nxl, ny, nzh) -> send (k, nxl, 6, nyl, nzh)."""
    six, nxl, ny, nzh = P.shape
    nyl = ny // k
    return np.ascontiguousarray(P.reshape(6, nxl, k, nyl, nzh).transpose(2, 1, 0, 3, 4))


def unpack(R, ny):
    """k_unpack: recv (k, nxl, 6, nyl, nzh) -> P (6, nxl, ny, nzh)."""
    k, nxl, six, nyl, nzh = R.shape
    return np.ascontiguousarray(R.transpose(2, 1, 0, 3, 4).reshape(6, nxl, ny, nzh))


def alltoall(buf):
    """Equal-block all-to-all of a complex array whose leading axis is the peer."""
    x = torch.from_numpy(np.ascontiguousarray(buf).view(np.float64).reshape(-1))
    y = torch.empty_like(x)
    dist.all_to_all_single(y, x)
    return y.numpy().view(np.complex128).reshape(buf.shape)


def forward(field, nx):
    """x-slab real field (6, nxl, ny, nz) -> ky-slab spectrum (nx, 6, nyl, nzh)."""
    k = dist.get_world_size()
    P = np.fft.rfftn(field, axes=(2, 3))
    R = alltoall(pack(P, k))  # (k src, nxl, 6, nyl, nzh) == (nx, 6, nyl, nzh)
    S = R.reshape(nx, 6, R.shape[3], R.shape[4])
    return np.fft.fft(S, axis=0)


def inverse(S, ny, nz):
    """ky-slab spectrum (nx, 6, nyl, nzh) -> x-slab real field (6, nxl, ny, nz)."""
    k = dist.get_world_size()
    nx = S.shape[0]
    T = np.fft.ifft(S, axis=0) * nx  # unnormalised like cuFFT's inverse
    send = T.reshape(k, nx // k, 6, S.shape[2], S.shape[3])
    R = alltoall(send)
    P = unpack(R, ny)
    return np.fft.irfftn(P, s=(ny, nz), axes=(2, 3)) * (ny * nz)


def plane_partials(S, y0, ny, nzh, parts=8):
    """k_fourier's reduction slots: per global ky plane and part, the sum over
    its (kx, kz) bins of a per-bin value (here |S_0|^2)."""
    nx, _, nyl, _ = S.shape
    out = np.zeros(ny * parts)
    v = np.abs(S[:, 0]) ** 2  # (nx, nyl, nzh)
    nb = nx * nzh
    for kyl in range(nyl):
        flat = v[:, kyl, :].reshape(-1)  # j = kx * nzh + kz
        for p in range(parts):
            lo, hi = nb * p // parts, nb * (p + 1) // parts
            out[(y0 + kyl) * parts + p] = flat[lo:hi].sum()
    return out
