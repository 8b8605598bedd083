// solver.cu -- the Moulinec-Suquet basic scheme (gsmkit homogenize.py:
// Homogenizer, GreenOperator, equilibrium_residual, reference_update,
// apply_isotropic) on one or more GPUs, and its C-ABI (am_solver_*,
// am_*_host).
//
// The grid is decomposed into x-slabs ("ranks").  A solver handle drives
// either
//   * all slabs of the grid from one process on the current device (local
//     mode: nslabs = 1 is the plain single-GPU solver; nslabs > 1 runs the
//     distributed algorithm with device-to-device copies as the transport,
//     which is how the slab code is tested on a single B200), or
//   * exactly one slab per process with an NCCL communicator over
//     NVLink / NVSwitch (nccl mode, one process per GPU).
//
// Device-resident state per slab (component-major SoA, fp64):
//   eps, eps_n, sigma (6, nxl, ny, nz)   strain iterate, committed strain, stress
//   S, ehat                             spectra of sigma / of eps (complex128)
//   per phase: slab-local gather index, committed + pending internal states
// Spectral layout: one slab: cuFFT's (6, nx, ny, nz/2+1); several slabs:
// ky-slabs [kx][c][ky_local][kz], the layout the x-transposes produce.
//
// One basic-scheme iteration (homogenize.py:445-465):
//   K1    sigma = material(eps_n, a_n, eps) per phase (gathered)
//   FFT   S = rfft(sigma)   3-D D2Z, or 2-D D2Z + pack + all-to-all + 1-D FFT(x)
//   K2    residual partials per (ky plane, part) and, for every bin but 0,
//         ehat' = -Gamma0 (S - C0 ehat) -> ehat, ehat'/N -> S
//   red   fixed-order partials (independent of the slab count) -> host
//   host  strict convergence test, mixed-BC solve (homogenize.py:454-464)
//   bin0  ehat(0) = N ebar;  eps = irfft(S)  (inverse of FFT above)
// Carrying ehat replaces the reference's FFT of tau = sigma - C0:eps
// (6 forward + 6 inverse transforms per iteration instead of 12 + 6).
#include <cufft.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "fft_cb.h"
#include "fourier.cuh"
#include "k1.cuh"
#include "laws.cuh"
#include "refupdate.cuh"
#include "xfused.cuh"

namespace am {

#define AM_CUFFT(expr)                                                                      \
    do {                                                                                    \
        cufftResult _r = (expr);                                                            \
        if (_r != CUFFT_SUCCESS) return ::am::fail(AM_ERR_CUDA, "%s:%d %s: cufft error %d", \
                                                   __FILE__, __LINE__, #expr, (int)_r);     \
    } while (0)
#define AM_NCCL(expr)                                                                        \
    do {                                                                                     \
        ncclResult_t _r = (expr);                                                            \
        if (_r != ncclSuccess) return ::am::fail(AM_ERR_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, \
                                                 #expr, ncclGetErrorString(_r));             \
    } while (0)

struct Vec6 {
    double v[6];
};

constexpr int kRedThreads = 256;
constexpr int kParts = 8;            // blocks per ky plane in the residual: fixed, so the
                                     // reduction order never depends on the slab count
constexpr int kRedBlocks = 148 * 4;  // k_refstats / standalone reductions

// ---------------------------------------------------------------- layouts
// spectral layout of one slab; bin (kx, ky_local, kz) of component c lives
// at c * cs + kx * xs + kyl * nzh + kz
struct Spec {
    int nx, ny, nz, nzh;
    int y0, nyl;
    int64_t cs, xs;
    int64_t N;  // global voxel count (normalisation)
};

static Spec spec_single(int nx, int ny, int nz) {
    const int nzh = nz / 2 + 1;
    return Spec{nx, ny, nz, nzh, 0, ny, (int64_t)nx * ny * nzh, (int64_t)ny * nzh, (int64_t)nx * ny * nz};
}
static Spec spec_slab(int nx, int ny, int nz, int y0, int nyl) {
    const int nzh = nz / 2 + 1;
    return Spec{nx, ny, nz, nzh, y0, nyl, (int64_t)nyl * nzh, (int64_t)6 * nyl * nzh, (int64_t)nx * ny * nz};
}

// ---------------------------------------------------------------- kernels
__device__ __forceinline__ double block_sum(double v, double* sh) {
    // deterministic: warp shuffle tree, then the warps' partials in order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
    __syncthreads();
    return s;
}

// eps = eps_n + d (start of a loading step, homogenize.py:439); n per component
__global__ void k_shift(double* __restrict__ eps, const double* __restrict__ eps_n, Vec6 d, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int c = 0; c < 6; ++c) eps[c * n + i] = eps_n[c * n + i] + d.v[c];
}

// K2: residual partials + Green update for every bin of the slab but the
// global origin.  Block b handles part (b % kParts) of ky plane (b / kParts);
// its partial goes to red[(y0 + kyl) * kParts + part].
// S: rfft(sigma) in, ehat'/N out (scaled = 0: S untouched, the inverse
// transform reads ehat' / N through its load callback, fft_cb.cu);
// ehat: rfft(eps) in, ehat' out.
#ifndef AM_FOURIER_MINB
#define AM_FOURIER_MINB 1
#endif
#ifndef AM_FOURIER_EARLY
#define AM_FOURIER_EARLY 1
#endif
__global__ void __launch_bounds__(kRedThreads, AM_FOURIER_MINB) k_fourier(Spec sp, RefMat ref, double2* __restrict__ S,
                                                         double2* __restrict__ ehat, double* __restrict__ red,
                                                         int update, int scaled) {
    __shared__ double sh[kRedThreads / 32];
    const int kyl = blockIdx.x / kParts, part = blockIdx.x % kParts;
    const int ky = sp.y0 + kyl;
    const int64_t nb = (int64_t)sp.nx * sp.nzh;
    const int64_t lo = nb * part / kParts, hi = nb * (part + 1) / kParts;
    const double invN = 1.0 / (double)sp.N;
    double acc = 0.0;
    for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) {
        const int kx = (int)(j / sp.nzh), kz = (int)(j % sp.nzh);
        const int64_t q = kx * sp.xs + (int64_t)kyl * sp.nzh + kz;
        const Bin b = make_bin(kx, ky, kz, sp.nx, sp.ny, sp.nz);
        cplx s[6];
#if AM_FOURIER_EARLY
        // both spectra's loads in flight together (one memory latency per bin)
        double2 ev[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            const double2 v = S[c * sp.cs + q];
            s[c] = cplx{v.x, v.y};
            ev[c] = update ? ehat[c * sp.cs + q] : make_double2(0.0, 0.0);
        }
#else
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            const double2 v = S[c * sp.cs + q];
            s[c] = cplx{v.x, v.y};
        }
#endif
        if (!b.zero) acc += rfft_weight(kz, sp.nz) * traction_sq(b, s);
        if (update && !b.zero) {
            double er[6], ei[6], cr[6], ci[6], tr[6], ti[6], outr[6], outi[6];
#pragma unroll
            for (int c = 0; c < 6; ++c) {
#if AM_FOURIER_EARLY
                const double2 v = ev[c];
#else
                const double2 v = ehat[c * sp.cs + q];
#endif
                er[c] = v.x;
                ei[c] = v.y;
            }
            iso_apply(ref, er, cr);
            iso_apply(ref, ei, ci);
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                tr[c] = s[c].re - cr[c];
                ti[c] = s[c].im - ci[c];
            }
            green_apply_real(ref, b, tr, outr);
            green_apply_real(ref, b, ti, outi);
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                ehat[c * sp.cs + q] = make_double2(outr[c], outi[c]);
                if (scaled) S[c * sp.cs + q] = make_double2(outr[c] * invN, outi[c] * invN);
            }
        }
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) red[(int64_t)ky * kParts + part] = t;
}

// k_fourier with the next bin's spectra loaded before the current bin's
// results are stored (software pipelining; AM_FOURIER_PF=1)
__global__ void __launch_bounds__(kRedThreads, AM_FOURIER_MINB) k_fourier_pf(Spec sp, RefMat ref, double2* __restrict__ S,
                                                            double2* __restrict__ ehat, double* __restrict__ red,
                                                            int update, int scaled) {
    __shared__ double sh[kRedThreads / 32];
    const int kyl = blockIdx.x / kParts, part = blockIdx.x % kParts;
    const int ky = sp.y0 + kyl;
    const int64_t nb = (int64_t)sp.nx * sp.nzh;
    const int64_t lo = nb * part / kParts, hi = nb * (part + 1) / kParts;
    const double invN = 1.0 / (double)sp.N;
    double acc = 0.0;
    auto qof = [&](int64_t j) { return (int64_t)(j / sp.nzh) * sp.xs + (int64_t)kyl * sp.nzh + (int)(j % sp.nzh); };
    double2 sv[6], ev[6];
    int64_t j = lo + threadIdx.x;
    if (j < hi) {
        const int64_t q = qof(j);
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            sv[c] = S[c * sp.cs + q];
            ev[c] = update ? ehat[c * sp.cs + q] : make_double2(0.0, 0.0);
        }
    }
    for (; j < hi; j += blockDim.x) {
        const int kx = (int)(j / sp.nzh), kz = (int)(j % sp.nzh);
        const int64_t q = kx * sp.xs + (int64_t)kyl * sp.nzh + kz;
        const Bin b = make_bin(kx, ky, kz, sp.nx, sp.ny, sp.nz);
        cplx s[6];
        double2 e[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            s[c] = cplx{sv[c].x, sv[c].y};
            e[c] = ev[c];
        }
        const int64_t jn = j + blockDim.x;
        if (jn < hi) {  // the next bin's loads in flight during this bin's work
            const int64_t qn = qof(jn);
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                sv[c] = S[c * sp.cs + qn];
                ev[c] = update ? ehat[c * sp.cs + qn] : make_double2(0.0, 0.0);
            }
        }
        if (!b.zero) acc += rfft_weight(kz, sp.nz) * traction_sq(b, s);
        if (update && !b.zero) {
            double er[6], ei[6], cr[6], ci[6], tr[6], ti[6], outr[6], outi[6];
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                er[c] = e[c].x;
                ei[c] = e[c].y;
            }
            iso_apply(ref, er, cr);
            iso_apply(ref, ei, ci);
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                tr[c] = s[c].re - cr[c];
                ti[c] = s[c].im - ci[c];
            }
            green_apply_real(ref, b, tr, outr);
            green_apply_real(ref, b, ti, outi);
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                ehat[c * sp.cs + q] = make_double2(outr[c], outi[c]);
                if (scaled) S[c * sp.cs + q] = make_double2(outr[c] * invN, outi[c] * invN);
            }
        }
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) red[(int64_t)ky * kParts + part] = t;
}

// per-(x plane, component) sums of a slab field f (6, nxl, ny, nz) ->
// out[(x0 + x) * 6 + c]: fixed per-thread strides and a fixed tree, so the
// host's plane-ordered sum (field_means) is independent of the slab count
__global__ void __launch_bounds__(kRedThreads) k_plane_sums(const double* __restrict__ f, int64_t Nl, int64_t plane,
                                                            int x0, double* __restrict__ out) {
    __shared__ double sh[kRedThreads / 32];
    const int x = blockIdx.x, c = blockIdx.y;
    const double* p = f + c * Nl + (int64_t)x * plane;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < plane; i += blockDim.x) acc += p[i];
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) out[(int64_t)(x0 + x) * 6 + c] = t;
}

// red[P*ny + 0..5] = Re S(origin) on the origin's owner (else 0),
// red[P*ny + 6] = 1 if a material point's Newton failed, [7] = 1 if an
// adaptive integration hit a cap, [8] = accepted substeps of the adaptive
// kernels in the sweep, [9] = 1 if a radial return stalled (summed over
// slabs: all exact)
__global__ void k_finish(const double2* __restrict__ S, int64_t cs, int owner, const uint32_t* __restrict__ flags,
                         const unsigned long long* __restrict__ subs, double* __restrict__ red, int64_t off) {
    const int c = threadIdx.x;
    if (c < 6) red[off + c] = owner ? S[c * cs].x : 0.0;
    if (c == 6) red[off + 6] = (flags && (*flags & AM_VOXEL_NEWTON_FAILED)) ? 1.0 : 0.0;
    if (c == 7) red[off + 7] = (flags && (*flags & AM_VOXEL_INTEGRATION)) ? 1.0 : 0.0;
    if (c == 8) red[off + 8] = subs ? (double)*subs : 0.0;
    if (c == 9) red[off + 9] = (flags && (*flags & AM_VOXEL_RADIAL)) ? 1.0 : 0.0;
}

// origin bin of the update: ehat(0) = N ebar, inverse-FFT input ebar
__global__ void k_origin(double2* S, double2* ehat, int64_t cs, Vec6 ebar, double N) {
    const int c = threadIdx.x;
    if (c < 6) {
        ehat[c * cs] = make_double2(ebar.v[c] * N, 0.0);
        S[c * cs] = make_double2(ebar.v[c], 0.0);
    }
}

// the same with the mean strain read from device memory (graph replays;
// S = nullptr: the inverse transform's load callback reads ebar itself)
__global__ void k_origin_dev(double2* S, double2* ehat, int64_t cs, const double* __restrict__ ebar, double N) {
    const int c = threadIdx.x;
    if (c < 6) {
        ehat[c * cs] = make_double2(ebar[c] * N, 0.0);
        if (S) S[c * cs] = make_double2(ebar[c], 0.0);
    }
}

// origin of the fused update (xfused.cuh) once the host has the new mean
// strain: ehat(0) = N ebar, and the inverse x transform of the origin bin,
// ebar along the (ky, kz) = 0 line of the 2-D spectra
__global__ void k_origin_x(double2* __restrict__ S, double2* __restrict__ ehat, int64_t cs, int64_t xs, int nx,
                           Vec6 ebar, double N) {
    const int c = blockIdx.x;
    for (int x = threadIdx.x; x < nx; x += blockDim.x) {
        double2 v = S[c * cs + x * xs];
        v.x += ebar.v[c];
        S[c * cs + x * xs] = v;
    }
    if (threadIdx.x == 0) ehat[c * cs] = make_double2(ebar.v[c] * N, 0.0);
}

// Transposes between the x-slab 2-D spectra P (6, nxl, ny, nzh) and the
// exchange blocks [rank j][xl][c][kyl][kz] (equal ky ranges nyl per slab).
// For a fixed (j, xl, c) both sides are one contiguous run of nyl * nzh
// elements, so every kernel is a batch of contiguous copies: block row
// blockIdx.y = run r = (j * nxl + xl) * 6 + c, threads over the run (no
// per-element index arithmetic, coalesced 16-byte accesses on both sides).
__device__ __forceinline__ void run_of(int r, int nxl, int& j, int& xl, int& c) {
    c = r % 6;
    xl = (r / 6) % nxl;
    j = r / (6 * nxl);
}

// forward transpose, pack: P -> send
__global__ void k_pack(const double2* __restrict__ P, double2* __restrict__ send, int nxl, int ny, int nzh, int nyl) {
    int j, xl, c;
    run_of(blockIdx.y, nxl, j, xl, c);
    const int64_t len = (int64_t)nyl * nzh;
    const double2* src = P + ((int64_t)(c * nxl + xl) * ny + (int64_t)j * nyl) * nzh;
    double2* dst = send + (int64_t)blockIdx.y * len;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// inverse transpose, unpack: receive blocks [src j][xl][c][kyl][kz] -> P
__global__ void k_unpack(const double2* __restrict__ recv, double2* __restrict__ P, int nxl, int ny, int nzh, int nyl) {
    int j, xl, c;
    run_of(blockIdx.y, nxl, j, xl, c);
    const int64_t len = (int64_t)nyl * nzh;
    const double2* src = recv + (int64_t)blockIdx.y * len;
    double2* dst = P + ((int64_t)(c * nxl + xl) * ny + (int64_t)j * nyl) * nzh;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// Fused transposes over peer memory (NVLink P2P / same-device siblings):
// the pack kernel stores each destination's block straight into that
// rank's spectrum buffer (peer[j] + rank * blk + ...), so pack and
// all-to-all are one pass; the inverse reads each source's block straight
// from that rank's spectrum buffer.  `peer` is a device array of the k
// ranks' buffers.
__global__ void k_pack_peer(const double2* __restrict__ P, double2* const* __restrict__ peer, int rank, int nxl, int ny,
                            int nzh, int nyl) {
    int j, xl, c;
    run_of(blockIdx.y, nxl, j, xl, c);
    const int64_t len = (int64_t)nyl * nzh, blk = (int64_t)nxl * 6 * len;
    const double2* src = P + ((int64_t)(c * nxl + xl) * ny + (int64_t)j * nyl) * nzh;
    double2* dst = peer[j] + rank * blk + (int64_t)(xl * 6 + c) * len;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
    __threadfence_system();  // remote stores visible before the barrier that follows
}

__global__ void k_unpack_peer(double2* const* __restrict__ peer, double2* __restrict__ P, int rank, int nxl, int ny,
                              int nzh, int nyl) {
    int j, xl, c;
    run_of(blockIdx.y, nxl, j, xl, c);
    const int64_t len = (int64_t)nyl * nzh, blk = (int64_t)nxl * 6 * len;
    const double2* src = peer[j] + rank * blk + (int64_t)(xl * 6 + c) * len;
    double2* dst = P + ((int64_t)(c * nxl + xl) * ny + (int64_t)j * nyl) * nzh;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// standalone Green application on a single-layout spectrum (GreenOperator.apply):
// every bin, origin -> 0, output scaled by 1/N for the Z2D
__global__ void k_green(Spec sp, RefMat ref, double2* __restrict__ h) {
    const double invN = 1.0 / (double)sp.N;
    const int64_t nbins = (int64_t)sp.nx * sp.ny * sp.nzh;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nbins; q += (int64_t)gridDim.x * blockDim.x) {
        const int kz = (int)(q % sp.nzh);
        const int64_t r = q / sp.nzh;
        const int ky = (int)(r % sp.ny), kx = (int)(r / sp.ny);
        const Bin b = make_bin(kx, ky, kz, sp.nx, sp.ny, sp.nz);
        double tr[6], ti[6], outr[6], outi[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            tr[c] = h[c * sp.cs + q].x;
            ti[c] = h[c * sp.cs + q].y;
        }
        green_apply_real(ref, b, tr, outr);
        green_apply_real(ref, b, ti, outi);
#pragma unroll
        for (int c = 0; c < 6; ++c)
            h[c * sp.cs + q] = b.zero ? make_double2(0.0, 0.0) : make_double2(outr[c] * invN, outi[c] * invN);
    }
}

// C_ref : eps over a (6, N) field
__global__ void k_isotropic(RefMat ref, const double* __restrict__ e, double* __restrict__ out, int64_t N) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        double x[6], y[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) x[c] = e[c * N + i];
        iso_apply(ref, x, y);
#pragma unroll
        for (int c = 0; c < 6; ++c) out[c * N + i] = y[c];
    }
}

// K5: per-voxel tangent bounds + C sums over tangents stored
// C[(i*6+j)*cs + b], b = first, first + step, ... < end.  Block results:
// sums[0..35] = sum C, sums[36] = non-finite count; mins[0..3] = min kappa,
// -max kappa, min mu_lo, -max mu_hi (all four combine by min, in any order)
constexpr int kStat = 41;
constexpr int kSum = 37;
constexpr int kSParts = 16;  // blocks per (phase, x plane) in the tangent sweep statistics
__device__ void refstats_block(const double* __restrict__ C, int64_t cs, int64_t first, int64_t step, int64_t end,
                               const DevBasis& db, double* __restrict__ sums, double* __restrict__ mins) {
    __shared__ double sh[kRedThreads / 32];
    __shared__ double red[kRedThreads];
    double sum[36];
#pragma unroll
    for (int i = 0; i < 36; ++i) sum[i] = 0.0;
    double kmin = INFINITY, kmax = -INFINITY, mlo = INFINITY, mhi = -INFINITY, bad = 0.0;
    for (int64_t b = first; b < end; b += step) {
        double c[6][6];
        bool fin = true;
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
            for (int j = 0; j < 6; ++j) {
                c[i][j] = C[(i * 6 + j) * cs + b];
                sum[i * 6 + j] += c[i][j];
                fin = fin && (c[i][j] - c[i][j] == 0.0);
            }
        if (!fin) {
            bad += 1.0;
            continue;
        }
        double k, lo, hi;
        tangent_bounds(c, db, k, lo, hi);
        kmin = fmin(kmin, k);
        kmax = fmax(kmax, k);
        mlo = fmin(mlo, lo);
        mhi = fmax(mhi, hi);
    }
#pragma unroll
    for (int i = 0; i < 36; ++i) {
        const double t = block_sum(sum[i], sh);
        if (threadIdx.x == 0) sums[i] = t;
    }
    const double t = block_sum(bad, sh);
    if (threadIdx.x == 0) sums[36] = t;
    const double vals[4] = {kmin, -kmax, mlo, -mhi};
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        red[threadIdx.x] = vals[v];
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + s]);
            __syncthreads();
        }
        if (threadIdx.x == 0) mins[v] = red[0];
        __syncthreads();
    }
}

// reference_update of a stored tangent field: grid-stride blocks, record
// b at stats[b * kStat] = [sums (37) | mins (4)]
__global__ void __launch_bounds__(kRedThreads) k_refstats(const double* __restrict__ C, int64_t cs, int64_t B,
                                                          DevBasis db, double* __restrict__ stats) {
    double* out = stats + (int64_t)blockIdx.x * kStat;
    refstats_block(C, cs, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x, B, db, out,
                   out + kSum);
}

// tangent sweep chunk = x planes [xa, xa + gridDim.x / kSParts) of one phase;
// block (plane, part) reduces part `part` of the plane's voxels (gidx range
// poff[x] .. poff[x + 1], chunk-relative by `base`) into record
// (plane, part) at sums[rec * kSum] / mins[rec * 4].  Records are indexed by
// the global plane, so their plane-ordered sum does not depend on the chunk
// size, the slab count or the GPU count.
__global__ void __launch_bounds__(kRedThreads) k_refstats_planes(const double* __restrict__ C, int64_t cs,
                                                                 const int64_t* __restrict__ poff, int xa,
                                                                 int64_t base, DevBasis db, double* __restrict__ sums,
                                                                 double* __restrict__ mins) {
    const int x = xa + blockIdx.x / kSParts, part = blockIdx.x % kSParts;
    const int64_t p0 = poff[x] - base, n = poff[x + 1] - poff[x];
    const int64_t lo = p0 + n * part / kSParts, hi = p0 + n * (part + 1) / kSParts;
    refstats_block(C, cs, lo + threadIdx.x, blockDim.x, hi, db, sums + (int64_t)blockIdx.x * kSum,
                   mins + (int64_t)blockIdx.x * 4);
}

__global__ void k_fill(double* __restrict__ p, int64_t n, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// ---------------------------------------------------------------- host helpers
static unsigned grid_for(int64_t n, int threads = 256) {
    int64_t b = (n + threads - 1) / threads;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)kSMs * 32));
}

// dense solve with partial pivoting (numpy.linalg.solve / LAPACK gesv,
// homogenize.py:463) for the <= 6x6 mixed-BC system
static bool small_solve(int n, double* A, double* x) {
    int piv[6];
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (std::fabs(A[i * n + k]) > std::fabs(A[p * n + k])) p = i;
        piv[k] = p;
        if (A[p * n + k] == 0.0) return false;
        if (p != k)
            for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[p * n + j]);
        for (int i = k + 1; i < n; ++i) {
            A[i * n + k] /= A[k * n + k];
            for (int j = k + 1; j < n; ++j) A[i * n + j] -= A[i * n + k] * A[k * n + j];
        }
    }
    for (int k = 0; k < n; ++k)
        if (piv[k] != k) std::swap(x[k], x[piv[k]]);
    for (int i = 1; i < n; ++i)
        for (int k = 0; k < i; ++k) x[i] -= A[i * n + k] * x[k];
    for (int i = n - 1; i >= 0; --i) {
        for (int j = i + 1; j < n; ++j) x[i] -= A[i * n + j] * x[j];
        x[i] /= A[i * n + i];
    }
    return true;
}

static void ref_matrix(double lam, double mu, double* C) {
    for (int i = 0; i < 36; ++i) C[i] = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) C[i * 6 + j] = lam;
    for (int i = 0; i < 3; ++i) C[i * 6 + i] = lam + 2.0 * mu;
    for (int i = 3; i < 6; ++i) C[i * 6 + i] = mu;
}

static double dup_norm(const double* s) {
    // sqrt(sigma_bar . SHEAR_DUP . sigma_bar) (homogenize.py:266, 449)
    const double dup[6] = {1, 1, 1, 2, 2, 2};
    double t = 0.0;
    for (int i = 0; i < 6; ++i) t += s[i] * dup[i] * s[i];
    return std::sqrt(t);
}

struct Stats {
    double Csum[36];
    double kmin, kmax, mlo, mhi, bad;
    void reset() {
        for (double& c : Csum) c = 0.0;
        kmin = mlo = INFINITY;
        kmax = mhi = -INFINITY;
        bad = 0.0;
    }
    void add_sums(const double* s) {
        for (int i = 0; i < 36; ++i) Csum[i] += s[i];
        bad += s[36];
    }
    void add_mins(const double* m) {
        kmin = std::fmin(kmin, m[0]);
        kmax = std::fmax(kmax, -m[1]);
        mlo = std::fmin(mlo, m[2]);
        mhi = std::fmax(mhi, -m[3]);
    }
    void add(const double* s) {  // one k_refstats record
        add_sums(s);
        add_mins(s + kSum);
    }
};

// ---------------------------------------------------------------- slabs
struct Phase {
    am_law law;
    int m = 0;
    int64_t count = 0;        // voxels of this phase in the slab
    int64_t* gidx = nullptr;  // slab-local voxel indices (sorted)
    double* a_n = nullptr;
    double* a_pend = nullptr;  // state of the last converged solve_step (committed by am_solver_commit)
    double* a_tmp = nullptr;   // state of the last evaluation: basic-scheme iterates, evaluate, tangent sweep
    std::vector<int64_t> poff; // gidx range of slab x-plane x: [poff[x], poff[x + 1])
    int64_t* dpoff = nullptr;  // device copy
};

struct Slab {
    int rank = 0;
    int x0 = 0, nxl = 0;  // real-space x planes
    int y0 = 0, nyl = 0;  // spectral ky planes (multi-slab layout)
    int64_t Nl = 0;       // nxl * ny * nz
    Spec sp{};
    double *eps = nullptr, *eps_n = nullptr, *sigma = nullptr;
    double2 *S = nullptr, *ehat = nullptr;   // spectra
    double2 *P = nullptr, *X = nullptr;      // 2-D spectra / exchange buffer (multi-slab)
    uint32_t* flags = nullptr;
    unsigned long long* subs = nullptr;  // accepted substeps of the last sweep (adaptive integrators)
    double2** peerS = nullptr;  // device arrays: every rank's S / ehat (P2P transport)
    double2** peerE = nullptr;
    cufftHandle x1i = 0;        // inverse x transform reading ehat' / N through the load callback
    void* d_cbinfo = nullptr;   // its AmZ2DCb
    cufftHandle r2p = 0, c2u = 0;  // 2-D D2Z storing / Z2D loading through the transpose callbacks
    void* d_packinfo = nullptr;    // their AmPackCb
    double2** dbase = nullptr;     // its block bases (device, one per slab)
    std::vector<Phase> phases;
};

}  // namespace am

struct am_solver {
    int nx = 0, ny = 0, nz = 0, nzh = 0;
    int64_t N = 0;
    int64_t nstate = 0;  // voxels of phases with internal state (whole grid)
    int device = 0;
    cudaStream_t stream = nullptr;
    am_cfg cfg{};
    int nslabs = 1;      // global slab count
    bool multi = false;  // slab (transpose) algorithm vs 3-D cuFFT
    bool xfused = false; // single slab, nx = 256, AM_XFUSED=1: 2-D cuFFT + fused x transforms (xfused.cuh)
    int64_t redP = 0;    // offset of the slots after the residual partials in red
    ncclComm_t comm = nullptr;  // nccl mode: this process holds one slab
    std::vector<am::Slab> slabs;  // slabs held by this process
    cufftHandle r3 = 0, c3 = 0;   // 3-D D2Z / Z2D (single slab)
    bool zpack = false;           // sigma's transposes ride on the 2-D transforms' callbacks (fft_cb.h)
    void* fftws = nullptr;        // the cufft plans' shared work area
    bool zcb = false;             // the inverse transform reads ehat' / N through a load callback (fft_cb.cu):
                                  // c3 (one slab) or every slab's x1i
    void* d_cbinfo = nullptr;     // c3's AmZ2DCb
    cufftHandle r2 = 0, c2 = 0;   // 2-D D2Z / Z2D over (y, z), batch 6 nxl
    cufftHandle x1 = 0;           // 1-D Z2Z over x, batch 6 nyl nzh
    double* red = nullptr;        // reduction vectors, one per local slab, length redlen
    double* hred = nullptr;       // pinned host copy
    int64_t redlen = 0;
    int64_t chunk = 0;            // tangent sweep chunk
    double* Cbuf = nullptr;
    uint8_t* status = nullptr;
    double* stats = nullptr;
    double* hstats = nullptr;
    double* dsmall = nullptr;     // nccl reductions of the tangent statistics
    double* pl = nullptr;         // per-plane sums of eps and sigma (2 x nx x 6), field_means
    double* d_eb = nullptr;       // mean strain of the next iteration (graph replays read it)
    double* h_eb = nullptr;       // pinned host copy
    bool graphs = true;           // steady-state iterations as a CUDA graph (AM_NO_GRAPHS=1: eager)
    double* hpl = nullptr;        // pinned host copy
    int64_t nstat = 0;            // tangent statistics records: present phases x nx x kSParts
    std::vector<int> phase_rec;   // record block of each phase (phases without voxels: -1)
    double* ps = nullptr;         // per-(phase, x plane, part) records of k_refstats_planes
    double* hps = nullptr;        // pinned host copy
    bool p2p = false;             // fused pack / unpack over peer memory instead of the all-to-all
    std::vector<void*> ipc_open;  // peer buffers opened with cudaIpcOpenMemHandle
    double lam = 0.0, mu = 0.0;
    double ebar_n[6] = {0, 0, 0, 0, 0, 0};
    bool pending = false;
    bool warm_start = false;  // Newton from the previous iterate's state (am_solver_set_warm_start)
    am::DevBasis db = am::DevBasis::make();
    bool timing = false;
    cudaEvent_t ev[6] = {};
    double t_ms[5] = {0, 0, 0, 0, 0};  // material, forward FFT, fourier+reduce, inverse FFT, iterations
};

namespace am {

static void solver_free(am_solver* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (auto& s : h->slabs) {
        for (auto& p : s.phases) {
            cudaFree(p.gidx);
            cudaFree(p.a_n);
            cudaFree(p.a_pend);
            cudaFree(p.a_tmp);
            cudaFree(p.dpoff);
        }
        cudaFree(s.eps); cudaFree(s.eps_n); cudaFree(s.sigma);
        cudaFree(s.S); cudaFree(s.ehat); cudaFree(s.P); cudaFree(s.X); cudaFree(s.flags); cudaFree(s.subs);
        cudaFree(s.peerS); cudaFree(s.peerE); cudaFree(s.d_cbinfo); cudaFree(s.d_packinfo); cudaFree(s.dbase);
        for (cufftHandle p : {s.x1i, s.r2p, s.c2u})
            if (p) cufftDestroy(p);
    }
    cudaFree(h->red); cudaFreeHost(h->hred);
    cudaFree(h->Cbuf); cudaFree(h->status); cudaFree(h->stats); cudaFreeHost(h->hstats); cudaFree(h->dsmall);
    cudaFree(h->pl); cudaFreeHost(h->hpl); cudaFree(h->ps); cudaFreeHost(h->hps);
    cudaFree(h->d_eb); cudaFreeHost(h->h_eb); cudaFree(h->d_cbinfo); cudaFree(h->fftws);
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
    for (cufftHandle p : {h->r3, h->c3, h->r2, h->c2, h->x1})
        if (p) cufftDestroy(p);
    for (void* p : h->ipc_open) cudaIpcCloseMemHandle(p);
    if (h->comm) ncclCommDestroy(h->comm);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

// ---------------------------------------------------------------- transport
// all-to-all of equal blocks: block j of slab i's `send` -> block i of slab j's `recv`
static int alltoall(am_solver* h, double2* Slab::*send, double2* Slab::*recv, size_t blk) {
    if (h->comm) {
        Slab& s = h->slabs[0];
        AM_NCCL(ncclAlltoAll(s.*send, s.*recv, 2 * blk, ncclDouble, h->comm, h->stream));
        return AM_OK;
    }
    for (auto& si : h->slabs)
        for (auto& sj : h->slabs)
            AM_CUDA(cudaMemcpyAsync(sj.*recv + (size_t)si.rank * blk, si.*send + (size_t)sj.rank * blk,
                                    blk * sizeof(double2), cudaMemcpyDeviceToDevice, h->stream));
    return AM_OK;
}

// element-wise sum of every slab's reduction vector -> host (disjoint
// supports, so the sum is exact and independent of the slab count):
// enqueue (stream-ordered, capturable) + collect (synchronises)
static int reduce_enqueue(am_solver* h) {
    const int64_t L = h->redlen;
    if (h->comm) AM_NCCL(ncclAllReduce(h->red, h->red, L, ncclDouble, ncclSum, h->comm, h->stream));
    const size_t nvec = h->comm ? 1 : h->slabs.size();
    AM_CUDA(cudaMemcpyAsync(h->hred, h->red, sizeof(double) * L * nvec, cudaMemcpyDeviceToHost, h->stream));
    return AM_OK;
}
static int reduce_collect(am_solver* h, double* out) {
    const int64_t L = h->redlen;
    const size_t nvec = h->comm ? 1 : h->slabs.size();
    AM_CUDA(cudaStreamSynchronize(h->stream));
    for (int64_t i = 0; i < L; ++i) {
        double v = 0.0;
        for (size_t s = 0; s < nvec; ++s) v += h->hred[s * L + i];
        out[i] = v;
    }
    return AM_OK;
}
static int reduce_to_host(am_solver* h, double* out) {
    AM_TRY(reduce_enqueue(h));
    return reduce_collect(h, out);
}

// stream-ordered barrier across ranks (a 1-element all-reduce); in local
// mode all slabs share one stream, which already orders them
static int barrier(am_solver* h) {
    if (h->comm) AM_NCCL(ncclAllReduce(h->dsmall + 63, h->dsmall + 63, 1, ncclDouble, ncclSum, h->comm, h->stream));
    return AM_OK;
}

// grid of the transpose kernels: one row of blocks per contiguous run
static dim3 runs_grid(const am_solver* h, const Slab& s) {
    const int64_t len = (int64_t)s.nyl * h->nzh;
    return dim3((unsigned)std::min<int64_t>((len + 255) / 256, 64), (unsigned)(h->nslabs * s.nxl * 6));
}

// ---------------------------------------------------------------- transforms
// rfft of a real slab field -> spectrum buffer `dst` (S or ehat) of every slab
static int forward(am_solver* h, double* Slab::*field, double2* Slab::*dst) {
    if (!h->multi) {
        Slab& s = h->slabs[0];
        AM_CUFFT(cufftExecD2Z(h->r3, s.*field, s.*dst));
        return AM_OK;
    }
    const bool fused = h->zpack && dst == &Slab::S;  // the D2Z stores the packed blocks itself
    if (h->p2p) {
        for (auto& s : h->slabs) {
            if (fused) {
                AM_CUFFT(cufftExecD2Z(s.r2p, s.*field, s.P));
                continue;
            }
            AM_CUFFT(cufftExecD2Z(h->r2, s.*field, s.P));
            k_pack_peer<<<runs_grid(h, s), 256, 0, h->stream>>>(s.P, dst == &Slab::S ? s.peerS : s.peerE, s.rank,
                                                                s.nxl, h->ny, h->nzh, s.nyl);
            AM_CUDA(cudaGetLastError());
        }
        AM_TRY(barrier(h));  // every block has landed
        for (auto& s : h->slabs) AM_CUFFT(cufftExecZ2Z(h->x1, s.*dst, s.*dst, CUFFT_FORWARD));
        return AM_OK;
    }
    for (auto& s : h->slabs) {
        if (fused) {
            AM_CUFFT(cufftExecD2Z(s.r2p, s.*field, s.P));
            continue;
        }
        AM_CUFFT(cufftExecD2Z(h->r2, s.*field, s.P));
        k_pack<<<runs_grid(h, s), 256, 0, h->stream>>>(s.P, s.X, s.nxl, h->ny, h->nzh, s.nyl);
        AM_CUDA(cudaGetLastError());
    }
    AM_TRY(alltoall(h, &Slab::X, dst, (size_t)6 * h->slabs[0].nxl * h->slabs[0].nyl * h->nzh));
    for (auto& s : h->slabs) AM_CUFFT(cufftExecZ2Z(h->x1, s.*dst, s.*dst, CUFFT_FORWARD));
    return AM_OK;
}

// real field of every slab = irfft of the spectrum buffer `src` (destroyed)
static int inverse(am_solver* h, double2* Slab::*src, double* Slab::*field) {
    if (!h->multi) {
        Slab& s = h->slabs[0];
        AM_CUFFT(cufftExecZ2D(h->c3, s.*src, s.*field));
        return AM_OK;
    }
    // S: the load callback reads ehat' / N instead (the caller skipped the copy)
    for (auto& s : h->slabs)
        AM_CUFFT(cufftExecZ2Z(h->zcb && src == &Slab::S ? s.x1i : h->x1, s.*src, s.*src, CUFFT_INVERSE));
    const bool fused = h->zpack && src == &Slab::S;  // the Z2D loads the blocks itself
    if (h->p2p) {
        AM_TRY(barrier(h));  // every rank's x-transform is done before it is read
        if (fused) {
            for (auto& s : h->slabs) AM_CUFFT(cufftExecZ2D(s.c2u, s.P, s.*field));
            AM_TRY(barrier(h));  // nobody overwrites a spectrum a peer is still reading
            return AM_OK;
        }
        for (auto& s : h->slabs) {
            k_unpack_peer<<<runs_grid(h, s), 256, 0, h->stream>>>(src == &Slab::S ? s.peerS : s.peerE, s.P, s.rank,
                                                                  s.nxl, h->ny, h->nzh, s.nyl);
            AM_CUDA(cudaGetLastError());
        }
        AM_TRY(barrier(h));  // nobody overwrites a spectrum a peer is still reading
        for (auto& s : h->slabs) AM_CUFFT(cufftExecZ2D(h->c2, s.P, s.*field));
        return AM_OK;
    }
    AM_TRY(alltoall(h, src, &Slab::X, (size_t)6 * h->slabs[0].nxl * h->slabs[0].nyl * h->nzh));
    for (auto& s : h->slabs) {
        if (fused) {
            AM_CUFFT(cufftExecZ2D(s.c2u, s.P, s.*field));
            continue;
        }
        k_unpack<<<runs_grid(h, s), 256, 0, h->stream>>>(s.X, s.P, s.nxl, h->ny, h->nzh, s.nyl);
        AM_CUDA(cudaGetLastError());
        AM_CUFFT(cufftExecZ2D(h->c2, s.P, s.*field));
    }
    return AM_OK;
}

// K1 over every phase of every local slab; states -> a_tmp
// warm: start each voxel's Newton from a_tmp (the previous basic-scheme
// iterate) instead of a_n (am_solver_set_warm_start)
static int material_sweep(am_solver* h, double dt, bool warm = false) {
    for (auto& s : h->slabs) {
        AM_CUDA(cudaMemsetAsync(s.flags, 0, sizeof(uint32_t), h->stream));
        AM_CUDA(cudaMemsetAsync(s.subs, 0, sizeof(unsigned long long), h->stream));
        for (auto& p : s.phases) {
            if (!p.count) continue;
            KArgs k{};
            k.sub_sum = (p.m && h->cfg.integrator != AM_INTEGRATOR_IMPLICIT_EULER) ? s.subs : nullptr;
            k.B = p.count;
            k.gidx = p.gidx;
            k.eps_n = s.eps_n; k.eps_np1 = s.eps; k.a_n = p.a_n; k.dt = nullptr; k.dt_scalar = dt;
            k.a_start = (warm && p.m && h->cfg.integrator == AM_INTEGRATOR_IMPLICIT_EULER) ? p.a_tmp : nullptr;
            k.le = {s.Nl, 1}; k.la = {p.count, 1}; k.lc = {0, 0};
            k.sigma = s.sigma; k.a_out = p.a_tmp; k.C = nullptr;
            k.iters = nullptr; k.status = nullptr; k.flags = s.flags;
            set_controls(k, &h->cfg);
            AM_TRY(launch_material(&p.law, k, h->stream));
        }
    }
    return AM_OK;
}

// residual partials (+ update) of every slab -> host vector
// [ny * kParts partials | Re S(origin) (6) | any Newton failure | 0]
static int fourier_enqueue(am_solver* h, bool update) {
    const RefMat ref = RefMat::make(h->lam, h->mu);
    const int64_t L = h->redlen;
    AM_CUDA(cudaMemsetAsync(h->red, 0, sizeof(double) * L * h->slabs.size(), h->stream));
    for (size_t i = 0; i < h->slabs.size(); ++i) {
        Slab& s = h->slabs[i];
        double* red = h->red + (int64_t)i * L;
#ifndef AM_FOURIER_PF
#define AM_FOURIER_PF 0
#endif
        if (AM_FOURIER_PF)
            k_fourier_pf<<<s.sp.nyl * kParts, kRedThreads, 0, h->stream>>>(s.sp, ref, s.S, s.ehat, red, update ? 1 : 0,
                                                                            h->zcb ? 0 : 1);
        else
            k_fourier<<<s.sp.nyl * kParts, kRedThreads, 0, h->stream>>>(s.sp, ref, s.S, s.ehat, red, update ? 1 : 0,
                                                                         h->zcb ? 0 : 1);
        AM_CUDA(cudaGetLastError());
        k_finish<<<1, 32, 0, h->stream>>>(s.S, s.sp.cs, s.y0 == 0 ? 1 : 0, s.flags, s.subs, red,
                                          (int64_t)h->ny * kParts);
        AM_CUDA(cudaGetLastError());
    }
    return reduce_enqueue(h);
}
static int fourier_pass(am_solver* h, bool update, std::vector<double>& out) {
    AM_TRY(fourier_enqueue(h, update));
    out.resize(h->redlen);
    return reduce_collect(h, out.data());
}

// the fused spectral step (xfused.cuh): 2-D spectra of sigma in S ->
// residual partials per tile + slots, ehat updated, S = 2-D spectra of the
// next eps without its origin (k_origin_x)
static int fourier_pass_x(am_solver* h, std::vector<double>& out) {
    const RefMat ref = RefMat::make(h->lam, h->mu);
    const int64_t L = h->redlen;
    Slab& s = h->slabs[0];
    AM_CUDA(cudaMemsetAsync(h->red, 0, sizeof(double) * L, h->stream));
    k_finish<<<1, 32, 0, h->stream>>>(s.S, s.sp.cs, 0, s.flags, s.subs, h->red, h->redP);
    AM_CUDA(cudaGetLastError());
    const int64_t ncol = (int64_t)h->ny * h->nzh;
    const int64_t tiles = (ncol + kXJ - 1) / kXJ;
    int sms = 148;
    AM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
    k_xfourier<<<(unsigned)std::min<int64_t>(tiles, (int64_t)sms * kXCtas), kXThreads, kXSmem, h->stream>>>(
        h->nx, h->ny, h->nz, s.sp.cs, ref, s.S, s.ehat, h->red, h->redP);
    AM_CUDA(cudaGetLastError());
    out.resize(L);
    return reduce_to_host(h, out.data());
}

// voxel means of eps and sigma (homogenize.py:448, 503-504: numpy's mean over
// the grid), as plane sums added in global plane order on the host
static int field_means(am_solver* h, double* ebar, double* sbar) {
    const int64_t L = (int64_t)h->nx * 6;
    AM_CUDA(cudaMemsetAsync(h->pl, 0, sizeof(double) * 2 * L, h->stream));
    const int64_t plane = (int64_t)h->ny * h->nz;
    for (auto& s : h->slabs) {
        k_plane_sums<<<dim3(s.nxl, 6), kRedThreads, 0, h->stream>>>(s.eps, s.Nl, plane, s.x0, h->pl);
        k_plane_sums<<<dim3(s.nxl, 6), kRedThreads, 0, h->stream>>>(s.sigma, s.Nl, plane, s.x0, h->pl + L);
        AM_CUDA(cudaGetLastError());
    }
    if (h->comm) AM_NCCL(ncclAllReduce(h->pl, h->pl, 2 * L, ncclDouble, ncclSum, h->comm, h->stream));
    AM_CUDA(cudaMemcpyAsync(h->hpl, h->pl, sizeof(double) * 2 * L, cudaMemcpyDeviceToHost, h->stream));
    AM_CUDA(cudaStreamSynchronize(h->stream));
    for (int c = 0; c < 6; ++c) {
        double e = 0.0, t = 0.0;
        for (int x = 0; x < h->nx; ++x) {
            e += h->hpl[x * 6 + c];
            t += h->hpl[L + x * 6 + c];
        }
        ebar[c] = e / (double)h->N;
        sbar[c] = t / (double)h->N;
    }
    return AM_OK;
}

}  // namespace am

using namespace am;

// ---------------------------------------------------------------- creation
static int solver_build(int nx, int ny, int nz, const uint8_t* ids, int nmat, const am_law* laws, const am_cfg* cfg,
                        int nslabs, int first, int nlocal, ncclComm_t comm, am_solver** out) {
    if (!out || !ids || !laws || nmat <= 0 || nx <= 0 || ny <= 0 || nz <= 0 || nslabs <= 0)
        return fail(AM_ERR_ARG, "am_solver_create: bad arguments");
    if (nslabs > 1 && (nx % nslabs || ny % nslabs))
        return fail(AM_ERR_ARG, "slab count %d must divide nx = %d and ny = %d", nslabs, nx, ny);
    AM_TRY(check_cfg(cfg));
    for (int i = 0; i < nmat; ++i) AM_TRY(check_law(&laws[i]));
    const int64_t N = (int64_t)nx * ny * nz;
    for (int64_t i = 0; i < N; ++i)
        if (ids[i] >= nmat) return fail(AM_ERR_ARG, "material id exceeds material table");
    auto* h = new am_solver();
    auto bail = [&](int code) {
        if (comm && h->comm == nullptr) ncclCommDestroy(comm);
        solver_free(h);
        return code;
    };
#define AMC(expr)                                                                                       \
    do {                                                                                                \
        cudaError_t _e = (expr);                                                                        \
        if (_e != cudaSuccess) return bail(fail(AM_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e))); \
    } while (0)
    AMC(cudaGetDevice(&h->device));
    h->comm = comm;
    h->nx = nx; h->ny = ny; h->nz = nz; h->nzh = nz / 2 + 1; h->N = N;
    h->cfg = *cfg;
    h->nslabs = nslabs;
    h->multi = nslabs > 1 || comm != nullptr;  // nccl mode always transposes (same bits for every rank count)
    AMC(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    const int nxl = nx / nslabs, nyl = ny / nslabs;
    const int64_t Nl = (int64_t)nxl * ny * nz;
    const int64_t spec = (int64_t)6 * nxl * ny * h->nzh;  // complex elements per slab spectrum
    for (int r = first; r < first + nlocal; ++r) {
        Slab s;
        s.rank = r;
        s.x0 = r * nxl; s.nxl = nxl; s.y0 = h->multi ? r * nyl : 0; s.nyl = h->multi ? nyl : ny; s.Nl = Nl;
        s.sp = h->multi ? spec_slab(nx, ny, nz, s.y0, nyl) : spec_single(nx, ny, nz);
        h->slabs.push_back(s);
        Slab& sl = h->slabs.back();
        AMC(cudaMalloc(&sl.eps, sizeof(double) * 6 * Nl));
        AMC(cudaMalloc(&sl.eps_n, sizeof(double) * 6 * Nl));
        AMC(cudaMalloc(&sl.sigma, sizeof(double) * 6 * Nl));
        AMC(cudaMemset(sl.eps, 0, sizeof(double) * 6 * Nl));
        AMC(cudaMemset(sl.eps_n, 0, sizeof(double) * 6 * Nl));
        AMC(cudaMemset(sl.sigma, 0, sizeof(double) * 6 * Nl));
        AMC(cudaMalloc(&sl.S, sizeof(double2) * spec));
        AMC(cudaMalloc(&sl.ehat, sizeof(double2) * spec));
        if (h->multi) {
            AMC(cudaMalloc(&sl.P, sizeof(double2) * spec));
            AMC(cudaMalloc(&sl.X, sizeof(double2) * spec));
        }
        AMC(cudaMalloc(&sl.flags, sizeof(uint32_t)));
        AMC(cudaMemset(sl.flags, 0, sizeof(uint32_t)));
        AMC(cudaMalloc(&sl.subs, sizeof(unsigned long long)));
        AMC(cudaMemset(sl.subs, 0, sizeof(unsigned long long)));
        // phases: slab-local sorted indices (the global order restricted to the slab)
        std::vector<std::vector<int64_t>> idx(nmat);
        const uint8_t* sid = ids + (int64_t)sl.x0 * ny * nz;
        for (int64_t i = 0; i < Nl; ++i) idx[sid[i]].push_back(i);
        for (int k = 0; k < nmat; ++k) {
            Phase p;
            p.law = laws[k];
            p.m = law_m(&laws[k]);
            p.count = (int64_t)idx[k].size();
            sl.phases.push_back(p);
            Phase& ph = sl.phases.back();
            ph.poff.resize(nxl + 1);
            for (int x = 0; x <= nxl; ++x)
                ph.poff[x] = std::lower_bound(idx[k].begin(), idx[k].end(), (int64_t)x * ny * nz) - idx[k].begin();
            if (!ph.count) continue;
            AMC(cudaMalloc(&ph.dpoff, sizeof(int64_t) * (nxl + 1)));
            AMC(cudaMemcpy(ph.dpoff, ph.poff.data(), sizeof(int64_t) * (nxl + 1), cudaMemcpyHostToDevice));
            AMC(cudaMalloc(&ph.gidx, sizeof(int64_t) * ph.count));
            AMC(cudaMemcpy(ph.gidx, idx[k].data(), sizeof(int64_t) * ph.count, cudaMemcpyHostToDevice));
            if (ph.m) {
                for (double** a : {&ph.a_n, &ph.a_pend, &ph.a_tmp}) {
                    AMC(cudaMalloc(a, sizeof(double) * ph.m * ph.count));
                    AMC(cudaMemset(*a, 0, sizeof(double) * ph.m * ph.count));
                }
            }
        }
    }
    // fused x transforms on one GPU when nx = 256, opt-in (AM_XFUSED=1):
    // correct, but slower than cuFFT's x passes + k_fourier at 256^3 so far
    // (profiles/r01/k1_variants.log, r26)
    {
        const char* on = getenv("AM_XFUSED");
        h->xfused = !h->multi && nx == kXN && on && on[0] == '1';
    }
    h->redP = h->xfused ? ((int64_t)ny * h->nzh + kXJ - 1) / kXJ : (int64_t)ny * kParts;
    h->redlen = h->redP + 10;
    for (int64_t i = 0; i < N; ++i)
        if (law_m(&laws[ids[i]])) ++h->nstate;
    AMC(cudaMalloc(&h->red, sizeof(double) * h->redlen * h->slabs.size()));
    AMC(cudaMallocHost(&h->hred, sizeof(double) * h->redlen * h->slabs.size()));
    // tangent sweep chunks are whole x planes of a phase: at least one plane
    h->chunk = std::max<int64_t>(std::min<int64_t>(Nl, int64_t(1) << 22), (int64_t)ny * nz);
    AMC(cudaMalloc(&h->Cbuf, sizeof(double) * 36 * h->chunk));
    AMC(cudaMalloc(&h->status, h->chunk));
    AMC(cudaMalloc(&h->stats, sizeof(double) * kStat * kRedBlocks));
    AMC(cudaMallocHost(&h->hstats, sizeof(double) * kStat * kRedBlocks));
    AMC(cudaMalloc(&h->dsmall, sizeof(double) * 64));
    AMC(cudaMalloc(&h->pl, sizeof(double) * 12 * nx));
    AMC(cudaMalloc(&h->d_eb, sizeof(double) * 6));
    AMC(cudaMallocHost(&h->h_eb, sizeof(double) * 6));
    {
        const char* off = getenv("AM_NO_GRAPHS");
        h->graphs = !(off && off[0] == '1');
    }
    AMC(cudaMallocHost(&h->hpl, sizeof(double) * 12 * nx));
    {  // records only for phases that have voxels somewhere in the grid
        std::vector<int64_t> cnt(nmat, 0);
        for (int64_t i = 0; i < N; ++i) ++cnt[ids[i]];
        int np = 0;
        h->phase_rec.assign(nmat, -1);
        for (int k = 0; k < nmat; ++k)
            if (cnt[k]) h->phase_rec[k] = np++;
        h->nstat = (int64_t)std::max(np, 1) * nx * kSParts;
    }
    AMC(cudaMalloc(&h->ps, sizeof(double) * kStat * h->nstat));
    AMC(cudaMallocHost(&h->hps, sizeof(double) * kStat * h->nstat));
#undef AMC
    // every plan runs on h->stream, one at a time: they share one work area
    // (640^3: the 3-D D2Z and Z2D each want 12.6 GB)
    size_t ws_max = 0;
    auto plan = [&](cufftHandle* p, int rank, long long* n, long long* inembed, long long istride, long long idist,
                    long long* onembed, long long ostride, long long odist, cufftType t, long long batch) -> bool {
        size_t ws = 0;
        const bool r = cufftCreate(p) == CUFFT_SUCCESS && cufftSetAutoAllocation(*p, 0) == CUFFT_SUCCESS &&
                       cufftMakePlanMany64(*p, rank, n, inembed, istride, idist, onembed, ostride, odist, t, batch,
                                           &ws) == CUFFT_SUCCESS &&
                       cufftSetStream(*p, h->stream) == CUFFT_SUCCESS;
        ws_max = std::max(ws_max, ws);
        return r;
    };
    bool ok;
    // the inverse transform with the load callback (fft_cb.cu) from 128^3
    // on, where the saved copy matters, for power-of-two voxel counts (the
    // origin's N ebar / N is then exact); AM_FFT_CALLBACK=0 / 1 forces it
    // off / on.  The callback's first link in a process costs ~2 s.
    const char* cbenv = getenv("AM_FFT_CALLBACK");
    // local slabs transpose through the siblings' spectra (the P2P kernels);
    // AM_LOCAL_ALLTOALL=1 runs them through the all-to-all buffers instead
    // (device copies in place of ncclAlltoAll: the NCCL transport's data
    // layout with more than one slab, testable on one GPU)
    const char* ltenv = getenv("AM_LOCAL_ALLTOALL");
    const bool local_p2p = !comm && !(ltenv && ltenv[0] == '1');
    const bool want_cb = !h->xfused && (N & (N - 1)) == 0 && (cbenv ? cbenv[0] == '1' : N >= (int64_t(1) << 21));
    if (!h->multi) {
        long long n3[3] = {nx, ny, nz};
        ok = plan(&h->r3, 3, n3, nullptr, 1, N, nullptr, 1, (long long)nx * ny * h->nzh, CUFFT_D2Z, 6);
        if (ok && want_cb) {
            const am::Slab& s0 = h->slabs[0];
            const AmZ2DCb info{s0.ehat, 1.0 / (double)N};
            h->zcb = cudaMalloc(&h->d_cbinfo, sizeof(info)) == cudaSuccess &&
                     cudaMemcpy(h->d_cbinfo, &info, sizeof(info), cudaMemcpyHostToDevice) == cudaSuccess &&
                     am_callback_plan(&h->c3, 3, n3, nullptr, 1, (long long)nx * ny * h->nzh, nullptr, 1, N, CUFFT_Z2D,
                                      6, h->stream, h->d_cbinfo, "am_z2d_load", CUFFT_CB_LD_COMPLEX_DOUBLE, &ws_max);
        }
        if (ok && !h->zcb)
            ok = plan(&h->c3, 3, n3, nullptr, 1, (long long)nx * ny * h->nzh, nullptr, 1, N, CUFFT_Z2D, 6);
        if (ok && h->xfused) {
            long long n2[2] = {ny, nz};
            ok = plan(&h->r2, 2, n2, nullptr, 1, (long long)ny * nz, nullptr, 1, (long long)ny * h->nzh, CUFFT_D2Z,
                      6LL * nx) &&
                 plan(&h->c2, 2, n2, nullptr, 1, (long long)ny * h->nzh, nullptr, 1, (long long)ny * nz, CUFFT_Z2D,
                      6LL * nx) &&
                 cudaFuncSetAttribute(k_xfourier, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kXSmem) ==
                     cudaSuccess;
        }
    } else {
        long long n2[2] = {ny, nz};
        long long n1[1] = {nx};
        const long long bx = (long long)6 * nyl * h->nzh;  // x stride = batch of the 1-D transforms
        ok = plan(&h->r2, 2, n2, nullptr, 1, (long long)ny * nz, nullptr, 1, (long long)ny * h->nzh, CUFFT_D2Z,
                  6LL * nxl) &&
             plan(&h->c2, 2, n2, nullptr, 1, (long long)ny * h->nzh, nullptr, 1, (long long)ny * nz, CUFFT_Z2D,
                  6LL * nxl) &&
             plan(&h->x1, 1, n1, n1, bx, 1, n1, bx, 1, CUFFT_Z2Z, bx);
        if (ok && want_cb) {  // every local slab's inverse x transform reads its own ehat'
            bool all = true;
            for (auto& sl : h->slabs) {
                const AmZ2DCb info{sl.ehat, 1.0 / (double)N};
                all = all && cudaMalloc(&sl.d_cbinfo, sizeof(info)) == cudaSuccess &&
                      cudaMemcpy(sl.d_cbinfo, &info, sizeof(info), cudaMemcpyHostToDevice) == cudaSuccess &&
                      am_callback_plan(&sl.x1i, 1, n1, n1, bx, 1, n1, bx, 1, CUFFT_Z2Z, bx, h->stream, sl.d_cbinfo,
                                       "am_z2d_load", CUFFT_CB_LD_COMPLEX_DOUBLE, &ws_max);
            }
            h->zcb = all;
        }
        // sigma's transposes on the 2-D transforms' callbacks (fft_cb.h):
        // block bases = the sibling slabs' spectra (local), the all-to-all
        // buffer (NCCL; am_solver_ipc_import switches them to the peers')
        const long long blk = (long long)nxl * 6 * nyl * h->nzh;
        const bool fits = 6.0 * nxl * ny * h->nzh < 4294967296.0;  // 32-bit element offsets in the callbacks
        // (power-of-two grids, like the load callback: cuFFT picks other kernels
        // for LTO plans of other sizes, and the fields would differ in the last bits)
        if (ok && fits && (N & (N - 1)) == 0 && !h->xfused && (cbenv ? cbenv[0] == '1' : N >= (int64_t(1) << 21))) {
            bool all = true;
            std::vector<double2*> byrank(nslabs, nullptr);
            for (auto& sl : h->slabs) byrank[sl.rank] = sl.S;
            for (auto& sl : h->slabs) {
                std::vector<double2*> base(nslabs);
                for (int j = 0; j < nslabs; ++j) base[j] = local_p2p ? byrank[j] + sl.rank * blk : sl.X + j * blk;
                const AmPackCb info{nullptr, (unsigned)h->nzh, (unsigned)ny, (unsigned)nxl, (unsigned)nyl};
                all = all && cudaMalloc(&sl.dbase, sizeof(double2*) * nslabs) == cudaSuccess &&
                      cudaMemcpy(sl.dbase, base.data(), sizeof(double2*) * nslabs, cudaMemcpyHostToDevice) ==
                          cudaSuccess &&
                      cudaMalloc(&sl.d_packinfo, sizeof(info)) == cudaSuccess;
                if (!all) break;
                AmPackCb dinfo = info;
                dinfo.base = sl.dbase;
                all = cudaMemcpy(sl.d_packinfo, &dinfo, sizeof(dinfo), cudaMemcpyHostToDevice) == cudaSuccess &&
                      am_callback_plan(&sl.r2p, 2, n2, nullptr, 1, (long long)ny * nz, nullptr, 1,
                                       (long long)ny * h->nzh, CUFFT_D2Z, 6LL * nxl, h->stream, sl.d_packinfo,
                                       "am_pack_store", CUFFT_CB_ST_COMPLEX_DOUBLE, &ws_max) &&
                      am_callback_plan(&sl.c2u, 2, n2, nullptr, 1, (long long)ny * h->nzh, nullptr, 1,
                                       (long long)ny * nz, CUFFT_Z2D, 6LL * nxl, h->stream, sl.d_packinfo,
                                       "am_unpack_load", CUFFT_CB_LD_COMPLEX_DOUBLE, &ws_max);
                if (!all) break;
            }
            h->zpack = all;
        }
    }
    if (!ok) return bail(fail(AM_ERR_CUDA, "cufft plan creation failed for %dx%dx%d / %d slabs", nx, ny, nz, nslabs));
    if (ws_max) {
        if (cudaMalloc(&h->fftws, ws_max) != cudaSuccess) return bail(fail(AM_ERR_CUDA, "out of memory (cufft work area)"));
        std::vector<cufftHandle> all = {h->r3, h->c3, h->r2, h->c2, h->x1};
        for (auto& sl : h->slabs) all.insert(all.end(), {sl.x1i, sl.r2p, sl.c2u});
        for (cufftHandle p : all)
            if (p && cufftSetWorkArea(p, h->fftws) != CUFFT_SUCCESS)
                return bail(fail(AM_ERR_CUDA, "cufft work area"));
    }
    if (h->multi) {
        for (auto& sl : h->slabs) {
            if (cudaMalloc(&sl.peerS, sizeof(double2*) * nslabs) != cudaSuccess ||
                cudaMalloc(&sl.peerE, sizeof(double2*) * nslabs) != cudaSuccess)
                return bail(fail(AM_ERR_CUDA, "out of memory"));
        }
        if (!comm) {  // all slabs are local: the fused transposes address them directly
            std::vector<double2*> S(nslabs), E(nslabs);
            for (auto& sl : h->slabs) {
                S[sl.rank] = sl.S;
                E[sl.rank] = sl.ehat;
            }
            for (auto& sl : h->slabs)
                if (cudaMemcpy(sl.peerS, S.data(), sizeof(double2*) * nslabs, cudaMemcpyHostToDevice) != cudaSuccess ||
                    cudaMemcpy(sl.peerE, E.data(), sizeof(double2*) * nslabs, cudaMemcpyHostToDevice) != cudaSuccess)
                    return bail(fail(AM_ERR_CUDA, "copy failed"));
            h->p2p = local_p2p;
        }
    }
    *out = h;
    return AM_OK;
}

extern "C" int am_solver_create(int nx, int ny, int nz, const uint8_t* ids, int nmat, const am_law* laws,
                                const am_cfg* cfg, am_solver** out) {
    return solver_build(nx, ny, nz, ids, nmat, laws, cfg, 1, 0, 1, nullptr, out);
}

extern "C" int am_solver_create_slabs(int nx, int ny, int nz, const uint8_t* ids, int nmat, const am_law* laws,
                                      const am_cfg* cfg, int nslabs, am_solver** out) {
    return solver_build(nx, ny, nz, ids, nmat, laws, cfg, nslabs, 0, nslabs, nullptr, out);
}

extern "C" int am_nccl_unique_id(void* id128) {
    if (!id128) return fail(AM_ERR_ARG, "null id buffer");
    ncclUniqueId id;
    AM_NCCL(ncclGetUniqueId(&id));
    std::memcpy(id128, &id, sizeof(id));
    return AM_OK;
}

extern "C" int am_solver_create_nccl(int nx, int ny, int nz, const uint8_t* ids, int nmat, const am_law* laws,
                                     const am_cfg* cfg, const void* id128, int rank, int nranks, am_solver** out) {
    if (!id128 || rank < 0 || rank >= nranks) return fail(AM_ERR_ARG, "bad rank / id");
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm = nullptr;
    AM_NCCL(ncclCommInitRank(&comm, nranks, id, rank));
    return solver_build(nx, ny, nz, ids, nmat, laws, cfg, nranks, rank, 1, comm, out);
}

// P2P transport for one-slab-per-process handles: export this rank's
// spectrum buffers as CUDA IPC handles (2 x 64 bytes: S, ehat) ...
extern "C" int am_solver_ipc_export(am_solver* h, void* out128) {
    if (!h || !out128 || !h->comm) return fail(AM_ERR_ARG, "am_solver_ipc_export needs an nccl-mode handle");
    AM_CUDA(cudaSetDevice(h->device));
    cudaIpcMemHandle_t hs[2];
    AM_CUDA(cudaIpcGetMemHandle(&hs[0], h->slabs[0].S));
    AM_CUDA(cudaIpcGetMemHandle(&hs[1], h->slabs[0].ehat));
    std::memcpy(out128, hs, sizeof(hs));
    return AM_OK;
}

// ... and map every rank's (nranks x 128 bytes, rank order), switching the
// transposes from ncclAlltoAll to the fused pack / unpack kernels over NVLink
extern "C" int am_solver_ipc_import(am_solver* h, const void* all, int nranks) {
    if (!h || !all || !h->comm || nranks != h->nslabs) return fail(AM_ERR_ARG, "am_solver_ipc_import: bad arguments");
    AM_CUDA(cudaSetDevice(h->device));
    Slab& sl = h->slabs[0];
    std::vector<double2*> S(nranks), E(nranks);
    const cudaIpcMemHandle_t* hs = (const cudaIpcMemHandle_t*)all;
    for (int r = 0; r < nranks; ++r) {
        if (r == sl.rank) {
            S[r] = sl.S;
            E[r] = sl.ehat;
            continue;
        }
        void *ps = nullptr, *pe = nullptr;
        AM_CUDA(cudaIpcOpenMemHandle(&ps, hs[2 * r], cudaIpcMemLazyEnablePeerAccess));
        h->ipc_open.push_back(ps);
        AM_CUDA(cudaIpcOpenMemHandle(&pe, hs[2 * r + 1], cudaIpcMemLazyEnablePeerAccess));
        h->ipc_open.push_back(pe);
        S[r] = (double2*)ps;
        E[r] = (double2*)pe;
    }
    AM_CUDA(cudaMemcpy(sl.peerS, S.data(), sizeof(double2*) * nranks, cudaMemcpyHostToDevice));
    AM_CUDA(cudaMemcpy(sl.peerE, E.data(), sizeof(double2*) * nranks, cudaMemcpyHostToDevice));
    if (h->zpack) {  // the transpose callbacks now address the peers' spectra (this rank's block)
        const long long blk = (long long)sl.nxl * 6 * sl.nyl * h->nzh;
        std::vector<double2*> base(nranks);
        for (int r = 0; r < nranks; ++r) base[r] = S[r] + sl.rank * blk;
        AM_CUDA(cudaMemcpy(sl.dbase, base.data(), sizeof(double2*) * nranks, cudaMemcpyHostToDevice));
    }
    AM_CUDA(cudaMemsetAsync(h->dsmall, 0, sizeof(double) * 64, h->stream));
    AM_CUDA(cudaStreamSynchronize(h->stream));
    h->p2p = true;
    return AM_OK;
}

extern "C" int am_solver_destroy(am_solver* h) {
    solver_free(h);
    return AM_OK;
}

extern "C" int am_solver_set_reference(am_solver* h, double lam, double mu) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    h->lam = lam;
    h->mu = mu;
    return AM_OK;
}

extern "C" int am_solver_get_reference(am_solver* h, double* lam, double* mu) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    *lam = h->lam;
    *mu = h->mu;
    return AM_OK;
}

extern "C" int am_solver_set_mean(am_solver* h, const double* ebar_n) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    std::memcpy(h->ebar_n, ebar_n, sizeof(h->ebar_n));
    return AM_OK;
}

extern "C" int am_solver_layout(am_solver* h, int* nslabs, int* first, int* nlocal) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    if (nslabs) *nslabs = h->nslabs;
    if (first) *first = h->slabs[0].rank;
    if (nlocal) *nlocal = (int)h->slabs.size();
    return AM_OK;
}

// ---------------------------------------------------------------- solve
extern "C" int am_solver_solve_step(am_solver* h, const double* ebar_target, double dt, const uint8_t* free_mask,
                                    double tol, int max_iterations, am_stepinfo* info, double* history,
                                    int history_cap) {
    if (!h || !ebar_target || !info) return fail(AM_ERR_ARG, "am_solver_solve_step: bad arguments");
    AM_CUDA(cudaSetDevice(h->device));
    bool fr[6];
    int nf = 0, fi[6];
    for (int i = 0; i < 6; ++i) {
        fr[i] = free_mask ? free_mask[i] != 0 : false;
        if (fr[i]) fi[nf++] = i;
    }
    double ebar[6];
    for (int i = 0; i < 6; ++i) ebar[i] = fr[i] ? h->ebar_n[i] : ebar_target[i];  // homogenize.py:436-437
    Vec6 shift;
    for (int i = 0; i < 6; ++i) shift.v[i] = ebar[i] - h->ebar_n[i];
    for (auto& s : h->slabs) {
        k_shift<<<grid_for(s.Nl), 256, 0, h->stream>>>(s.eps, s.eps_n, shift, s.Nl);
        AM_CUDA(cudaGetLastError());
    }
    AM_TRY(forward(h, &Slab::eps, &Slab::ehat));
    double Cff[36];
    {
        double C0[36];
        ref_matrix(h->lam, h->mu, C0);
        for (int a = 0; a < nf; ++a)
            for (int b = 0; b < nf; ++b) Cff[a * nf + b] = C0[fi[a] * 6 + fi[b]];
    }
    info->iterations = 0;
    info->converged = 0;
    info->residual = 0.0;
    info->mean_substeps = 1.0;  // implicit Euler: one substep per voxel (evaluator.py:130)
    const double Nd = (double)h->N;
    const int64_t P = h->redP;
    std::vector<double> o;
    auto mark = [&](int i) -> int {
        if (h->timing) AM_CUDA(cudaEventRecord(h->ev[i], h->stream));
        return AM_OK;
    };
    auto acc = [&](int a, int b, int slot) -> int {
        float ms = 0.f;
        AM_CUDA(cudaEventElapsedTime(&ms, h->ev[a], h->ev[b]));
        h->t_ms[slot] += ms;
        return AM_OK;
    };
    // Steady-state iterations (2, 3, ...) on one slab: origin + Z2D, the
    // material sweep, D2Z, the Fourier kernels and the reduction's D2H are
    // one CUDA graph (captured once per load step, since dt, the reference
    // material and the state buffers are fixed within a step), replayed
    // after the host's convergence test and mixed-BC update: one launch per
    // iteration instead of ~12.  Same kernels in the same order as the
    // eager path; AM_NO_GRAPHS=1 or the phase timers select the eager path.
    const bool use_graph = h->graphs && !h->multi && !h->xfused && !h->timing;
    struct GraphGuard {
        cudaGraph_t g = nullptr;
        cudaGraphExec_t x = nullptr;
        ~GraphGuard() {
            if (x) cudaGraphExecDestroy(x);
            if (g) cudaGraphDestroy(g);
        }
    } gg;
    auto capture = [&]() -> int {
        Slab& s0 = h->slabs[0];
        AM_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        auto body = [&]() -> int {
            k_origin_dev<<<1, 32, 0, h->stream>>>(h->zcb ? nullptr : s0.S, s0.ehat, s0.sp.cs, h->d_eb, Nd);
            AM_CUDA(cudaGetLastError());
            AM_TRY(inverse(h, &Slab::S, &Slab::eps));
            AM_TRY(material_sweep(h, dt, h->warm_start));
            AM_TRY(forward(h, &Slab::sigma, &Slab::S));
            return fourier_enqueue(h, true);
        };
        const int rc = body();
        cudaGraph_t g = nullptr;
        const cudaError_t e = cudaStreamEndCapture(h->stream, &g);
        if (rc != AM_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        AM_CUDA(e);
        gg.g = g;
        AM_CUDA(cudaGraphInstantiate(&gg.x, gg.g, 0));
        return AM_OK;
    };
    bool have = false;  // o already holds this iteration's reduction (graph replay)
    for (int it = 1; it <= max_iterations; ++it) {
        if (!have) {
        AM_TRY(mark(0));
        AM_TRY(material_sweep(h, dt, h->warm_start && it > 1));
        AM_TRY(mark(1));
        if (h->xfused) {
            AM_CUFFT(cufftExecD2Z(h->r2, h->slabs[0].sigma, h->slabs[0].S));
            AM_TRY(mark(2));
            AM_TRY(fourier_pass_x(h, o));  // synchronises the stream
        } else {
            AM_TRY(forward(h, &Slab::sigma, &Slab::S));
            AM_TRY(mark(2));
            AM_TRY(fourier_pass(h, true, o));  // synchronises the stream
        }
        }
        have = false;
        if (h->timing) {
            AM_CUDA(cudaEventRecord(h->ev[3], h->stream));
            AM_CUDA(cudaEventSynchronize(h->ev[3]));
            AM_TRY(acc(0, 1, 0));
            AM_TRY(acc(1, 2, 1));
            AM_TRY(acc(2, 3, 2));
            h->t_ms[4] += 1.0;
        }
        if (o[P + 6] != 0.0 || o[P + 7] != 0.0 || o[P + 9] != 0.0) {
            info->iterations = it;
            if (o[P + 6] != 0.0)
                return fail(AM_ERR_NEWTON, "implicit Euler Newton failed for at least one voxel (iteration %d)", it);
            if (o[P + 7] != 0.0) return fail(AM_ERR_INTEGRATION, "adaptive integration hit a cap (iteration %d)", it);
            return fail(AM_ERR_RADIAL, "radial return stalled for at least one voxel (iteration %d)", it);
        }
        // Homogenizer's mean substeps (homogenize.py:420-421): implicit Euler,
        // frozen points and laws without state take one substep per voxel
        if (h->cfg.integrator != AM_INTEGRATOR_IMPLICIT_EULER)
            info->mean_substeps = (o[P + 8] + (double)(h->N - h->nstate)) / (double)h->N;
        double fsum = 0.0;
        for (int64_t i = 0; i < P; ++i) fsum += o[i];  // fixed order: ky plane, then part
        double sbar[6];
        for (int i = 0; i < 6; ++i) sbar[i] = o[P + i] / Nd;
        // equilibrium_residual (homogenize.py:264-267)
        const double scale = std::max(dup_norm(sbar), 1e-300);
        const double res = std::sqrt(fsum / (Nd * Nd)) / scale;
        double res_bc = 0.0;
        if (nf) {
            double t = 0.0;
            for (int a = 0; a < nf; ++a) t += sbar[fi[a]] * sbar[fi[a]];
            res_bc = std::sqrt(t) / scale;
        }
        const double hres = std::max(res, res_bc);
        if (history && it <= history_cap) history[it - 1] = hres;
        info->iterations = it;
        info->residual = hres;
        for (int i = 0; i < 6; ++i) {
            info->ebar[i] = ebar[i];
            info->sig_bar[i] = sbar[i];
        }
        if (res < tol && res_bc < tol) {  // strict (homogenize.py:454)
            info->converged = 1;
            AM_TRY(field_means(h, info->ebar, info->sig_bar));
            // the converged evaluation's state becomes the pending state
            // (homogenize.py:455-457); earlier evaluations never touch it
            for (auto& s : h->slabs)
                for (auto& p : s.phases) std::swap(p.a_pend, p.a_tmp);
            h->pending = true;
            return AM_OK;
        }
        if (nf) {  // mixed BC (homogenize.py:462-464)
            double A[36], x[6];
            std::memcpy(A, Cff, sizeof(double) * nf * nf);
            for (int a = 0; a < nf; ++a) x[a] = -sbar[fi[a]];
            if (!small_solve(nf, A, x)) return fail(AM_ERR_SINGULAR, "singular reference block");
            for (int a = 0; a < nf; ++a) ebar[fi[a]] += x[a];
        }
        if (use_graph && it < max_iterations) {  // iteration it + 1 as a graph replay
            for (int i = 0; i < 6; ++i) h->h_eb[i] = ebar[i];
            AM_CUDA(cudaMemcpyAsync(h->d_eb, h->h_eb, sizeof(double) * 6, cudaMemcpyHostToDevice, h->stream));
            if (!gg.x) AM_TRY(capture());
            AM_CUDA(cudaGraphLaunch(gg.x, h->stream));
            o.resize(h->redlen);
            AM_TRY(reduce_collect(h, o.data()));
            have = true;
            continue;
        }
        AM_TRY(mark(4));
        Vec6 eb;
        for (int i = 0; i < 6; ++i) eb.v[i] = ebar[i];
        if (h->xfused) {
            Slab& s = h->slabs[0];
            k_origin_x<<<6, 256, 0, h->stream>>>(s.S, s.ehat, s.sp.cs, (int64_t)h->ny * h->nzh, h->nx, eb, Nd);
            AM_CUDA(cudaGetLastError());
            AM_CUFFT(cufftExecZ2D(h->c2, s.S, s.eps));
        } else if (h->zcb && !h->multi) {  // the callback reads the origin's N ebar from ehat
            Slab& s0 = h->slabs[0];
            for (int i = 0; i < 6; ++i) h->h_eb[i] = ebar[i];
            AM_CUDA(cudaMemcpyAsync(h->d_eb, h->h_eb, sizeof(double) * 6, cudaMemcpyHostToDevice, h->stream));
            k_origin_dev<<<1, 32, 0, h->stream>>>(nullptr, s0.ehat, s0.sp.cs, h->d_eb, Nd);
            AM_CUDA(cudaGetLastError());
            AM_TRY(inverse(h, &Slab::S, &Slab::eps));
        } else {
            for (auto& s : h->slabs)
                if (s.y0 == 0) {
                    k_origin<<<1, 32, 0, h->stream>>>(s.S, s.ehat, s.sp.cs, eb, Nd);
                    AM_CUDA(cudaGetLastError());
                }
            AM_TRY(inverse(h, &Slab::S, &Slab::eps));
        }
        if (h->timing) {
            AM_TRY(mark(5));
            AM_CUDA(cudaEventSynchronize(h->ev[5]));
            AM_TRY(acc(4, 5, 3));
        }
    }
    return fail(AM_ERR_NOT_CONVERGED, "basic scheme did not converge in %d iterations (last residual %.3e)",
                max_iterations, info->residual);
}

extern "C" int am_solver_set_warm_start(am_solver* h, int on) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    h->warm_start = on != 0;
    return AM_OK;
}

extern "C" int am_solver_fft_callback(const am_solver* h, int* on) {
    if (!h || !on) return fail(AM_ERR_ARG, "null argument");
    *on = (h->zcb ? 1 : 0) | (h->zpack ? 2 : 0);
    return AM_OK;
}

// eps_n <- eps, ebar_n <- ebar, a_n <- pending (homogenize.py:474-480)
extern "C" int am_solver_commit(am_solver* h, const double* ebar) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    AM_CUDA(cudaSetDevice(h->device));
    for (auto& s : h->slabs)
        AM_CUDA(cudaMemcpyAsync(s.eps_n, s.eps, sizeof(double) * 6 * s.Nl, cudaMemcpyDeviceToDevice, h->stream));
    if (ebar) std::memcpy(h->ebar_n, ebar, sizeof(h->ebar_n));
    if (h->pending) {
        for (auto& s : h->slabs)
            for (auto& p : s.phases) std::swap(p.a_n, p.a_pend);
        h->pending = false;
    }
    AM_CUDA(cudaStreamSynchronize(h->stream));
    return AM_OK;
}

// any per-voxel failure bit of the last sweep (OR over local slabs and ranks)
static int sweep_flags(am_solver* h, uint32_t* any) {
    uint32_t a = 0;
    for (auto& s : h->slabs) {
        uint32_t f = 0;
        AM_CUDA(cudaMemcpyAsync(&f, s.flags, sizeof(f), cudaMemcpyDeviceToHost, h->stream));
        AM_CUDA(cudaStreamSynchronize(h->stream));
        a |= f;
    }
    if (h->comm) {
        double v[5] = {0, 0, 0, 0, 0};
        const uint32_t bits[5] = {AM_VOXEL_NEWTON_FAILED, AM_VOXEL_SINGULAR, AM_VOXEL_NONFINITE, AM_VOXEL_INTEGRATION,
                                  AM_VOXEL_RADIAL};
        for (int i = 0; i < 5; ++i) v[i] = (a & bits[i]) ? 1.0 : 0.0;
        AM_CUDA(cudaMemcpyAsync(h->dsmall, v, sizeof(v), cudaMemcpyHostToDevice, h->stream));
        AM_NCCL(ncclAllReduce(h->dsmall, h->dsmall, 5, ncclDouble, ncclMax, h->comm, h->stream));
        AM_CUDA(cudaMemcpyAsync(v, h->dsmall, sizeof(v), cudaMemcpyDeviceToHost, h->stream));
        AM_CUDA(cudaStreamSynchronize(h->stream));
        a = 0;
        for (int i = 0; i < 5; ++i)
            if (v[i] > 0.0) a |= bits[i];
    }
    *any = a;
    return AM_OK;
}

// the exception the reference raises first for a sweep's failure bits
static int sweep_error(uint32_t any) {
    if (any & AM_VOXEL_NEWTON_FAILED) return fail(AM_ERR_NEWTON, "implicit Euler Newton failed for at least one voxel");
    if (any & AM_VOXEL_INTEGRATION) return fail(AM_ERR_INTEGRATION, "adaptive integration hit a cap");
    if (any & AM_VOXEL_RADIAL) return fail(AM_ERR_RADIAL, "radial return stalled for at least one voxel");
    return AM_OK;
}

// material evaluation of the current eps field (Homogenizer.evaluate_field,
// homogenize.py:389-421) without tangent: sigma field, states -> a_tmp.
// The pending state of the last solve_step is not touched.
extern "C" int am_solver_evaluate(am_solver* h, double dt) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    AM_CUDA(cudaSetDevice(h->device));
    AM_TRY(material_sweep(h, dt));
    uint32_t any = 0;
    AM_TRY(sweep_flags(h, &any));
    return sweep_error(any);
}

// Tangent sweep of the current eps from the committed state (the
// evaluate_field(want_tangent=True) of run_loading_path, homogenize.py:509)
// fused with reference_update (homogenize.py:307-329): C is produced in
// chunks of whole x planes and reduced per (phase, plane, part) to C_bar
// (36) and the spectral bounds; it is stored only if C_out (host,
// (N_local, 6, 6) in voxel order of the local slabs) is given.  Refreshes
// sigma; states -> a_tmp (the pending state of solve_step is kept, as the
// reference commits solve_step's state, homogenize.py:508-512).
extern "C" int am_solver_tangent_sweep(am_solver* h, double dt, double* Cbar, double* lam_mu, double* C_out) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    AM_CUDA(cudaSetDevice(h->device));
    const int64_t ns = h->nstat;
    double* dsum = h->ps;             // ns x kSum
    double* dmin = h->ps + ns * kSum; // ns x 4
    AM_CUDA(cudaMemsetAsync(dsum, 0, sizeof(double) * ns * kSum, h->stream));
    k_fill<<<grid_for(ns * 4), 256, 0, h->stream>>>(dmin, ns * 4, INFINITY);
    AM_CUDA(cudaGetLastError());
    std::vector<double> hC;
    std::vector<int64_t> hidx;
    int64_t vbase = 0;
    for (auto& s : h->slabs) {
        AM_CUDA(cudaMemsetAsync(s.flags, 0, sizeof(uint32_t), h->stream));
        for (size_t ip = 0; ip < s.phases.size(); ++ip) {
            Phase& p = s.phases[ip];
            if (!p.count) continue;
            if (C_out) {
                hidx.resize(p.count);
                AM_CUDA(cudaMemcpy(hidx.data(), p.gidx, sizeof(int64_t) * p.count, cudaMemcpyDeviceToHost));
            }
            for (int xa = 0; xa < s.nxl;) {
                int xb = xa + 1;  // planes [xa, xb): as many as fit the chunk
                while (xb < s.nxl && p.poff[xb + 1] - p.poff[xa] <= h->chunk) ++xb;
                const int64_t lo = p.poff[xa], n = p.poff[xb] - lo;
                if (n > 0) {
                    KArgs k{};
                    k.B = n;
                    k.gidx = p.gidx + lo;
                    k.eps_n = s.eps_n; k.eps_np1 = s.eps;
                    k.a_n = p.m ? p.a_n + lo : nullptr;
                    k.dt = nullptr; k.dt_scalar = dt;
                    k.le = {s.Nl, 1}; k.la = {p.count, 1}; k.lc = {n, 1};
                    k.sigma = s.sigma; k.a_out = p.m ? p.a_tmp + lo : nullptr; k.C = h->Cbuf;
                    k.iters = nullptr; k.status = h->status; k.flags = s.flags;
                    set_controls(k, &h->cfg);
                    AM_TRY(launch_material(&p.law, k, h->stream));
                    const int64_t rec = ((int64_t)h->phase_rec[ip] * h->nx + s.x0 + xa) * kSParts;
                    k_refstats_planes<<<(unsigned)((xb - xa) * kSParts), kRedThreads, 0, h->stream>>>(
                        h->Cbuf, n, p.dpoff, xa, lo, h->db, dsum + rec * kSum, dmin + rec * 4);
                    AM_CUDA(cudaGetLastError());
                    if (C_out) {
                        hC.resize((size_t)36 * n);
                        AM_CUDA(cudaMemcpyAsync(hC.data(), h->Cbuf, sizeof(double) * 36 * n, cudaMemcpyDeviceToHost,
                                                h->stream));
                        AM_CUDA(cudaStreamSynchronize(h->stream));
                        for (int64_t b = 0; b < n; ++b)
                            for (int e = 0; e < 36; ++e)
                                C_out[(vbase + hidx[lo + b]) * 36 + e] = hC[(size_t)e * n + b];
                    }
                }
                xa = xb;
            }
        }
        vbase += s.Nl;
    }
    if (h->comm) {
        // records are disjoint across ranks (zero / +inf where not owned)
        AM_NCCL(ncclAllReduce(dsum, dsum, ns * kSum, ncclDouble, ncclSum, h->comm, h->stream));
        AM_NCCL(ncclAllReduce(dmin, dmin, ns * 4, ncclDouble, ncclMin, h->comm, h->stream));
    }
    AM_CUDA(cudaMemcpyAsync(h->hps, h->ps, sizeof(double) * ns * kStat, cudaMemcpyDeviceToHost, h->stream));
    AM_CUDA(cudaStreamSynchronize(h->stream));
    uint32_t any = 0;
    AM_TRY(sweep_flags(h, &any));
    Stats st;
    st.reset();
    for (int64_t r = 0; r < ns; ++r) {  // fixed order: phase, global x plane, part
        st.add_sums(h->hps + r * kSum);
        st.add_mins(h->hps + ns * kSum + r * 4);
    }
    AM_TRY(sweep_error(any));
    if (Cbar)
        for (int i = 0; i < 36; ++i) Cbar[i] = st.Csum[i] / (double)h->N;
    // the tangent LU raises inside evaluate_field (odeint.py:424), before
    // reference_update sees the field (homogenize.py:316-317)
    if (any & AM_VOXEL_SINGULAR) return fail(AM_ERR_SINGULAR, "pivot below 1e-14 * max|A| in the tangent LU");
    if (st.bad > 0.0 || (any & AM_VOXEL_NONFINITE))
        return fail(AM_ERR_NONFINITE, "tangent field contains non-finite entries");
    if (lam_mu) {
        const double mu_ref = 0.5 * (st.mlo + st.mhi);
        const double kappa_ref = 0.5 * (st.kmin + st.kmax);
        lam_mu[0] = kappa_ref - 2.0 * mu_ref / 3.0;
        lam_mu[1] = mu_ref;
    }
    return AM_OK;
}

// ---------------------------------------------------------------- host transfer
// which: 0 eps, 1 eps_n, 2 sigma.  Host layout (6, nx_local, ny, nz): the
// whole grid in local mode, this rank's x-slab in nccl mode.
static double* Slab::*field_member(int which) {
    return which == 0 ? &Slab::eps : which == 1 ? &Slab::eps_n : which == 2 ? &Slab::sigma : nullptr;
}

static int field_copy(am_solver* h, int which, double* host, bool to_host) {
    auto f = field_member(which);
    if (!h || !host || !f) return fail(AM_ERR_ARG, "bad field arguments");
    AM_CUDA(cudaSetDevice(h->device));
    AM_CUDA(cudaStreamSynchronize(h->stream));
    const int64_t nloc = (int64_t)h->slabs.size() * h->slabs[0].Nl;  // voxels held by this process
    for (size_t i = 0; i < h->slabs.size(); ++i) {
        Slab& s = h->slabs[i];
        for (int c = 0; c < 6; ++c) {
            double* hp = host + (int64_t)c * nloc + (int64_t)i * s.Nl;
            double* dp = s.*f + (int64_t)c * s.Nl;
            if (to_host) AM_CUDA(cudaMemcpy(hp, dp, sizeof(double) * s.Nl, cudaMemcpyDeviceToHost));
            else AM_CUDA(cudaMemcpy(dp, hp, sizeof(double) * s.Nl, cudaMemcpyHostToDevice));
        }
    }
    return AM_OK;
}

extern "C" int am_solver_get_field(am_solver* h, int which, double* out) { return field_copy(h, which, out, true); }

extern "C" int am_solver_set_field(am_solver* h, int which, const double* in) {
    return field_copy(h, which, const_cast<double*>(in), false);
}

// per-phase state, host (count, m) in voxel order over the local slabs;
// pending = 0 committed, 1 pending (last converged solve_step), 2 the last
// evaluation (evaluate / tangent sweep)
static int state_copy(am_solver* h, int phase, int pending, double* host, bool to_host) {
    if (!h || phase < 0 || phase >= (int)h->slabs[0].phases.size()) return fail(AM_ERR_ARG, "bad phase");
    AM_CUDA(cudaSetDevice(h->device));
    AM_CUDA(cudaStreamSynchronize(h->stream));
    int64_t off = 0;
    for (auto& s : h->slabs) {
        const Phase& p = s.phases[phase];
        if (p.m && p.count) {
            std::vector<double> soa((size_t)p.m * p.count);
            double* dp = pending == 2 ? p.a_tmp : pending ? p.a_pend : p.a_n;
            if (to_host) {
                AM_CUDA(cudaMemcpy(soa.data(), dp, sizeof(double) * soa.size(), cudaMemcpyDeviceToHost));
                for (int64_t b = 0; b < p.count; ++b)
                    for (int c = 0; c < p.m; ++c) host[(off + b) * p.m + c] = soa[(size_t)c * p.count + b];
            } else {
                for (int64_t b = 0; b < p.count; ++b)
                    for (int c = 0; c < p.m; ++c) soa[(size_t)c * p.count + b] = host[(off + b) * p.m + c];
                AM_CUDA(cudaMemcpy(dp, soa.data(), sizeof(double) * soa.size(), cudaMemcpyHostToDevice));
            }
        }
        off += p.count;
    }
    return AM_OK;
}

extern "C" int am_solver_get_state(am_solver* h, int phase, int pending, double* out) {
    return state_copy(h, phase, pending, out, true);
}

extern "C" int am_solver_set_state(am_solver* h, int phase, const double* in) {
    return state_copy(h, phase, 0, const_cast<double*>(in), false);
}

extern "C" int am_solver_phase_count(am_solver* h, int phase, int64_t* count) {
    if (!h || !count || phase < 0 || phase >= (int)h->slabs[0].phases.size()) return fail(AM_ERR_ARG, "bad phase");
    int64_t c = 0;
    for (auto& s : h->slabs) c += s.phases[phase].count;
    *count = c;
    return AM_OK;
}

// Per-phase device time of solve_step iterations (CUDA events on the solver
// stream): out[0..4] = ms in material sweeps, forward FFT, Fourier kernel +
// reduction, origin + inverse FFT, and the number of iterations timed.
// enable: 1 on (resets the accumulators), 0 off, -1 query only.
extern "C" int am_solver_timing(am_solver* h, int enable, double* out) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    AM_CUDA(cudaSetDevice(h->device));
    if (enable >= 0) {
        if (enable && !h->ev[0])
            for (auto& e : h->ev) AM_CUDA(cudaEventCreate(&e));
        h->timing = enable != 0;
        for (double& t : h->t_ms) t = 0.0;
    }
    if (out)
        for (int i = 0; i < 5; ++i) out[i] = h->t_ms[i];
    return AM_OK;
}

extern "C" int am_solver_synchronize(am_solver* h) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    AM_CUDA(cudaStreamSynchronize(h->stream));
    return AM_OK;
}

extern "C" int am_solver_stream(am_solver* h, void** stream) {
    if (!h || !stream) return fail(AM_ERR_ARG, "bad arguments");
    *stream = (void*)h->stream;
    return AM_OK;
}

// ---------------------------------------------------------------- standalone field operators
// GreenOperator(dims, ref).apply(tau) (homogenize.py:229-233), host (6,nx,ny,nz)
extern "C" int am_green_apply_host(int nx, int ny, int nz, double lam, double mu, const double* tau, double* out) {
    if (nx <= 0 || ny <= 0 || nz <= 0 || !tau || !out) return fail(AM_ERR_ARG, "am_green_apply_host: bad arguments");
    const Spec sp = spec_single(nx, ny, nz);
    const int64_t N = sp.N, Nh = sp.cs;
    double* f = nullptr;
    double2* c = nullptr;
    cufftHandle p1 = 0, p2 = 0;
    int rc = AM_OK;
    long long n3[3] = {nx, ny, nz};
    size_t ws;
    if (cudaMalloc(&f, sizeof(double) * 6 * N) != cudaSuccess || cudaMalloc(&c, sizeof(double2) * 6 * Nh) != cudaSuccess)
        rc = fail(AM_ERR_CUDA, "am_green_apply_host: out of memory");
    if (rc == AM_OK && (cufftCreate(&p1) != CUFFT_SUCCESS || cufftCreate(&p2) != CUFFT_SUCCESS ||
                        cufftMakePlanMany64(p1, 3, n3, nullptr, 1, N, nullptr, 1, Nh, CUFFT_D2Z, 6, &ws) != CUFFT_SUCCESS ||
                        cufftMakePlanMany64(p2, 3, n3, nullptr, 1, Nh, nullptr, 1, N, CUFFT_Z2D, 6, &ws) != CUFFT_SUCCESS))
        rc = fail(AM_ERR_CUDA, "am_green_apply_host: cufft plan failed");
    if (rc == AM_OK && cudaMemcpy(f, tau, sizeof(double) * 6 * N, cudaMemcpyHostToDevice) != cudaSuccess)
        rc = fail(AM_ERR_CUDA, "copy failed");
    if (rc == AM_OK && cufftExecD2Z(p1, f, c) != CUFFT_SUCCESS) rc = fail(AM_ERR_CUDA, "D2Z failed");
    if (rc == AM_OK) {
        k_green<<<grid_for(Nh), 256>>>(sp, RefMat::make(lam, mu), c);
        if (cudaGetLastError() != cudaSuccess) rc = fail(AM_ERR_CUDA, "k_green launch failed");
    }
    if (rc == AM_OK && cufftExecZ2D(p2, c, f) != CUFFT_SUCCESS) rc = fail(AM_ERR_CUDA, "Z2D failed");
    if (rc == AM_OK && cudaMemcpy(out, f, sizeof(double) * 6 * N, cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = fail(AM_ERR_CUDA, "copy failed");
    if (p1) cufftDestroy(p1);
    if (p2) cufftDestroy(p2);
    cudaFree(f);
    cudaFree(c);
    return rc;
}

// equilibrium_residual(sig) (homogenize.py:241-267), host (6,nx,ny,nz)
extern "C" int am_equilibrium_residual_host(int nx, int ny, int nz, const double* sig, double* res) {
    if (nx <= 0 || ny <= 0 || nz <= 0 || !sig || !res) return fail(AM_ERR_ARG, "bad arguments");
    const Spec sp = spec_single(nx, ny, nz);
    const int64_t N = sp.N, Nh = sp.cs, L = (int64_t)ny * kParts + 10;
    double *f = nullptr, *red = nullptr;
    double2* c = nullptr;
    cufftHandle p1 = 0;
    int rc = AM_OK;
    long long n3[3] = {nx, ny, nz};
    size_t ws;
    std::vector<double> o(L);
    if (cudaMalloc(&f, sizeof(double) * 6 * N) != cudaSuccess || cudaMalloc(&c, sizeof(double2) * 6 * Nh) != cudaSuccess ||
        cudaMalloc(&red, sizeof(double) * L) != cudaSuccess)
        rc = fail(AM_ERR_CUDA, "out of memory");
    if (rc == AM_OK && (cufftCreate(&p1) != CUFFT_SUCCESS ||
                        cufftMakePlanMany64(p1, 3, n3, nullptr, 1, N, nullptr, 1, Nh, CUFFT_D2Z, 6, &ws) != CUFFT_SUCCESS))
        rc = fail(AM_ERR_CUDA, "cufft plan failed");
    if (rc == AM_OK && cudaMemcpy(f, sig, sizeof(double) * 6 * N, cudaMemcpyHostToDevice) != cudaSuccess)
        rc = fail(AM_ERR_CUDA, "copy failed");
    if (rc == AM_OK && cufftExecD2Z(p1, f, c) != CUFFT_SUCCESS) rc = fail(AM_ERR_CUDA, "D2Z failed");
    if (rc == AM_OK) {
        k_fourier<<<ny * kParts, kRedThreads>>>(sp, RefMat::make(1.0, 1.0), c, nullptr, red, 0, 0);
        k_finish<<<1, 32>>>(c, sp.cs, 1, nullptr, nullptr, red, (int64_t)ny * kParts);
        if (cudaMemcpy(o.data(), red, sizeof(double) * L, cudaMemcpyDeviceToHost) != cudaSuccess)
            rc = fail(AM_ERR_CUDA, "residual kernel failed");
    }
    if (rc == AM_OK) {
        double fsum = 0.0;
        for (int64_t i = 0; i < (int64_t)ny * kParts; ++i) fsum += o[i];
        // the reference's sigma_bar is the voxel mean: rfft(sigma)(0) / N
        double sbar[6];
        for (int i = 0; i < 6; ++i) sbar[i] = o[(int64_t)ny * kParts + i] / (double)N;
        *res = std::sqrt(fsum / ((double)N * (double)N)) / std::max(dup_norm(sbar), 1e-300);
    }
    if (p1) cufftDestroy(p1);
    cudaFree(f); cudaFree(c); cudaFree(red);
    return rc;
}

// apply_isotropic(ref, eps) (homogenize.py:270-281), host (6, N)
extern "C" int am_apply_isotropic_host(int64_t N, double lam, double mu, const double* eps, double* out) {
    if (N < 0 || (N && (!eps || !out))) return fail(AM_ERR_ARG, "bad arguments");
    if (!N) return AM_OK;
    double* f;
    AM_CUDA(cudaMalloc(&f, sizeof(double) * 12 * N));
    int rc = AM_OK;
    if (cudaMemcpy(f, eps, sizeof(double) * 6 * N, cudaMemcpyHostToDevice) != cudaSuccess) rc = fail(AM_ERR_CUDA, "copy");
    if (rc == AM_OK) {
        k_isotropic<<<grid_for(N), 256>>>(RefMat::make(lam, mu), f, f + 6 * N, N);
        if (cudaMemcpy(out, f + 6 * N, sizeof(double) * 6 * N, cudaMemcpyDeviceToHost) != cudaSuccess)
            rc = fail(AM_ERR_CUDA, "copy");
    }
    cudaFree(f);
    return rc;
}

// reference_update(C_field) (homogenize.py:307-329), host (n, 6, 6)
extern "C" int am_reference_update_host(int64_t n, const double* C, double* lam, double* mu) {
    if (n <= 0 || !C || !lam || !mu) return fail(AM_ERR_ARG, "reference_update needs at least one tangent");
    double *d = nullptr, *stats = nullptr;
    AM_CUDA(cudaMalloc(&d, sizeof(double) * 36 * n));
    int rc = AM_OK;
    std::vector<double> soa((size_t)36 * n), hs((size_t)kStat * kRedBlocks);
    for (int64_t b = 0; b < n; ++b)
        for (int e = 0; e < 36; ++e) soa[(size_t)e * n + b] = C[b * 36 + e];
    if (cudaMalloc(&stats, sizeof(double) * kStat * kRedBlocks) != cudaSuccess) rc = fail(AM_ERR_CUDA, "oom");
    if (rc == AM_OK && cudaMemcpy(d, soa.data(), sizeof(double) * soa.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        rc = fail(AM_ERR_CUDA, "copy");
    if (rc == AM_OK) {
        k_refstats<<<kRedBlocks, kRedThreads>>>(d, n, n, DevBasis::make(), stats);
        if (cudaMemcpy(hs.data(), stats, sizeof(double) * hs.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
            rc = fail(AM_ERR_CUDA, "reference_update kernel failed");
    }
    if (rc == AM_OK) {
        Stats st;
        st.reset();
        for (int b = 0; b < kRedBlocks; ++b) st.add(hs.data() + (size_t)b * kStat);
        if (st.bad > 0.0) {
            rc = fail(AM_ERR_NONFINITE, "tangent field contains non-finite entries");
        } else {
            const double mu_ref = 0.5 * (st.mlo + st.mhi);
            const double kappa_ref = 0.5 * (st.kmin + st.kmax);
            *lam = kappa_ref - 2.0 * mu_ref / 3.0;
            *mu = mu_ref;
        }
    }
    cudaFree(d);
    cudaFree(stats);
    return rc;
}
