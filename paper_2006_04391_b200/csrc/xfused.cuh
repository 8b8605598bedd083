// xfused.cuh -- the single-GPU basic scheme's spectral step with the x
// transforms fused into the Fourier update (nx = 256).
//
// The 3-D D2Z / Z2D of sigma / eps are split into a batched 2-D (y, z)
// cuFFT and the x direction, and the x direction is done here, in shared
// memory, together with the per-bin work of k_fourier:
//
//   S  (6, nx, ny, nzh)  2-D spectra of sigma            (in)
//   x-FFT -> sigma_hat -> residual partial, ehat' = -Gamma0 (sigma_hat - C0 ehat)
//   ehat (6, nx, ny, nzh) rfft(eps), same layout as the 3-D cuFFT spectrum (in / out)
//   x-IFFT of ehat'/N (origin bin 0) -> S, the 2-D spectra of the next eps (out)
//
// which removes the two x passes of cuFFT (each a full read + write of the
// spectrum) from every iteration: the kernel moves 4 x 96 bytes per rfft
// bin, the same as k_fourier alone.  The origin bin is added afterwards by
// k_origin_x, once the host has solved the mixed boundary conditions
// (its inverse x transform is the constant ebar along the (ky, kz) = 0 line).
//
// CTA tile (v3): XJ = 2 consecutive (ky, kz) columns j = ky * nzh + kz (a
// 32-byte sector for each (c, x)), all 256 x and 6 components, staged in
// shared memory (52 KB: 4 CTAs per SM, a persistent grid).  Each of the 12
// lines is transformed by 16 threads of one warp with a 16 x 16
// decomposition (radix-16 DFTs in registers, one table of 256 twiddles,
// lines padded to 17-element rows against bank conflicts) and only warp
// barriers; CTA barriers separate load / Fourier update / store.  v2 (4
// columns, 384 threads, CTA-wide barriers inside the FFTs, 1 CTA per SM)
// was issue-latency bound at 12 warps per SM (1.44 ms at 256^3).
// Residual partials are per tile, reduced in a fixed order.
//
// Status: opt-in (AM_XFUSED=1).  Parity-tested; at 256^3 v3 takes 1.30 ms
// (2 CTAs/SM, no spills; 1.38 at 3, 1.93 at 4 with spills) against 1.16 ms
// for k_fourier + cuFFT's two x passes, so the 3-D cuFFT path stays the
// default: the 32-byte (c, x) rows of a 2-column tile give the DRAM poor
// locality, and tiles wide enough for 128-byte rows need ~200 KB of shared
// memory (profiles/r01/k1_variants.log, r2 entries).
#pragma once

#include "fourier.cuh"

namespace am {

constexpr int kXN = 256;                 // supported nx
#ifndef AM_XF_J
#define AM_XF_J 2
#endif
constexpr int kXJ = AM_XF_J;             // (ky, kz) columns per tile
constexpr int kXLines = 6 * kXJ;         // lines per tile
constexpr int kXThreads = kXLines * 16;  // 16 threads per line: 192
#ifndef AM_XF_CTAS
#define AM_XF_CTAS 2
#endif
constexpr int kXCtas = AM_XF_CTAS;       // resident CTAs per SM
constexpr int kXRow = 273;               // padded line: pos(x) = (x & 15) + 17 (x >> 4) < 271;
                                         // odd, so the two columns of a component sit in different banks

__device__ __forceinline__ int xpos(int x) { return (x & 15) + 17 * (x >> 4); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 w) {
    return make_double2(a.x * w.x - a.y * w.y, a.x * w.y + a.y * w.x);
}
// a * (S i)
template <int S>
__device__ __forceinline__ double2 mul_i(double2 a) {
    return S < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}
// a * exp(S i pi m / 8) for the constant m of the 16-point DFT
template <int S, int M>
__device__ __forceinline__ double2 w16(double2 a) {
    constexpr double c1 = 0.92387953251128674, s1 = 0.38268343236508978, h = 0.70710678118654757;
    if constexpr (M == 0) return a;
    else if constexpr (M == 4) return mul_i<S>(a);
    else {
        constexpr double cr = M == 1 ? c1 : M == 2 ? h : M == 3 ? s1 : M == 6 ? -h : -c1;  // 9: -c1
        constexpr double ci = M == 1 ? s1 : M == 2 ? h : M == 3 ? c1 : M == 6 ? h : -s1;   // 9: -s1
        return cmul(a, make_double2(cr, S * ci));
    }
}

template <int S>
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
    const double2 t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = mul_i<S>(csub(a1, a3));
    a0 = cadd(t0, t2);
    a2 = csub(t0, t2);
    a1 = cadd(t1, t3);
    a3 = csub(t1, t3);
}

// in-place 16-point DFT, sign S, natural order in and out
template <int S>
__device__ __forceinline__ void dft16(double2* v) {
    // n = n1 + 4 n2: DFT4 over n2 -> A[n1][k1] at v[n1 + 4 k1]
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) dft4<S>(v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]);
    // twiddles W16^(n1 k1)
    v[5] = w16<S, 1>(v[5]);
    v[6] = w16<S, 2>(v[6]);
    v[7] = w16<S, 3>(v[7]);
    v[9] = w16<S, 2>(v[9]);
    v[10] = w16<S, 4>(v[10]);
    v[11] = w16<S, 6>(v[11]);
    v[13] = w16<S, 3>(v[13]);
    v[14] = w16<S, 6>(v[14]);
    v[15] = w16<S, 9>(v[15]);
    // DFT4 over n1 for each k1: X[k1 + 4 k2] at v[4 k1 + k2]
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4<S>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
    // transpose the 4 x 4 index to natural order
    double2 t;
    t = v[1]; v[1] = v[4]; v[4] = t;
    t = v[2]; v[2] = v[8]; v[8] = t;
    t = v[3]; v[3] = v[12]; v[12] = t;
    t = v[6]; v[6] = v[9]; v[9] = t;
    t = v[7]; v[7] = v[13]; v[13] = t;
    t = v[11]; v[11] = v[14]; v[14] = t;
}

// 256-point DFT (sign S) of one line, natural order at xpos(); thread i
// (0..15) of the 16 threads of its line, which share a warp (warp barriers
// only).  tw[m] = exp(-2 pi i m / 256).
template <int S>
__device__ __forceinline__ void line_fft256(double2* line, const double2* tw, int i) {
    double2 v[16];
    // x = n1 + 16 n2, n1 = i: DFT16 over n2, twiddle W256^(n1 k1)
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) v[n2] = line[i + 17 * n2];
    dft16<S>(v);
#pragma unroll
    for (int k1 = 1; k1 < 16; ++k1) {
        const double2 w = tw[i * k1];
        v[k1] = cmul(v[k1], make_double2(w.x, S < 0 ? w.y : -w.y));
    }
    __syncwarp();
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) line[i + 17 * k1] = v[k1];
    __syncwarp();
    // k1 = i: DFT16 over n1 -> X[k1 + 16 k2]
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) v[n1] = line[n1 + 17 * i];
    dft16<S>(v);
    __syncwarp();
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) line[i + 17 * k2] = v[k2];
    __syncwarp();
}

// 16-byte asynchronous global -> shared copy; zero fill when !valid
__device__ __forceinline__ void cp_async16(double2* dst, const double2* src, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

#ifndef AM_XF_PREFETCH
#define AM_XF_PREFETCH 0
#endif
constexpr int kXNB = AM_XF_PREFETCH ? 2 : 1;  // tile buffers (2: the next tile prefetched with cp.async)

// stage tile `tile` of the 2-D spectra into buf (asynchronous)
__device__ __forceinline__ void xtile_prefetch(double2* buf, const double2* __restrict__ S, int64_t cs, int64_t ncol,
                                               int64_t tile) {
    const int64_t j0 = tile * kXJ;
#pragma unroll
    for (int r = 0; r < kXLines * kXN / kXThreads; ++r) {
        const int e = threadIdx.x + r * kXThreads;
        const int jj = e & (kXJ - 1), x = (e / kXJ) & (kXN - 1), c = e / (kXJ * kXN);
        const int64_t j = j0 + jj;
        cp_async16(buf + (c * kXJ + jj) * kXRow + xpos(x), S + (j < ncol ? c * cs + x * ncol + j : 0), j < ncol);
    }
}

// Persistent: CTA b handles tiles b, b + grid, ...  red[tile] = the tile's
// residual partial; red[P + c] = Re sigma_hat(origin) (the caller zeroes the
// slots).  S: 2-D spectra (c, x, j) in, 2-D spectra of the next eps (without
// its origin, k_origin_x) out; ehat: rfft(eps) (c, kx, j) in / out.
__global__ void __launch_bounds__(kXThreads, kXCtas) k_xfourier(int nx, int ny, int nz, int64_t cs, RefMat ref,
                                                                double2* __restrict__ S, double2* __restrict__ ehat,
                                                                double* __restrict__ red, int64_t P) {
    extern __shared__ double2 xsm[];
    double2* tw = xsm + kXNB * kXLines * kXRow;  // [256]
    __shared__ double rsh[kXThreads / 32];
    const int nzh = nz / 2 + 1;
    const int64_t ncol = (int64_t)ny * nzh;  // = x stride of the 2-D spectra
    const int64_t ntiles = (ncol + kXJ - 1) / kXJ;
    const int t = threadIdx.x;
    for (int m = t; m < kXN; m += kXThreads) {
        double s, c;
        sincospi(-(double)m / 128.0, &s, &c);
        tw[m] = make_double2(c, s);
    }
    const int L = t >> 4, i = t & 15;  // line L = c * kXJ + jj
    const double invN = 1.0 / ((double)nx * ny * nz);
    constexpr int kE = kXLines * kXN / kXThreads;  // tile elements per thread: 16
    if (kXNB == 2) {
        if (blockIdx.x < ntiles) xtile_prefetch(xsm, S, cs, ncol, blockIdx.x);
        cp_async_commit();
    }
    int cur = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, cur ^= (kXNB - 1)) {
        const int64_t j0 = tile * kXJ;
        double2* xs = xsm + cur * kXLines * kXRow;  // this tile's lines
        double2* line = xs + L * kXRow;
        if constexpr (kXNB == 2) {
            // the next tile streams in while this one is transformed
            if (tile + gridDim.x < ntiles) xtile_prefetch(xsm + (cur ^ 1) * kXLines * kXRow, S, cs, ncol, tile + gridDim.x);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            // load: element e -> (c, x, jj), consecutive threads take the
            // columns of one (c, x) row
#pragma unroll
            for (int r = 0; r < kE; ++r) {
                const int e = t + r * kXThreads;
                const int jj = e & (kXJ - 1), x = (e / kXJ) & (kXN - 1), c = e / (kXJ * kXN);
                const int64_t j = j0 + jj;
                xs[(c * kXJ + jj) * kXRow + xpos(x)] =
                    j < ncol ? __ldg(S + c * cs + x * ncol + j) : make_double2(0.0, 0.0);
            }
        }
        __syncthreads();
        line_fft256<-1>(line, tw, i);
        __syncthreads();
        // Fourier update of the tile's 2 x 256 bins
        double acc = 0.0;
        for (int b = t; b < kXN * kXJ; b += kXThreads) {
            const int jj = b & (kXJ - 1), kx = b / kXJ;
            const int64_t j = j0 + jj;
            if (j >= ncol) continue;
            const int ky = (int)(j / nzh), kz = (int)(j - (int64_t)ky * nzh);
            const Bin bn = make_bin(kx, ky, kz, nx, ny, nz);
            double2* cell = xs + jj * kXRow + xpos(kx);  // component c at cell[c * kXJ * kXRow]
            cplx s[6];
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                const double2 w = cell[c * kXJ * kXRow];
                s[c] = cplx{w.x, w.y};
            }
            if (bn.zero) {
#pragma unroll
                for (int c = 0; c < 6; ++c) {
                    red[P + c] = s[c].re;
                    cell[c * kXJ * kXRow] = make_double2(0.0, 0.0);
                }
                continue;
            }
            acc += rfft_weight(kz, nz) * traction_sq(bn, s);
            const int64_t q = (int64_t)kx * ncol + j;
            double er[6], ei[6], cr[6], ci[6], tr[6], ti[6], outr[6], outi[6];
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                const double2 w = ehat[c * cs + q];
                er[c] = w.x;
                ei[c] = w.y;
            }
            iso_apply(ref, er, cr);
            iso_apply(ref, ei, ci);
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                tr[c] = s[c].re - cr[c];
                ti[c] = s[c].im - ci[c];
            }
            green_apply_real(ref, bn, tr, outr);
            green_apply_real(ref, bn, ti, outi);
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                ehat[c * cs + q] = make_double2(outr[c], outi[c]);
                cell[c * kXJ * kXRow] = make_double2(outr[c] * invN, outi[c] * invN);
            }
        }
        // deterministic block reduction of the tile's partial
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
        if ((t & 31) == 0) rsh[t >> 5] = acc;
        __syncthreads();
        if (t == 0) {
            double sum = 0.0;
            for (int w = 0; w < kXThreads / 32; ++w) sum += rsh[w];
            red[tile] = sum;
        }
        line_fft256<1>(line, tw, i);
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kE; ++r) {
            const int e = t + r * kXThreads;
            const int jj = e & (kXJ - 1), x = (e / kXJ) & (kXN - 1), c = e / (kXJ * kXN);
            const int64_t j = j0 + jj;
            if (j < ncol) S[c * cs + x * ncol + j] = xs[(c * kXJ + jj) * kXRow + xpos(x)];
        }
        __syncthreads();  // the lines are read before the next tile overwrites them
    }
    if constexpr (kXNB == 2) cp_async_wait<0>();
}

constexpr size_t kXSmem = sizeof(double2) * (kXNB * kXLines * kXRow + kXN);

}  // namespace am
