// fourier.cuh -- per-frequency math of the Moulinec-Suquet basic scheme:
// numpy frequency conventions, the isotropic Green operator and the
// equilibrium-residual traction, for one rfft bin.  Host + device.
//
// Follows gsmkit/homogenize.py: GreenOperator (174-233), equilibrium_residual
// (241-267), apply_isotropic (270-281).
#pragma once

#include <cmath>
#include <cstdint>

#include "ad.cuh"  // AM_HD

namespace am {

struct cplx {
    double re, im;
};

// numpy.fft.fftfreq(n, 1/n)[i]: 0, 1, ..., (n-1)//2, -(n//2), ..., -1
AM_HD int fftfreq(int i, int n) { return i < (n + 1) / 2 ? i : i - n; }

// isotropic reference (ReferenceMaterial, homogenize.py:37-49) and the
// constants of its Green operator (homogenize.py:213-214) and compliance
// (the Nyquist-bin operator C_ref^-1, homogenize.py:197-203)
struct RefMat {
    double lam, mu;
    double c1, c2;       // 1/(4 mu), (lam + mu)/(mu (lam + 2 mu))
    double s11, s12, s44;  // compliance: normal diag / off-diag, shear (engineering)

    AM_HD static RefMat make(double lam, double mu) {
        RefMat r;
        r.lam = lam; r.mu = mu;
        r.c1 = 1.0 / (4.0 * mu);
        r.c2 = (lam + mu) / (mu * (lam + 2.0 * mu));
        const double d = mu * (3.0 * lam + 2.0 * mu);
        r.s11 = (lam + mu) / d;
        r.s12 = -lam / (2.0 * d);
        r.s44 = 1.0 / mu;
        return r;
    }
};

// unit wave vector of bin (ix, iy, iz) of an (nx, ny, nz/2+1) half spectrum;
// zero at the origin (norm set to 1 there, homogenize.py:209-211)
struct Bin {
    double n0, n1, n2;
    bool zero, nyquist;
};

AM_HD Bin make_bin(int ix, int iy, int iz, int nx, int ny, int nz) {
    const int fx = fftfreq(ix, nx), fy = fftfreq(iy, ny), fz = iz;
    const double x = fx, y = fy, z = fz;
    double norm = sqrt(x * x + y * y + z * z);
    Bin b;
    b.zero = (fx == 0 && fy == 0 && fz == 0);
    if (b.zero) norm = 1.0;
    b.n0 = x / norm; b.n1 = y / norm; b.n2 = z / norm;
    // |f| == n/2 on any axis (only for even n)
    b.nyquist = (2 * (fx < 0 ? -fx : fx) == nx) || (2 * (fy < 0 ? -fy : fy) == ny) || (2 * fz == nz);
    return b;
}

// residual weight of an rfft bin: 2 for the implicit conjugate half, 1 on the
// self-conjugate planes kz = 0 and (even nz) kz = nz/2 (homogenize.py:259-262)
AM_HD double rfft_weight(int iz, int nz) { return (iz == 0 || (nz % 2 == 0 && 2 * iz == nz)) ? 1.0 : 2.0; }

// |t|^2 of the Fourier traction n . sigma_hat (homogenize.py:253-256)
AM_HD double traction_sq(const Bin& b, const cplx* s) {
    const double t0r = b.n0 * s[0].re + b.n1 * s[5].re + b.n2 * s[4].re;
    const double t0i = b.n0 * s[0].im + b.n1 * s[5].im + b.n2 * s[4].im;
    const double t1r = b.n0 * s[5].re + b.n1 * s[1].re + b.n2 * s[3].re;
    const double t1i = b.n0 * s[5].im + b.n1 * s[1].im + b.n2 * s[3].im;
    const double t2r = b.n0 * s[4].re + b.n1 * s[3].re + b.n2 * s[2].re;
    const double t2i = b.n0 * s[4].im + b.n1 * s[3].im + b.n2 * s[2].im;
    return (t0r * t0r + t0i * t0i) + (t1r * t1r + t1i * t1i) + (t2r * t2r + t2i * t2i);
}

// C_ref : eps for engineering-shear strain components (homogenize.py:270-281),
// real or complex (applied to re and im separately)
AM_HD void iso_apply(const RefMat& r, const double* e, double* out) {
    const double tr = e[0] + e[1] + e[2];
    out[0] = r.lam * tr + 2.0 * r.mu * e[0];
    out[1] = r.lam * tr + 2.0 * r.mu * e[1];
    out[2] = r.lam * tr + 2.0 * r.mu * e[2];
    out[3] = r.mu * e[3];
    out[4] = r.mu * e[4];
    out[5] = r.mu * e[5];
}

// corr = -Gamma0(n) tau for one real part (re or im) of a Voigt stress-like
// tau (GreenOperator._assemble, homogenize.py:207-227, contracted with tau):
//   Gamma_khij tau_ij = 2 c1 (n_h (tau n)_k + n_k (tau n)_h) - c2 n_k n_h (n . tau n)
// with the row weight 2 on shear components (engineering strain out).
// Nyquist bins: corr = -C_ref^-1 tau (homogenize.py:197-203).
AM_HD void green_apply_real(const RefMat& r, const Bin& b, const double* t, double* out) {
    if (b.nyquist) {
        const double n = t[0] + t[1] + t[2];
        out[0] = -(r.s12 * n + (r.s11 - r.s12) * t[0]);
        out[1] = -(r.s12 * n + (r.s11 - r.s12) * t[1]);
        out[2] = -(r.s12 * n + (r.s11 - r.s12) * t[2]);
        out[3] = -r.s44 * t[3];
        out[4] = -r.s44 * t[4];
        out[5] = -r.s44 * t[5];
        return;
    }
    // (tau n)_k with Voigt (xx, yy, zz, yz, xz, xy)
    const double u0 = t[0] * b.n0 + t[5] * b.n1 + t[4] * b.n2;
    const double u1 = t[5] * b.n0 + t[1] * b.n1 + t[3] * b.n2;
    const double u2 = t[4] * b.n0 + t[3] * b.n1 + t[2] * b.n2;
    const double s = b.n0 * u0 + b.n1 * u1 + b.n2 * u2;
    const double a = 2.0 * r.c1, c = r.c2 * s;
    // (k, h) = (0,0), (1,1), (2,2), (1,2), (0,2), (0,1)
    out[0] = -(a * (2.0 * b.n0 * u0) - c * b.n0 * b.n0);
    out[1] = -(a * (2.0 * b.n1 * u1) - c * b.n1 * b.n1);
    out[2] = -(a * (2.0 * b.n2 * u2) - c * b.n2 * b.n2);
    out[3] = -2.0 * (a * (b.n2 * u1 + b.n1 * u2) - c * b.n1 * b.n2);
    out[4] = -2.0 * (a * (b.n2 * u0 + b.n0 * u2) - c * b.n0 * b.n2);
    out[5] = -2.0 * (a * (b.n1 * u0 + b.n0 * u1) - c * b.n0 * b.n1);
}

}  // namespace am
