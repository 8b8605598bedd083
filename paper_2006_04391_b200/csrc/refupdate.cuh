// refupdate.cuh -- per-voxel spectral bounds of a consistent tangent for the
// reference-material update (gsmkit/homogenize.py:288-329, reference_update):
//   C <- (C + C^T)/2, C^ = M C M (Mandel, sqrt 2 on shear),
//   kappa = vol . C^ vol / 3, mu_lo/hi = extreme eigenvalues of the 5x5
//   deviatoric block B^T C^ B, halved.
// The reference takes all eigenvalues with LAPACK eigvalsh and keeps the
// extremes; here a cyclic Jacobi iteration in registers (accurate to a few
// ulp of the spectral radius) gives the same extremes.  Host + device.
#pragma once

#include <cmath>

#include "ad.cuh"  // AM_HD, sfor

namespace am {

// the orthonormal deviatoric basis of the reference (_dev_basis,
// homogenize.py:292-304): Gram-Schmidt of (I - vol vol^T) e_i, first five
// vectors; Bt[p][i] = B[i][p]
struct DevBasis {
    double Bt[5][6];
    double vol[6];

    static DevBasis make() {
        DevBasis d;
        const double v = 1.0 / std::sqrt(3.0);
        for (int i = 0; i < 6; ++i) d.vol[i] = i < 3 ? v : 0.0;
        double basis[6][6];
        int nb = 0;
        for (int e = 0; e < 6 && nb < 5; ++e) {
            double x[6];
            double dv = 0.0;
            for (int i = 0; i < 6; ++i) dv += (i == e ? 1.0 : 0.0) * d.vol[i];
            for (int i = 0; i < 6; ++i) x[i] = (i == e ? 1.0 : 0.0) - dv * d.vol[i];
            for (int b = 0; b < nb; ++b) {
                double p = 0.0;
                for (int i = 0; i < 6; ++i) p += x[i] * basis[b][i];
                for (int i = 0; i < 6; ++i) x[i] -= p * basis[b][i];
            }
            double nrm = 0.0;
            for (int i = 0; i < 6; ++i) nrm += x[i] * x[i];
            nrm = std::sqrt(nrm);
            if (nrm > 1e-12) {
                for (int i = 0; i < 6; ++i) basis[nb][i] = x[i] / nrm;
                ++nb;
            }
        }
        for (int p = 0; p < 5; ++p)
            for (int i = 0; i < 6; ++i) d.Bt[p][i] = basis[p][i];
        return d;
    }
};

// extreme eigenvalues of a symmetric 5x5 matrix (destroys A)
AM_HD void sym5_extremes(double (&A)[5][5], double& lo, double& hi) {
    for (int sweep = 0; sweep < 12; ++sweep) {
        double off = 0.0, dia = 0.0;
#pragma unroll
        for (int p = 0; p < 5; ++p) {
            dia += A[p][p] * A[p][p];
#pragma unroll
            for (int q = p + 1; q < 5; ++q) off += A[p][q] * A[p][q];
        }
        if (!(off > 1e-36 * dia)) break;  // also stops on NaN
        sfor<5>([&](auto P) {
            constexpr int p = decltype(P)::value;
            sfor<5>([&](auto Q) {
                constexpr int q = decltype(Q)::value;
                if constexpr (q > p) {
                    const double apq = A[p][q];
                    if (apq != 0.0) {
                        // Golub & Van Loan sym.schur2
                        const double tau = (A[q][q] - A[p][p]) / (2.0 * apq);
                        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
#pragma unroll
                        for (int k = 0; k < 5; ++k) {
                            const double akp = A[k][p], akq = A[k][q];
                            A[k][p] = c * akp - s * akq;
                            A[k][q] = s * akp + c * akq;
                        }
#pragma unroll
                        for (int k = 0; k < 5; ++k) {
                            const double apk = A[p][k], aqk = A[q][k];
                            A[p][k] = c * apk - s * aqk;
                            A[q][k] = s * apk + c * aqk;
                        }
                    }
                }
            });
        });
    }
    lo = A[0][0];
    hi = A[0][0];
#pragma unroll
    for (int p = 1; p < 5; ++p) {
        lo = fmin(lo, A[p][p]);
        hi = fmax(hi, A[p][p]);
    }
}

// kappa and the halved deviatoric eigenvalue extremes of one tangent
AM_HD void tangent_bounds(const double (*C)[6], const DevBasis& db, double& kappa, double& mu_lo, double& mu_hi) {
    const double r2 = 1.4142135623730951;  // np.sqrt(2.0)
    double H[6][6];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            const double s = 0.5 * (C[i][j] + C[j][i]);
            H[i][j] = s * (i < 3 ? 1.0 : r2) * (j < 3 ? 1.0 : r2);
        }
    double k = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) k += db.vol[i] * H[i][j] * db.vol[j];
    kappa = k / 3.0;
    double T[5][6], A[5][5];
#pragma unroll
    for (int p = 0; p < 5; ++p)
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < 6; ++i) s += db.Bt[p][i] * H[i][j];
            T[p][j] = s;
        }
#pragma unroll
    for (int p = 0; p < 5; ++p)
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < 6; ++j) s += T[p][j] * db.Bt[q][j];
            A[p][q] = s;
        }
    // symmetrise exactly (the reference's eigvalsh reads one triangle)
#pragma unroll
    for (int p = 0; p < 5; ++p)
#pragma unroll
        for (int q = p + 1; q < 5; ++q) A[q][p] = A[p][q];
    double lo, hi;
    sym5_extremes(A, lo, hi);
    mu_lo = lo / 2.0;
    mu_hi = hi / 2.0;
}

}  // namespace am
