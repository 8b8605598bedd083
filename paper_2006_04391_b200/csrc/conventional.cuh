// conventional.cuh -- the paper's hand-derived baseline for the Michel-Suquet
// law: a single backward-Euler step reduced to a scalar Newton solve on the
// plastic multiplier (radial return) with its closed-form consistent tangent
// (gsmkit gsm.py:332-404 MichelSuquet.conventional_step; the
// strategy="conventional" route of evaluator.py:172-174).  Host + device.
//
// Per point, like every other route here.  The reference's scalar Newton
// stops when the largest relative step over the whole batch is below
// 1e-14; per point that is "this point's step", which changes results by
// round-off only (the extra batch iterations move x by less than an ulp).
#pragma once

#include "semi.cuh"

namespace am {

enum : int { ST_RADIAL = 16 };  // gsm.NewtonError: radial return stalled (gsm.py:377-378)

// returns status; writes sigma, the new state and (C != nullptr) the tangent
AM_HD int conventional_point(const SemiLaw<MichelSuquetLaw>& S, const double* eps_np1, const double* a_n, double h,
                             double* sig, double* a_new, double (*C)[6]) {
    const MichelSuquetLaw& p = S.base;
    const double mu = p.mu;
    const auto e = tup(plain(eps_np1[0]), plain(eps_np1[1]), plain(eps_np1[2]), plain(eps_np1[3]),
                       plain(eps_np1[4]), plain(eps_np1[5]));
    const auto an = tup(plain(a_n[0]), plain(a_n[1]), plain(a_n[2]), plain(a_n[3]), plain(a_n[4]), plain(a_n[5]),
                        plain(a_n[6]));
    const auto A = S.hand_gen_stress(e, an);
    const double At[6] = {get<0>(A).v, get<1>(A).v, get<2>(A).v, get<3>(A).v, get<4>(A).v, get<5>(A).v};
    // s_tr = A_tr[:6] @ DEV6.T
    const double third = 1.0 / 3.0, dd = 1.0 - third;
    double s[6];
    s[0] = At[0] * dd + At[1] * (-third) + At[2] * (-third);
    s[1] = At[0] * (-third) + At[1] * dd + At[2] * (-third);
    s[2] = At[0] * (-third) + At[1] * (-third) + At[2] * dd;
    s[3] = At[3];
    s[4] = At[4];
    s[5] = At[5];
    const double dup[6] = {1, 1, 1, 2, 2, 2};
    double q = 0.0;
    for (int i = 0; i < 6; ++i) q += s[i] * dup[i] * s[i];
    q *= 1.5;
    const double Ntr = sqrt(fmax(q, 0.0));
    const double ytr = Ntr - p.sigma_Y;
    const double keff = 3.0 * mu + p.H;
    const bool plastic = (ytr > 0.0) && (h > 0.0);
    int status = 0;
    double dgam = 0.0;
    if (plastic) {
        const double hi = fmax(ytr / keff * (1.0 - 1e-15), 0.0);
        const double scale = fmax(hi, 1e-30);
        double x = 0.0;
        bool conv = false;
        for (int it = 0; it < 50; ++it) {
            const double ye = ytr - keff * x;
            const double g = h * p.eps0_dot * ::pow(ye / p.sigma_d, p.n);
            const double r = x - g;
            const double rp = 1.0 + keff * h * p.eps0_dot * p.n / p.sigma_d * ::pow(ye / p.sigma_d, p.n - 1.0);
            const double step = r / rp;
            x = fmin(fmax(x - step, 0.0), hi);
            if (fabs(step) / scale < 1e-14) {
                conv = true;
                break;
            }
        }
        if (!conv) status |= ST_RADIAL;
        dgam = x;
    }
    const double safeN = plastic ? Ntr : 1.0;
    const double pl = plastic ? 1.0 : 0.0;
    for (int i = 0; i < 6; ++i) a_new[i] = a_n[i] + dgam * (1.5 * dup[i] * s[i] / safeN * pl);
    a_new[6] = a_n[6] + dgam;
    const auto an1 = tup(plain(a_new[0]), plain(a_new[1]), plain(a_new[2]), plain(a_new[3]), plain(a_new[4]),
                         plain(a_new[5]), plain(a_new[6]));
    const auto sg = S.hand_stress(e, an1);
    sig[0] = get<0>(sg).v; sig[1] = get<1>(sg).v; sig[2] = get<2>(sg).v;
    sig[3] = get<3>(sg).v; sig[4] = get<4>(sg).v; sig[5] = get<5>(sg).v;
    if (C) {
        S.Ce(C);
        if (plastic) {
            const double ye = ytr - keff * dgam;
            const double gp = h * p.eps0_dot * p.n / p.sigma_d * ::pow(ye / p.sigma_d, p.n - 1.0);
            const double beta = gp / (1.0 + keff * gp);
            double ns[6];
            for (int i = 0; i < 6; ++i) ns[i] = 1.5 * s[i] / safeN;
            const double c1 = 4.0 * mu * mu * (beta - dgam / safeN) * pl;
            const double c2 = 6.0 * mu * mu * (dgam / safeN) * pl;
            for (int i = 0; i < 6; ++i)
                for (int j = 0; j < 6; ++j) {
                    double dev;  // DEV6 with the shear block 0.5 I
                    if (i < 3 && j < 3) dev = (i == j ? 1.0 : 0.0) - third;
                    else dev = (i == j) ? 0.5 : 0.0;
                    C[i][j] -= c1 * ns[i] * ns[j];
                    C[i][j] -= c2 * dev;
                }
        }
    }
    return status;
}

}  // namespace am
