// semi.cuh -- the semi-automatic strategy: hand-coded first partials of the
// laws (gsm.py:122-153 LinearElastic.hand_*, gsm.py:258-328
// MichelSuquet.hand_*) and the nested-Jacobian assembly of
// LawOps.rhs_jac_generic (gsm.py:463-481) / stress_and_tangent
// (gsm.py:531-536).
//
// SemiLaw<Base> wraps a law: the sweeps of material.cuh dispatch on it (if
// constexpr is_semi<Law>) to these formulas instead of the reverse AD.  The
// hand formulas are generic over payload tuples, so forward duals flow
// through them exactly as Dual1 payloads flow through the reference's hand
// code (rhs_dual / stress_dual, odeint.py:298-304, 343-352).  Operation
// order follows the Python expressions.  Host + device.
#pragma once

#include "ad.cuh"
#include "laws.cuh"

namespace am {

template <class Base>
struct SemiLaw;

template <class T>
struct is_semi : std::false_type {};
template <class B>
struct is_semi<SemiLaw<B>> : std::true_type {};
template <class T>
constexpr bool is_semi_v = is_semi<T>::value;

// LinearElastic.hand_stress (gsm.py:122-133)
template <>
struct SemiLaw<LinearElasticLaw> {
    static constexpr int m = 0;
    LinearElasticLaw base;
    AM_HD static SemiLaw make(double E, double nu) { return SemiLaw{LinearElasticLaw::make(E, nu)}; }

    template <class E, class A>
    AM_HD auto hand_stress(const E& e, const A&) const {
        const auto lam = plain(base.lam), mu2 = plain(2.0 * base.mu), mu = plain(base.mu);
        auto tr = get<0>(e) + get<1>(e) + get<2>(e);
        return tup(lam * tr + mu2 * get<0>(e), lam * tr + mu2 * get<1>(e), lam * tr + mu2 * get<2>(e),
                   mu * get<3>(e), mu * get<4>(e), mu * get<5>(e));
    }
    // d2w_ee (isotropic_stiffness, linalg.py:56-63)
    AM_HD void Ce(double (*C)[6]) const {
        for (int i = 0; i < 6; ++i)
            for (int j = 0; j < 6; ++j) C[i][j] = 0.0;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) C[i][j] = base.lam;
        for (int i = 0; i < 3; ++i) C[i][i] = base.lam + 2.0 * base.mu;
        for (int i = 3; i < 6; ++i) C[i][i] = base.mu;
    }
};

template <>
struct SemiLaw<MichelSuquetLaw> {
    static constexpr int m = 7;
    MichelSuquetLaw base;
    AM_HD static SemiLaw make(double E, double nu, double sigma_Y, double H, double eps0_dot, double sigma_d,
                              double n) {
        return SemiLaw{MichelSuquetLaw::make(E, nu, sigma_Y, H, eps0_dot, sigma_d, n)};
    }

    // gsm.py:260-271
    template <class E, class A>
    AM_HD auto hand_stress(const E& e, const A& a) const {
        const auto lam = plain(base.lam), mu2 = plain(2.0 * base.mu), mu = plain(base.mu);
        auto ee0 = get<0>(e) - get<0>(a);
        auto ee1 = get<1>(e) - get<1>(a);
        auto ee2 = get<2>(e) - get<2>(a);
        auto ee3 = get<3>(e) - get<3>(a);
        auto ee4 = get<4>(e) - get<4>(a);
        auto ee5 = get<5>(e) - get<5>(a);
        auto tr = ee0 + ee1 + ee2;
        return tup(lam * tr + mu2 * ee0, lam * tr + mu2 * ee1, lam * tr + mu2 * ee2, mu * ee3, mu * ee4, mu * ee5);
    }
    // gsm.py:273-286
    template <class E, class A>
    AM_HD auto hand_gen_stress(const E& e, const A& a) const {
        auto s = hand_stress(e, a);
        const double kin = 2.0 * base.H / 3.0;
        const auto k1 = plain(kin), k2 = plain(0.5 * kin);
        return tup(get<0>(s) - k1 * get<0>(a), get<1>(s) - k1 * get<1>(a), get<2>(s) - k1 * get<2>(a),
                   get<3>(s) - k2 * get<3>(a), get<4>(s) - k2 * get<4>(a), get<5>(s) - k2 * get<5>(a),
                   plain(-base.sigma_Y) + plain(0.0) * get<6>(a));
    }

    // _flow_pieces (gsm.py:288-296) with mises_components (gsm.py:68-79)
    template <class A, class F>
    AM_HD auto flow_pieces(const A& A_, F&& use) const {
        auto p = (get<0>(A_) + get<1>(A_) + get<2>(A_)) * plain(1.0 / 3.0);
        auto d0 = get<0>(A_) - p;
        auto d1 = get<1>(A_) - p;
        auto d2 = get<2>(A_) - p;
        const auto& d3 = get<3>(A_);
        const auto& d4 = get<4>(A_);
        const auto& d5 = get<5>(A_);
        auto q = plain(1.5) * (d0 * d0 + d1 * d1 + d2 * d2 + plain(2.0) * (d3 * d3 + d4 * d4 + d5 * d5));
        const double mask = q.v > 0.0 ? 1.0 : 0.0;
        auto norm = dsqrt(q + plain(1.0 - mask)) * plain(mask);
        auto y = norm + get<6>(A_);
        const double gate = y.v > 0.0 ? 1.0 : 0.0;
        auto denom = norm + plain(1.0 - gate);
        auto x = dpos(y * plain(1.0 / base.sigma_d));
        auto gdot = plain(base.eps0_dot) * dpow(x, base.n);
        const auto g = plain(gate);
        // 1.5 * SHEAR_DUP[i] * d[i] / denom * gate
        auto P0 = plain(1.5) * d0 / denom * g;
        auto P1 = plain(1.5) * d1 / denom * g;
        auto P2 = plain(1.5) * d2 / denom * g;
        auto P3 = plain(3.0) * d3 / denom * g;
        auto P4 = plain(3.0) * d4 / denom * g;
        auto P5 = plain(3.0) * d5 / denom * g;
        return use(gdot, tup(P0, P1, P2, P3, P4, P5), x, denom, gate);
    }
    // hand_flow (gsm.py:298-300)
    template <class A>
    AM_HD auto hand_flow(const A& A_) const {
        return flow_pieces(A_, [](const auto& gdot, const auto& P, const auto&, const auto&, double) {
            return tup(gdot * get<0>(P), gdot * get<1>(P), gdot * get<2>(P), gdot * get<3>(P), gdot * get<4>(P),
                       gdot * get<5>(P), gdot);
        });
    }

    // rhs_jac_generic (gsm.py:463-481) on plain values: f, d f/d a (dense
    // leading 6 columns; column 6 is the empty sum 0), d f/d eps
    template <bool WithJe>
    AM_HD void rhs_jac_t(const double* e, const double* a, double* f, double (*J)[6], double (*Je)[6]) const {
        double psi2[7][7];
        auto Av = hand_gen_stress(tup(plain(e[0]), plain(e[1]), plain(e[2]), plain(e[3]), plain(e[4]), plain(e[5])),
                                  tup(plain(a[0]), plain(a[1]), plain(a[2]), plain(a[3]), plain(a[4]), plain(a[5]),
                                      plain(a[6])));
        flow_pieces(Av, [&](const auto&, const auto& Pt, const auto& x, const auto& denom_, double gate) {
            const double denom = denom_.v;
            const double P[6] = {get<0>(Pt).v, get<1>(Pt).v, get<2>(Pt).v, get<3>(Pt).v, get<4>(Pt).v, get<5>(Pt).v};
            // x^n (gdot) and x^(n-1) (gprime) from one power, as the
            // automatic path's powjet (ad.cuh): <= 1e-14 relative to pow()
            const double xv = x.v, c = base.n;
            double p1, pn;
            if (xv > 0.0) {
#ifdef AM_EXACT_POW
                p1 = ::pow(xv, c - 1.0);
                pn = ::pow(xv, c);
#else
                p1 = ::exp((c - 1.0) * ::log(xv));
                pn = p1 * xv;
#endif
            } else {
                p1 = ::pow(xv, c - 1.0);
                pn = ::pow(xv, c);
            }
            const double gdot = base.eps0_dot * pn;
            const double gprime = (base.eps0_dot * base.n / base.sigma_d) * p1;
            // x / denom for the 36 entries: the correctly rounded reciprocal
            // and one FMA correction of x * rd give the correctly rounded
            // quotient (Markstein), i.e. the bits of the IEEE division
            const double rd = 1.0 / denom;
            auto qdiv = [&](double num) {
                const double q = num * rd;
                return fma(fma(-q, denom, num), rd, q);
            };
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                f[i] = gdot * P[i];
                const double dup_i = i < 3 ? 1.5 : 3.0;
#pragma unroll
                for (int j = 0; j < 6; ++j) {
                    const double dev = (i == j ? 1.0 : 0.0) - ((i < 3 && j < 3) ? 1.0 / 3.0 : 0.0);
                    const double curv = qdiv(dup_i * dev - P[i] * P[j]) * gate;
                    psi2[i][j] = gprime * P[i] * P[j] + gdot * curv;
                }
                psi2[i][6] = gprime * P[i];
                psi2[6][i] = gprime * P[i];
            }
            psi2[6][6] = gprime;
            f[6] = gdot;
            return 0;
        });
        // d2w_aa = [Ce + (2/3) Hmat, 0; 0, 0], d2w_ae = [-Ce; 0] (gsm.py:221-227).
        // The reference sums psi2[i][j] * w[j][k] over the j with w[j][k] != 0
        // in increasing j: for a normal column k < 3 that is j = 0, 1, 2 (the
        // off-diagonal entries are lam, skipped when lam == 0), for a shear
        // column only j = k.  The sparsity is spelled out at compile time.
        const double lam = base.lam, mu = base.mu, H = base.H;
        const double k23 = 2.0 / 3.0;
        const bool lam_nz = lam != 0.0;
        const double aa_n = lam + 2.0 * mu + k23 * H, aa_s = mu + k23 * (H / 2.0);
        const double ae_n = -(lam + 2.0 * mu), ae_o = -lam, ae_s = -mu;
#pragma unroll
        for (int i = 0; i < 7; ++i) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                double s = 0.0, se = 0.0;
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    if (j == k) {
                        s += psi2[i][j] * aa_n;
                        se += psi2[i][j] * ae_n;
                    } else if (lam_nz) {
                        s += psi2[i][j] * lam;
                        se += psi2[i][j] * ae_o;
                    }
                }
                J[i][k] = -s;
                if (WithJe) Je[i][k] = -se;
            }
#pragma unroll
            for (int k = 3; k < 6; ++k) {
                J[i][k] = -(0.0 + psi2[i][k] * aa_s);
                if (WithJe) Je[i][k] = -(0.0 + psi2[i][k] * ae_s);
            }
        }
    }
    AM_HD void rhs_jac(const double* e, const double* a, double* f, double (*J)[6], double (*Je)[6]) const {
        if (Je) rhs_jac_t<true>(e, a, f, J, Je);
        else rhs_jac_t<false>(e, a, f, J, nullptr);
    }

    AM_HD void Ce(double (*C)[6]) const {
        for (int i = 0; i < 6; ++i)
            for (int j = 0; j < 6; ++j) C[i][j] = 0.0;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) C[i][j] = base.lam;
        for (int i = 0; i < 3; ++i) C[i][i] = base.lam + 2.0 * base.mu;
        for (int i = 3; i < 6; ++i) C[i][i] = base.mu;
    }
};

}  // namespace am
