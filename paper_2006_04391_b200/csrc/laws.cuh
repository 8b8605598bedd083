// laws.cuh -- the SPEC's material laws as device-side potentials.
//
// A generalized standard material is its two potentials: the free energy
// omega(eps, a) and the force potential psi(A).  Each law below writes them
// over component lists (Tup) of generic reverse nodes, exactly as the
// reference writes them over Python lists of generic payloads
// (gsm.py:82-97); the AD in ad.cuh derives everything else.  Expression
// shapes follow Python's left-to-right operator evaluation so the tree the
// compiler sees is the tree the reference builds.
#pragma once

#include "ad.cuh"

namespace am {

// linalg.py:49-53
AM_HD void lame_parameters(double E, double nu, double& lam, double& mu) {
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    mu = E / (2.0 * (1.0 + nu));
}

// sum of squares as Python builds x0*x0 + x1*x1 + x2*x2
template <class X0, class X1, class X2>
AM_HD auto sq3(const X0& x0, const X1& x1, const X2& x2) {
    return x0 * x0 + x1 * x1 + x2 * x2;
}

// LinearElastic (gsm.py:100-153): m = 0, psi = 0
struct LinearElasticLaw {
    static constexpr int m = 0;
    double lam, mu;

    AM_HD static LinearElasticLaw make(double E, double nu) {
        LinearElasticLaw L;
        lame_parameters(E, nu, L.lam, L.mu);
        return L;
    }

    // gsm.py:112-117
    template <class E, class A>
    AM_HD auto omega(const E& e, const A&) const {
        auto tr = get<0>(e) + get<1>(e) + get<2>(e);
        auto w = cst(0.5 * lam) * tr * tr;
        auto w1 = w + cst(mu) * sq3(get<0>(e), get<1>(e), get<2>(e));
        return w1 + cst(0.5 * mu) * sq3(get<3>(e), get<4>(e), get<5>(e));
    }
};

// MichelSuquet (gsm.py:210-256): a = (eps_vp[6], alpha), m = 7
struct MichelSuquetLaw {
    static constexpr int m = 7;
    double lam, mu, H, sigma_Y, eps0_dot, sigma_d, n;

#ifdef __CUDA_ARCH__
    __device__ void launder() {
        asm volatile("" : "+d"(lam), "+d"(mu), "+d"(H), "+d"(sigma_Y), "+d"(eps0_dot), "+d"(sigma_d), "+d"(n));
    }
#endif

    AM_HD static MichelSuquetLaw make(double E, double nu, double sigma_Y, double H, double eps0_dot,
                                      double sigma_d, double n) {
        MichelSuquetLaw L;
        lame_parameters(E, nu, L.lam, L.mu);
        L.H = H; L.sigma_Y = sigma_Y; L.eps0_dot = eps0_dot; L.sigma_d = sigma_d; L.n = n;
        return L;
    }

    // gsm.py:234-244
    template <class E, class A>
    AM_HD auto omega(const E& e, const A& a) const {
        auto ee0 = get<0>(e) - get<0>(a);
        auto ee1 = get<1>(e) - get<1>(a);
        auto ee2 = get<2>(e) - get<2>(a);
        auto ee3 = get<3>(e) - get<3>(a);
        auto ee4 = get<4>(e) - get<4>(a);
        auto ee5 = get<5>(e) - get<5>(a);
        auto tr = ee0 + ee1 + ee2;
        auto w = cst(0.5 * lam) * tr * tr;
        auto w1 = w + cst(mu) * sq3(ee0, ee1, ee2);
        auto w2 = w1 + cst(0.5 * mu) * sq3(ee3, ee4, ee5);
        auto w3 = w2 + cst(H / 3.0) * sq3(get<0>(a), get<1>(a), get<2>(a));
        auto w4 = w3 + cst(H / 6.0) * sq3(get<3>(a), get<4>(a), get<5>(a));
        return w4 + cst(sigma_Y) * get<6>(a);
    }

    // gsm.py:246-250 with mises_components (gsm.py:62-79): the guarded
    // sqrt masks on the primal value of q.
    template <class A>
    AM_HD auto psi(const A& s) const {
        auto p = (get<0>(s) + get<1>(s) + get<2>(s)) * cst(1.0 / 3.0);
        auto d0 = get<0>(s) - p;
        auto d1 = get<1>(s) - p;
        auto d2 = get<2>(s) - p;
        auto q = cst(1.5) * (sq3(d0, d1, d2) + cst(2.0) * sq3(get<3>(s), get<4>(s), get<5>(s)));
        const double mask = v(q).v > 0.0 ? 1.0 : 0.0;
        auto norm = nsqrt(q + cst(1.0 - mask)) * cst(mask);
        auto y = norm + get<6>(s);
        const double K = sigma_d * eps0_dot / (n + 1.0);
        return cst(K) * npow(npos(y * cst(1.0 / sigma_d)), n + 1.0);
    }
};

}  // namespace am
