// material.cuh -- per-voxel automatic implicit-Euler material evaluation.
//
// One call evaluates one voxel entirely in registers:
//   * the reverse sweeps of LawOps (gsm.py:431-461) over forward-dual
//     payloads (tangent-over-adjoint) give f = dpsi/dA(-domega/da) and its
//     Jacobians (gsm.py:494-518);
//   * the masked Newton of _newton_implicit_euler (odeint.py:357-401) with
//     a 7x7 partially pivoted LU (linalg.py:75-143);
//   * the tangent post-process of implicit_euler_step (odeint.py:417-426:
//     "six additional linear system solves");
//   * clamp_state and the stress / consistent-tangent sweep
//     (evaluator.py:198-202, gsm.py:520-551);
//   * the m == 0 and dt == 0 paths of _evaluate_chunk (evaluator.py:134-170).
// The same code compiles for the host (g++) so the test-suite can check the
// device logic on a CPU build before any GPU time is spent.
#pragma once

#include "ad.cuh"
#include "laws.cuh"

namespace am {

template <int N>
using seq = std::make_integer_sequence<int, N>;

enum : int { ST_NEWTON = 1, ST_SINGULAR = 2, ST_NONFINITE = 4 };

struct NewtonCfg {
    int mode;      // 0 internal (RMS of the applied step), 1 stress
    int max_it;    // odeint.py:371
    double tol;    // implicit_euler_step newton_tol (odeint.py:404)
};

// ---------------------------------------------------------------- tuple helpers
template <int N, int... I>
AM_HD auto plain_tup(const double* x, std::integer_sequence<int, I...>) {
    return tup(plain(x[I])...);
}
template <int Off, int... I>
AM_HD auto seed_tup(const double* x, double s, std::integer_sequence<int, I...>) {
    return tup(seed<Off + I>(x[I], s)...);
}
template <class T, int... I>
AM_HD auto csts_of(const T& t, std::integer_sequence<int, I...>) {
    return tup(cst(get<I>(t))...);
}
template <class T, int... I>
AM_HD auto leaves_of(const T& t, std::integer_sequence<int, I...>) {
    return tup(leaf<I>(get<I>(t))...);
}
template <class Root, class T, int... I>
AM_HD auto grads_of(const Root& r, const T& t, std::integer_sequence<int, I...>) {
    return tup(gradient<I>(r, get<I>(t))...);
}
template <class T, int... I>
AM_HD auto negs_of(const T& t, std::integer_sequence<int, I...>) {
    return tup((-get<I>(t))...);
}

// ---------------------------------------------------------------- LawOps sweeps
// stress_generic (gsm.py:431-439): eps leaves, a constants
template <class Law, class PE, class PA>
AM_HD auto stress_sweep(const Law& L, const PE& pe, const PA& pa) {
    auto w = L.omega(leaves_of(pe, seq<6>{}), csts_of(pa, seq<Law::m>{}));
    return grads_of(w, pe, seq<6>{});
}
// gen_stress_generic (gsm.py:441-449): eps constants, a leaves, A = -adj
template <class Law, class PE, class PA>
AM_HD auto gen_stress_sweep(const Law& L, const PE& pe, const PA& pa) {
    auto w = L.omega(csts_of(pe, seq<6>{}), leaves_of(pa, seq<Law::m>{}));
    return negs_of(grads_of(w, pa, seq<Law::m>{}), seq<Law::m>{});
}
// flow_generic (gsm.py:451-458)
template <class Law, class PA>
AM_HD auto flow_sweep(const Law& L, const PA& A) {
    return grads_of(L.psi(leaves_of(A, seq<Law::m>{})), A, seq<Law::m>{});
}
// rhs_generic (gsm.py:460-461)
template <class Law, class PE, class PA>
AM_HD auto rhs_sweep(const Law& L, const PE& pe, const PA& pa) {
    return flow_sweep(L, gen_stress_sweep(L, pe, pa));
}

// f and df/da (a seeded with directions 0..m-1, eps plain): the part of
// rhs_and_jacobians (gsm.py:494-518) the Newton iteration consumes.
template <class Law>
AM_HD void rhs_jac_a(const Law& L, const double* e, const double* a, double* f, double (*J)[Law::m]) {
    auto fv = rhs_sweep(L, plain_tup<6>(e, seq<6>{}), seed_tup<0>(a, 1.0, seq<Law::m>{}));
    sfor<Law::m>([&](auto I) {
        constexpr int i = decltype(I)::value;
        f[i] = get<i>(fv).v;
        sfor<Law::m>([&](auto K) { J[i][decltype(K)::value] = get<i>(fv).template dir<decltype(K)::value>(); });
    });
}
// df/deps_{n+1} with eps seeded r*I and zero state tangents: rhs_dual
// (odeint.py:298-304) as used by the tangent post-process.
template <class Law>
AM_HD void rhs_jac_eps(const Law& L, const double* e, double r, const double* a, double (*dfp)[6]) {
    auto fv = rhs_sweep(L, seed_tup<0>(e, r, seq<6>{}), plain_tup<Law::m>(a, seq<Law::m>{}));
    sfor<Law::m>([&](auto I) {
        constexpr int i = decltype(I)::value;
        sfor<6>([&](auto K) { dfp[i][decltype(K)::value] = get<i>(fv).template dir<decltype(K)::value>(); });
    });
}
// stress_of (odeint.py:339-341): plain payloads
template <class Law>
AM_HD void stress_plain(const Law& L, const double* e, const double* a, double* sig) {
    auto s = stress_sweep(L, plain_tup<6>(e, seq<6>{}), plain_tup<Law::m>(a, seq<Law::m>{}));
    sfor<6>([&](auto I) { sig[decltype(I)::value] = get<decltype(I)::value>(s).v; });
}

// state payload with tangent da[k][0..5] (gsm.py:532)
template <int... I>
AM_HD auto da_tup(const double* a, const double (*da)[6], std::integer_sequence<int, I...>) {
    auto mk = [&](int k) {
        D<0x3Fu> p; p.v = a[k];
        for (int j = 0; j < 6; ++j) p.d[j] = da[k][j];
        return p;
    };
    return tup(mk(I)...);
}

// stress_and_tangent (gsm.py:520-551): sigma and C[i][j] = dsigma_i/deps_j
template <class Law>
AM_HD void stress_tangent(const Law& L, const double* e, const double* a, const double (*da)[6], double* sig,
                          double (*C)[6]) {
    auto pe = seed_tup<0>(e, 1.0, seq<6>{});
    auto run = [&](const auto& pa) {
        auto s = stress_sweep(L, pe, pa);
        sfor<6>([&](auto I) {
            constexpr int i = decltype(I)::value;
            sig[i] = get<i>(s).v;
            sfor<6>([&](auto K) { C[i][decltype(K)::value] = get<i>(s).template dir<decltype(K)::value>(); });
        });
    };
    if constexpr (Law::m == 0) run(Tup<>{});
    else if (da) run(da_tup(a, da, seq<Law::m>{}));
    else run(plain_tup<Law::m>(a, seq<Law::m>{}));  // elastic_tangent: frozen state
}

// ---------------------------------------------------------------- LU
// lu_factor (linalg.py:75-109): partial pivoting with numpy.argmax
// semantics (first maximum, first NaN wins); row swaps are done with
// predicated selects so every index stays compile-time and the matrix
// stays in registers.  Returns the reference's ok flag:
// all |pivot| >= 1e-14 * max|A|.
template <int N>
AM_HD bool lu_factor(double (&A)[N][N], int (&piv)[N]) {
    double scale = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double v = fabs(A[i][j]);
            scale = (v > scale || v != v) ? v : scale;
        }
    bool ok = scale > 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        int p = k;
        double best = fabs(A[k][k]);
        bool stop = best != best;
#pragma unroll
        for (int i = k + 1; i < N; ++i) {
            const double v = fabs(A[i][k]);
            const bool take = !stop && (v != v || v > best);
            stop = stop || (v != v);
            best = take ? v : best;
            p = take ? i : p;
        }
        piv[k] = p;
#pragma unroll
        for (int i = k + 1; i < N; ++i) {
            const bool s = (p == i);
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const double t = A[k][j];
                A[k][j] = s ? A[i][j] : t;
                A[i][j] = s ? t : A[i][j];
            }
        }
        const double pivot = A[k][k];
        ok = ok && (fabs(pivot) >= 1e-14 * scale);
        if (k < N - 1) {
            const double safe = pivot == 0.0 ? 1.0 : pivot;
#pragma unroll
            for (int i = k + 1; i < N; ++i) A[i][k] /= safe;
#pragma unroll
            for (int i = k + 1; i < N; ++i)
#pragma unroll
                for (int j = k + 1; j < N; ++j) A[i][j] -= A[i][k] * A[k][j];
        }
    }
    return ok;
}

// numpy's einsum contraction order for the substitutions (linalg.py:133,
// 137): two interleaved partial sums (even / odd terms) added at the end.
template <int Len>
AM_HD double dot2(const double* l, const double* x) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int j = 0; j < Len; ++j) {
        if (j & 1) s1 += l[j] * x[j];
        else s0 += l[j] * x[j];
    }
    return s0 + s1;
}

// lu_solve_factored (linalg.py:112-143) for one right-hand side
template <int N>
AM_HD void lu_solve(const double (&A)[N][N], const int (&piv)[N], double (&x)[N]) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
#pragma unroll
        for (int i = k + 1; i < N; ++i) {
            const bool s = (piv[k] == i);
            const double t = x[k];
            x[k] = s ? x[i] : t;
            x[i] = s ? t : x[i];
        }
    }
    sfor<N - 1>([&](auto K) {
        constexpr int k = decltype(K)::value + 1;
        x[k] -= dot2<k>(A[k], x);
    });
    sfor<N>([&](auto K) {
        constexpr int k = N - 1 - decltype(K)::value;
        if constexpr (k < N - 1) x[k] -= dot2<N - 1 - k>(A[k] + k + 1, x + k + 1);
        x[k] /= A[k][k];
    });
}

template <int N>
AM_HD double rms(const double* x) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) s += x[i] * x[i];
    return sqrt(s / N);
}

// ---------------------------------------------------------------- Newton
// _newton_implicit_euler (odeint.py:357-401) for one voxel: solves
// a - a0 - h f(eps(t1), a) = 0 from a = a0.  Returns ok; iters counts the
// rhs_and_jac evaluations (the reference's per-voxel Newton count).
template <class Law>
AM_HD bool newton_ie(const Law& L, const NewtonCfg& cfg, const double* e1, double h, const double* a0,
                     double* a, int& iters) {
    constexpr int m = Law::m;
    double res_prev = INFINITY;
    int growth = 0;
    double sig_prev[6];
#pragma unroll
    for (int i = 0; i < m; ++i) a[i] = a0[i];
    if (cfg.mode == 1) stress_plain(L, e1, a, sig_prev);
    iters = 0;
    for (int pass = 0; pass < cfg.max_it; ++pass) {
        ++iters;
        double f[m], M[m][m], F[m], dl[m], an[m], sc[m];
        int piv[m];
        rhs_jac_a(L, e1, a, f, M);
        bool finite = true;
#pragma unroll
        for (int i = 0; i < m; ++i) {
            F[i] = a[i] - a0[i] - h * f[i];
            finite = finite && (F[i] - F[i] == 0.0);  // isfinite
        }
#pragma unroll
        for (int i = 0; i < m; ++i)
#pragma unroll
            for (int k = 0; k < m; ++k) M[i][k] = (i == k ? 1.0 : 0.0) - h * M[i][k];
        const bool fac_ok = lu_factor(M, piv);
        const bool bad = !fac_ok || !finite;
#pragma unroll
        for (int i = 0; i < m; ++i) dl[i] = bad ? 0.0 : F[i];
        lu_solve(M, piv, dl);
#pragma unroll
        for (int i = 0; i < m; ++i) {
            an[i] = a[i] - dl[i];
            sc[i] = F[i] / (1.0 + fabs(a[i]));
        }
        const double res = rms<m>(sc);
        growth = res > res_prev ? growth + 1 : 0;
        res_prev = res;
        bool conv;
        if (cfg.mode == 1) {
            double sn[6], ds[6];
            stress_plain(L, e1, an, sn);
#pragma unroll
            for (int i = 0; i < 6; ++i) ds[i] = sn[i] - sig_prev[i];
            const double dsig = rms<6>(ds), ref = rms<6>(sn);
            conv = dsig <= cfg.tol * (ref > 1e-300 ? ref : 1e-300);
#pragma unroll
            for (int i = 0; i < 6; ++i) sig_prev[i] = sn[i];
        } else {
#pragma unroll
            for (int i = 0; i < m; ++i) sc[i] = dl[i] / (1.0 + fabs(an[i]));
            conv = rms<m>(sc) <= cfg.tol;
        }
#pragma unroll
        for (int i = 0; i < m; ++i) a[i] = an[i];
        if (bad || growth >= 5) return false;
        if (conv) return true;
    }
    return false;  // iteration cap (odeint.py:400)
}

// ---------------------------------------------------------------- one voxel
// _evaluate_chunk (evaluator.py:124-203) for the automatic strategy and the
// implicit-Euler integrator.  C (if non-null) receives C[i][j].
template <class Law>
AM_HD int eval_voxel(const Law& L, const NewtonCfg& cfg, const double* eps_n, const double* a_n,
                     const double* eps_np1, double dt, double* sig, double* a_out, double (*C)[6], int& iters) {
    constexpr int m = Law::m;
    iters = 0;
    if constexpr (m == 0) {
        if (C) stress_tangent(L, eps_np1, a_n, nullptr, sig, C);
        else stress_plain(L, eps_np1, a_n, sig);
        return 0;
    } else {
        if (dt == 0.0) {  // frozen (evaluator.py:142-170): a = a_n, no clamp
#pragma unroll
            for (int i = 0; i < m; ++i) a_out[i] = a_n[i];
            stress_plain(L, eps_np1, a_n, sig);
            if (C) {
                double s2[6];
                stress_tangent(L, eps_np1, a_n, nullptr, s2, C);
            }
            return 0;
        }
        int status = 0;
        // MaterialStepProblem (odeint.py:241-264): t1 = 0 + h, ramp r = min(t1/dt, 1)
        const double h = dt, t1 = 0.0 + h;
        double r = t1 / dt;
        r = (r > 1.0) ? 1.0 : r;
        double e1[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) e1[i] = eps_n[i] + r * (eps_np1[i] - eps_n[i]);
        double a[m];
        if (!newton_ie(L, cfg, e1, h, a_n, a, iters)) status |= ST_NEWTON;
        double da[m][6];
        if (C) {
            // tangent post-process (odeint.py:417-426) at the integrated,
            // not yet clamped, state: (I - h J) da = 0 + h df/deps
            double J[m][m], f[m];
            int piv[m];
            rhs_jac_eps(L, e1, r, a, da);
            rhs_jac_a(L, e1, a, f, J);
#pragma unroll
            for (int i = 0; i < m; ++i)
#pragma unroll
                for (int k = 0; k < m; ++k) J[i][k] = (i == k ? 1.0 : 0.0) - h * J[i][k];
            if (!lu_factor(J, piv)) status |= ST_SINGULAR;
#pragma unroll
            for (int j = 0; j < 6; ++j) {
                double x[m];
#pragma unroll
                for (int i = 0; i < m; ++i) x[i] = 0.0 + h * da[i][j];
                lu_solve(J, piv, x);
#pragma unroll
                for (int i = 0; i < m; ++i) da[i][j] = x[i];
            }
        }
        a[6] = a[6] < 0.0 ? 0.0 : a[6];  // clamp_state (gsm.py:252-256, evaluator.py:198)
#pragma unroll
        for (int i = 0; i < m; ++i) a_out[i] = a[i];
        if (C) stress_tangent(L, eps_np1, a, da, sig, C);
        else stress_plain(L, eps_np1, a, sig);
        return status;
    }
}

}  // namespace am
