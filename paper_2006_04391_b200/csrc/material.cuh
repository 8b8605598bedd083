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
#include "semi.cuh"

#include "newton_cfg.cuh"

namespace am {

template <int N>
using seq = std::make_integer_sequence<int, N>;

enum : int { ST_NEWTON = 1, ST_SINGULAR = 2, ST_NONFINITE = 4 };


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
// (semi-automatic: the hand partials of semi.cuh, gsm.py:431-458)
template <class Law, class PE, class PA>
AM_HD auto stress_sweep(const Law& L, const PE& pe, const PA& pa) {
    if constexpr (is_semi_v<Law>) {
        return L.hand_stress(pe, pa);
    } else {
        auto w = L.omega(leaves_of(pe, seq<6>{}), csts_of(pa, seq<Law::m>{}));
        return grads_of(w, pe, seq<6>{});
    }
}
// gen_stress_generic (gsm.py:441-449): eps constants, a leaves, A = -adj
template <class Law, class PE, class PA>
AM_HD auto gen_stress_sweep(const Law& L, const PE& pe, const PA& pa) {
    if constexpr (is_semi_v<Law>) {
        return L.hand_gen_stress(pe, pa);
    } else {
        auto w = L.omega(csts_of(pe, seq<6>{}), leaves_of(pa, seq<Law::m>{}));
        return negs_of(grads_of(w, pa, seq<Law::m>{}), seq<Law::m>{});
    }
}
// flow_generic (gsm.py:451-458)
template <class Law, class PA>
AM_HD auto flow_sweep(const Law& L, const PA& A) {
    if constexpr (is_semi_v<Law>) return L.hand_flow(A);
    else return grads_of(L.psi(leaves_of(A, seq<Law::m>{})), A, seq<Law::m>{});
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
    if constexpr (is_semi_v<Law>) {  // rhs_jac_generic (gsm.py:463-481)
        double J6[Law::m][6];
        L.rhs_jac(e, a, f, J6, nullptr);
        for (int i = 0; i < Law::m; ++i) {
            for (int k = 0; k < 6; ++k) J[i][k] = J6[i][k];
            J[i][6] = 0.0;
        }
        return;
    }
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
// semi-automatic: sigma by hand, C = d2w_ee + d2w_ae^T da (gsm.py:531-536)
template <class Law>
AM_HD void semi_stress_tangent_cols(const Law& L, const double* e, const double* a, const double* dacol,
                                    int dstride, int j, double* sig, double* c) {
    stress_plain(L, e, a, sig);
    double Ce[6][6];
    L.Ce(Ce);
    for (int i = 0; i < 6; ++i) {
        double s = 0.0;
        if (dacol) {  // einsum("ki,kj->ij", d2w_ae, da): d2w_ae = [-Ce; 0]
            for (int k = 0; k < 6; ++k) s += (-Ce[k][i]) * dacol[k * dstride];
            if (Law::m > 6) s += 0.0 * dacol[6 * dstride];
        }
        c[i] = dacol ? Ce[i][j] + s : Ce[i][j];
    }
}

template <class Law>
AM_HD void stress_tangent(const Law& L, const double* e, const double* a, const double (*da)[6], double* sig,
                          double (*C)[6]) {
    if constexpr (is_semi_v<Law>) {
        for (int j = 0; j < 6; ++j) {
            double c[6];
            semi_stress_tangent_cols(L, e, a, (Law::m && da) ? &da[0][j] : nullptr, 6, j, sig, c);
            for (int i = 0; i < 6; ++i) C[i][j] = c[i];
        }
        return;
    }
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

// mean square (the square of rms without the sqrt and the division; used
// for comparisons, which sqrt preserves)
template <int N>
AM_HD double msq(const double* x) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) s += x[i] * x[i];
    return s * (1.0 / N);
}

// reciprocal for finite nonzero y: hardware approximation + two
// Newton-Raphson steps (within an ulp of 1/y; the IEEE division costs an
// extra multiply-correct sequence and a slow-path branch).  Non-finite or
// zero y give NaN / inf; callers only use it where those cases are already
// flagged by other tests.
AM_HD double frcp(double y) {
#ifdef __CUDA_ARCH__
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
    double e = fma(-y, r, 1.0);
    r = fma(r, e, r);
    e = fma(-y, r, 1.0);
    return fma(r, e, r);
#else
    return 1.0 / y;
#endif
}


// The exact-LU fallback is rarely executed but inlined: an out-of-line call
// makes the caller save its live registers around the call site, and that
// spill traffic costs more (2-6%, r23) than the larger SASS.
#ifndef AM_INLINE_COLD
#define AM_INLINE_COLD 1
#endif
#if defined(__CUDACC__) && AM_INLINE_COLD
#define AM_COLD __host__ __device__ __forceinline__
#elif defined(__CUDACC__)
#define AM_COLD __host__ __device__ __noinline__
#else
#define AM_COLD __attribute__((noinline))
#endif

// ---------------------------------------------------------------- Jacobian shape
// The AD proves at compile time which columns of df/da are structurally
// zero: the tangent mask of every f_i lacks them.  For the Michel-Suquet
// law omega is linear in alpha, so A does not depend on a_6 and column 6
// vanishes ("zero last column"); M = I - h J is then block
// lower triangular [[D, 0], [R, I]] with a dense nd x nd block D.
template <class FT, int... I>
constexpr uint32_t tup_mask(std::integer_sequence<int, I...>) {
    return (0u | ... | std::decay_t<decltype(get<I>(std::declval<FT&>()))>::mask);
}
template <class Law>
struct JacShape {
    static constexpr int m = Law::m;
    using FT = decltype(rhs_sweep(std::declval<const Law&>(), plain_tup<6>((const double*)nullptr, seq<6>{}),
                                  seed_tup<0>((const double*)nullptr, 1.0, seq<m>{})));
    static constexpr uint32_t mask = tup_mask<FT>(seq<m>{});
    // dense block = leading columns when the nonzero columns are a prefix;
    // the semi-automatic Jacobian has an explicitly empty last column
    // (d2w_aa's last row and column vanish, gsm.py:221-225)
    static constexpr int nd = is_semi_v<Law> ? m - 1 : (mask == ((1u << popc(mask)) - 1u)) ? popc(mask) : m;
    static constexpr int nr = m - nd;
};

// f and the nd leading (structurally nonzero) columns of df/da
template <class Law, int nd>
AM_HD void rhs_jac_dense(const Law& L, const double* e, const double* a, double* f, double (*J)[nd]) {
    if constexpr (is_semi_v<Law>) {
        static_assert(nd == 6, "semi-automatic Jacobian has 6 dense columns");
        L.rhs_jac(e, a, f, J, nullptr);
        return;
    }
    auto fv = rhs_sweep(L, plain_tup<6>(e, seq<6>{}), seed_tup<0>(a, 1.0, seq<Law::m>{}));
    sfor<Law::m>([&](auto I) {
        constexpr int i = decltype(I)::value;
        f[i] = get<i>(fv).v;
        sfor<nd>([&](auto K) { J[i][decltype(K)::value] = get<i>(fv).template dir<decltype(K)::value>(); });
    });
}

// ---------------------------------------------------------------- structured LU
// Unpivoted factorisation of M = [[D, 0], [R, I]] (fast path).  It is used
// only when it is as good as the reference's partially pivoted LU
// (linalg.py:75-109): the multipliers must stay small (sum of |l| <= 1e3,
// so there is no element growth that pivoting would have avoided) and every
// pivot must be at least 1e-9 of the diagonal scale of M (far from the
// reference's 1e-14 singularity threshold); otherwise the caller falls
// back to the exact reference LU (cold path).  Mathematically the same
// solve; results differ from the pivoted one by round-off only.
template <int m, int nd>
struct SFact {
    static constexpr int nr = m - nd;
    double D[nd][nd];
    double R[nr > 0 ? nr : 1][nd];
    double inv[nd];

    // M = I - h J from the dense columns
    AM_HD void build(const double (*J)[nd], double h) {
#pragma unroll
        for (int i = 0; i < nd; ++i)
#pragma unroll
            for (int k = 0; k < nd; ++k) D[i][k] = (i == k ? 1.0 : 0.0) - h * J[i][k];
#pragma unroll
        for (int r = 0; r < nr; ++r)
#pragma unroll
            for (int k = 0; k < nd; ++k) R[r][k] = 0.0 - h * J[nd + r][k];
    }

    AM_HD bool factor() {
        // guard terms are sums of absolute values (DADD with |.| operand
        // modifiers, no compare/select chains): lsum bounds every multiplier,
        // dsum is the diagonal scale of M
        double dsum = double(nr), lsum = 0.0;
#pragma unroll
        for (int k = 0; k < nd; ++k) dsum += fabs(D[k][k]);
        bool ok = true;
#pragma unroll
        for (int k = 0; k < nd; ++k) {
            const double p = D[k][k];
            ok = ok && (fabs(p) >= 1e-9 * dsum);
            const double iv = frcp(p);
            inv[k] = iv;
#pragma unroll
            for (int i = k + 1; i < nd; ++i) {
                const double l = D[i][k] * iv;
                lsum += fabs(l);
                D[i][k] = l;
#pragma unroll
                for (int j = k + 1; j < nd; ++j) D[i][j] = fma(-l, D[k][j], D[i][j]);
            }
#pragma unroll
            for (int r = 0; r < nr; ++r) {
                const double l = R[r][k] * iv;
                lsum += fabs(l);
                R[r][k] = l;
#pragma unroll
                for (int j = k + 1; j < nd; ++j) R[r][j] = fma(-l, D[k][j], R[r][j]);
            }
        }
        // NaN anywhere makes a comparison false; inf makes dsum or lsum inf
        return ok && lsum <= 1e3 && dsum < INFINITY;
    }

    AM_HD void solve(double* x) const {
#pragma unroll
        for (int i = 1; i < nd; ++i)
#pragma unroll
            for (int k = 0; k < i; ++k) x[i] = fma(-D[i][k], x[k], x[i]);
#pragma unroll
        for (int r = 0; r < nr; ++r)
#pragma unroll
            for (int k = 0; k < nd; ++k) x[nd + r] = fma(-R[r][k], x[k], x[nd + r]);
#pragma unroll
        for (int i = nd - 1; i >= 0; --i) {
#pragma unroll
            for (int j = i + 1; j < nd; ++j) x[i] = fma(-D[i][j], x[j], x[i]);
            x[i] *= inv[i];
        }
    }
};

// ---------------------------------------------------------------- exact (cold) path
// The reference's dense partially pivoted LU (linalg.py:75-143) on
// M = I - h df/da at state a, solving M x = rhs in place.  Returns the
// reference's ok flag (all |pivot| >= 1e-14 max|M|).  Used when the fast
// path's pivot guard trips (ill-conditioned or non-finite iteration
// matrix) so that such voxels see exactly the reference's arithmetic;
// `zero_rhs_if_bad` reproduces odeint.py:381-382 (solve with a zero
// right-hand side when the factorisation or F is bad).
template <class Law>
AM_COLD bool exact_solve(const Law& L, const double* e1, const double* a, double h, double* xp, bool zero_rhs_if_bad,
                         bool rhs_finite) {
    constexpr int m = Law::m;
    double f[m], M[m][m], x[m];
    int piv[m];
    for (int i = 0; i < m; ++i) x[i] = xp[i];
    rhs_jac_a(L, e1, a, f, M);
    for (int i = 0; i < m; ++i)
        for (int k = 0; k < m; ++k) M[i][k] = (i == k ? 1.0 : 0.0) - h * M[i][k];
    const bool ok = lu_factor(M, piv);
    if (zero_rhs_if_bad && (!ok || !rhs_finite))
        for (int i = 0; i < m; ++i) x[i] = 0.0;
    lu_solve(M, piv, x);
    for (int i = 0; i < m; ++i) xp[i] = x[i];
    return ok;
}

// ---------------------------------------------------------------- tangent sinks
// Receivers of the consistent tangent C[i][j] = dsigma_i/deps_j, one
// column j (compile-time after inlining) at a time.
struct NoSink {
    AM_HD void col(int, const double*) {}
};
template <class Sink>
AM_HD void put_all(Sink& sink, const double (*C)[6]) {
    sfor<6>([&](auto J) {
        constexpr int j = decltype(J)::value;
        double c[6];
        for (int i = 0; i < 6; ++i) c[i] = C[i][j];
        sink.col(j, c);
    });
}

// strain payloads: eps_i seeded with direction i - J0 (value s) for
// J0 <= i < J0 + NJ, plain otherwise
template <int J0, int NJ, int I>
AM_HD auto seed_or_plain(double v, double s) {
    if constexpr (I >= J0 && I < J0 + NJ) return seed<I - J0>(v, s);
    else return plain(v);
}
template <int J0, int NJ, int... I>
AM_HD auto eps_seed_block(const double* e, double s, std::integer_sequence<int, I...>) {
    return tup(seed_or_plain<J0, NJ, I>(e[I], s)...);
}
// state payloads (a_k, da[k][0..NJ-1]) (gsm.py:532)
template <int NJ, int... I>
AM_HD auto da_block_tup(const double* a, const double (*da)[NJ], std::integer_sequence<int, I...>) {
    auto mk = [&](int k) {
        D<(1u << NJ) - 1u> p;
        p.v = a[k];
        for (int j = 0; j < NJ; ++j) p.d[j] = da[k][j];
        return p;
    };
    return tup(mk(I)...);
}

// stress_and_tangent columns J0 .. J0+NJ-1 at (eps_{n+1}, clamped a) seeded
// (e_j, da[:, j]) (gsm.py:520-551; semi-automatic: C = d2w_ee + d2w_ae^T da)
template <int J0, int NJ, class Law, class Sink>
AM_HD void tangent_stress_block(const Law& L, const double* ac, const double* eps_np1, const double (*da)[NJ],
                                double* sig, Sink& sink) {
    constexpr int m = Law::m;
    if constexpr (is_semi_v<Law>) {
        sfor<NJ>([&](auto Jc) {
            constexpr int jj = decltype(Jc)::value;
            double c[6];
            semi_stress_tangent_cols(L, eps_np1, ac, &da[0][jj], NJ, J0 + jj, sig, c);
            sink.col(J0 + jj, c);
        });
        return;
    }
    auto s = stress_sweep(L, eps_seed_block<J0, NJ>(eps_np1, 1.0, seq<6>{}), da_block_tup<NJ>(ac, da, seq<m>{}));
    sfor<NJ>([&](auto Jc) {
        constexpr int jj = decltype(Jc)::value;
        double c[6];
        sfor<6>([&](auto I) {
            constexpr int i = decltype(I)::value;
            c[i] = get<i>(s).template dir<jj>();
            sig[i] = get<i>(s).v;
        });
        sink.col(J0 + jj, c);
    });
}

// Columns J0 .. J0+NJ-1 of the consistent tangent (odeint.py:417-426 then
// gsm.py:520-551): df/deps_{n+1} for these strain directions (rhs_dual,
// eps seeded r * e_j), (I - h J) da = 0 + h df/deps per column with the
// factorisation of the converged iteration matrix, then the stress sweep at
// (eps_{n+1}, clamped a) seeded (e_j, da[:, j]).  Each direction of a
// forward dual is computed independently, so blocks of directions give the
// same numbers as the reference's W = 6 sweeps; blocks keep the register
// footprint of the tangent phase small.
template <int J0, int NJ, class Law, class Fact, class Sink>
AM_HD void tangent_block(const Law& L, const double* e1, double r, double h, const double* a, const double* ac,
                         const double* eps_np1, const Fact& fac, bool fast, double* sig, Sink& sink) {
    constexpr int m = Law::m;
    auto fv = rhs_sweep(L, eps_seed_block<J0, NJ>(e1, r, seq<6>{}), plain_tup<m>(a, seq<m>{}));
    double da[m][NJ];
    sfor<NJ>([&](auto Jc) {
        constexpr int jj = decltype(Jc)::value;
        double x[m];
        sfor<m>([&](auto I) { x[decltype(I)::value] = 0.0 + h * get<decltype(I)::value>(fv).template dir<jj>(); });
        if (fast) fac.solve(x);
        else exact_solve(L, e1, a, h, x, false, true);
#pragma unroll
        for (int i = 0; i < m; ++i) da[i][jj] = x[i];
    });
    tangent_stress_block<J0, NJ>(L, ac, eps_np1, da, sig, sink);
}

// ---------------------------------------------------------------- one point
// _evaluate_chunk (evaluator.py:124-203) for strategy="automatic" and the
// implicit-Euler integrator is split in two phases so that the hot Newton
// loop and the once-per-point tangent post-process can run as separate
// kernels with different register budgets:
//   newton_point:  MaterialStepProblem + _newton_implicit_euler
//                  (odeint.py:241-264, 357-401) -> unclamped state a
//   stress_point:  clamp_state (evaluator.py:198) + stress (evaluator.py:202)
//   tangent_point: tangent post-process (odeint.py:417-426) at the unclamped
//                  a, clamp, stress_and_tangent (gsm.py:520-551)
// Both phases are pure functions of the point's inputs, so the split does
// not change any result.

// MaterialStepProblem (odeint.py:241-264): t1 = 0 + h, ramp r = min(t1/dt, 1),
// eps(t1) = eps_n + r (eps_{n+1} - eps_n)
AM_HD double step_strain(const double* eps_n, const double* eps_np1, double dt, double* e1) {
    const double h = dt, t1 = 0.0 + h;
    double r = t1 / dt;
    r = (r > 1.0) ? 1.0 : r;
#pragma unroll
    for (int i = 0; i < 6; ++i) e1[i] = eps_n[i] + r * (eps_np1[i] - eps_n[i]);
    return r;
}

// Newton of one point; returns status bits (ST_NEWTON on failure), writes the
// unclamped state to a and the per-point Newton count (the number of
// rhs_and_jac evaluations the reference makes for this point) to iters.
// Mode: 0 internal / 1 stress convergence (odeint.py:388-395).
// dt == 0 (frozen, evaluator.py:142-170): a = a_n, no iteration.
template <class Law, int Mode>
struct NewtonState {
    static constexpr int m = Law::m;
    static constexpr int ms = m > 0 ? m : 1;
    double a0[ms], a[ms], e1[6], h, res_prev;
    double sig_prev[Mode == 1 ? 6 : 1];
    int growth, iters;

    // MaterialStepProblem set-up; false when no iteration is needed
    // (no state, or frozen dt == 0: a = a_n)
    // a_start: optional first iterate (default a_n, odeint.py:371)
    AM_HD bool init(const Law& L, const double* eps_n, const double* a_n, const double* eps_np1, double dt,
                    const double* a_start = nullptr) {
        iters = 0;
#pragma unroll
        for (int i = 0; i < m; ++i) a0[i] = a[i] = a_n[i];
        if (a_start && m > 0 && dt != 0.0) {
#pragma unroll
            for (int i = 0; i < m; ++i) a[i] = a_start[i];
        }
        if (m == 0 || dt == 0.0) return false;
        h = dt;
        step_strain(eps_n, eps_np1, dt, e1);
        res_prev = INFINITY;
        growth = 0;
        if constexpr (Mode == 1) stress_plain(L, e1, a, sig_prev);
        return true;
    }

    // one iteration of _newton_implicit_euler (odeint.py:371-399):
    // 0 = continue, 1 = converged, 2 = failed (odeint.py:397, 400)
    AM_HD int step(const Law& L, const NewtonCfg& cfg) {
        if constexpr (m == 0) {
            return 1;
        } else {
            constexpr int nd = JacShape<Law>::nd;
            double f[m], J[m][nd], F[m], dl[m];
            rhs_jac_dense<Law, nd>(L, e1, a, f, J);
            SFact<m, nd> fac;
            fac.build(J, h);
            const bool fast = fac.factor();
            ++iters;
            bool finite = true;
#pragma unroll
            for (int i = 0; i < m; ++i) {
                F[i] = a[i] - a0[i] - h * f[i];
                finite = finite && (F[i] - F[i] == 0.0);  // isfinite
                dl[i] = F[i];
            }
            bool bad;
            if (fast) {
                bad = !finite;
                if (bad) {
#pragma unroll
                    for (int i = 0; i < m; ++i) dl[i] = 0.0;
                }
                fac.solve(dl);
            } else {
                bad = !exact_solve(L, e1, a, h, dl, true, finite) || !finite;
            }
            double an[m], sc[m];
#pragma unroll
            for (int i = 0; i < m; ++i) {
                an[i] = a[i] - dl[i];
                sc[i] = F[i] * frcp(1.0 + fabs(a[i]));
            }
            // residual RMS (odeint.py:384); compared in squares (sqrt is monotone)
            const double res = msq<m>(sc);
            growth = res > res_prev ? growth + 1 : 0;
            res_prev = res;
            bool conv;
            if constexpr (Mode == 1) {
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
                for (int i = 0; i < m; ++i) sc[i] = dl[i] * frcp(1.0 + fabs(an[i]));
                conv = msq<m>(sc) <= cfg.tol * cfg.tol;  // rms <= tol (odeint.py:395)
            }
#pragma unroll
            for (int i = 0; i < m; ++i) a[i] = an[i];
            if (bad || growth >= 5) return 2;
            if (conv) return 1;
            if (iters >= cfg.max_it) return 2;
            return 0;
        }
    }
};

template <class Law, int Mode>
AM_HD int newton_point(const Law& L, const NewtonCfg& cfg, const double* eps_n, const double* a_n,
                       const double* eps_np1, double dt, double* a, int& iters, const double* a_start = nullptr) {
    NewtonState<Law, Mode> S;
    int r = 1;
    if (S.init(L, eps_n, a_n, eps_np1, dt, a_start))
        while ((r = S.step(L, cfg)) == 0) {
        }
#pragma unroll
    for (int i = 0; i < Law::m; ++i) a[i] = S.a[i];
    iters = S.iters;
    return r == 2 ? ST_NEWTON : 0;
}

// clamp_state (gsm.py:252-256): alpha >= 0; identity for laws without state
template <class Law>
AM_HD void clamp_state(const double* a, double* ac) {
    constexpr int m = Law::m;
#pragma unroll
    for (int i = 0; i < m; ++i) ac[i] = a[i];
    if constexpr (m > 0) ac[m - 1] = ac[m - 1] < 0.0 ? 0.0 : ac[m - 1];
}

// sigma at eps_{n+1} and the clamped state (evaluator.py:198-202); writes
// the clamped state to ac
template <class Law>
AM_HD void stress_point(const Law& L, const double* eps_np1, const double* a, double* ac, double* sig) {
    clamp_state<Law>(a, ac);
    stress_plain(L, eps_np1, ac, sig);
}

// Tangent phase for a point whose Newton converged to the unclamped state a:
// the post-process of implicit_euler_step (odeint.py:417-426: M = I - h J at
// a, "six additional linear system solves") and stress_and_tangent at the
// clamped state (gsm.py:520-551).  Frozen points (dt == 0) get the elastic
// tangent at a_n (evaluator.py:145-148), laws without state the stiffness
// (evaluator.py:134-138).  Writes the clamped state to ac, sigma, and C to
// the sink.  Returns ST_SINGULAR when the reference's check_singular LU
// would raise (odeint.py:424).
template <class Law, class Sink>
AM_HD int tangent_point(const Law& L, const double* eps_n, const double* eps_np1, double dt, const double* a,
                        double* ac, double* sig, Sink& sink) {
    constexpr int m = Law::m;
    clamp_state<Law>(a, ac);
    if constexpr (m == 0) {
        double C[6][6];
        stress_tangent(L, eps_np1, a, nullptr, sig, C);
        put_all(sink, C);
        return 0;
    } else {
        if (dt == 0.0) {
            double C[6][6], s2[6];
            stress_plain(L, eps_np1, a, sig);
            stress_tangent(L, eps_np1, a, nullptr, s2, C);
            put_all(sink, C);
            return 0;
        }
        constexpr int nd = JacShape<Law>::nd;
        const double h = dt;
        double e1[6];
        const double r = step_strain(eps_n, eps_np1, dt, e1);
        int status = 0;
#ifndef AM_TAN_BLOCK
#define AM_TAN_BLOCK 3
#endif
#ifndef AM_TAN_COMBINED
#define AM_TAN_COMBINED 1
#endif
        if constexpr (AM_TAN_COMBINED && !is_semi_v<Law>) {
            // one sweep for the whole post-process: the state seeded with
            // directions 0..m-1 (df/da, odeint.py:421) and eps_{n+1} with
            // directions m..m+5 scaled by the ramp (rhs_dual, odeint.py:420)
            static_assert(m + 6 <= kMaxDir, "too many directions");
            auto fv = rhs_sweep(L, seed_tup<m>(e1, r, seq<6>{}), seed_tup<0>(a, 1.0, seq<m>{}));
            double J[m][nd], dfp[m][6];
            sfor<m>([&](auto I) {
                constexpr int i = decltype(I)::value;
                sfor<nd>([&](auto K) { J[i][decltype(K)::value] = get<i>(fv).template dir<decltype(K)::value>(); });
                sfor<6>([&](auto K) { dfp[i][decltype(K)::value] = get<i>(fv).template dir<m + decltype(K)::value>(); });
            });
            SFact<m, nd> fac;
            fac.build(J, h);
            const bool fast = fac.factor();
            if (!fast) {
                double x[m];
                for (int i = 0; i < m; ++i) x[i] = 0.0;
                if (!exact_solve(L, e1, a, h, x, false, true)) status |= ST_SINGULAR;
            }
            sfor<6 / AM_TAN_BLOCK>([&](auto Bk) {
                constexpr int J0 = decltype(Bk)::value * AM_TAN_BLOCK;
                double da[m][AM_TAN_BLOCK];
                sfor<AM_TAN_BLOCK>([&](auto Jc) {
                    constexpr int jj = decltype(Jc)::value;
                    double x[m];
#pragma unroll
                    for (int i = 0; i < m; ++i) x[i] = 0.0 + h * dfp[i][J0 + jj];
                    if (fast) fac.solve(x);
                    else exact_solve(L, e1, a, h, x, false, true);
#pragma unroll
                    for (int i = 0; i < m; ++i) da[i][jj] = x[i];
                });
                tangent_stress_block<J0, AM_TAN_BLOCK>(L, ac, eps_np1, da, sig, sink);
            });
            return status;
        } else {
        double f[m], J[m][nd];
        rhs_jac_dense<Law, nd>(L, e1, a, f, J);
        SFact<m, nd> fac;
        fac.build(J, h);
        const bool fast = fac.factor();
        if (!fast) {
            double x[m];
            for (int i = 0; i < m; ++i) x[i] = 0.0;
            if (!exact_solve(L, e1, a, h, x, false, true)) status |= ST_SINGULAR;
        }
        // strain directions in blocks of columns (semi-automatic: 6, measured
        // 1.20e9 vs 1.18e9 evals/s with 3)
        constexpr int kBlk = is_semi_v<Law> ? 6 : AM_TAN_BLOCK;
        sfor<6 / kBlk>([&](auto Bk) {
            tangent_block<decltype(Bk)::value * kBlk, kBlk>(L, e1, r, h, a, ac, eps_np1, fac, fast, sig, sink);
        });
        return status;
        }
    }
}

// A failed point has no tangent (the reference raises NewtonDivergenceError
// before the post-process, odeint.py:415-416): NaN columns, stress at the
// returned state.
template <class Law, class Sink>
AM_HD void failed_point(const Law& L, const double* eps_np1, const double* a, double* ac, double* sig, Sink& sink) {
    stress_point(L, eps_np1, a, ac, sig);
    double c[6];
    for (int i = 0; i < 6; ++i) c[i] = NAN;
    sfor<6>([&](auto J) { sink.col(decltype(J)::value, c); });
}

}  // namespace am
