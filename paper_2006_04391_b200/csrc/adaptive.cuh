// adaptive.cuh -- adaptive explicit embedded integration of one material
// point (gsmkit odeint.py: ode12 / ode23 SchemeSpec 92-113, _explicit_step
// 429-475, error_norm 564-617, adaptive_integrate 636-756, StepController
// 198-214), automatic strategy, with optional coupled sensitivity transport
// (Theorem 2 / Corollary 1 of the paper: the sensitivity da/deps_{n+1} is
// advanced by the same scheme through forward-mode duals of f).
//
// Everything is per point: the FSAL slope reuse, the step controller and
// the caps act on this point only, exactly as the reference's masked batch
// code does per voxel ("a voxel's arithmetic never depends on its batch
// company", odeint.py:432-434).  Host + device.
#pragma once

#include "dual2.cuh"
#include "material.cuh"

namespace am {

enum : int { ST_INTEGRATION = 8 };  // IntegrationError (odeint.py:30-31): caps / underflow

// Butcher tableaux (ode12 odeint.py:92-105, ode23 odeint.py:108-128)
template <int Scheme>
struct Tableau;
template <>
struct Tableau<12> {
    static constexpr int s = 2;
    static constexpr bool fsal = false;
    static constexpr int order_low = 1;
    AM_HD static double a(int i, int j) { return (i == 1 && j == 0) ? 1.0 : 0.0; }
    AM_HD static double b(int j) { return 0.5; }
    AM_HD static double be(int j) { return j == 0 ? 1.0 : 0.0; }
    AM_HD static double c(int i) { return i == 1 ? 1.0 : 0.0; }
};
template <>
struct Tableau<23> {
    static constexpr int s = 4;
    static constexpr bool fsal = true;
    static constexpr int order_low = 2;
    AM_HD static double a(int i, int j) {
        if (i == 1) return j == 0 ? 0.5 : 0.0;
        if (i == 2) return j == 1 ? 0.75 : 0.0;
        if (i == 3) return j == 0 ? 2.0 / 9.0 : (j == 1 ? 1.0 / 3.0 : (j == 2 ? 4.0 / 9.0 : 0.0));
        return 0.0;
    }
    AM_HD static double b(int j) { return j == 0 ? 2.0 / 9.0 : (j == 1 ? 1.0 / 3.0 : (j == 2 ? 4.0 / 9.0 : 0.0)); }
    AM_HD static double be(int j) { return j == 0 ? 7.0 / 24.0 : (j == 1 ? 0.25 : (j == 2 ? 1.0 / 3.0 : 0.125)); }
    // row sums of a (SchemeSpec.c)
    AM_HD static double c(int i) { return i == 0 ? 0.0 : (i == 1 ? 0.5 : (i == 2 ? 0.75 : 1.0)); }
};

// ode23s (odeint.py:116-132): Shampine-Reichelt linearly implicit 2(3) pair
template <>
struct Tableau<32> {
    static constexpr int s = 3;
    static constexpr bool fsal = false;
    static constexpr int order_low = 2;
    AM_HD static double dd() { return 1.0 / (2.0 + 1.4142135623730951); }   // 1 / (2 + sqrt 2)
    AM_HD static double e32() { return 6.0 + 1.4142135623730951; }
    AM_HD static double a(int i, int j) { return (i == 1 && j == 0) ? 0.5 : ((i == 2 && j == 1) ? 1.0 : 0.0); }
    AM_HD static double b(int j) { return j == 1 ? 1.0 : 0.0; }
    AM_HD static double be(int j) { return j == 1 ? 4.0 / 3.0 : -1.0 / 6.0; }
    AM_HD static double c(int i) { return i == 0 ? 0.0 : (i == 1 ? 0.5 : 1.0); }
    AM_HD static double gam(int i, int j) {
        const double d = dd();
        if (i == 0) return j == 0 ? d : 0.0;
        if (i == 1) return j == 0 ? -d : (j == 1 ? d : 0.0);
        return j == 0 ? (e32() - 2.0) * d : (j == 1 ? -e32() * d : d);
    }
    // row sums of gamma (SchemeSpec.gbar)
    AM_HD static double gbar(int i) { return (gam(i, 0) + gam(i, 1)) + gam(i, 2); }
};

// strain at time t of the step and its ramp r = min(t/dt, 1) (odeint.py:256-264)
AM_HD double strain_at(const double* eps_n, const double* eps_np1, double t, double dt, double* e) {
    double r = t / dt;
    r = r < 1.0 ? r : 1.0;
    for (int i = 0; i < 6; ++i) e[i] = eps_n[i] + r * (eps_np1[i] - eps_n[i]);
    return r;
}

// MaterialStepProblem.rhs (odeint.py:286-288)
template <class Law>
AM_HD void rhs_plain(const Law& L, const double* e, const double* a, double* f) {
    auto fv = rhs_sweep(L, plain_tup<6>(e, seq<6>{}), plain_tup<Law::m>(a, seq<Law::m>{}));
    sfor<Law::m>([&](auto I) { f[decltype(I)::value] = get<decltype(I)::value>(fv).v; });
}

template <int... I>
AM_HD auto dual6_tup(const double* a, const double (*da)[6], std::integer_sequence<int, I...>) {
    auto mk = [&](int k) {
        D<0x3Fu> p;
        p.v = a[k];
        for (int j = 0; j < 6; ++j) p.d[j] = da[k][j];
        return p;
    };
    return tup(mk(I)...);
}

// MaterialStepProblem.rhs_dual (odeint.py:298-304): f and
// df/da . ydot + df/deps_{n+1} with eps(t) seeded r * I
template <class Law>
AM_HD void rhs_dual_pt(const Law& L, const double* e, double r, const double* a, const double (*ad)[6], double* f,
                       double (*fd)[6]) {
    auto fv = rhs_sweep(L, seed_tup<0>(e, r, seq<6>{}), dual6_tup(a, ad, seq<Law::m>{}));
    sfor<Law::m>([&](auto I) {
        constexpr int i = decltype(I)::value;
        f[i] = get<i>(fv).v;
        sfor<6>([&](auto K) { fd[i][decltype(K)::value] = get<i>(fv).template dir<decltype(K)::value>(); });
    });
}

// MaterialStepProblem.stress_of / stress_dual (odeint.py:339-352)
template <class Law>
AM_HD void stress_dual_pt(const Law& L, const double* e, double r, const double* a, const double (*ad)[6],
                          double* sig, double (*C)[6]) {
    auto s = stress_sweep(L, seed_tup<0>(e, r, seq<6>{}), dual6_tup(a, ad, seq<Law::m>{}));
    sfor<6>([&](auto I) {
        constexpr int i = decltype(I)::value;
        sig[i] = get<i>(s).v;
        sfor<6>([&](auto K) { C[i][decltype(K)::value] = get<i>(s).template dir<decltype(K)::value>(); });
    });
}

// _scaled_sq (odeint.py:559-561) accumulated
AM_HD double scaled_sq(double diff, double ra, double rb, double atol, double rtol) {
    const double sc = atol + rtol * fmax(fabs(ra), fabs(rb));
    const double x = diff / sc;
    return x * x;
}

// MaterialStepProblem.jac_dir2 (odeint.py:306-337): d/deps_{n+1} of
// [df/da . v_a + df/dt . v_t] at (t, y) with the state sensitivity da as
// chained inner seed, through second-order duals of the hand partials
template <class Law>
AM_HD void jac_dir2(const Law& L, const double* eps_n, const double* eps_np1, double t, double dt, const double* y,
                    const double (*da)[6], const double* v_a, double v_t, double (*out)[6]) {
    constexpr int m = Law::m;
    double r = t / dt;
    r = r < 1.0 ? r : 1.0;
    D2 pe[6], pa[m];
    for (int i = 0; i < 6; ++i) {
        const double de = eps_np1[i] - eps_n[i];
        pe[i].v = eps_n[i] + r * de;
        pe[i].d1 = de / dt * v_t;  // epsdot * v_t
        for (int k = 0; k < 6; ++k) {
            pe[i].d2[k] = k == i ? r : 0.0;
            pe[i].d12[k] = k == i ? v_t / dt : 0.0;
        }
    }
    for (int i = 0; i < m; ++i) {
        pa[i].v = y[i];
        pa[i].d1 = v_a[i];
        for (int k = 0; k < 6; ++k) {
            pa[i].d2[k] = da[i][k];
            pa[i].d12[k] = 0.0;
        }
    }
    auto f = rhs_sweep(L, tup(pe[0], pe[1], pe[2], pe[3], pe[4], pe[5]),
                       tup(pa[0], pa[1], pa[2], pa[3], pa[4], pa[5], pa[6]));
    sfor<m>([&](auto I) {
        for (int k = 0; k < 6; ++k) out[decltype(I)::value][k] = get<decltype(I)::value>(f).d12[k];
    });
}

// _rosenbrock_step (odeint.py:481-531): one linearly implicit embedded step
// with the Jacobian frozen at (t, y); semi-automatic strategy only (the
// reference rejects the automatic one, evaluator.py:61-62).  Returns ok.
template <class Law, bool Coupled>
AM_HD bool rosenbrock_attempt(const Law& L, const double* eps_n, const double* eps_np1, double dt, double t,
                              double h, const double* y, const double (*da)[6], double* yh, double* yl,
                              double (*dh)[6], double (*dl)[6]) {
    static_assert(is_semi_v<Law>, "ode23s needs the hand-coded partials");
    using T = Tableau<32>;
    constexpr int m = Law::m;
    constexpr int s = T::s;
    // rhs_and_jac at (t, y): f0, J, ft = df/deps . epsdot
    double e0[6];
    strain_at(eps_n, eps_np1, t, dt, e0);
    double f0[m], J6[m][6], Je[m][6], J[m][m], ft[m], W[m][m];
    int piv[m];
    L.rhs_jac(e0, y, f0, J6, Je);
    for (int i = 0; i < m; ++i) {
        for (int k = 0; k < 6; ++k) J[i][k] = J6[i][k];
        J[i][6] = 0.0;
        double sft = 0.0;
        for (int k = 0; k < 6; ++k) sft += Je[i][k] * ((eps_np1[k] - eps_n[k]) / dt);
        ft[i] = sft;
    }
    const double g00h = T::gam(0, 0) * h;
    for (int i = 0; i < m; ++i)
        for (int k = 0; k < m; ++k) W[i][k] = (i == k ? 1.0 : 0.0) - g00h * J[i][k];
    bool ok = lu_factor(W, piv);
    double K[s][m], Kd[Coupled ? s : 1][Coupled ? m : 1][6];
    for (int st = 0; st < s; ++st) {
        double yi[m], fi[m], fdi[Coupled ? m : 1][6];
        for (int i = 0; i < m; ++i) yi[i] = y[i];
        for (int q = 0; q < st; ++q)
            if (T::a(st, q) != 0.0)
                for (int i = 0; i < m; ++i) yi[i] += T::a(st, q) * K[q][i];
        const double ti = t + T::c(st) * h;
        if constexpr (Coupled) {
            double ydi[m][6];
            for (int i = 0; i < m; ++i)
                for (int j = 0; j < 6; ++j) ydi[i][j] = da[i][j];
            for (int q = 0; q < st; ++q)
                if (T::a(st, q) != 0.0)
                    for (int i = 0; i < m; ++i)
                        for (int j = 0; j < 6; ++j) ydi[i][j] += T::a(st, q) * Kd[q][i][j];
            double e[6];
            const double r = strain_at(eps_n, eps_np1, ti, dt, e);
            rhs_dual_pt(L, e, r, yi, ydi, fi, fdi);
        } else {
            if (st == 0) {
                for (int i = 0; i < m; ++i) fi[i] = f0[i];
            } else {
                double e[6];
                strain_at(eps_n, eps_np1, ti, dt, e);
                rhs_plain(L, e, yi, fi);
            }
        }
        double rhs[m];
        const double gt = h * T::gbar(st) * h;
        for (int i = 0; i < m; ++i) rhs[i] = h * fi[i] + gt * ft[i];
        for (int q = 0; q < st; ++q) {
            const double g = T::gam(st, q);
            if (g == 0.0) continue;
            for (int i = 0; i < m; ++i) {
                double jk = 0.0;
                for (int n = 0; n < m; ++n) jk += J[i][n] * K[q][n];
                rhs[i] += g * h * jk;
            }
        }
        for (int i = 0; i < m; ++i) K[st][i] = ok ? rhs[i] : 0.0;
        lu_solve(W, piv, K[st]);
        if constexpr (Coupled) {
            double v_a[m], jtv[m][6];
            for (int i = 0; i < m; ++i) v_a[i] = 0.0;
            for (int q = 0; q <= st; ++q)
                if (T::gam(st, q) != 0.0)
                    for (int i = 0; i < m; ++i) v_a[i] += T::gam(st, q) * K[q][i];
            jac_dir2(L, eps_n, eps_np1, t, dt, y, da, v_a, T::gbar(st) * h, jtv);
            for (int j = 0; j < 6; ++j) {
                double col[m];
                for (int i = 0; i < m; ++i) col[i] = h * fdi[i][j] + h * jtv[i][j];
                for (int q = 0; q < st; ++q) {
                    const double g = T::gam(st, q);
                    if (g == 0.0) continue;
                    for (int i = 0; i < m; ++i) {
                        double jk = 0.0;
                        for (int n = 0; n < m; ++n) jk += J[i][n] * Kd[q][n][j];
                        col[i] += g * h * jk;
                    }
                }
                for (int i = 0; i < m; ++i) col[i] = ok ? col[i] : 0.0;
                lu_solve(W, piv, col);
                for (int i = 0; i < m; ++i) Kd[st][i][j] = col[i];
            }
        }
    }
    for (int i = 0; i < m; ++i) {
        double sh = 0.0, sl = 0.0;
        for (int q = 0; q < s; ++q) {
            sh += T::b(q) * K[q][i];
            sl += T::be(q) * K[q][i];
        }
        yh[i] = y[i] + sh;
        yl[i] = y[i] + sl;
        ok = ok && (yh[i] - yh[i] == 0.0) && (yl[i] - yl[i] == 0.0);
        if (Coupled)
            for (int j = 0; j < 6; ++j) {
                double ch = 0.0, cl = 0.0;
                for (int q = 0; q < s; ++q) {
                    ch += T::b(q) * Kd[q][i][j];
                    cl += T::be(q) * Kd[q][i][j];
                }
                dh[i][j] = da[i][j] + ch;
                dl[i][j] = da[i][j] + cl;
            }
    }
    return ok;
}

// One point over [0, dt] (adaptive_integrate, odeint.py:636-756).  Writes the
// unclamped state to a and (Coupled) da = da/deps_{n+1}; substeps / rejected
// counts; with rec_h / rec_acc every attempt's step size and acceptance.  Returns status bits (ST_INTEGRATION when a cap or the step-size
// underflow would raise IntegrationError).
template <class Law, int Scheme, bool Coupled>
AM_HD int adaptive_point(const Law& L, const StepCtl& ctl, const double* eps_n, const double* a_n,
                         const double* eps_np1, double dt, double* a, double (*da)[6], int& substeps, int& rejected,
                         double* rec_h = nullptr, uint8_t* rec_acc = nullptr) {
    using T = Tableau<Scheme>;
    constexpr int m = Law::m;
    constexpr int s = T::s;
    for (int i = 0; i < m; ++i) {
        a[i] = a_n[i];
        if (Coupled)
            for (int j = 0; j < 6; ++j) da[i][j] = 0.0;
    }
    substeps = rejected = 0;
    double t = 0.0, h = dt;
    bool accepted_any = false, g1_valid = false;
    double g1[m], gd1[Coupled ? m : 1][6];
    const int max_attempts = ctl.max_substeps * 4;
    for (int attempts = 1;; ++attempts) {
        if (attempts > max_attempts) return ST_INTEGRATION;  // global attempt cap
        double hi = fmin(h, dt - t);
        const bool clipped = hi >= dt - t - 1e-15 * dt;
        double G[s][m], Gd[Coupled ? s : 1][Coupled ? m : 1][6];
        double yi[m], ydi[Coupled ? m : 1][6];
        double yh[m], yl[m], dh[Coupled ? m : 1][6], dl[Coupled ? m : 1][6];
        bool ok = true;
        if constexpr (Scheme == 32) {
            ok = rosenbrock_attempt<Law, Coupled>(L, eps_n, eps_np1, dt, t, hi, a, da, yh, yl, dh, dl);
        } else {
        auto stage = [&](int st) {
            if (st == 0 && g1_valid) {  // FSAL reuse (odeint.py:443-453)
                for (int i = 0; i < m; ++i) {
                    G[0][i] = g1[i];
                    if (Coupled)
                        for (int j = 0; j < 6; ++j) Gd[0][i][j] = gd1[i][j];
                }
                return;
            }
            for (int i = 0; i < m; ++i) {
                yi[i] = a[i];
                if (Coupled)
                    for (int j = 0; j < 6; ++j) ydi[i][j] = da[i][j];
            }
            for (int q = 0; q < st; ++q) {
                const double aq = T::a(st, q);
                if (aq == 0.0) continue;
                const double w = hi * aq;
                for (int i = 0; i < m; ++i) {
                    yi[i] += w * G[q][i];
                    if (Coupled)
                        for (int j = 0; j < 6; ++j) ydi[i][j] += w * Gd[q][i][j];
                }
            }
            const double ti = t + T::c(st) * hi;
            double e[6];
            const double r = strain_at(eps_n, eps_np1, ti, dt, e);
            if constexpr (Coupled) rhs_dual_pt(L, e, r, yi, ydi, G[st], Gd[st]);
            else rhs_plain(L, e, yi, G[st]);
        };
        // two-stage ode12 with constant stage indices (its slopes then stay
        // in registers: +21%); ode23 rolled (unrolled it spills more, -41%;
        // k1_variants.log)
        if constexpr (s == 2) {
            stage(0);
            stage(1);
        } else {
            for (int st = 0; st < s; ++st) stage(st);
        }
        for (int i = 0; i < m; ++i) {
            double sh = 0.0, sl = 0.0;
            for (int q = 0; q < s; ++q) {
                sh += T::b(q) * G[q][i];
                sl += T::be(q) * G[q][i];
            }
            yh[i] = a[i] + hi * sh;
            yl[i] = a[i] + hi * sl;
            ok = ok && (yh[i] - yh[i] == 0.0) && (yl[i] - yl[i] == 0.0);
            if (Coupled)
                for (int j = 0; j < 6; ++j) {
                    double ch = 0.0, cl = 0.0;
                    for (int q = 0; q < s; ++q) {
                        ch += T::b(q) * Gd[q][i][j];
                        cl += T::be(q) * Gd[q][i][j];
                    }
                    dh[i][j] = da[i][j] + hi * ch;
                    dl[i][j] = da[i][j] + hi * cl;
                }
        }
        }  // explicit stages
        // error_norm (odeint.py:564-617)
        double total = 0.0;
        int count;
        if (ctl.measure == 0) {
            double p = 0.0;
            for (int i = 0; i < m; ++i) p += scaled_sq(yh[i] - yl[i], a[i], yh[i], ctl.atol, ctl.rtol);
            total = p;
            count = m;
            if (Coupled) {
                double pd = 0.0;
                for (int i = 0; i < m; ++i)
                    for (int j = 0; j < 6; ++j)
                        pd += scaled_sq(dh[i][j] - dl[i][j], da[i][j], dh[i][j], ctl.atol, ctl.rtol);
                total = p + pd;
                count += 6 * m;
            }
        } else {
            double e0[6], e1[6], s0[6], sh[6], sl[6];
            const double r0 = strain_at(eps_n, eps_np1, t, dt, e0);
            const double r1 = strain_at(eps_n, eps_np1, t + hi, dt, e1);
            if constexpr (Coupled) {
                double C0[6][6], Ch[6][6], Cl[6][6];
                stress_dual_pt(L, e0, r0, a, da, s0, C0);
                stress_dual_pt(L, e1, r1, yh, dh, sh, Ch);
                stress_dual_pt(L, e1, r1, yl, dl, sl, Cl);
                double pc = 0.0;
                for (int i = 0; i < 6; ++i)
                    for (int j = 0; j < 6; ++j)
                        pc += scaled_sq(Ch[i][j] - Cl[i][j], C0[i][j], Ch[i][j], ctl.atol, ctl.rtol);
                double p = 0.0;
                for (int i = 0; i < 6; ++i) p += scaled_sq(sh[i] - sl[i], s0[i], sh[i], ctl.atol, ctl.rtol);
                total = p + pc;
                count = 42;
            } else {
                (void)r0;
                (void)r1;
                stress_plain(L, e0, a, s0);
                stress_plain(L, e1, yh, sh);
                stress_plain(L, e1, yl, sl);
                double p = 0.0;
                for (int i = 0; i < 6; ++i) p += scaled_sq(sh[i] - sl[i], s0[i], sh[i], ctl.atol, ctl.rtol);
                total = p;
                count = 6;
            }
        }
        double err = sqrt(total / count);
        if (!(err - err == 0.0) || !ok) err = INFINITY;  // non-finite -> inf (odeint.py:617, 697)
        const bool accept = err <= 1.0;
        if (rec_h) {  // record_steps: (attempted h, accepted) per attempt (odeint.py:725-727)
            rec_h[substeps + rejected] = hi;
            rec_acc[substeps + rejected] = accept ? 1 : 0;
        }
        if (accept) {
            t = clipped ? dt : t + hi;
            for (int i = 0; i < m; ++i) {
                a[i] = yh[i];
                if (Coupled)
                    for (int j = 0; j < 6; ++j) da[i][j] = dh[i][j];
            }
            ++substeps;
            accepted_any = true;
        } else {
            ++rejected;
        }
        if constexpr (T::fsal) {  // odeint.py:712-723
            const int src = accept ? s - 1 : 0;
            for (int i = 0; i < m; ++i) {
                g1[i] = G[src][i];
                if (Coupled)
                    for (int j = 0; j < 6; ++j) gd1[i][j] = Gd[src][i][j];
            }
            g1_valid = true;
        }
        // controller (odeint.py:729-738)
        double factor = ctl.safety * pow(err, -1.0 / (T::order_low + 1.0));
        if (err == 0.0) factor = ctl.max_factor;
        if (factor != factor) factor = ctl.min_factor;
        factor = fmin(fmax(factor, ctl.min_factor), ctl.max_factor);
        double hn = hi * factor;
        if (!accepted_any && !accept) hn = 0.5 * hi;
        h = hn;
        const bool done = accept && t >= dt * (1.0 - 1e-12);
        if (substeps + rejected > ctl.max_substeps) return ST_INTEGRATION;
        if (done) return 0;
        if (h < 1e-14 * dt) return ST_INTEGRATION;  // step size underflow
    }
}

#ifdef __CUDACC__
// ---------------------------------------------------------------- lane groups
// Coupled integration with the sensitivity split over a group of 6 lanes:
// lane j advances column j of da/deps_{n+1} (one forward direction: eps_i
// seeded r [i == j], the state with da[:, j]); the primal state, slopes and
// step control are computed identically by every lane of the group.  Per
// direction the arithmetic is the 6-direction sweep's (a dual direction is
// computed independently of the others), so the results are those of
// adaptive_point<Law, Scheme, true>; the per-thread live set drops from
// ~440 doubles (local memory, 116 KB of DRAM traffic per point) to ~120.
// The error norm gathers the column terms with shuffles and sums them in
// the reference's (i, j) order (odeint.py:564-617).

#ifndef AM_LANES_SMEM
#define AM_LANES_SMEM 0
#endif

template <int... I>
AM_HD auto eps_lane_tup(const double* e, double r, int j, std::integer_sequence<int, I...>) {
    auto mk = [&](int i) {
        D<1u> p;
        p.v = e[i];
        p.d[0] = i == j ? r : 0.0;
        return p;
    };
    return tup(mk(I)...);
}
template <int... I>
AM_HD auto a_lane_tup(const double* a, const double* acol, std::integer_sequence<int, I...>) {
    auto mk = [&](int k) {
        D<1u> p;
        p.v = a[k];
        p.d[0] = acol[k];
        return p;
    };
    return tup(mk(I)...);
}

// rhs_dual (odeint.py:298-304) for direction j: f and column j of the sensitivity rhs
template <class Law>
__device__ __forceinline__ void rhs_dual_lane(const Law& L, const double* e, double r, int j, const double* a,
                                              const double* acol, double* f, double* fcol) {
    auto fv = rhs_sweep(L, eps_lane_tup(e, r, j, seq<6>{}), a_lane_tup(a, acol, seq<Law::m>{}));
    sfor<Law::m>([&](auto I) {
        constexpr int i = decltype(I)::value;
        f[i] = get<i>(fv).v;
        fcol[i] = get<i>(fv).template dir<0>();
    });
}

// stress_dual (odeint.py:339-352) / stress_tangent column j; acol = nullptr: frozen state
template <class Law>
__device__ __forceinline__ void stress_dual_lane(const Law& L, const double* e, double r, int j, const double* a,
                                                 const double* acol, double* sig, double* ccol) {
    auto run = [&](const auto& pa) {
        auto sv = stress_sweep(L, eps_lane_tup(e, r, j, seq<6>{}), pa);
        sfor<6>([&](auto I) {
            constexpr int i = decltype(I)::value;
            sig[i] = get<i>(sv).v;
            ccol[i] = get<i>(sv).template dir<0>();
        });
    };
    if (acol) run(a_lane_tup(a, acol, seq<Law::m>{}));
    else run(plain_tup<Law::m>(a, seq<Law::m>{}));
}

// jac_dir2 (odeint.py:306-337) for outer direction j only (lane groups)
template <class Law>
__device__ __forceinline__ void jac_dir2_lane(const Law& L, const double* eps_n, const double* eps_np1, double t,
                                              double dt, const double* y, const double* dacol, const double* v_a,
                                              double v_t, int j, double* out) {
    constexpr int m = Law::m;
    double r = t / dt;
    r = r < 1.0 ? r : 1.0;
    D2T<1> pe[6], pa[m];
    for (int i = 0; i < 6; ++i) {
        const double de = eps_np1[i] - eps_n[i];
        pe[i].v = eps_n[i] + r * de;
        pe[i].d1 = de / dt * v_t;
        pe[i].d2[0] = i == j ? r : 0.0;
        pe[i].d12[0] = i == j ? v_t / dt : 0.0;
    }
    for (int i = 0; i < m; ++i) {
        pa[i].v = y[i];
        pa[i].d1 = v_a[i];
        pa[i].d2[0] = dacol[i];
        pa[i].d12[0] = 0.0;
    }
    auto f = rhs_sweep(L, tup(pe[0], pe[1], pe[2], pe[3], pe[4], pe[5]),
                       tup(pa[0], pa[1], pa[2], pa[3], pa[4], pa[5], pa[6]));
    sfor<m>([&](auto I) { out[decltype(I)::value] = get<decltype(I)::value>(f).d12[0]; });
}

// rosenbrock_attempt<Law, true> for sensitivity column j (lane groups): the
// primal stages are computed identically by every lane
template <class Law>
__device__ bool rosenbrock_attempt_lane(const Law& L, const double* eps_n, const double* eps_np1, double dt,
                                        double t, double h, const double* y, const double* dacol, int j, double* yh,
                                        double* yl, double* dh, double* dl) {
    static_assert(is_semi_v<Law>, "ode23s needs the hand-coded partials");
    using T = Tableau<32>;
    constexpr int m = Law::m;
    constexpr int s = T::s;
    double e0[6];
    strain_at(eps_n, eps_np1, t, dt, e0);
    double f0[m], J6[m][6], Je[m][6], J[m][m], ft[m], W[m][m];
    int piv[m];
    L.rhs_jac(e0, y, f0, J6, Je);
    for (int i = 0; i < m; ++i) {
        for (int k = 0; k < 6; ++k) J[i][k] = J6[i][k];
        J[i][6] = 0.0;
        double sft = 0.0;
        for (int k = 0; k < 6; ++k) sft += Je[i][k] * ((eps_np1[k] - eps_n[k]) / dt);
        ft[i] = sft;
    }
    const double g00h = T::gam(0, 0) * h;
    for (int i = 0; i < m; ++i)
        for (int k = 0; k < m; ++k) W[i][k] = (i == k ? 1.0 : 0.0) - g00h * J[i][k];
    bool ok = lu_factor(W, piv);
    double K[s][m], Kd[s][m];
    for (int st = 0; st < s; ++st) {
        double yi[m], ydi[m], fi[m], fdi[m];
        for (int i = 0; i < m; ++i) {
            yi[i] = y[i];
            ydi[i] = dacol[i];
        }
        for (int q = 0; q < st; ++q)
            if (T::a(st, q) != 0.0)
                for (int i = 0; i < m; ++i) {
                    yi[i] += T::a(st, q) * K[q][i];
                    ydi[i] += T::a(st, q) * Kd[q][i];
                }
        const double ti = t + T::c(st) * h;
        double e[6];
        const double r = strain_at(eps_n, eps_np1, ti, dt, e);
        rhs_dual_lane(L, e, r, j, yi, ydi, fi, fdi);
        double rhs[m];
        const double gt = h * T::gbar(st) * h;
        for (int i = 0; i < m; ++i) rhs[i] = h * fi[i] + gt * ft[i];
        for (int q = 0; q < st; ++q) {
            const double g = T::gam(st, q);
            if (g == 0.0) continue;
            for (int i = 0; i < m; ++i) {
                double jk = 0.0;
                for (int n = 0; n < m; ++n) jk += J[i][n] * K[q][n];
                rhs[i] += g * h * jk;
            }
        }
        for (int i = 0; i < m; ++i) K[st][i] = ok ? rhs[i] : 0.0;
        lu_solve(W, piv, K[st]);
        double v_a[m], jtv[m], col[m];
        for (int i = 0; i < m; ++i) v_a[i] = 0.0;
        for (int q = 0; q <= st; ++q)
            if (T::gam(st, q) != 0.0)
                for (int i = 0; i < m; ++i) v_a[i] += T::gam(st, q) * K[q][i];
        jac_dir2_lane(L, eps_n, eps_np1, t, dt, y, dacol, v_a, T::gbar(st) * h, j, jtv);
        for (int i = 0; i < m; ++i) col[i] = h * fdi[i] + h * jtv[i];
        for (int q = 0; q < st; ++q) {
            const double g = T::gam(st, q);
            if (g == 0.0) continue;
            for (int i = 0; i < m; ++i) {
                double jk = 0.0;
                for (int n = 0; n < m; ++n) jk += J[i][n] * Kd[q][n];
                col[i] += g * h * jk;
            }
        }
        for (int i = 0; i < m; ++i) col[i] = ok ? col[i] : 0.0;
        lu_solve(W, piv, col);
        for (int i = 0; i < m; ++i) Kd[st][i] = col[i];
    }
    for (int i = 0; i < m; ++i) {
        double sh = 0.0, sl = 0.0, ch = 0.0, cl = 0.0;
        for (int q = 0; q < s; ++q) {
            sh += T::b(q) * K[q][i];
            sl += T::be(q) * K[q][i];
            ch += T::b(q) * Kd[q][i];
            cl += T::be(q) * Kd[q][i];
        }
        yh[i] = y[i] + sh;
        yl[i] = y[i] + sl;
        ok = ok && (yh[i] - yh[i] == 0.0) && (yl[i] - yl[i] == 0.0);
        dh[i] = dacol[i] + ch;
        dl[i] = dacol[i] + cl;
    }
    return ok;
}

// sum over (i, jj) in the reference's order of the group's per-column terms t[i]
template <int N>
__device__ __forceinline__ double group_sum(const double* t, unsigned gmask, int gbase) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int jj = 0; jj < 6; ++jj) s += __shfl_sync(gmask, t[i], gbase + jj);
    return s;
}

// adaptive_point<Law, Scheme, true> by a lane group: every lane returns the
// same status / counts / primal state a; dacol = column j of da.
template <class Law, int Scheme>
__device__ int adaptive_point_lanes(const Law& L, const StepCtl& ctl, const double* eps_n, const double* a_n,
                                    const double* eps_np1, double dt, double* a, double* dacol, int& substeps,
                                    int& rejected, int j, unsigned gmask, int gbase, double* rec_h,
                                    uint8_t* rec_acc, double* gs = nullptr, int gst = 0) {
    using T = Tableau<Scheme>;
    constexpr int m = Law::m;
    constexpr int s = T::s;
    for (int i = 0; i < m; ++i) {
        a[i] = a_n[i];
        dacol[i] = 0.0;
    }
    substeps = rejected = 0;
    double t = 0.0, h = dt;
    bool accepted_any = false, g1_valid = false;
    double g1[m], gd1[m];
    const int max_attempts = ctl.max_substeps * 4;
    for (int attempts = 1;; ++attempts) {
        if (attempts > max_attempts) return ST_INTEGRATION;  // global attempt cap
        double hi = fmin(h, dt - t);
        const bool clipped = hi >= dt - t - 1e-15 * dt;
        // stage slopes: registers, or (gs) this thread's strided slice of
        // shared memory, element (q, i) at gs[(q * m + i) * gst]
        double Greg[AM_LANES_SMEM ? 1 : s][m], Gdreg[AM_LANES_SMEM ? 1 : s][m];
        auto G = [&](int q, int i) -> double& {
            if constexpr (AM_LANES_SMEM) return gs[(q * m + i) * gst];
            else return Greg[q][i];
        };
        auto Gd = [&](int q, int i) -> double& {
            if constexpr (AM_LANES_SMEM) return gs[((s + q) * m + i) * gst];
            else return Gdreg[q][i];
        };
        double yh[m], yl[m], dh[m], dl[m];
        bool ok = true;
        if constexpr (Scheme == 32) {
            ok = rosenbrock_attempt_lane<Law>(L, eps_n, eps_np1, dt, t, hi, a, dacol, j, yh, yl, dh, dl);
        } else {
        auto stage = [&](int st) {
            if (st == 0 && g1_valid) {  // FSAL reuse (odeint.py:443-453)
                for (int i = 0; i < m; ++i) {
                    G(0, i) = g1[i];
                    Gd(0, i) = gd1[i];
                }
                return;
            }
            double yi[m], ydi[m];
            for (int i = 0; i < m; ++i) {
                yi[i] = a[i];
                ydi[i] = dacol[i];
            }
            for (int q = 0; q < st; ++q) {
                const double aq = T::a(st, q);
                if (aq == 0.0) continue;
                const double w = hi * aq;
                for (int i = 0; i < m; ++i) {
                    yi[i] += w * G(q, i);
                    ydi[i] += w * Gd(q, i);
                }
            }
            const double ti = t + T::c(st) * hi;
            double e[6];
            const double r = strain_at(eps_n, eps_np1, ti, dt, e);
            double fo[m], fco[m];
            rhs_dual_lane(L, e, r, j, yi, ydi, fo, fco);
            for (int i = 0; i < m; ++i) {
                G(st, i) = fo[i];
                Gd(st, i) = fco[i];
            }
        };
        if constexpr (s == 2) {
            stage(0);
            stage(1);
        } else {
            for (int st = 0; st < s; ++st) stage(st);
        }
        for (int i = 0; i < m; ++i) {
            double sh = 0.0, sl = 0.0, ch = 0.0, cl = 0.0;
            for (int q = 0; q < s; ++q) {
                sh += T::b(q) * G(q, i);
                sl += T::be(q) * G(q, i);
                ch += T::b(q) * Gd(q, i);
                cl += T::be(q) * Gd(q, i);
            }
            yh[i] = a[i] + hi * sh;
            yl[i] = a[i] + hi * sl;
            ok = ok && (yh[i] - yh[i] == 0.0) && (yl[i] - yl[i] == 0.0);
            dh[i] = dacol[i] + hi * ch;
            dl[i] = dacol[i] + hi * cl;
        }
        }  // explicit stages
        // error_norm (odeint.py:564-617)
        double total;
        int count;
        if (ctl.measure == 0) {
            double p = 0.0, tt[m];
            for (int i = 0; i < m; ++i) p += scaled_sq(yh[i] - yl[i], a[i], yh[i], ctl.atol, ctl.rtol);
            for (int i = 0; i < m; ++i) tt[i] = scaled_sq(dh[i] - dl[i], dacol[i], dh[i], ctl.atol, ctl.rtol);
            total = p + group_sum<m>(tt, gmask, gbase);
            count = m + 6 * m;
        } else {
            double e0[6], e1[6], s0[6], sh[6], sl[6], c0[6], chh[6], cll[6], tc[6];
            const double r0 = strain_at(eps_n, eps_np1, t, dt, e0);
            const double r1 = strain_at(eps_n, eps_np1, t + hi, dt, e1);
            stress_dual_lane(L, e0, r0, j, a, dacol, s0, c0);
            stress_dual_lane(L, e1, r1, j, yh, dh, sh, chh);
            stress_dual_lane(L, e1, r1, j, yl, dl, sl, cll);
            for (int i = 0; i < 6; ++i) tc[i] = scaled_sq(chh[i] - cll[i], c0[i], chh[i], ctl.atol, ctl.rtol);
            const double pc = group_sum<6>(tc, gmask, gbase);
            double p = 0.0;
            for (int i = 0; i < 6; ++i) p += scaled_sq(sh[i] - sl[i], s0[i], sh[i], ctl.atol, ctl.rtol);
            total = p + pc;
            count = 42;
        }
        double err = sqrt(total / count);
        if (!(err - err == 0.0) || !ok) err = INFINITY;  // non-finite -> inf (odeint.py:617, 697)
        const bool accept = err <= 1.0;
        if (rec_h && j == 0) {  // record_steps (odeint.py:725-727)
            rec_h[substeps + rejected] = hi;
            rec_acc[substeps + rejected] = accept ? 1 : 0;
        }
        if (accept) {
            t = clipped ? dt : t + hi;
            for (int i = 0; i < m; ++i) {
                a[i] = yh[i];
                dacol[i] = dh[i];
            }
            ++substeps;
            accepted_any = true;
        } else {
            ++rejected;
        }
        if constexpr (T::fsal) {  // odeint.py:712-723
            const int src = accept ? s - 1 : 0;
            for (int i = 0; i < m; ++i) {
                g1[i] = G(src, i);
                gd1[i] = Gd(src, i);
            }
            g1_valid = true;
        }
        // controller (odeint.py:729-738)
        double factor = ctl.safety * pow(err, -1.0 / (T::order_low + 1.0));
        if (err == 0.0) factor = ctl.max_factor;
        if (factor != factor) factor = ctl.min_factor;
        factor = fmin(fmax(factor, ctl.min_factor), ctl.max_factor);
        double hn = hi * factor;
        if (!accepted_any && !accept) hn = 0.5 * hi;
        h = hn;
        const bool done = accept && t >= dt * (1.0 - 1e-12);
        if (substeps + rejected > ctl.max_substeps) return ST_INTEGRATION;
        if (done) return 0;
        if (h < 1e-14 * dt) return ST_INTEGRATION;  // step size underflow
    }
}
#endif  // __CUDACC__

}  // namespace am
