// Host (g++) build of the device material code in csrc/material.cuh.
// TEST INFRASTRUCTURE ONLY: lets the CPU test-suite check the AD / Newton /
// tangent logic of the CUDA kernel against the oracle without a GPU.  The
// product package never loads this library.
#include <cstdint>
#include <cstring>

#include "../../paper_2006_04391_b200/csrc/material.cuh"

using namespace am;

struct HostSink {
    double (*C)[6];
    void col(int j, const double* c) {
        for (int i = 0; i < 6; ++i) C[i][j] = c[i];
    }
};

// the GPU's two phases in sequence (material.cu k_material / k_tangent)
template <class Law, int Mode, bool Tangent>
static int point(const Law& L, const NewtonCfg& cfg, const double* en, const double* an, const double* ep, double dt,
                 double* sig, double* ao, double (*Cv)[6], int& it) {
    double a[8];
    int st = newton_point<Law, Mode>(L, cfg, en, an, ep, dt, a, it);
    if (!Tangent) {
        stress_point(L, ep, a, ao, sig);
        return st;
    }
    HostSink s{Cv};
    if (st & ST_NEWTON) {
        failed_point(L, ep, a, ao, sig, s);
        return st;
    }
    return st | tangent_point(L, en, ep, dt, a, ao, sig, s);
}

template <class Law>
static int run(const Law& L, const NewtonCfg& cfg, int64_t B, const double* eps_n, const double* a_n,
               const double* eps_np1, const double* dt, int want_tangent, double* sig, double* a_out, double* C,
               int32_t* iters, uint8_t* status) {
    constexpr int m = Law::m;
    int any = 0;
    for (int64_t b = 0; b < B; ++b) {
        double Cv[6][6];
        double an[7] = {0}, ao[7] = {0};
        if (m) std::memcpy(an, a_n + m * b, sizeof(double) * m);
        int it = 0;
        int st;
        const double *en = eps_n + 6 * b, *ep = eps_np1 + 6 * b;
        if (cfg.mode == 1)
            st = want_tangent ? point<Law, 1, true>(L, cfg, en, an, ep, dt[b], sig + 6 * b, ao, Cv, it)
                              : point<Law, 1, false>(L, cfg, en, an, ep, dt[b], sig + 6 * b, ao, Cv, it);
        else
            st = want_tangent ? point<Law, 0, true>(L, cfg, en, an, ep, dt[b], sig + 6 * b, ao, Cv, it)
                              : point<Law, 0, false>(L, cfg, en, an, ep, dt[b], sig + 6 * b, ao, Cv, it);
        if (m) std::memcpy(a_out + m * b, ao, sizeof(double) * m);
        if (want_tangent) std::memcpy(C + 36 * b, Cv, sizeof(Cv));
        iters[b] = it;
        status[b] = (uint8_t)st;
        any |= st;
    }
    return any;
}

extern "C" int hostcheck_eval(int kind, const double* prm, int mode, double tol, int64_t B, const double* eps_n,
                              const double* a_n, const double* eps_np1, const double* dt, int want_tangent,
                              double* sig, double* a_out, double* C, int32_t* iters, uint8_t* status, int semi) {
    NewtonCfg cfg{mode, 50, tol};
    if (kind == 1) {
        if (semi) {
            auto L = SemiLaw<MichelSuquetLaw>::make(prm[0], prm[1], prm[2], prm[3], prm[4], prm[5], prm[6]);
            return run(L, cfg, B, eps_n, a_n, eps_np1, dt, want_tangent, sig, a_out, C, iters, status);
        }
        auto L = MichelSuquetLaw::make(prm[0], prm[1], prm[2], prm[3], prm[4], prm[5], prm[6]);
        return run(L, cfg, B, eps_n, a_n, eps_np1, dt, want_tangent, sig, a_out, C, iters, status);
    }
    if (semi) {
        auto L = SemiLaw<LinearElasticLaw>::make(prm[0], prm[1]);
        return run(L, cfg, B, eps_n, a_n, eps_np1, dt, want_tangent, sig, a_out, C, iters, status);
    }
    auto L = LinearElasticLaw::make(prm[0], prm[1]);
    return run(L, cfg, B, eps_n, a_n, eps_np1, dt, want_tangent, sig, a_out, C, iters, status);
}

// the tangent post-process alone at a given (unclamped, "converged") state:
// the singular-tangent route (odeint.py:424 check_singular) without a Newton
extern "C" int hostcheck_tangent_point(const double* prm, int64_t B, const double* eps_n, const double* a,
                                       const double* eps_np1, const double* dt, double* sig, double* C,
                                       uint8_t* status) {
    auto L = MichelSuquetLaw::make(prm[0], prm[1], prm[2], prm[3], prm[4], prm[5], prm[6]);
    int any = 0;
    for (int64_t b = 0; b < B; ++b) {
        double ac[7], Cv[6][6];
        HostSink sink{Cv};
        const int st = tangent_point(L, eps_n + 6 * b, eps_np1 + 6 * b, dt[b], a + 7 * b, ac, sig + 6 * b, sink);
        std::memcpy(C + 36 * b, Cv, sizeof(Cv));
        status[b] = (uint8_t)st;
        any |= st;
    }
    return any;
}

// adaptive ode12 / ode23 (material.cu k_adaptive on the host)
#include "../../paper_2006_04391_b200/csrc/adaptive.cuh"

template <int Scheme, bool Coupled, class Law>
static int run_adaptive(const Law& L, const StepCtl& ctl, int64_t B, const double* eps_n,
                        const double* a_n, const double* eps_np1, const double* dt, double* sig, double* a_out,
                        double* C, int32_t* sub, int32_t* rej, uint8_t* status) {
    int any = 0;
    for (int64_t b = 0; b < B; ++b) {
        const double *en = eps_n + 6 * b, *ep = eps_np1 + 6 * b, *an = a_n + 7 * b;
        double a[7], ac[7], da[7][6], Cv[6][6];
        int s = 1, r = 0, st = 0;
        HostSink sink{Cv};
        if (dt[b] == 0.0) {
            for (int i = 0; i < 7; ++i) ac[i] = an[i];
            stress_plain(L, ep, an, sig + 6 * b);
            if (Coupled) {
                double s2[6];
                stress_tangent(L, ep, an, nullptr, s2, Cv);
            }
        } else {
            st = adaptive_point<Law, Scheme, Coupled>(L, ctl, en, an, ep, dt[b], a, da, s, r);
            clamp_state<Law>(a, ac);
            if (Coupled) stress_tangent(L, ep, ac, da, sig + 6 * b, Cv);
            else stress_plain(L, ep, ac, sig + 6 * b);
        }
        std::memcpy(a_out + 7 * b, ac, sizeof(ac));
        if (Coupled) std::memcpy(C + 36 * b, Cv, sizeof(Cv));
        sub[b] = s;
        rej[b] = r;
        status[b] = (uint8_t)st;
        any |= st;
    }
    return any;
}

extern "C" int hostcheck_adaptive(const double* prm, int scheme, int coupled, int measure, double atol, double rtol,
                                  int max_sub, int64_t B, const double* eps_n, const double* a_n, const double* eps_np1,
                                  const double* dt, double* sig, double* a_out, double* C, int32_t* sub, int32_t* rej,
                                  uint8_t* status, int semi) {
    StepCtl ctl;
    ctl.atol = atol;
    ctl.rtol = rtol;
    ctl.max_substeps = max_sub;
    ctl.measure = measure;
    if (scheme == 32) {  // ode23s: semi-automatic only
        auto L = SemiLaw<MichelSuquetLaw>::make(prm[0], prm[1], prm[2], prm[3], prm[4], prm[5], prm[6]);
        return coupled ? run_adaptive<32, true>(L, ctl, B, eps_n, a_n, eps_np1, dt, sig, a_out, C, sub, rej, status)
                       : run_adaptive<32, false>(L, ctl, B, eps_n, a_n, eps_np1, dt, sig, a_out, C, sub, rej, status);
    }
    auto go = [&](const auto& L) {
        if (scheme == 23)
            return coupled ? run_adaptive<23, true>(L, ctl, B, eps_n, a_n, eps_np1, dt, sig, a_out, C, sub, rej, status)
                           : run_adaptive<23, false>(L, ctl, B, eps_n, a_n, eps_np1, dt, sig, a_out, C, sub, rej,
                                                     status);
        return coupled ? run_adaptive<12, true>(L, ctl, B, eps_n, a_n, eps_np1, dt, sig, a_out, C, sub, rej, status)
                       : run_adaptive<12, false>(L, ctl, B, eps_n, a_n, eps_np1, dt, sig, a_out, C, sub, rej, status);
    };
    if (semi) return go(SemiLaw<MichelSuquetLaw>::make(prm[0], prm[1], prm[2], prm[3], prm[4], prm[5], prm[6]));
    return go(MichelSuquetLaw::make(prm[0], prm[1], prm[2], prm[3], prm[4], prm[5], prm[6]));
}

// conventional radial return (material.cu k_conventional on the host)
#include "../../paper_2006_04391_b200/csrc/conventional.cuh"

extern "C" int hostcheck_conventional(const double* prm, int64_t B, const double* eps_np1, const double* a_n,
                                      const double* dt, int want_tangent, double* sig, double* a_out, double* C) {
    auto S = SemiLaw<MichelSuquetLaw>::make(prm[0], prm[1], prm[2], prm[3], prm[4], prm[5], prm[6]);
    int any = 0;
    for (int64_t b = 0; b < B; ++b) {
        double Cv[6][6];
        if (dt[b] == 0.0) {
            std::memcpy(a_out + 7 * b, a_n + 7 * b, 7 * sizeof(double));
            stress_plain(S, eps_np1 + 6 * b, a_n + 7 * b, sig + 6 * b);
            S.Ce(Cv);
        } else {
            any |= conventional_point(S, eps_np1 + 6 * b, a_n + 7 * b, dt[b], sig + 6 * b, a_out + 7 * b,
                                      want_tangent ? Cv : nullptr);
        }
        if (want_tangent) std::memcpy(C + 36 * b, Cv, sizeof(Cv));
    }
    return any;
}
