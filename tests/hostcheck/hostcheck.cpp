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
                              double* sig, double* a_out, double* C, int32_t* iters, uint8_t* status) {
    NewtonCfg cfg{mode, 50, tol};
    if (kind == 1) {
        auto L = MichelSuquetLaw::make(prm[0], prm[1], prm[2], prm[3], prm[4], prm[5], prm[6]);
        return run(L, cfg, B, eps_n, a_n, eps_np1, dt, want_tangent, sig, a_out, C, iters, status);
    }
    auto L = LinearElasticLaw::make(prm[0], prm[1]);
    return run(L, cfg, B, eps_n, a_n, eps_np1, dt, want_tangent, sig, a_out, C, iters, status);
}
