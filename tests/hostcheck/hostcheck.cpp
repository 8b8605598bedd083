// Host (g++) build of the device material code in csrc/material.cuh.
// TEST INFRASTRUCTURE ONLY: lets the CPU test-suite check the AD / Newton /
// tangent logic of the CUDA kernel against the oracle without a GPU.  The
// product package never loads this library.
#include <cstdint>
#include <cstring>

#include "../../paper_2006_04391_b200/csrc/material.cuh"

using namespace am;

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
        int st = eval_voxel(L, cfg, eps_n + 6 * b, an, eps_np1 + 6 * b, dt[b], sig + 6 * b, ao,
                            want_tangent ? Cv : nullptr, it);
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
