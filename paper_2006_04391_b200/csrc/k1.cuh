// k1.cuh -- launch interface of the material kernel (K1) shared by the
// material-point entry points (material.cu) and the basic-scheme solver
// (solver.cu).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/automat.h"
#include "newton_cfg.cuh"

namespace am {

struct Layout {
    int64_t cs, es;  // element (c, b) at p[c * cs + b * es]
};

struct KArgs {
    int64_t B;
    const int64_t* gidx;  // optional gather/scatter index for eps_n / eps_np1 / sigma
    const double* eps_n;
    const double* a_n;
    const double* a_start;  // optional first Newton iterate (same layout as a_n; may alias a_out)
    const double* eps_np1;
    const double* dt;
    double dt_scalar;
    Layout le, la, lc;
    double* sigma;
    double* a_out;
    double* C;
    int32_t* iters;     // Newton count (implicit Euler) / accepted substeps (adaptive)
    int32_t* rejected;  // rejected attempts (adaptive), optional
    uint8_t* status;
    uint32_t* flags;
    NewtonCfg ncfg;
    int integrator;     // AM_INTEGRATOR_*
    int strategy;       // AM_STRATEGY_*
    StepCtl sctl;
    unsigned long long* sub_sum;  // optional: += accepted substeps of the adaptive kernels
    // optional step records of the adaptive kernels: point b's attempts at
    // rec_h / rec_acc [rec_off[b], rec_off[b+1]) (record_steps)
    const int64_t* rec_off;
    double* rec_h;
    uint8_t* rec_acc;
};

// validation and dispatch (material.cu)
int check_law(const am_law* law);
int check_cfg(const am_cfg* cfg);
int law_m(const am_law* law);
NewtonCfg newton_cfg(const am_cfg* cfg);
StepCtl step_ctl(const am_cfg* cfg);
// fills ncfg, integrator and sctl of k from cfg
void set_controls(KArgs& k, const am_cfg* cfg);
// enqueue K1 on stream s: Newton (+ clamp + stress), or with k.C the Newton
// then tangent kernels; per-point status bits OR-ed into *k.flags
int launch_material(const am_law* law, const KArgs& k, cudaStream_t s);

}  // namespace am
