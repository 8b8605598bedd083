// fft_cb.h -- load callback of the basic scheme's inverse transform (fft_cb.cu)
#pragma once
#include <cuda_runtime.h>
#include <cufft.h>

// layout shared with the callback source compiled at run time (fft_cb.cu)
struct AmZ2DCb {
    const double2* ehat;  // carried spectrum ehat' (origin bins: N ebar)
    double inv_n;         // 1 / (nx ny nz), a power of two
};

bool am_z2d_callback_plan(cufftHandle* p, long long* n3, long long idist, long long odist, long long batch,
                          cudaStream_t stream, void* d_info);
