// fft_cb.h -- load callback of the basic scheme's inverse transform (fft_cb.cu)
#pragma once
#include <cuda_runtime.h>
#include <cufft.h>

// layout shared with the callback source compiled at run time (fft_cb.cu)
struct AmZ2DCb {
    const double2* ehat;  // carried spectrum ehat' (origin bins: N ebar)
    double inv_n;         // 1 / (nx ny nz), a power of two
};

bool am_callback_plan(cufftHandle* p, int rank, long long* n, long long* inembed, long long istride, long long idist,
                      long long* onembed, long long ostride, long long odist, cufftType type, long long batch,
                      cudaStream_t stream, void* d_info);
