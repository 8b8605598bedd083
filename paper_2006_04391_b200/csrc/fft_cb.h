// fft_cb.h -- load callback of the basic scheme's inverse transform (fft_cb.cu)
#pragma once
#include <cuda_runtime.h>
#include <cufftXt.h>

// layout shared with the callback source compiled at run time (fft_cb.cu)
struct AmZ2DCb {
    const double2* ehat;  // carried spectrum ehat' (origin bins: N ebar)
    double inv_n;         // 1 / (nx ny nz), a power of two
};

// the slab algorithm's transposes riding on the 2-D transforms: element
// offset o of a slab's 2-D spectra (c, xl, ky, kz) <-> block j = ky / nyl
// of the x-pencil layout, base[j] + ((xl * 6 + c) * nyl + ky % nyl) * nzh + kz
// (base[j]: the peer's spectrum at this rank's block, or the all-to-all
// buffer's block j).  The D2Z stores through am_pack_store, the Z2D loads
// through am_unpack_load: k_pack / k_unpack and their pass over P vanish.
struct AmPackCb {
    double2* const* base;  // device array of the destination / source blocks
    unsigned nzh, ny, nxl, nyl;
};

bool am_callback_plan(cufftHandle* p, int rank, long long* n, long long* inembed, long long istride, long long idist,
                      long long* onembed, long long ostride, long long odist, cufftType type, long long batch,
                      cudaStream_t stream, void* d_info, const char* symbol, int cb_type, size_t* ws_max);
