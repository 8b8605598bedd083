// LTO load callback for tools/cufft_cb_probe.cu: the Z2D reads the carried
// spectrum (callerInfo->carry) scaled by 1/N instead of a scaled copy.
#include <cufftXt.h>

struct CbInfo {
    const double2* carry;
    double inv_n;
};

__device__ cufftDoubleComplex cb_load_scaled(void* dataIn, unsigned long long offset, void* callerInfo, void* shared) {
    const CbInfo* ci = static_cast<const CbInfo*>(callerInfo);
    double2 v = ci->carry[offset];
    return make_double2(v.x * ci->inv_n, v.y * ci->inv_n);
}
