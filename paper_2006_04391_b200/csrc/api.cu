// api.cu -- library-level C-ABI entry points (errors, version, devices).
#include "common.cuh"

namespace am {
std::string& last_error() {
    static thread_local std::string msg;
    return msg;
}
}  // namespace am

extern "C" const char* am_last_error(void) { return am::last_error().c_str(); }

extern "C" const char* am_version(void) { return "automat-b200 0.1 (sm_100a, fp64)"; }

extern "C" int am_device_count(int* count) {
    AM_CUDA(cudaGetDeviceCount(count));
    return AM_OK;
}

extern "C" int am_set_device(int device) {
    AM_CUDA(cudaSetDevice(device));
    return AM_OK;
}
