// common.cuh -- error plumbing shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/automat.h"

namespace am {

// thread-local message for am_last_error()
std::string& last_error();

inline int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    last_error() = buf;
    return code;
}

#define AM_CUDA(expr)                                                                         \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            return ::am::fail(AM_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,         \
                              cudaGetErrorString(_e));                                        \
    } while (0)

#define AM_TRY(expr)                 \
    do {                             \
        int _rc = (expr);            \
        if (_rc != AM_OK) return _rc; \
    } while (0)

constexpr int kSMs = 148;  // B200

}  // namespace am
