// api.cu -- library-level C-ABI entry points (errors, version, devices).
#include <algorithm>

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

// ---------------------------------------------------------------- pinned host pool
// Page-locked host blocks for result arrays handed to the caller (the Python
// shim's evaluate_arrays outputs): the D2H copies land in them directly.
// Freed blocks are cached by size and reused; at most kKeep bytes are kept.
#include <map>
#include <mutex>

namespace {
struct PinnedPool {
    std::mutex mu;
    std::multimap<size_t, void*> free_blocks;
    std::map<void*, size_t> size_of;
    size_t cached = 0;
    static constexpr size_t kKeep = size_t(8) << 30;
};
PinnedPool& pinned_pool() {
    static PinnedPool* p = new PinnedPool();  // never destroyed: blocks may outlive static destruction
    return *p;
}
}  // namespace

extern "C" int am_host_alloc(int64_t bytes, void** out) {
    if (!out || bytes < 0) return am::fail(AM_ERR_ARG, "am_host_alloc: bad arguments");
    const size_t want = std::max<size_t>((size_t)bytes, 64);
    PinnedPool& P = pinned_pool();
    {
        std::lock_guard<std::mutex> lk(P.mu);
        auto it = P.free_blocks.lower_bound(want);
        if (it != P.free_blocks.end() && it->first <= 2 * want) {
            *out = it->second;
            P.cached -= it->first;
            P.free_blocks.erase(it);
            return AM_OK;
        }
    }
    void* p = nullptr;
    AM_CUDA(cudaHostAlloc(&p, want, cudaHostAllocPortable));
    std::lock_guard<std::mutex> lk(P.mu);
    P.size_of[p] = want;
    *out = p;
    return AM_OK;
}

extern "C" int am_host_free(void* p) {
    if (!p) return AM_OK;
    PinnedPool& P = pinned_pool();
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = P.size_of.find(p);
    if (it == P.size_of.end()) return am::fail(AM_ERR_ARG, "am_host_free: not a pool block");
    const size_t n = it->second;
    // evict the largest cached blocks while over budget
    while (P.cached + n > PinnedPool::kKeep && !P.free_blocks.empty()) {
        auto last = std::prev(P.free_blocks.end());
        P.size_of.erase(last->second);
        P.cached -= last->first;
        cudaFreeHost(last->second);
        P.free_blocks.erase(last);
    }
    if (n > PinnedPool::kKeep) {
        P.size_of.erase(it);
        AM_CUDA(cudaFreeHost(p));
        return AM_OK;
    }
    P.free_blocks.emplace(n, p);
    P.cached += n;
    return AM_OK;
}
