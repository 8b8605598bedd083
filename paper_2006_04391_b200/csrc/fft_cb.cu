// fft_cb.cu -- the basic scheme's inverse transform reading the carried
// spectrum through a cuFFT load callback (one slab: the 3-D Z2D; x slabs:
// each slab's inverse 1-D x transform).
//
// k_fourier leaves ehat' (the carried spectrum of the next strain) in ehat;
// the Z2D destroys its input, so without a callback k_fourier also writes a
// scaled copy ehat'/N into S for the transform to consume (96 B per rfft
// bin, a quarter of k_fourier's traffic).  With the callback the transform's
// first pass loads ehat'[q] * (1 / N) directly, and S -- whose sigma-hat is
// dead by then -- is only the transform's nominal input and workspace.
// Same products as the copy, so the fields are bitwise those of the copy
// path.  The origin bins hold N ebar (k_origin_dev), and the copy path
// feeds ebar there: N is a power of two for the callback path, so
// (N ebar) / N == ebar exactly and the callback needs no branch (an origin
// test in the callback made the transform 30% slower).
//
// cuFFT links callbacks as LTO IR with the nvJitLink of the cuFFT in the
// process (the one torch loaded, or the system one).  IR from a newer
// compiler than that linker is rejected, so the IR is compiled at run time
// by the NVRTC that sits next to the cuFFT in use (same CUDA release), and
// any failure along the way leaves the caller on the copy path.
#include <cuda_runtime.h>
#include <cufftXt.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "fft_cb.h"

namespace {

const char* kSource = R"(
struct AmZ2DCb { const double2* ehat; double inv_n; };
__device__ double2 am_z2d_load(void* in, unsigned long long off, void* info, void* sh) {
    const AmZ2DCb* c = (const AmZ2DCb*)info;
    const double2 v = c->ehat[off];
    return make_double2(v.x * c->inv_n, v.y * c->inv_n);
}
struct AmPackCb { double2* const* base; unsigned nzh, ny, nxl, nyl; };
__device__ __forceinline__ double2* am_pack_addr(const AmPackCb* p, unsigned o) {
    const unsigned kz = o % p->nzh, t = o / p->nzh;
    const unsigned ky = t % p->ny, cx = t / p->ny;
    const unsigned c = cx / p->nxl, xl = cx - c * p->nxl;
    const unsigned j = ky / p->nyl, kyl = ky - j * p->nyl;
    return p->base[j] + ((unsigned long long)(xl * 6 + c) * p->nyl + kyl) * p->nzh + kz;
}
__device__ void am_pack_store(void* out, unsigned long long off, double2 v, void* info, void* sh) {
    *am_pack_addr((const AmPackCb*)info, (unsigned)off) = v;
}
__device__ double2 am_unpack_load(void* in, unsigned long long off, void* info, void* sh) {
    return *am_pack_addr((const AmPackCb*)info, (unsigned)off);
}
)";

struct Nvrtc {
    void* lib = nullptr;
    nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*);
    nvrtcResult (*compile)(nvrtcProgram, int, const char* const*);
    nvrtcResult (*ir_size)(nvrtcProgram, size_t*);
    nvrtcResult (*ir)(nvrtcProgram, char*);
    nvrtcResult (*destroy)(nvrtcProgram*);
    bool bind(void* h) {
        lib = h;
        create = (decltype(create))dlsym(h, "nvrtcCreateProgram");
        compile = (decltype(compile))dlsym(h, "nvrtcCompileProgram");
        ir_size = (decltype(ir_size))dlsym(h, "nvrtcGetLTOIRSize");
        ir = (decltype(ir))dlsym(h, "nvrtcGetLTOIR");
        destroy = (decltype(destroy))dlsym(h, "nvrtcDestroyProgram");
        return create && compile && ir_size && ir && destroy;
    }
};

// libnvrtc.so.12 of the CUDA release of the cuFFT in this process:
// <...>/nvidia/cufft/lib -> <...>/nvidia/cuda_nvrtc/lib (pip wheels),
// <cuda>/lib64 -> the same directory (toolkit); then the default search.
std::vector<std::string> nvrtc_candidates() {
    std::vector<std::string> out;
    Dl_info di{};
    if (dladdr((void*)&cufftCreate, &di) && di.dli_fname) {
        std::string p = di.dli_fname;
        const size_t slash = p.rfind('/');
        if (slash != std::string::npos) {
            const std::string dir = p.substr(0, slash);
            const std::string wheel = "/cufft/lib";
            if (dir.size() > wheel.size() && dir.compare(dir.size() - wheel.size(), wheel.size(), wheel) == 0)
                out.push_back(dir.substr(0, dir.size() - wheel.size()) + "/cuda_nvrtc/lib/libnvrtc.so.12");
            out.push_back(dir + "/libnvrtc.so.12");
        }
    }
    out.push_back("libnvrtc.so.12");
    return out;
}

bool lto_ir(const std::string& path, std::vector<char>& ir) {
    void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
    if (!h) return false;
    Nvrtc r;
    if (!r.bind(h)) return false;
    nvrtcProgram prog = nullptr;
    if (r.create(&prog, kSource, "am_z2d_load.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) return false;
    const char* opts[] = {"-arch=sm_100a", "-dlto", "-rdc=true"};
    bool ok = r.compile(prog, 3, opts) == NVRTC_SUCCESS;
    size_t n = 0;
    if (ok) ok = r.ir_size(prog, &n) == NVRTC_SUCCESS && n > 0;
    if (ok) {
        ir.resize(n);
        ok = r.ir(prog, ir.data()) == NVRTC_SUCCESS;
    }
    r.destroy(&prog);
    return ok;  // the library stays loaded (cheap; cuFFT may link lazily)
}

std::mutex g_mu;
int g_state = 0;  // 0 untried, 1 IR ready, -1 unavailable
std::vector<char> g_ir;
std::vector<std::string> g_cands;
size_t g_next = 0;

}  // namespace

// cufft plan *p (created here; cufftMakePlanMany64 geometry) with the
// callback `symbol` of kSource (a cufftXtCallbackType) reading d_info
// (its device argument struct).  ws_max != nullptr: no work area of its
// own; *ws_max is raised to the plan's need (the caller sets a shared
// one).  Returns false, with *p = 0, if the callback cannot be linked in
// this process; a failed link moves on to the next NVRTC candidate, and
// once none is left the process stays on the copy / pack-kernel paths.
bool am_callback_plan(cufftHandle* p, int rank, long long* n, long long* inembed, long long istride, long long idist,
                      long long* onembed, long long ostride, long long odist, cufftType type, long long batch,
                      cudaStream_t stream, void* d_info, const char* symbol, int cb_type, size_t* ws_max) {
    std::lock_guard<std::mutex> lk(g_mu);
    *p = 0;
    if (g_state == 0) g_cands = nvrtc_candidates();
    while (g_state >= 0) {
        if (g_state == 0) {  // next NVRTC candidate
            if (g_next >= g_cands.size()) {
                g_state = -1;
                break;
            }
            if (!lto_ir(g_cands[g_next++], g_ir)) continue;
            g_state = 1;
        }
        cufftHandle h = 0;
        size_t ws = 0;
        void* info = d_info;
        bool ok = cufftCreate(&h) == CUFFT_SUCCESS &&
                  (!ws_max || cufftSetAutoAllocation(h, 0) == CUFFT_SUCCESS) &&
                  cufftXtSetJITCallback(h, symbol, g_ir.data(), g_ir.size(), (cufftXtCallbackType)cb_type, &info) ==
                      CUFFT_SUCCESS &&
                  cufftMakePlanMany64(h, rank, n, inembed, istride, idist, onembed, ostride, odist, type, batch,
                                      &ws) == CUFFT_SUCCESS &&
                  cufftSetStream(h, stream) == CUFFT_SUCCESS;
        if (ok) {
            *p = h;
            if (ws_max && ws > *ws_max) *ws_max = ws;
            return true;
        }
        if (h) cufftDestroy(h);
        g_state = 0;  // this IR does not link here: try the next compiler
    }
    return false;
}
