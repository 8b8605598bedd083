// material.cu -- K1: the one-thread-per-voxel fp64 material kernel and its
// C-ABI entry points (am_eval_batch, am_eval_batch_host,
// am_constitutive_host).
//
// Replaces gsmkit.evaluator.evaluate_arrays (evaluator.py:206-248) for
// StrategyConfig(strategy="automatic", integrator="implicit-euler"): each
// thread runs material.cuh's eval_voxel -- reverse AD of the two potentials
// over forward duals, the implicit-Euler Newton, the tangent post-process,
// clamp, stress and consistent tangent -- with all intermediates in
// registers.  Inputs and outputs are read/written through (component
// stride, item stride) pairs so the same kernel serves SoA device fields
// (coalesced: consecutive threads touch consecutive doubles) and the
// reference's AoS host layout on the host-pointer path.
#include <algorithm>
#include <condition_variable>
#include <emmintrin.h>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "k1_kernels.cuh"

namespace am {

// gsm.py:574-602 at B points (AoS); used by the module-level API and the AD
// unit tests.  eps dirs and a dirs are separate sweeps, like rhs_dual /
// rhs_and_jac.
template <class Law>
__global__ void k_constitutive(Law L, int64_t B, const double* eps, const double* a, double* sigma, double* A,
                               double* f, double* dfda, double* dfde) {
    constexpr int m = Law::m;
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= B) return;
    double e[6], s[6], av[m > 0 ? m : 1];
    for (int c = 0; c < 6; ++c) e[c] = eps[6 * b + c];
    for (int c = 0; c < m; ++c) av[c] = a[m * b + c];
    stress_plain(L, e, av, s);
    if (sigma)
        for (int c = 0; c < 6; ++c) sigma[6 * b + c] = s[c];
    if constexpr (m > 0) {
        if (A) {
            auto Av = gen_stress_sweep(L, plain_tup<6>(e, seq<6>{}), plain_tup<m>(av, seq<m>{}));
            sfor<m>([&](auto I) { A[m * b + decltype(I)::value] = get<decltype(I)::value>(Av).v; });
        }
        double fv[m], J[m][m], Je[m][6];
        rhs_jac_a(L, e, av, fv, J);
        rhs_jac_eps(L, e, 1.0, av, Je);
        for (int i = 0; i < m; ++i) {
            if (f) f[m * b + i] = fv[i];
            for (int k = 0; k < m; ++k)
                if (dfda) dfda[(m * b + i) * m + k] = J[i][k];
            for (int k = 0; k < 6; ++k)
                if (dfde) dfde[(m * b + i) * 6 + k] = Je[i][k];
        }
    }
}

// LawOps (gsm.py:412-566) at B points for either strategy: sigma, A, f,
// df/da, df/deps (rhs_and_jacobians, gsm.py:488-518; semi-automatic:
// rhs_jac_generic, gsm.py:463-481) and, with da (B, m, 6), the consistent
// tangent C = stress_and_tangent (gsm.py:520-551); all AoS, any output NULL.
template <class Law>
__global__ void k_lawops(Law L, int64_t B, const double* eps, const double* a, const double* da, double* sigma,
                         double* A, double* f, double* dfda, double* dfde, double* C) {
    constexpr int m = Law::m;
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= B) return;
    double e[6], s[6], av[m > 0 ? m : 1];
    for (int c = 0; c < 6; ++c) e[c] = eps[6 * b + c];
    for (int c = 0; c < m; ++c) av[c] = a[m * b + c];
    stress_plain(L, e, av, s);
    if (sigma)
        for (int c = 0; c < 6; ++c) sigma[6 * b + c] = s[c];
    if (C) {
        double Cv[6][6], s2[6], dav[m > 0 ? m : 1][6];
        for (int k = 0; k < m; ++k)
            for (int j = 0; j < 6; ++j) dav[k][j] = da ? da[(m * b + k) * 6 + j] : 0.0;
        stress_tangent(L, e, av, (m && da) ? dav : nullptr, s2, Cv);
        for (int i = 0; i < 6; ++i)
            for (int j = 0; j < 6; ++j) C[36 * b + 6 * i + j] = Cv[i][j];
    }
    if constexpr (m > 0) {
        if (A) {
            auto Av = gen_stress_sweep(L, plain_tup<6>(e, seq<6>{}), plain_tup<m>(av, seq<m>{}));
            sfor<m>([&](auto I) { A[m * b + decltype(I)::value] = get<decltype(I)::value>(Av).v; });
        }
        if (f || dfda || dfde) {
            double fv[m], J[m][m], Je[m][6];
            if constexpr (is_semi_v<Law>) {
                double J6[m][6];
                L.rhs_jac(e, av, fv, J6, Je);
                for (int i = 0; i < m; ++i) {
                    for (int k = 0; k < 6; ++k) J[i][k] = J6[i][k];
                    J[i][6] = 0.0;
                }
            } else {
                rhs_jac_a(L, e, av, fv, J);
                rhs_jac_eps(L, e, 1.0, av, Je);
            }
            for (int i = 0; i < m; ++i) {
                if (f) f[m * b + i] = fv[i];
                for (int k = 0; k < m; ++k)
                    if (dfda) dfda[(m * b + i) * m + k] = J[i][k];
                for (int k = 0; k < 6; ++k)
                    if (dfde) dfde[(m * b + i) * 6 + k] = Je[i][k];
            }
        }
    }
}

int check_law(const am_law* law) {
    if (!law) return fail(AM_ERR_ARG, "law is NULL");
    if (law->kind != AM_LAW_LINEAR_ELASTIC && law->kind != AM_LAW_MICHEL_SUQUET)
        return fail(AM_ERR_CONFIG, "unknown law kind %d (only LinearElastic and MichelSuquet have device potentials)",
                    law->kind);
    return AM_OK;
}

int check_cfg(const am_cfg* cfg) {
    if (!cfg) return fail(AM_ERR_ARG, "cfg is NULL");
    const bool integ = cfg->integrator == AM_INTEGRATOR_IMPLICIT_EULER || cfg->integrator == AM_INTEGRATOR_ODE12 ||
                       cfg->integrator == AM_INTEGRATOR_ODE23 ||
                       (cfg->integrator == AM_INTEGRATOR_ODE23S && cfg->strategy == AM_STRATEGY_SEMI_AUTOMATIC);
    const bool strat = cfg->strategy == AM_STRATEGY_AUTOMATIC || cfg->strategy == AM_STRATEGY_SEMI_AUTOMATIC ||
                       (cfg->strategy == AM_STRATEGY_CONVENTIONAL && cfg->integrator == AM_INTEGRATOR_IMPLICIT_EULER);
    if (!strat || !integ)
        return fail(AM_ERR_CONFIG,
                    "the device implements the automatic and semi-automatic strategies with integrator "
                    "implicit-euler, ode12 or ode23, ode23s with the semi-automatic strategy, and the "
                    "conventional implicit-Euler route (got strategy %d, integrator %d)",
                    cfg->strategy, cfg->integrator);
    if (cfg->newton_mode != AM_NEWTON_INTERNAL && cfg->newton_mode != AM_NEWTON_STRESS)
        return fail(AM_ERR_CONFIG, "unknown newton mode %d", cfg->newton_mode);
    if (cfg->error_measure != 0 && cfg->error_measure != 1)
        return fail(AM_ERR_CONFIG, "unknown error measure %d", cfg->error_measure);
    if (cfg->max_newton <= 0) return fail(AM_ERR_ARG, "max_newton must be positive");
    if (cfg->integrator != AM_INTEGRATOR_IMPLICIT_EULER && (cfg->max_substeps <= 0 || !(cfg->atol >= 0.0) ||
                                                            !(cfg->rtol >= 0.0)))
        return fail(AM_ERR_ARG, "bad step controller settings");
    return AM_OK;
}

NewtonCfg newton_cfg(const am_cfg* cfg) { return NewtonCfg{cfg->newton_mode, cfg->max_newton, cfg->newton_tol}; }

StepCtl step_ctl(const am_cfg* cfg) {
    StepCtl c;
    c.atol = cfg->atol;
    c.rtol = cfg->rtol;
    c.max_substeps = cfg->max_substeps;
    c.measure = cfg->error_measure;
    return c;
}

void set_controls(KArgs& k, const am_cfg* cfg) {
    k.ncfg = newton_cfg(cfg);
    k.integrator = cfg->integrator;
    k.strategy = cfg->strategy;
    k.sctl = step_ctl(cfg);
}

// Stream-ordered scratch comes from the device's default memory pool; keep
// freed blocks in the pool (release threshold = max) so per-call
// allocations do not return memory to the driver at every synchronisation.
void keep_pool_memory() {
    static std::mutex mu;
    static std::vector<int> done;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(done.begin(), done.end(), dev) != done.end()) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~uint64_t(0);
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done.push_back(dev);
}

// Per-kernel device time of the two-kernel tangent route (am_k1_timing):
// events before the Newton kernel, between the kernels and after the
// tangent kernel, on the launching stream.
namespace {
struct K1Timing {
    bool on = false;
    cudaEvent_t e[3] = {};
    double ms[2] = {0.0, 0.0};
    int64_t launches = 0;
    std::mutex mu;
};
K1Timing& k1_timing() {
    static K1Timing t;
    return t;
}
}  // namespace

void k1_mark(int i, cudaStream_t s) {
    K1Timing& t = k1_timing();
    if (!t.on) return;
    cudaEventRecord(t.e[i], s);
    if (i == 2) {
        float a = 0.f, b = 0.f;
        cudaEventSynchronize(t.e[2]);
        cudaEventElapsedTime(&a, t.e[0], t.e[1]);
        cudaEventElapsedTime(&b, t.e[1], t.e[2]);
        t.ms[0] += a;
        t.ms[1] += b;
        ++t.launches;
    }
}

int launch_material(const am_law* law, const KArgs& k, cudaStream_t s) {
    if (k.B == 0) return AM_OK;
    const bool semi = k.strategy == AM_STRATEGY_SEMI_AUTOMATIC || k.strategy == AM_STRATEGY_CONVENTIONAL;
    if (law->kind == AM_LAW_MICHEL_SUQUET && k.strategy == AM_STRATEGY_CONVENTIONAL) {
        const auto S = SemiLaw<MichelSuquetLaw>::make(law->E, law->nu, law->sigma_Y, law->H, law->eps0_dot,
                                                      law->sigma_d, law->n);
        return launch_conventional(S, k, s);
    }
    if (law->kind == AM_LAW_MICHEL_SUQUET) {
        if (semi)
            return launch_law_ms_semi(SemiLaw<MichelSuquetLaw>::make(law->E, law->nu, law->sigma_Y, law->H,
                                                                     law->eps0_dot, law->sigma_d, law->n),
                                      k, s);
        return launch_law_ms(
            MichelSuquetLaw::make(law->E, law->nu, law->sigma_Y, law->H, law->eps0_dot, law->sigma_d, law->n), k, s);
    }
    if (semi) return launch_law_le_semi(SemiLaw<LinearElasticLaw>::make(law->E, law->nu), k, s);
    return launch_law_le(LinearElasticLaw::make(law->E, law->nu), k, s);
}

int law_m(const am_law* law) { return law->kind == AM_LAW_MICHEL_SUQUET ? 7 : 0; }

}  // namespace am

using namespace am;

extern "C" int am_k1_timing(int enable, double* out) {
    K1Timing& t = k1_timing();
    std::lock_guard<std::mutex> lk(t.mu);
    if (enable >= 0) {
        if (enable && !t.e[0])
            for (auto& e : t.e) AM_CUDA(cudaEventCreate(&e));
        t.on = enable != 0;
        t.ms[0] = t.ms[1] = 0.0;
        t.launches = 0;
    }
    if (out) {
        out[0] = t.ms[0];
        out[1] = t.ms[1];
        out[2] = (double)t.launches;
    }
    return AM_OK;
}

extern "C" int am_eval_batch(const am_law* law, const am_cfg* cfg, int64_t B, const double* eps_n,
                             const double* a_n, const double* eps_np1, const double* dt, double dt_scalar,
                             int want_tangent, double* sigma, double* a_out, double* C, int32_t* newton_iters,
                             int32_t* rejected, uint8_t* status, uint32_t* flags, void* stream) {
    AM_TRY(check_law(law));
    AM_TRY(check_cfg(cfg));
    if (B < 0) return fail(AM_ERR_ARG, "negative batch size");
    const int m = law_m(law);
    if (B > 0 && (!eps_n || !eps_np1 || !sigma || (m && (!a_n || !a_out)) || (want_tangent && !C)))
        return fail(AM_ERR_ARG, "missing array argument");
    KArgs k{};
    k.B = B; k.gidx = nullptr;
    k.eps_n = eps_n; k.a_n = a_n; k.eps_np1 = eps_np1; k.dt = dt; k.dt_scalar = dt_scalar;
    k.le = {B, 1}; k.la = {B, 1}; k.lc = {B, 1};
    k.sigma = sigma; k.a_out = a_out; k.C = want_tangent ? C : nullptr;
    k.iters = newton_iters; k.rejected = rejected; k.status = status; k.flags = flags;
    set_controls(k, cfg);
    return launch_material(law, k, (cudaStream_t)stream);
}

namespace {

// Parallel host memcpy for the staging of pageable host arrays: a small
// persistent pool; run() splits the copies into 1 MiB segments that the
// workers and the caller take in order and returns when all are done.
struct CopyPool {
    struct Seg {
        char* d;
        const char* s;
        size_t n;
    };
    std::vector<std::thread> workers;
    std::mutex mu;
    std::condition_variable cv_work, cv_done;
    std::vector<Seg> jobs;
    size_t idx = 0, remaining = 0;
    bool stop = false;

    void ensure() {
        if (!workers.empty()) return;
        // measured on the B200 boxes (16 vCPUs, tools/e2e_probe.py): 5 workers + the caller
        // saturate the host memory bandwidth the copies share with the DMA
        int n = std::min(5, (int)std::thread::hardware_concurrency() - 1);
        if (const char* e = std::getenv("AM_COPY_THREADS")) n = std::atoi(e);
        n = std::max(0, std::min(n, 16));
        for (int i = 0; i < n; ++i) workers.emplace_back([this] { loop(); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
        cv_work.notify_all();
        for (auto& t : workers) t.join();
    }
    // streaming (non-temporal) stores: the staging buffers are read next by
    // the DMA engine, not by this CPU, and skipping the read-for-ownership
    // of the destination saves a sixth of the host memory traffic of the
    // path (which is host-DRAM bound with pageable inputs)
    static void copy_nt(char* d, const char* s, size_t n) {
        size_t head = (16 - ((uintptr_t)d & 15)) & 15;
        if (head > n) head = n;
        std::memcpy(d, s, head);
        d += head, s += head, n -= head;
        const size_t body = n & ~size_t(63);
        for (size_t o = 0; o < body; o += 64) {
            const __m128i a = _mm_loadu_si128((const __m128i*)(s + o));
            const __m128i b = _mm_loadu_si128((const __m128i*)(s + o + 16));
            const __m128i c = _mm_loadu_si128((const __m128i*)(s + o + 32));
            const __m128i e = _mm_loadu_si128((const __m128i*)(s + o + 48));
            _mm_stream_si128((__m128i*)(d + o), a);
            _mm_stream_si128((__m128i*)(d + o + 16), b);
            _mm_stream_si128((__m128i*)(d + o + 32), c);
            _mm_stream_si128((__m128i*)(d + o + 48), e);
        }
        std::memcpy(d + body, s + body, n - body);
        _mm_sfence();
    }
    void drain(std::unique_lock<std::mutex>& lk) {
        while (idx < jobs.size()) {
            const Seg g = jobs[idx++];
            lk.unlock();
            copy_nt(g.d, g.s, g.n);
            lk.lock();
            if (--remaining == 0) cv_done.notify_all();
        }
    }
    void loop() {
        std::unique_lock<std::mutex> lk(mu);
        for (;;) {
            cv_work.wait(lk, [&] { return stop || idx < jobs.size(); });
            if (stop) return;
            drain(lk);
        }
    }
    static void add(std::vector<Seg>& v, void* d, const void* s, size_t n) {
        constexpr size_t kSeg = size_t(1) << 20;
        for (size_t o = 0; o < n; o += kSeg) v.push_back({(char*)d + o, (const char*)s + o, std::min(kSeg, n - o)});
    }
    void run(std::vector<Seg>& segs) {
        if (segs.empty()) return;
        ensure();
        std::unique_lock<std::mutex> lk(mu);
        jobs.swap(segs);
        idx = 0;
        remaining = jobs.size();
        cv_work.notify_all();
        drain(lk);
        cv_done.wait(lk, [&] { return remaining == 0; });
        jobs.clear();
        segs.clear();
        idx = 0;
    }
};

bool host_pinned(const void* p) {
    if (!p) return true;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// Device staging for the host-pointer path: chunks of 2^17 points cycle
// through three slots / streams so that the H2D copy of one chunk, the
// kernels of another and the D2H copy of a third overlap (the paper's
// two-stream staging, with device-resident buffers reused
// across calls).  The path is PCIe-bound by the D2H of C (288 B/point);
// 3 x 2^17 measured best (tools/e2e_variants.py: 8.67 ms per 2^20 vs
// 9.0-9.2 ms for 2 x 2^18).  Pageable (unregistered) host arrays go through
// pinned per-slot staging buffers, filled / drained by the CopyPool while
// the other slots' DMA runs (a pageable cudaMemcpyAsync would stage
// synchronously and serialise the pipeline).
struct HostPipe {
#ifndef AM_HOST_SLOTS
#define AM_HOST_SLOTS 3
#endif
#ifndef AM_HOST_CHUNK_LOG2
#define AM_HOST_CHUNK_LOG2 17
#endif
    static constexpr int kSlots = AM_HOST_SLOTS;
    int device = -1;
    int64_t cap = 0;
    cudaStream_t stream[kSlots] = {};
    cudaEvent_t done[kSlots] = {};
    double* in[kSlots] = {};     // eps_n | a_n | eps_np1 | dt
    double* out[kSlots] = {};    // sigma | a_out | C
    int32_t* iters[kSlots] = {};
    uint8_t* status[kSlots] = {};
    char* hin[kSlots] = {};      // pinned staging: inputs (20 doubles / point)
    char* hout[kSlots] = {};     // pinned staging: outputs (49 doubles + 2 int32 + 1 byte / point)
    uint32_t* flags = nullptr;   // kSlots words
    CopyPool pool;
    std::mutex mu;

    static constexpr size_t kInBytes = 20 * sizeof(double);
    static constexpr size_t kOutBytes = 49 * sizeof(double) + 2 * sizeof(int32_t) + 1;

    int ensure(int64_t chunk) {
        int dev;
        AM_CUDA(cudaGetDevice(&dev));
        if (dev == device && chunk <= cap) return AM_OK;
        release();
        device = dev;
        for (int s = 0; s < kSlots; ++s) {
            AM_CUDA(cudaStreamCreateWithFlags(&stream[s], cudaStreamNonBlocking));
            AM_CUDA(cudaEventCreateWithFlags(&done[s], cudaEventDisableTiming));
            AM_CUDA(cudaMalloc(&in[s], sizeof(double) * chunk * 20));
            AM_CUDA(cudaMalloc(&out[s], sizeof(double) * chunk * 49));
            AM_CUDA(cudaMalloc(&iters[s], sizeof(int32_t) * 2 * chunk));  // iters | rejected
            AM_CUDA(cudaMalloc(&status[s], chunk));
        }
        AM_CUDA(cudaMalloc(&flags, sizeof(uint32_t) * kSlots));
        cap = chunk;
        return AM_OK;
    }
    int ensure_staging() {
        for (int s = 0; s < kSlots; ++s) {
            if (!hin[s]) AM_CUDA(cudaHostAlloc((void**)&hin[s], kInBytes * cap, cudaHostAllocPortable));
            if (!hout[s]) AM_CUDA(cudaHostAlloc((void**)&hout[s], kOutBytes * cap, cudaHostAllocPortable));
        }
        return AM_OK;
    }
    void release() {
        if (device < 0) return;
        for (int s = 0; s < kSlots; ++s) {
            cudaFree(in[s]); cudaFree(out[s]); cudaFree(iters[s]); cudaFree(status[s]);
            cudaFreeHost(hin[s]); cudaFreeHost(hout[s]);
            if (stream[s]) cudaStreamDestroy(stream[s]);
            if (done[s]) cudaEventDestroy(done[s]);
            in[s] = out[s] = nullptr; iters[s] = nullptr; status[s] = nullptr; stream[s] = nullptr;
            hin[s] = hout[s] = nullptr; done[s] = nullptr;
        }
        cudaFree(flags);
        flags = nullptr;
        cap = 0;
        device = -1;
    }
};

HostPipe& host_pipe() {
    static HostPipe p;
    return p;
}

}  // namespace

extern "C" int am_eval_batch_host(const am_law* law, const am_cfg* cfg, int64_t B, const double* eps_n,
                                  const double* a_n, const double* eps_np1, const double* dt, int want_tangent,
                                  double* sigma, double* a_out, double* C, int32_t* newton_iters,
                                  int32_t* rejected, uint8_t* status) {
    AM_TRY(check_law(law));
    AM_TRY(check_cfg(cfg));
    if (B < 0) return fail(AM_ERR_ARG, "negative batch size");
    if (B == 0) return AM_OK;
    const int m = law_m(law);
    if (!eps_n || !eps_np1 || !dt || !sigma || (m && (!a_n || !a_out)) || (want_tangent && !C))
        return fail(AM_ERR_ARG, "missing array argument");
    HostPipe& P = host_pipe();
    std::lock_guard<std::mutex> lock(P.mu);
    const int64_t chunk = B < (int64_t(1) << AM_HOST_CHUNK_LOG2) ? B : (int64_t(1) << AM_HOST_CHUNK_LOG2);
    AM_TRY(P.ensure(chunk));
    // on every return (including errors) no copy into or out of the
    // caller's arrays is still in flight
    struct Drain {
        HostPipe& p;
        ~Drain() {
            for (int s = 0; s < HostPipe::kSlots; ++s)
                if (p.stream[s]) cudaStreamSynchronize(p.stream[s]);
        }
    } drain_all{P};
    // which host arrays need staging (pageable memory)
    const double* ins[4] = {eps_n, m ? a_n : nullptr, eps_np1, dt};
    const int inw[4] = {6, m, 6, 1};                         // doubles per point
    void* outs[6] = {sigma, m ? a_out : nullptr, want_tangent ? C : nullptr, newton_iters, rejected, status};
    const int outb[6] = {6 * 8, m * 8, 36 * 8, 4, 4, 1};     // bytes per point
    bool stage_in[4], stage_out[6], any_stage = false;
    for (int i = 0; i < 4; ++i) any_stage |= (stage_in[i] = ins[i] && !host_pinned(ins[i]));
    for (int i = 0; i < 6; ++i) any_stage |= (stage_out[i] = outs[i] && !host_pinned(outs[i]));
    if (any_stage) AM_TRY(P.ensure_staging());
    AM_CUDA(cudaMemsetAsync(P.flags, 0, sizeof(uint32_t) * HostPipe::kSlots, P.stream[0]));
    AM_CUDA(cudaStreamSynchronize(P.stream[0]));
    std::vector<CopyPool::Seg> segs;
    int64_t plo[HostPipe::kSlots], pn[HostPipe::kSlots];
    bool live[HostPipe::kSlots] = {};
    // staged outputs of the chunk in slot s -> the caller's arrays
    auto drain = [&](int s) -> int {
        if (!live[s]) return AM_OK;
        AM_CUDA(cudaEventSynchronize(P.done[s]));
        size_t off = 0;
        for (int i = 0; i < 6; ++i) {
            if (!outs[i]) continue;
            const size_t nb = (size_t)outb[i] * pn[s];
            if (stage_out[i]) CopyPool::add(segs, (char*)outs[i] + (size_t)outb[i] * plo[s], P.hout[s] + off, nb);
            off += nb;
        }
        P.pool.run(segs);
        live[s] = false;
        return AM_OK;
    };
    // chunk sizes ramp up from 2^AM_HOST_RAMP_LOG2 so the first D2H starts
    // early (pipeline fill), then stay at `chunk`
#ifndef AM_HOST_RAMP_LOG2
#define AM_HOST_RAMP_LOG2 12
#endif
    int64_t lo = 0, c = 0;
    for (; lo < B; ++c) {
        const int s = int(c % HostPipe::kSlots);
        cudaStream_t st = P.stream[s];
        AM_TRY(drain(s));  // the slot's previous chunk is complete
        int64_t want = chunk;
        if (AM_HOST_RAMP_LOG2 + c < AM_HOST_CHUNK_LOG2) want = int64_t(1) << (AM_HOST_RAMP_LOG2 + c);
        const int64_t n = (B - lo) < want ? (B - lo) : want;
        double* d_in[4];
        d_in[0] = P.in[s];
        d_in[1] = d_in[0] + 6 * n;
        d_in[2] = d_in[1] + 7 * n;
        d_in[3] = d_in[2] + 6 * n;
        // inputs: stage the pageable ones, then H2D
        {
            size_t off = 0;
            const char* src[4];
            for (int i = 0; i < 4; ++i) {
                if (!ins[i]) continue;
                const size_t nb = sizeof(double) * inw[i] * n;
                const char* user = (const char*)(ins[i] + (size_t)inw[i] * lo);
                if (stage_in[i]) {
                    CopyPool::add(segs, P.hin[s] + off, user, nb);
                    src[i] = P.hin[s] + off;
                    off += nb;
                } else {
                    src[i] = user;
                }
            }
            P.pool.run(segs);
            for (int i = 0; i < 4; ++i)
                if (ins[i])
                    AM_CUDA(cudaMemcpyAsync(d_in[i], src[i], sizeof(double) * inw[i] * n, cudaMemcpyHostToDevice, st));
        }
        double* d_sig = P.out[s];
        double* d_ao = d_sig + 6 * n;
        double* d_C = d_ao + 7 * n;
        KArgs k{};
        k.B = n; k.gidx = nullptr;
        k.eps_n = d_in[0]; k.a_n = d_in[1]; k.eps_np1 = d_in[2]; k.dt = d_in[3]; k.dt_scalar = 0.0;
        k.le = {1, 6}; k.la = {1, m}; k.lc = {1, 36};
        k.sigma = d_sig; k.a_out = d_ao; k.C = want_tangent ? d_C : nullptr;
        k.iters = P.iters[s]; k.rejected = P.iters[s] + n; k.status = P.status[s]; k.flags = P.flags + s;
        set_controls(k, cfg);
        AM_TRY(launch_material(law, k, st));
        // outputs: D2H straight into pinned caller arrays, else into the slot's staging
        {
            const void* dsrc[6] = {d_sig, d_ao, d_C, P.iters[s], P.iters[s] + n, P.status[s]};
            size_t off = 0;
            for (int i = 0; i < 6; ++i) {
                if (!outs[i]) continue;
                const size_t nb = (size_t)outb[i] * n;
                void* dst = stage_out[i] ? (void*)(P.hout[s] + off) : (void*)((char*)outs[i] + (size_t)outb[i] * lo);
                AM_CUDA(cudaMemcpyAsync(dst, dsrc[i], nb, cudaMemcpyDeviceToHost, st));
                off += nb;
            }
        }
        AM_CUDA(cudaEventRecord(P.done[s], st));
        plo[s] = lo;
        pn[s] = n;
        live[s] = true;
        lo += n;
    }
    // drain the remaining slots in chunk order
    for (int64_t j = c; j < c + HostPipe::kSlots; ++j) AM_TRY(drain(int(j % HostPipe::kSlots)));
    uint32_t flags[HostPipe::kSlots];
    AM_CUDA(cudaMemcpyAsync(flags, P.flags, sizeof(flags), cudaMemcpyDeviceToHost, P.stream[0]));
    for (int s = 0; s < HostPipe::kSlots; ++s) AM_CUDA(cudaStreamSynchronize(P.stream[s]));
    uint32_t any = 0;
    for (int s = 0; s < HostPipe::kSlots; ++s) any |= flags[s];
    if (any & AM_VOXEL_NEWTON_FAILED)
        return fail(AM_ERR_NEWTON, "implicit Euler Newton failed for at least one voxel");
    if (any & AM_VOXEL_INTEGRATION)
        return fail(AM_ERR_INTEGRATION, "adaptive integration: substep cap or step size underflow");
    if (any & AM_VOXEL_RADIAL) return fail(AM_ERR_RADIAL, "radial return stalled");
    if (any & AM_VOXEL_SINGULAR) return fail(AM_ERR_SINGULAR, "pivot below 1e-14 * max|A|");
    return AM_OK;
}

// record_steps of the adaptive integrators: the same evaluation as
// am_eval_batch_host (no chunking; meant for the reference's step-record
// diagnostics), writing each point's attempts (step size, accepted) to
// rec_h / rec_acc [offsets[b], offsets[b+1]); offsets (B + 1) come from the
// substep + rejected counts of a previous evaluation of the same inputs.
extern "C" int am_eval_batch_record_host(const am_law* law, const am_cfg* cfg, int64_t B, const double* eps_n,
                                         const double* a_n, const double* eps_np1, const double* dt, int want_tangent,
                                         double* sigma, double* a_out, double* C, int32_t* substeps,
                                         int32_t* rejected, const int64_t* offsets, double* rec_h, uint8_t* rec_acc) {
    AM_TRY(check_law(law));
    AM_TRY(check_cfg(cfg));
    if (B <= 0) return B == 0 ? AM_OK : fail(AM_ERR_ARG, "negative batch size");
    const int m = law_m(law);
    if (!eps_n || !eps_np1 || !dt || !sigma || !offsets || !rec_h || !rec_acc || (m && (!a_n || !a_out)) ||
        (want_tangent && !C))
        return fail(AM_ERR_ARG, "missing array argument");
    const int64_t nrec = offsets[B];
    std::vector<void*> bufs;
    auto dalloc = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (cudaMalloc(&p, bytes ? bytes : 1) != cudaSuccess) return nullptr;
        bufs.push_back(p);
        return p;
    };
    auto cleanup = [&]() {
        for (void* p : bufs) cudaFree(p);
    };
    double* d_in = (double*)dalloc(sizeof(double) * B * 20);
    double* d_out = (double*)dalloc(sizeof(double) * B * 49);
    int32_t* d_cnt = (int32_t*)dalloc(sizeof(int32_t) * B * 2);
    uint8_t* d_st = (uint8_t*)dalloc(B);
    int64_t* d_off = (int64_t*)dalloc(sizeof(int64_t) * (B + 1));
    double* d_rh = (double*)dalloc(sizeof(double) * nrec);
    uint8_t* d_ra = (uint8_t*)dalloc(nrec);
    uint32_t* d_fl = (uint32_t*)dalloc(sizeof(uint32_t));
    if (!d_in || !d_out || !d_cnt || !d_st || !d_off || !d_rh || !d_ra || !d_fl) {
        cleanup();
        return fail(AM_ERR_CUDA, "am_eval_batch_record_host: out of device memory");
    }
    double *d_en = d_in, *d_an = d_in + 6 * B, *d_e1 = d_in + 13 * B, *d_dt = d_in + 19 * B;
    double *d_sig = d_out, *d_ao = d_out + 6 * B, *d_C = d_out + 13 * B;
    cudaError_t e = cudaMemcpy(d_en, eps_n, sizeof(double) * 6 * B, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && m) e = cudaMemcpy(d_an, a_n, sizeof(double) * m * B, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_e1, eps_np1, sizeof(double) * 6 * B, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_dt, dt, sizeof(double) * B, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_off, offsets, sizeof(int64_t) * (B + 1), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(d_fl, 0, sizeof(uint32_t));
    if (e != cudaSuccess) {
        cleanup();
        return fail(AM_ERR_CUDA, "am_eval_batch_record_host: %s", cudaGetErrorString(e));
    }
    KArgs k{};
    k.B = B;
    k.eps_n = d_en; k.a_n = d_an; k.eps_np1 = d_e1; k.dt = d_dt;
    k.le = {1, 6}; k.la = {1, m}; k.lc = {1, 36};
    k.sigma = d_sig; k.a_out = d_ao; k.C = want_tangent ? d_C : nullptr;
    k.iters = d_cnt; k.rejected = d_cnt + B; k.status = d_st; k.flags = d_fl;
    k.rec_off = d_off; k.rec_h = d_rh; k.rec_acc = d_ra;
    set_controls(k, cfg);
    int rc = launch_material(law, k, 0);
    uint32_t any = 0;
    if (rc == AM_OK) {
        e = cudaMemcpy(sigma, d_sig, sizeof(double) * 6 * B, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && m) e = cudaMemcpy(a_out, d_ao, sizeof(double) * m * B, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && want_tangent) e = cudaMemcpy(C, d_C, sizeof(double) * 36 * B, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && substeps) e = cudaMemcpy(substeps, d_cnt, sizeof(int32_t) * B, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && rejected) e = cudaMemcpy(rejected, d_cnt + B, sizeof(int32_t) * B, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(rec_h, d_rh, sizeof(double) * nrec, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(rec_acc, d_ra, nrec, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(&any, d_fl, sizeof(any), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) rc = fail(AM_ERR_CUDA, "am_eval_batch_record_host: %s", cudaGetErrorString(e));
    }
    cleanup();
    if (rc != AM_OK) return rc;
    if (any & AM_VOXEL_NEWTON_FAILED) return fail(AM_ERR_NEWTON, "implicit Euler Newton failed for at least one voxel");
    if (any & AM_VOXEL_INTEGRATION) return fail(AM_ERR_INTEGRATION, "adaptive integration: substep cap");
    if (any & AM_VOXEL_SINGULAR) return fail(AM_ERR_SINGULAR, "pivot below 1e-14 * max|A|");
    return AM_OK;
}

extern "C" int am_lawops_host(const am_law* law, int strategy, int64_t B, const double* eps, const double* a,
                              const double* da, double* sigma, double* A, double* f, double* dfda, double* dfde,
                              double* C) {
    AM_TRY(check_law(law));
    if (strategy != AM_STRATEGY_AUTOMATIC && strategy != AM_STRATEGY_SEMI_AUTOMATIC &&
        strategy != AM_STRATEGY_CONVENTIONAL)
        return fail(AM_ERR_CONFIG, "unsupported strategy %d", strategy);
    if (B <= 0) return B == 0 ? AM_OK : fail(AM_ERR_ARG, "negative batch size");
    const int m = law_m(law);
    const bool semi = strategy != AM_STRATEGY_AUTOMATIC;  // _ops_for: conventional -> semi-automatic
    const size_t sz[] = {6, (size_t)m, (size_t)m * 6, 6, (size_t)m, (size_t)m, (size_t)m * m, (size_t)m * 6, 36};
    const double* hin[] = {eps, a, da};
    double* hout[] = {sigma, A, f, dfda, dfde, C};
    std::vector<double*> d(9, nullptr);
    int rc = AM_OK;
    for (int i = 0; i < 9 && rc == AM_OK; ++i) {
        const bool want = i < 3 ? hin[i] != nullptr : hout[i - 3] != nullptr;
        if (want && sz[i] && cudaMalloc(&d[i], sizeof(double) * sz[i] * B) != cudaSuccess)
            rc = fail(AM_ERR_CUDA, "am_lawops_host: out of memory");
        if (rc == AM_OK && i < 3 && d[i] &&
            cudaMemcpy(d[i], hin[i], sizeof(double) * sz[i] * B, cudaMemcpyHostToDevice) != cudaSuccess)
            rc = fail(AM_ERR_CUDA, "am_lawops_host: copy failed");
    }
    if (rc == AM_OK) {
        const unsigned blocks = unsigned((B + 127) / 128);
        auto go = [&](const auto& L) {
            k_lawops<<<blocks, 128>>>(L, B, d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], d[8]);
        };
        if (law->kind == AM_LAW_MICHEL_SUQUET) {
            if (semi)
                go(SemiLaw<MichelSuquetLaw>::make(law->E, law->nu, law->sigma_Y, law->H, law->eps0_dot, law->sigma_d,
                                                  law->n));
            else go(MichelSuquetLaw::make(law->E, law->nu, law->sigma_Y, law->H, law->eps0_dot, law->sigma_d, law->n));
        } else {
            if (semi) go(SemiLaw<LinearElasticLaw>::make(law->E, law->nu));
            else go(LinearElasticLaw::make(law->E, law->nu));
        }
        if (cudaGetLastError() != cudaSuccess) rc = fail(AM_ERR_CUDA, "am_lawops_host: launch failed");
    }
    for (int i = 3; i < 9 && rc == AM_OK; ++i)
        if (d[i] && cudaMemcpy(hout[i - 3], d[i], sizeof(double) * sz[i] * B, cudaMemcpyDeviceToHost) != cudaSuccess)
            rc = fail(AM_ERR_CUDA, "am_lawops_host: kernel failed");
    for (double* p : d) cudaFree(p);
    return rc;
}

extern "C" int am_constitutive_host(const am_law* law, int64_t B, const double* eps, const double* a,
                                    double* sigma, double* A, double* f, double* dfda, double* dfde) {
    AM_TRY(check_law(law));
    if (B <= 0) return B == 0 ? AM_OK : fail(AM_ERR_ARG, "negative batch size");
    const int m = law_m(law);
    const size_t n_in = 6 + m, n_out = 6 + m + m + m * m + 6 * m;
    double *d_in, *d_out;
    AM_CUDA(cudaMalloc(&d_in, sizeof(double) * n_in * B));
    AM_CUDA(cudaMalloc(&d_out, sizeof(double) * n_out * B));
    double* d_e = d_in;
    double* d_a = d_in + 6 * B;
    double* d_s = d_out;
    double* d_A = d_s + 6 * B;
    double* d_f = d_A + m * B;
    double* d_J = d_f + m * B;
    double* d_Je = d_J + m * m * B;
    int rc = AM_OK;
    cudaError_t e = cudaMemcpy(d_e, eps, sizeof(double) * 6 * B, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && m) e = cudaMemcpy(d_a, a, sizeof(double) * m * B, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        const unsigned blocks = unsigned((B + 127) / 128);
        if (law->kind == AM_LAW_MICHEL_SUQUET) {
            auto L = MichelSuquetLaw::make(law->E, law->nu, law->sigma_Y, law->H, law->eps0_dot, law->sigma_d, law->n);
            k_constitutive<<<blocks, 128>>>(L, B, d_e, d_a, d_s, d_A, d_f, d_J, d_Je);
        } else {
            auto L = LinearElasticLaw::make(law->E, law->nu);
            k_constitutive<<<blocks, 128>>>(L, B, d_e, d_a, d_s, d_A, d_f, d_J, d_Je);
        }
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && sigma) e = cudaMemcpy(sigma, d_s, sizeof(double) * 6 * B, cudaMemcpyDeviceToHost);
    if (m) {
        if (e == cudaSuccess && A) e = cudaMemcpy(A, d_A, sizeof(double) * m * B, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && f) e = cudaMemcpy(f, d_f, sizeof(double) * m * B, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && dfda) e = cudaMemcpy(dfda, d_J, sizeof(double) * m * m * B, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && dfde) e = cudaMemcpy(dfde, d_Je, sizeof(double) * 6 * m * B, cudaMemcpyDeviceToHost);
    }
    if (e != cudaSuccess) rc = fail(AM_ERR_CUDA, "am_constitutive_host: %s", cudaGetErrorString(e));
    cudaFree(d_in);
    cudaFree(d_out);
    return rc;
}
