// k1_kernels.cuh -- the K1 kernel templates and their launch logic, shared by
// the per-law translation units (k1_*.cu; split so nvcc compiles the heavy
// instantiations in parallel).  See material.cu for the C-ABI.
#pragma once

#include <algorithm>

#include "adaptive.cuh"
#include "common.cuh"
#include "conventional.cuh"
#include "k1.cuh"
#include "material.cuh"

namespace am {

// default-pool release threshold (material.cu)
void keep_pool_memory();
void k1_mark(int i, cudaStream_t s);  // am_k1_timing events (material.cu)

// writes C[i][j] of item `off` to C[(i * 6 + j) * cs + off]
struct GlobalSink {
    double* C;
    int64_t cs, off;
    bool finite = true;
    __device__ void col(int j, const double* c) {
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            C[(i * 6 + j) * cs + off] = c[i];
            finite = finite && (c[i] - c[i] == 0.0);
        }
    }
};

// K1: one thread per material point, grid-stride, all intermediates in
// registers.  Two phases (material.cuh):
//   k_material<Law, Mode, Raw>  Newton (+ clamp + stress unless Raw).  With
//                               Raw the unclamped state goes to a_out for
//                               the tangent phase.
//   k_tangent<Law>              tangent post-process + clamp + stress + C.
// Mode = Newton convergence measure; each combination is its own
// instantiation so the hot Newton loop carries no dead code
// (instruction-cache footprint).  The Newton kernel runs best at 3 CTAs per
// SM (168 registers), the tangent kernel with the full 255-register budget
// (tools/k1_variants.py measurements).
#ifndef AM_K1_MINB_N
#define AM_K1_MINB_N 3
#endif
#ifndef AM_K1_MINB_T
#define AM_K1_MINB_T 1
#endif

struct PointIO {
    const KArgs& k;
    int64_t b, eo, ao;
    __device__ PointIO(const KArgs& k_, int64_t b_) : k(k_), b(b_) {
        const int64_t g = k.gidx ? k.gidx[b] : b;
        eo = g * k.le.es;
        ao = b * k.la.es;
    }
    // with the gather index already loaded (prefetched by the caller)
    __device__ PointIO(const KArgs& k_, int64_t b_, int64_t g) : k(k_), b(b_) {
        eo = g * k.le.es;
        ao = b * k.la.es;
    }
    __device__ void eps(double* en, double* ep) const {
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            en[c] = __ldg(k.eps_n + c * k.le.cs + eo);
            ep[c] = __ldg(k.eps_np1 + c * k.le.cs + eo);
        }
    }
    template <int m>
    __device__ void load_a(const double* src, double* a) const {
#pragma unroll
        for (int c = 0; c < m; ++c) a[c] = src[c * k.la.cs + ao];
    }
    template <int m>
    __device__ void store_a(const double* a) const {
#pragma unroll
        for (int c = 0; c < m; ++c) k.a_out[c * k.la.cs + ao] = a[c];
    }
    __device__ void store_sigma(const double* sig) const {
#pragma unroll
        for (int c = 0; c < 6; ++c) k.sigma[c * k.le.cs + eo] = sig[c];
    }
    __device__ double dt() const { return k.dt ? __ldg(k.dt + b) : k.dt_scalar; }
    __device__ void status(int st) const {
        if (k.status) k.status[b] = (uint8_t)st;
        if (st && k.flags) atomicOr(k.flags, (uint32_t)st);
    }
};

#ifndef AM_GS_WAVES
#define AM_GS_WAVES 16
#endif
#ifndef AM_GS_PREFETCH
#define AM_GS_PREFETCH 0
#endif
#ifndef AM_TAN_WAVES
#define AM_TAN_WAVES 0
#endif
#ifndef AM_TAN_PREFETCH
#define AM_TAN_PREFETCH 0
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
template <class Law, int Mode, bool Raw>
__global__ void __launch_bounds__(128, AM_K1_MINB_N) k_material(Law L, KArgs k) {
    constexpr int m = Law::m;
    constexpr int ms = m > 0 ? m : 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    // gathered (solver) launches: the next point's gather index is loaded
    // while this point is evaluated (one dependent-load latency fewer)
    int64_t gnext = (k.gidx && b < k.B) ? k.gidx[b] : b;
    for (; b < k.B; b += stride) {
        const int64_t g = gnext;
        if (k.gidx && b + stride < k.B) {
            gnext = k.gidx[b + stride];
            if (AM_GS_PREFETCH) {  // the next point's inputs into L2 (no registers held)
#pragma unroll
                for (int c = 0; c < 6; ++c) {
                    prefetch_l2(k.eps_n + c * k.le.cs + gnext * k.le.es);
                    prefetch_l2(k.eps_np1 + c * k.le.cs + gnext * k.le.es);
                }
#pragma unroll
                for (int c = 0; c < m; ++c) prefetch_l2(k.a_n + c * k.la.cs + (b + stride) * k.la.es);
            }
        }
        const PointIO io(k, b, k.gidx ? g : b);
        double en[6], ep[6], an[ms], a[ms];
        io.eps(en, ep);
        io.load_a<m>(k.a_n, an);
        int it = 0;
        // warm start (solver option): the previous basic-scheme iterate
        double as[ms];
        const bool warm = !Raw && k.a_start;
        if (warm) io.load_a<m>(k.a_start, as);
        const int st = newton_point<Law, Mode>(L, k.ncfg, en, an, ep, io.dt(), a, it, warm ? as : nullptr);
        if constexpr (Raw) {
            io.store_a<m>(a);
        } else {
            double ac[ms], sig[6];
            stress_point(L, ep, a, ac, sig);
            io.store_sigma(sig);
            io.store_a<m>(ac);
        }
        if (k.iters) k.iters[b] = it;
        io.status(st);
    }
}

// reads the unclamped state from a_out and the Newton status from status
template <class Law>
__global__ void __launch_bounds__(128, AM_K1_MINB_T) k_tangent(Law L, KArgs k) {
    constexpr int m = Law::m;
    constexpr int ms = m > 0 ? m : 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < k.B; b += stride) {
        if (AM_TAN_PREFETCH && b + stride < k.B) {  // the next point's inputs into L2
            const int64_t bn = b + stride;
            const int64_t gn = k.gidx ? k.gidx[bn] : bn;
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                prefetch_l2(k.eps_n + c * k.le.cs + gn * k.le.es);
                prefetch_l2(k.eps_np1 + c * k.le.cs + gn * k.le.es);
            }
#pragma unroll
            for (int c = 0; c < m; ++c) prefetch_l2(k.a_out + c * k.la.cs + bn * k.la.es);
        }
        const PointIO io(k, b);
        double en[6], ep[6], a[ms], ac[ms], sig[6];
        io.eps(en, ep);
        if constexpr (m > 0) io.load_a<m>(k.a_out, a);
        int st = (m > 0) ? k.status[b] : 0;
        GlobalSink sink{k.C, k.lc.cs, b * k.lc.es};
        if (st & ST_NEWTON) failed_point(L, ep, a, ac, sig, sink);
        else st |= tangent_point(L, en, ep, io.dt(), a, ac, sig, sink);
        if (!sink.finite) st |= ST_NONFINITE;
        io.store_sigma(sig);
        io.store_a<m>(ac);
        io.status(st);
    }
}

// adaptive explicit integrators (odeint.py:636-756): one thread per point;
// substeps -> iters, rejected attempts -> rejected.  Coupled = tangent.
template <class Law, int Scheme, bool Coupled>
__global__ void __launch_bounds__(128) k_adaptive(Law L, KArgs k) {
    constexpr int m = Law::m;
    constexpr int ms = m > 0 ? m : 1;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < k.B; b += (int64_t)gridDim.x * blockDim.x) {
        const PointIO io(k, b);
        double en[6], ep[6], an[ms], a[ms], ac[ms], sig[6], da[ms][6];
        io.eps(en, ep);
        io.load_a<m>(k.a_n, an);
        const double dt = io.dt();
        int sub = 1, rej = 0, st = 0;
        GlobalSink sink{k.C, k.lc.cs, b * k.lc.es};
        if (dt == 0.0) {  // frozen (evaluator.py:142-150): a_n, elastic tangent, no clamp
            for (int i = 0; i < m; ++i) ac[i] = an[i];
            stress_plain(L, ep, an, sig);
            if (Coupled) {
                double C[6][6], s2[6];
                stress_tangent(L, ep, an, nullptr, s2, C);
                put_all(sink, C);
            }
        } else {
            double* rh = k.rec_h ? k.rec_h + k.rec_off[b] : nullptr;
            uint8_t* ra = k.rec_h ? k.rec_acc + k.rec_off[b] : nullptr;
            st = adaptive_point<Law, Scheme, Coupled>(L, k.sctl, en, an, ep, dt, a, da, sub, rej, rh, ra);
            clamp_state<Law>(a, ac);  // evaluator.py:198
            if (Coupled) {
                double C[6][6];
                stress_tangent(L, ep, ac, da, sig, C);  // evaluator.py:200
                put_all(sink, C);
            } else {
                stress_plain(L, ep, ac, sig);
            }
        }
        if (Coupled && !sink.finite) st |= ST_NONFINITE;
        io.store_sigma(sig);
        io.store_a<m>(ac);
        if (k.iters) k.iters[b] = sub;
        if (k.rejected) k.rejected[b] = rej;
        if (k.sub_sum) {  // warp sum, one atomic per warp (integer: order independent)
            const unsigned mask = __activemask();
            const unsigned v = __reduce_add_sync(mask, (unsigned)sub);
            if ((threadIdx.x & 31) == (unsigned)(__ffs(mask) - 1)) atomicAdd(k.sub_sum, (unsigned long long)v);
        }
        io.status(st);
    }
}

// coupled adaptive integration (ode12 / ode23 with tangent) by 6-lane groups
// (adaptive.cuh adaptive_point_lanes): 5 points per warp, lane j of a group
// advances and writes column j of the tangent; lane 0 writes the rest.
#ifndef AM_LANES_MINB
#define AM_LANES_MINB 1
#endif
template <class Law, int Scheme>
__global__ void __launch_bounds__(128, AM_LANES_MINB) k_adaptive_lanes(Law L, KArgs k) {
    constexpr int m = Law::m;
    const int lane = threadIdx.x & 31;
    const int grp = lane / 6;
    if (grp >= 5) return;  // lanes 30, 31 idle (never part of a group mask)
    const int j = lane - 6 * grp, gbase = 6 * grp;
    const unsigned gmask = 0x3Fu << gbase;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = warp * 5 + grp; b < k.B; b += nwarps * 5) {
        const PointIO io(k, b);
        double en[6], ep[6], an[m], a[m], ac[m], sig[6], dacol[m], ccol[6];
        io.eps(en, ep);
        io.load_a<m>(k.a_n, an);
        const double dt = io.dt();
        int sub = 1, rej = 0, st = 0;
        if (dt == 0.0) {  // frozen (evaluator.py:142-150): a_n, elastic tangent, no clamp
            for (int i = 0; i < m; ++i) ac[i] = an[i];
            if constexpr (is_semi_v<Law>) semi_stress_tangent_cols(L, ep, an, nullptr, 1, j, sig, ccol);
            else stress_dual_lane(L, ep, 1.0, j, an, nullptr, sig, ccol);
        } else {
            double* rh = k.rec_h ? k.rec_h + k.rec_off[b] : nullptr;
            uint8_t* ra = k.rec_h ? k.rec_acc + k.rec_off[b] : nullptr;
            double* gs = nullptr;
            if constexpr (AM_LANES_SMEM) {
                extern __shared__ double lanes_smem[];
                gs = lanes_smem + threadIdx.x;  // slice of this thread, stride blockDim.x
            }
            st = adaptive_point_lanes<Law, Scheme>(L, k.sctl, en, an, ep, dt, a, dacol, sub, rej, j, gmask, gbase, rh,
                                                   ra, gs, (int)blockDim.x);
            clamp_state<Law>(a, ac);  // evaluator.py:198
            // evaluator.py:200 (semi-automatic: the hand-coded tangent, gsm.py:553-560)
            if constexpr (is_semi_v<Law>) semi_stress_tangent_cols(L, ep, ac, dacol, 1, j, sig, ccol);
            else stress_dual_lane(L, ep, 1.0, j, ac, dacol, sig, ccol);
        }
        bool fin = true;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            k.C[(i * 6 + j) * k.lc.cs + b * k.lc.es] = ccol[i];
            fin = fin && (ccol[i] - ccol[i] == 0.0);
        }
        if (__any_sync(gmask, !fin)) st |= ST_NONFINITE;
        if (k.sub_sum) {  // one add per group (integer: order independent)
            const unsigned mask = __activemask();
            const unsigned v = __reduce_add_sync(mask, j == 0 ? (unsigned)sub : 0u);
            if ((threadIdx.x & 31) == (unsigned)(__ffs(mask) - 1)) atomicAdd(k.sub_sum, (unsigned long long)v);
        }
        if (j == 0) {
            io.store_sigma(sig);
            io.store_a<m>(ac);
            if (k.iters) k.iters[b] = sub;
            if (k.rejected) k.rejected[b] = rej;
            io.status(st);
        }
    }
}

// strategy="conventional" (evaluator.py:172-174): radial return of the
// Michel-Suquet law; frozen points use the semi-automatic operations
// (evaluator.py:128, 142-150)
template <bool Tangent>
__global__ void __launch_bounds__(128) k_conventional(SemiLaw<MichelSuquetLaw> S, KArgs k) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < k.B; b += (int64_t)gridDim.x * blockDim.x) {
        const PointIO io(k, b);
        double en[6], ep[6], an[7], a[7], sig[6], C[6][6];
        io.eps(en, ep);
        io.load_a<7>(k.a_n, an);
        const double dt = io.dt();
        int st = 0;
        if (dt == 0.0) {
            for (int i = 0; i < 7; ++i) a[i] = an[i];
            stress_plain(S, ep, an, sig);
            if (Tangent) S.Ce(C);
        } else {
            st = conventional_point(S, ep, an, dt, sig, a, Tangent ? C : nullptr);
        }
        if (Tangent) {
            GlobalSink sink{k.C, k.lc.cs, b * k.lc.es};
            put_all(sink, C);
            if (!sink.finite) st |= ST_NONFINITE;
        }
        io.store_sigma(sig);
        io.store_a<7>(a);
        if (k.iters) k.iters[b] = 1;
        if (k.rejected) k.rejected[b] = 0;
        io.status(st);
    }
}

#ifndef AM_ADAPT_LANES
#define AM_ADAPT_LANES 1
#endif
#ifndef AM_LANES_ROS
#define AM_LANES_ROS 0
#endif
template <class Law, int Scheme>
int launch_adaptive(const Law& L, const KArgs& k, unsigned g, cudaStream_t s) {
    // lane groups for ode23 (automatic): 26.3 vs 21.0 M evals/s (internal
    // measure), 12.9 vs 8.6 (stress); ode12's unrolled one-thread kernel
    // stays faster (12.3 vs 7.1) -- k1_variants.log, round 2
    if (k.C && AM_ADAPT_LANES && (Scheme == 23 || (Scheme == 32 && AM_LANES_ROS))) {
        int64_t blocks = (k.B + 19) / 20;  // 4 warps x 5 points
        if (blocks > (int64_t)kSMs * 512) blocks = (int64_t)kSMs * 512;
        const size_t smem = AM_LANES_SMEM ? sizeof(double) * 2 * Tableau<Scheme>::s * Law::m * 128 : 0;
        if (smem > 48 * 1024) {
            static bool opted = false;  // per instantiation and process (the attribute is per function)
            if (!opted) {
                AM_CUDA(cudaFuncSetAttribute(k_adaptive_lanes<Law, Scheme>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
                opted = true;
            }
        }
        k_adaptive_lanes<Law, Scheme><<<(unsigned)blocks, 128, smem, s>>>(L, k);
    } else if (k.C) k_adaptive<Law, Scheme, true><<<g, 128, 0, s>>>(L, k);
    else k_adaptive<Law, Scheme, false><<<g, 128, 0, s>>>(L, k);
    AM_CUDA(cudaGetLastError());
    return AM_OK;
}

// adaptive integrators of one law (k1_adapt_*.cu)
int launch_adaptive_law(const MichelSuquetLaw& L, const KArgs& k, unsigned g, cudaStream_t s);
int launch_adaptive_law(const SemiLaw<MichelSuquetLaw>& L, const KArgs& k, unsigned g, cudaStream_t s);

template <class Law>
int launch_law(const Law& L, KArgs k, cudaStream_t s) {
    const int threads = 128;
    int64_t blocks = (k.B + threads - 1) / threads;
    if (blocks > (int64_t)kSMs * 1024) blocks = (int64_t)kSMs * 1024;
    const unsigned g = (unsigned)blocks;
    const bool stress = k.ncfg.mode == AM_NEWTON_STRESS;
    if constexpr (Law::m > 0) {
        if (k.integrator == AM_INTEGRATOR_ODE23 || k.integrator == AM_INTEGRATOR_ODE12 ||
            k.integrator == AM_INTEGRATOR_ODE23S)
            return launch_adaptive_law(L, k, g, s);  // k1_adapt_*.cu
    }
    if (!k.C) {
        unsigned gg = g;
        if (AM_GS_WAVES && k.gidx && gg > (unsigned)(kSMs * AM_K1_MINB_N * AM_GS_WAVES))
            gg = (unsigned)(kSMs * AM_K1_MINB_N * AM_GS_WAVES);  // grid-stride: the gidx prefetch pays
        if (stress) k_material<Law, 1, false><<<gg, threads, 0, s>>>(L, k);
        else k_material<Law, 0, false><<<gg, threads, 0, s>>>(L, k);
        AM_CUDA(cudaGetLastError());
        return AM_OK;
    }
    // tangent: Newton (raw state) then the tangent phase; the Newton status
    // travels through `status` (a stream-ordered scratch when the caller
    // does not want it)
    uint8_t* scratch = nullptr;
    if (Law::m > 0 && !k.status) {
        keep_pool_memory();
        AM_CUDA(cudaMallocAsync((void**)&scratch, (size_t)k.B, s));
        k.status = scratch;
    }
    k1_mark(0, s);
    if (Law::m > 0) {
        KArgs kn = k;
        kn.flags = nullptr;  // the tangent kernel reports the combined status
        if (stress) k_material<Law, 1, true><<<g, threads, 0, s>>>(L, kn);
        else k_material<Law, 0, true><<<g, threads, 0, s>>>(L, kn);
        AM_CUDA(cudaGetLastError());
    }
    k1_mark(1, s);
    unsigned gt = g;
    if (AM_TAN_WAVES && gt > (unsigned)(kSMs * 2 * AM_TAN_WAVES)) gt = (unsigned)(kSMs * 2 * AM_TAN_WAVES);
    k_tangent<Law><<<gt, threads, 0, s>>>(L, k);
    AM_CUDA(cudaGetLastError());
    k1_mark(2, s);
    if (scratch) AM_CUDA(cudaFreeAsync(scratch, s));
    return AM_OK;
}

// per-law launchers (k1_*.cu)
int launch_law_ms(const MichelSuquetLaw& L, const KArgs& k, cudaStream_t s);
int launch_law_ms_semi(const SemiLaw<MichelSuquetLaw>& L, const KArgs& k, cudaStream_t s);
int launch_law_le(const LinearElasticLaw& L, const KArgs& k, cudaStream_t s);
int launch_law_le_semi(const SemiLaw<LinearElasticLaw>& L, const KArgs& k, cudaStream_t s);
int launch_conventional(const SemiLaw<MichelSuquetLaw>& S, const KArgs& k, cudaStream_t s);

}  // namespace am
