// solver.cu -- the Moulinec-Suquet basic scheme on one GPU (gsmkit
// homogenize.py: Homogenizer, GreenOperator, equilibrium_residual,
// reference_update, apply_isotropic) and its C-ABI (am_solver_*, am_*_host).
//
// Device-resident state (component-major SoA, fp64):
//   eps, eps_n, sigma   (6, N)           strain iterate, committed strain, stress
//   ehat                (6, N^)  cplx    rfft of eps (unnormalised), carried across iterations
//   shat                (6, N^)  cplx    rfft of sigma, then the Z2D input of the update
//   per phase: gidx (Bm) i64, a_n and a_pending (m, Bm)
// with N = nx ny nz, N^ = nx ny (nz/2+1).
//
// One basic-scheme iteration (homogenize.py:445-465):
//   K1   sigma = material(eps_n, a_n, eps)           per phase, gathered by gidx
//   D2Z  shat = rfft(sigma)                          6 batched 3-D transforms
//   K2   residual partials and, for every bin but 0, the update
//        ehat' = -Gamma0 (shat - C0 ehat)          (= rfft of the new fluctuation)
//        written to ehat and, scaled by 1/N, to shat (Z2D input)
//   red  fixed-order sum of the partials; sigma_bar = shat(0)/N; D2H of 8 doubles
//   host convergence test (strict <, homogenize.py:454), mixed-BC update of ebar
//   bin0 ehat(0) = N ebar; Z2D eps = irfft(shat)
// Carrying ehat replaces the reference's FFT of tau = sigma - C0:eps
// (6 forward + 6 inverse transforms per iteration instead of 12 + 6): the
// reference's tau_hat is rfft(sigma) - C0 rfft(eps), and rfft(eps) is the
// previous update plus the mean.
#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "fourier.cuh"
#include "k1.cuh"
#include "laws.cuh"
#include "refupdate.cuh"

namespace am {

#define AM_CUFFT(expr)                                                                      \
    do {                                                                                    \
        cufftResult _r = (expr);                                                            \
        if (_r != CUFFT_SUCCESS) return ::am::fail(AM_ERR_CUDA, "%s:%d %s: cufft error %d", \
                                                   __FILE__, __LINE__, #expr, (int)_r);     \
    } while (0)

struct Vec6 {
    double v[6];
};

constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 148 * 4;  // fixed: the reduction order never depends on the launch

// ---------------------------------------------------------------- kernels
__device__ __forceinline__ double block_sum(double v, double* sh) {
    // deterministic tree: warp shuffle then the warps' partials in order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
    __syncthreads();
    return s;
}

// eps = eps_n + d (start of a loading step, homogenize.py:439)
__global__ void k_shift(double* __restrict__ eps, const double* __restrict__ eps_n, Vec6 d, int64_t N) {
    const int64_t n6 = 6 * N;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n6; i += (int64_t)gridDim.x * blockDim.x)
        eps[i] = eps_n[i] + d.v[i / N];
}

struct Dims {
    int nx, ny, nz, nzh;
    int64_t N, Nh;
};

__device__ __forceinline__ void bin_coords(const Dims& d, int64_t q, int& ix, int& iy, int& iz) {
    iz = (int)(q % d.nzh);
    const int64_t r = q / d.nzh;
    iy = (int)(r % d.ny);
    ix = (int)(r / d.ny);
}

// K2: residual partials + Green update for every bin but the origin.
// shat: rfft(sigma) in, ehat'/N out;  ehat: rfft(eps) in, ehat' out.
__global__ void __launch_bounds__(kRedThreads) k_fourier(Dims d, RefMat ref, cufftDoubleComplex* __restrict__ shat,
                                                         cufftDoubleComplex* __restrict__ ehat, double* __restrict__ partial,
                                                         int update) {
    __shared__ double sh[kRedThreads / 32];
    const double invN = 1.0 / (double)d.N;
    double acc = 0.0;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < d.Nh; q += (int64_t)gridDim.x * blockDim.x) {
        int ix, iy, iz;
        bin_coords(d, q, ix, iy, iz);
        const Bin b = make_bin(ix, iy, iz, d.nx, d.ny, d.nz);
        cplx s[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            const cufftDoubleComplex v = shat[c * d.Nh + q];
            s[c] = cplx{v.x, v.y};
        }
        if (!b.zero) acc += rfft_weight(iz, d.nz) * traction_sq(b, s);
        if (update && !b.zero) {
            double er[6], ei[6], cr[6], ci[6], tr[6], ti[6], outr[6], outi[6];
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                const cufftDoubleComplex v = ehat[c * d.Nh + q];
                er[c] = v.x;
                ei[c] = v.y;
            }
            iso_apply(ref, er, cr);
            iso_apply(ref, ei, ci);
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                tr[c] = s[c].re - cr[c];
                ti[c] = s[c].im - ci[c];
            }
            green_apply_real(ref, b, tr, outr);
            green_apply_real(ref, b, ti, outi);
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                ehat[c * d.Nh + q] = make_cuDoubleComplex(outr[c], outi[c]);
                shat[c * d.Nh + q] = make_cuDoubleComplex(outr[c] * invN, outi[c] * invN);
            }
        }
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// out[0] = sum of partials (fixed order), out[1..6] = Re shat(0) (= N sigma_bar),
// out[7] = material status flags
__global__ void k_finish(const double* __restrict__ partial, int np, const cufftDoubleComplex* __restrict__ shat,
                         int64_t Nh, const uint32_t* __restrict__ flags, double* __restrict__ out) {
    __shared__ double sh[32];
    double v = 0.0;
    for (int i = threadIdx.x; i < np; i += blockDim.x) v += partial[i];
    const double t = block_sum(v, sh);
    if (threadIdx.x == 0) {
        out[0] = t;
        for (int c = 0; c < 6; ++c) out[1 + c] = shat[c * Nh].x;
        out[7] = (double)(flags ? *flags : 0u);
    }
}

// origin bin of the update: ehat(0) = N ebar, Z2D input ebar
__global__ void k_origin(cufftDoubleComplex* shat, cufftDoubleComplex* ehat, int64_t Nh, Vec6 ebar, double N) {
    const int c = threadIdx.x;
    if (c < 6) {
        ehat[c * Nh] = make_cuDoubleComplex(ebar.v[c] * N, 0.0);
        shat[c * Nh] = make_cuDoubleComplex(ebar.v[c], 0.0);
    }
}

// standalone Green application on a spectrum (GreenOperator.apply): every
// bin, the origin -> 0, output scaled by 1/N for the Z2D
__global__ void k_green(Dims d, RefMat ref, cufftDoubleComplex* __restrict__ h) {
    const double invN = 1.0 / (double)d.N;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < d.Nh; q += (int64_t)gridDim.x * blockDim.x) {
        int ix, iy, iz;
        bin_coords(d, q, ix, iy, iz);
        const Bin b = make_bin(ix, iy, iz, d.nx, d.ny, d.nz);
        double tr[6], ti[6], outr[6], outi[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            tr[c] = h[c * d.Nh + q].x;
            ti[c] = h[c * d.Nh + q].y;
        }
        green_apply_real(ref, b, tr, outr);
        green_apply_real(ref, b, ti, outi);
#pragma unroll
        for (int c = 0; c < 6; ++c)
            h[c * d.Nh + q] = b.zero ? make_cuDoubleComplex(0.0, 0.0)
                                     : make_cuDoubleComplex(outr[c] * invN, outi[c] * invN);
    }
}

// C_ref : eps over a (6, N) field
__global__ void k_isotropic(RefMat ref, const double* __restrict__ e, double* __restrict__ out, int64_t N) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        double x[6], y[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) x[c] = e[c * N + i];
        iso_apply(ref, x, y);
#pragma unroll
        for (int c = 0; c < 6; ++c) out[c * N + i] = y[c];
    }
}

// K5: per-voxel tangent bounds + C sums over a chunk of tangents stored
// C[(i*6+j)*cs + b].  Per block: [sum C (36), min kappa, max kappa,
// min mu_lo, max mu_hi, nonfinite count] -> stats[blockIdx * 41 + ...]
constexpr int kStat = 41;
__global__ void __launch_bounds__(kRedThreads) k_refstats(const double* __restrict__ C, int64_t cs, int64_t B,
                                                          DevBasis db, double* __restrict__ stats) {
    __shared__ double sh[kRedThreads / 32];
    __shared__ double red[kRedThreads];
    double sum[36];
#pragma unroll
    for (int i = 0; i < 36; ++i) sum[i] = 0.0;
    double kmin = INFINITY, kmax = -INFINITY, mlo = INFINITY, mhi = -INFINITY, bad = 0.0;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
        double c[6][6];
        bool fin = true;
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
            for (int j = 0; j < 6; ++j) {
                c[i][j] = C[(i * 6 + j) * cs + b];
                sum[i * 6 + j] += c[i][j];
                fin = fin && (c[i][j] - c[i][j] == 0.0);
            }
        if (!fin) {
            bad += 1.0;
            continue;
        }
        double k, lo, hi;
        tangent_bounds(c, db, k, lo, hi);
        kmin = fmin(kmin, k);
        kmax = fmax(kmax, k);
        mlo = fmin(mlo, lo);
        mhi = fmax(mhi, hi);
    }
    double* out = stats + (int64_t)blockIdx.x * kStat;
#pragma unroll 1
    for (int i = 0; i < 36; ++i) {
        const double t = block_sum(sum[i], sh);
        if (threadIdx.x == 0) out[i] = t;
    }
    const double t = block_sum(bad, sh);
    if (threadIdx.x == 0) out[40] = t;
    // min / max are order independent
    double vals[4] = {kmin, -kmax, mlo, -mhi};
#pragma unroll 1
    for (int v = 0; v < 4; ++v) {
        red[threadIdx.x] = vals[v];
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + s]);
            __syncthreads();
        }
        if (threadIdx.x == 0) out[36 + v] = (v & 1) ? -red[0] : red[0];
        __syncthreads();
    }
}

// gather-scatter copy of a phase's C chunk into an (N, 6, 6) field is done on
// the host (API path only)

// ---------------------------------------------------------------- host helpers
static unsigned grid_for(int64_t n, int threads = 256) {
    int64_t b = (n + threads - 1) / threads;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)kSMs * 32));
}

// LAPACK-style dense solve with partial pivoting (numpy.linalg.solve,
// homogenize.py:463) for the <= 6x6 mixed-BC system
static bool small_solve(int n, double* A, double* x) {
    int piv[6];
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (std::fabs(A[i * n + k]) > std::fabs(A[p * n + k])) p = i;
        piv[k] = p;
        if (A[p * n + k] == 0.0) return false;
        if (p != k)
            for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[p * n + j]);
        for (int i = k + 1; i < n; ++i) {
            A[i * n + k] /= A[k * n + k];
            for (int j = k + 1; j < n; ++j) A[i * n + j] -= A[i * n + k] * A[k * n + j];
        }
    }
    for (int k = 0; k < n; ++k)
        if (piv[k] != k) std::swap(x[k], x[piv[k]]);
    for (int i = 1; i < n; ++i)
        for (int k = 0; k < i; ++k) x[i] -= A[i * n + k] * x[k];
    for (int i = n - 1; i >= 0; --i) {
        for (int j = i + 1; j < n; ++j) x[i] -= A[i * n + j] * x[j];
        x[i] /= A[i * n + i];
    }
    return true;
}

static void ref_matrix(double lam, double mu, double* C) {
    for (int i = 0; i < 36; ++i) C[i] = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) C[i * 6 + j] = lam;
    for (int i = 0; i < 3; ++i) C[i * 6 + i] = lam + 2.0 * mu;
    for (int i = 3; i < 6; ++i) C[i * 6 + i] = mu;
}

// ---------------------------------------------------------------- the solver
struct Phase {
    am_law law;
    int m = 0;
    int64_t count = 0;
    int64_t* gidx = nullptr;
    double* a_n = nullptr;
    double* a_pend = nullptr;
};

struct Stats {
    double Csum[36];
    double kmin, kmax, mlo, mhi;
    double bad;
    void reset() {
        for (double& c : Csum) c = 0.0;
        kmin = mlo = INFINITY;
        kmax = mhi = -INFINITY;
        bad = 0.0;
    }
    void add(const double* s) {
        for (int i = 0; i < 36; ++i) Csum[i] += s[i];
        kmin = std::fmin(kmin, s[36]);
        kmax = std::fmax(kmax, s[37]);
        mlo = std::fmin(mlo, s[38]);
        mhi = std::fmax(mhi, s[39]);
        bad += s[40];
    }
};

}  // namespace am

struct am_solver {
    am::Dims d{};
    int device = 0;
    cudaStream_t stream = nullptr;
    am_cfg cfg{};
    std::vector<am::Phase> phases;
    double *eps = nullptr, *eps_n = nullptr, *sigma = nullptr;
    cufftDoubleComplex *shat = nullptr, *ehat = nullptr;
    cufftHandle r2c = 0, c2r = 0;
    double* partial = nullptr;
    double* dsmall = nullptr;
    double* hsmall = nullptr;  // pinned
    uint32_t* flags = nullptr;
    // tangent sweep scratch
    int64_t chunk = 0;
    double* Cbuf = nullptr;
    uint8_t* status = nullptr;
    double* stats = nullptr;
    double* hstats = nullptr;  // pinned
    double lam = 0.0, mu = 0.0;
    double ebar_n[6] = {0, 0, 0, 0, 0, 0};
    double ebar[6] = {0, 0, 0, 0, 0, 0};  // mean strain of the current iterate
    bool pending = false;
    am::DevBasis db = am::DevBasis::make();
    // optional per-phase device timing of solve_step (am_solver_timing)
    bool timing = false;
    cudaEvent_t ev[6] = {};
    double t_ms[5] = {0, 0, 0, 0, 0};  // material, d2z, fourier+reduce, z2d+origin, iterations
};

namespace am {

static int solver_free(am_solver* h) {
    if (!h) return AM_OK;
    cudaSetDevice(h->device);
    for (auto& p : h->phases) {
        cudaFree(p.gidx);
        cudaFree(p.a_n);
        cudaFree(p.a_pend);
    }
    cudaFree(h->eps); cudaFree(h->eps_n); cudaFree(h->sigma);
    cudaFree(h->shat); cudaFree(h->ehat);
    cudaFree(h->partial); cudaFree(h->dsmall); cudaFreeHost(h->hsmall); cudaFree(h->flags);
    cudaFree(h->Cbuf); cudaFree(h->status); cudaFree(h->stats); cudaFreeHost(h->hstats);
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
    if (h->r2c) cufftDestroy(h->r2c);
    if (h->c2r) cufftDestroy(h->c2r);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return AM_OK;
}

// K1 over every phase: sigma field and pending states from (eps_n, a_n, eps)
static int material_sweep(am_solver* h, double dt) {
    AM_CUDA(cudaMemsetAsync(h->flags, 0, sizeof(uint32_t), h->stream));
    for (auto& p : h->phases) {
        if (!p.count) continue;
        KArgs k{};
        k.B = p.count;
        k.gidx = p.gidx;
        k.eps_n = h->eps_n; k.eps_np1 = h->eps; k.a_n = p.a_n; k.dt = nullptr; k.dt_scalar = dt;
        k.le = {h->d.N, 1}; k.la = {p.count, 1}; k.lc = {0, 0};
        k.sigma = h->sigma; k.a_out = p.a_pend; k.C = nullptr;
        k.iters = nullptr; k.status = nullptr; k.flags = h->flags;
        k.ncfg = newton_cfg(&h->cfg);
        AM_TRY(launch_material(&p.law, k, h->stream));
    }
    return AM_OK;
}

static int fft_forward(am_solver* h, double* field, cufftDoubleComplex* out) {
    AM_CUFFT(cufftExecD2Z(h->r2c, field, out));
    return AM_OK;
}

static int fft_inverse(am_solver* h, cufftDoubleComplex* in, double* field) {
    AM_CUFFT(cufftExecZ2D(h->c2r, in, field));
    return AM_OK;
}

// residual of the current sigma (whose rfft is in shat) and, when `update`,
// the Green update of every bin but the origin; returns the 8 host values
static int fourier_pass(am_solver* h, bool update, double* out8) {
    RefMat ref = RefMat::make(h->lam, h->mu);
    k_fourier<<<kRedBlocks, kRedThreads, 0, h->stream>>>(h->d, ref, h->shat, h->ehat, h->partial, update ? 1 : 0);
    AM_CUDA(cudaGetLastError());
    k_finish<<<1, 1024, 0, h->stream>>>(h->partial, kRedBlocks, h->shat, h->d.Nh, h->flags, h->dsmall);
    AM_CUDA(cudaGetLastError());
    AM_CUDA(cudaMemcpyAsync(h->hsmall, h->dsmall, 8 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    AM_CUDA(cudaStreamSynchronize(h->stream));
    std::memcpy(out8, h->hsmall, 8 * sizeof(double));
    return AM_OK;
}

static double dup_norm(const double* s) {
    // sqrt(sigma_bar . SHEAR_DUP . sigma_bar) (homogenize.py:266, 449)
    const double dup[6] = {1, 1, 1, 2, 2, 2};
    double t = 0.0;
    for (int i = 0; i < 6; ++i) t += s[i] * dup[i] * s[i];
    return std::sqrt(t);
}

}  // namespace am

using namespace am;

extern "C" int am_solver_create(int nx, int ny, int nz, const uint8_t* ids, int nmat, const am_law* laws,
                                const am_cfg* cfg, am_solver** out) {
    if (!out || !ids || !laws || nmat <= 0 || nx <= 0 || ny <= 0 || nz <= 0)
        return fail(AM_ERR_ARG, "am_solver_create: bad arguments");
    AM_TRY(check_cfg(cfg));
    for (int i = 0; i < nmat; ++i) AM_TRY(check_law(&laws[i]));
    const int64_t N = (int64_t)nx * ny * nz;
    std::vector<std::vector<int64_t>> idx(nmat);
    for (int64_t i = 0; i < N; ++i) {
        if (ids[i] >= nmat) return fail(AM_ERR_ARG, "material id exceeds material table");
        idx[ids[i]].push_back(i);
    }
    auto* h = new am_solver();
    int rc = AM_OK;
    auto bail = [&](int code) {
        solver_free(h);
        return code;
    };
    if (cudaGetDevice(&h->device) != cudaSuccess) return bail(fail(AM_ERR_CUDA, "no CUDA device"));
    h->d = Dims{nx, ny, nz, nz / 2 + 1, N, (int64_t)nx * ny * (nz / 2 + 1)};
    h->cfg = *cfg;
#define AMC(expr)                                                                                     \
    do {                                                                                              \
        cudaError_t _e = (expr);                                                                      \
        if (_e != cudaSuccess) return bail(fail(AM_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e))); \
    } while (0)
    AMC(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    AMC(cudaMalloc(&h->eps, sizeof(double) * 6 * N));
    AMC(cudaMalloc(&h->eps_n, sizeof(double) * 6 * N));
    AMC(cudaMalloc(&h->sigma, sizeof(double) * 6 * N));
    AMC(cudaMemset(h->eps_n, 0, sizeof(double) * 6 * N));
    AMC(cudaMemset(h->eps, 0, sizeof(double) * 6 * N));
    AMC(cudaMemset(h->sigma, 0, sizeof(double) * 6 * N));
    AMC(cudaMalloc(&h->shat, sizeof(cufftDoubleComplex) * 6 * h->d.Nh));
    AMC(cudaMalloc(&h->ehat, sizeof(cufftDoubleComplex) * 6 * h->d.Nh));
    AMC(cudaMalloc(&h->partial, sizeof(double) * kRedBlocks));
    AMC(cudaMalloc(&h->dsmall, sizeof(double) * 8));
    AMC(cudaMallocHost(&h->hsmall, sizeof(double) * 8));
    AMC(cudaMalloc(&h->flags, sizeof(uint32_t)));
    h->chunk = std::min<int64_t>(N, int64_t(1) << 22);
    AMC(cudaMalloc(&h->Cbuf, sizeof(double) * 36 * h->chunk));
    AMC(cudaMalloc(&h->status, h->chunk));
    AMC(cudaMalloc(&h->stats, sizeof(double) * kStat * kRedBlocks));
    AMC(cudaMallocHost(&h->hstats, sizeof(double) * kStat * kRedBlocks));
    for (int i = 0; i < nmat; ++i) {
        Phase p;
        p.law = laws[i];
        p.m = law_m(&laws[i]);
        p.count = (int64_t)idx[i].size();
        if (p.count) {
            AMC(cudaMalloc(&p.gidx, sizeof(int64_t) * p.count));
            AMC(cudaMemcpy(p.gidx, idx[i].data(), sizeof(int64_t) * p.count, cudaMemcpyHostToDevice));
            if (p.m) {
                AMC(cudaMalloc(&p.a_n, sizeof(double) * p.m * p.count));
                AMC(cudaMalloc(&p.a_pend, sizeof(double) * p.m * p.count));
                AMC(cudaMemset(p.a_n, 0, sizeof(double) * p.m * p.count));
                AMC(cudaMemset(p.a_pend, 0, sizeof(double) * p.m * p.count));
            }
        }
        h->phases.push_back(p);
    }
#undef AMC
    long long n3[3] = {nx, ny, nz};
    size_t ws = 0;
    if (cufftCreate(&h->r2c) != CUFFT_SUCCESS || cufftCreate(&h->c2r) != CUFFT_SUCCESS)
        return bail(fail(AM_ERR_CUDA, "cufftCreate failed"));
    if (cufftMakePlanMany64(h->r2c, 3, n3, nullptr, 1, N, nullptr, 1, h->d.Nh, CUFFT_D2Z, 6, &ws) != CUFFT_SUCCESS ||
        cufftMakePlanMany64(h->c2r, 3, n3, nullptr, 1, h->d.Nh, nullptr, 1, N, CUFFT_Z2D, 6, &ws) != CUFFT_SUCCESS)
        return bail(fail(AM_ERR_CUDA, "cufft plan creation failed for %dx%dx%d", nx, ny, nz));
    cufftSetStream(h->r2c, h->stream);
    cufftSetStream(h->c2r, h->stream);
    *out = h;
    return rc;
}

extern "C" int am_solver_destroy(am_solver* h) { return solver_free(h); }

extern "C" int am_solver_set_reference(am_solver* h, double lam, double mu) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    h->lam = lam;
    h->mu = mu;
    return AM_OK;
}

extern "C" int am_solver_get_reference(am_solver* h, double* lam, double* mu) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    *lam = h->lam;
    *mu = h->mu;
    return AM_OK;
}

extern "C" int am_solver_set_mean(am_solver* h, const double* ebar_n) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    std::memcpy(h->ebar_n, ebar_n, sizeof(h->ebar_n));
    return AM_OK;
}

extern "C" int am_solver_solve_step(am_solver* h, const double* ebar_target, double dt, const uint8_t* free_mask,
                                    double tol, int max_iterations, am_stepinfo* info, double* history,
                                    int history_cap) {
    if (!h || !ebar_target || !info) return fail(AM_ERR_ARG, "am_solver_solve_step: bad arguments");
    AM_CUDA(cudaSetDevice(h->device));
    const Dims& d = h->d;
    bool free[6];
    int nf = 0, fi[6];
    for (int i = 0; i < 6; ++i) {
        free[i] = free_mask ? free_mask[i] != 0 : false;
        if (free[i]) fi[nf++] = i;
    }
    double ebar[6];
    for (int i = 0; i < 6; ++i) ebar[i] = free[i] ? h->ebar_n[i] : ebar_target[i];  // homogenize.py:436-437
    Vec6 shift;
    for (int i = 0; i < 6; ++i) shift.v[i] = ebar[i] - h->ebar_n[i];
    k_shift<<<grid_for(6 * d.N), 256, 0, h->stream>>>(h->eps, h->eps_n, shift, d.N);
    AM_CUDA(cudaGetLastError());
    AM_TRY(fft_forward(h, h->eps, h->ehat));
    double Cff[36];
    {
        double C0[36];
        ref_matrix(h->lam, h->mu, C0);
        for (int a = 0; a < nf; ++a)
            for (int b = 0; b < nf; ++b) Cff[a * nf + b] = C0[fi[a] * 6 + fi[b]];
    }
    info->iterations = 0;
    info->converged = 0;
    info->residual = 0.0;
    info->mean_substeps = 1.0;  // implicit Euler: one substep per voxel (evaluator.py:130)
    const double Nd = (double)d.N;
    auto mark = [&](int i) -> int {
        if (h->timing) AM_CUDA(cudaEventRecord(h->ev[i], h->stream));
        return AM_OK;
    };
    auto acc = [&](int a, int b, int slot) -> int {
        float ms = 0.f;
        AM_CUDA(cudaEventElapsedTime(&ms, h->ev[a], h->ev[b]));
        h->t_ms[slot] += ms;
        return AM_OK;
    };
    for (int it = 1; it <= max_iterations; ++it) {
        AM_TRY(mark(0));
        AM_TRY(material_sweep(h, dt));
        AM_TRY(mark(1));
        AM_TRY(fft_forward(h, h->sigma, h->shat));
        AM_TRY(mark(2));
        double o[8];
        AM_TRY(fourier_pass(h, true, o));  // synchronises the stream
        if (h->timing) {
            AM_CUDA(cudaEventRecord(h->ev[3], h->stream));
            AM_CUDA(cudaEventSynchronize(h->ev[3]));
            AM_TRY(acc(0, 1, 0));
            AM_TRY(acc(1, 2, 1));
            AM_TRY(acc(2, 3, 2));
            h->t_ms[4] += 1.0;
        }
        if ((uint32_t)o[7] & AM_VOXEL_NEWTON_FAILED) {
            info->iterations = it;
            return fail(AM_ERR_NEWTON, "implicit Euler Newton failed for at least one voxel (iteration %d)", it);
        }
        double sbar[6];
        for (int i = 0; i < 6; ++i) sbar[i] = o[1 + i] / Nd;
        // equilibrium_residual (homogenize.py:264-267)
        const double scale = std::max(dup_norm(sbar), 1e-300);
        const double res = std::sqrt(o[0] / (Nd * Nd)) / scale;
        double res_bc = 0.0;
        if (nf) {
            double t = 0.0;
            for (int a = 0; a < nf; ++a) t += sbar[fi[a]] * sbar[fi[a]];
            res_bc = std::sqrt(t) / scale;
        }
        const double hres = std::max(res, res_bc);
        if (history && it <= history_cap) history[it - 1] = hres;
        info->iterations = it;
        info->residual = hres;
        for (int i = 0; i < 6; ++i) {
            info->ebar[i] = ebar[i];
            info->sig_bar[i] = sbar[i];
        }
        if (res < tol && res_bc < tol) {  // strict (homogenize.py:454)
            info->converged = 1;
            h->pending = true;
            std::memcpy(h->ebar, ebar, sizeof(ebar));
            return AM_OK;
        }
        if (nf) {  // mixed BC (homogenize.py:462-464)
            double A[36], x[6];
            std::memcpy(A, Cff, sizeof(double) * nf * nf);
            for (int a = 0; a < nf; ++a) x[a] = -sbar[fi[a]];
            if (!small_solve(nf, A, x)) return fail(AM_ERR_SINGULAR, "singular reference block");
            for (int a = 0; a < nf; ++a) ebar[fi[a]] += x[a];
        }
        Vec6 eb;
        for (int i = 0; i < 6; ++i) eb.v[i] = ebar[i];
        AM_TRY(mark(4));
        k_origin<<<1, 32, 0, h->stream>>>(h->shat, h->ehat, d.Nh, eb, Nd);
        AM_CUDA(cudaGetLastError());
        AM_TRY(fft_inverse(h, h->shat, h->eps));
        if (h->timing) {
            AM_TRY(mark(5));
            AM_CUDA(cudaEventSynchronize(h->ev[5]));
            AM_TRY(acc(4, 5, 3));
        }
    }
    std::memcpy(h->ebar, ebar, sizeof(ebar));
    return fail(AM_ERR_NOT_CONVERGED, "basic scheme did not converge in %d iterations (last residual %.3e)",
                max_iterations, info->residual);
}

// eps_n <- eps, ebar_n <- ebar, a_n <- pending (homogenize.py:474-480)
extern "C" int am_solver_commit(am_solver* h, const double* ebar) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    AM_CUDA(cudaSetDevice(h->device));
    AM_CUDA(cudaMemcpyAsync(h->eps_n, h->eps, sizeof(double) * 6 * h->d.N, cudaMemcpyDeviceToDevice, h->stream));
    if (ebar) std::memcpy(h->ebar_n, ebar, sizeof(h->ebar_n));
    if (h->pending) {
        for (auto& p : h->phases) std::swap(p.a_n, p.a_pend);
        h->pending = false;
    }
    AM_CUDA(cudaStreamSynchronize(h->stream));
    return AM_OK;
}

// material evaluation of the current eps field (Homogenizer.evaluate_field,
// homogenize.py:389-421) without tangent: sigma field + pending states
extern "C" int am_solver_evaluate(am_solver* h, double dt) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    AM_CUDA(cudaSetDevice(h->device));
    AM_TRY(material_sweep(h, dt));
    uint32_t f = 0;
    AM_CUDA(cudaMemcpyAsync(&f, h->flags, sizeof(f), cudaMemcpyDeviceToHost, h->stream));
    AM_CUDA(cudaStreamSynchronize(h->stream));
    h->pending = true;
    if (f & AM_VOXEL_NEWTON_FAILED) return fail(AM_ERR_NEWTON, "implicit Euler Newton failed for at least one voxel");
    return AM_OK;
}

// Tangent sweep of the current eps from the committed state (the
// evaluate_field(want_tangent=True) of run_loading_path, homogenize.py:509)
// fused with reference_update (homogenize.py:307-329): C is produced in
// chunks, reduced to C_bar (36) and the spectral bounds, and never stored
// as a field unless C_out (N, 6, 6, host) is given.  Also refreshes sigma and
// the pending states.  lam_mu (optional) receives reference_update's result.
extern "C" int am_solver_tangent_sweep(am_solver* h, double dt, double* Cbar, double* lam_mu, double* C_out) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    AM_CUDA(cudaSetDevice(h->device));
    Stats st;
    st.reset();
    uint32_t any = 0;
    AM_CUDA(cudaMemsetAsync(h->flags, 0, sizeof(uint32_t), h->stream));
    std::vector<double> hC;
    std::vector<int64_t> hidx;
    for (auto& p : h->phases) {
        if (!p.count) continue;
        if (C_out) {
            hidx.resize(p.count);
            AM_CUDA(cudaMemcpy(hidx.data(), p.gidx, sizeof(int64_t) * p.count, cudaMemcpyDeviceToHost));
        }
        for (int64_t lo = 0; lo < p.count; lo += h->chunk) {
            const int64_t n = std::min(h->chunk, p.count - lo);
            KArgs k{};
            k.B = n;
            k.gidx = p.gidx + lo;
            k.eps_n = h->eps_n; k.eps_np1 = h->eps;
            k.a_n = p.m ? p.a_n + lo : nullptr;
            k.dt = nullptr; k.dt_scalar = dt;
            k.le = {h->d.N, 1}; k.la = {p.count, 1}; k.lc = {n, 1};
            k.sigma = h->sigma; k.a_out = p.m ? p.a_pend + lo : nullptr; k.C = h->Cbuf;
            k.iters = nullptr; k.status = h->status; k.flags = h->flags;
            k.ncfg = newton_cfg(&h->cfg);
            AM_TRY(launch_material(&p.law, k, h->stream));
            k_refstats<<<kRedBlocks, kRedThreads, 0, h->stream>>>(h->Cbuf, n, n, h->db, h->stats);
            AM_CUDA(cudaGetLastError());
            AM_CUDA(cudaMemcpyAsync(h->hstats, h->stats, sizeof(double) * kStat * kRedBlocks, cudaMemcpyDeviceToHost,
                                    h->stream));
            if (C_out) {
                hC.resize((size_t)36 * n);
                AM_CUDA(cudaMemcpyAsync(hC.data(), h->Cbuf, sizeof(double) * 36 * n, cudaMemcpyDeviceToHost, h->stream));
            }
            AM_CUDA(cudaStreamSynchronize(h->stream));
            for (int b = 0; b < kRedBlocks; ++b) st.add(h->hstats + (size_t)b * kStat);
            if (C_out)
                for (int64_t b = 0; b < n; ++b)
                    for (int e = 0; e < 36; ++e) C_out[hidx[lo + b] * 36 + e] = hC[(size_t)e * n + b];
        }
    }
    AM_CUDA(cudaMemcpy(&any, h->flags, sizeof(any), cudaMemcpyDeviceToHost));
    h->pending = true;
    if (any & AM_VOXEL_NEWTON_FAILED) return fail(AM_ERR_NEWTON, "implicit Euler Newton failed for at least one voxel");
    if (Cbar)
        for (int i = 0; i < 36; ++i) Cbar[i] = st.Csum[i] / (double)h->d.N;
    if (st.bad > 0.0 || (any & AM_VOXEL_NONFINITE))
        return fail(AM_ERR_NONFINITE, "tangent field contains non-finite entries");
    if (any & AM_VOXEL_SINGULAR) return fail(AM_ERR_SINGULAR, "pivot below 1e-14 * max|A| in the tangent LU");
    if (lam_mu) {
        const double mu_ref = 0.5 * (st.mlo + st.mhi);
        const double kappa_ref = 0.5 * (st.kmin + st.kmax);
        lam_mu[0] = kappa_ref - 2.0 * mu_ref / 3.0;
        lam_mu[1] = mu_ref;
    }
    return AM_OK;
}

// which: 0 eps, 1 eps_n, 2 sigma; host layout (6, nx, ny, nz)
static double* field_ptr(am_solver* h, int which) {
    return which == 0 ? h->eps : which == 1 ? h->eps_n : which == 2 ? h->sigma : nullptr;
}

extern "C" int am_solver_get_field(am_solver* h, int which, double* out) {
    if (!h || !out || !field_ptr(h, which)) return fail(AM_ERR_ARG, "am_solver_get_field: bad arguments");
    AM_CUDA(cudaSetDevice(h->device));
    AM_CUDA(cudaStreamSynchronize(h->stream));
    AM_CUDA(cudaMemcpy(out, field_ptr(h, which), sizeof(double) * 6 * h->d.N, cudaMemcpyDeviceToHost));
    return AM_OK;
}

extern "C" int am_solver_set_field(am_solver* h, int which, const double* in) {
    if (!h || !in || !field_ptr(h, which)) return fail(AM_ERR_ARG, "am_solver_set_field: bad arguments");
    AM_CUDA(cudaSetDevice(h->device));
    AM_CUDA(cudaStreamSynchronize(h->stream));
    AM_CUDA(cudaMemcpy(field_ptr(h, which), in, sizeof(double) * 6 * h->d.N, cudaMemcpyHostToDevice));
    return AM_OK;
}

// per-phase state, host AoS (count, m); pending = 0 committed, 1 pending
extern "C" int am_solver_get_state(am_solver* h, int phase, int pending, double* out) {
    if (!h || phase < 0 || phase >= (int)h->phases.size()) return fail(AM_ERR_ARG, "bad phase");
    const Phase& p = h->phases[phase];
    if (!p.m || !p.count) return AM_OK;
    std::vector<double> soa((size_t)p.m * p.count);
    AM_CUDA(cudaSetDevice(h->device));
    AM_CUDA(cudaStreamSynchronize(h->stream));
    AM_CUDA(cudaMemcpy(soa.data(), pending ? p.a_pend : p.a_n, sizeof(double) * soa.size(), cudaMemcpyDeviceToHost));
    for (int64_t b = 0; b < p.count; ++b)
        for (int c = 0; c < p.m; ++c) out[b * p.m + c] = soa[(size_t)c * p.count + b];
    return AM_OK;
}

extern "C" int am_solver_set_state(am_solver* h, int phase, const double* in) {
    if (!h || phase < 0 || phase >= (int)h->phases.size()) return fail(AM_ERR_ARG, "bad phase");
    const Phase& p = h->phases[phase];
    if (!p.m || !p.count) return AM_OK;
    std::vector<double> soa((size_t)p.m * p.count);
    for (int64_t b = 0; b < p.count; ++b)
        for (int c = 0; c < p.m; ++c) soa[(size_t)c * p.count + b] = in[b * p.m + c];
    AM_CUDA(cudaSetDevice(h->device));
    AM_CUDA(cudaStreamSynchronize(h->stream));
    AM_CUDA(cudaMemcpy(p.a_n, soa.data(), sizeof(double) * soa.size(), cudaMemcpyHostToDevice));
    return AM_OK;
}

extern "C" int am_solver_phase_count(am_solver* h, int phase, int64_t* count) {
    if (!h || phase < 0 || phase >= (int)h->phases.size()) return fail(AM_ERR_ARG, "bad phase");
    *count = h->phases[phase].count;
    return AM_OK;
}

// Per-phase device time of solve_step iterations (CUDA events on the solver
// stream): out[0..4] = ms in material sweeps, D2Z, Fourier kernel +
// reduction, origin + Z2D, and the number of iterations timed.  enable:
// 1 on (resets the accumulators), 0 off, -1 query only.
extern "C" int am_solver_timing(am_solver* h, int enable, double* out) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    AM_CUDA(cudaSetDevice(h->device));
    if (enable >= 0) {
        if (enable && !h->ev[0])
            for (auto& e : h->ev) AM_CUDA(cudaEventCreate(&e));
        h->timing = enable != 0;
        for (double& t : h->t_ms) t = 0.0;
    }
    if (out)
        for (int i = 0; i < 5; ++i) out[i] = h->t_ms[i];
    return AM_OK;
}

extern "C" int am_solver_synchronize(am_solver* h) {
    if (!h) return fail(AM_ERR_ARG, "null solver");
    AM_CUDA(cudaStreamSynchronize(h->stream));
    return AM_OK;
}

extern "C" int am_solver_stream(am_solver* h, void** stream) {
    if (!h || !stream) return fail(AM_ERR_ARG, "bad arguments");
    *stream = (void*)h->stream;
    return AM_OK;
}

// ---------------------------------------------------------------- standalone field operators
// GreenOperator(dims, ref).apply(tau) (homogenize.py:229-233), host (6,nx,ny,nz)
extern "C" int am_green_apply_host(int nx, int ny, int nz, double lam, double mu, const double* tau, double* out) {
    if (nx <= 0 || ny <= 0 || nz <= 0 || !tau || !out) return fail(AM_ERR_ARG, "am_green_apply_host: bad arguments");
    const int64_t N = (int64_t)nx * ny * nz, Nh = (int64_t)nx * ny * (nz / 2 + 1);
    double* f = nullptr;
    cufftDoubleComplex* c = nullptr;
    cufftHandle p1 = 0, p2 = 0;
    int rc = AM_OK;
    long long n3[3] = {nx, ny, nz};
    size_t ws;
    if (cudaMalloc(&f, sizeof(double) * 6 * N) != cudaSuccess || cudaMalloc(&c, sizeof(cufftDoubleComplex) * 6 * Nh) != cudaSuccess)
        rc = fail(AM_ERR_CUDA, "am_green_apply_host: out of memory");
    if (rc == AM_OK && (cufftCreate(&p1) != CUFFT_SUCCESS || cufftCreate(&p2) != CUFFT_SUCCESS ||
                        cufftMakePlanMany64(p1, 3, n3, nullptr, 1, N, nullptr, 1, Nh, CUFFT_D2Z, 6, &ws) != CUFFT_SUCCESS ||
                        cufftMakePlanMany64(p2, 3, n3, nullptr, 1, Nh, nullptr, 1, N, CUFFT_Z2D, 6, &ws) != CUFFT_SUCCESS))
        rc = fail(AM_ERR_CUDA, "am_green_apply_host: cufft plan failed");
    if (rc == AM_OK && cudaMemcpy(f, tau, sizeof(double) * 6 * N, cudaMemcpyHostToDevice) != cudaSuccess)
        rc = fail(AM_ERR_CUDA, "copy failed");
    if (rc == AM_OK && cufftExecD2Z(p1, f, c) != CUFFT_SUCCESS) rc = fail(AM_ERR_CUDA, "D2Z failed");
    if (rc == AM_OK) {
        Dims d{nx, ny, nz, nz / 2 + 1, N, Nh};
        k_green<<<grid_for(Nh), 256>>>(d, RefMat::make(lam, mu), c);
        if (cudaGetLastError() != cudaSuccess) rc = fail(AM_ERR_CUDA, "k_green launch failed");
    }
    if (rc == AM_OK && cufftExecZ2D(p2, c, f) != CUFFT_SUCCESS) rc = fail(AM_ERR_CUDA, "Z2D failed");
    if (rc == AM_OK && cudaMemcpy(out, f, sizeof(double) * 6 * N, cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = fail(AM_ERR_CUDA, "copy failed");
    if (p1) cufftDestroy(p1);
    if (p2) cufftDestroy(p2);
    cudaFree(f);
    cudaFree(c);
    return rc;
}

// equilibrium_residual(sig) (homogenize.py:241-267), host (6,nx,ny,nz)
extern "C" int am_equilibrium_residual_host(int nx, int ny, int nz, const double* sig, double* res) {
    if (nx <= 0 || ny <= 0 || nz <= 0 || !sig || !res) return fail(AM_ERR_ARG, "bad arguments");
    const int64_t N = (int64_t)nx * ny * nz, Nh = (int64_t)nx * ny * (nz / 2 + 1);
    double *f = nullptr, *part = nullptr, *small = nullptr;
    cufftDoubleComplex* c = nullptr;
    cufftHandle p1 = 0;
    int rc = AM_OK;
    long long n3[3] = {nx, ny, nz};
    size_t ws;
    if (cudaMalloc(&f, sizeof(double) * 6 * N) != cudaSuccess ||
        cudaMalloc(&c, sizeof(cufftDoubleComplex) * 6 * Nh) != cudaSuccess ||
        cudaMalloc(&part, sizeof(double) * kRedBlocks) != cudaSuccess || cudaMalloc(&small, sizeof(double) * 8) != cudaSuccess)
        rc = fail(AM_ERR_CUDA, "out of memory");
    if (rc == AM_OK && (cufftCreate(&p1) != CUFFT_SUCCESS ||
                        cufftMakePlanMany64(p1, 3, n3, nullptr, 1, N, nullptr, 1, Nh, CUFFT_D2Z, 6, &ws) != CUFFT_SUCCESS))
        rc = fail(AM_ERR_CUDA, "cufft plan failed");
    if (rc == AM_OK && cudaMemcpy(f, sig, sizeof(double) * 6 * N, cudaMemcpyHostToDevice) != cudaSuccess)
        rc = fail(AM_ERR_CUDA, "copy failed");
    if (rc == AM_OK && cufftExecD2Z(p1, f, c) != CUFFT_SUCCESS) rc = fail(AM_ERR_CUDA, "D2Z failed");
    double o[8];
    if (rc == AM_OK) {
        Dims d{nx, ny, nz, nz / 2 + 1, N, Nh};
        k_fourier<<<kRedBlocks, kRedThreads>>>(d, RefMat::make(1.0, 1.0), c, nullptr, part, 0);
        k_finish<<<1, 1024>>>(part, kRedBlocks, c, Nh, nullptr, small);
        if (cudaMemcpy(o, small, sizeof(o), cudaMemcpyDeviceToHost) != cudaSuccess) rc = fail(AM_ERR_CUDA, "failed");
    }
    if (rc == AM_OK) {
        // the reference's sigma_bar is the voxel mean; rfft(sigma)(0) / N
        double sbar[6];
        for (int i = 0; i < 6; ++i) sbar[i] = o[1 + i] / (double)N;
        *res = std::sqrt(o[0] / ((double)N * (double)N)) / std::max(dup_norm(sbar), 1e-300);
    }
    if (p1) cufftDestroy(p1);
    cudaFree(f); cudaFree(c); cudaFree(part); cudaFree(small);
    return rc;
}

// apply_isotropic(ref, eps) (homogenize.py:270-281), host (6, N)
extern "C" int am_apply_isotropic_host(int64_t N, double lam, double mu, const double* eps, double* out) {
    if (N < 0 || (N && (!eps || !out))) return fail(AM_ERR_ARG, "bad arguments");
    if (!N) return AM_OK;
    double* f;
    AM_CUDA(cudaMalloc(&f, sizeof(double) * 12 * N));
    int rc = AM_OK;
    if (cudaMemcpy(f, eps, sizeof(double) * 6 * N, cudaMemcpyHostToDevice) != cudaSuccess) rc = fail(AM_ERR_CUDA, "copy");
    if (rc == AM_OK) {
        k_isotropic<<<grid_for(N), 256>>>(RefMat::make(lam, mu), f, f + 6 * N, N);
        if (cudaMemcpy(out, f + 6 * N, sizeof(double) * 6 * N, cudaMemcpyDeviceToHost) != cudaSuccess)
            rc = fail(AM_ERR_CUDA, "copy");
    }
    cudaFree(f);
    return rc;
}

// reference_update(C_field) (homogenize.py:307-329), host (n, 6, 6)
extern "C" int am_reference_update_host(int64_t n, const double* C, double* lam, double* mu) {
    if (n <= 0 || !C || !lam || !mu) return fail(AM_ERR_ARG, "reference_update needs at least one tangent");
    double *d = nullptr, *stats = nullptr;
    AM_CUDA(cudaMalloc(&d, sizeof(double) * 36 * n));
    int rc = AM_OK;
    std::vector<double> soa((size_t)36 * n), hs((size_t)kStat * kRedBlocks);
    for (int64_t b = 0; b < n; ++b)
        for (int e = 0; e < 36; ++e) soa[(size_t)e * n + b] = C[b * 36 + e];
    if (cudaMalloc(&stats, sizeof(double) * kStat * kRedBlocks) != cudaSuccess) rc = fail(AM_ERR_CUDA, "oom");
    if (rc == AM_OK && cudaMemcpy(d, soa.data(), sizeof(double) * soa.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        rc = fail(AM_ERR_CUDA, "copy");
    if (rc == AM_OK) {
        k_refstats<<<kRedBlocks, kRedThreads>>>(d, n, n, DevBasis::make(), stats);
        if (cudaMemcpy(hs.data(), stats, sizeof(double) * hs.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
            rc = fail(AM_ERR_CUDA, "reference_update kernel failed");
    }
    if (rc == AM_OK) {
        Stats st;
        st.reset();
        for (int b = 0; b < kRedBlocks; ++b) st.add(hs.data() + (size_t)b * kStat);
        if (st.bad > 0.0) {
            rc = fail(AM_ERR_NONFINITE, "tangent field contains non-finite entries");
        } else {
            const double mu_ref = 0.5 * (st.mlo + st.mhi);
            const double kappa_ref = 0.5 * (st.kmin + st.kmax);
            *lam = kappa_ref - 2.0 * mu_ref / 3.0;
            *mu = mu_ref;
        }
    }
    cudaFree(d);
    cudaFree(stats);
    return rc;
}
