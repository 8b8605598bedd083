// cuFFT timing of the layouts considered for the basic scheme's spectral
// step (tools experiment, not product code):
//   3d      3-D D2Z / Z2D, batch 6 (the current solver)
//   2d      2-D (y, z) D2Z / Z2D, batch 6 nx, natural layout (c, x, ky, kz)
//   2d_col  2-D (y, z) with the spectrum column-major: (ky, kz, c, x), i.e.
//           odist = 1, ostride = 6 nx (x-lines contiguous for the fused x pass)
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fft_layout_probe.cu -lcufft -o /tmp/fftp
#include <cufft.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                              \
    do {                                                                   \
        auto rc_ = (x);                                                      \
        if (rc_ != 0) {                                                    \
            std::printf("%s:%d error %d\n", __FILE__, __LINE__, (int)rc_); \
            std::exit(1);                                                  \
        }                                                                  \
    } while (0)

static float time_exec(cufftHandle p, bool fwd, double* r, double2* c) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) CK(fwd ? cufftExecD2Z(p, r, c) : cufftExecZ2D(p, c, r));
    cudaEventRecord(a);
    const int n = 10;
    for (int i = 0; i < n; ++i) CK(fwd ? cufftExecD2Z(p, r, c) : cufftExecZ2D(p, c, r));
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / n;
}

int main(int argc, char** argv) {
    const long long n = argc > 1 ? atoll(argv[1]) : 256;
    const long long nx = n, ny = n, nz = n, nzh = nz / 2 + 1;
    const long long N = nx * ny * nz, Nh = nx * ny * nzh;
    double* r;
    double2* c;
    CK(cudaMalloc(&r, sizeof(double) * 6 * N));
    CK(cudaMalloc(&c, sizeof(double2) * 6 * Nh));
    CK(cudaMemset(r, 0, sizeof(double) * 6 * N));
    size_t ws;
    {
        cufftHandle f, i;
        long long d3[3] = {nx, ny, nz};
        CK(cufftCreate(&f));
        CK(cufftCreate(&i));
        CK(cufftMakePlanMany64(f, 3, d3, nullptr, 1, N, nullptr, 1, Nh, CUFFT_D2Z, 6, &ws));
        CK(cufftMakePlanMany64(i, 3, d3, nullptr, 1, Nh, nullptr, 1, N, CUFFT_Z2D, 6, &ws));
        std::printf("3d      D2Z %.3f ms  Z2D %.3f ms\n", time_exec(f, true, r, c), time_exec(i, false, r, c));
        cufftDestroy(f);
        cufftDestroy(i);
    }
    {
        cufftHandle f, i;
        long long d2[2] = {ny, nz};
        CK(cufftCreate(&f));
        CK(cufftCreate(&i));
        CK(cufftMakePlanMany64(f, 2, d2, nullptr, 1, ny * nz, nullptr, 1, ny * nzh, CUFFT_D2Z, 6 * nx, &ws));
        CK(cufftMakePlanMany64(i, 2, d2, nullptr, 1, ny * nzh, nullptr, 1, ny * nz, CUFFT_Z2D, 6 * nx, &ws));
        std::printf("2d      D2Z %.3f ms  Z2D %.3f ms\n", time_exec(f, true, r, c), time_exec(i, false, r, c));
        cufftDestroy(f);
        cufftDestroy(i);
    }
    {
        cufftHandle f, i;
        long long d2[2] = {ny, nz};
        long long inr[2] = {ny, nz}, onc[2] = {ny, nzh};
        CK(cufftCreate(&f));
        CK(cufftCreate(&i));
        CK(cufftMakePlanMany64(f, 2, d2, inr, 1, ny * nz, onc, 6 * nx, 1, CUFFT_D2Z, 6 * nx, &ws));
        CK(cufftMakePlanMany64(i, 2, d2, onc, 6 * nx, 1, inr, 1, ny * nz, CUFFT_Z2D, 6 * nx, &ws));
        std::printf("2d_col  D2Z %.3f ms  Z2D %.3f ms\n", time_exec(f, true, r, c), time_exec(i, false, r, c));
        cufftDestroy(f);
        cufftDestroy(i);
    }
    // 1-D x transforms over the natural 2-D layout (the cuFFT x pass)
    {
        cufftHandle x1;
        long long d1[1] = {nx};
        const long long bx = ny * nzh;
        CK(cufftCreate(&x1));
        for (int cc = 0; cc < 1; ++cc)
            CK(cufftMakePlanMany64(x1, 1, d1, d1, bx, 1, d1, bx, 1, CUFFT_Z2Z, bx, &ws));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int k = 0; k < 3; ++k)
            for (int cc = 0; cc < 6; ++cc) CK(cufftExecZ2Z(x1, c + cc * nx * bx, c + cc * nx * bx, CUFFT_FORWARD));
        cudaEventRecord(a);
        for (int k = 0; k < 10; ++k)
            for (int cc = 0; cc < 6; ++cc) CK(cufftExecZ2Z(x1, c + cc * nx * bx, c + cc * nx * bx, CUFFT_FORWARD));
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        std::printf("x-pass  Z2Z (6 components) %.3f ms\n", ms / 10);
    }
    std::printf("bytes of one spectrum pass (read + write): %.3f GB\n", 2.0 * 16 * 6 * Nh / 1e9);
    return 0;
}
