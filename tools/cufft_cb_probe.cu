// Does a cuFFT LTO load callback on the basic scheme's Z2D (reading the
// carried spectrum scaled by 1/N, so k_fourier need not write a scaled copy
// that the transform then destroys) cost less than the copy it saves?
// Times the batch-6 3-D Z2D plain vs with the callback, and the plan time.
// build: nvcc -gencode arch=compute_100a,code=lto_100a -dc -fatbin tools/cufft_cb_cb.cu -o /tmp/cb.fatbin
//        nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/cufft_cb_probe.cu -lcufft -o /tmp/cbp
// usage: /tmp/cbp /tmp/cb.fatbin [n]
#include <cufftXt.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                              \
    do {                                                                   \
        auto rc_ = (x);                                                    \
        if (rc_ != 0) {                                                    \
            std::printf("%s:%d error %d\n", __FILE__, __LINE__, (int)rc_); \
            std::exit(1);                                                  \
        }                                                                  \
    } while (0)

struct CbInfo {
    const double2* carry;
    double inv_n;
};

static float time_z2d(cufftHandle p, double2* c, double* r) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) CK(cufftExecZ2D(p, c, r));
    cudaEventRecord(a);
    const int n = 20;
    for (int i = 0; i < n; ++i) CK(cufftExecZ2D(p, c, r));
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / n;
}

__global__ void scale_copy(const double2* __restrict__ in, double2* __restrict__ out, long long n, double s) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double2 v = in[i];
        out[i] = make_double2(v.x * s, v.y * s);
    }
}

int main(int argc, char** argv) {
    FILE* f = std::fopen(argv[1], "rb");
    if (!f) return 1;
    std::vector<char> fat;
    char buf[65536];
    size_t k;
    while ((k = std::fread(buf, 1, sizeof buf, f)) > 0) fat.insert(fat.end(), buf, buf + k);
    std::fclose(f);
    const long long n = argc > 2 ? atoll(argv[2]) : 256;
    const long long N = n * n * n, Nh = n * n * (n / 2 + 1);
    long long n3[3] = {n, n, n};
    double2 *carry, *scr;
    double* real;
    CK(cudaMalloc(&carry, sizeof(double2) * 6 * Nh));
    CK(cudaMalloc(&scr, sizeof(double2) * 6 * Nh));
    CK(cudaMalloc(&real, sizeof(double) * 6 * N));
    CK(cudaMemset(carry, 0, sizeof(double2) * 6 * Nh));
    CK(cudaMemset(scr, 0, sizeof(double2) * 6 * Nh));
    size_t ws;
    cufftHandle plain, cb;
    auto t0 = std::chrono::steady_clock::now();
    CK(cufftCreate(&plain));
    CK(cufftMakePlanMany64(plain, 3, n3, nullptr, 1, Nh, nullptr, 1, N, CUFFT_Z2D, 6, &ws));
    auto t1 = std::chrono::steady_clock::now();
    CbInfo hinfo{carry, 1.0 / double(N)};
    CbInfo* dinfo;
    CK(cudaMalloc(&dinfo, sizeof(CbInfo)));
    CK(cudaMemcpy(dinfo, &hinfo, sizeof hinfo, cudaMemcpyHostToDevice));
    CK(cufftCreate(&cb));
    void* ci = dinfo;
    CK(cufftXtSetJITCallback(cb, "cb_load_scaled", fat.data(), fat.size(), CUFFT_CB_LD_COMPLEX_DOUBLE, &ci));
    CK(cufftMakePlanMany64(cb, 3, n3, nullptr, 1, Nh, nullptr, 1, N, CUFFT_Z2D, 6, &ws));
    auto t2 = std::chrono::steady_clock::now();
    float tp = time_z2d(plain, scr, real);
    float tc = time_z2d(cb, scr, real);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) scale_copy<<<148 * 8, 256>>>(carry, scr, 6 * Nh, 1.0 / double(N));
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) scale_copy<<<148 * 8, 256>>>(carry, scr, 6 * Nh, 1.0 / double(N));
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float tcopy;
    cudaEventElapsedTime(&tcopy, a, b);
    std::printf("{\"n\": %lld, \"plan_plain_s\": %.3f, \"plan_callback_s\": %.3f, \"z2d_plain_ms\": %.4f, "
                "\"z2d_callback_ms\": %.4f, \"scaled_copy_kernel_ms\": %.4f}\n",
                n, std::chrono::duration<double>(t1 - t0).count(), std::chrono::duration<double>(t2 - t1).count(), tp,
                tc, tcopy / 20);
    return 0;
}
