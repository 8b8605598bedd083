// Can the slab algorithm's pack (2-D spectra -> x-pencil layout of every
// destination slab) ride on the 2-D D2Z as a store callback?  Times, for k
// local slabs of an n^3 grid: the batch-6 nxl 2-D D2Z per slab + a pack
// copy kernel, vs the D2Z with the store callback writing the packed layout.
// build: nvcc -gencode arch=compute_100a,code=lto_100a -dc -fatbin tools/cufft_cb_pack_cb.cu -o /tmp/pk.fatbin
//        nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/cufft_cb_pack_probe.cu -lcufft -o /tmp/pkp
// usage: /tmp/pkp /tmp/pk.fatbin [n] [slabs]
#include <cufftXt.h>
#include <cuda_runtime.h>

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

struct PackCb {
    double2* const* peer;
    unsigned nzh, ny, nxl, nyl;
    unsigned long long blk;
    unsigned rank;
};

__global__ void k_pack(const double2* __restrict__ P, double2* const* __restrict__ peer, int rank, int nxl, int ny,
                       int nzh, int nyl) {
    const int run = blockIdx.y;  // (j, xl, c)
    const int c = run % 6, xl = (run / 6) % nxl, j = run / (6 * nxl);
    const long long len = (long long)nyl * nzh, blk = (long long)nxl * 6 * len;
    const double2* src = P + ((long long)(c * nxl + xl) * ny + (long long)j * nyl) * nzh;
    double2* dst = peer[j] + rank * blk + (long long)(xl * 6 + c) * len;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main(int argc, char** argv) {
    FILE* f = std::fopen(argv[1], "rb");
    std::vector<char> fat;
    char buf[65536];
    size_t r;
    while ((r = std::fread(buf, 1, sizeof buf, f)) > 0) fat.insert(fat.end(), buf, buf + r);
    std::fclose(f);
    const int n = argc > 2 ? atoi(argv[2]) : 256, k = argc > 3 ? atoi(argv[3]) : 8;
    const int nxl = n / k, nyl = n / k, nzh = n / 2 + 1;
    const long long spec = 6LL * nxl * n * nzh;  // complex elements per slab
    std::vector<double*> R(k);
    std::vector<double2*> P(k), S(k);
    for (int s = 0; s < k; ++s) {
        CK(cudaMalloc(&R[s], sizeof(double) * 6LL * nxl * n * n));
        CK(cudaMalloc(&P[s], sizeof(double2) * spec));
        CK(cudaMalloc(&S[s], sizeof(double2) * spec));
        CK(cudaMemset(R[s], 0, sizeof(double) * 6LL * nxl * n * n));
    }
    double2** dpeer;
    CK(cudaMalloc(&dpeer, sizeof(double2*) * k));
    CK(cudaMemcpy(dpeer, S.data(), sizeof(double2*) * k, cudaMemcpyHostToDevice));
    long long n2[2] = {n, n};
    size_t ws;
    cufftHandle plain;
    CK(cufftCreate(&plain));
    CK(cufftMakePlanMany64(plain, 2, n2, nullptr, 1, (long long)n * n, nullptr, 1, (long long)n * nzh, CUFFT_D2Z,
                           6LL * nxl, &ws));
    std::vector<cufftHandle> cb(k);
    for (int s = 0; s < k; ++s) {
        PackCb h{dpeer, (unsigned)nzh, (unsigned)n, (unsigned)nxl, (unsigned)nyl,
                 (unsigned long long)nxl * 6 * nyl * nzh, (unsigned)s};
        PackCb* d;
        CK(cudaMalloc(&d, sizeof h));
        CK(cudaMemcpy(d, &h, sizeof h, cudaMemcpyHostToDevice));
        void* ci = d;
        CK(cufftCreate(&cb[s]));
        CK(cufftXtSetJITCallback(cb[s], "cb_pack_store", fat.data(), fat.size(), CUFFT_CB_ST_COMPLEX_DOUBLE, &ci));
        CK(cufftMakePlanMany64(cb[s], 2, n2, nullptr, 1, (long long)n * n, nullptr, 1, (long long)n * nzh, CUFFT_D2Z,
                               6LL * nxl, &ws));
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run_plain = [&]() {
        for (int s = 0; s < k; ++s) {
            CK(cufftExecD2Z(plain, R[s], P[s]));
            k_pack<<<dim3(8, k * nxl * 6), 256>>>(P[s], dpeer, s, nxl, n, nzh, nyl);
        }
    };
    auto run_cb = [&]() {
        for (int s = 0; s < k; ++s) CK(cufftExecD2Z(cb[s], R[s], P[s]));
    };
    float t[2];
    for (int v = 0; v < 2; ++v) {
        for (int i = 0; i < 3; ++i) v ? run_cb() : run_plain();
        cudaEventRecord(a);
        for (int i = 0; i < 10; ++i) v ? run_cb() : run_plain();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&t[v], a, b);
        t[v] /= 10;
    }
    // the D2Z alone
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i)
        for (int s = 0; s < k; ++s) CK(cufftExecD2Z(plain, R[s], P[s]));
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float td;
    cudaEventElapsedTime(&td, a, b);
    std::printf("{\"n\": %d, \"slabs\": %d, \"d2z_only_ms\": %.4f, \"d2z_plus_pack_ms\": %.4f, \"d2z_store_callback_ms\": %.4f}\n",
                n, k, td / 10, t[0], t[1]);
    return 0;
}
