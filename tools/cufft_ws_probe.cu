#include <cufft.h>
#include <cstdio>
int main() {
    for (long long n : {256LL, 512LL, 640LL}) {
        long long n3[3] = {n, n, n}, N = n * n * n, Nh = n * n * (n / 2 + 1);
        size_t w1 = 0, w2 = 0;
        cufftHandle a, b;
        cufftCreate(&a); cufftSetAutoAllocation(a, 0);
        cufftCreate(&b); cufftSetAutoAllocation(b, 0);
        int r1 = cufftMakePlanMany64(a, 3, n3, nullptr, 1, N, nullptr, 1, Nh, CUFFT_D2Z, 6, &w1);
        int r2 = cufftMakePlanMany64(b, 3, n3, nullptr, 1, Nh, nullptr, 1, N, CUFFT_Z2D, 6, &w2);
        printf("n=%lld rc %d %d  D2Z ws %.3f GB  Z2D ws %.3f GB  spectrum %.3f GB\n", n, r1, r2, w1 / 1e9, w2 / 1e9,
               6.0 * Nh * 16 / 1e9);
        cufftDestroy(a); cufftDestroy(b);
    }
}
