// k1_misc.cu -- linear elasticity (automatic and semi-automatic) and the conventional radial return.
// (one translation unit per law / strategy so the heavy template
// instantiations compile in parallel; kernels in k1_kernels.cuh)
#include "k1_kernels.cuh"

namespace am {

int launch_law_le(const LinearElasticLaw& L, const KArgs& k, cudaStream_t s) { return launch_law(L, k, s); }

int launch_law_le_semi(const SemiLaw<LinearElasticLaw>& L, const KArgs& k, cudaStream_t s) {
    return launch_law(L, k, s);
}

int launch_conventional(const SemiLaw<MichelSuquetLaw>& S, const KArgs& k, cudaStream_t s) {
    int64_t blocks = (k.B + 127) / 128;
    if (blocks > (int64_t)kSMs * 1024) blocks = (int64_t)kSMs * 1024;
    if (k.C) k_conventional<true><<<(unsigned)blocks, 128, 0, s>>>(S, k);
    else k_conventional<false><<<(unsigned)blocks, 128, 0, s>>>(S, k);
    AM_CUDA(cudaGetLastError());
    return AM_OK;
}

}  // namespace am
