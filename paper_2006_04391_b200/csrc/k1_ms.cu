// k1_ms.cu -- Michel-Suquet, automatic strategy: Newton and tangent kernels.
// (one translation unit per law / strategy so the heavy template
// instantiations compile in parallel; kernels in k1_kernels.cuh)
#include "k1_kernels.cuh"

namespace am {

int launch_law_ms(const MichelSuquetLaw& L, const KArgs& k, cudaStream_t s) { return launch_law(L, k, s); }

}  // namespace am
