// k1_adapt_ms_semi.cu -- Michel-Suquet, semi-automatic strategy: adaptive ode12 / ode23 / ode23s kernels.
// (one translation unit per law / strategy so the heavy template
// instantiations compile in parallel; kernels in k1_kernels.cuh)
#include "k1_kernels.cuh"

namespace am {

int launch_adaptive_law(const SemiLaw<MichelSuquetLaw>& L, const KArgs& k, unsigned g, cudaStream_t s) {
    using Law = SemiLaw<MichelSuquetLaw>;
    if (k.integrator == AM_INTEGRATOR_ODE23S) return launch_adaptive<Law, 32>(L, k, g, s);
    return k.integrator == AM_INTEGRATOR_ODE23 ? launch_adaptive<Law, 23>(L, k, g, s)
                                               : launch_adaptive<Law, 12>(L, k, g, s);
}

}  // namespace am
