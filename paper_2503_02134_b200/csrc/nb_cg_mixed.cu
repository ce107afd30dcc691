// nb_cg_mixed.cu -- instantiates the Ax / CG kernels of nb_cg.cuh for the mixed policy
// (one translation unit per policy so the build compiles them in parallel).
// mixed policy, N = 10: one element per 128-thread block, three resident blocks (AxCfg::E1S, nb_cg.cuh)
#define NB_E1_S10 3
#include "nb_mega_launch.cuh"

namespace nb {
NB_INSTANTIATE_CG(NB_MIXED)
}  // namespace nb
