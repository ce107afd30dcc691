// nb_cg_mixed.cu -- instantiates the Ax / CG kernels of nb_cg.cuh for the mixed policy
// (one translation unit per policy so the build compiles them in parallel).
#include "nb_mega_launch.cuh"

namespace nb {
NB_INSTANTIATE_CG(NB_MIXED)
}  // namespace nb
