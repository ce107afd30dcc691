// nb_cg_fp32.cu -- instantiates the Ax / CG kernels of nb_cg.cuh for the fp32 policy
// (one translation unit per policy so the build compiles them in parallel).
#include "nb_mega_launch.cuh"

namespace nb {
NB_INSTANTIATE_CG(NB_FP32)
}  // namespace nb
