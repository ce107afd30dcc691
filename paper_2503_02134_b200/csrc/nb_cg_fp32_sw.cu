// nb_cg_fp32_sw.cu -- the fp32 policy's Schwarz-preconditioned megakernel and solveM kernel
// (NB_PC_SCHWARZ), in their own translation unit (parallel build).
#include "nb_mega_launch.cuh"

namespace nb {
NB_INSTANTIATE_CG_SW(NB_FP32)
}  // namespace nb
