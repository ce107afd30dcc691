// nb_cg_dot2.cu -- instantiates the Ax / CG kernels of nb_cg.cuh for the fp32 policy with
// compensated (Dot2) dot products (Sec. 5.2.1).
#include "nb_mega_launch.cuh"

namespace nb {
NB_INSTANTIATE_CG(NB_FP32_DOT2)
}  // namespace nb
