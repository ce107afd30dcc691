// nb_cg_fp64_var.cu -- the fp64 policy's megakernels for the preconditioner / x_fp64 variants
// (VAR = 1), in their own translation unit so the build runs in parallel.
#include "nb_mega_launch.cuh"

namespace nb {
NB_INSTANTIATE_CG_VAR(NB_FP64)
}  // namespace nb
