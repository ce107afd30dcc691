// nb_cg_fp32_var.cu -- the fp32 policy's megakernels for the preconditioner / x_fp64 variants
// (VAR = 1), in their own translation unit so the build runs in parallel.
// fp32 policy, N = 12: the TMA stage for the geometric factors with two resident blocks instead of three
// (AxCfg::GSTAGE bit 2, NB_MINB_N12; 32^3 p11: phase A 580 -> 480 us, phase B 238 -> 273 us, iteration -8%)
#define NB_GSTAGE 7
#define NB_MINB_N12 2
#include "nb_mega_launch.cuh"

namespace nb {
NB_INSTANTIATE_CG_VAR(NB_FP32)
}  // namespace nb
