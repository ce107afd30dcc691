// nb_cg_fp32.cu -- instantiates the Ax / CG kernels of nb_cg.cuh for the fp32 policy
// (one translation unit per policy so the build compiles them in parallel).
// fp32 policy, N = 12: the TMA stage for the geometric factors with two resident blocks instead of three
// (AxCfg::GSTAGE bit 2, NB_MINB_N12; 32^3 p11: phase A 580 -> 480 us, phase B 238 -> 273 us, iteration -8%)
#define NB_GSTAGE 7
#define NB_MINB_N12 2
#include "nb_mega_launch.cuh"

namespace nb {
NB_INSTANTIATE_CG(NB_FP32)
}  // namespace nb
