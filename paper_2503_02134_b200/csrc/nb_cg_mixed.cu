// nb_cg_mixed.cu -- instantiates the Ax / CG kernels of nb_cg.cuh for the mixed policy
// (one translation unit per policy so the build compiles them in parallel).
// mixed policy, N = 10: one element per 128-thread block, three resident blocks (AxCfg::E1S, nb_cg.cuh)
#define NB_E1_S10 3
// mixed policy, N = 12: the TMA stage for the geometric factors with two resident blocks instead of three
// (AxCfg::GSTAGE bit 2, NB_MINB_N12; 32^3 p11: phase A 593 -> 493 us, phase B 332 -> 342 us)
#define NB_GSTAGE 7
#define NB_MINB_N12 2
#include "nb_mega_launch.cuh"

namespace nb {
NB_INSTANTIATE_CG(NB_MIXED)
}  // namespace nb
