// nb_gs.cu -- gather-scatter (direct stiffness summation, QQ^T) over the precomputed
// shared-node CSR segments: gslib's gs_op / jl_gs_gather in the
// paper, accumulated in the policy's gather-scatter precision
// (the mixed strategy keeps the GS in double).
//
// One thread per shared global node (segment); segments are ascending in global id and
// each lists its copies in ascending local index.
//   NB_GS_CONSISTENT: s = sum of the copies in that order, written to every copy.
//   NB_GS_PER_COPY  : copy l receives w_l + sum_{m != l, ascending} w_m -- the arithmetic of
//                     the paper's pairwise exchange, where each rank adds its neighbours'
//                     contributions to its own (Table 3).
//   NB_GS_PAIRWISE / NB_GS_ALLREDUCE: the same exchange between the ranks of a logical element
//                     partition (rank partials first; NEXT-2, nb.h).
#include "nb_gs.cuh"

namespace nb {

constexpr int GS_NT = 256;

template <int PREC, int ORDER, typename TVX, typename TGX>
__global__ void __launch_bounds__(GS_NT)
k_gs(const int32_t nseg, const int32_t *__restrict__ off, const int32_t *__restrict__ idx, TVX *__restrict__ w,
     const MeshDev m, const RankPart rp)
{
    const int32_t s = blockIdx.x * GS_NT + threadIdx.x;
    if (s < nseg) gs_segment<PREC, ORDER, 0, TVX, TGX, LD_DEF>(s, off, idx, w, (const TVX *)nullptr, &m, rp);
}

int grid_gs(const nb_handle *h) { return (int)((h->nseg + GS_NT - 1) / GS_NT); }

template <int PREC, typename TVX, typename TGX>
static cudaError_t gs_launch_t(const nb_handle *h, int order, void *u, RankPart rp, cudaStream_t st)
{
    if (h->nseg == 0) return cudaSuccess;
    const int g = grid_gs(h);
    const MeshDev m = h->md();
    auto L = [&](auto kern) {
        kern<<<g, GS_NT, 0, st>>>((int32_t)h->nseg, h->gs_off, h->gs_idx, (TVX *)u, m, rp);
        return cudaGetLastError();
    };
    switch (order) {
    case NB_GS_CONSISTENT: return L(k_gs<PREC, NB_GS_CONSISTENT, TVX, TGX>);
    case NB_GS_PER_COPY: return L(k_gs<PREC, NB_GS_PER_COPY, TVX, TGX>);
    case NB_GS_PAIRWISE: return L(k_gs<PREC, NB_GS_PAIRWISE, TVX, TGX>);
    default: return L(k_gs<PREC, NB_GS_ALLREDUCE, TVX, TGX>);
    }
}

cudaError_t launch_dssum(const nb_handle *h, int prec, int order, void *u, cudaStream_t st, RankPart rp)
{
    if (prec == NB_FP64) return gs_launch_t<NB_FP64, double, double>(h, order, u, rp, st);
    if (prec == NB_FP32 || prec == NB_FP32_DOT2) return gs_launch_t<NB_FP32, float, float>(h, order, u, rp, st);
    return gs_launch_t<NB_MIXED, float, double>(h, order, u, rp, st);
}

}  // namespace nb
