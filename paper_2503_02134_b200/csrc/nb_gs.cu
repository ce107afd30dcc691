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
// MODE 1 (CG, per-copy path): also the shared-node part of pap = glsc3(w, c, p)
// and the alpha finalize; K1 (MODE 2) contributed the unshared nodes.
#include "nb_gs.cuh"

namespace nb {

constexpr int GS_NT = 256;

template <int PREC, int ORDER, int MODE, typename TVX, typename TGX>
__global__ void __launch_bounds__(GS_NT)
k_gs(const int32_t nseg, const int32_t *__restrict__ off, const int32_t *__restrict__ idx, TVX *__restrict__ w,
     const TVX *__restrict__ pv, Scal *__restrict__ scal, const RedWs rw)
{
    using TS = typename Pol<PREC>::TS;
    if (MODE == 1 && scal->done) return;
    TS acc = 0;
    const int32_t s = blockIdx.x * GS_NT + threadIdx.x;
    if (s < nseg) acc = gs_segment<PREC, ORDER, MODE, TVX, TGX, LD_DEF>(s, off, idx, w, pv).value();
    if (MODE == 1) {
        __shared__ TS red[32];
        TS vv[1] = {block_sum<TS>(acc, red)};
        TS tot[1];
        if (grid_reduce<TS, 1>(vv, rw, tot) && threadIdx.x == 0) {
            // pap = (unshared part from K1, stored in scal->pap) + shared part
            const TS pap = (TS)scal->pap + tot[0];
            const TS rho = (TS)scal->rho;
            scal->pap = (double)pap;
            if (!(pap > (TS)0) || !isfinite((double)pap) || !isfinite((double)rho)) {
                scal->status = NB_BROKEDOWN;
                scal->done = 1;
                scal->pending = 0;
            } else {
                scal->alpha = (double)(rho / pap);
                scal->pending = 1;
            }
        }
    }
}

int grid_gs(const nb_handle *h) { return (int)((h->nseg + GS_NT - 1) / GS_NT); }

template <int PREC, int ORDER, int MODE, typename TVX, typename TGX>
static cudaError_t gs_launch_t(const nb_handle *h, void *u, const void *pv, Scal *scal, const RedWs &rw, cudaStream_t st)
{
    if (h->nseg == 0 && MODE == 0) return cudaSuccess;
    const int grid = grid_gs(h) > 0 ? grid_gs(h) : 1;
    k_gs<PREC, ORDER, MODE, TVX, TGX><<<grid, GS_NT, 0, st>>>((int32_t)h->nseg, h->gs_off, h->gs_idx, (TVX *)u,
                                                              (const TVX *)pv, scal, rw);
    return cudaGetLastError();
}

cudaError_t launch_dssum(const nb_handle *h, int prec, int order, void *u, cudaStream_t st)
{
    const RedWs n = {nullptr, nullptr, nullptr};
    if (prec == NB_FP64)
        return order == NB_GS_CONSISTENT ? gs_launch_t<NB_FP64, NB_GS_CONSISTENT, 0, double, double>(h, u, nullptr, nullptr, n, st)
                                         : gs_launch_t<NB_FP64, NB_GS_PER_COPY, 0, double, double>(h, u, nullptr, nullptr, n, st);
    if (prec == NB_FP32)
        return order == NB_GS_CONSISTENT ? gs_launch_t<NB_FP32, NB_GS_CONSISTENT, 0, float, float>(h, u, nullptr, nullptr, n, st)
                                         : gs_launch_t<NB_FP32, NB_GS_PER_COPY, 0, float, float>(h, u, nullptr, nullptr, n, st);
    return order == NB_GS_CONSISTENT ? gs_launch_t<NB_MIXED, NB_GS_CONSISTENT, 0, float, double>(h, u, nullptr, nullptr, n, st)
                                     : gs_launch_t<NB_MIXED, NB_GS_PER_COPY, 0, float, double>(h, u, nullptr, nullptr, n, st);
}

cudaError_t launch_cg_gs(const nb_handle *h, int prec, int order, Workspace &ws, cudaStream_t st)
{
    if (prec == NB_FP64)
        return order == NB_GS_CONSISTENT
                   ? gs_launch_t<NB_FP64, NB_GS_CONSISTENT, 1, double, double>(h, ws.w, ws.p, ws.scal, ws.red, st)
                   : gs_launch_t<NB_FP64, NB_GS_PER_COPY, 1, double, double>(h, ws.w, ws.p, ws.scal, ws.red, st);
    if (prec == NB_FP32)
        return order == NB_GS_CONSISTENT
                   ? gs_launch_t<NB_FP32, NB_GS_CONSISTENT, 1, float, float>(h, ws.w, ws.p, ws.scal, ws.red, st)
                   : gs_launch_t<NB_FP32, NB_GS_PER_COPY, 1, float, float>(h, ws.w, ws.p, ws.scal, ws.red, st);
    return order == NB_GS_CONSISTENT
               ? gs_launch_t<NB_MIXED, NB_GS_CONSISTENT, 1, float, double>(h, ws.w, ws.p, ws.scal, ws.red, st)
               : gs_launch_t<NB_MIXED, NB_GS_PER_COPY, 1, float, double>(h, ws.w, ws.p, ws.scal, ws.red, st);
}

}  // namespace nb
