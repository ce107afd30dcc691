// nb_gs.cuh -- one gather-scatter segment (direct stiffness summation over the copies of one
// shared global node), shared by the CSR kernel (nb_gs.cu) and the
// per-copy phase of the CG megakernel (nb_cg.cuh).  gslib's gs_op / jl_gs_gather in the
// paper, accumulated in the policy's gather-scatter precision
// (the mixed strategy keeps the GS in double).
//   NB_GS_CONSISTENT: s = sum of the copies in ascending local index, written to every copy.
//   NB_GS_PER_COPY  : copy l receives w_l + sum_{m != l, ascending} w_m -- the arithmetic of
//                     the paper's pairwise exchange, where each rank adds its neighbours'
//                     contributions to its own (Table 3).
// With PAP = 1 it returns the segment's part of pap = glsc3(w, c, p).
#pragma once
#include "nb_common.cuh"

namespace nb {

// Rank of element e in the partition rp of the element box (NB_GS_PAIRWISE / NB_GS_ALLREDUCE,
// nb.h): block b of an axis holds elements [b nel / P, (b+1) nel / P), so the block of element
// index i is floor(((i + 1) P - 1) / nel).
__device__ __forceinline__ int elem_rank(const MeshDev &m, const RankPart &rp, int32_t e)
{
    const int32_t t = e / m.nelx, ex = e - t * m.nelx;
    const int32_t ez = t / m.nely, ey = t - ez * m.nely;
    const int bx = ((ex + 1) * rp.px - 1) / m.nelx;
    const int by = ((ey + 1) * rp.py - 1) / m.nely;
    const int bz = ((ez + 1) * rp.pz - 1) / m.nelz;
    return bx + rp.px * (by + rp.py * bz);
}

template <int PREC, int ORDER, int PAP, typename TVX, typename TGX, int H>
__device__ __forceinline__ Acc<PREC> gs_segment(int32_t s, const int32_t *__restrict__ off,
                                                const int32_t *__restrict__ idx, TVX *__restrict__ w,
                                                const TVX *__restrict__ pv, const MeshDev *m = nullptr,
                                                RankPart rp = RankPart{1, 1, 1})
{
    using TS = typename Pol<PREC>::TS;
    Acc<PREC> acc;
    const int32_t a0 = __ldg(off + s);
    const int32_t cnt = __ldg(off + s + 1) - a0;
    int32_t id[8];
    TVX v[8];
#pragma unroll
    for (int c = 0; c < 8; c++)
        if (c < cnt) id[c] = __ldg(idx + a0 + c);
#pragma unroll
    for (int c = 0; c < 8; c++)
        if (c < cnt) v[c] = ldv<H>(w + id[c]);
    if (ORDER == NB_GS_CONSISTENT) {
        TGX t = (TGX)v[0];
#pragma unroll
        for (int c = 1; c < 8; c++)
            if (c < cnt) t += (TGX)v[c];
        const TVX tv = (TVX)t;
#pragma unroll
        for (int c = 0; c < 8; c++)
            if (c < cnt) w[id[c]] = tv;
        if (PAP) acc.add((TS)tv, (TS)ldv<H>(pv + id[0]));   // sum_copies c w p = sigma p (p continuous)
    } else if (ORDER == NB_GS_PAIRWISE || ORDER == NB_GS_ALLREDUCE) {
        // rank partials (each rank's copies in ascending local index), then the exchange
        const int n3 = m->n * m->n * m->n;
        int rk[8];
        TGX part[8];
#pragma unroll
        for (int c = 0; c < 8; c++)
            if (c < cnt) rk[c] = elem_rank(*m, rp, id[c] / n3);
#pragma unroll
        for (int c = 0; c < 8; c++) {
            if (c < cnt) {
                TGX t = 0;
#pragma unroll
                for (int c2 = 0; c2 < 8; c2++)
                    if (c2 < cnt && rk[c2] == rk[c]) t += (TGX)v[c2];
                part[c] = t;
            }
        }
        const TS cinv = (TS)1 / (TS)cnt;
#pragma unroll
        for (int c = 0; c < 8; c++) {
            if (c < cnt) {
                // distinct ranks in ascending order: copy c2 contributes when it is the first copy of
                // its rank (ascending local index = the rank's lowest copy) -- ordered by rank value
                TGX t = ORDER == NB_GS_PAIRWISE ? part[c] : (TGX)0;
                int prev = -1;
#pragma unroll 1
                for (int k = 0; k < cnt; k++) {
                    int best = -1, br = 0x7fffffff;
#pragma unroll
                    for (int c2 = 0; c2 < 8; c2++)
                        if (c2 < cnt && rk[c2] > prev && rk[c2] < br) { best = c2; br = rk[c2]; }
                    if (best < 0) break;
                    prev = br;
                    if (!(ORDER == NB_GS_PAIRWISE && br == rk[c])) {
#pragma unroll
                        for (int c2 = 0; c2 < 8; c2++)   // static register indices
                            if (c2 == best) t += part[c2];
                    }
                }
                const TVX tv = (TVX)t;
                w[id[c]] = tv;
                if (PAP) acc.add((TS)tv * cinv, (TS)ldv<H>(pv + id[c]));
            }
        }
    } else {
        const TS cinv = (TS)1 / (TS)cnt;
#pragma unroll
        for (int c = 0; c < 8; c++) {
            if (c < cnt) {
                TGX t = (TGX)v[c];
#pragma unroll
                for (int r = 0; r < 8; r++)
                    if (r < cnt && r != c) t += (TGX)v[r];
                const TVX tv = (TVX)t;
                w[id[c]] = tv;
                if (PAP) acc.add((TS)tv * cinv, (TS)ldv<H>(pv + id[c]));
            }
        }
    }
    return acc;
}

}  // namespace nb
