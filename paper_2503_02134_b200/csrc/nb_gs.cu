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
#include "nb_cg.cuh"   // DevCache

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

// ---------------------------------------------------------------------------
// Consistent order on the box, without the CSR (nb_dssum / nb_ax default path).
// Every shared global node is handled by its "owner" copy: the copy in the highest-numbered
// element, i.e. the one whose local coordinate is 0 on every shared axis.  Owners lie on an
// element's three lower faces, enumerated once each: item t < N^2 -> (i, j, 0); then (i, 0, k >= 1);
// then (0, j >= 1, k >= 1) -- M = 3N^2 - 3N + 1 items, one thread each.  The owner reads the copies
// in the lower neighbours (their upper faces), sums them in ascending element order
// (lexicographic (dz, dy, dx), negative offsets first, the owner last) -- the CSR consistent
// order, so the sums are bit-identical -- and writes the rounded sum to every copy.  Each local
// node belongs to one global node and each global node to one owner: the kernel is in-place safe
// without any ordering between blocks, and no index arrays are read (the CSR reads 4 B per copy
// and 4 B per node more).
// A block streams chunks of CH consecutive elements along x: each element is read once, whole and
// coalesced, into shared memory (double-buffered, the next element prefetched in registers while
// this one is summed); the i = 0 face (one value per pencil -- strided in i-fastest storage) and
// the x-partner column of the previous element then come from shared memory, the y/z partner
// faces (contiguous rows / planes of other elements, recently streamed: L2) from global memory.
// z-neighbours only inside the handle's layers (a slab's nb_dssum acts on the slab alone, like the
// slab's CSR).
// ---------------------------------------------------------------------------
template <int N, typename TVX> struct DsRow {
    static constexpr int N3 = N * N * N;
    static constexpr int M = 3 * N * N - 3 * N + 1;
    static constexpr int NT = ((M + 31) / 32) * 32 < 128 ? 128 : ((M + 31) / 32) * 32;
    // elements per step (gathers in flight): up to 4, at most ~96 KB of double-buffered stage
    static constexpr int ELM = 98304 / (2 * N3 * (int)sizeof(TVX));
    // measured (tools/ab_ops.sh, 32^3 p7/p9/p11 with an L2 flush per call): 2 for 4-byte data,
    // 1 for 8-byte data (EL = 4 and the register-only variant EU = 4 / 8 were slower or equal)
#ifndef NB_DS_EL
#define NB_DS_EL (sizeof(TVX) == 4 ? 2 : 1)
#endif
    static constexpr int EL = ELM < 1 ? 1 : (ELM > NB_DS_EL ? NB_DS_EL : ELM);
    static constexpr int PV = (EL * N3 + NT - 1) / NT;      // staged values per thread (prefetch)
    static constexpr int CH = 16;                           // elements per chunk along x
    static constexpr int SMEM = 2 * EL * N3 * (int)sizeof(TVX);
};

#ifndef NB_DS_PF
#define NB_DS_PF 0
#endif
template <typename TVX, typename TGX, int N>
__global__ void __launch_bounds__(DsRow<N, TVX>::NT) k_dssum_rows(const MeshDev m, TVX *__restrict__ u)
{
    using R = DsRow<N, TVX>;
    constexpr int N2 = N * N, N3 = N2 * N, M = R::M, NT = R::NT, PV = R::PV, CH = R::CH, EL = R::EL;
    extern __shared__ __align__(16) unsigned char ds_raw[];
    TVX *const buf = reinterpret_cast<TVX *>(ds_raw);   // [2][EL * N3]
    const int t = threadIdx.x;
    int i, j, k;
    if (t < N2) { i = t % N; j = t / N; k = 0; }
    else if (t < N2 + N * (N - 1)) { const int q = t - N2; i = q % N; j = 0; k = 1 + q / N; }
    else { const int q = t - N2 - N * (N - 1); i = 0; j = 1 + q % (N - 1); k = 1 + q / (N - 1); }
    const bool item = t < M;
    const int qown = i + N * j + N2 * k;
    const int qxp = (N - 1) + N * j + N2 * k;   // x-partner (i = N-1) in the lower x-neighbour
    const int64_t ox = N3 - (N - 1);
    const int64_t oy = (int64_t)m.nelx * N3 - (int64_t)(N - 1) * N;
    const int64_t oz = (int64_t)m.nelx * m.nely * N3 - (int64_t)(N - 1) * N2;
    const int cpr = (m.nelx + CH - 1) / CH;
    const int64_t units = (int64_t)cpr * m.nely * m.nelzl;
#pragma unroll 1
    for (int64_t unit = blockIdx.x; unit < units; unit += gridDim.x) {
        const int c = (int)(unit % cpr);
        const int64_t row = unit / cpr;
        const int ey = (int)(row % m.nely), ez = (int)(row / m.nely);
        const int exa = c * CH, exb = min(m.nelx, exa + CH);
        const int64_t erow = (int64_t)m.nelx * (ey + (int64_t)m.nely * ez);
#if NB_DS_PF
        // the block's next unit (a contiguous run of elements) into L2 while this one is summed
        // (measured slower at 32^3: mixed p9 84 -> 93 us, fp64 p11 192 -> 227 us; off)
        if (threadIdx.x == 0 && unit + gridDim.x < units) {
            const int64_t un = unit + gridDim.x;
            const int cn = (int)(un % cpr);
            const int64_t rn = un / cpr;
            const int xa = cn * CH, xb = min(m.nelx, xa + CH);
            l2_prefetch(u + (rn * m.nelx + xa) * (int64_t)N3, (size_t)(xb - xa) * N3 * sizeof(TVX));
        }
#endif
        const bool sy = j == 0 && ey > 0, sz = k == 0 && ez > 0;
        const bool upyz = (j == N - 1 && ey < m.nely - 1) || (k == N - 1 && ez < m.nelzl - 1);
        TVX pre[PV];
        {
            const int cnt = min(EL, exb - exa) * N3;
#pragma unroll
            for (int v = 0; v < PV; v++) {
                const int q = t + v * NT;
                if (q < cnt) pre[v] = u[(erow + exa) * N3 + q];
            }
        }
#pragma unroll 1
        for (int ex0 = exa, step = 0; ex0 < exb; ex0 += EL, step++) {
            const int ne = min(EL, exb - ex0);
            TVX *const bc = buf + (step & 1) * EL * N3;
            const TVX *const bp = buf + ((step & 1) ^ 1) * EL * N3;
#pragma unroll
            for (int v = 0; v < PV; v++) {
                const int q = t + v * NT;
                if (q < ne * N3) bc[q] = pre[v];
            }
            __syncthreads();
            if (ex0 + EL < exb) {   // prefetch the next EL elements of the chunk
                const int cnt = min(EL, exb - ex0 - EL) * N3;
#pragma unroll
                for (int v = 0; v < PV; v++) {
                    const int q = t + v * NT;
                    if (q < cnt) pre[v] = u[(erow + ex0 + EL) * N3 + q];
                }
            }
            TVX v[EL][8];   // v[.][c]: c = (iz, iy, ix) bits, 1 = the lower neighbour on that axis
            bool own[EL], sxa[EL];
#pragma unroll
            for (int uu = 0; uu < EL; uu++) {
                const int ex = ex0 + uu;
                const bool sx = i == 0 && ex > 0;
                const bool up = upyz || (i == N - 1 && ex < m.nelx - 1);
                own[uu] = item && uu < ne && (sx || sy || sz) && !up;
                sxa[uu] = sx;
                if (!own[uu]) continue;
                const int64_t l = (erow + ex) * N3 + qown;
#pragma unroll
                for (int cc = 0; cc < 8; cc++) {
                    const bool need = ((cc & 1) == 0 || sx) && ((cc & 2) == 0 || sy) && ((cc & 4) == 0 || sz);
                    if (!need) continue;
                    if (cc == 0) v[uu][cc] = bc[uu * N3 + qown];
                    else if (cc == 1)
                        v[uu][cc] = uu > 0 ? bc[(uu - 1) * N3 + qxp]
                                           : (ex0 > exa ? bp[(EL - 1) * N3 + qxp] : u[l - ox]);
                    else v[uu][cc] = u[l - ((cc & 4) ? oz : 0) - ((cc & 2) ? oy : 0) - ((cc & 1) ? ox : 0)];
                }
            }
#pragma unroll
            for (int uu = 0; uu < EL; uu++) {
                if (!own[uu]) continue;
                const bool sx = sxa[uu];
                const int64_t l = (erow + ex0 + uu) * N3 + qown;
                TGX acc = 0;
                bool first = true;
#pragma unroll
                for (int oc = 0; oc < 8; oc++) {   // (1,1,1) first ... (0,0,0) = the owner last
                    const int cc = 7 - oc;
                    if (((cc & 1) && !sx) || ((cc & 2) && !sy) || ((cc & 4) && !sz)) continue;
                    acc = first ? (TGX)v[uu][cc] : acc + (TGX)v[uu][cc];
                    first = false;
                }
                const TVX r = (TVX)acc;
#pragma unroll
                for (int cc = 0; cc < 8; cc++) {
                    if (((cc & 1) && !sx) || ((cc & 2) && !sy) || ((cc & 4) && !sz)) continue;
                    u[l - ((cc & 4) ? oz : 0) - ((cc & 2) ? oy : 0) - ((cc & 1) ? ox : 0)] = r;
                }
            }
            __syncthreads();   // bp is overwritten two steps later
        }
    }
}

template <typename TVX, typename TGX, int N>
static cudaError_t dssum_rows_t(const nb_handle *h, void *u, cudaStream_t st)
{
    using R = DsRow<N, TVX>;
    static DevCache cache;
    int &occ = cache.here();
    if (occ < 0) {
        cudaFuncSetAttribute(k_dssum_rows<TVX, TGX, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, R::SMEM);
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_dssum_rows<TVX, TGX, N>, R::NT, R::SMEM);
        occ = o > 0 ? o : 1;
    }
    const int64_t units = (int64_t)((h->nelx + R::CH - 1) / R::CH) * h->nely * h->nelzl;
    int64_t grid = (int64_t)h->sm_count * occ;
    if (grid > units) grid = units;
    if (grid < 1) grid = 1;
    k_dssum_rows<TVX, TGX, N><<<(int)grid, R::NT, R::SMEM, st>>>(h->md(), (TVX *)u);
    return cudaGetLastError();
}

template <typename TVX, typename TGX>
static cudaError_t dssum_box(const nb_handle *h, void *u, cudaStream_t st)
{
    NB_DISPATCH_N(h->n, return (dssum_rows_t<TVX, TGX, NN>(h, u, st)))
}

cudaError_t launch_dssum(const nb_handle *h, int prec, int order, void *u, cudaStream_t st, RankPart rp)
{
    if (order == NB_GS_CONSISTENT && !h->dssum_csr) {
        if (h->nseg == 0) return cudaSuccess;
        if (prec == NB_FP64) return dssum_box<double, double>(h, u, st);
        if (prec == NB_FP32 || prec == NB_FP32_DOT2) return dssum_box<float, float>(h, u, st);
        return dssum_box<float, double>(h, u, st);
    }
    if (prec == NB_FP64) return gs_launch_t<NB_FP64, double, double>(h, order, u, rp, st);
    if (prec == NB_FP32 || prec == NB_FP32_DOT2) return gs_launch_t<NB_FP32, float, float>(h, order, u, rp, st);
    return gs_launch_t<NB_MIXED, float, double>(h, order, u, rp, st);
}

}  // namespace nb
