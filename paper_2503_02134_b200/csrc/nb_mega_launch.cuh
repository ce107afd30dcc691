// nb_mega_launch.cuh -- host launchers of the CG megakernels (nb_cg.cuh): occupancy-sized
// persistent grids (every block resident: cooperative launches), the shared-memory carve-out,
// the kernel arguments of one slab or whole box, and the multi-rank (z-slab) launch.
// Included by the per-policy translation units (nb_cg_<policy>[_var].cu).
// (A variant that staged every phase operand through 1-D TMA bulk copies and an mbarrier ring
// measured slower on B200 and was removed.)
#pragma once
#include "nb_cg.cuh"

#include <cstdlib>

namespace nb {

// Shared-memory carve-out: just what the resident blocks need, the rest of the 256 KB stays L1
// (phase B's neighbour-copy loads hit in L1).  NB_CARVEOUT=0 leaves the driver's choice.
static void set_carveout(const void *fn, int occ, int smem)   // called once per device and kernel
{
    static int mode = -1;
    if (mode < 0) {
        const char *s = std::getenv("NB_CARVEOUT");
        mode = (s && s[0] == '0') ? 0 : 1;
    }
    if (!mode) return;
    cudaFuncAttributes fa{};
    const int stat = cudaFuncGetAttributes(&fa, fn) == cudaSuccess ? (int)fa.sharedSizeBytes : 0;
    const int need = occ * (smem + stat + 1024) + 1024;            // + static + per-block reservation
    int pct = (int)((100LL * need + 228 * 1024 - 1) / (228 * 1024));
    // close to the maximum: ask for all of it (a preference that maps to a smaller supported size than
    // the resident blocks need lowers the cooperative-launch limit: "too many blocks")
    if (pct > 80) pct = 100;
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

template <int PREC, int N, int FUSED, int VAR>
static int mega_grid_t(const nb_handle *h)
{
    using C = AxCfg<typename Pol<PREC>::TV, N>;
    constexpr int SMEM_MEGA = C::SMEM_CG;
    const void *fn = (const void *)k_cg_mega<PREC, N, FUSED, VAR>;
    static DevCache cache;   // the attributes and the residency are per device
    int &occ = cache.here();
    if (occ < 0) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MEGA);
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, C::NT, SMEM_MEGA);
        occ = o > 0 ? o : 1;
        set_carveout(fn, occ, SMEM_MEGA);
    }
    return h->sm_count * occ;
}

template <int PREC, int VAR>
int grid_mega_var(const nb_handle *h)
{
    NB_DISPATCH_N(h->n, return (mega_grid_t<PREC, NN, 1, VAR>(h) > mega_grid_t<PREC, NN, 0, VAR>(h)
                                    ? mega_grid_t<PREC, NN, 1, VAR>(h)
                                    : mega_grid_t<PREC, NN, 0, VAR>(h)))
}

// grid size of every megakernel of the policy (sizes the per-block partials)
template <int PREC>
int grid_mega(const nb_handle *h)
{
    const int g0 = grid_mega_var<PREC, 0>(h), g1 = grid_mega_var<PREC, 1>(h);
    return g0 > g1 ? g0 : g1;
}

// element groups on the busiest SM when G blocks split ng groups into contiguous ranges
// (split(): block i gets [i ng / G, (i+1) ng / G)) and block i runs on SM i mod S
static long long balanced_sm_max(long long ng, long long G, int S)
{
    if (S < 1) S = 1;
    long long best = 0;
    for (int j = 0; j < S && j < G; j++) {
        long long w = 0;
        for (long long i = j; i < G; i += S) w += (i + 1) * ng / G - i * ng / G;
        if (w > best) best = w;
    }
    return best;
}

template <int PREC, int N, int FUSED, int VAR>
static cudaError_t mega_launch_t(const nb_handle *h, const MegaArgs &args, cudaStream_t st)
{
    using TV = typename Pol<PREC>::TV;
    using C = AxCfg<TV, N>;
    constexpr int SMEM_MEGA = C::SMEM_CG;
    DMat<TV, N> D = make_dmat<TV, N>(h->D);
    MegaArgs a2 = args;
    void *params[2] = {(void *)&a2, (void *)&D};
    int grid = mega_grid_t<PREC, N, FUSED, VAR>(h);
    const int full = grid;
    // Balanced grid: the fewest blocks that keep the same number of element groups on the
    // busiest block (configs[1]: 1024 groups on 256 blocks x 4 instead of 296 blocks x 3-4), so
    // no wave is partly idle and the barriers have fewer arrivals -- unless that raises the
    // busiest SM's group count (blocks i -> SM i mod #SMs; e.g. 20^3 p = 11: 55 -> 57 groups,
    // measured +4%).  DESIGN.md §6.  NB_GRID_BALANCE=0: the full occupancy grid.
    static int balance = -1;
    if (balance < 0) {
        const char *s = std::getenv("NB_GRID_BALANCE");
        balance = (s && s[0] == '0') ? 0 : 1;
    }
    if (balance) {
        const long long ng = ((long long)h->E + C::EPB - 1) / C::EPB;
        const long long waves = (ng + grid - 1) / grid;
        const long long g = waves > 0 ? (ng + waves - 1) / waves : grid;
        if (g >= 1 && g < grid && balanced_sm_max(ng, g, h->sm_count) <= balanced_sm_max(ng, grid, h->sm_count))
            grid = (int)g;
    }
    // Per-SM split (grp_range, nb_cg.cuh; the blocks find their SM at the start of the solve): the full
    // grid with every SM's share of the groups split over its resident blocks, where that lowers the
    // busiest SM's group count against occ blocks of the (balanced) grid's busiest kind (configs[1] in
    // single precision: 7 instead of 2 x 4 groups).  NB_SM_SPLIT=0: off.
    static int smsplit = -1;
    if (smsplit < 0) {
        const char *s = std::getenv("NB_SM_SPLIT");
        smsplit = (s && s[0] == '0') ? 0 : 1;
    }
    a2.sm_split = 0;
    if (smsplit && h->sm_count > 0 && h->sm_count < SMID_MAX && full > h->sm_count && full % h->sm_count == 0) {
        const long long ng = ((long long)h->E + C::EPB - 1) / C::EPB;
        const long long per_sm = (ng + h->sm_count - 1) / h->sm_count;
        const long long occ = full / h->sm_count;
        if (ng >= full && per_sm < occ * ((ng + grid - 1) / grid)) {
            grid = full;
            a2.sm_split = h->sm_count;
        }
    }
    return cudaLaunchCooperativeKernel((const void *)k_cg_mega<PREC, N, FUSED, VAR>, dim3(grid), dim3(C::NT), params,
                                       (size_t)SMEM_MEGA, st);
}

template <int PREC, int VAR>
cudaError_t launch_cg_mega_var(const nb_handle *h, const MegaArgs &A, bool fused, cudaStream_t st)
{
    if (fused) { NB_DISPATCH_N(h->n, return (mega_launch_t<PREC, NN, 1, VAR>(h, A, st))) }
    NB_DISPATCH_N(h->n, return (mega_launch_t<PREC, NN, 0, VAR>(h, A, st)))
}

template <int PREC>
void fill_mega_args(const nb_handle *h, Workspace &ws, const void *b, int order, int max_iter, double rtol, int precond,
                    int x64, unsigned long long *tim, MegaArgs &A)
{
    A.m = h->md();
    A.b = b;
    A.pc = precond;
    A.x64 = (PREC == NB_MIXED && x64) ? 1 : 0;
    A.phase_only = h->phase_only;
    A.x = A.x64 ? (void *)ws.xd : ws.x; A.p = ws.p; A.r = ws.r; A.w = ws.w;
    A.z = precond == NB_PC_IDENTITY ? ws.r : ws.z;   // identity: z aliases r (never stored)
    A.g = (sizeof(typename Pol<PREC>::TV) == 8) ? (const void *)h->g64 : (const void *)h->g32;
    A.dinv = (sizeof(typename Pol<PREC>::TJ) == 4 || precond == NB_PC_JACOBI_F32) ? (const void *)h->dinv32
                                                                                  : (const void *)h->dinv64;
    A.gs_off = h->gs_off; A.gs_idx = h->gs_idx; A.nseg = (int32_t)h->nseg;
    A.order = order; A.max_iter = max_iter; A.rtol = rtol;
    A.rp = RankPart{1, 1, 1};
    A.hist = ws.hist; A.shist = ws.shist; A.tim = tim;
    // per-block partials: W doubles per accumulator (2 for the Dot2 expansions)
    const size_t W = (size_t)Acc<PREC>::W;
    A.partA = ws.part; A.partS = ws.part + W * ws.mega_G; A.partB = ws.part + 2 * W * ws.mega_G;
    A.bar = ws.bar;
    A.sm_split = 0;
    A.scal = ws.scal;
    A.wlo = ws.peer.wlo;
    A.whi = ws.peer.whi;
}

template <int PREC>
cudaError_t launch_cg_mega(const nb_handle *h, Workspace &ws, const void *b, int order, int max_iter, double rtol,
                           int precond, int x64, unsigned long long *tim, cudaStream_t st, RankPart rp)
{
    MegaArgs A;
    fill_mega_args<PREC>(h, ws, b, order, max_iter, rtol, precond, x64, tim, A);
    A.wlo = A.whi = nullptr;
    A.rp = rp;
    const bool fused = order == NB_GS_CONSISTENT && !h->cg_csr;
    cudaError_t e = cudaMemsetAsync(ws.bar, 0, BAR_WORDS * sizeof(unsigned int), st);   // barrier epoch 0
    if (e != cudaSuccess) return e;
    const bool var = precond != NB_PC_JACOBI || A.x64;
    return var ? launch_cg_mega_var<PREC, 1>(h, A, fused, st) : launch_cg_mega_var<PREC, 0>(h, A, fused, st);
}

// ---- Schwarz-preconditioned solve (k_cg_sw) and solveM alone (k_sw_apply), NEXT-4 ----
// Full occupancy grid (every block resident), at most `gmax` blocks (the workspace's partials).
template <int PREC, int N, bool APPLY, int FUSED>
static cudaError_t sw_launch_t(const nb_handle *h, const MegaArgs &A, int gmax, cudaStream_t st)
{
    using TV = typename Pol<PREC>::TV;
    using C = AxCfg<TV, N>;
    constexpr int SMEM = C::SMEM_CG > SwCfg<TV, N>::SMEM ? C::SMEM_CG : SwCfg<TV, N>::SMEM;
    const void *fn = APPLY ? (const void *)k_sw_apply<PREC, N> : (const void *)k_cg_sw<PREC, N, FUSED>;
    static DevCache cache;
    int &occ = cache.here();
    if (occ < 0) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, C::NT, SMEM);
        occ = o > 0 ? o : 1;
        set_carveout(fn, occ, SMEM);
    }
    int grid = h->sm_count * occ;
    if (gmax > 0 && grid > gmax) grid = gmax;
    const long long ng = ((long long)h->E + C::EPB - 1) / C::EPB;
    if (grid > ng) grid = (int)ng;
    if (grid < 1) grid = 1;
    DMat<TV, N> D = make_dmat<TV, N>(h->D);
    void *params[2] = {(void *)&A, (void *)&D};
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(C::NT), params, (size_t)SMEM, st);
}

template <int PREC>
cudaError_t launch_cg_sw(const nb_handle *h, const MegaArgs &A, int gmax, bool apply_only, cudaStream_t st)
{
    if (apply_only) { NB_DISPATCH_N(h->n, return (sw_launch_t<PREC, NN, true, 1>(h, A, gmax, st))) }
    if (A.order == NB_GS_CONSISTENT && !h->cg_csr) { NB_DISPATCH_N(h->n, return (sw_launch_t<PREC, NN, false, 1>(h, A, gmax, st))) }
    NB_DISPATCH_N(h->n, return (sw_launch_t<PREC, NN, false, 0>(h, A, gmax, st)))
}

// ---- multi-rank (z-slab) megakernel: consistent order, runtime options ----
template <int PREC, int N>
static int mr_occupancy()
{
    using C = AxCfg<typename Pol<PREC>::TV, N>;
    constexpr int SMEM_MEGA = C::SMEM;
    static DevCache cache;
    int &occ = cache.here();
    if (occ < 0) {
        const void *fn = (const void *)k_cg_mega_mr<PREC, N>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MEGA);
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, C::NT, SMEM_MEGA);
        occ = o > 0 ? o : 1;
    }
    return occ;
}

template <int PREC>
int grid_mega_mr(const nb_handle *h)
{
    NB_DISPATCH_N(h->n, return (h->sm_count * mr_occupancy<PREC, NN>()))
}

template <int PREC, int N>
static cudaError_t mr_launch_t(const nb_handle *h, const MultiArgs &M, cudaStream_t st)
{
    using TV = typename Pol<PREC>::TV;
    using C = AxCfg<TV, N>;
    constexpr int SMEM_MEGA = C::SMEM;
    DMat<TV, N> D = make_dmat<TV, N>(h->D);
    void *params[2] = {(void *)&M, (void *)&D};
    (void)mr_occupancy<PREC, N>();
    return cudaLaunchCooperativeKernel((const void *)k_cg_mega_mr<PREC, N>, dim3(M.mr.nloc * M.mr.Gr), dim3(C::NT),
                                       params, (size_t)SMEM_MEGA, st);
}

template <int PREC>
cudaError_t launch_cg_mr(const nb_handle *h0, const MultiArgs &M, cudaStream_t st)
{
    NB_DISPATCH_N(h0->n, return (mr_launch_t<PREC, NN>(h0, M, st)))
}

}  // namespace nb
