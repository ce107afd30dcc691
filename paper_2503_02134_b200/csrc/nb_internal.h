// nb_internal.h -- private declarations shared by the host layer (nb_api.cu) and the
// kernel translation units.  No torch, no oracle.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "nb.h"

namespace nb {

struct SwState;   // NB_PC_SCHWARZ host state (nb_sw_setup.cu)

// Device-resident CG scalars.  Values of the policy's scalar
// precision (float under NB_FP32, double otherwise) are stored widened to double.
struct Scal {
    double rho;        // rho_k = glsc3(r, c, z) for the next p update
    double beta;       // beta used by the next p update
    double alpha;      // alpha of the last completed pap
    double pap;
    double rtr;        // rtr after the last update
    double rtr0;
    double rtol;
    int32_t iter;      // completed iterations
    int32_t max_iter;
    int32_t done;      // 1: no further updates (kernels no-op)
    int32_t status;    // NB_CONVERGED / NB_MAXITER / NB_BROKEDOWN (stagnation decided on host)
    int32_t pending;   // 1: x += alpha*p of the last iteration not yet applied (deferred x update)
    int32_t epochs;    // multi-rank megakernel: cross-rank barrier epochs used by the solve
    int32_t aborted;   // multi-rank megakernel: a cross-rank wait timed out or a rank aborted
};

// Multi-rank (z-slab) solves: ranks per solve, slabs per launch (one GPU)
constexpr int NB_MAX_RANKS = 8;
constexpr int NB_MAX_DEVICES = 64;   // per-device caches of kernel residency
constexpr int NB_MAX_LOCAL = 4;
// per-rank control block (peer-visible): arrival flag (offset 0), abort word (offset 64), then
// rank-partial slots [2 parities][NB_MAX_RANKS][4 doubles] (K <= 2 accumulators x W <= 2 doubles)
constexpr int NB_CTL_FLAG_BYTES = 128;
constexpr int NB_CTL_ABORT_OFF = 64;
constexpr int NB_CTL_BYTES = NB_CTL_FLAG_BYTES + 2 * NB_MAX_RANKS * 4 * 8;
struct PeerState {
    int32_t nrank = 0, rank = 0;       // nrank 0: not attached
    const void *wlo = nullptr, *whi = nullptr;   // neighbours' w (below / above), rebased (nb_cg.cuh)
    unsigned int *flag[NB_MAX_RANKS] = {};
    unsigned int *abrt[NB_MAX_RANKS] = {};
    double *slot[NB_MAX_RANKS] = {};
    bool broken = false;               // a solve aborted: flags/epochs out of step, re-attach needed
    uint32_t epoch = 0;                // cross-rank barrier epochs completed by earlier solves
    void *opened[NB_MAX_RANKS + 2] = {};   // IPC mappings to close
    int nopened = 0;
};

// Rank partition of the NB_GS_PAIRWISE / NB_GS_ALLREDUCE gather-scatter orders (NEXT-2)
struct RankPart {
    int32_t px, py, pz;
};

// Geometry needed by kernels, passed by value.
struct MeshDev {
    int32_t nelx, nely, nelz, p, n;   // the whole box (nelz: global layer count)
    int32_t E;                        // elements held here (a z-slab of the box, or all of it)
    int64_t NL, NX, NY, NZ, NG;       // NL local; NX, NY, NZ, NG: the global node lattice
    int32_t nseg;
    int32_t ez0, nelzl;               // slab: first global z layer and layer count (box: 0, nelz)
    int64_t NZl, NGl;                 // the slab's own node lattice (its GS segments)
};

// Two-level Schwarz preconditioner (NEXT-4, nb_schwarz.cuh / nb_sw_setup.cu): device tables and
// scratch of one handle and policy.  P3 = p + 3 points per axis of an extended element box.
struct SwArgs {
    int32_t on;                 // 1: tables valid (nb_cg with NB_PC_SCHWARZ, nb_precond_apply)
    int32_t nv[3];              // interior element vertices per axis (nel_a - 1); coarse level iff all > 0
    const uint8_t *cs[3];       // [nel_a]: case (1-D table) of each element position along axis a
    const uint8_t *cnt[3];      // [nel_a][P3]: overlap count of the extended point (0: not an unknown)
    const void *S[3];           // [ncase_a][P3][P3] (TV): fast-diagonalisation eigenvectors, row = point
    const double *lam[3];       // [ncase_a][P3]: eigenvalues (padded modes: 1)
    const void *S0[3];          // [nv_a][nv_a] (TV): coarse eigenvectors
    const double *lam0[3];      // [nv_a]
    const double *phL, *phR;    // [p+1]: (1 - xi_i)/2, (1 + xi_i)/2 at the GLL points
    void *zext;                 // [E][P3^3] (TV): unweighted local solutions
    void *cpart;                // [E][8] (TG): coarse restriction partials, element corners
    void *c0, *c1;              // [V] (TV): coarse vectors (b0 / transforms; x0 ends in c0)
};

// Arguments of the persistent CG megakernel (nb_cg.cuh), one slab's (or the whole box's) solve
constexpr int SMID_MAX = 1024;            // SM ids tracked by the per-SM split
constexpr int BAR_WORDS = 2 + SMID_MAX;   // Workspace::bar

struct MegaArgs {
    MeshDev m;
    const void *b;
    void *x, *p, *r, *z, *w;
    const void *g, *dinv;
    const int32_t *gs_off, *gs_idx;
    int32_t nseg;
    int32_t order;          // NB_GS_CONSISTENT / NB_GS_PER_COPY / NB_GS_PAIRWISE / NB_GS_ALLREDUCE
    RankPart rp;            // partition of the ranked orders
    int32_t max_iter;
    double rtol;
    double *hist;           // [max_iter + 1]
    double *shist;          // nullable: [3 * max_iter] rho_k, alpha_k, beta_k (block 0)
    unsigned long long *tim;  // nullable: [3 * (max_iter + 1)] globaltimer stamps (block 0)
    double *partA, *partS, *partB;   // per-block partials, [G], [G], [2G] (x Acc::W)
    int32_t pc;             // nb_precond (z aliases r for the identity)
    int32_t x64;            // NB_MIXED: x is double (x_fp64 option)
    int32_t phase_only;     // measurement only (NB_PHASE_ONLY=A|B at setup): 1 = phase A alone,
                            // 2 = phase B alone, max_iter iterations, no stop test (ncu traffic per phase)
    unsigned int *bar;      // [BAR_WORDS] grid barrier: arrival count, generation; then the resident-block
                            // count of every SM id (sm_split), all zeroed before the launch
    int32_t sm_split;       // S > 0 (a full grid of occ * S blocks): the element groups are split per SM first
                            // and each SM's contiguous share over the blocks resident on it (the blocks find
                            // their SM and slot at the start of the solve; grp_range()); 0: per block
    Scal *scal;             // result scalars (written by block 0)
    // multi-rank (z-slab) solves only: the neighbour slabs' w, rebased so that the element
    // index of this slab addresses them (wlo + e*N3 for e < 0, whi + e*N3 for e >= E); else null
    const void *wlo, *whi;
    SwArgs sw;              // NB_PC_SCHWARZ solves (k_cg_sw) only
};

// Multi-rank solve over z-slabs: every rank's block 0 pushes its rank partial
// into every rank's control block (peer stores over NVLink, or plain stores when the slabs share
// a GPU), then bumps every rank's arrival flag; the phase-B gather reads the neighbour slabs'
// w directly from peer memory.  Flags count monotonically across solves (epoch0).
struct MrArgs {
    int32_t nrank;           // ranks R of the solve
    int32_t rank0;           // global rank of this launch's first slab
    int32_t nloc;            // slabs in this launch (1: one per GPU; >1: slabs sharing this GPU)
    int32_t Gr;              // blocks per slab
    uint32_t epoch0;         // barrier epochs completed by earlier solves
    int32_t sys;             // 1: ranks on other GPUs (system-scope flags); 0: all in this launch
    unsigned long long timeout_ns;   // bound of every cross-rank wait (NB_PEER_TIMEOUT_MS)
    unsigned int *flag[NB_MAX_RANKS];
    unsigned int *abrt[NB_MAX_RANKS];   // abort words: a rank that gives up tells every rank
    double *slot[NB_MAX_RANKS];
};
struct MultiArgs {
    MegaArgs a[NB_MAX_LOCAL];
    MrArgs mr;
};

struct Workspace {          // per-policy CG workspace (lazily allocated)
    bool ready = false;
    void *r = nullptr, *p = nullptr, *w = nullptr, *x = nullptr, *z = nullptr;
    double *xd = nullptr;       // x accumulated in double (x_fp64 option), lazily allocated
    unsigned char *ctl = nullptr;   // multi-rank control block (NB_CTL_BYTES), lazily allocated
    PeerState peer;
    double *part = nullptr;     // megakernel per-block partials
    Scal *scal = nullptr;       // device scalars
    Scal *scal_host = nullptr;  // pinned mirror
    double *hist = nullptr;     // device history, capacity hist_cap
    double *shist = nullptr;    // device scalar history [3 * hist_cap] (rho, alpha, beta)
    int32_t hist_cap = 0;
    // megakernel: grid size, barrier words [2], globaltimer stamps [3 * hist_cap]
    int32_t mega_G = 0;
    unsigned int *bar = nullptr;
    unsigned long long *tim = nullptr;
};

}  // namespace nb

struct nb_handle {
    int32_t device;
    int32_t nelx, nely, nelz, p, n;   // nelz: the whole box
    int32_t ez0 = 0, nelzl = 0;       // z-slab held by this handle
    int64_t E, NL, NX, NY, NZ, NG;    // E, NL: the slab's; NX..NG: the global lattice
    int64_t NZl = 0, NGl = 0;         // the slab's node lattice
    nb_handle *ext = nullptr;         // slab with one ghost layer per side (setup data: diag, rhs)
    int64_t ext_off = 0;              // first owned element inside ext
    int64_t n_unmasked, nseg, ncopies;
    double deform;
    uint64_t seed;
    double nodes[16], weights[16], D[256];
    int sm_count;
    // device data owned by the handle
    double *g64 = nullptr;      // [E][6][n^3]
    float *g32 = nullptr;       // one-time cast, lazily
    double *B = nullptr;        // [NL]
    double *dinv64 = nullptr;   // [NL]
    float *dinv32 = nullptr;    // lazily
    int32_t *gs_off = nullptr;  // [nseg+1]
    int32_t *gs_idx = nullptr;  // [ncopies]
    int32_t *flag = nullptr;    // device error flags for setup checks
    cudaStream_t cap_stream = nullptr;   // private stream used for setup
    int cg_csr = 0;             // 1: consistent-order CG also through the CSR dssum kernel (A/B)
    int phase_only = 0;         // NB_PHASE_ONLY=A (1) / B (2): measurement runs of one megakernel phase
    int dssum_csr = 0;          // NB_DSSUM=csr: consistent nb_dssum through the CSR kernel (A/B, tests)
    nb::Workspace ws[4];   // one per nb_policy
    nb::SwState *sw = nullptr;      // NB_PC_SCHWARZ tables and scratch (nb_sw_setup.cu), lazily
    nb::MeshDev md() const {
        nb::MeshDev m;
        m.nelx = nelx; m.nely = nely; m.nelz = nelz; m.p = p; m.n = n;
        m.E = (int32_t)E; m.ez0 = ez0; m.nelzl = nelzl;
        m.NL = NL; m.NX = NX; m.NY = NY; m.NZ = NZ; m.NG = NG; m.NZl = NZl; m.NGl = NGl;
        m.nseg = (int32_t)nseg;
        return m;
    }
};

namespace nb {

// C-3 deformation phases phi_a = pi (1 + U(seed, 3, a)) (host, nb_api.cu)
void deform_phases(uint64_t seed, double ph[3]);

// ---- setup launchers (nb_setup_k.cu), asynchronous on `st` unless stated ----
cudaError_t launch_geometry(const nb_handle *h, const double phi[3], cudaStream_t st);
cudaError_t launch_jacobi(nb_handle *h, double *diag_scratch, cudaStream_t st);
cudaError_t build_gs(nb_handle *h, cudaStream_t st);   // allocates gs_off/gs_idx (synchronizes)
cudaError_t launch_cast(const double *src, float *dst, int64_t n, cudaStream_t st);
cudaError_t launch_maps(const nb_handle *h, int64_t *gid, uint8_t *mask, cudaStream_t st);
cudaError_t launch_rhs(const nb_handle *h, int kind, double noise, uint64_t seed, int prec,
                       void *b, cudaStream_t st);

// ---- CSR gather-scatter (nb_gs.cu) ----
int grid_gs(const nb_handle *h);
cudaError_t launch_dssum(const nb_handle *h, int prec, int order, void *u, cudaStream_t st,
                         RankPart rp = RankPart{1, 1, 1});

// ---- Ax + CG kernels, one translation unit per policy (nb_cg_<policy>.cu) ----
template <int PREC> cudaError_t launch_ax_local(const nb_handle *h, const void *u, void *w, bool mask, cudaStream_t st);
// the whole solve as one persistent cooperative kernel (grid size: grid_mega)
template <int PREC> int grid_mega(const nb_handle *h);
struct MegaArgs;
struct MultiArgs;
template <int PREC, int VAR> int grid_mega_var(const nb_handle *h);
// multi-rank (z-slab) solves: args of one slab, grid of one GPU, the launch (nb_mega_launch.cuh)
template <int PREC>
void fill_mega_args(const nb_handle *h, Workspace &ws, const void *b, int order, int max_iter, double rtol,
                    int precond, int x64, unsigned long long *tim, MegaArgs &A);
template <int PREC> int grid_mega_mr(const nb_handle *h);
// NB_PC_SCHWARZ: the Schwarz-preconditioned solve (k_cg_sw) or solveM alone (k_sw_apply)
template <int PREC>
cudaError_t launch_cg_sw(const nb_handle *h, const MegaArgs &A, int gmax, bool apply_only, cudaStream_t st);
// Schwarz tables of the handle + the policy's scratch (nb_sw_setup.cu); fill / free
int sw_ensure(nb_handle *h, int prec, const char **msg);   // NB_OK or an nb_status (msg set)
void sw_fill(const nb_handle *h, int prec, SwArgs &a);
void sw_free(nb_handle *h);
template <int PREC> cudaError_t launch_cg_mr(const nb_handle *h0, const MultiArgs &M, cudaStream_t st);
template <int PREC, int VAR>
cudaError_t launch_cg_mega_var(const nb_handle *h, const MegaArgs &A, bool fused, cudaStream_t st);
template <int PREC> cudaError_t launch_cg_mega(const nb_handle *h, Workspace &ws, const void *b, int order,
                                              int max_iter, double rtol, int precond, int x64,
                                              unsigned long long *tim, cudaStream_t st, RankPart rp);

}  // namespace nb
