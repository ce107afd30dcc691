/*
 * nb.h -- C ABI of the B200 (sm_100a) Nekbone-style mixed-precision SEM Jacobi-PCG.
 *
 * The only public header.  C99; no C++ or torch types cross it.  Every entry
 * point returns an nb_status code and never aborts or throws; on a non-OK
 * return nb_last_error() gives a thread-local message.
 *
 * What is computed (arxiv 2503.02134, PAPER.md):
 *   - the Nekbone CG loop of Table 2 (:158-168): solveM (Jacobi, :444), glsc3,
 *     add2s1, ax, glsc3, add2s2 x2, glsc3;
 *   - ax = per-element local_grad3 / geometric scaling / local_grad3_t (:147),
 *     followed by gather-scatter "to ensure continuity" of the unassembled
 *     per-element representation (:404) and the Dirichlet mask;
 *   - under three precision policies: fp64, fp32, and the paper's mixed
 *     strategy "single precision PCG loop with the global communication via
 *     the Gather-Scatter library performed in double" plus double dot products
 *     and preconditioner (:53, :429-431, :537; BASELINE.json north_star).
 * Readings where the paper is silent (mesh, deformation, numbering, RHS,
 * stopping rule) are SURVEY.md §8(c) C-1..C-17 and are listed in DESIGN.md §3.
 *
 * Conventions shared by every call:
 *   - Local ("L-vector") layout: n = p+1, index
 *     l = e*n^3 + i + n*j + n^2*k, element e = ex + nelx*(ey + nely*ez).
 *     A vector has n_local contiguous entries (double for NB_FP64, float for
 *     NB_FP32 / NB_MIXED).
 *   - Device pointers must be 16-byte aligned and point into memory of the
 *     handle's device.  The caller owns every vector it passes; the library
 *     never frees or retains them past the call.
 *   - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *     nb_rhs / nb_ax / nb_dssum are asynchronous on it; nb_cg returns after
 *     the solve has finished (its report is host data).
 *   - A handle is not re-entrant: one call in flight per handle.
 */
#ifndef NB_H
#define NB_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nb_handle nb_handle;

/* Precision policy: selects both element type and arithmetic.
 *   NB_FP64 : double data, double arithmetic everywhere.
 *   NB_FP32 : float data, float arithmetic, float gather-scatter accumulation,
 *             float dot products and scalars, float Jacobi copy.
 *   NB_MIXED: float data and float Ax arithmetic; gather-scatter accumulated in
 *             double and rounded once to float; Jacobi z = (float)((double)r * dinv64);
 *             glsc3 products and accumulation and the CG scalars in double. */
/*   NB_FP32_DOT2: the NB_FP32 policy with every glsc3 (pap, rtr, rho) computed by the
 *             compensated Dot2 (TwoProduct/TwoSum error-free transformations in binary32,
 *             block and grid partials combined as expansions of size two) -- PAPER.md:434,
 *             Sec. 5.2.1; SURVEY.md §8(f) NEXT-1.  For nb_rhs / nb_ax / nb_dssum it is NB_FP32. */
typedef enum { NB_FP64 = 0, NB_FP32 = 1, NB_MIXED = 2, NB_FP32_DOT2 = 3 } nb_policy;

/* Gather-scatter summation order:
 *   NB_GS_CONSISTENT: one sum per shared global node, copies ascending, written to all copies.
 *   NB_GS_PER_COPY  : copy l receives w_l + sum_{m != l, ascending} w_m, emulating the
 *                     pairwise exchange mode whose fp32 stagnation the paper reports
 *                     (Table 3) with every element its own rank.
 *   NB_GS_PAIRWISE / NB_GS_ALLREDUCE: the gather-scatter of a run whose
 *                     elements are split over px x py x pz ranks (contiguous blocks as even as
 *                     possible: block b of an axis holds elements [b nel/P, (b+1) nel/P)).  Each
 *                     rank sums its own copies of a node (ascending local index) into a partial P_q
 *                     in the GS precision; PAIRWISE: a copy on rank r receives P_r + sum over the
 *                     other ranks q ascending of P_q (gslib's pairwise exchange: each rank adds its
 *                     neighbours' contributions to its own); ALLREDUCE: every copy receives
 *                     sum over q ascending of P_q (one global reduction).  PAPER.md:339-341, Table 3.
 *                     Emulated in one launch on one GPU (the partition is logical). */
typedef enum { NB_GS_CONSISTENT = 0, NB_GS_PER_COPY = 1, NB_GS_PAIRWISE = 2, NB_GS_ALLREDUCE = 3 } nb_gs_order;

/* Right-hand sides, generated in fp64 and cast once:
 *   NB_RHS_UNIFORM     : b_l = mask_l * U(seed, 1, gid_l), U the counter SplitMix64 in [-1,1).
 *   NB_RHS_MANUFACTURED: b = mask . QQ^T (B . f), f = 3 pi^2 sin(pi x) sin(pi y) sin(pi z)
 *                        + noise_amp * U(seed, 2, gid). */
typedef enum { NB_RHS_UNIFORM = 0, NB_RHS_MANUFACTURED = 1 } nb_rhs_kind;

typedef enum {
    NB_OK = 0,
    NB_EINVAL = 1,      /* bad sizes/arguments, NULL or misaligned pointers, p outside [1,15] */
    NB_ENOMEM = 2,      /* device or host allocation failed */
    NB_ECUDA = 3,       /* CUDA runtime error; message in nb_last_error() */
    NB_EGEOM = 4,       /* non-positive Jacobian or Jacobi diagonal at setup */
    NB_EBREAKDOWN = 5,  /* pap <= 0 with rtr > 0, or a non-finite scalar */
    NB_ESTATE = 6,      /* handle destroyed / used from the wrong device; a peer-attached handle
                           whose last multi-rank solve aborted (nb_peer_detach + attach again) */
    NB_ETIMEOUT = 7     /* multi-rank solve: a peer rank did not arrive within NB_PEER_TIMEOUT_MS
                           (default 20000 ms) or another rank gave up; the solve stopped on every
                           rank (no hang) and the attachment must be renewed */
} nb_status;

/* nb_cg_report.status (stagnation is NB_OK with status NB_STAGNATED) */
enum { NB_CONVERGED = 0, NB_MAXITER = 1, NB_STAGNATED = 2, NB_BROKEDOWN = 3 };

/* nb_ax flags */
enum { NB_AX_LOCAL = 1u };   /* w = A_L u only: no gather-scatter, no mask */

typedef struct {
    int64_t E, n_local, n_global, n_unmasked, n_shared_global, n_shared_copies;  /* E, n_local, n_shared_*:
                                            this handle's slab; n_global, n_unmasked: the whole box */
    int32_t p, nelx, nely, nelz;           /* nelz: the whole box */
    int32_t ez0, nelz_local;               /* the slab's first z layer and layer count (box: 0, nelz) */
} nb_info;

/* Preconditioner of nb_cg:
 *   NB_PC_JACOBI    : the policy's Jacobi z = M^-1 r (C-10 table: fp64 diagonal for NB_FP64 and
 *                     NB_MIXED, its one-time float copy for NB_FP32 / NB_FP32_DOT2).
 *   NB_PC_IDENTITY  : none, z = r -- "CG with the identity ... preconditioner".
 *   NB_PC_JACOBI_F32: Neko's "single precision copy of the preconditioner":
 *                     z = r * (float)dinv in binary32.  Same as NB_PC_JACOBI for NB_FP32 /
 *                     NB_FP32_DOT2; NB_EINVAL for NB_FP64.
 *   NB_PC_SCHWARZ   : the two-level overlapping Schwarz preconditioner of SURVEY.md §8(f) NEXT-4
 *                     (reading 28; Nekbone's multigrid-preconditioned CG, PAPER.md:160,
 *                     :324-328, :537, :704-709): M^-1 = sum_e R_e^T W K_e^-1 W R_e + Phi A0^-1 Phi^T,
 *                     local solves on the element boxes extended by one GLL layer by fast
 *                     diagonalisation, weights W = 1/sqrt(overlap count) ("the square roots"),
 *                     Galerkin coarse level on the interior element vertices.  Precision: the
 *                     policy's vector type for the fast-diagonalisation arithmetic; square roots,
 *                     weights and the sums over subdomains in the gather-scatter precision (fp64
 *                     under NB_MIXED, the paper's "sqrt and GS in fp64").  Whole-box handles
 *                     (NB_EINVAL otherwise); every gs_order: the per-copy / pairwise / allreduce
 *                     orders also combine the overlapping local solutions at each copy in that
 *                     order (own element's / own rank's contribution first, ...). */
typedef enum { NB_PC_JACOBI = 0, NB_PC_IDENTITY = 1, NB_PC_JACOBI_F32 = 2, NB_PC_SCHWARZ = 3 } nb_precond;

typedef struct {
    nb_policy policy;
    int32_t max_iter;          /* >= 0 */
    double rtol;               /* stop when sqrt(rtr/rtr0) <= rtol; 0 = run exactly max_iter */
    nb_gs_order gs_order;
    int32_t stag_window;       /* C-11 window W (default 200 when <= 0) */
    int32_t reserved0;         /* must be 0 */
    double *rel_res_history;   /* host, length max_iter+1, nullable: [0] = 1, [k] = sqrt(rtr_k/rtr0) */
    nb_precond precond;        /* 0 = NB_PC_JACOBI (zero-initialised options keep the default) */
    int32_t x_fp64;            /* NB_MIXED only (else NB_EINVAL): x += alpha p accumulated in double
                                  with the double alpha, and x returned as n_local DOUBLES (C-15 variant) */
    double *scal_history;      /* host, length 3*max_iter, nullable: for k = 1..iterations,
                                  [3(k-1) + 0..2] = rho_k, alpha_k, beta_k of Table 2
                                  as the policy computes them: binary64 under NB_FP64 / NB_MIXED,
                                  binary32 (widened exactly) under NB_FP32 / NB_FP32_DOT2 (C-10 table) */
    int32_t ranks[3];          /* px, py, pz of gs_order NB_GS_PAIRWISE / NB_GS_ALLREDUCE (0 = 1) */
} nb_cg_opts;

typedef struct {
    int32_t iterations;        /* completed CG iterations */
    int32_t status;            /* NB_CONVERGED / NB_MAXITER / NB_STAGNATED / NB_BROKEDOWN */
    double rtr0, rtr_final, rel_res_final, rel_res_min;
    double solve_ms;           /* device time of the solve (CUDA events on the caller stream) */
    int64_t kernel_launches;   /* kernels of this library launched by the solve */
    double k_ax_ms, k_gs_ms, k_upd_ms;  /* summed per-phase device time over the iterations (block 0's
                                           %globaltimer stamps after each grid barrier of the
                                           megakernel): phase A (p update + Ax), the CSR gather-
                                           scatter phase (per-copy order only), phase B (gather +
                                           update + dots) */
} nb_cg_report;

/* Build the box mesh [0,1]^3 of nelx*nely*nelz hexes of order p on `device`
 * (SURVEY.md C-1..C-9): GLL nodes/weights/D, deformed trilinear geometry
 * (deform_amp = vertex amplitude as a fraction of element size, 0 = undeformed;
 * phases seeded by `seed`), g1..g6 and B, numbering, mask, GS segments and the
 * Jacobi diagonal.  All device data is allocated here and owned by the handle.
 * Errors: NB_EINVAL (p not in [1,15], nel < 1, n_local >= 2^31), NB_ENOMEM, NB_ECUDA, NB_EGEOM. */
int nb_setup(int32_t nelx, int32_t nely, int32_t nelz, int32_t p, double deform_amp, uint64_t seed,
             int32_t device, nb_handle **out);
int nb_destroy(nb_handle *h);                 /* NULL is a no-op; frees all device memory */

/* A z-slab of the same box for multi-GPU runs: the elements with
 * ez0 <= ez < ez1 (element e = ex + nelx*(ey + nely*(ez - ez0)) locally, vectors hold only them).
 * Global numbering, mask, multiplicity c and geometry are those of the whole box; the Jacobi
 * diagonal and the manufactured RHS include the neighbour slabs' contributions (computed
 * redundantly on a one-ghost-layer twin, bit-identical to the whole box).  nb_ax / nb_dssum act
 * on the slab alone; nb_cg on a slab needs its neighbours: nb_cg_group (slabs on one device, one
 * launch) or nb_peer_attach (one slab per process/GPU).  nb_setup = nb_setup_slab(.., 0, nelz, ..).
 * Errors as nb_setup, plus NB_EINVAL unless 0 <= ez0 < ez1 <= nelz. */
int nb_setup_slab(int32_t nelx, int32_t nely, int32_t nelz, int32_t ez0, int32_t ez1, int32_t p,
                  double deform_amp, uint64_t seed, int32_t device, nb_handle **out);
int nb_query(const nb_handle *h, nb_info *out);   /* sizes of the handle's mesh (nb_info) */

/* Fill device vector b (policy precision of `prec`) with a right-hand side. Async. */
int nb_rhs(nb_handle *h, nb_rhs_kind kind, double noise_amp, uint64_t seed, nb_policy prec,
           void *b, void *stream);

/* w = mask . QQ^T A_L u  (or w = A_L u with NB_AX_LOCAL).  u, w: device, distinct,
 * precision of `prec` (NB_MIXED: float data, float Ax, double GS accumulation).  Async.
 * PAPER.md:163 ("call ax(w,p,g,ur,us,ut,wk,n)"), :147. */
int nb_ax(nb_handle *h, nb_policy prec, const void *u, void *w, uint32_t flags, void *stream);

/* In place u = QQ^T u over the shared-node segments (no mask).  Async.  PAPER.md:309, :404.
 * order NB_GS_PAIRWISE / NB_GS_ALLREDUCE need a partition: nb_dssum_ranked. */
int nb_dssum(nb_handle *h, nb_policy prec, nb_gs_order order, void *u, void *stream);
/* Same with the rank partition px x py x pz of the NB_GS_PAIRWISE / NB_GS_ALLREDUCE orders
 * (NB_EINVAL unless 1 <= p_a <= nel_a; the handle must hold the whole box). */
int nb_dssum_ranked(nb_handle *h, nb_policy prec, nb_gs_order order, int32_t px, int32_t py, int32_t pz,
                    void *u, void *stream);

/* Jacobi-PCG (Table 2 order) from x0 = 0.  b, x: device vectors in the
 * policy precision (x: double when o->x_fp64); b must be continuous and masked (e.g. from
 * nb_rhs).  Blocks until done.  The graph driver (env NB_CG_DRIVER=graph) supports the default
 * options only (policies 0-2, NB_PC_JACOBI, x_fp64 = 0): NB_EINVAL otherwise.  The default
 * driver sizes its persistent grid to balance element groups per block (env NB_GRID_BALANCE=0:
 * full occupancy grid); the grid changes only the summation order of the dot-product partials.
 * Returns NB_OK for converged / max_iter / stagnated runs, NB_EBREAKDOWN on breakdown
 * (report filled in either case); NB_EINVAL for bad options or a mesh without unknowns
 * (every node on the Dirichlet boundary, e.g. p = 1 with one element along an axis). */
int nb_cg(nb_handle *h, const nb_cg_opts *o, const void *b, void *x, nb_cg_report *rep, void *stream);

/* solveM alone (Table 2 line 2): z = M^-1 r for `pc` = NB_PC_SCHWARZ (the NEXT-4
 * preconditioner of nb_cg, same arithmetic).  r, z: device, distinct, policy precision; r must be
 * continuous and masked.  Builds the handle's Schwarz tables on first use (synchronizes then).
 * One cooperative launch.  Errors: NB_EINVAL (other pc, slab handle, aliasing), NB_ECUDA. */
int nb_precond_apply(nb_handle *h, nb_policy prec, nb_precond pc, const void *r, void *z, void *stream);

/* Same solve with HOST buffers (pinned or pageable): copies b in and x out on `stream`. */
int nb_cg_host(nb_handle *h, const nb_cg_opts *o, const void *b_host, void *x_host,
               nb_cg_report *rep, void *stream);

/* ---- multi-rank z-slab solves (slabs from nb_setup_slab) ----
 * The z-slabs of one box are solved together: Ax stays slab-local; the phase-B gather reads
 * the neighbour slabs' w of the interface layers directly (peer memory over NVLink, or plain
 * device memory for slabs on one GPU), and the three dot products are reduced per rank, the
 * rank partials pushed into every rank's control block and merged in rank order (every rank
 * takes bit-identical scalar decisions).  Consistent GS order, fused megakernel only
 * (NB_EINVAL otherwise); the per-slab reports carry the same iterations/status/residuals. */

/* Slabs of one box that share a GPU (1 <= nslab <= 4, bottom to top, tiling the box): one
 * cooperative launch over all of them.  b[r], x[r]: slab r's device vectors; reps: nslab reports.
 * This is also how the multi-rank path is verified on one GPU. */
int nb_cg_group(nb_handle *const *hs, int32_t nslab, const nb_cg_opts *o, const void *const *b,
                void *const *x, nb_cg_report *reps, void *stream);

/* One slab per process/GPU: each rank exports an NB_PEER_BLOB_BYTES blob (CUDA IPC handles of
 * its policy workspace's w and control block), the blobs are exchanged (e.g. all_gather over
 * torch.distributed), and every rank attaches with all nrank blobs in rank order (rank r holds
 * the r-th slab from the bottom).  Afterwards nb_cg / nb_cg_host on this handle and policy run the
 * multi-rank solve; every rank must call them with the same options.  All ranks must attach before
 * any rank solves.  Errors: NB_EINVAL (bad blobs, slabs not tiling the box), NB_ECUDA (IPC). */
#define NB_PEER_BLOB_BYTES 256
int nb_peer_export(nb_handle *h, nb_policy policy, void *blob);
int nb_peer_attach(nb_handle *h, nb_policy policy, int32_t nrank, int32_t rank, const void *blobs);
int nb_peer_detach(nb_handle *h, nb_policy policy);

/* Host copies of the integer maps (caller-allocated host arrays, each nullable):
 * gid[n_local], mask[n_local], gs_off[n_shared_global+1], gs_idx[n_shared_copies]. */
int nb_export_maps(const nb_handle *h, int64_t *gid, uint8_t *mask, int32_t *gs_off, int32_t *gs_idx);
/* Host copies of the fp64 setup data (nullable): g6[6*n_local] factor-major (g1..g6 each
 * n_local long, C-6 ordering g1=Grr,g2=Grs,g3=Grt,g4=Gss,g5=Gst,g6=Gtt), B, dinv[n_local]. */
int nb_export_geom(const nb_handle *h, double *g6, double *B, double *dinv);
/* GLL nodes[p+1], weights[p+1], D[(p+1)^2] (row-major, D[i*(p+1)+j] = l_j'(x_i)). */
int nb_export_basis(const nb_handle *h, double *nodes, double *weights, double *D);

const char *nb_last_error(void);
const char *nb_version(void);

#ifdef __cplusplus
}
#endif
#endif
