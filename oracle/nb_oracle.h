/*
 * nb_oracle.h -- TEST INFRASTRUCTURE ONLY (parity oracle).
 *
 * Plain, slow, single-threaded C implementation of the Nekbone-style
 * Jacobi-preconditioned CG solve of the spectral-element Poisson operator
 * (arxiv 2503.02134, Table 2) under the three precision
 * policies of SURVEY.md §8(c) C-10.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this.  It
 * shares no code with the CUDA path (paper_2503_02134_b200/csrc) and the
 * CUDA path never links or calls it.
 *
 * Built with: gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared
 * (no FMA contraction, C float/double exactly as each policy states).
 */
#ifndef NB_ORACLE_H
#define NB_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* OR_FP32_DOT2: the fp32 policy with every glsc3 computed by the
 * compensated Dot2 in binary32. */
enum { OR_FP64 = 0, OR_FP32 = 1, OR_MIXED = 2, OR_FP32_DOT2 = 3 };
/* OR_GS_PAIRWISE / OR_GS_ALLREDUCE: the gather-scatter of a rank-partitioned
 * run (partition set by or_set_ranks; Table 3). */
enum { OR_GS_CONSISTENT = 0, OR_GS_PER_COPY = 1, OR_GS_PAIRWISE = 2, OR_GS_ALLREDUCE = 3 };
enum { OR_RHS_UNIFORM = 0, OR_RHS_MANUFACTURED = 1 };
enum { OR_CONVERGED = 0, OR_MAXITER = 1, OR_STAGNATED = 2, OR_BREAKDOWN = 3 };

typedef struct or_mesh or_mesh;

typedef struct {
    int32_t iterations;
    int32_t status;
    double rtr0, rtr_final, rel_res_final, rel_res_min;
    double true_res;   /* ||b - A x||_c / ||b||_c in fp64 at exit (C-14, report only) */
} or_report;

/* C-1: GLL nodes/weights and derivative matrix D[i*(p+1)+j]; returns 0 on success. */
int or_gll(int p, double *nodes, double *weights, double *D);

/* C-2..C-9: box mesh [0,1]^3 of nelx*nely*nelz hexes, order p, vertex deformation. NULL on error. */
or_mesh *or_mesh_new(int nelx, int nely, int nelz, int p, double deform_amp, uint64_t seed);
void or_mesh_free(or_mesh *m);
/* info[0..7] = E, n_local, n_global, n_unmasked, n_shared_global, n_shared_copies, p, min J sign ok */
void or_mesh_info(const or_mesh *m, int64_t *info);
/* rank partition px x py x pz of the element box for OR_GS_PAIRWISE / OR_GS_ALLREDUCE (default 1x1x1);
 * returns 1 unless 1 <= p_a <= nel_a. */
int or_set_ranks(or_mesh *m, int px, int py, int pz);
void or_export_maps(const or_mesh *m, int64_t *gid, uint8_t *mask, int32_t *gs_off, int32_t *gs_idx);
/* g6: 6*n_local factor-major (g1..g6), B, dinv, c (=1/mult), xyz: 3*n_local (x,y,z factor-major), jac: n_local */
void or_export_geom(const or_mesh *m, double *g6, double *B, double *dinv, double *c, double *xyz, double *jac);

/* C-5: counter-based SplitMix64 uniform in [-1,1). */
uint64_t or_splitmix64(uint64_t seed, uint64_t stream, uint64_t i);
double or_prng_u(uint64_t seed, uint64_t stream, uint64_t i);
void or_rhs(const or_mesh *m, int kind, double noise_amp, uint64_t seed, double *b);

/* C-7: one-element local gradient (fp64), for the u = r pin. */
void or_local_grad3(int p, const double *D, const double *u, double *ur, double *us, double *ut);

/* C-7 local operator A_L (no dssum, no mask). */
void or_ax_local_d(const or_mesh *m, const double *u, double *w);
void or_ax_local_f(const or_mesh *m, const float *u, float *w);
/* C-8 dssum (QQ^T), no mask.  _d: double data/double accumulate; _f: float/float; _fd: float data, double accumulate. */
void or_dssum_d(const or_mesh *m, int order, double *u);
void or_dssum_f(const or_mesh *m, int order, float *u);
void or_dssum_fd(const or_mesh *m, int order, float *u);
/* full operator w = mask . QQ^T A_L u under a policy (fp64 uses the _d arrays, fp32/mixed the _f arrays). */
void or_ax_d(const or_mesh *m, int order, const double *u, double *w);
void or_ax_f(const or_mesh *m, int policy, int order, const float *u, float *w);

/* glsc3 variants (C-10 table). */
double or_glsc3_d(const double *a, const double *c, const double *b, int64_t n);
double or_glsc3_mixed(const float *a, const double *c, const float *b, int64_t n);
float or_glsc3_f_tree(const float *a, const float *c, const float *b, int64_t n);
float or_glsc3_f_seq(const float *a, const float *c, const float *b, int64_t n);
/* error-free transformations and the compensated Dot2 (binary32) */
void or_two_sum_f(float a, float b, float *s, float *e);
void or_two_prod_f(float a, float b, float *p, float *e);
float or_glsc3_f_dot2(const float *a, const float *c, const float *b, int64_t n);

/*
 * C-10 PCG.  b64: fp64 RHS (cast once to the policy precision).  x_out: n_local doubles
 * (the policy-precision solution widened).  hist: nullable, len max_iter+1 (hist[0] = 1).
 * seqdot: fp32 policy uses Nekbone's sequential float dot instead of the pairwise tree.
 * x64: mixed policy keeps x in fp64 (C-15 variant).
 * precond: OR_PC_JACOBI = the policy's Jacobi (C-10 table);
 *   OR_PC_IDENTITY = none, z = r ("CG with the identity ... preconditioner");
 *   OR_PC_JACOBI_F32 = Neko's single-precision copy of the Jacobi diagonal, z = r * (float)dinv in
 *   binary32 -- for fp32/dot2 the same as OR_PC_JACOBI; rejected for fp64;
 *   OR_PC_SCHWARZ = the NEXT-4 two-level Schwarz preconditioner below (the policy's variant).
 * scal: nullable, len 3*max_iter: scal[3(k-1) + 0..2] = rho_k, alpha_k, beta_k of iteration k (the
 *   policy's own scalar values widened to double: binary64 under fp64/mixed, binary32 under fp32).
 * Returns 0, or 1 on bad arguments.
 */
enum { OR_PC_JACOBI = 0, OR_PC_IDENTITY = 1, OR_PC_JACOBI_F32 = 2, OR_PC_SCHWARZ = 3 };
/*
 * NEXT-4: two-level overlapping Schwarz preconditioner z = M^-1 r on the local
 * copies (reading 28):
 *   M^-1 = sum_e R_e^T W K_e^-1 W R_e + Phi A0^-1 Phi^T, W = diag(1/sqrt(overlap count)),
 * K_e the 1-D Kronecker-sum operator of the element box extended by one GLL layer, A0 its
 * Galerkin coarse operator on the interior element vertices; both by fast diagonalisation.
 * _d: fp64.  _f: policy OR_MIXED (fp32 arithmetic, sqrt / weights and the sums over subdomains
 * in fp64) or OR_FP32 / OR_FP32_DOT2 (all fp32).  Also or_cg(precond = OR_PC_SCHWARZ).
 * order: the gather-scatter order of the overlap sum (OR_GS_*; the ranked orders use the
 * or_set_ranks partition): the box contributions at a copy are combined like the copies of a
 * node in or_dssum (own element's box / own rank's partial first, ...); or_cg passes its gs_order.
 * or_schwarz_tables: the 1-D tables of axis a (0 x, 1 y, 2 z) at element position ex: first
 * lattice index and size of the extended index set, S ((p+3) x (p+3), row-major) and lambda
 * (p+3); the coarse S0 (nv x nv, nv = nel_a - 1) and lambda0 (nullable outputs).
 */
int or_schwarz_apply_d(or_mesh *m, int order, const double *r, double *z);
int or_schwarz_apply_f(or_mesh *m, int policy, int order, const float *r, float *z);
int or_schwarz_tables(or_mesh *m, int axis, int ex, int *t0, int *nt, double *S, double *lam, double *S0, double *lam0);
int or_cg(const or_mesh *m, int policy, int max_iter, double rtol, int gs_order, int stag_window,
          int seqdot, int x64, int precond, const double *b64, double *x_out, double *hist, double *scal,
          or_report *rep);

#ifdef __cplusplus
}
#endif
#endif
