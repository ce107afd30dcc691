/*
 * nb_oracle.c -- TEST INFRASTRUCTURE ONLY: the parity oracle for the B200 path.
 *
 * A plain, slow, single-threaded CPU implementation of what the hot path
 * computes, written from the paper and the readings of SURVEY.md §8(c)
 * (listed in DESIGN.md §3).  Only tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline legs may load it; the product path
 * (paper_2503_02134_b200/) never does.  No code is shared with the CUDA path.
 *
 * Paper passages followed (PAPER.md line numbers):
 *   - Nekbone CG loop, Table 2 (:158-168): solveM, glsc3 (beta), add2s1, ax,
 *     glsc3 (pap), add2s2 x2, glsc3 (rtr).
 *   - ax -> local_grad3 / local_grad3_t / mxm / add2, call graph (:147).
 *   - gather-scatter "ensure continuity" on an unassembled per-element
 *     matrix (:404), GS precision as the stagnation mechanism (:339-341, :429-431).
 *   - Jacobi J^-1 = 1/diag(A), one-time cast (:444).
 *   - mixed policy: fp32 loop, fp64 dots + gather-scatter + init (:53, :537).
 *
 * Compiled -O2 -ffp-contract=off -fno-fast-math: no FMA contraction, C float
 * and double exactly as each policy states.
 *
 * Parity pins live in tests/test_oracle_*.py (closed forms, dense assembly,
 * patch test, spectral convergence, dense solve, stagnation).
 */
#include "nb_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

struct or_mesh {
    int nelx, nely, nelz, p, n;
    int64_t E, NL, NX, NY, NZ, NG;
    int64_t n_unmasked, n_shared_global, n_shared_copies;
    double z[16], w[16], D[256];   /* GLL nodes, weights, D[i*n+j] */
    float Df[256];                 /* one-time float cast of D */
    double *xyz;                   /* 3*NL, factor-major */
    double *jac;                   /* NL */
    double *g;                     /* 6*NL factor-major g1..g6 (C-6 ordering) */
    float *gf;                     /* one-time float cast */
    double *B;                     /* NL */
    int64_t *gid;                  /* NL */
    uint8_t *mask;                 /* NL */
    double *c;                     /* NL, 1/multiplicity */
    float *cf;
    int32_t nseg;
    int32_t *off, *idx;            /* GS CSR */
    double *dinv;                  /* NL fp64 */
    float *dinvf;                  /* one-time float cast */
    int px, py, pz;                /* rank partition of the ranked gather-scatter orders (or_set_ranks) */
    struct or_schwarz *sw;         /* NEXT-4 Schwarz preconditioner tables (built on first use) */
};
static void schwarz_free(struct or_schwarz *sw);

/* ------------------------------------------------------------------ */
/* C-1: GLL basis                     */
/* ------------------------------------------------------------------ */

/* Legendre P_p(x) and P_{p-1}(x) by the three-term recurrence. */
static void legendre(int p, double x, double *Pp, double *Ppm1)
{
    double P0 = 1.0, P1 = x;
    if (p == 0) { *Pp = 1.0; *Ppm1 = 0.0; return; }
    for (int k = 2; k <= p; k++) {
        double P2 = ((2.0 * k - 1.0) * x * P1 - (k - 1.0) * P0) / k;
        P0 = P1;
        P1 = P2;
    }
    *Pp = P1;
    *Ppm1 = P0;
}

int or_gll(int p, double *nodes, double *weights, double *D)
{
    if (p < 1 || p > 15) return 1;
    const int n = p + 1;
    const double pi = 3.14159265358979323846;
    /* Newton on f(x) = (1-x^2) P_p'(x) = p (P_{p-1} - x P_p), f'(x) = -p(p+1) P_p(x)
       (Legendre ODE), from x_i = -cos(pi i / p); stop at |dx| < 1e-16 (100 its max). */
    for (int i = 0; i < n; i++) {
        double x = -cos(pi * i / p);
        if (i == 0) x = -1.0;
        if (i == p) x = 1.0;
        int it = 0;
        for (; it < 100; it++) {
            double Pp, Pm;
            legendre(p, x, &Pp, &Pm);
            double dx = (Pm - x * Pp) / ((p + 1.0) * Pp);
            x += dx;
            if (fabs(dx) < 1e-16) break;
        }
        if (it == 100) {
            /* rounding can leave |dx| oscillating at ~1 ulp; accept if f(x) is at roundoff */
            double Pp, Pm;
            legendre(p, x, &Pp, &Pm);
            if (fabs(Pm - x * Pp) > 1e-13) return 2;
        }
        nodes[i] = x;
    }
    /* weights w_i = 2 / (p(p+1) P_p(x_i)^2) */
    double Pn[16];
    for (int i = 0; i < n; i++) {
        double Pp, Pm;
        legendre(p, nodes[i], &Pp, &Pm);
        Pn[i] = Pp;
        weights[i] = 2.0 / (p * (p + 1.0) * Pp * Pp);
    }
    /* D_ij = P_p(x_i) / (P_p(x_j) (x_i - x_j)), i != j; D_ii = -sum_{j!=i} D_ij (C-1 reading) */
    for (int i = 0; i < n; i++) {
        double s = 0.0;
        for (int j = 0; j < n; j++) {
            if (j == i) continue;
            D[i * n + j] = Pn[i] / (Pn[j] * (nodes[i] - nodes[j]));
            s += D[i * n + j];
        }
        D[i * n + i] = -s;
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* C-5: counter-based SplitMix64                                        */
/* ------------------------------------------------------------------ */

uint64_t or_splitmix64(uint64_t seed, uint64_t stream, uint64_t i)
{
    uint64_t z = (seed ^ (stream * 0xD1B54A32D192ED03ull)) + (i + 1ull) * 0x9E3779B97F4A7C15ull;
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

double or_prng_u(uint64_t seed, uint64_t stream, uint64_t i)
{
    uint64_t z = or_splitmix64(seed, stream, i);
    return (double)(z >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
}

/* ------------------------------------------------------------------ */
/* helpers                                                              */
/* ------------------------------------------------------------------ */

/* local index l -> element e and (i,j,k) ; C-4: l = e n^3 + i + n j + n^2 k */
static void split_local(const or_mesh *m, int64_t l, int64_t *e, int *i, int *j, int *k)
{
    int64_t n3 = (int64_t)m->n * m->n * m->n;
    *e = l / n3;
    int64_t r = l % n3;
    *i = (int)(r % m->n);
    *j = (int)((r / m->n) % m->n);
    *k = (int)(r / ((int64_t)m->n * m->n));
}

static void element_xyz(const or_mesh *m, int64_t e, int *ex, int *ey, int *ez)
{
    *ex = (int)(e % m->nelx);
    *ey = (int)((e / m->nelx) % m->nely);
    *ez = (int)(e / ((int64_t)m->nelx * m->nely));
}

/* C-3: deformed vertex position */
static void vertex_pos(int ix, int iy, int iz, int nelx, int nely, int nelz, double amp,
                       const double phi[3], double out[3])
{
    const double pi = 3.14159265358979323846;
    double X = (double)ix / nelx, Y = (double)iy / nely, Z = (double)iz / nelz;
    out[0] = X;
    out[1] = Y;
    out[2] = Z;
    if (amp == 0.0) return;
    if (ix == 0 || ix == nelx || iy == 0 || iy == nely || iz == 0 || iz == nelz) return;
    double bubble = sin(pi * X) * sin(pi * Y) * sin(pi * Z);
    const int kv[3][3] = {{1, 2, 1}, {2, 1, 1}, {1, 1, 2}};
    const double h[3] = {1.0 / nelx, 1.0 / nely, 1.0 / nelz};
    for (int a = 0; a < 3; a++) {
        double kdot = kv[a][0] * X + kv[a][1] * Y + kv[a][2] * Z;
        out[a] += amp * h[a] * bubble * cos(2.0 * pi * kdot + phi[a]);
    }
}

/* ------------------------------------------------------------------ */
/* mesh setup (C-2 .. C-9)                                              */
/* ------------------------------------------------------------------ */

void or_mesh_free(or_mesh *m)
{
    if (!m) return;
    free(m->xyz); free(m->jac); free(m->g); free(m->gf); free(m->B); free(m->gid);
    free(m->mask); free(m->c); free(m->cf); free(m->off); free(m->idx); free(m->dinv); free(m->dinvf);
    schwarz_free(m->sw);
    free(m);
}

or_mesh *or_mesh_new(int nelx, int nely, int nelz, int p, double deform_amp, uint64_t seed)
{
    if (nelx < 1 || nely < 1 || nelz < 1 || p < 1 || p > 15) return NULL;
    or_mesh *m = (or_mesh *)calloc(1, sizeof(or_mesh));
    m->nelx = nelx; m->nely = nely; m->nelz = nelz; m->p = p; m->n = p + 1;
    m->px = m->py = m->pz = 1;
    const int n = m->n;
    const int64_t n3 = (int64_t)n * n * n;
    m->E = (int64_t)nelx * nely * nelz;
    m->NL = m->E * n3;
    m->NX = (int64_t)nelx * p + 1; m->NY = (int64_t)nely * p + 1; m->NZ = (int64_t)nelz * p + 1;
    m->NG = m->NX * m->NY * m->NZ;
    if (m->NL >= 2147483647LL) { free(m); return NULL; }
    if (or_gll(p, m->z, m->w, m->D)) { free(m); return NULL; }
    for (int a = 0; a < n * n; a++) m->Df[a] = (float)m->D[a];

    const int64_t NL = m->NL;
    m->xyz = (double *)malloc(3 * NL * sizeof(double));
    m->jac = (double *)malloc(NL * sizeof(double));
    m->g = (double *)malloc(6 * NL * sizeof(double));
    m->gf = (float *)malloc(6 * NL * sizeof(float));
    m->B = (double *)malloc(NL * sizeof(double));
    m->gid = (int64_t *)malloc(NL * sizeof(int64_t));
    m->mask = (uint8_t *)malloc(NL);
    m->c = (double *)malloc(NL * sizeof(double));
    m->cf = (float *)malloc(NL * sizeof(float));
    m->dinv = (double *)malloc(NL * sizeof(double));
    m->dinvf = (float *)malloc(NL * sizeof(float));

    /* C-3 phases */
    double phi[3];
    const double pi = 3.14159265358979323846;
    for (int a = 0; a < 3; a++) phi[a] = pi * (1.0 + or_prng_u(seed, 3, (uint64_t)a));

    /* C-2/C-3: GLL node coordinates by trilinear interpolation of the 8 moved vertices */
    int ok = 1;
    for (int64_t e = 0; e < m->E; e++) {
        int ex, ey, ez;
        element_xyz(m, e, &ex, &ey, &ez);
        double V[2][2][2][3];
        for (int cz = 0; cz < 2; cz++)
            for (int cy = 0; cy < 2; cy++)
                for (int cx = 0; cx < 2; cx++)
                    vertex_pos(ex + cx, ey + cy, ez + cz, nelx, nely, nelz, deform_amp, phi, V[cz][cy][cx]);
        double *X = m->xyz, *Y = m->xyz + NL, *Z = m->xyz + 2 * NL;
        for (int k = 0; k < n; k++)
            for (int j = 0; j < n; j++)
                for (int i = 0; i < n; i++) {
                    double Nx[2] = {(1.0 - m->z[i]) / 2.0, (1.0 + m->z[i]) / 2.0};
                    double Ny[2] = {(1.0 - m->z[j]) / 2.0, (1.0 + m->z[j]) / 2.0};
                    double Nz[2] = {(1.0 - m->z[k]) / 2.0, (1.0 + m->z[k]) / 2.0};
                    double pos[3] = {0.0, 0.0, 0.0};
                    for (int cz = 0; cz < 2; cz++)
                        for (int cy = 0; cy < 2; cy++)
                            for (int cx = 0; cx < 2; cx++)
                                for (int a = 0; a < 3; a++)
                                    pos[a] += Nx[cx] * Ny[cy] * Nz[cz] * V[cz][cy][cx][a];
                    int64_t l = e * n3 + i + n * j + (int64_t)n * n * k;
                    X[l] = pos[0]; Y[l] = pos[1]; Z[l] = pos[2];
                }
        /* C-6: Jacobian via D, G = W J R R^T, B = W J */
        for (int k = 0; k < n; k++)
            for (int j = 0; j < n; j++)
                for (int i = 0; i < n; i++) {
                    int64_t l = e * n3 + i + n * j + (int64_t)n * n * k;
                    double M[3][3]; /* M[a][b] = d x_a / d r_b */
                    const double *F[3] = {X, Y, Z};
                    for (int a = 0; a < 3; a++) {
                        double dr = 0.0, ds = 0.0, dt = 0.0;
                        for (int q = 0; q < n; q++) {
                            dr += m->D[i * n + q] * F[a][e * n3 + q + n * j + (int64_t)n * n * k];
                            ds += m->D[j * n + q] * F[a][e * n3 + i + n * q + (int64_t)n * n * k];
                            dt += m->D[k * n + q] * F[a][e * n3 + i + n * j + (int64_t)n * n * q];
                        }
                        M[a][0] = dr; M[a][1] = ds; M[a][2] = dt;
                    }
                    double det = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1])
                               - M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0])
                               + M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
                    if (!(det > 0.0)) ok = 0;
                    double R[3][3]; /* R[a][b] = d r_a / d x_b = inverse of M */
                    R[0][0] = (M[1][1] * M[2][2] - M[1][2] * M[2][1]) / det;
                    R[0][1] = (M[0][2] * M[2][1] - M[0][1] * M[2][2]) / det;
                    R[0][2] = (M[0][1] * M[1][2] - M[0][2] * M[1][1]) / det;
                    R[1][0] = (M[1][2] * M[2][0] - M[1][0] * M[2][2]) / det;
                    R[1][1] = (M[0][0] * M[2][2] - M[0][2] * M[2][0]) / det;
                    R[1][2] = (M[0][2] * M[1][0] - M[0][0] * M[1][2]) / det;
                    R[2][0] = (M[1][0] * M[2][1] - M[1][1] * M[2][0]) / det;
                    R[2][1] = (M[0][1] * M[2][0] - M[0][0] * M[2][1]) / det;
                    R[2][2] = (M[0][0] * M[1][1] - M[0][1] * M[1][0]) / det;
                    double W = m->w[i] * m->w[j] * m->w[k];
                    double G[3][3];
                    for (int a = 0; a < 3; a++)
                        for (int b = 0; b < 3; b++) {
                            double s = 0.0;
                            for (int q = 0; q < 3; q++) s += R[a][q] * R[b][q];
                            G[a][b] = W * det * s;
                        }
                    m->jac[l] = det;
                    m->g[0 * NL + l] = G[0][0];
                    m->g[1 * NL + l] = G[0][1];
                    m->g[2 * NL + l] = G[0][2];
                    m->g[3 * NL + l] = G[1][1];
                    m->g[4 * NL + l] = G[1][2];
                    m->g[5 * NL + l] = G[2][2];
                    m->B[l] = W * det;
                }
    }
    for (int64_t a = 0; a < 6 * NL; a++) m->gf[a] = (float)m->g[a];

    /* C-4: global ids and mask */
    for (int64_t l = 0; l < NL; l++) {
        int64_t e; int i, j, k, ex, ey, ez;
        split_local(m, l, &e, &i, &j, &k);
        element_xyz(m, e, &ex, &ey, &ez);
        int64_t I = (int64_t)ex * p + i, J = (int64_t)ey * p + j, K = (int64_t)ez * p + k;
        m->gid[l] = I + m->NX * (J + m->NY * K);
        int bnd = (I == 0 || I == m->NX - 1 || J == 0 || J == m->NY - 1 || K == 0 || K == m->NZ - 1);
        m->mask[l] = bnd ? 0 : 1;
    }
    /* multiplicity by brute-force counting of copies per global id */
    int32_t *cnt = (int32_t *)calloc(m->NG, sizeof(int32_t));
    for (int64_t l = 0; l < NL; l++) cnt[m->gid[l]]++;
    for (int64_t l = 0; l < NL; l++) {
        m->c[l] = 1.0 / cnt[m->gid[l]];
        m->cf[l] = (float)m->c[l];
    }
    /* GS segments: shared global nodes (count >= 2) ascending gid, copies ascending l */
    int32_t *seg = (int32_t *)malloc(m->NG * sizeof(int32_t));
    int64_t nseg = 0, ncopies = 0, nunm = 0;
    for (int64_t gg = 0; gg < m->NG; gg++) {
        if (cnt[gg] >= 2) { seg[gg] = (int32_t)nseg++; ncopies += cnt[gg]; }
        else seg[gg] = -1;
    }
    m->nseg = (int32_t)nseg;
    m->off = (int32_t *)malloc((nseg + 1) * sizeof(int32_t));
    m->idx = (int32_t *)malloc((ncopies > 0 ? ncopies : 1) * sizeof(int32_t));
    m->off[0] = 0;
    for (int64_t gg = 0; gg < m->NG; gg++)
        if (seg[gg] >= 0) m->off[seg[gg] + 1] = m->off[seg[gg]] + cnt[gg];
    int32_t *fill = (int32_t *)calloc(nseg > 0 ? nseg : 1, sizeof(int32_t));
    for (int64_t l = 0; l < NL; l++) {
        int32_t s = seg[m->gid[l]];
        if (s >= 0) m->idx[m->off[s] + fill[s]++] = (int32_t)l;
    }
    free(fill);
    free(seg);
    /* unmasked unique nodes */
    {
        uint8_t *seen = (uint8_t *)calloc(m->NG, 1);
        for (int64_t l = 0; l < NL; l++)
            if (m->mask[l] && !seen[m->gid[l]]) { seen[m->gid[l]] = 1; nunm++; }
        free(seen);
    }
    free(cnt);
    m->n_unmasked = nunm;
    m->n_shared_global = nseg;
    m->n_shared_copies = ncopies;

    /* C-9: Jacobi diagonal, closed form, then consistent fp64 dssum, dinv = 1/diag (0 on mask) */
    double *diag = (double *)malloc(NL * sizeof(double));
    for (int64_t e = 0; e < m->E; e++)
        for (int k = 0; k < n; k++)
            for (int j = 0; j < n; j++)
                for (int i = 0; i < n; i++) {
                    int64_t base = e * n3;
                    int64_t l = base + i + n * j + (int64_t)n * n * k;
                    double s = 0.0;
                    for (int q = 0; q < n; q++) {
                        double d = m->D[q * n + i];
                        s += d * d * m->g[0 * NL + base + q + n * j + (int64_t)n * n * k];
                    }
                    for (int q = 0; q < n; q++) {
                        double d = m->D[q * n + j];
                        s += d * d * m->g[3 * NL + base + i + n * q + (int64_t)n * n * k];
                    }
                    for (int q = 0; q < n; q++) {
                        double d = m->D[q * n + k];
                        s += d * d * m->g[5 * NL + base + i + n * j + (int64_t)n * n * q];
                    }
                    s += 2.0 * m->D[i * n + i] * m->D[j * n + j] * m->g[1 * NL + l];
                    s += 2.0 * m->D[i * n + i] * m->D[k * n + k] * m->g[2 * NL + l];
                    s += 2.0 * m->D[j * n + j] * m->D[k * n + k] * m->g[4 * NL + l];
                    diag[l] = s;
                }
    or_dssum_d(m, OR_GS_CONSISTENT, diag);
    for (int64_t l = 0; l < NL; l++) {
        if (m->mask[l]) {
            if (!(diag[l] > 0.0)) ok = 0;
            m->dinv[l] = 1.0 / diag[l];
        } else {
            m->dinv[l] = 0.0;
        }
        m->dinvf[l] = (float)m->dinv[l];
    }
    free(diag);
    if (!ok) { or_mesh_free(m); return NULL; }
    return m;
}

void or_mesh_info(const or_mesh *m, int64_t *info)
{
    info[0] = m->E;
    info[1] = m->NL;
    info[2] = m->NG;
    info[3] = m->n_unmasked;
    info[4] = m->n_shared_global;
    info[5] = m->n_shared_copies;
    info[6] = m->p;
    info[7] = 1;
}

void or_export_maps(const or_mesh *m, int64_t *gid, uint8_t *mask, int32_t *gs_off, int32_t *gs_idx)
{
    if (gid) memcpy(gid, m->gid, m->NL * sizeof(int64_t));
    if (mask) memcpy(mask, m->mask, m->NL);
    if (gs_off) memcpy(gs_off, m->off, (m->nseg + 1) * sizeof(int32_t));
    if (gs_idx) memcpy(gs_idx, m->idx, m->n_shared_copies * sizeof(int32_t));
}

void or_export_geom(const or_mesh *m, double *g6, double *B, double *dinv, double *c, double *xyz, double *jac)
{
    if (g6) memcpy(g6, m->g, 6 * m->NL * sizeof(double));
    if (B) memcpy(B, m->B, m->NL * sizeof(double));
    if (dinv) memcpy(dinv, m->dinv, m->NL * sizeof(double));
    if (c) memcpy(c, m->c, m->NL * sizeof(double));
    if (xyz) memcpy(xyz, m->xyz, 3 * m->NL * sizeof(double));
    if (jac) memcpy(jac, m->jac, m->NL * sizeof(double));
}

/* ------------------------------------------------------------------ */
/* C-7: local operator ("ax_e": local_grad3, geometric scaling, local_grad3_t) */
/* ------------------------------------------------------------------ */

void or_local_grad3(int p, const double *D, const double *u, double *ur, double *us, double *ut)
{
    const int n = p + 1;
    for (int k = 0; k < n; k++)
        for (int j = 0; j < n; j++)
            for (int i = 0; i < n; i++) {
                double a = 0.0, b = 0.0, c = 0.0;
                for (int l = 0; l < n; l++) {
                    a += D[i * n + l] * u[l + n * j + n * n * k];
                    b += D[j * n + l] * u[i + n * l + n * n * k];
                    c += D[k * n + l] * u[i + n * j + n * n * l];
                }
                int q = i + n * j + n * n * k;
                ur[q] = a; us[q] = b; ut[q] = c;
            }
}

void or_ax_local_d(const or_mesh *m, const double *u, double *w)
{
    const int n = m->n;
    const int64_t n3 = (int64_t)n * n * n, NL = m->NL;
    double *ur = (double *)malloc(n3 * sizeof(double)), *us = (double *)malloc(n3 * sizeof(double));
    double *ut = (double *)malloc(n3 * sizeof(double));
    const double *D = m->D;
    for (int64_t e = 0; e < m->E; e++) {
        const double *ue = u + e * n3;
        or_local_grad3(m->p, D, ue, ur, us, ut);
        for (int64_t q = 0; q < n3; q++) {
            int64_t l = e * n3 + q;
            double g1 = m->g[l], g2 = m->g[NL + l], g3 = m->g[2 * NL + l];
            double g4 = m->g[3 * NL + l], g5 = m->g[4 * NL + l], g6 = m->g[5 * NL + l];
            double a = ur[q], b = us[q], c = ut[q];
            ur[q] = (g1 * a + g2 * b) + g3 * c;
            us[q] = (g2 * a + g4 * b) + g5 * c;
            ut[q] = (g3 * a + g5 * b) + g6 * c;
        }
        for (int k = 0; k < n; k++)
            for (int j = 0; j < n; j++)
                for (int i = 0; i < n; i++) {
                    double a = 0.0, b = 0.0, c = 0.0;
                    for (int l = 0; l < n; l++) {
                        a += D[l * n + i] * ur[l + n * j + n * n * k];
                        b += D[l * n + j] * us[i + n * l + n * n * k];
                        c += D[l * n + k] * ut[i + n * j + n * n * l];
                    }
                    w[e * n3 + i + n * j + n * n * k] = (a + b) + c;
                }
    }
    free(ur); free(us); free(ut);
}

void or_ax_local_f(const or_mesh *m, const float *u, float *w)
{
    const int n = m->n;
    const int64_t n3 = (int64_t)n * n * n, NL = m->NL;
    float *ur = (float *)malloc(n3 * sizeof(float)), *us = (float *)malloc(n3 * sizeof(float));
    float *ut = (float *)malloc(n3 * sizeof(float));
    const float *D = m->Df;
    for (int64_t e = 0; e < m->E; e++) {
        const float *ue = u + e * n3;
        for (int k = 0; k < n; k++)
            for (int j = 0; j < n; j++)
                for (int i = 0; i < n; i++) {
                    float a = 0.0f, b = 0.0f, c = 0.0f;
                    for (int l = 0; l < n; l++) {
                        a += D[i * n + l] * ue[l + n * j + n * n * k];
                        b += D[j * n + l] * ue[i + n * l + n * n * k];
                        c += D[k * n + l] * ue[i + n * j + n * n * l];
                    }
                    int q = i + n * j + n * n * k;
                    ur[q] = a; us[q] = b; ut[q] = c;
                }
        for (int64_t q = 0; q < n3; q++) {
            int64_t l = e * n3 + q;
            float g1 = m->gf[l], g2 = m->gf[NL + l], g3 = m->gf[2 * NL + l];
            float g4 = m->gf[3 * NL + l], g5 = m->gf[4 * NL + l], g6 = m->gf[5 * NL + l];
            float a = ur[q], b = us[q], c = ut[q];
            ur[q] = (g1 * a + g2 * b) + g3 * c;
            us[q] = (g2 * a + g4 * b) + g5 * c;
            ut[q] = (g3 * a + g5 * b) + g6 * c;
        }
        for (int k = 0; k < n; k++)
            for (int j = 0; j < n; j++)
                for (int i = 0; i < n; i++) {
                    float a = 0.0f, b = 0.0f, c = 0.0f;
                    for (int l = 0; l < n; l++) {
                        a += D[l * n + i] * ur[l + n * j + n * n * k];
                        b += D[l * n + j] * us[i + n * l + n * n * k];
                        c += D[l * n + k] * ut[i + n * j + n * n * l];
                    }
                    w[e * n3 + i + n * j + n * n * k] = (a + b) + c;
                }
    }
    free(ur); free(us); free(ut);
}

/* ------------------------------------------------------------------ */
/* C-8: gather-scatter QQ^T over the CSR segments                      */
/* ------------------------------------------------------------------ */

/* Rank of element e in a px x py x pz partition of the element box:
 * contiguous blocks as even as possible, block b of an axis with nel elements and P parts
 * holding elements [floor(b nel / P), floor((b+1) nel / P)). */
int or_set_ranks(or_mesh *m, int px, int py, int pz)
{
    if (px < 1 || py < 1 || pz < 1 || px > m->nelx || py > m->nely || pz > m->nelz) return 1;
    m->px = px; m->py = py; m->pz = pz;
    return 0;
}
static int block_of(int i, int nel, int P)
{
    int b = 0;
    while (b + 1 < P && (int64_t)(b + 1) * nel / P <= i) b++;
    return b;
}
static int elem_rank(const or_mesh *m, int64_t e)
{
    int ex, ey, ez;
    element_xyz(m, e, &ex, &ey, &ez);
    return block_of(ex, m->nelx, m->px) + m->px * (block_of(ey, m->nely, m->py) + m->py * block_of(ez, m->nelz, m->pz));
}

/* The gather-scatter of a rank-partitioned run (Table 3: gslib's pairwise and
 * allreduce modes).  Each rank first sums its own copies of a node in ascending local index (the
 * local gather, GS precision TG); the rank partials P_q are then exchanged in TG:
 *   OR_GS_PAIRWISE : a copy on rank r receives P_r + sum_{q != r, ascending q} P_q -- each rank
 *                    adds its neighbours' contributions to its own;
 *   OR_GS_ALLREDUCE: every copy receives sum_{ascending q} P_q -- one reduction, the same value on
 *                    every rank.
 * Copies of a node on one rank always agree; copies on different ranks agree under pairwise only
 * when at most two ranks share the node (a + b = b + a), so a 1-D partition stays consistent. */
#define OR_DSSUM_RANKED(NAME, TVX, TGX)                                                        \
    static void NAME(const or_mesh *m, int order, TVX *u)                                     \
    {                                                                                          \
        const int64_t n3 = (int64_t)m->n * m->n * m->n;                                        \
        for (int32_t s = 0; s < m->nseg; s++) {                                                \
            const int32_t a = m->off[s], cnt = m->off[s + 1] - a;                              \
            TVX v[8];                                                                          \
            int rk[8];                                                                         \
            TGX part[8];                                                                       \
            for (int q = 0; q < cnt; q++) {                                                    \
                v[q] = u[m->idx[a + q]];                                                       \
                rk[q] = elem_rank(m, m->idx[a + q] / n3);                                      \
            }                                                                                  \
            for (int q = 0; q < cnt; q++) {          /* local gather: P of copy q's rank */    \
                TGX t = 0;                                                                     \
                for (int q2 = 0; q2 < cnt; q2++)                                               \
                    if (rk[q2] == rk[q]) t += (TGX)v[q2];                                      \
                part[q] = t;                                                                   \
            }                                                                                  \
            for (int q = 0; q < cnt; q++) {                                                    \
                TGX t = (order == OR_GS_PAIRWISE) ? part[q] : (TGX)0;                          \
                int prev = -1;                                                                 \
                for (;;) {                           /* ranks in ascending order */            \
                    int best = -1;                                                             \
                    for (int q2 = 0; q2 < cnt; q2++)                                           \
                        if (rk[q2] > prev && (best < 0 || rk[q2] < rk[best])) best = q2;       \
                    if (best < 0) break;                                                       \
                    prev = rk[best];                                                           \
                    if (order == OR_GS_PAIRWISE && rk[best] == rk[q]) continue;                \
                    t += part[best];                                                           \
                }                                                                              \
                u[m->idx[a + q]] = (TVX)t;                                                     \
            }                                                                                  \
        }                                                                                      \
    }
OR_DSSUM_RANKED(dssum_ranked_d, double, double)
OR_DSSUM_RANKED(dssum_ranked_f, float, float)
OR_DSSUM_RANKED(dssum_ranked_fd, float, double)

void or_dssum_d(const or_mesh *m, int order, double *u)
{
    if (order == OR_GS_PAIRWISE || order == OR_GS_ALLREDUCE) { dssum_ranked_d(m, order, u); return; }
    double vals[8];
    for (int32_t s = 0; s < m->nseg; s++) {
        int32_t a = m->off[s], cnt = m->off[s + 1] - a;
        for (int q = 0; q < cnt; q++) vals[q] = u[m->idx[a + q]];
        if (order == OR_GS_CONSISTENT) {
            double t = 0.0;
            for (int q = 0; q < cnt; q++) t += vals[q];
            for (int q = 0; q < cnt; q++) u[m->idx[a + q]] = t;
        } else {
            for (int q = 0; q < cnt; q++) {
                double t = vals[q];
                for (int r = 0; r < cnt; r++)
                    if (r != q) t += vals[r];
                u[m->idx[a + q]] = t;
            }
        }
    }
}

void or_dssum_f(const or_mesh *m, int order, float *u)
{
    if (order == OR_GS_PAIRWISE || order == OR_GS_ALLREDUCE) { dssum_ranked_f(m, order, u); return; }
    float vals[8];
    for (int32_t s = 0; s < m->nseg; s++) {
        int32_t a = m->off[s], cnt = m->off[s + 1] - a;
        for (int q = 0; q < cnt; q++) vals[q] = u[m->idx[a + q]];
        if (order == OR_GS_CONSISTENT) {
            float t = 0.0f;
            for (int q = 0; q < cnt; q++) t += vals[q];
            for (int q = 0; q < cnt; q++) u[m->idx[a + q]] = t;
        } else {
            for (int q = 0; q < cnt; q++) {
                float t = vals[q];
                for (int r = 0; r < cnt; r++)
                    if (r != q) t += vals[r];
                u[m->idx[a + q]] = t;
            }
        }
    }
}

void or_dssum_fd(const or_mesh *m, int order, float *u)
{
    if (order == OR_GS_PAIRWISE || order == OR_GS_ALLREDUCE) { dssum_ranked_fd(m, order, u); return; }
    float vals[8];
    for (int32_t s = 0; s < m->nseg; s++) {
        int32_t a = m->off[s], cnt = m->off[s + 1] - a;
        for (int q = 0; q < cnt; q++) vals[q] = u[m->idx[a + q]];
        if (order == OR_GS_CONSISTENT) {
            double t = 0.0;
            for (int q = 0; q < cnt; q++) t += (double)vals[q];
            for (int q = 0; q < cnt; q++) u[m->idx[a + q]] = (float)t;
        } else {
            for (int q = 0; q < cnt; q++) {
                double t = (double)vals[q];
                for (int r = 0; r < cnt; r++)
                    if (r != q) t += (double)vals[r];
                u[m->idx[a + q]] = (float)t;
            }
        }
    }
}

void or_ax_d(const or_mesh *m, int order, const double *u, double *w)
{
    or_ax_local_d(m, u, w);
    or_dssum_d(m, order, w);
    for (int64_t l = 0; l < m->NL; l++)
        if (!m->mask[l]) w[l] = 0.0;
}

void or_ax_f(const or_mesh *m, int policy, int order, const float *u, float *w)
{
    or_ax_local_f(m, u, w);
    if (policy == OR_MIXED) or_dssum_fd(m, order, w);
    else or_dssum_f(m, order, w);
    for (int64_t l = 0; l < m->NL; l++)
        if (!m->mask[l]) w[l] = 0.0f;
}

/* ------------------------------------------------------------------ */
/* glsc3 (Table 2 lines 3, 6, 9)                                        */
/* ------------------------------------------------------------------ */

double or_glsc3_d(const double *a, const double *c, const double *b, int64_t n)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) s += (a[i] * c[i]) * b[i];
    return s;
}

double or_glsc3_mixed(const float *a, const double *c, const float *b, int64_t n)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) s += ((double)a[i] * c[i]) * (double)b[i];
    return s;
}

static float tree_f(const float *a, const float *c, const float *b, int64_t lo, int64_t hi)
{
    if (hi - lo <= 32) {
        float s = 0.0f;
        for (int64_t i = lo; i < hi; i++) s += (a[i] * c[i]) * b[i];
        return s;
    }
    int64_t mid = lo + (hi - lo) / 2;
    float left = tree_f(a, c, b, lo, mid);
    float right = tree_f(a, c, b, mid, hi);
    return left + right;
}

float or_glsc3_f_tree(const float *a, const float *c, const float *b, int64_t n)
{
    if (n <= 0) return 0.0f;
    return tree_f(a, c, b, 0, n);
}

float or_glsc3_f_seq(const float *a, const float *c, const float *b, int64_t n)
{
    float s = 0.0f;
    for (int64_t i = 0; i < n; i++) s += (a[i] * c[i]) * b[i];
    return s;
}

/* Error-free transformations in binary32 (Sec. 5.2.1; SPEC.md eft module).
 * two_sum: Knuth's branch-free TwoSum, s = fl(a+b), s + e = a + b exactly.
 * two_prod: p = fl(a*b), e = fma(a, b, -p), p + e = a*b exactly (fma-class hardware). */
void or_two_sum_f(float a, float b, float *s, float *e)
{
    /* binary32 per operation: -ffp-contract=off, FLT_EVAL_METHOD 0 on x86-64 */
    const float x = a + b;
    const float bv = x - a;
    const float av = x - bv;
    *s = x;
    *e = (a - av) + (b - bv);
}
void or_two_prod_f(float a, float b, float *p, float *e)
{
    const float x = a * b;
    *p = x;
    *e = fmaf(a, b, -x);
}

/* Dot2 (Ogita, Rump, Oishi 2005, Algorithm 5.3) of x_i = a_i c_i (exact: c_i = 2^-k) and b_i,
 * sequential, in binary32: [p, s] = TwoProduct(x_1, y_1); for i >= 2: [h, r] = TwoProduct(x_i, y_i);
 * [p, q] = TwoSum(p, h); s = s + (q + r); result fl(p + s). */
float or_glsc3_f_dot2(const float *a, const float *c, const float *b, int64_t n)
{
    if (n <= 0) return 0.0f;
    float p, s, h, r, q;
    or_two_prod_f(a[0] * c[0], b[0], &p, &s);
    for (int64_t i = 1; i < n; i++) {
        or_two_prod_f(a[i] * c[i], b[i], &h, &r);
        or_two_sum_f(p, h, &p, &q);
        s = s + (q + r);
    }
    return p + s;
}

/* ------------------------------------------------------------------ */
/* NEXT-4: two-level overlapping Schwarz preconditioner (DESIGN.md      */
/* reading 28).  The paper fixes only that Nekbone's multigrid-preconditioned CG spends ~70% of */
/* its time in solveM (Table 1), that its Schwarz weights routine                */
/* h1mg_schwarz_wt3d2 "relies on square-root operations" and that the winning   */
/* mixed strategies keep those square roots, the dots and the gather-scatter in fp64 while the */
/* PCG loop runs in fp32.  Reading (not the paper's text):            */
/*   M^-1 r = sum_e R_e^T W K_e^-1 W R_e r  +  Phi A0^-1 Phi^T r                               */
/*   R_e   restriction of the global (lattice) vector to the element's box extended by one     */
/*         GLL layer on every side, Dirichlet (boundary) lattice points excluded;              */
/*   W     diag(1/sqrt(count)), count(I,J,K) = number of extended boxes containing the point   */
/*         (so sum_e R_e^T W^2 R_e = I: the square roots make the additive sum symmetric);     */
/*   K_e   the Kronecker sum A1x(x)B1y(x)B1z + B1x(x)A1y(x)B1z + B1x(x)B1y(x)A1z of the 1-D    */
/*         assembled GLL stiffness/mass on the box lattice (spacing 1/nel_a), restricted to    */
/*         the extended box -- equal to R_e A R_e^T on an undeformed box, an approximation     */
/*         (still SPD) on a deformed one -- inverted by fast diagonalisation (1-D generalised  */
/*         eigenproblems A1 S = B1 S Lambda, S^T B1 S = I);                                    */
/*   Phi   trilinear hat functions of the interior element vertices evaluated on the lattice,  */
/*         A0 = Phi^T A_box Phi (the same Kronecker sum), also inverted by fast                */
/*         diagonalisation (B0 = Phi^T B1 Phi is tridiagonal: Cholesky-reduced).               */
/* ------------------------------------------------------------------ */
struct or_sw_axis {
    int nel, n;          /* elements along the axis, lattice points nel*p + 1 */
    int *t0, *nt;        /* per element position: first lattice index and size of the extended set */
    double *S, *lam;     /* per element position: S[(ex*(p+3) + row)*(p+3) + col], lam[ex*(p+3) + col] */
    int nv;              /* interior vertices nel - 1 */
    double *S0, *lam0;   /* coarse: S0[row*nv + col], lam0[col] */
    double *phiL, *phiR; /* hat values on an element's local points: phiL[i] = (1 - xi_i)/2, phiR = (1 + xi_i)/2 */
};
struct or_schwarz {
    struct or_sw_axis ax[3];
};

static void schwarz_free(struct or_schwarz *sw)
{
    if (!sw) return;
    for (int a = 0; a < 3; a++) {
        struct or_sw_axis *A = &sw->ax[a];
        free(A->t0); free(A->nt); free(A->S); free(A->lam); free(A->S0); free(A->lam0); free(A->phiL); free(A->phiR);
    }
    free(sw);
}

/* Cyclic Jacobi eigenvalue algorithm for a symmetric n x n matrix C (overwritten): C = Q diag(lam) Q^T. */
static void jacobi_eig(int n, double *C, double *Q, double *lam)
{
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) Q[i * n + j] = (i == j) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 100; sweep++) {
        double off = 0.0, tot = 0.0;
        for (int i = 0; i < n; i++)
            for (int j = 0; j < n; j++) {
                tot += C[i * n + j] * C[i * n + j];
                if (i != j) off += C[i * n + j] * C[i * n + j];
            }
        if (off <= 1e-30 * tot) break;
        for (int p = 0; p < n - 1; p++)
            for (int q = p + 1; q < n; q++) {
                const double apq = C[p * n + q];
                if (apq == 0.0) continue;
                const double theta = (C[q * n + q] - C[p * n + p]) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
                for (int k = 0; k < n; k++) {   /* columns p, q of C */
                    const double ckp = C[k * n + p], ckq = C[k * n + q];
                    C[k * n + p] = c * ckp - sn * ckq;
                    C[k * n + q] = sn * ckp + c * ckq;
                }
                for (int k = 0; k < n; k++) {   /* rows p, q */
                    const double cpk = C[p * n + k], cqk = C[q * n + k];
                    C[p * n + k] = c * cpk - sn * cqk;
                    C[q * n + k] = sn * cpk + c * cqk;
                }
                for (int k = 0; k < n; k++) {
                    const double qkp = Q[k * n + p], qkq = Q[k * n + q];
                    Q[k * n + p] = c * qkp - sn * qkq;
                    Q[k * n + q] = sn * qkp + c * qkq;
                }
            }
    }
    for (int i = 0; i < n; i++) lam[i] = C[i * n + i];
}

/* 1-D reference stiffness Ahat[a][b] = sum_q w_q D[q][a] D[q][b] on [-1, 1]. */
static double ahat(const or_mesh *m, int a, int b)
{
    double s = 0.0;
    for (int q = 0; q < m->n; q++) s += m->w[q] * m->D[q * m->n + a] * m->D[q * m->n + b];
    return s;
}
/* assembled 1-D lattice stiffness / mass entries (element length h = 1/nel) */
static double a1(const or_mesh *m, int nel, int I, int J)
{
    const int p = m->p;
    const double h = 1.0 / nel;
    double s = 0.0;
    for (int ex = 0; ex < nel; ex++) {
        const int a = I - ex * p, b = J - ex * p;
        if (a >= 0 && a <= p && b >= 0 && b <= p) s += (2.0 / h) * ahat(m, a, b);
    }
    return s;
}
static double b1(const or_mesh *m, int nel, int I)
{
    const int p = m->p;
    const double h = 1.0 / nel;
    double s = 0.0;
    for (int ex = 0; ex < nel; ex++) {
        const int a = I - ex * p;
        if (a >= 0 && a <= p) s += (h / 2.0) * m->w[a];
    }
    return s;
}
/* hat function of vertex v (lattice index v*p) at lattice point I */
static double hat(const or_mesh *m, int v, int I)
{
    const int p = m->p;
    if (I >= (v - 1) * p && I <= v * p && v >= 1) return (1.0 + m->z[I - (v - 1) * p]) / 2.0;
    if (I >= v * p && I <= (v + 1) * p) return (1.0 - m->z[I - v * p]) / 2.0;
    return 0.0;
}

/* Generalised symmetric-definite eigenproblem A S = B S Lambda, S^T B S = I, B SPD (n x n dense):
   Cholesky B = L L^T, C = L^-1 A L^-T, C = Q Lambda Q^T, S = L^-T Q. */
static void gen_eig(int n, const double *A, const double *B, double *S, double *lam)
{
    double *L = (double *)calloc((size_t)n * n, sizeof(double));
    double *T = (double *)calloc((size_t)n * n, sizeof(double));
    double *C = (double *)calloc((size_t)n * n, sizeof(double));
    double *Q = (double *)calloc((size_t)n * n, sizeof(double));
    for (int j = 0; j < n; j++) {
        double d = B[j * n + j];
        for (int k = 0; k < j; k++) d -= L[j * n + k] * L[j * n + k];
        L[j * n + j] = sqrt(d);
        for (int i = j + 1; i < n; i++) {
            double v = B[i * n + j];
            for (int k = 0; k < j; k++) v -= L[i * n + k] * L[j * n + k];
            L[i * n + j] = v / L[j * n + j];
        }
    }
    /* T = L^-1 A (forward substitution per column), C = T L^-T = (L^-1 T^T)^T */
    for (int c = 0; c < n; c++)
        for (int i = 0; i < n; i++) {
            double v = A[i * n + c];
            for (int k = 0; k < i; k++) v -= L[i * n + k] * T[k * n + c];
            T[i * n + c] = v / L[i * n + i];
        }
    for (int r = 0; r < n; r++)           /* C[r][:] = L^-1 applied to row r of T, as a column */
        for (int i = 0; i < n; i++) {
            double v = T[r * n + i];
            for (int k = 0; k < i; k++) v -= L[i * n + k] * C[r * n + k];
            C[r * n + i] = v / L[i * n + i];
        }
    for (int i = 0; i < n; i++)           /* symmetrise the rounding */
        for (int j = i + 1; j < n; j++) {
            const double v = 0.5 * (C[i * n + j] + C[j * n + i]);
            C[i * n + j] = v; C[j * n + i] = v;
        }
    jacobi_eig(n, C, Q, lam);
    /* S = L^-T Q: back substitution L^T S = Q per column */
    for (int c = 0; c < n; c++)
        for (int i = n - 1; i >= 0; i--) {
            double v = Q[i * n + c];
            for (int k = i + 1; k < n; k++) v -= L[k * n + i] * S[k * n + c];
            S[i * n + c] = v / L[i * n + i];
        }
    free(L); free(T); free(C); free(Q);
}

static struct or_schwarz *schwarz_setup(or_mesh *m)
{
    if (m->sw) return m->sw;
    const int p = m->p, P3 = p + 3;
    struct or_schwarz *sw = (struct or_schwarz *)calloc(1, sizeof(struct or_schwarz));
    const int nels[3] = {m->nelx, m->nely, m->nelz};
    for (int a = 0; a < 3; a++) {
        struct or_sw_axis *X = &sw->ax[a];
        const int nel = nels[a], n = nel * p + 1;
        X->nel = nel; X->n = n;
        X->t0 = (int *)calloc(nel, sizeof(int));
        X->nt = (int *)calloc(nel, sizeof(int));
        X->S = (double *)calloc((size_t)nel * P3 * P3, sizeof(double));
        X->lam = (double *)calloc((size_t)nel * P3, sizeof(double));
        X->phiL = (double *)calloc(p + 1, sizeof(double));
        X->phiR = (double *)calloc(p + 1, sizeof(double));
        for (int i = 0; i <= p; i++) { X->phiL[i] = (1.0 - m->z[i]) / 2.0; X->phiR[i] = (1.0 + m->z[i]) / 2.0; }
        for (int ex = 0; ex < nel; ex++) {
            int lo = ex * p - 1, hi = ex * p + p + 1;
            if (lo < 1) lo = 1;
            if (hi > n - 2) hi = n - 2;
            const int nt = hi - lo + 1;
            X->t0[ex] = lo; X->nt[ex] = nt;
            if (nt <= 0) continue;
            double *Ae = (double *)calloc((size_t)nt * nt, sizeof(double)), *Be = (double *)calloc((size_t)nt * nt, sizeof(double));
            double *Se = (double *)calloc((size_t)nt * nt, sizeof(double));
            for (int i = 0; i < nt; i++) {
                for (int j = 0; j < nt; j++) Ae[i * nt + j] = a1(m, nel, lo + i, lo + j);
                Be[i * nt + i] = b1(m, nel, lo + i);
            }
            gen_eig(nt, Ae, Be, Se, X->lam + (size_t)ex * P3);
            for (int i = 0; i < nt; i++)
                for (int j = 0; j < nt; j++) X->S[((size_t)ex * P3 + i) * P3 + j] = Se[i * nt + j];
            free(Ae); free(Be); free(Se);
        }
        const int nv = nel - 1;
        X->nv = nv;
        if (nv > 0) {
            double *A0 = (double *)calloc((size_t)nv * nv, sizeof(double)), *B0 = (double *)calloc((size_t)nv * nv, sizeof(double));
            /* A0 = Phi^T A1 Phi, B0 = Phi^T B1 Phi over all lattice points (hat supports) */
            for (int u = 1; u <= nv; u++)
                for (int v = 1; v <= nv; v++) {
                    double sa = 0.0, sb = 0.0;
                    for (int I = (u - 1) * p; I <= (u + 1) * p; I++) {
                        const double hu = hat(m, u, I);
                        if (hu == 0.0) continue;
                        sb += hu * b1(m, nel, I) * hat(m, v, I);
                        for (int J = (v - 1) * p; J <= (v + 1) * p; J++) {
                            const double hv = hat(m, v, J);
                            if (hv != 0.0) sa += hu * a1(m, nel, I, J) * hv;
                        }
                    }
                    A0[(u - 1) * nv + (v - 1)] = sa;
                    B0[(u - 1) * nv + (v - 1)] = sb;
                }
            X->S0 = (double *)calloc((size_t)nv * nv, sizeof(double));
            X->lam0 = (double *)calloc(nv, sizeof(double));
            gen_eig(nv, A0, B0, X->S0, X->lam0);
            free(A0); free(B0);
        }
    }
    m->sw = sw;
    return sw;
}

/* overlap count of lattice index I along an axis: extended sets [ex p - 1, ex p + p + 1] containing I */
static int ov_count(int nel, int p, int I)
{
    int c = 0;
    for (int ex = 0; ex < nel; ex++)
        if (I >= ex * p - 1 && I <= ex * p + p + 1) c++;
    return c;
}

/* Schwarz precision variants (reading 28), selected by the CG policy:
   SW_D   fp64 everything;
   SW_MIX mixed: fp32 vectors and fast-diagonalisation arithmetic, weights 1/sqrt(count) in fp64
          applied in fp64, the sums over subdomains (overlap and coarse assembly) in fp64;
   SW_F   fp32 everything (weights 1.0f / sqrtf((float)count)). */
enum { SW_D = 0, SW_MIX = 1, SW_F = 2 };

/* 3-D fast-diagonalisation apply in working precision T (T = double or float by macro):
   u = (Sz(x)Sy(x)Sx) diag(1/(lx+ly+lz)) (Sz(x)Sy(x)Sx)^T f on an nx x ny x nz box (x fastest).
   S given row-major with leading dimension ld.  Sums are sequential in the index order. */
#define OR_FDM_APPLY(NAME, T)                                                                               \
    static void NAME(int nx, int ny, int nz, const T *Sx, const T *Sy, const T *Sz, int ldx, int ldy, int ldz, \
                     const T *dinvl, const T *f, T *u, T *w1, T *w2)                                        \
    {                                                                                                       \
        /* w1 = Sx^T along x */                                                                             \
        for (int k = 0; k < nz; k++)                                                                        \
            for (int j = 0; j < ny; j++)                                                                    \
                for (int i = 0; i < nx; i++) {                                                              \
                    T s = 0;                                                                                \
                    for (int l = 0; l < nx; l++) s = s + Sx[l * ldx + i] * f[l + nx * (j + ny * k)];        \
                    w1[i + nx * (j + ny * k)] = s;                                                          \
                }                                                                                           \
        for (int k = 0; k < nz; k++) /* w2 = Sy^T along y */                                                \
            for (int j = 0; j < ny; j++)                                                                    \
                for (int i = 0; i < nx; i++) {                                                              \
                    T s = 0;                                                                                \
                    for (int l = 0; l < ny; l++) s = s + Sy[l * ldy + j] * w1[i + nx * (l + ny * k)];       \
                    w2[i + nx * (j + ny * k)] = s;                                                          \
                }                                                                                           \
        for (int k = 0; k < nz; k++) /* w1 = Sz^T along z, then the eigenvalue scaling */                   \
            for (int j = 0; j < ny; j++)                                                                    \
                for (int i = 0; i < nx; i++) {                                                              \
                    T s = 0;                                                                                \
                    for (int l = 0; l < nz; l++) s = s + Sz[l * ldz + k] * w2[i + nx * (j + ny * l)];       \
                    w1[i + nx * (j + ny * k)] = s * dinvl[i + nx * (j + ny * k)];                           \
                }                                                                                           \
        for (int k = 0; k < nz; k++) /* w2 = Sz along z */                                                  \
            for (int j = 0; j < ny; j++)                                                                    \
                for (int i = 0; i < nx; i++) {                                                              \
                    T s = 0;                                                                                \
                    for (int l = 0; l < nz; l++) s = s + Sz[k * ldz + l] * w1[i + nx * (j + ny * l)];       \
                    w2[i + nx * (j + ny * k)] = s;                                                          \
                }                                                                                           \
        for (int k = 0; k < nz; k++) /* w1 = Sy along y */                                                  \
            for (int j = 0; j < ny; j++)                                                                    \
                for (int i = 0; i < nx; i++) {                                                              \
                    T s = 0;                                                                                \
                    for (int l = 0; l < ny; l++) s = s + Sy[j * ldy + l] * w2[i + nx * (l + ny * k)];       \
                    w1[i + nx * (j + ny * k)] = s;                                                          \
                }                                                                                           \
        for (int k = 0; k < nz; k++) /* u = Sx along x */                                                   \
            for (int j = 0; j < ny; j++)                                                                    \
                for (int i = 0; i < nx; i++) {                                                              \
                    T s = 0;                                                                                \
                    for (int l = 0; l < nx; l++) s = s + Sx[i * ldx + l] * w1[l + nx * (j + ny * k)];       \
                    u[i + nx * (j + ny * k)] = s;                                                           \
                }                                                                                           \
    }
OR_FDM_APPLY(fdm_apply_d, double)
OR_FDM_APPLY(fdm_apply_f, float)

/* z = M^-1 r on the local copies (r consistent: every copy of a global node holds its value).
   rd / zd: double vectors (SW_D); rf / zf: float vectors (SW_MIX, SW_F). */
/* the overlap sum of the local solutions at one copy under the gather-scatter orders of the
   per-copy / rank-partitioned modes (NEXT-2 crossed with NEXT-4, reading 28): the
   contributions c_k (k ascending in element order, element e_k of rank r_k, TG values) of the
   boxes holding the node are combined like the copies of a node in the ranked dssum
   (OR_DSSUM_RANKED): OR_GS_PER_COPY: the copy's own element's box first, then the others
   ascending; OR_GS_PAIRWISE: rank partials (ascending within a rank), the copy's own rank's first,
   then the other ranks ascending; OR_GS_ALLREDUCE: all rank partials in ascending rank order. */
#define OR_SW_COMBINE(NAME, TGX)                                                                  \
    static TGX NAME(int order, int cnt, const TGX *c, const int64_t *ek, const int *rk, int64_t eown, int rown) \
    {                                                                                             \
        TGX t = 0;                                                                                \
        if (order == OR_GS_PER_COPY) {                                                            \
            for (int k = 0; k < cnt; k++)                                                         \
                if (ek[k] == eown) t += c[k];                                                     \
            for (int k = 0; k < cnt; k++)                                                         \
                if (ek[k] != eown) t += c[k];                                                     \
            return t;                                                                             \
        }                                                                                         \
        TGX part[27];                                                                             \
        for (int k = 0; k < cnt; k++) {                                                           \
            TGX u = 0;                                                                            \
            for (int k2 = 0; k2 < cnt; k2++)                                                      \
                if (rk[k2] == rk[k]) u += c[k2];                                                  \
            part[k] = u;                                                                          \
        }                                                                                         \
        int own = -1;                                                                             \
        for (int k = 0; k < cnt; k++)                                                             \
            if (rk[k] == rown) { own = k; break; }                                                \
        if (order == OR_GS_PAIRWISE && own >= 0) t = part[own];                                   \
        int prev = -1;                                                                            \
        for (;;) {                                                                                \
            int best = -1;                                                                        \
            for (int k = 0; k < cnt; k++)                                                         \
                if (rk[k] > prev && (best < 0 || rk[k] < rk[best])) best = k;                     \
            if (best < 0) break;                                                                  \
            prev = rk[best];                                                                      \
            if (order == OR_GS_PAIRWISE && own >= 0 && rk[best] == rown) continue;                \
            t += part[best];                                                                      \
        }                                                                                         \
        return t;                                                                                 \
    }
OR_SW_COMBINE(sw_combine_d, double)
OR_SW_COMBINE(sw_combine_f, float)

static void schwarz_apply_ord(or_mesh *m, int var, int order, const double *rd, double *zd, const float *rf, float *zf);
static inline void schwarz_apply(or_mesh *m, int var, const double *rd, double *zd, const float *rf, float *zf)
{
    schwarz_apply_ord(m, var, OR_GS_CONSISTENT, rd, zd, rf, zf);
}

static void schwarz_apply_ord(or_mesh *m, int var, int order, const double *rd, double *zd, const float *rf, float *zf)
{
    struct or_schwarz *sw = schwarz_setup(m);
    const int p = m->p, P3 = p + 3, n = m->n;
    const int64_t NX = m->NX, NY = m->NY, NZ = m->NZ, NG = m->NG, NL = m->NL;
    const struct or_sw_axis *X = &sw->ax[0], *Y = &sw->ax[1], *Z = &sw->ax[2];
    /* 1. the global lattice vector (any copy) and the accumulator (fp64 unless SW_F) */
    double *rg = (double *)calloc(NG, sizeof(double)), *zg = (double *)calloc(NG, sizeof(double));
    float *rgf = (float *)calloc(NG, sizeof(float)), *zgf = (float *)calloc(NG, sizeof(float));
    for (int64_t l = 0; l < NL; l++) {
        if (var == SW_D) rg[m->gid[l]] = rd[l];
        else rgf[m->gid[l]] = rf[l];
    }
    const int mx = P3 * P3 * P3;
    double *fd = (double *)malloc(mx * sizeof(double)), *ud = (double *)malloc(mx * sizeof(double));
    double *w1d = (double *)malloc(mx * sizeof(double)), *w2d = (double *)malloc(mx * sizeof(double));
    double *dld = (double *)malloc(mx * sizeof(double));
    float *ff = (float *)malloc(mx * sizeof(float)), *uf = (float *)malloc(mx * sizeof(float));
    float *w1f = (float *)malloc(mx * sizeof(float)), *w2f = (float *)malloc(mx * sizeof(float));
    float *dlf = (float *)malloc(mx * sizeof(float));
    float *Sxf = (float *)malloc(P3 * P3 * sizeof(float)), *Syf = (float *)malloc(P3 * P3 * sizeof(float));
    float *Szf = (float *)malloc(P3 * P3 * sizeof(float));
    /* per element (other orders): the unweighted local solution on its box (TG values) */
    const int ordered = order != OR_GS_CONSISTENT;
    double *ue_d = ordered && var != SW_F ? (double *)calloc((size_t)m->E * P3 * P3 * P3, sizeof(double)) : NULL;
    float *ue_f = ordered && var == SW_F ? (float *)calloc((size_t)m->E * P3 * P3 * P3, sizeof(float)) : NULL;
    double *cgd = (double *)calloc(NG, sizeof(double));   /* coarse term per node (TV value widened) */
    /* 2. local solves on the extended boxes, elements in ascending order */
    for (int64_t e = 0; e < m->E; e++) {
        int ex, ey, ez;
        element_xyz(m, e, &ex, &ey, &ez);
        const int nx = X->nt[ex], ny = Y->nt[ey], nz = Z->nt[ez];
        if (nx <= 0 || ny <= 0 || nz <= 0) continue;
        const int I0 = X->t0[ex], J0 = Y->t0[ey], K0 = Z->t0[ez];
        const double *Sx = X->S + (size_t)ex * P3 * P3, *Sy = Y->S + (size_t)ey * P3 * P3, *Sz = Z->S + (size_t)ez * P3 * P3;
        const double *lx = X->lam + (size_t)ex * P3, *ly = Y->lam + (size_t)ey * P3, *lz = Z->lam + (size_t)ez * P3;
        for (int k = 0; k < nz; k++)
            for (int j = 0; j < ny; j++)
                for (int i = 0; i < nx; i++) {
                    const int q = i + nx * (j + ny * k);
                    const int64_t G = (I0 + i) + NX * ((J0 + j) + NY * (int64_t)(K0 + k));
                    const int cnt = ov_count(m->nelx, p, I0 + i) * ov_count(m->nely, p, J0 + j) * ov_count(m->nelz, p, K0 + k);
                    const double dl = 1.0 / (lx[i] + ly[j] + lz[k]);
                    if (var == SW_D) {
                        fd[q] = rg[G] * (1.0 / sqrt((double)cnt));
                        dld[q] = dl;
                    } else if (var == SW_MIX) {
                        ff[q] = (float)((double)rgf[G] * (1.0 / sqrt((double)cnt)));
                        dlf[q] = (float)dl;
                    } else {
                        ff[q] = rgf[G] * (1.0f / sqrtf((float)cnt));
                        dlf[q] = (float)dl;
                    }
                }
        if (var == SW_D) {
            fdm_apply_d(nx, ny, nz, Sx, Sy, Sz, P3, P3, P3, dld, fd, ud, w1d, w2d);
        } else {
            for (int i = 0; i < P3 * P3; i++) { Sxf[i] = (float)Sx[i]; Syf[i] = (float)Sy[i]; Szf[i] = (float)Sz[i]; }
            fdm_apply_f(nx, ny, nz, Sxf, Syf, Szf, P3, P3, P3, dlf, ff, uf, w1f, w2f);
        }
        for (int k = 0; k < nz; k++)
            for (int j = 0; j < ny; j++)
                for (int i = 0; i < nx; i++) {
                    const int q = i + nx * (j + ny * k);
                    const int64_t G = (I0 + i) + NX * ((J0 + j) + NY * (int64_t)(K0 + k));
                    const int cnt = ov_count(m->nelx, p, I0 + i) * ov_count(m->nely, p, J0 + j) * ov_count(m->nelz, p, K0 + k);
                    if (var == SW_D) zg[G] = zg[G] + ud[q] * (1.0 / sqrt((double)cnt));
                    else if (var == SW_MIX) zg[G] = zg[G] + (double)uf[q] * (1.0 / sqrt((double)cnt));
                    else zgf[G] = zgf[G] + uf[q] * (1.0f / sqrtf((float)cnt));
                    if (ue_d) ue_d[(size_t)e * P3 * P3 * P3 + q] = var == SW_D ? ud[q] : (double)uf[q];
                    if (ue_f) ue_f[(size_t)e * P3 * P3 * P3 + q] = uf[q];
                }
    }
    /* 3. coarse correction: b0 = Phi^T r (sums in fp64 unless SW_F), x0 = A0^-1 b0, z += Phi x0 */
    const int nvx = X->nv, nvy = Y->nv, nvz = Z->nv;
    if (nvx > 0 && nvy > 0 && nvz > 0) {
        const int64_t V = (int64_t)nvx * nvy * nvz;
        double *b0 = (double *)calloc(V, sizeof(double)), *x0 = (double *)calloc(V, sizeof(double));
        double *c1 = (double *)calloc(V, sizeof(double)), *c2 = (double *)calloc(V, sizeof(double));
        double *dl0 = (double *)calloc(V, sizeof(double));
        float *b0f = (float *)calloc(V, sizeof(float)), *x0f = (float *)calloc(V, sizeof(float));
        float *c1f = (float *)calloc(V, sizeof(float)), *c2f = (float *)calloc(V, sizeof(float));
        float *dl0f = (float *)calloc(V, sizeof(float));
        float *S0x = (float *)malloc((size_t)nvx * nvx * sizeof(float)), *S0y = (float *)malloc((size_t)nvy * nvy * sizeof(float));
        float *S0z = (float *)malloc((size_t)nvz * nvz * sizeof(float));
        for (int64_t v = 0; v < V; v++) {
            const int vx = (int)(v % nvx), vy = (int)((v / nvx) % nvy), vz = (int)(v / ((int64_t)nvx * nvy));
            /* b0[v] = sum over the lattice points of the vertex's support, ascending lattice id */
            double sd = 0.0;
            float sf = 0.0f;
            for (int K = vz * p; K <= (vz + 2) * p; K++)
                for (int J = vy * p; J <= (vy + 2) * p; J++)
                    for (int I = vx * p; I <= (vx + 2) * p; I++) {
                        const double ph = hat(m, vx + 1, I) * hat(m, vy + 1, J) * hat(m, vz + 1, K);
                        if (ph == 0.0) continue;
                        const int64_t G = I + NX * (J + NY * (int64_t)K);
                        if (var == SW_D) sd = sd + ph * rg[G];
                        else if (var == SW_MIX) sd = sd + ph * (double)rgf[G];
                        else sf = sf + (float)ph * rgf[G];
                    }
            b0[v] = sd;
            b0f[v] = (var == SW_MIX) ? (float)sd : sf;
            const double dl = 1.0 / (X->lam0[vx] + Y->lam0[vy] + Z->lam0[vz]);
            dl0[v] = dl;
            dl0f[v] = (float)dl;
        }
        if (var == SW_D) {
            fdm_apply_d(nvx, nvy, nvz, X->S0, Y->S0, Z->S0, nvx, nvy, nvz, dl0, b0, x0, c1, c2);
        } else {
            for (int i = 0; i < nvx * nvx; i++) S0x[i] = (float)X->S0[i];
            for (int i = 0; i < nvy * nvy; i++) S0y[i] = (float)Y->S0[i];
            for (int i = 0; i < nvz * nvz; i++) S0z[i] = (float)Z->S0[i];
            fdm_apply_f(nvx, nvy, nvz, S0x, S0y, S0z, nvx, nvy, nvz, dl0f, b0f, x0f, c1f, c2f);
        }
        /* z[G] += sum over the (up to 8) interior vertices whose hats cover G, ascending vertex id */
        for (int64_t K = 1; K < NZ - 1; K++)
            for (int64_t J = 1; J < NY - 1; J++)
                for (int64_t I = 1; I < NX - 1; I++) {
                    const int64_t G = I + NX * (J + NY * K);
                    double sd = 0.0;
                    float sf = 0.0f;
                    const int ix = (int)(I / p), iy = (int)(J / p), iz = (int)(K / p);
                    for (int vz = iz - 1; vz <= iz + 1; vz++)
                        for (int vy = iy - 1; vy <= iy + 1; vy++)
                            for (int vx = ix - 1; vx <= ix + 1; vx++) {
                                if (vx < 1 || vx > nvx || vy < 1 || vy > nvy || vz < 1 || vz > nvz) continue;
                                const double ph = hat(m, vx, (int)I) * hat(m, vy, (int)J) * hat(m, vz, (int)K);
                                if (ph == 0.0) continue;
                                const int64_t v = (vx - 1) + nvx * ((vy - 1) + (int64_t)nvy * (vz - 1));
                                if (var == SW_D) sd = sd + ph * x0[v];
                                else sf = sf + (float)ph * x0f[v];
                            }
                    if (var == SW_D) zg[G] = zg[G] + sd;
                    else if (var == SW_MIX) zg[G] = zg[G] + (double)sf;
                    else zgf[G] = zgf[G] + sf;
                    cgd[G] = var == SW_D ? sd : (double)sf;
                }
        free(b0); free(x0); free(c1); free(c2); free(dl0); free(b0f); free(x0f); free(c1f); free(c2f); free(dl0f);
        free(S0x); free(S0y); free(S0z);
    }
    /* 4. back to the local copies (Dirichlet copies 0: the boxes and hats exclude them) */
    for (int64_t l = 0; l < NL; l++) {
        const int64_t G = m->gid[l];
        if (var == SW_D) zd[l] = m->mask[l] ? zg[G] : 0.0;
        else if (var == SW_MIX) zf[l] = m->mask[l] ? (float)zg[G] : 0.0f;
        else zf[l] = m->mask[l] ? zgf[G] : 0.0f;
    }
    /* 4'. other gather-scatter orders: every copy combines the box contributions of its node in
       its own order (OR_SW_COMBINE), then adds the coarse term */
    if (ordered) {
        const int64_t n3 = (int64_t)n * n * n;
        for (int64_t l = 0; l < NL; l++) {
            if (!m->mask[l]) continue;
            const int64_t G = m->gid[l];
            const int I = (int)(G % NX), J = (int)((G / NX) % NY), K = (int)(G / (NX * NY));
            const int cnt = ov_count(m->nelx, p, I) * ov_count(m->nely, p, J) * ov_count(m->nelz, p, K);
            double cd[27];
            float cf[27];
            int64_t ek[27];
            int rk[27];
            int nc = 0;
            for (int ez = K / p - 1; ez <= K / p + 1; ez++)
                for (int ey = J / p - 1; ey <= J / p + 1; ey++)
                    for (int ex = I / p - 1; ex <= I / p + 1; ex++) {
                        if (ex < 0 || ex >= m->nelx || ey < 0 || ey >= m->nely || ez < 0 || ez >= m->nelz) continue;
                        const int I0 = X->t0[ex], J0 = Y->t0[ey], K0 = Z->t0[ez];
                        const int nx = X->nt[ex], ny = Y->nt[ey], nz = Z->nt[ez];
                        if (I < I0 || I >= I0 + nx || J < J0 || J >= J0 + ny || K < K0 || K >= K0 + nz) continue;
                        const int64_t e = ex + (int64_t)m->nelx * (ey + (int64_t)m->nely * ez);
                        const size_t q = (size_t)e * P3 * P3 * P3 + (size_t)((I - I0) + nx * ((J - J0) + ny * (K - K0)));
                        if (var == SW_F) cf[nc] = ue_f[q] * (1.0f / sqrtf((float)cnt));
                        else cd[nc] = ue_d[q] * (1.0 / sqrt((double)cnt));
                        ek[nc] = e;
                        rk[nc] = elem_rank(m, e);
                        nc++;
                    }
            const int64_t eown = l / n3;
            const int rown = elem_rank(m, eown);
            if (var == SW_D) zd[l] = sw_combine_d(order, nc, cd, ek, rk, eown, rown) + cgd[G];
            else if (var == SW_MIX) zf[l] = (float)(sw_combine_d(order, nc, cd, ek, rk, eown, rown) + cgd[G]);
            else zf[l] = sw_combine_f(order, nc, cf, ek, rk, eown, rown) + (float)cgd[G];
        }
    }
    free(ue_d); free(ue_f); free(cgd);
    free(rg); free(zg); free(rgf); free(zgf); free(fd); free(ud); free(w1d); free(w2d); free(dld);
    free(ff); free(uf); free(w1f); free(w2f); free(dlf); free(Sxf); free(Syf); free(Szf);
}

int or_schwarz_apply_d(or_mesh *m, int order, const double *r, double *z)
{
    if (!m || !r || !z || order < OR_GS_CONSISTENT || order > OR_GS_ALLREDUCE) return 1;
    schwarz_apply_ord(m, SW_D, order, r, z, NULL, NULL);
    return 0;
}
int or_schwarz_apply_f(or_mesh *m, int policy, int order, const float *r, float *z)
{
    if (!m || !r || !z || policy == OR_FP64 || order < OR_GS_CONSISTENT || order > OR_GS_ALLREDUCE) return 1;
    schwarz_apply_ord(m, policy == OR_MIXED ? SW_MIX : SW_F, order, NULL, NULL, r, z);
    return 0;
}
/* the fast-diagonalisation tables: per axis a and element position ex, t0/nt and S, lambda
   (S[(ex*(p+3)+i)*(p+3)+j]); coarse S0 (nv x nv), lam0.  Pointers valid while the mesh lives. */
int or_schwarz_tables(or_mesh *m, int axis, int ex, int *t0, int *nt, double *S, double *lam, double *S0, double *lam0)
{
    if (!m || axis < 0 || axis > 2) return 1;
    struct or_schwarz *sw = schwarz_setup(m);
    const struct or_sw_axis *X = &sw->ax[axis];
    const int P3 = m->p + 3;
    if (ex < 0 || ex >= X->nel) return 1;
    if (t0) *t0 = X->t0[ex];
    if (nt) *nt = X->nt[ex];
    if (S) memcpy(S, X->S + (size_t)ex * P3 * P3, sizeof(double) * P3 * P3);
    if (lam) memcpy(lam, X->lam + (size_t)ex * P3, sizeof(double) * P3);
    if (S0 && X->nv > 0) memcpy(S0, X->S0, sizeof(double) * X->nv * X->nv);
    if (lam0 && X->nv > 0) memcpy(lam0, X->lam0, sizeof(double) * X->nv);
    return 0;
}

/* ------------------------------------------------------------------ */
/* C-10 / C-11: PCG and the stagnation rule                             */
/* ------------------------------------------------------------------ */

/* C-11: status of a run that did not converge by max_iter. */
static int classify(const double *res, int k, int W)
{
    /* running minimum m_j = min_{i<=j} res_i */
    double mk = res[0];
    for (int i = 1; i <= k; i++) if (res[i] < mk) mk = res[i];
    if (res[k] > 100.0 * mk) return OR_STAGNATED;
    if (W > 0 && k >= W) {
        double mkw = res[0];
        for (int i = 1; i <= k - W; i++) if (res[i] < mkw) mkw = res[i];
        if (mk > 0.1 * mkw) return OR_STAGNATED;
    }
    return OR_MAXITER;
}

static void finish_report(or_report *rep, const double *res, int k, int status, double rtr0, double rtr)
{
    rep->iterations = k;
    rep->status = status;
    rep->rtr0 = rtr0;
    rep->rtr_final = rtr;
    rep->rel_res_final = res[k];
    double mn = res[0];
    for (int i = 1; i <= k; i++) if (res[i] < mn) mn = res[i];
    rep->rel_res_min = mn;
}

static double true_residual(const or_mesh *m, const double *b64, const double *x)
{
    const int64_t NL = m->NL;
    double *w = (double *)malloc(NL * sizeof(double));
    double *r = (double *)malloc(NL * sizeof(double));
    or_ax_d(m, OR_GS_CONSISTENT, x, w);
    for (int64_t l = 0; l < NL; l++) r[l] = b64[l] - w[l];
    double rr = or_glsc3_d(r, m->c, r, NL), bb = or_glsc3_d(b64, m->c, b64, NL);
    free(w); free(r);
    return bb > 0.0 ? sqrt(rr / bb) : 0.0;
}

/* sc (nullable): per iteration k = 1..iterations, sc[3(k-1) + 0..2] = rho_k, alpha_k, beta_k as
   the policy computes them (widened to double) -- the scalar recurrence of Table 2, exported so
   that tests can pin its precision (C-10 table, "rho, pap, alpha, beta" row). */
static void put_scal(double *sc, int k, double rho, double alpha, double beta)
{
    if (!sc) return;
    sc[3 * (k - 1) + 0] = rho;
    sc[3 * (k - 1) + 1] = alpha;
    sc[3 * (k - 1) + 2] = beta;
}

static int cg_fp64(const or_mesh *m, int max_iter, double rtol, int order, int W, int pc, const double *b64,
                   double *x, double *res, double *sc, or_report *rep)
{
    const int64_t NL = m->NL;
    double *r = (double *)malloc(NL * sizeof(double)), *p = (double *)malloc(NL * sizeof(double));
    double *z = (double *)malloc(NL * sizeof(double)), *w = (double *)malloc(NL * sizeof(double));
    for (int64_t l = 0; l < NL; l++) { x[l] = 0.0; r[l] = b64[l]; p[l] = 0.0; }
    double rtr0 = or_glsc3_d(r, m->c, r, NL), rtr = rtr0, rho = 0.0, rho_old = 1.0;
    res[0] = 1.0;
    int k = 0, status = OR_MAXITER;
    if (rtr0 == 0.0) { status = OR_CONVERGED; res[0] = 0.0; }
    else {
        for (k = 1; k <= max_iter; k++) {
            if (pc == OR_PC_IDENTITY) for (int64_t l = 0; l < NL; l++) z[l] = r[l];  /* solveM: none */
            else if (pc == OR_PC_SCHWARZ) schwarz_apply_ord((or_mesh *)m, SW_D, order, r, z, NULL, NULL);   /* NEXT-4 */
            else for (int64_t l = 0; l < NL; l++) z[l] = r[l] * m->dinv[l];          /* solveM */
            rho = or_glsc3_d(r, m->c, z, NL);                                        /* glsc3 */
            double beta = (k == 1) ? 0.0 : rho / rho_old;
            rho_old = rho;
            for (int64_t l = 0; l < NL; l++) p[l] = z[l] + beta * p[l];              /* add2s1 */
            or_ax_d(m, order, p, w);                                                 /* ax */
            double pap = or_glsc3_d(w, m->c, p, NL);                                 /* glsc3 */
            if (!(pap > 0.0) || !isfinite(pap) || !isfinite(rho)) { status = OR_BREAKDOWN; res[k] = res[k - 1]; break; }
            double alpha = rho / pap;
            put_scal(sc, k, rho, alpha, beta);
            for (int64_t l = 0; l < NL; l++) x[l] = x[l] + alpha * p[l];             /* add2s2 */
            for (int64_t l = 0; l < NL; l++) r[l] = r[l] - alpha * w[l];             /* add2s2 */
            rtr = or_glsc3_d(r, m->c, r, NL);                                        /* glsc3 */
            res[k] = sqrt(rtr / rtr0);
            if (!isfinite(rtr)) { status = OR_BREAKDOWN; break; }
            if (res[k] <= rtol || rtr == 0.0) { status = OR_CONVERGED; break; }
        }
        if (k > max_iter) { k = max_iter; status = rtol > 0.0 ? classify(res, k, W) : OR_MAXITER; }
    }
    finish_report(rep, res, k, status, rtr0, rtr);
    free(r); free(p); free(z); free(w);
    return 0;
}

/* fp32 and mixed policies (C-10 table). */
static int cg_f32(const or_mesh *m, int policy, int max_iter, double rtol, int order, int W, int seqdot,
                  int x64, int pc, const double *b64, double *x_out, double *res, double *sc, or_report *rep)
{
    const int64_t NL = m->NL;
    const int mixed = (policy == OR_MIXED);
    const int dot2 = (policy == OR_FP32_DOT2);   /* fp32 policy with compensated dot products */
    float *x = (float *)malloc(NL * sizeof(float)), *r = (float *)malloc(NL * sizeof(float));
    float *p = (float *)malloc(NL * sizeof(float)), *z = (float *)malloc(NL * sizeof(float));
    float *w = (float *)malloc(NL * sizeof(float));
    double *xd = (x64 && mixed) ? (double *)malloc(NL * sizeof(double)) : NULL;
    for (int64_t l = 0; l < NL; l++) { x[l] = 0.0f; r[l] = (float)b64[l]; p[l] = 0.0f; }
    if (xd) for (int64_t l = 0; l < NL; l++) xd[l] = 0.0;

    /* scalar recurrences: double under mixed, float under fp32 */
#define DOT(a, b) (mixed ? or_glsc3_mixed((a), m->c, (b), NL) \
                   : dot2 ? (double)or_glsc3_f_dot2((a), m->cf, (b), NL) \
                         : (double)(seqdot ? or_glsc3_f_seq((a), m->cf, (b), NL) : or_glsc3_f_tree((a), m->cf, (b), NL)))
    double rtr0 = DOT(r, r), rtr = rtr0;
    double rho = 0.0, rho_old = 1.0;
    float rho_f = 0.0f, rho_old_f = 1.0f;
    res[0] = 1.0;
    int k = 0, status = OR_MAXITER;
    if (rtr0 == 0.0) { status = OR_CONVERGED; res[0] = 0.0; }
    else {
        for (k = 1; k <= max_iter; k++) {
            /* solveM: mixed z = (float)((double)r * dinv64); fp32 (and the Neko-style fp32 copy
               under mixed) z = r * dinv32; identity z = r */
            if (pc == OR_PC_IDENTITY) for (int64_t l = 0; l < NL; l++) z[l] = r[l];
            else if (pc == OR_PC_SCHWARZ) schwarz_apply_ord((or_mesh *)m, mixed ? SW_MIX : SW_F, order, NULL, NULL, r, z);
            else if (mixed && pc == OR_PC_JACOBI) for (int64_t l = 0; l < NL; l++) z[l] = (float)((double)r[l] * m->dinv[l]);
            else for (int64_t l = 0; l < NL; l++) z[l] = r[l] * m->dinvf[l];
            float beta_f;
            double beta_sc;
            if (mixed) {
                rho = DOT(r, z);
                double beta = (k == 1) ? 0.0 : rho / rho_old;
                rho_old = rho;
                beta_sc = beta;
                beta_f = (float)beta;
            } else {
                rho_f = (float)DOT(r, z);
                beta_f = (k == 1) ? 0.0f : rho_f / rho_old_f;
                rho_old_f = rho_f;
                rho = rho_f;
                beta_sc = beta_f;
            }
            for (int64_t l = 0; l < NL; l++) p[l] = z[l] + beta_f * p[l];           /* add2s1 */
            or_ax_f(m, policy, order, p, w);                                         /* ax */
            float alpha_f;
            double pap;
            if (mixed) {
                pap = DOT(w, p);
                if (!(pap > 0.0) || !isfinite(pap) || !isfinite(rho)) { status = OR_BREAKDOWN; res[k] = res[k - 1]; break; }
                alpha_f = (float)(rho / pap);
                put_scal(sc, k, rho, rho / pap, beta_sc);
                if (xd) {
                    double alpha = rho / pap;
                    for (int64_t l = 0; l < NL; l++) xd[l] = xd[l] + alpha * (double)p[l];
                }
            } else {
                float pap_f = (float)DOT(w, p);
                pap = pap_f;
                if (!(pap_f > 0.0f) || !isfinite(pap_f) || !isfinite(rho_f)) { status = OR_BREAKDOWN; res[k] = res[k - 1]; break; }
                alpha_f = rho_f / pap_f;
                put_scal(sc, k, rho_f, alpha_f, beta_sc);
            }
            for (int64_t l = 0; l < NL; l++) x[l] = x[l] + alpha_f * p[l];           /* add2s2 */
            for (int64_t l = 0; l < NL; l++) r[l] = r[l] - alpha_f * w[l];           /* add2s2 */
            rtr = DOT(r, r);                                                         /* glsc3 */
            res[k] = sqrt(rtr / rtr0);
            if (!isfinite(rtr)) { status = OR_BREAKDOWN; break; }
            if (res[k] <= rtol || rtr == 0.0) { status = OR_CONVERGED; break; }
        }
        if (k > max_iter) { k = max_iter; status = rtol > 0.0 ? classify(res, k, W) : OR_MAXITER; }
    }
#undef DOT
    finish_report(rep, res, k, status, rtr0, rtr);
    for (int64_t l = 0; l < NL; l++) x_out[l] = xd ? xd[l] : (double)x[l];
    free(x); free(r); free(p); free(z); free(w); free(xd);
    return 0;
}

int or_cg(const or_mesh *m, int policy, int max_iter, double rtol, int gs_order, int stag_window,
          int seqdot, int x64, int precond, const double *b64, double *x_out, double *hist, double *scal,
          or_report *rep)
{
    if (!m || !b64 || !x_out || !rep || max_iter < 0 || rtol < 0.0) return 1;
    if (policy < OR_FP64 || policy > OR_FP32_DOT2) return 1;
    if (precond < OR_PC_JACOBI || precond > OR_PC_SCHWARZ) return 1;
    if (policy == OR_FP64 && precond == OR_PC_JACOBI_F32) return 1;
    if (x64 && policy != OR_MIXED) return 1;
    double *res = (double *)calloc((size_t)max_iter + 1, sizeof(double));
    int rc;
    if (policy == OR_FP64) rc = cg_fp64(m, max_iter, rtol, gs_order, stag_window, precond, b64, x_out, res, scal, rep);
    else rc = cg_f32(m, policy, max_iter, rtol, gs_order, stag_window, seqdot, x64, precond, b64, x_out, res, scal, rep);
    if (hist) for (int i = 0; i <= rep->iterations; i++) hist[i] = res[i];
    rep->true_res = true_residual(m, b64, x_out);
    free(res);
    return rc;
}

/* ------------------------------------------------------------------ */
/* C-5: right-hand sides                                                */
/* ------------------------------------------------------------------ */

void or_rhs(const or_mesh *m, int kind, double noise_amp, uint64_t seed, double *b)
{
    const int64_t NL = m->NL;
    if (kind == OR_RHS_UNIFORM) {
        for (int64_t l = 0; l < NL; l++)
            b[l] = m->mask[l] ? or_prng_u(seed, 1, (uint64_t)m->gid[l]) : 0.0;
        return;
    }
    const double pi = 3.14159265358979323846;
    const double *X = m->xyz, *Y = m->xyz + NL, *Z = m->xyz + 2 * NL;
    for (int64_t l = 0; l < NL; l++) {
        double f = 3.0 * pi * pi * sin(pi * X[l]) * sin(pi * Y[l]) * sin(pi * Z[l])
                 + noise_amp * or_prng_u(seed, 2, (uint64_t)m->gid[l]);
        b[l] = m->B[l] * f;
    }
    or_dssum_d(m, OR_GS_CONSISTENT, b);
    for (int64_t l = 0; l < NL; l++)
        if (!m->mask[l]) b[l] = 0.0;
}
