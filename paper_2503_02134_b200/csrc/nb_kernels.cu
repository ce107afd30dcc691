// nb_kernels.cu -- the sm_100a kernels of the SEM Jacobi-PCG hot path and of its setup.
//
//   k_ax   (K1)  local operator A_L ("ax_e": local_grad3, geometric scaling,
//                local_grad3_t), register pencils + shared-memory
//                transposes, D from constant memory; in CG mode fused with solveM +
//                add2s1 (p = z + beta p) on its loads and the interior part of
//                glsc3(w,c,p) in its epilogue.
//   k_gs   (K2)  gather-scatter QQ^T over the shared-node CSR segments (PAPER.md:309,
//                :404), consistent or per-copy order, accumulation in the policy's GS
//                precision; in CG mode + shared part of pap and
//                the alpha finalize.
//   k_upd  (K3)  add2s2 x2 + glsc3(r,c,r) + next solveM/glsc3(r,c,z) + finalize
//                (PAPER.md:165-167, :161).
//   setup kernels: geometry (C-2/C-3/C-6), Jacobi diagonal (C-9), GS segments (C-4),
//                RHS (C-5), casts, map export.
#include <cub/device/device_scan.cuh>

#include "nb_common.cuh"

namespace nb {

cudaError_t upload_basis(int n, const double *D)
{
    float Df[256];
    for (int i = 0; i < n * n; i++) Df[i] = (float)D[i];
    cudaError_t e = cudaMemcpyToSymbol(c_D64, D, sizeof(double) * n * n, sizeof(double) * n * 256);
    if (e != cudaSuccess) return e;
    return cudaMemcpyToSymbol(c_D32, Df, sizeof(float) * n * n, sizeof(float) * n * 256);
}

// ===========================================================================
// K1: local operator
// ===========================================================================
template <typename T, int N> struct AxGeom {
    static constexpr int N2 = N * N;
    static constexpr int N3 = N * N * N;
    static constexpr int BANKS = (sizeof(T) == 4) ? 32 : 16;
    // plane pitch P >= N^2 with P == N (mod BANKS): the stride-N s-pencil reads of a warp
    // (threads q = a + N b, address a + N j + P b) hit consecutive banks.
    static constexpr int P = N2 + (((N - N2) % BANKS) + BANKS) % BANKS;
    static constexpr int ESZ = P * N;                       // one array, one element
    static constexpr int EPB = (N2 >= 256) ? 1 : (256 / N2);  // elements per block
    static constexpr int NT = ((EPB * N2 + 31) / 32) * 32;   // threads per block
    static constexpr size_t SMEM = (size_t)3 * EPB * ESZ * sizeof(T);
};

// MODE 0: standalone w = A_L u (+ mask unless local).  MODE 1: CG K1.
template <int PREC, int N, int MODE>
__global__ void __launch_bounds__(AxGeom<typename Pol<PREC>::TV, N>::NT)
k_ax(const MeshDev m, const typename Pol<PREC>::TV *__restrict__ u_or_r,
     const typename Pol<PREC>::TJ *__restrict__ dinv, typename Pol<PREC>::TV *__restrict__ pv,
     const typename Pol<PREC>::TV *__restrict__ g, typename Pol<PREC>::TV *__restrict__ w, int apply_mask,
     const Scal *__restrict__ scal, double *__restrict__ part)
{
    using TV = typename Pol<PREC>::TV;
    using TJ = typename Pol<PREC>::TJ;
    using TS = typename Pol<PREC>::TS;
    using T = TV;
    using G = AxGeom<T, N>;
    extern __shared__ __align__(16) unsigned char smraw[];
    T *sm = reinterpret_cast<T *>(smraw);

    if (MODE == 1 && scal->done) return;   // block-uniform
    const int tid = threadIdx.x;
    const int el = tid / G::N2;
    const int q = tid - el * G::N2;
    const int a = q % N, b = q / N;
    const bool slot = el < G::EPB;
    T *A0 = sm + (slot ? el : 0) * 3 * G::ESZ;
    T *A1 = A0 + G::ESZ;
    T *A2 = A1 + G::ESZ;
    const int rp = N * a + G::P * b;          // smem offset of this thread's r-pencil (i, a, b)
    const int sp = a + G::P * b;              // s-pencil (a, j, b) base, stride N
    const int tp = a + N * b;                 // t-pencil (a, b, k) base, stride P

    TV beta_v = 0;
    if (MODE == 1) beta_v = (TV)(TS)scal->beta;
    TS acc = 0;
    const int64_t ngroups = (m.E + G::EPB - 1) / G::EPB;

    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const int64_t e = grp * G::EPB + el;
        const bool active = slot && e < m.E;
        const int64_t gbase = e * G::N3 + (int64_t)N * q;   // global offset of the r-pencil
        T ru[N];
        // ---- 1. load u (CG: p = z + beta p, z = M^-1 r) as r-pencils, stage in shared
        if (active) {
            if (MODE == 1) {
                TV rr[N], pp[N];
                TJ dd[N];
                ld_pencil<TV, N>(u_or_r + gbase, rr);
                ld_pencil<TJ, N>(dinv + gbase, dd);
                ld_pencil<TV, N>(pv + gbase, pp);
#pragma unroll
                for (int i = 0; i < N; i++) {
                    TV z = (TV)((TJ)rr[i] * dd[i]);          // solveM (Jacobi)
                    ru[i] = fma(beta_v, pp[i], z);           // add2s1
                }
                st_pencil<TV, N>(pv + gbase, ru);
            } else {
                ld_pencil<TV, N>(u_or_r + gbase, ru);
            }
            st_pencil<T, N>(A0 + rp, ru);
        }
        __syncthreads();
        // ---- 2. us along s, ut along t (local_grad3), pencils read from shared
        if (active) {
            T v[N], o[N];
#pragma unroll
            for (int j = 0; j < N; j++) v[j] = A0[sp + N * j];
            contract<T, N>(v, o);
#pragma unroll
            for (int j = 0; j < N; j++) A1[sp + N * j] = o[j];
#pragma unroll
            for (int k = 0; k < N; k++) v[k] = A0[tp + G::P * k];
            contract<T, N>(v, o);
#pragma unroll
            for (int k = 0; k < N; k++) A2[tp + G::P * k] = o[k];
        }
        __syncthreads();
        // ---- 3. ur in registers; geometric scaling; r-part of local_grad3_t
        T wr_t[N];
        if (active) {
            T ur[N], us[N], ut[N];
            contract<T, N>(ru, ur);
            ld_pencil<T, N>(A1 + rp, us);
            ld_pencil<T, N>(A2 + rp, ut);
            const T *ge = g + e * 6 * G::N3 + (int64_t)N * q;
            T g1[N], g2[N], g3[N];
            ld_pencil<T, N>(ge, g1);
            ld_pencil<T, N>(ge + G::N3, g2);
            ld_pencil<T, N>(ge + 2 * G::N3, g3);
            T wr[N], ws[N], wt[N];
#pragma unroll
            for (int i = 0; i < N; i++) {
                wr[i] = g1[i] * ur[i] + g2[i] * us[i] + g3[i] * ut[i];
                ws[i] = g2[i] * ur[i];
                wt[i] = g3[i] * ur[i];
            }
            T g4[N], g5[N], g6[N];
            ld_pencil<T, N>(ge + 3 * G::N3, g4);
            ld_pencil<T, N>(ge + 4 * G::N3, g5);
            ld_pencil<T, N>(ge + 5 * G::N3, g6);
#pragma unroll
            for (int i = 0; i < N; i++) {
                ws[i] = ws[i] + g4[i] * us[i] + g5[i] * ut[i];
                wt[i] = wt[i] + g5[i] * us[i] + g6[i] * ut[i];
            }
            st_pencil<T, N>(A1 + rp, ws);
            st_pencil<T, N>(A2 + rp, wt);
            contract_t<T, N>(wr, wr_t);
        }
        __syncthreads();
        // ---- 4. s- and t-parts of local_grad3_t, in place on the owner's pencils
        if (active) {
            T v[N], o[N];
#pragma unroll
            for (int j = 0; j < N; j++) v[j] = A1[sp + N * j];
            contract_t<T, N>(v, o);
#pragma unroll
            for (int j = 0; j < N; j++) A1[sp + N * j] = o[j];
#pragma unroll
            for (int k = 0; k < N; k++) v[k] = A2[tp + G::P * k];
            contract_t<T, N>(v, o);
#pragma unroll
            for (int k = 0; k < N; k++) A2[tp + G::P * k] = o[k];
        }
        __syncthreads();
        // ---- 5. w = (w_r + w_s) + w_t, mask, store; CG: interior pap partial
        if (active) {
            T ws_t[N], wt_t[N], out[N];
            ld_pencil<T, N>(A1 + rp, ws_t);
            ld_pencil<T, N>(A2 + rp, wt_t);
#pragma unroll
            for (int i = 0; i < N; i++) out[i] = (wr_t[i] + ws_t[i]) + wt_t[i];
            if (MODE == 1 || apply_mask) {
                const ElemPos P = elem_pos(m, e);
                const bool mjk = axis_bnd(a, N, P.ey, m.nely) || axis_bnd(b, N, P.ez, m.nelz);
                const bool sjk = axis_mult(a, N, P.ey, m.nely) * axis_mult(b, N, P.ez, m.nelz) > 1;
                T pp[N];
                if (MODE == 1) ld_pencil<T, N>(A0 + rp, pp);
#pragma unroll
                for (int i = 0; i < N; i++) {
                    const bool msk = mjk || axis_bnd(i, N, P.ex, m.nelx);
                    if (msk) out[i] = T(0);
                    if (MODE == 1) {
                        const bool shared = sjk || axis_mult(i, N, P.ex, m.nelx) > 1;
                        if (!shared) acc += (TS)out[i] * (TS)pp[i];   // c = 1 on unshared nodes
                    }
                }
            }
            st_pencil<T, N>(w + gbase, out);
        }
        __syncthreads();
    }
    if (MODE == 1) {
        __shared__ TS red[32];
        TS s = block_sum<TS>(acc, red);
        if (tid == 0) part[blockIdx.x] = (double)s;
    }
}

// ===========================================================================
// K2: gather-scatter over CSR segments
// ===========================================================================
// MODE 0: standalone.  MODE 1: CG (shared pap partial + finalize alpha).
template <int PREC, int ORDER, int MODE, typename TVX, typename TGX>
__global__ void __launch_bounds__(256)
k_gs(const int32_t nseg, const int32_t *__restrict__ off, const int32_t *__restrict__ idx,
     TVX *__restrict__ w, const TVX *__restrict__ pv, Scal *__restrict__ scal, double *__restrict__ part,
     const int nblk_ax, cudaGraphConditionalHandle cond, int use_cond)
{
    using TS = typename Pol<PREC>::TS;
    if (MODE == 1 && scal->done) return;
    TS acc = 0;
    for (int32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < nseg; s += gridDim.x * blockDim.x) {
        const int32_t a0 = off[s];
        const int32_t cnt = off[s + 1] - a0;
        int32_t id[8];
        TGX v[8];
#pragma unroll
        for (int c = 0; c < 8; c++)
            if (c < cnt) { id[c] = idx[a0 + c]; v[c] = (TGX)w[id[c]]; }
        if (ORDER == NB_GS_CONSISTENT) {
            TGX t = v[0];
#pragma unroll
            for (int c = 1; c < 8; c++)
                if (c < cnt) t += v[c];
            const TVX tv = (TVX)t;
#pragma unroll
            for (int c = 0; c < 8; c++)
                if (c < cnt) w[id[c]] = tv;
            if (MODE == 1) acc += (TS)tv * (TS)pv[id[0]];   // sum_copies c*w*p = sigma*p (p continuous)
        } else {
            const TS cinv = (TS)1 / (TS)cnt;
#pragma unroll
            for (int c = 0; c < 8; c++) {
                if (c < cnt) {
                    TGX t = v[c];
#pragma unroll
                    for (int r = 0; r < 8; r++)
                        if (r < cnt && r != c) t += v[r];
                    const TVX tv = (TVX)t;
                    w[id[c]] = tv;
                    if (MODE == 1) acc += ((TS)tv * cinv) * (TS)pv[id[c]];
                }
            }
        }
    }
    if (MODE == 1) {
        __shared__ TS red[32];
        TS s = block_sum<TS>(acc, red);
        if (threadIdx.x == 0) part[nblk_ax + blockIdx.x] = (double)s;
        if (last_block(&scal->cnt_gs)) {
            TS pap = block_sum_array<TS>(part, nblk_ax + gridDim.x, 1, red);
            if (threadIdx.x == 0) {
                const TS rho = (TS)scal->rho;
                scal->pap = (double)pap;
                if (!(pap > (TS)0) || !isfinite((double)pap) || !isfinite((double)rho)) {
                    scal->status = NB_BROKEDOWN;
                    scal->done = 1;
                } else {
                    scal->alpha = (double)(rho / pap);
                }
                scal->cnt_gs = 0;
            }
        }
    }
}

// ===========================================================================
// K3: x += alpha p; r -= alpha w; rtr; rho_next = glsc3(r, c, M^-1 r); finalize.
// One thread per r-pencil; c = 1/mult is analytic on the box.
// ===========================================================================
template <int PREC, int N>
__global__ void __launch_bounds__(256)
k_upd(const MeshDev m, typename Pol<PREC>::TV *__restrict__ x, const typename Pol<PREC>::TV *__restrict__ pv,
      typename Pol<PREC>::TV *__restrict__ r, const typename Pol<PREC>::TV *__restrict__ w,
      const typename Pol<PREC>::TJ *__restrict__ dinv, Scal *__restrict__ scal, double *__restrict__ part,
      double *__restrict__ hist, cudaGraphConditionalHandle cond, int use_cond)
{
    using TV = typename Pol<PREC>::TV;
    using TJ = typename Pol<PREC>::TJ;
    using TS = typename Pol<PREC>::TS;
    if (scal->done) {
        if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    const TV alpha_v = (TV)(TS)scal->alpha;
    TS rtr = 0, rho = 0;
    const int64_t npen = m.E * N * N;
    for (int64_t pid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pid < npen;
         pid += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = pid / (N * N);
        const int q = (int)(pid - e * (N * N));
        const int a = q % N, b = q / N;
        const int64_t base = pid * N;
        TV xx[N], pp[N], rr[N], ww[N];
        TJ dd[N];
        ld_pencil<TV, N>(x + base, xx);
        ld_pencil<TV, N>(pv + base, pp);
        ld_pencil<TV, N>(r + base, rr);
        ld_pencil<TV, N>(w + base, ww);
        ld_pencil<TJ, N>(dinv + base, dd);
        const ElemPos P = elem_pos(m, e);
        const int mjk = axis_mult(a, N, P.ey, m.nely) * axis_mult(b, N, P.ez, m.nelz);
#pragma unroll
        for (int i = 0; i < N; i++) {
            xx[i] = fma(alpha_v, pp[i], xx[i]);      // add2s2(x, p, alpha)
            rr[i] = fma(-alpha_v, ww[i], rr[i]);     // add2s2(r, w, -alpha)
            const TS c = (TS)1 / (TS)(mjk * axis_mult(i, N, P.ex, m.nelx));
            const TS rs = (TS)rr[i];
            rtr += (rs * c) * rs;
            const TV z = (TV)((TJ)rr[i] * dd[i]);
            rho += (rs * c) * (TS)z;
        }
        st_pencil<TV, N>(x + base, xx);
        st_pencil<TV, N>(r + base, rr);
    }
    __shared__ TS red[32];
    TS s1 = block_sum<TS>(rtr, red);
    TS s2 = block_sum<TS>(rho, red);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = (double)s1;
        part[2 * blockIdx.x + 1] = (double)s2;
    }
    if (last_block(&scal->cnt_upd)) {
        TS trtr = block_sum_array<TS>(part, gridDim.x, 2, red);
        TS trho = block_sum_array<TS>(part + 1, gridDim.x, 2, red);
        if (threadIdx.x == 0) {
            const int it = scal->iter + 1;
            const double res = sqrt((double)trtr / scal->rtr0);
            hist[it] = res;
            int done = 0;
            if (!isfinite((double)trtr) || !isfinite((double)trho)) {
                scal->status = NB_BROKEDOWN;
                done = 1;
            } else if (res <= scal->rtol || trtr == (TS)0) {
                scal->status = NB_CONVERGED;
                done = 1;
            } else if (it >= scal->max_iter) {
                scal->status = NB_MAXITER;
                done = 1;
            }
            const TS rho_old = (TS)scal->rho;
            scal->beta = (double)(trho / rho_old);
            scal->rho = (double)trho;
            scal->rtr = (double)trtr;
            scal->iter = it;
            scal->done = done;
            scal->cnt_upd = 0;
            if (done && use_cond) cudaGraphSetConditional(cond, 0);
        }
    }
}

// CG prologue on the workspace: r already holds b.  x = 0, p = 0, rtr0, rho_1.
template <int PREC, int N>
__global__ void __launch_bounds__(256)
k_init(const MeshDev m, typename Pol<PREC>::TV *__restrict__ x, typename Pol<PREC>::TV *__restrict__ pv,
       const typename Pol<PREC>::TV *__restrict__ r, const typename Pol<PREC>::TJ *__restrict__ dinv,
       Scal *__restrict__ scal, double *__restrict__ part, double *__restrict__ hist)
{
    using TV = typename Pol<PREC>::TV;
    using TJ = typename Pol<PREC>::TJ;
    using TS = typename Pol<PREC>::TS;
    TS rtr = 0, rho = 0;
    const int64_t npen = m.E * N * N;
    for (int64_t pid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pid < npen;
         pid += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = pid / (N * N);
        const int q = (int)(pid - e * (N * N));
        const int a = q % N, b = q / N;
        const int64_t base = pid * N;
        TV rr[N], zero[N];
        TJ dd[N];
        ld_pencil<TV, N>(r + base, rr);
        ld_pencil<TJ, N>(dinv + base, dd);
        const ElemPos P = elem_pos(m, e);
        const int mjk = axis_mult(a, N, P.ey, m.nely) * axis_mult(b, N, P.ez, m.nelz);
#pragma unroll
        for (int i = 0; i < N; i++) {
            zero[i] = TV(0);
            const TS c = (TS)1 / (TS)(mjk * axis_mult(i, N, P.ex, m.nelx));
            const TS rs = (TS)rr[i];
            rtr += (rs * c) * rs;
            const TV z = (TV)((TJ)rr[i] * dd[i]);
            rho += (rs * c) * (TS)z;
        }
        st_pencil<TV, N>(x + base, zero);
        st_pencil<TV, N>(pv + base, zero);
    }
    __shared__ TS red[32];
    TS s1 = block_sum<TS>(rtr, red);
    TS s2 = block_sum<TS>(rho, red);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = (double)s1;
        part[2 * blockIdx.x + 1] = (double)s2;
    }
    if (last_block(&scal->cnt_init)) {
        TS trtr = block_sum_array<TS>(part, gridDim.x, 2, red);
        TS trho = block_sum_array<TS>(part + 1, gridDim.x, 2, red);
        if (threadIdx.x == 0) {
            scal->rtr0 = (double)trtr;
            scal->rtr = (double)trtr;
            scal->rho = (double)trho;
            scal->beta = 0.0;
            scal->iter = 0;
            hist[0] = 1.0;
            if (trtr == (TS)0) {
                scal->status = NB_CONVERGED;
                scal->done = 1;
                hist[0] = 0.0;
            } else if (!isfinite((double)trtr)) {
                scal->status = NB_BROKEDOWN;
                scal->done = 1;
            } else if (scal->max_iter <= 0) {
                scal->status = NB_MAXITER;
                scal->done = 1;
            }
            scal->cnt_init = 0;
        }
    }
}

// ===========================================================================
// setup kernels
// ===========================================================================
// C-3: deformed vertex position (the CUDA path's own implementation of the reading)
__device__ void vertex_xyz(int ix, int iy, int iz, const MeshDev &m, double amp, double phx, double phy,
                           double phz, double out[3])
{
    const double X = (double)ix / m.nelx, Y = (double)iy / m.nely, Z = (double)iz / m.nelz;
    out[0] = X; out[1] = Y; out[2] = Z;
    if (amp == 0.0) return;
    if (ix == 0 || ix == m.nelx || iy == 0 || iy == m.nely || iz == 0 || iz == m.nelz) return;
    const double pi = 3.14159265358979323846;
    const double bub = sin(pi * X) * sin(pi * Y) * sin(pi * Z);
    out[0] += amp / m.nelx * bub * cos(2.0 * pi * (X + 2.0 * Y + Z) + phx);
    out[1] += amp / m.nely * bub * cos(2.0 * pi * (2.0 * X + Y + Z) + phy);
    out[2] += amp / m.nelz * bub * cos(2.0 * pi * (X + Y + 2.0 * Z) + phz);
}

// node position and trilinear Jacobian d x_a / d r_b at reference point (xi, eta, zeta)
__device__ void trilinear_map(const double V[8][3], double xi, double eta, double zeta, double pos[3],
                              double J[3][3])
{
    const double lx[2] = {0.5 * (1.0 - xi), 0.5 * (1.0 + xi)};
    const double ly[2] = {0.5 * (1.0 - eta), 0.5 * (1.0 + eta)};
    const double lz[2] = {0.5 * (1.0 - zeta), 0.5 * (1.0 + zeta)};
    const double d[2] = {-0.5, 0.5};
    for (int a = 0; a < 3; a++) {
        pos[a] = 0.0;
        J[a][0] = J[a][1] = J[a][2] = 0.0;
    }
    for (int c = 0; c < 8; c++) {
        const int cx = c & 1, cy = (c >> 1) & 1, cz = c >> 2;
        for (int a = 0; a < 3; a++) {
            const double v = V[c][a];
            pos[a] += lx[cx] * ly[cy] * lz[cz] * v;
            J[a][0] += d[cx] * ly[cy] * lz[cz] * v;
            J[a][1] += lx[cx] * d[cy] * lz[cz] * v;
            J[a][2] += lx[cx] * ly[cy] * d[cz] * v;
        }
    }
}

__device__ void element_vertices(const MeshDev &m, const ElemPos &P, double amp, const double *ph, double V[8][3])
{
    for (int c = 0; c < 8; c++)
        vertex_xyz(P.ex + (c & 1), P.ey + ((c >> 1) & 1), P.ez + (c >> 2), m, amp, ph[0], ph[1], ph[2], V[c]);
}

struct Basis {
    double z[16], w[16];
};

__global__ void k_geometry(const MeshDev m, const Basis bs, double amp, double ph0, double ph1, double ph2,
                           double *__restrict__ g, double *__restrict__ B, int32_t *__restrict__ flag)
{
    const int n = m.n;
    const int64_t n3 = (int64_t)n * n * n;
    const double ph[3] = {ph0, ph1, ph2};
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < m.NL; l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = l / n3;
        const int rq = (int)(l - e * n3);
        const int i = rq % n, j = (rq / n) % n, k = rq / (n * n);
        const ElemPos P = elem_pos(m, e);
        double V[8][3], pos[3], J[3][3];
        element_vertices(m, P, amp, ph, V);
        trilinear_map(V, bs.z[i], bs.z[j], bs.z[k], pos, J);
        // cofactor inverse: R = J^-1 (R[a][b] = d r_a / d x_b)
        const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
        const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
        const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
        const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
        if (!(det > 0.0)) atomicOr(flag, 1);
        double R[3][3];
        R[0][0] = c00 / det;
        R[1][0] = c01 / det;
        R[2][0] = c02 / det;
        R[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
        R[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
        R[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
        R[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
        R[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
        R[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
        const double W = bs.w[i] * bs.w[j] * bs.w[k];
        const double WJ = W * det;
        auto G = [&](int a, int b2) { return WJ * (R[a][0] * R[b2][0] + R[a][1] * R[b2][1] + R[a][2] * R[b2][2]); };
        double *ge = g + e * 6 * n3 + rq;
        ge[0 * n3] = G(0, 0);
        ge[1 * n3] = G(0, 1);
        ge[2 * n3] = G(0, 2);
        ge[3 * n3] = G(1, 1);
        ge[4 * n3] = G(1, 2);
        ge[5 * n3] = G(2, 2);
        B[l] = WJ;
    }
}

// C-9 closed-form local diagonal of A_L
__global__ void k_diag_local(const MeshDev m, const double *__restrict__ g, double *__restrict__ diag)
{
    const int n = m.n;
    const int64_t n3 = (int64_t)n * n * n;
    const double *D = c_D64 + n * 256;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < m.NL; l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = l / n3;
        const int rq = (int)(l - e * n3);
        const int i = rq % n, j = (rq / n) % n, k = rq / (n * n);
        const double *ge = g + e * 6 * n3;
        double s = 0.0;
        for (int q = 0; q < n; q++) {
            const double d1 = D[q * n + i], d2 = D[q * n + j], d3 = D[q * n + k];
            s += d1 * d1 * ge[0 * n3 + q + n * j + n * n * k];
            s += d2 * d2 * ge[3 * n3 + i + n * q + n * n * k];
            s += d3 * d3 * ge[5 * n3 + i + n * j + n * n * q];
        }
        const double dii = D[i * n + i], djj = D[j * n + j], dkk = D[k * n + k];
        s += 2.0 * dii * djj * ge[1 * n3 + rq] + 2.0 * dii * dkk * ge[2 * n3 + rq] + 2.0 * djj * dkk * ge[4 * n3 + rq];
        diag[l] = s;
    }
}

__global__ void k_dinv(const MeshDev m, const double *__restrict__ diag, double *__restrict__ dinv,
                       int32_t *__restrict__ flag)
{
    const int n = m.n;
    const int64_t n3 = (int64_t)n * n * n;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < m.NL; l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = l / n3;
        const int rq = (int)(l - e * n3);
        const int i = rq % n, j = (rq / n) % n, k = rq / (n * n);
        const ElemPos P = elem_pos(m, e);
        const bool msk = axis_bnd(i, n, P.ex, m.nelx) || axis_bnd(j, n, P.ey, m.nely) || axis_bnd(k, n, P.ez, m.nelz);
        if (msk) {
            dinv[l] = 0.0;
        } else {
            const double d = diag[l];
            if (!(d > 0.0)) atomicOr(flag, 2);
            dinv[l] = 1.0 / d;
        }
    }
}

// GS segments (C-4): global nodes with multiplicity >= 2 in ascending gid; copies ascending l.
__device__ __forceinline__ int lattice_mult(int64_t I, int64_t NX, int p)
{
    return (I % p == 0 && I > 0 && I < NX - 1) ? 2 : 1;
}
__global__ void k_gs_count(const MeshDev m, int32_t *__restrict__ flag, int32_t *__restrict__ cnt)
{
    for (int64_t gg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gg < m.NG; gg += (int64_t)gridDim.x * blockDim.x) {
        const int64_t I = gg % m.NX;
        const int64_t t = gg / m.NX;
        const int64_t J = t % m.NY, K = t / m.NY;
        const int mu = lattice_mult(I, m.NX, m.p) * lattice_mult(J, m.NY, m.p) * lattice_mult(K, m.NZ, m.p);
        flag[gg] = mu >= 2;
        cnt[gg] = mu >= 2 ? mu : 0;
    }
}
__global__ void k_gs_offsets(const MeshDev m, const int32_t *__restrict__ flag, const int32_t *__restrict__ segid,
                             const int32_t *__restrict__ segoff, int32_t *__restrict__ off, int32_t nseg, int32_t ncopies)
{
    for (int64_t gg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gg < m.NG; gg += (int64_t)gridDim.x * blockDim.x)
        if (flag[gg]) off[segid[gg]] = segoff[gg];
    if (blockIdx.x == 0 && threadIdx.x == 0) off[nseg] = ncopies;
}
__global__ void k_gs_fill(const MeshDev m, const int32_t *__restrict__ flag, const int32_t *__restrict__ segoff,
                          int32_t *__restrict__ idx)
{
    const int n = m.n, p = m.p;
    const int64_t n3 = (int64_t)n * n * n;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < m.NL; l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = l / n3;
        const int rq = (int)(l - e * n3);
        const int i = rq % n, j = (rq / n) % n, k = rq / (n * n);
        const ElemPos P = elem_pos(m, e);
        const int64_t I = (int64_t)P.ex * p + i, J = (int64_t)P.ey * p + j, K = (int64_t)P.ez * p + k;
        const int64_t gg = I + m.NX * (J + m.NY * K);
        if (!flag[gg]) continue;
        // copies of gg are ordered by ascending element index = lexicographic (ez, ey, ex)
        const int cx = axis_mult(i, n, P.ex, m.nelx), cy = axis_mult(j, n, P.ey, m.nely);
        const int rx = (cx == 2 && i == 0) ? 1 : 0;
        const int ry = (cy == 2 && j == 0) ? 1 : 0;
        const int rz = (axis_mult(k, n, P.ez, m.nelz) == 2 && k == 0) ? 1 : 0;
        idx[segoff[gg] + rz * cy * cx + ry * cx + rx] = (int32_t)l;
    }
}

__global__ void k_cast(const double *__restrict__ s, float *__restrict__ d, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = (float)s[i];
}

__global__ void k_maps(const MeshDev m, int64_t *__restrict__ gid, uint8_t *__restrict__ mask)
{
    const int n = m.n, p = m.p;
    const int64_t n3 = (int64_t)n * n * n;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < m.NL; l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = l / n3;
        const int rq = (int)(l - e * n3);
        const int i = rq % n, j = (rq / n) % n, k = rq / (n * n);
        const ElemPos P = elem_pos(m, e);
        const int64_t I = (int64_t)P.ex * p + i, J = (int64_t)P.ey * p + j, K = (int64_t)P.ez * p + k;
        if (gid) gid[l] = I + m.NX * (J + m.NY * K);
        if (mask)
            mask[l] = (axis_bnd(i, n, P.ex, m.nelx) || axis_bnd(j, n, P.ey, m.nely) || axis_bnd(k, n, P.ez, m.nelz)) ? 0 : 1;
    }
}

// C-5 right-hand sides, fp64.  kind 0: mask*U(seed,1,gid).  kind 1: B*f (before dssum/mask).
__global__ void k_rhs(const MeshDev m, const Basis bs, double amp, double ph0, double ph1, double ph2, int kind,
                      double noise, uint64_t seed, const double *__restrict__ B, double *__restrict__ out)
{
    const int n = m.n, p = m.p;
    const int64_t n3 = (int64_t)n * n * n;
    const double ph[3] = {ph0, ph1, ph2};
    const double pi = 3.14159265358979323846;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < m.NL; l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = l / n3;
        const int rq = (int)(l - e * n3);
        const int i = rq % n, j = (rq / n) % n, k = rq / (n * n);
        const ElemPos P = elem_pos(m, e);
        const int64_t I = (int64_t)P.ex * p + i, J = (int64_t)P.ey * p + j, K = (int64_t)P.ez * p + k;
        const uint64_t gid = (uint64_t)(I + m.NX * (J + m.NY * K));
        if (kind == NB_RHS_UNIFORM) {
            const bool msk = axis_bnd(i, n, P.ex, m.nelx) || axis_bnd(j, n, P.ey, m.nely) || axis_bnd(k, n, P.ez, m.nelz);
            out[l] = msk ? 0.0 : unif(seed, 1, gid);
        } else {
            double V[8][3], pos[3], Jm[3][3];
            element_vertices(m, P, amp, ph, V);
            trilinear_map(V, bs.z[i], bs.z[j], bs.z[k], pos, Jm);
            const double f = 3.0 * pi * pi * sin(pi * pos[0]) * sin(pi * pos[1]) * sin(pi * pos[2]) + noise * unif(seed, 2, gid);
            out[l] = B[l] * f;
        }
    }
}

__global__ void k_mask_cast(const MeshDev m, const double *__restrict__ s, void *__restrict__ d, int to_float)
{
    const int n = m.n;
    const int64_t n3 = (int64_t)n * n * n;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < m.NL; l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = l / n3;
        const int rq = (int)(l - e * n3);
        const int i = rq % n, j = (rq / n) % n, k = rq / (n * n);
        const ElemPos P = elem_pos(m, e);
        const bool msk = axis_bnd(i, n, P.ex, m.nelx) || axis_bnd(j, n, P.ey, m.nely) || axis_bnd(k, n, P.ez, m.nelz);
        const double v = msk ? 0.0 : s[l];
        if (to_float) static_cast<float *>(d)[l] = (float)v;
        else static_cast<double *>(d)[l] = v;
    }
}

// ===========================================================================
// launchers
// ===========================================================================
static int grid_for(int64_t work, int threads, int sm_count, int per_sm = 8)
{
    int64_t g = (work + threads - 1) / threads;
    int64_t cap = (int64_t)sm_count * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

template <int PREC, int N, int MODE>
static int ax_grid_t(const nb_handle *h)
{
    using G = AxGeom<typename Pol<PREC>::TV, N>;
    static int occ = -1;
    if (occ < 0) {
        cudaFuncSetAttribute(k_ax<PREC, N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_ax<PREC, N, MODE>, G::NT, G::SMEM);
        occ = o > 0 ? o : 1;
    }
    const int64_t ngroups = (h->E + G::EPB - 1) / G::EPB;
    int64_t grid = (int64_t)h->sm_count * occ;
    if (grid > ngroups) grid = ngroups;
    return (int)(grid < 1 ? 1 : grid);
}

template <int PREC, int N, int MODE>
static cudaError_t ax_launch_t(const nb_handle *h, const void *u_or_r, const void *dinv, void *pv, void *w,
                               int apply_mask, const Scal *scal, double *part, cudaStream_t st)
{
    using TV = typename Pol<PREC>::TV;
    using TJ = typename Pol<PREC>::TJ;
    using G = AxGeom<TV, N>;
    const int grid = ax_grid_t<PREC, N, MODE>(h);
    const TV *g = (const TV *)(sizeof(TV) == 8 ? (const void *)h->g64 : (const void *)h->g32);
    k_ax<PREC, N, MODE><<<grid, G::NT, G::SMEM, st>>>(h->md(), (const TV *)u_or_r, (const TJ *)dinv, (TV *)pv, g,
                                                     (TV *)w, apply_mask, scal, part);
    return cudaGetLastError();
}

#define NB_DISPATCH_N(n, CALL)                 \
    switch (n) {                               \
    case 2: { constexpr int NN = 2; CALL; }    \
    case 3: { constexpr int NN = 3; CALL; }    \
    case 4: { constexpr int NN = 4; CALL; }    \
    case 5: { constexpr int NN = 5; CALL; }    \
    case 6: { constexpr int NN = 6; CALL; }    \
    case 7: { constexpr int NN = 7; CALL; }    \
    case 8: { constexpr int NN = 8; CALL; }    \
    case 9: { constexpr int NN = 9; CALL; }    \
    case 10: { constexpr int NN = 10; CALL; }  \
    case 11: { constexpr int NN = 11; CALL; }  \
    case 12: { constexpr int NN = 12; CALL; }  \
    case 13: { constexpr int NN = 13; CALL; }  \
    case 14: { constexpr int NN = 14; CALL; }  \
    case 15: { constexpr int NN = 15; CALL; }  \
    case 16: { constexpr int NN = 16; CALL; }  \
    default: return cudaErrorInvalidValue;     \
    }

cudaError_t launch_ax(const nb_handle *h, int prec, const void *u, void *w, bool local, cudaStream_t st)
{
    cudaError_t e;
    if (prec == NB_FP64) {
        NB_DISPATCH_N(h->n, e = (ax_launch_t<NB_FP64, NN, 0>(h, u, nullptr, nullptr, w, !local, nullptr, nullptr, st)); break)
    } else {
        NB_DISPATCH_N(h->n, e = (ax_launch_t<NB_FP32, NN, 0>(h, u, nullptr, nullptr, w, !local, nullptr, nullptr, st)); break)
    }
    if (e != cudaSuccess || local) return e;
    return launch_dssum(h, prec, NB_GS_CONSISTENT, w, st);
}

int grid_gs(const nb_handle *h) { return grid_for(h->nseg, 256, h->sm_count, 8); }

template <int PREC, int ORDER, int MODE, typename TVX, typename TGX>
static cudaError_t gs_launch_t(const nb_handle *h, void *u, const void *pv, Scal *scal, double *part, int nblk_ax,
                               cudaGraphConditionalHandle cond, int use_cond, cudaStream_t st)
{
    if (h->nseg == 0 && MODE == 0) return cudaSuccess;
    const int grid = grid_gs(h);
    k_gs<PREC, ORDER, MODE, TVX, TGX><<<grid, 256, 0, st>>>((int32_t)h->nseg, h->gs_off, h->gs_idx, (TVX *)u,
                                                            (const TVX *)pv, scal, part, nblk_ax, cond, use_cond);
    return cudaGetLastError();
}

cudaError_t launch_dssum(const nb_handle *h, int prec, int order, void *u, cudaStream_t st)
{
    cudaGraphConditionalHandle c = 0;
    if (prec == NB_FP64) {
        return order == NB_GS_CONSISTENT
                   ? gs_launch_t<NB_FP64, NB_GS_CONSISTENT, 0, double, double>(h, u, nullptr, nullptr, nullptr, 0, c, 0, st)
                   : gs_launch_t<NB_FP64, NB_GS_PER_COPY, 0, double, double>(h, u, nullptr, nullptr, nullptr, 0, c, 0, st);
    } else if (prec == NB_FP32) {
        return order == NB_GS_CONSISTENT
                   ? gs_launch_t<NB_FP32, NB_GS_CONSISTENT, 0, float, float>(h, u, nullptr, nullptr, nullptr, 0, c, 0, st)
                   : gs_launch_t<NB_FP32, NB_GS_PER_COPY, 0, float, float>(h, u, nullptr, nullptr, nullptr, 0, c, 0, st);
    }
    return order == NB_GS_CONSISTENT
               ? gs_launch_t<NB_MIXED, NB_GS_CONSISTENT, 0, float, double>(h, u, nullptr, nullptr, nullptr, 0, c, 0, st)
               : gs_launch_t<NB_MIXED, NB_GS_PER_COPY, 0, float, double>(h, u, nullptr, nullptr, nullptr, 0, c, 0, st);
}

// ---- CG pieces ----
int grid_ax(const nb_handle *h, int prec)
{
    if (prec == NB_FP64) { NB_DISPATCH_N(h->n, return (ax_grid_t<NB_FP64, NN, 1>(h))) }
    if (prec == NB_FP32) { NB_DISPATCH_N(h->n, return (ax_grid_t<NB_FP32, NN, 1>(h))) }
    NB_DISPATCH_N(h->n, return (ax_grid_t<NB_MIXED, NN, 1>(h)))
}
int grid_upd(const nb_handle *h, int prec)
{
    (void)prec;
    return grid_for(h->E * h->n * h->n, 256, h->sm_count, 8);
}

cudaError_t launch_cg_init(const nb_handle *h, int prec, Workspace &ws, const void *b, cudaStream_t st)
{
    (void)b;
    const int grid = grid_upd(h, prec);
#define NB_INIT(P) NB_DISPATCH_N(h->n, (k_init<P, NN><<<grid, 256, 0, st>>>(h->md(), (Pol<P>::TV *)ws.x, (Pol<P>::TV *)ws.p, \
        (const Pol<P>::TV *)ws.r, (const Pol<P>::TJ *)(P == NB_FP32 ? (const void *)h->dinv32 : (const void *)h->dinv64),     \
        ws.scal, ws.part, ws.hist)); break)
    if (prec == NB_FP64) { NB_INIT(NB_FP64) }
    else if (prec == NB_FP32) { NB_INIT(NB_FP32) }
    else { NB_INIT(NB_MIXED) }
#undef NB_INIT
    return cudaGetLastError();
}

cudaError_t launch_cg_ax(const nb_handle *h, int prec, Workspace &ws, cudaStream_t st)
{
    cudaError_t e;
    if (prec == NB_FP64) {
        NB_DISPATCH_N(h->n, e = (ax_launch_t<NB_FP64, NN, 1>(h, ws.r, h->dinv64, ws.p, ws.w, 1, ws.scal, ws.part, st)); break)
    } else if (prec == NB_FP32) {
        NB_DISPATCH_N(h->n, e = (ax_launch_t<NB_FP32, NN, 1>(h, ws.r, h->dinv32, ws.p, ws.w, 1, ws.scal, ws.part, st)); break)
    } else {
        NB_DISPATCH_N(h->n, e = (ax_launch_t<NB_MIXED, NN, 1>(h, ws.r, h->dinv64, ws.p, ws.w, 1, ws.scal, ws.part, st)); break)
    }
    return e;
}

cudaError_t launch_cg_gs(const nb_handle *h, int prec, int order, Workspace &ws, cudaStream_t st,
                         cudaGraphConditionalHandle cond, bool use_cond)
{
    const int nax = grid_ax(h, prec);
    const int uc = use_cond ? 1 : 0;
    if (prec == NB_FP64)
        return order == NB_GS_CONSISTENT
                   ? gs_launch_t<NB_FP64, NB_GS_CONSISTENT, 1, double, double>(h, ws.w, ws.p, ws.scal, ws.part, nax, cond, uc, st)
                   : gs_launch_t<NB_FP64, NB_GS_PER_COPY, 1, double, double>(h, ws.w, ws.p, ws.scal, ws.part, nax, cond, uc, st);
    if (prec == NB_FP32)
        return order == NB_GS_CONSISTENT
                   ? gs_launch_t<NB_FP32, NB_GS_CONSISTENT, 1, float, float>(h, ws.w, ws.p, ws.scal, ws.part, nax, cond, uc, st)
                   : gs_launch_t<NB_FP32, NB_GS_PER_COPY, 1, float, float>(h, ws.w, ws.p, ws.scal, ws.part, nax, cond, uc, st);
    return order == NB_GS_CONSISTENT
               ? gs_launch_t<NB_MIXED, NB_GS_CONSISTENT, 1, float, double>(h, ws.w, ws.p, ws.scal, ws.part, nax, cond, uc, st)
               : gs_launch_t<NB_MIXED, NB_GS_PER_COPY, 1, float, double>(h, ws.w, ws.p, ws.scal, ws.part, nax, cond, uc, st);
}

cudaError_t launch_cg_upd(const nb_handle *h, int prec, Workspace &ws, cudaStream_t st,
                          cudaGraphConditionalHandle cond, bool use_cond)
{
    const int grid = grid_upd(h, prec);
    const int uc = use_cond ? 1 : 0;
#define NB_UPD(P) NB_DISPATCH_N(h->n, (k_upd<P, NN><<<grid, 256, 0, st>>>(h->md(), (Pol<P>::TV *)ws.x, (const Pol<P>::TV *)ws.p, \
        (Pol<P>::TV *)ws.r, (const Pol<P>::TV *)ws.w,                                                                       \
        (const Pol<P>::TJ *)(P == NB_FP32 ? (const void *)h->dinv32 : (const void *)h->dinv64), ws.scal, ws.part, ws.hist,   \
        cond, uc)); break)
    if (prec == NB_FP64) { NB_UPD(NB_FP64) }
    else if (prec == NB_FP32) { NB_UPD(NB_FP32) }
    else { NB_UPD(NB_MIXED) }
#undef NB_UPD
    return cudaGetLastError();
}

// ---- setup launchers ----
static Basis make_basis(const nb_handle *h)
{
    Basis b;
    for (int i = 0; i < 16; i++) {
        b.z[i] = i < h->n ? h->nodes[i] : 0.0;
        b.w[i] = i < h->n ? h->weights[i] : 0.0;
    }
    return b;
}

cudaError_t launch_geometry(const nb_handle *h, const double phi[3], cudaStream_t st)
{
    const int grid = grid_for(h->NL, 256, h->sm_count, 16);
    k_geometry<<<grid, 256, 0, st>>>(h->md(), make_basis(h), h->deform, phi[0], phi[1], phi[2], h->g64, h->B, h->flag);
    return cudaGetLastError();
}

cudaError_t launch_jacobi(nb_handle *h, double *diag, cudaStream_t st)
{
    const int grid = grid_for(h->NL, 256, h->sm_count, 16);
    k_diag_local<<<grid, 256, 0, st>>>(h->md(), h->g64, diag);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = launch_dssum(h, NB_FP64, NB_GS_CONSISTENT, diag, st);
    if (e != cudaSuccess) return e;
    k_dinv<<<grid, 256, 0, st>>>(h->md(), diag, h->dinv64, h->flag);
    return cudaGetLastError();
}

cudaError_t build_gs(nb_handle *h, cudaStream_t st)
{
    const MeshDev m = h->md();
    int32_t *flag = nullptr, *cnt = nullptr, *segid = nullptr, *segoff = nullptr;
    void *tmp = nullptr;
    size_t tb1 = 0, tb2 = 0;
    cudaError_t e;
#define CK(x) do { e = (x); if (e != cudaSuccess) goto done; } while (0)
    CK(cudaMalloc(&flag, sizeof(int32_t) * m.NG));
    CK(cudaMalloc(&cnt, sizeof(int32_t) * m.NG));
    CK(cudaMalloc(&segid, sizeof(int32_t) * m.NG));
    CK(cudaMalloc(&segoff, sizeof(int32_t) * m.NG));
    {
        const int grid = grid_for(m.NG, 256, h->sm_count, 16);
        k_gs_count<<<grid, 256, 0, st>>>(m, flag, cnt);
        CK(cudaGetLastError());
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tb1, flag, segid, (int)m.NG, st));
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnt, segoff, (int)m.NG, st));
        CK(cudaMalloc(&tmp, tb1 > tb2 ? tb1 : tb2));
        CK(cub::DeviceScan::ExclusiveSum(tmp, tb1, flag, segid, (int)m.NG, st));
        CK(cub::DeviceScan::ExclusiveSum(tmp, tb2, cnt, segoff, (int)m.NG, st));
        int32_t last[4];
        CK(cudaMemcpyAsync(&last[0], segid + m.NG - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&last[1], flag + m.NG - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&last[2], segoff + m.NG - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&last[3], cnt + m.NG - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        h->nseg = (int64_t)last[0] + last[1];
        h->ncopies = (int64_t)last[2] + last[3];
        CK(cudaMalloc(&h->gs_off, sizeof(int32_t) * (h->nseg + 1)));
        CK(cudaMalloc(&h->gs_idx, sizeof(int32_t) * (h->ncopies > 0 ? h->ncopies : 1)));
        k_gs_offsets<<<grid, 256, 0, st>>>(m, flag, segid, segoff, h->gs_off, (int32_t)h->nseg, (int32_t)h->ncopies);
        CK(cudaGetLastError());
        const int gl = grid_for(m.NL, 256, h->sm_count, 16);
        k_gs_fill<<<gl, 256, 0, st>>>(m, flag, segoff, h->gs_idx);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
    }
#undef CK
done:
    cudaFree(flag); cudaFree(cnt); cudaFree(segid); cudaFree(segoff); cudaFree(tmp);
    return e;
}

cudaError_t launch_cast(const double *src, float *dst, int64_t n, cudaStream_t st)
{
    k_cast<<<1184, 256, 0, st>>>(src, dst, n);
    return cudaGetLastError();
}

cudaError_t launch_maps(const nb_handle *h, int64_t *gid, uint8_t *mask, cudaStream_t st)
{
    const int grid = grid_for(h->NL, 256, h->sm_count, 16);
    k_maps<<<grid, 256, 0, st>>>(h->md(), gid, mask);
    return cudaGetLastError();
}

cudaError_t launch_rhs(const nb_handle *h, int kind, double noise, uint64_t seed, int prec, void *b, cudaStream_t st)
{
    const int grid = grid_for(h->NL, 256, h->sm_count, 16);
    double *tmp = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&tmp, sizeof(double) * h->NL, st);
    if (e != cudaSuccess) return e;
    double ph[3];
    deform_phases(h->seed, ph);
    k_rhs<<<grid, 256, 0, st>>>(h->md(), make_basis(h), h->deform, ph[0], ph[1], ph[2], kind, noise, seed, h->B, tmp);
    e = cudaGetLastError();
    if (e == cudaSuccess && kind == NB_RHS_MANUFACTURED) e = launch_dssum(h, NB_FP64, NB_GS_CONSISTENT, tmp, st);
    if (e == cudaSuccess) {
        k_mask_cast<<<grid, 256, 0, st>>>(h->md(), tmp, b, prec == NB_FP64 ? 0 : 1);
        e = cudaGetLastError();
    }
    cudaError_t e2 = cudaFreeAsync(tmp, st);
    return e != cudaSuccess ? e : e2;
}

}  // namespace nb
