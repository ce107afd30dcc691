// nb_setup_k.cu -- setup kernels (readings C-2..C-9): geometry,
// Jacobi diagonal, gather-scatter segments, right-hand sides, casts, map export.
// Setup time is not part of the metric (Nekbone's own init is kept in fp64).
#include <cub/device/device_scan.cuh>

#include "nb_common.cuh"

namespace nb {

struct DFull {
    double d[256];   // D[i*n + j]
};

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
        const ElemPos P = elem_pos(m, (int32_t)e);
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
__global__ void k_diag_local(const MeshDev m, const __grid_constant__ DFull Dm, const double *__restrict__ g,
                             double *__restrict__ diag)
{
    const int n = m.n;
    const int64_t n3 = (int64_t)n * n * n;
    const double *D = Dm.d;
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
        const ElemPos P = elem_pos(m, (int32_t)e);
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
// Built over the handle's own node lattice (a slab's nodes, multiplicity among its own copies).
__device__ __forceinline__ int lattice_mult(int64_t I, int64_t NX, int p)
{
    return (I % p == 0 && I > 0 && I < NX - 1) ? 2 : 1;
}
__global__ void k_gs_count(const MeshDev m, int32_t *__restrict__ flag, int32_t *__restrict__ cnt)
{
    for (int64_t gg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gg < m.NGl; gg += (int64_t)gridDim.x * blockDim.x) {
        const int64_t I = gg % m.NX;
        const int64_t t = gg / m.NX;
        const int64_t J = t % m.NY, K = t / m.NY;
        const int mu = lattice_mult(I, m.NX, m.p) * lattice_mult(J, m.NY, m.p) * lattice_mult(K, m.NZl, m.p);
        flag[gg] = mu >= 2;
        cnt[gg] = mu >= 2 ? mu : 0;
    }
}
__global__ void k_gs_offsets(const MeshDev m, const int32_t *__restrict__ flag, const int32_t *__restrict__ segid,
                             const int32_t *__restrict__ segoff, int32_t *__restrict__ off, int32_t nseg, int32_t ncopies)
{
    for (int64_t gg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gg < m.NGl; gg += (int64_t)gridDim.x * blockDim.x)
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
        const ElemPos P = elem_pos(m, (int32_t)e);
        const int zl = P.ez - m.ez0;   // layer within the slab
        const int64_t I = (int64_t)P.ex * p + i, J = (int64_t)P.ey * p + j, K = (int64_t)zl * p + k;
        const int64_t gg = I + m.NX * (J + m.NY * K);
        if (!flag[gg]) continue;
        // copies of gg are ordered by ascending element index = lexicographic (ez, ey, ex)
        const int cx = axis_mult(i, n, P.ex, m.nelx), cy = axis_mult(j, n, P.ey, m.nely);
        const int rx = (cx == 2 && i == 0) ? 1 : 0;
        const int ry = (cy == 2 && j == 0) ? 1 : 0;
        const int rz = (axis_mult(k, n, zl, m.nelzl) == 2 && k == 0) ? 1 : 0;
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
        const ElemPos P = elem_pos(m, (int32_t)e);
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
        const ElemPos P = elem_pos(m, (int32_t)e);
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
        const ElemPos P = elem_pos(m, (int32_t)e);
        const bool msk = axis_bnd(i, n, P.ex, m.nelx) || axis_bnd(j, n, P.ey, m.nely) || axis_bnd(k, n, P.ez, m.nelz);
        const double v = msk ? 0.0 : s[l];
        if (to_float) static_cast<float *>(d)[l] = (float)v;
        else static_cast<double *>(d)[l] = v;
    }
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
    DFull Dm;
    for (int i = 0; i < 256; i++) Dm.d[i] = i < h->n * h->n ? h->D[i] : 0.0;
    k_diag_local<<<grid, 256, 0, st>>>(h->md(), Dm, h->g64, diag);
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
    CK(cudaMalloc(&flag, sizeof(int32_t) * m.NGl));
    CK(cudaMalloc(&cnt, sizeof(int32_t) * m.NGl));
    CK(cudaMalloc(&segid, sizeof(int32_t) * m.NGl));
    CK(cudaMalloc(&segoff, sizeof(int32_t) * m.NGl));
    {
        const int grid = grid_for(m.NGl, 256, h->sm_count, 16);
        k_gs_count<<<grid, 256, 0, st>>>(m, flag, cnt);
        CK(cudaGetLastError());
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tb1, flag, segid, (int)m.NGl, st));
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnt, segoff, (int)m.NGl, st));
        CK(cudaMalloc(&tmp, tb1 > tb2 ? tb1 : tb2));
        CK(cub::DeviceScan::ExclusiveSum(tmp, tb1, flag, segid, (int)m.NGl, st));
        CK(cub::DeviceScan::ExclusiveSum(tmp, tb2, cnt, segoff, (int)m.NGl, st));
        int32_t last[4];
        CK(cudaMemcpyAsync(&last[0], segid + m.NGl - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&last[1], flag + m.NGl - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&last[2], segoff + m.NGl - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&last[3], cnt + m.NGl - 1, 4, cudaMemcpyDeviceToHost, st));
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
