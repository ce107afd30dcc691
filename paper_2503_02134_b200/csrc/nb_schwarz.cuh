// nb_schwarz.cuh -- the two-level overlapping Schwarz preconditioner z = M^-1 r (SURVEY.md §8(f)
// NEXT-4; reading 28), as grid-wide phases of a persistent cooperative kernel:
//
//   M^-1 r = sum_e R_e^T W K_e^-1 W R_e r  +  Phi A0^-1 Phi^T r
//
//   S1 (sw_local, one element per block step): gather r on the element box extended by one GLL
//      layer (the neighbours' copies, diagonal neighbours included), the coarse restriction
//      partials of the element's 8 corners (Phi^T r), weights W = 1/sqrt(overlap count) -- the
//      square roots of Nekbone's h1mg_schwarz_wt, in the gather-scatter precision
//      TG: fp64 under NB_FP64 / NB_MIXED ("sqrt in fp64"), binary32 otherwise
//      -- and the fast-diagonalisation solve (S_z S_y S_x) Lambda^-1 (S_z S_y S_x)^T in the vector
//      precision TV: six 1-D contractions, one line of P3 values per thread through shared memory.
//   C0..C6 (sw_coarse): the coarse vertex RHS assembled from the corner partials, then the six
//      1-D passes of the coarse fast diagonalisation, one output per thread over the whole grid.
//   S2 (sw_gather_pencil, one r-pencil per thread): z at every copy = the sum, in ascending
//      element order, of the weighted local solutions of the (up to 8) extended boxes holding
//      the node, accumulated in TG (the preconditioner's gather-scatter: fp64 under NB_MIXED),
//      plus the trilinear interpolation of the coarse solution; glsc3(r, c, z) partial.
// Grid barriers separate the phases (the caller passes the barrier counter and target).
#pragma once
#include "nb_common.cuh"
#include "nb_gs.cuh"   // elem_rank

namespace nb {

#ifndef NB_SW_EB
#define NB_SW_EB 0   // 0: the measured choice per data size and order (SwCfg::EBW)
#endif
template <typename TV, int N> struct SwCfg {
    static constexpr int P3 = N + 2, P2 = P3 * P3, PV = P2 * P3;
    // one slot: F, T [PV] (TV); S_x, S_y, S_z and their transposes [P2] (TV); lambda_x,y,z [P3] (double);
    static constexpr int OFF_S = 2 * PV * (int)sizeof(TV);
    static constexpr int OFF_L = ((OFF_S + 6 * P2 * (int)sizeof(TV)) + 15) / 16 * 16;
    // D [PV] (TV): 1/(lambda_x + lambda_y + lambda_z) per box point, rebuilt with the tables
    static constexpr int OFF_D = ((OFF_L + 3 * P3 * 8) + 15) / 16 * 16;
    static constexpr int SLOT = ((OFF_D + PV * (int)sizeof(TV)) + 15) / 16 * 16;
    // elements per S1 step (slots), while the slots fit in 110 KB, else 1.  Measured (solveM alone,
    // 32^3, profiles/r2_ab_schwarz_eb.txt): 2 for p = 7 and fp64; single precision p = 9: 3
    // (1077 -> 1035 us), p = 11: 1 (1950 -> 1761 us)
    static constexpr int EBW = NB_SW_EB ? NB_SW_EB
                             : (sizeof(TV) == 4 && N == 10) ? 3 : (sizeof(TV) == 4 && N == 12) ? 1 : 2;
    static constexpr int EB = (EBW * SLOT <= 110 * 1024) ? (EBW > 3 ? 3 : EBW) : 1;   // <= 3 named barriers
    static constexpr int SMEM = EB * SLOT;
};

// W = 1/sqrt(count) in the gather-scatter precision (count 0: not an unknown)
template <typename TG>
__device__ __forceinline__ TG sw_weight(int c)
{
    if (c == 0) return TG(0);
    if constexpr (sizeof(TG) == 8) return 1.0 / sqrt((double)c);
    else return 1.0f / sqrtf((float)c);
}

// the weights of every possible count (1..27: up to 3 boxes per axis), in a block's shared memory
template <typename TG>
__device__ __forceinline__ void sw_weights_init(TG *wlut)
{
    if (threadIdx.x < 28) wlut[threadIdx.x] = sw_weight<TG>((int)threadIdx.x);
    __syncthreads();
}

// one 1-D pass over the P3^3 box of one slot (its tps threads, lt = thread in the slot): axis 0
// (x), 1 (y), 2 (z), one line per thread:
// o[i] = sum_l M[l*P3 + i] in_l with M = S (S^T applied) or M = S^T (S applied), both stored
// row-major in the slot's shared memory so a row of M is contiguous: single precision pairs the
// outputs in packed FMAs (FFMA2) fed by 8-byte shared loads.  l outermost (unrolled by 2): one row
// of M live at a time (all P3^2 coefficients hoisted into registers would spill at the
// megakernel's register cap).  SCALE: multiply output (ti,tj,tk) by 1/(lx[ti] + ly[tj] + lz[tk])
// (the slot's table at SwCfg::OFF_D, computed in double and rounded once to TV when the slot's
// 1-D tables change).  Byte offsets within a slot: IN, OUT (OUT < 0: the global zext of the
// slot's element), M.
template <typename TV, int N, int AXIS, bool SCALE>
__device__ __forceinline__ void sw_pass(unsigned char *slot, int lt, int tps, int in_off, int out_off, int m_off,
                                        TV *__restrict__ zext, int e)
{
    using C = SwCfg<TV, N>;
    constexpr int P3 = C::P3, P2 = C::P2;
    constexpr bool PAIR = sizeof(TV) == 4 && P3 % 2 == 0 && NB_FFMA2;
    const TV *in = reinterpret_cast<const TV *>(slot + in_off);
    const TV *M = reinterpret_cast<const TV *>(slot + m_off);
    const TV *dl = reinterpret_cast<const TV *>(slot + C::OFF_D);
    TV *out = out_off >= 0 ? reinterpret_cast<TV *>(slot + out_off) : zext + (size_t)e * C::PV;
    for (int line = lt; line < P2; line += tps) {
        const int u = line % P3, w = line / P3;
        // base index and stride of the line along AXIS
        const int base = AXIS == 0 ? P3 * line : AXIS == 1 ? u + P2 * w : line;
        constexpr int st = AXIS == 0 ? 1 : AXIS == 1 ? P3 : P2;
        TV o[P3];
        if constexpr (PAIR) {
            unsigned long long acc[P3 / 2];
#pragma unroll
            for (int i = 0; i < P3 / 2; i++) acc[i] = 0ull;
#pragma unroll 2
            for (int l = 0; l < P3; l++) {
                const float vl = (float)in[base + st * l];
                const unsigned long long vv = pack2(vl, vl);
                unsigned long long row[P3 / 2];
                if constexpr (P3 % 4 == 0) {   // 16-byte shared loads of the M row (rows are 16-byte aligned)
                    const ulonglong2 *r2 = reinterpret_cast<const ulonglong2 *>(M + l * P3);
#pragma unroll
                    for (int i = 0; i < P3 / 4; i++) { const ulonglong2 t = r2[i]; row[2 * i] = t.x; row[2 * i + 1] = t.y; }
                } else {
                    const unsigned long long *r1 = reinterpret_cast<const unsigned long long *>(M + l * P3);
#pragma unroll
                    for (int i = 0; i < P3 / 2; i++) row[i] = r1[i];
                }
#pragma unroll
                for (int i = 0; i < P3 / 2; i++) acc[i] = ffma2(row[i], vv, acc[i]);
            }
#pragma unroll
            for (int i = 0; i < P3 / 2; i++) { o[2 * i] = (TV)lo2(acc[i]); o[2 * i + 1] = (TV)hi2(acc[i]); }
        } else {
#pragma unroll
            for (int i = 0; i < P3; i++) o[i] = TV(0);
#pragma unroll 2
            for (int l = 0; l < P3; l++) {
                const TV vl = in[base + st * l];
                if constexpr (sizeof(TV) == 8 && P3 % 2 == 0) {   // 16-byte shared loads of the M row
                    const double2 *r2 = reinterpret_cast<const double2 *>(M + l * P3);
#pragma unroll
                    for (int i = 0; i < P3 / 2; i++) {
                        const double2 t = r2[i];
                        o[2 * i] = fma((TV)t.x, vl, o[2 * i]);
                        o[2 * i + 1] = fma((TV)t.y, vl, o[2 * i + 1]);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < P3; i++) o[i] = fma(M[l * P3 + i], vl, o[i]);
                }
            }
        }
#pragma unroll
        for (int l = 0; l < P3; l++) {
            TV val = o[l];
            if (SCALE) val = val * dl[base + st * l];   // AXIS == 2: point (u, w, l)
            out[base + st * l] = val;
        }
    }
}

// barrier of the tps threads of slot sl (named barrier 1 + sl, immediate ids so that ptxas
// reserves only barriers 0..3 -- a register id reserves all 16 and can cost residency)
__device__ __forceinline__ void slot_sync(int sl, int tps)
{
    if (sl == 0) asm volatile("bar.sync 1, %0;" ::"r"(tps) : "memory");
    else if (sl == 1) asm volatile("bar.sync 2, %0;" ::"r"(tps) : "memory");
    else asm volatile("bar.sync 3, %0;" ::"r"(tps) : "memory");
}

// S1 for one element e on slot sl (the slot's tps = SwCfg::TPS threads, warp-aligned, lt = thread
// in the slot; the slots of a block proceed independently, synchronised by named barriers):
// writes S.zext[e] and S.cpart[e].  cur: the cases of the tables the slot holds (kept across
// elements when they match).  red: the slot's 8 x (tps/32) partials.
template <int PREC, int N>
__device__ __forceinline__ void sw_local(const MeshDev &m, const SwArgs &S, const typename Pol<PREC>::TV *__restrict__ r,
                                         int e, int sl, int lt, int tps, unsigned char *slot,
                                         typename Pol<PREC>::TG *red, int (&cur)[3],
                                         const typename Pol<PREC>::TG *__restrict__ wlut)
{
    using TV = typename Pol<PREC>::TV;
    using TG = typename Pol<PREC>::TG;
    using C = SwCfg<TV, N>;
    constexpr int P3 = C::P3, P2 = C::P2, N3 = N * N * N;
    const ElemPos P = elem_pos<false>(m, e);
    // the element's 1-D tables: S_a at [a], S_a^T at [3 + a]; 1/(lx + ly + lz) per point
    {
        const int pos[3] = {P.ex, P.ey, P.ez};
        const int cs0 = S.cs[0][P.ex], cs1 = S.cs[1][P.ey], cs2 = S.cs[2][P.ez];
        if (cs0 != cur[0] || cs1 != cur[1] || cs2 != cur[2]) {
            TV *Sm = reinterpret_cast<TV *>(slot + C::OFF_S);
            double *lm = reinterpret_cast<double *>(slot + C::OFF_L);
            for (int q = lt; q < 3 * P2; q += tps) {
                const int a = q / P2, k = q - a * P2;
                const TV v = ((const TV *)S.S[a])[(size_t)S.cs[a][pos[a]] * P2 + k];
                Sm[q] = v;
                Sm[(3 + a) * P2 + (k % P3) * P3 + k / P3] = v;
            }
            for (int q = lt; q < 3 * P3; q += tps) {
                const int a = q / P3, k = q - a * P3;
                lm[q] = S.lam[a][(size_t)S.cs[a][pos[a]] * P3 + k];
            }
            slot_sync(sl, tps);
            TV *dl = reinterpret_cast<TV *>(slot + C::OFF_D);
            for (int q = lt; q < C::PV; q += tps) {   // in double, rounded once to TV
                const int ti = q % P3, tj = (q / P3) % P3, tk = q / P2;
                dl[q] = (TV)(1.0 / (lm[ti] + lm[P3 + tj] + lm[2 * P3 + tk]));
            }
            cur[0] = cs0; cur[1] = cs1; cur[2] = cs2;
        }
    }
    // R_e r, its coarse restriction partials and W R_e r, one x-line (tj, tk) of the extended box
    // per thread: the line is a row of the (y, z)-neighbour element's copy (N contiguous values)
    // plus one value from each x-neighbour of that element
    TG cp[8];
#pragma unroll
    for (int c = 0; c < 8; c++) cp[c] = TG(0);
    const bool coarse = S.nv[0] > 0 && S.nv[1] > 0 && S.nv[2] > 0;
    {
        const uint8_t *cx = S.cnt[0] + (size_t)P.ex * P3, *cy = S.cnt[1] + (size_t)P.ey * P3, *cz = S.cnt[2] + (size_t)P.ez * P3;
        TV *F = reinterpret_cast<TV *>(slot);
        for (int line = lt; line < P2; line += tps) {
            const int tj = line % P3, tk = line / P3;
            const int cyz = cy[tj] * cz[tk];
            TV v[P3];
#pragma unroll
            for (int t = 0; t < P3; t++) v[t] = TV(0);
            if (cyz) {
                const int dy = tj == 0 ? -1 : (tj == P3 - 1 ? 1 : 0);
                const int dz = tk == 0 ? -1 : (tk == P3 - 1 ? 1 : 0);
                const int lj = tj == 0 ? N - 2 : (tj == P3 - 1 ? 1 : tj - 1);
                const int lk = tk == 0 ? N - 2 : (tk == P3 - 1 ? 1 : tk - 1);
                const int64_t e2 = (int64_t)e + (int64_t)m.nelx * (dy + (int64_t)m.nely * dz);
                const TV *row = r + e2 * N3 + N * (lj + N * lk);
                TV own[N];
                ld_pencil<TV, N>(row, own);
                v[0] = cx[0] ? row[-N3 + N - 2] : TV(0);
                v[P3 - 1] = cx[P3 - 1] ? row[N3 + 1] : TV(0);
#pragma unroll
                for (int i = 0; i < N; i++) v[i + 1] = cx[i + 1] ? own[i] : TV(0);
                if (coarse && dy == 0 && dz == 0) {   // the element's own copies: c_l phi r per corner
                    const int j = tj - 1, k = tk - 1;
                    const double cjk = 1.0 / (double)(axis_mult(j, N, P.ey, m.nely) * axis_mult(k, N, P.ez, m.nelz));
#pragma unroll
                    for (int i = 0; i < N; i++) {
                        const double cl = cjk / (double)axis_mult(i, N, P.ex, m.nelx);
                        const TG vi = (TG)v[i + 1];
#pragma unroll
                        for (int c = 0; c < 8; c++) {
                            const double ph = ((c & 1) ? S.phR[i] : S.phL[i]) * ((c & 2) ? S.phR[j] : S.phL[j]) *
                                              ((c & 4) ? S.phR[k] : S.phL[k]);
                            cp[c] += (TG)(ph * cl) * vi;
                        }
                    }
                }
#pragma unroll
                for (int t = 0; t < P3; t++) v[t] = (TV)((TG)v[t] * wlut[cx[t] * cyz]);
            }
#pragma unroll
            for (int t = 0; t < P3; t++) F[P3 * line + t] = v[t];
        }
    }
    if (coarse) {   // the slot's sum of the 8 partials over its warps (fixed tree)
        const int lane = lt & 31, wl = lt >> 5, wps = tps >> 5;
#pragma unroll
        for (int c = 0; c < 8; c++)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) cp[c] += __shfl_down_sync(0xffffffffu, cp[c], o);
        if (lane == 0)
#pragma unroll
            for (int c = 0; c < 8; c++) red[wl * 8 + c] = cp[c];
        slot_sync(sl, tps);
        if (lt < 8) {
            TG sacc = TG(0);
            for (int w = 0; w < wps; w++) sacc += red[w * 8 + lt];
            ((TG *)S.cpart)[(size_t)e * 8 + lt] = sacc;
        }
    } else {
        slot_sync(sl, tps);
    }
    // K_e^-1 by fast diagonalisation: S_x^T, S_y^T, S_z^T + Lambda^-1, S_z, S_y, S_x
    constexpr int oF = 0, oT = C::PV * (int)sizeof(TV), oS = C::OFF_S, P2B = P2 * (int)sizeof(TV);
    TV *zx = (TV *)S.zext;
    sw_pass<TV, N, 0, false>(slot, lt, tps, oF, oT, oS, zx, e);
    slot_sync(sl, tps);
    sw_pass<TV, N, 1, false>(slot, lt, tps, oT, oF, oS + P2B, zx, e);
    slot_sync(sl, tps);
    sw_pass<TV, N, 2, true>(slot, lt, tps, oF, oT, oS + 2 * P2B, zx, e);
    slot_sync(sl, tps);
    sw_pass<TV, N, 2, false>(slot, lt, tps, oT, oF, oS + 5 * P2B, zx, e);
    slot_sync(sl, tps);
    sw_pass<TV, N, 1, false>(slot, lt, tps, oF, oT, oS + 4 * P2B, zx, e);
    slot_sync(sl, tps);
    sw_pass<TV, N, 0, false>(slot, lt, tps, oT, -1, oS + 3 * P2B, zx, e);
    slot_sync(sl, tps);   // the slot's smem is reused by its next element
}

// S1 over elements [e0, e1) of the block: slot sl takes e0 + sl, e0 + sl + EB, ... (its threads
// only; threads beyond the slots idle until the caller's block barrier)
template <int PREC, int N>
__device__ __forceinline__ void sw_local_range(const MeshDev &m, const SwArgs &S, const typename Pol<PREC>::TV *__restrict__ r,
                                               int e0, int e1, unsigned char *smraw, typename Pol<PREC>::TG *red,
                                               const typename Pol<PREC>::TG *__restrict__ wlut)
{
    using C = SwCfg<typename Pol<PREC>::TV, N>;
    constexpr int EB = C::EB;
    const int tps = ((int)(blockDim.x >> 5) / EB) * 32;
    const int sl = (int)threadIdx.x / tps, lt = (int)threadIdx.x - sl * tps;
    if (sl >= EB) return;
    int cur[3] = {-1, -1, -1};
    for (int e = e0 + sl; e < e1; e += EB)
        sw_local<PREC, N>(m, S, r, e, sl, lt, tps, smraw + sl * C::SLOT, red + sl * 8 * (tps >> 5), cur, wlut);
}

// coarse pass `pass` (0: assemble b0; 1..6: the fast-diagonalisation passes), thread gt of gn
template <int PREC>
__device__ __forceinline__ void sw_coarse(const MeshDev &m, const SwArgs &S, int pass, int64_t gt, int64_t gn)
{
    using TV = typename Pol<PREC>::TV;
    using TG = typename Pol<PREC>::TG;
    const int nx = S.nv[0], ny = S.nv[1], nz = S.nv[2];
    const int64_t V = (int64_t)nx * ny * nz;
    TV *c0 = (TV *)S.c0, *c1 = (TV *)S.c1;
    for (int64_t v = gt; v < V; v += gn) {
        const int vx = (int)(v % nx), vy = (int)((v / nx) % ny), vz = (int)(v / ((int64_t)nx * ny));
        if (pass == 0) {
            // vertex (vx+1, vy+1, vz+1): corners of the elements around it, ascending element order
            TG s = TG(0);
            for (int dz = 0; dz < 2; dz++)
                for (int dy = 0; dy < 2; dy++)
                    for (int dx = 0; dx < 2; dx++) {
                        const int ex = vx + dx, ey = vy + dy, ez = vz + dz;   // element; its corner (1-dx, 1-dy, 1-dz)
                        const int64_t e = ex + (int64_t)m.nelx * (ey + (int64_t)m.nely * ez);
                        const int c = (1 - dx) + 2 * (1 - dy) + 4 * (1 - dz);
                        s += __ldcg((const TG *)S.cpart + e * 8 + c);
                    }
            c0[v] = (TV)s;
            continue;
        }
        // 1: Sx^T c0 -> c1; 2: Sy^T c1 -> c0; 3: Sz^T c0 * dl -> c1; 4: Sz c1 -> c0; 5: Sy c0 -> c1; 6: Sx c1 -> c0
        const int ax = (pass == 1 || pass == 6) ? 0 : (pass == 2 || pass == 5) ? 1 : 2;
        const bool tr = pass >= 4;
        const TV *in = (pass & 1) ? c0 : c1;
        TV *out = (pass & 1) ? c1 : c0;
        const int n = S.nv[ax], idx = ax == 0 ? vx : ax == 1 ? vy : vz;
        const int64_t st = ax == 0 ? 1 : ax == 1 ? nx : (int64_t)nx * ny;
        const int64_t base = v - (int64_t)idx * st;
        const TV *M = (const TV *)S.S0[ax];
        TV s = TV(0);
        for (int l = 0; l < n; l++) s = fma(tr ? M[idx * n + l] : M[l * n + idx], __ldcg(in + base + st * l), s);
        if (pass == 3) s = s * (TV)(1.0 / (S.lam0[0][vx] + S.lam0[1][vy] + S.lam0[2][vz]));
        out[v] = s;
    }
}

// S2: z on the r-pencil (a, b) of element e = W (sum of the local solutions holding each node,
// ascending element order, in TG) + the coarse interpolation; glsc3(r, c, z) partial.
// Per candidate box row (iy, iz): the element's own box row (P3 contiguous values, 16-byte
// loads) and, for the pencil's end nodes, the x-neighbours' boxes; the element's interior corner
// values of the coarse solution are loaded once per pencil.
template <int PREC, int N>
__device__ __forceinline__ void sw_gather_pencil(const MeshDev &m, const SwArgs &S, const typename Pol<PREC>::TV *__restrict__ r,
                                                 typename Pol<PREC>::TV *__restrict__ z, int64_t pid, Acc<PREC> &rho,
                                                 const typename Pol<PREC>::TG *__restrict__ wlut)
{
    using TV = typename Pol<PREC>::TV;
    using TG = typename Pol<PREC>::TG;
    using TS = typename Pol<PREC>::TS;
    constexpr int N2 = N * N, P3 = N + 2, P2 = P3 * P3, PV = P2 * P3;
    constexpr int VR = (P3 * sizeof(TV)) % 16 == 0 ? 16 / (int)sizeof(TV) : 1;   // row load width
    const int e = (int)(pid / N2);
    const int q = (int)(pid - (int64_t)e * N2);
    const int a = q % N, b = q / N;
    const ElemPos P = elem_pos<false>(m, e);
    const TV *zx = (const TV *)S.zext;
    const bool coarse = S.nv[0] > 0 && S.nv[1] > 0 && S.nv[2] > 0;
    // candidate boxes along y and z (element offset d, index t in that element's box): the node at
    // local a lies at box index a + 1 of its own element, a + N of the lower neighbour's (a <= 1)
    // and a - N + 2 of the upper neighbour's (a >= N - 2); three boxes for p <= 2
    int ny_ = 0, nz_ = 0, dy[3], ty[3], dz[3], tz[3];
    if (a <= 1 && P.ey > 0) { dy[ny_] = -1; ty[ny_++] = a + N; }
    dy[ny_] = 0; ty[ny_++] = a + 1;
    if (a >= N - 2 && P.ey < m.nely - 1) { dy[ny_] = 1; ty[ny_++] = a - N + 2; }
    if (b <= 1 && P.ez > 0) { dz[nz_] = -1; tz[nz_++] = b + N; }
    dz[nz_] = 0; tz[nz_++] = b + 1;
    if (b >= N - 2 && P.ez < m.nelz - 1) { dz[nz_] = 1; tz[nz_++] = b - N + 2; }
    const bool xl = P.ex > 0, xr = P.ex < m.nelx - 1;
    const int cyz = S.cnt[1][(size_t)P.ey * P3 + a + 1] * S.cnt[2][(size_t)P.ez * P3 + b + 1];
    // independent loads first: r (for rho) and the element's interior corner values of x0
    TV rr[N];
    const size_t base = (size_t)pid * N;
    ld_pencil<TV, N>(r + base, rr);
    TV xc[8];
#pragma unroll
    for (int c = 0; c < 8; c++) {
        const int vx = P.ex + (c & 1), vy = P.ey + ((c >> 1) & 1), vz = P.ez + (c >> 2);
        const bool in = coarse && vx >= 1 && vx <= S.nv[0] && vy >= 1 && vy <= S.nv[1] && vz >= 1 && vz <= S.nv[2];
        xc[c] = in ? __ldcg((const TV *)S.c0 + (vx - 1) + (int64_t)S.nv[0] * ((vy - 1) + (int64_t)S.nv[1] * (vz - 1))) : TV(0);
    }
    // sum of the local solutions at the node, then the node's weight (constant over its boxes);
    // the next box row is loaded while the current one is summed
    TG acc[N];
#pragma unroll
    for (int i = 0; i < N; i++) acc[i] = TG(0);
    if (cyz) {
        const int nrow = ny_ * nz_;
        TV v[P3], l0, l1, r0, r1;
        auto load_row = [&](int k, TV (&vv)[P3], TV &a0, TV &a1, TV &b0, TV &b1) {
            const int iz = k / ny_, iy = k - iz * ny_;
            const int64_t eyz = (int64_t)e + (int64_t)m.nelx * (dy[iy] + (int64_t)m.nely * dz[iz]);
            const TV *row = zx + eyz * PV + (int64_t)P3 * (ty[iy] + P3 * tz[iz]);
#pragma unroll
            for (int c = 0; c < P3 / VR; c++) {
                if constexpr (VR == 4) {
                    const float4 t = __ldcg(reinterpret_cast<const float4 *>(row) + c);
                    vv[4 * c] = t.x; vv[4 * c + 1] = t.y; vv[4 * c + 2] = t.z; vv[4 * c + 3] = t.w;
                } else if constexpr (VR == 2) {
                    const double2 t = __ldcg(reinterpret_cast<const double2 *>(row) + c);
                    vv[2 * c] = t.x; vv[2 * c + 1] = t.y;
                } else {
                    vv[c] = __ldcg(row + c);
                }
            }
            // x-neighbours' boxes: values at their indices N, N + 1 (nodes 0, 1) and 0, 1 (nodes N - 2, N - 1)
            a0 = xl ? __ldcg(row - PV + N) : TV(0); a1 = xl ? __ldcg(row - PV + N + 1) : TV(0);
            b0 = xr ? __ldcg(row + PV) : TV(0); b1 = xr ? __ldcg(row + PV + 1) : TV(0);
        };
        load_row(0, v, l0, l1, r0, r1);
        for (int k = 0; k < nrow; k++) {
            TV vn[P3], nl0 = TV(0), nl1 = TV(0), nr0 = TV(0), nr1 = TV(0);
            if (k + 1 < nrow) load_row(k + 1, vn, nl0, nl1, nr0, nr1);
#pragma unroll
            for (int i = 0; i < N; i++) {
                if (i <= 1 && xl) acc[i] += (TG)(i == 0 ? l0 : l1);
                acc[i] += (TG)v[i + 1];
                if (i >= N - 2 && xr) acc[i] += (TG)(i == N - 2 ? r0 : r1);
            }
            if (k + 1 < nrow) {
#pragma unroll
                for (int t = 0; t < P3; t++) v[t] = vn[t];
                l0 = nl0; l1 = nl1; r0 = nr0; r1 = nr1;
            }
        }
#pragma unroll
        for (int i = 0; i < N; i++) acc[i] *= wlut[S.cnt[0][(size_t)P.ex * P3 + i + 1] * cyz];
    }
    if (coarse) {   // trilinear interpolation of x0 from the element's interior corner vertices:
        // g[cx] = sum_{cz, cy} hz hy x0(corner) once per pencil, then per node hx0 g[0] + hx1 g[1]
        // (corner values of boundary vertices are 0; the same arithmetic at every copy of a node)
        const TV hy[2] = {(TV)S.phL[a], (TV)S.phR[a]}, hz[2] = {(TV)S.phL[b], (TV)S.phR[b]};
        TV g[2] = {TV(0), TV(0)};
#pragma unroll
        for (int c = 0; c < 8; c++) g[c & 1] = fma(hz[c >> 2] * hy[(c >> 1) & 1], xc[c], g[c & 1]);
#pragma unroll
        for (int i = 0; i < N; i++) {
            if (!(cyz && S.cnt[0][(size_t)P.ex * P3 + i + 1])) continue;   // Dirichlet node
            acc[i] += (TG)fma((TV)S.phL[i], g[0], (TV)S.phR[i] * g[1]);
        }
    }
    TV zz[N];
    const int mjk = axis_mult(a, N, P.ey, m.nely) * axis_mult(b, N, P.ez, m.nelz);
#pragma unroll
    for (int i = 0; i < N; i++) {
        zz[i] = (TV)acc[i];
        const TS c = (TS)1 / (TS)(mjk * axis_mult(i, N, P.ex, m.nelx));
        const TS rs = (TS)rr[i];
        rho.add(rs * c, (TS)zz[i]);
    }
    st_pencil<TV, N>(z + base, zz);
}

// S2 under the per-copy / rank-partitioned gather-scatter orders (NEXT-2 x NEXT-4; the oracle's
// OR_SW_COMBINE): per node, the weighted contributions of the boxes holding it (ascending element
// order, with each box's element and rank) are combined -- per-copy: the pencil's own element's box
// first, then the others; pairwise: rank partials (ascending within a rank), the own rank's first,
// then the other ranks ascending; allreduce: all rank partials ascending.  Then the coarse term.
template <int PREC, int N>
__device__ __forceinline__ void sw_gather_pencil_ordered(const MeshDev &m, const SwArgs &S, int order, const RankPart &rp,
                                                         const typename Pol<PREC>::TV *__restrict__ r,
                                                         typename Pol<PREC>::TV *__restrict__ z, int64_t pid,
                                                         Acc<PREC> &rho, const typename Pol<PREC>::TG *__restrict__ wlut)
{
    using TV = typename Pol<PREC>::TV;
    using TG = typename Pol<PREC>::TG;
    using TS = typename Pol<PREC>::TS;
    constexpr int N2 = N * N, P3 = N + 2, P2 = P3 * P3, PV = P2 * P3;
    const int e = (int)(pid / N2);
    const int q = (int)(pid - (int64_t)e * N2);
    const int a = q % N, b = q / N;
    const ElemPos P = elem_pos<false>(m, e);
    const TV *zx = (const TV *)S.zext;
    const bool coarse = S.nv[0] > 0 && S.nv[1] > 0 && S.nv[2] > 0;
    const int rown = elem_rank(m, rp, e);
    TV xc[8];
#pragma unroll
    for (int c = 0; c < 8; c++) {
        const int vx = P.ex + (c & 1), vy = P.ey + ((c >> 1) & 1), vz = P.ez + (c >> 2);
        const bool in = coarse && vx >= 1 && vx <= S.nv[0] && vy >= 1 && vy <= S.nv[1] && vz >= 1 && vz <= S.nv[2];
        xc[c] = in ? __ldcg((const TV *)S.c0 + (vx - 1) + (int64_t)S.nv[0] * ((vy - 1) + (int64_t)S.nv[1] * (vz - 1))) : TV(0);
    }
    const TV hy[2] = {(TV)S.phL[a], (TV)S.phR[a]}, hz[2] = {(TV)S.phL[b], (TV)S.phR[b]};
    TV g[2] = {TV(0), TV(0)};
#pragma unroll
    for (int c = 0; c < 8; c++) g[c & 1] = fma(hz[c >> 2] * hy[(c >> 1) & 1], xc[c], g[c & 1]);
    const int cyz = S.cnt[1][(size_t)P.ey * P3 + a + 1] * S.cnt[2][(size_t)P.ez * P3 + b + 1];
    TV rr[N], zz[N];
    const size_t base = (size_t)pid * N;
    ld_pencil<TV, N>(r + base, rr);
    const int mjk = axis_mult(a, N, P.ey, m.nely) * axis_mult(b, N, P.ez, m.nelz);
    for (int i = 0; i < N; i++) {
        const int cnt = S.cnt[0][(size_t)P.ex * P3 + i + 1] * cyz;
        TG acc = TG(0);
        if (cnt) {
            const TG w = wlut[cnt];
            TG cv[27];
            int ce[27], cr[27], nc = 0;
            for (int dz = -1; dz <= 1; dz++) {
                const int tz = b + 1 - dz * (N - 1);   // the node's index in that element's box
                if (P.ez + dz < 0 || P.ez + dz >= m.nelz || tz < 0 || tz >= P3) continue;
                for (int dy = -1; dy <= 1; dy++) {
                    const int ty = a + 1 - dy * (N - 1);
                    if (P.ey + dy < 0 || P.ey + dy >= m.nely || ty < 0 || ty >= P3) continue;
                    for (int dx = -1; dx <= 1; dx++) {
                        const int tx = i + 1 - dx * (N - 1);
                        if (P.ex + dx < 0 || P.ex + dx >= m.nelx || tx < 0 || tx >= P3) continue;
                        const int e2 = e + dx + m.nelx * (dy + m.nely * dz);
                        cv[nc] = (TG)__ldcg(zx + (int64_t)e2 * PV + tx + P3 * (ty + P3 * tz)) * w;
                        ce[nc] = e2;
                        cr[nc] = elem_rank(m, rp, e2);
                        nc++;
                    }
                }
            }
            if (order == NB_GS_PER_COPY) {
                for (int k = 0; k < nc; k++)
                    if (ce[k] == e) acc += cv[k];
                for (int k = 0; k < nc; k++)
                    if (ce[k] != e) acc += cv[k];
            } else {
                int own = -1;
                for (int k = 0; k < nc; k++)
                    if (cr[k] == rown) { own = k; break; }
                auto part = [&](int rk) {
                    TG u = TG(0);
                    for (int k2 = 0; k2 < nc; k2++)
                        if (cr[k2] == rk) u += cv[k2];
                    return u;
                };
                if (order == NB_GS_PAIRWISE && own >= 0) acc = part(rown);
                int prev = -1;
                for (;;) {
                    int best = -1;
                    for (int k = 0; k < nc; k++)
                        if (cr[k] > prev && (best < 0 || cr[k] < cr[best])) best = k;
                    if (best < 0) break;
                    prev = cr[best];
                    if (order == NB_GS_PAIRWISE && own >= 0 && cr[best] == rown) continue;
                    acc += part(cr[best]);
                }
            }
            if (coarse) acc += (TG)fma((TV)S.phL[i], g[0], (TV)S.phR[i] * g[1]);
        }
        zz[i] = (TV)acc;
        const TS c = (TS)1 / (TS)(mjk * axis_mult(i, N, P.ex, m.nelx));
        const TS rs = (TS)rr[i];
        rho.add(rs * c, (TS)zz[i]);
    }
    st_pencil<TV, N>(z + base, zz);
}

}  // namespace nb
