// nb_cg.cuh -- the per-iteration work of the Jacobi-PCG hot path (templates; the translation
// units nb_cg_<policy>.cu (default options) and nb_cg_<policy>_var.cu (preconditioner / x_fp64
// variants and the multi-rank kernel) instantiate them per precision policy: fp64, fp32,
// mixed, fp32_dot2).
//
// One CG iteration (Table 2 of the paper) is two phases in consistent
// gather-scatter order:
//
//   A (ax_group):  p = z + beta p               (add2s1, :162; z = M^-1 r stored by phase B)
//                  x += alpha_prev p_old        (add2s2(x,p,alpha) of the previous iteration,
//                                                deferred so x is streamed once, :165)
//                  w = mask . A_L p             (ax -> ax_e: local_grad3, geometric scaling,
//                                                local_grad3_t, add2; :147, :163)
//                  pap = p^T A_L p              (glsc3(w,c,p), :164: for continuous p, zero on
//                                                the Dirichlet nodes, the c-weighted sum over
//                                                the assembled w equals p^T A_L p, taken here
//                                                in its energy form (Dp)^T G (Dp))
//                  alpha = rho / pap
//   B (upd_pencil): w <- QQ^T w on the fly      (gather-scatter "to ensure continuity",
//                                                :309, :404 -- each copy gathers the copies of
//                                                its node in ascending element order, so all
//                                                copies compute the same sum bit for bit)
//                  r -= alpha w                 (add2s2(r,w,-alpha), :166)
//                  z = M^-1 r                   (solveM, Jacobi, :160, :444)
//                  rtr = glsc3(r,c,r), rho = glsc3(r,c,z)   (:167, :161); beta; stop test
//
// Under the per-copy gather-scatter order (the emulation of the paper's pairwise
// exchange) the copies differ, so pap must be taken over the per-copy
// sums: phase A contributes only the unshared nodes, a CSR phase (nb_gs.cuh) does QQ^T and
// the shared part of pap, and phase B runs without the gather.
//
// The driver is ONE persistent cooperative kernel per solve (k_cg_mega).  Every block owns a
// contiguous element range; grid-wide barriers separate the phases; after each barrier every
// block reduces the per-block partials itself, in the same fixed order, so all blocks take the
// same (bit-identical) scalar decisions -- no host round trip, no launch gaps, no serial
// last-block tail.  k_cg_mega_mr is the same body for z-slabs of a box spread over ranks (GPUs,
// or slabs sharing one launch): the gather reads the neighbour slab's w, the reductions add a
// per-rank push/flag step (mr_reduce).  Body: nb_mega_body.inc.  k_ax is the standalone
// operator of nb_ax.
#pragma once
#include "nb_common.cuh"
#include "nb_gs.cuh"
#include "nb_schwarz.cuh"

namespace nb {

// ===========================================================================
// phase A: local operator A_L, register pencils + shared-memory transposes
// ===========================================================================
template <typename T, int N> struct AxCfg {
    static constexpr int N2 = N * N;
    static constexpr int N3 = N * N * N;
    static constexpr int BANKS = (sizeof(T) == 4) ? 32 : 16;
    // plane pitch P >= N^2 with P == N (mod BANKS): the stride-N s-pencil reads and the
    // stride-P t-pencil reads of a warp hit distinct banks.
#ifndef NB_PADR
#define NB_PADR 1
#endif
    // Shared-memory layout of one element array: index(i, j, k) = i + R j + P k.
    // fp32, N = 8: row pitch R = 12 so the 16-byte r-pencil accesses of 8 consecutive threads
    // (48-byte stride) hit 8 distinct 4-bank groups; P = 104 == 8 (mod 32) keeps the s-pencil
    // reads conflict-free; t-pencils are then assigned transposed (thread (a,b) takes (i=b, j=a)),
    // which makes them conflict-free too.  Otherwise R = N and P == N (mod banks).
    // fp64, N = 8: R = 10 (80-byte stride: 5a mod 8 distinct 16-byte bank groups), P = 88 == 8
    // (mod 16) for the half-warp s-pencil reads, t-pencils transposed.
    // fp32 N = 10: R = 14, P = 140; fp64 N = 12: R = 14, P = 172, transposed t-pencils.
    // (bank-conflict model and search: tools/smem_layout.py)
    static constexpr int LAY = !NB_PADR ? 0
                             : (N == 8) ? (sizeof(T) == 4 ? 1 : 2)
                             : (N == 10 && sizeof(T) == 4) ? 3 : (N == 12 && sizeof(T) == 8) ? 4 : 0;
    static constexpr int R = LAY == 1 ? 12 : LAY == 2 ? 10 : LAY == 3 ? 14 : LAY == 4 ? 14 : N;
    static constexpr bool TT = LAY == 1 || LAY == 2 || LAY == 4;
    static constexpr int P = LAY == 1 ? 104 : LAY == 2 ? 88 : LAY == 3 ? 140 : LAY == 4 ? 172
                           : N2 + (((N - N2) % BANKS) + BANKS) % BANKS;
    static constexpr int ESZ = P * N;                          // one array, one element
    // threads per element slot: N^2 (one per r-pencil), padded to whole warps for N = 10 so that
    // the elements of a group can synchronise separately (named barriers, elem_sync); measured
    // neutral at p = 9 (fp32 -2.5%, mixed +1%, fp64 +1%: the padding costs registers), so off
#ifndef NB_PAD_ELEM
#define NB_PAD_ELEM 0
#endif
    // fp64, p = 7: two threads per r-pencil (ax_group_half), four arrays per element, 16 warps/SM.
    // Parity-clean but off: at the 128-register cap of two blocks per SM the kernel spills 416 B
    // (phase A 347 -> 411 us, phase B 176 -> 167 us at 32^3 p7).
#ifndef NB_HALF64
#define NB_HALF64 0
#endif
    static constexpr bool HALF = NB_HALF64 && sizeof(T) == 8 && N == 8;
    static constexpr int N2P = HALF ? 2 * N2 : (NB_PAD_ELEM && N == 10) ? 128 : N2;
    static constexpr int NARR = HALF ? 4 : 3;
    // fp64, N = 10: one element per 128-thread block and NB_E1_D10 resident blocks (0: two elements per
    // 224-thread block, NB_MINB_D blocks): independent blocks desynchronise, so one block's loads
    // overlap the other's contractions
#ifndef NB_E1_D10
#define NB_E1_D10 2
#endif
    // Single precision N = 10 the same way with NB_E1_S10 resident blocks -- set to 3 by the MIXED
    // policy's translation units only (nb_cg_mixed.cu, nb_cg_mixed_var.cu): 12 warps at 168 registers
    // and 122 KB of shared memory per SM instead of 14 warps at 128 registers and 163 KB leave phase B
    // more L1 and registers (32^3 p9 mixed: phase B 208 -> 187 us, iteration 496 -> 476 us; 20^3 -7%,
    // 50^3 -6%).  The fp32 policy measured 3% slower with it (its phase B has no fp64 diagonal and
    // sums), so AxCfg<float, 10> deliberately differs between the mixed and the fp32 / Dot2 / Schwarz
    // translation units: every use is a compile-time constant inside one unit (the library exports
    // no AxCfg symbol, device code is per unit), and the workspace is sized by the policy's largest grid.
#ifndef NB_E1_S10
#define NB_E1_S10 0
#endif
    static constexpr bool E1S = NB_E1_S10 && sizeof(T) == 4 && N == 10 && !HALF && !(NB_PAD_ELEM);
    static constexpr bool E1D = (NB_E1_D10 && sizeof(T) == 8 && N == 10 && !HALF) || E1S;
    static constexpr int EPB = E1D ? 1 : (N2P >= 256) ? 1 : (256 / N2P);  // elements per group
    static constexpr int NT = ((EPB * N2P + 31) / 32) * 32;     // threads per block
    static constexpr int SMEM = NARR * EPB * ESZ * (int)sizeof(T);
    // Geometric factors of the solve's phase A staged through shared memory (NB_GSTAGE bit 0: fp64
    // N = 10, bit 1: single precision N = 10, bit 2: single precision N = 12): one 1-D TMA bulk copy
    // per element (its 6 N^3 factors are contiguous) issued by one thread right after the element's
    // threads consumed the previous group's, completing on the slot's mbarrier: the fetch (half of
    // phase A's bytes) overlaps the rest of this group and the start of the next without registers,
    // load instructions or L1 tag lookups (a pencil's 40 / 80-byte stride costs 10 / 20 tag lookups
    // per warp load at N = 10).  The stage keeps the global layout: pencil reads at a 10- or 12-word
    // stride are bank-conflict-free.
#ifndef NB_GSTAGE
#define NB_GSTAGE 3
#endif
    static constexpr bool GSTAGE = !HALF && N2P == N2 &&
                                   ((N == 10 && sizeof(T) == 8 && (NB_GSTAGE & 1)) || (N == 10 && sizeof(T) == 4 && (NB_GSTAGE & 2)) ||
                                    (N == 12 && sizeof(T) == 4 && (NB_GSTAGE & 4)) || (N == 8 && sizeof(T) == 8 && (NB_GSTAGE & 8)));
    static constexpr int GSB = GSTAGE ? 6 * N3 * (int)sizeof(T) : 0;   // staged bytes per element
    static constexpr int SMEM_CG = SMEM + EPB * GSB;                   // k_cg_mega / k_cg_sw
    // the standalone operator k_ax (no phase B that wants the L1): also single precision N = 12 (bit 0)
    // and N = 8 (bit 1; 32^3 p7 mixed 127 -> 100 us, 50^3 p7 504 -> 330 us = 0.95 of the copy peak)
#ifndef NB_GSTAGE_AX
#define NB_GSTAGE_AX 3
#endif
    static constexpr bool GSTAGE_AX = !HALF && N2P == N2 && (((NB_GSTAGE_AX & 1) && (N == 10 || (N == 12 && sizeof(T) == 4))) ||
                                                             ((NB_GSTAGE_AX & 2) && N == 8 && sizeof(T) == 4));
    static constexpr int GSB_AX = GSTAGE_AX ? 6 * N3 * (int)sizeof(T) : 0;
    static constexpr int SMEM_AX = SMEM + EPB * GSB_AX;                // k_ax
    // resident blocks per SM the register allocation must allow (launch bound); fp64 pencils
    // need twice the registers
// Phase-B loads of w (own pencil, neighbour copies): w was written by other blocks in phase A,
// before the grid barrier whose acquire (ld.acquire.gpu) invalidates this SM's L1
// (CCTL.IVALL), so L1-cached loads see the new values and x-/y-neighbour copies just loaded by
// a neighbouring warp hit in L1.  NB_WLD = LD_CG keeps them L2-only.
#ifndef NB_WLD
#define NB_WLD LD_DEF
#endif
// register cap for MINB resident blocks of NT threads via __maxnreg__ instead of the minimum-
// blocks launch bound (NB_MAXNREG=1): lets ptxas use the whole budget (144 instead of 128 at
// p = 9) but measured 25-40% slower at p = 9 / 11 in single precision (not investigated), so off
#ifndef NB_MAXNREG
#define NB_MAXNREG 0
#endif
#if NB_MAXNREG
#define NB_KERNEL_BOUNDS(...) __launch_bounds__(__VA_ARGS__::NT) __maxnreg__((__VA_ARGS__::MAXNREG))
#else
#define NB_KERNEL_BOUNDS(...) __launch_bounds__(__VA_ARGS__::NT, __VA_ARGS__::MINB)
#endif
#ifndef NB_MINB_MODE
#define NB_MINB_MODE 3
#endif
// p = 11 in single precision: 3 resident blocks of 160 threads (128 registers, a few spills)
// instead of 2 -- phase B gains from the extra warps (fp32 32^3: 829 -> 795 us/iteration;
// mixed neutral to -3%)
#ifndef NB_MINB_N12
#define NB_MINB_N12 3
#endif
// fp64, N = 10 (p = 9): one resident block (255 registers, no spills) instead of two at 128
// registers with ~670 bytes of spills -- measured 1388 -> 1187 us/iteration at 32^3 p9 deformed
// (phase A 1008 -> 845 us); at N = 12 the same change is slower (1952 -> 2377 us), so only N = 10
#ifndef NB_MINB_D
#define NB_MINB_D 1
#endif
    static constexpr int MINB = E1S ? NB_E1_S10 : E1D ? NB_E1_D10 : (NB_MINB_D && sizeof(T) == 8 && N == 10) ? NB_MINB_D
                              : (NB_MINB_N12 && N == 12 && sizeof(T) == 4) ? NB_MINB_N12
                              : NB_MINB_MODE == 0 ? 1
                              : NB_MINB_MODE == 3 ? ((sizeof(T) == 4) ? (NT <= 128 ? 4 : 2) : (N <= 8 && !HALF ? 1 : 2))
                              : NB_MINB_MODE == 1 ? ((sizeof(T) == 4) ? ((NT <= 128) ? 8 : (NT <= 256 ? 4 : 2)) : ((NT <= 128) ? 4 : 2))
                                                  : ((sizeof(T) == 4) ? ((NT <= 128) ? 6 : (NT <= 256 ? 3 : 1)) : 1);
    static constexpr int MAXNREG = (65536 / (MINB * NT)) / 8 * 8 > 255 ? 255 : (65536 / (MINB * NT)) / 8 * 8;
};

template <typename T, int V>
__device__ __forceinline__ void ld_chunk(const T *__restrict__ p, T (&d)[V])
{
    using W = typename VT<T, V>::type;
    VAcc<T, V>::get(*reinterpret_cast<const W *>(p), d);
}
template <typename T, int V, int H = LD_DEF>
__device__ __forceinline__ void ld_chunk_h(const T *__restrict__ p, T (&d)[V])
{
    using W = typename VT<T, V>::type;
    VAcc<T, V>::get(ldv<H>(reinterpret_cast<const W *>(p)), d);
}
template <typename T, int V>
__device__ __forceinline__ void st_chunk(T *__restrict__ p, const T (&d)[V])
{
    using W = typename VT<T, V>::type;
    *reinterpret_cast<W *>(p) = VAcc<T, V>::put(d);
}

// One group of EPB elements, all threads of the block.  MODE 0: standalone w = A_L u
// (+ mask).  MODE 1: CG with pap over all nodes.  MODE 2: CG with the unshared-node part of
// pap only.  Returns this thread's pap partial.  Contains 4 __syncthreads; consecutive calls
// need no barrier in between (phase 1 of the next group touches only the caller's own
// r-pencil slots, which only the caller read in phase 5).
// Phase-A step 3 variants (measured per data size, tools/ab_run.sh): NB_AXV32 / NB_AXV64 for
// 4- / 8-byte data.  0: w_r^T kept in registers, pap = sum w p (p from shared); 2: register-lean
// (fp64 needs 255 registers otherwise): the geometric factors streamed chunk by chunk through a
// non-unrolled loop, w_r^T via shared memory, pap in its energy form.
#ifndef NB_AXV32
#define NB_AXV32 0
#endif
#ifndef NB_AXV64
#define NB_AXV64 2
#endif
#ifndef NB_LEAN_UNROLL
#define NB_LEAN_UNROLL 2
#endif
#ifndef NB_POLL_NS
#define NB_POLL_NS 32
#endif
#ifndef NB_ELEM_BAR
#define NB_ELEM_BAR 1
#endif
#ifndef NB_PHASE_ATTR
#define NB_PHASE_ATTR __forceinline__
#endif
// Barrier over the threads of one element of the group: a named barrier per element when the
// elements are warp-aligned (their shared-memory slots are disjoint, so elements of one block
// need not wait for each other), else the block barrier.
template <int N2, int EPB>
__device__ __forceinline__ void elem_sync()
{
#if NB_ELEM_BAR
    if constexpr (N2 % 32 == 0 && EPB > 1 && EPB < 16) {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x / N2)), "r"(N2) : "memory");
        return;
    }
#endif
    __syncthreads();
}

// mbarriers and wait parities of the element slots' staged geometric factors (AxCfg::GSTAGE)
struct GStage {
    unsigned long long bar[4];
    unsigned par[4];
};
// element e's 6 N^3 factors into the slot's stage (one thread)
template <typename TV, int N>
__device__ __forceinline__ void gstage_issue(const TV *__restrict__ g, int e, TV *__restrict__ gst, unsigned long long *bar)
{
    constexpr int N3 = N * N * N;
    tma_load_1d(gst, g + (size_t)e * 6 * N3, 6 * N3 * (unsigned)sizeof(TV), bar);
}

template <int PREC, int N, int MODE, bool SLAB = false, bool GS = false>
__device__ NB_PHASE_ATTR Acc<PREC>
ax_group(const MeshDev &m, const DMat<typename Pol<PREC>::TV, N> &D, const typename Pol<PREC>::TV *__restrict__ in,
         typename Pol<PREC>::TV *__restrict__ pv, typename Pol<PREC>::TV *__restrict__ xv,
         const typename Pol<PREC>::TV *__restrict__ g, typename Pol<PREC>::TV *__restrict__ w, bool apply_mask,
         typename Pol<PREC>::TV beta, typename Pol<PREC>::TV alpha, int e, bool active, int a, int b,
         typename Pol<PREC>::TV *__restrict__ S0, double *__restrict__ xd = nullptr, double alpha_d = 0.0,
         typename Pol<PREC>::TV *__restrict__ gst = nullptr, int e_next = -1, GStage *gsh = nullptr, int el = 0)
{
    using TV = typename Pol<PREC>::TV;
    using TS = typename Pol<PREC>::TS;
    using C = AxCfg<TV, N>;
    constexpr int V = VecW<TV, N>::V;
    constexpr int AXV = sizeof(TV) == 8 ? NB_AXV64 : NB_AXV32;
    TV *A1 = S0 + C::ESZ;
    TV *A2 = A1 + C::ESZ;
    const int q = a + N * b;
    const int rp = C::R * a + C::P * b;   // r-pencil (i, a, b): contiguous
    const int sp = a + C::P * b;       // s-pencil (a, j, b): stride R
    const int tp = C::TT ? b + C::R * a : a + C::R * b;   // t-pencil: stride P
    const size_t gbase = (size_t)e * C::N3 + (size_t)N * q;

    // ---- 1. operand: u, or (CG) p = z + beta p_old with the deferred x update
    if (active) {
        TV u[N];
        if (MODE == 0) {
            ld_pencil<TV, N>(in + gbase, u);
        } else if (PREC == NB_MIXED && xd) {
            // x_fp64 variant (C-15): x += alpha p in double with the double alpha
            TV zz[N], po[N];
            double xx[N];
            ldg_pencil<TV, N, LD_CS>(in + gbase, zz);
            ldg_pencil<TV, N>(pv + gbase, po);
            ldg_pencil<double, N, LD_CS>(xd + gbase, xx);
#pragma unroll
            for (int i = 0; i < N; i++) {
                u[i] = fma(beta, po[i], zz[i]);                 // add2s1
                xx[i] = fma(alpha_d, (double)po[i], xx[i]);     // add2s2(x, p_old, alpha_prev)
            }
            stg_pencil<TV, N>(pv + gbase, u);
            stg_pencil<double, N, LD_CS>(xd + gbase, xx);
        } else {
            TV zz[N], po[N], xx[N];
            ldg_pencil<TV, N, LD_CS>(in + gbase, zz);
            ldg_pencil<TV, N>(pv + gbase, po);
            ldg_pencil<TV, N, LD_CS>(xv + gbase, xx);
#pragma unroll
            for (int i = 0; i < N; i++) {
                u[i] = fma(beta, po[i], zz[i]);      // add2s1
                xx[i] = fma(alpha, po[i], xx[i]);    // add2s2(x, p_old, alpha_prev)
            }
            stg_pencil<TV, N>(pv + gbase, u);
            stg_pencil<TV, N, LD_CS>(xv + gbase, xx);
        }
        st_pencil<TV, N>(S0 + rp, u);
    }
    elem_sync<C::N2P, C::EPB>();
    // ---- 2. us (D along s) and ut (D along t) from shared pencils
    if (active) {
        TV v[N], o[N];
#pragma unroll
        for (int j = 0; j < N; j++) v[j] = S0[sp + C::R * j];
        contract<TV, N>(D, v, o);
#pragma unroll
        for (int j = 0; j < N; j++) A1[sp + C::R * j] = o[j];
#pragma unroll
        for (int k = 0; k < N; k++) v[k] = S0[tp + C::P * k];
        contract<TV, N>(D, v, o);
#pragma unroll
        for (int k = 0; k < N; k++) A2[tp + C::P * k] = o[k];
    }
    elem_sync<C::N2P, C::EPB>();
    Acc<PREC> acc;
    if constexpr (AXV == 0) {
    // ---- 3. ur in registers; geometric factors (C-7); r-part of local_grad3_t
    TV wrt[N];
    if (active) {
        TV ur[N], wr[N];
        {
            TV v[N];
            ld_pencil<TV, N>(S0 + rp, v);
            contract<TV, N>(D, v, ur);
        }
        const TV *ge = g + (size_t)e * 6 * C::N3 + (size_t)N * q;
        if constexpr (GS) mbar_wait(&gsh->bar[el], gsh->par[el]);
#pragma unroll
        for (int c = 0; c < N / V; c++) {
            TV g1[V], g2[V], g3[V], g4[V], g5[V], g6[V], us[V], ut[V], ws[V], wt[V];
            if constexpr (GS) {
                ld_chunk<TV, V>(gst + 0 * C::N3 + N * q + c * V, g1);
                ld_chunk<TV, V>(gst + 1 * C::N3 + N * q + c * V, g2);
                ld_chunk<TV, V>(gst + 2 * C::N3 + N * q + c * V, g3);
                ld_chunk<TV, V>(gst + 3 * C::N3 + N * q + c * V, g4);
                ld_chunk<TV, V>(gst + 4 * C::N3 + N * q + c * V, g5);
                ld_chunk<TV, V>(gst + 5 * C::N3 + N * q + c * V, g6);
            } else {
            ld_chunk_h<TV, V, LD_CS>(ge + 0 * C::N3 + c * V, g1);
            ld_chunk_h<TV, V, LD_CS>(ge + 1 * C::N3 + c * V, g2);
            ld_chunk_h<TV, V, LD_CS>(ge + 2 * C::N3 + c * V, g3);
            ld_chunk_h<TV, V, LD_CS>(ge + 3 * C::N3 + c * V, g4);
            ld_chunk_h<TV, V, LD_CS>(ge + 4 * C::N3 + c * V, g5);
            ld_chunk_h<TV, V, LD_CS>(ge + 5 * C::N3 + c * V, g6);
            }
            ld_chunk<TV, V>(A1 + rp + c * V, us);
            ld_chunk<TV, V>(A2 + rp + c * V, ut);
#pragma unroll
            for (int t = 0; t < V; t++) {
                const TV r_ = ur[c * V + t];
                wr[c * V + t] = fma(g3[t], ut[t], fma(g2[t], us[t], g1[t] * r_));
                ws[t] = fma(g5[t], ut[t], fma(g4[t], us[t], g2[t] * r_));
                wt[t] = fma(g6[t], ut[t], fma(g5[t], us[t], g3[t] * r_));
            }
            st_chunk<TV, V>(A1 + rp + c * V, ws);
            st_chunk<TV, V>(A2 + rp + c * V, wt);
        }
        contract_t<TV, N>(D, wr, wrt);
    }
    elem_sync<C::N2P, C::EPB>();
    if constexpr (GS) {   // the element's threads are done with the stage: flip its parity, fetch the next group's
        if (active && q == 0) {
            gsh->par[el] ^= 1u;
            if (e_next >= 0) gstage_issue<TV, N>(g, e_next, gst, &gsh->bar[el]);
        }
    }
    // ---- 4. s- and t-parts of local_grad3_t, in place on the owner's pencils
    if (active) {
        TV v[N], o[N];
#pragma unroll
        for (int j = 0; j < N; j++) v[j] = A1[sp + C::R * j];
        contract_t<TV, N>(D, v, o);
#pragma unroll
        for (int j = 0; j < N; j++) A1[sp + C::R * j] = o[j];
#pragma unroll
        for (int k = 0; k < N; k++) v[k] = A2[tp + C::P * k];
        contract_t<TV, N>(D, v, o);
#pragma unroll
        for (int k = 0; k < N; k++) A2[tp + C::P * k] = o[k];
    }
    elem_sync<C::N2P, C::EPB>();
    // ---- 5. w = (w_r + w_s) + w_t, Dirichlet mask, store; CG: pap partial (p from S0)
    if (active) {
        TV out[N];
        {
            TV t1[N], t2[N];
            ld_pencil<TV, N>(A1 + rp, t1);
            ld_pencil<TV, N>(A2 + rp, t2);
#pragma unroll
            for (int i = 0; i < N; i++) out[i] = (wrt[i] + t1[i]) + t2[i];
        }
        if (MODE != 0 || apply_mask) {
            const ElemPos P = elem_pos<SLAB>(m, e);
            const bool mjk = axis_bnd(a, N, P.ey, m.nely) || axis_bnd(b, N, P.ez, m.nelz);
#pragma unroll
            for (int i = 0; i < N; i++)
                if (mjk || axis_bnd(i, N, P.ex, m.nelx)) out[i] = TV(0);
            if (MODE == 2) {   // unshared nodes only (c = 1); the CSR phase adds the shared ones
                const bool sjk = axis_mult(a, N, P.ey, m.nely) * axis_mult(b, N, P.ez, m.nelz) > 1;
                TV pp[N];
                ld_pencil<TV, N>(S0 + rp, pp);
#pragma unroll
                for (int i = 0; i < N; i++)
                    if (!sjk && axis_mult(i, N, P.ex, m.nelx) == 1) acc.add((TS)out[i], (TS)pp[i]);
            }
        }
        if (MODE == 1) {
            TV pp[N];
            ld_pencil<TV, N>(S0 + rp, pp);
#pragma unroll
            for (int i = 0; i < N; i++) acc.add((TS)out[i], (TS)pp[i]);
        }
        stg_pencil<TV, N>(w + gbase, out);
    }
    } else {
    // ---- 3. (register-lean) ur to the owner's S0 slots; the geometric factors streamed in
    // chunks of V values (loop not unrolled: one chunk of operands live at a time); pap in
    // energy form (MODE 1); w_r^T back into S0.
    if (active) {
        {
            TV v[N], o[N];
            ld_pencil<TV, N>(S0 + rp, v);
            contract<TV, N>(D, v, o);
            st_pencil<TV, N>(S0 + rp, o);
        }
        const TV *ge = g + (size_t)e * 6 * C::N3 + (size_t)N * q;
// two chunks of geometric factors in flight for p >= 7 (fp64 phase A -3% / -14% / -7% at p = 7 / 9 / 11;
// +2% at p = 5, so not below)
constexpr int LEAN_U = N >= 8 ? NB_LEAN_UNROLL : 1;
        if constexpr (GS) mbar_wait(&gsh->bar[el], gsh->par[el]);
#pragma unroll LEAN_U
        for (int c = 0; c < N / V; c++) {
            TV g1[V], g2[V], g3[V], g4[V], g5[V], g6[V], ur[V], us[V], ut[V], wr[V], ws[V], wt[V];
            if constexpr (GS) {
                ld_chunk<TV, V>(gst + 0 * C::N3 + N * q + c * V, g1);
                ld_chunk<TV, V>(gst + 1 * C::N3 + N * q + c * V, g2);
                ld_chunk<TV, V>(gst + 2 * C::N3 + N * q + c * V, g3);
                ld_chunk<TV, V>(gst + 3 * C::N3 + N * q + c * V, g4);
                ld_chunk<TV, V>(gst + 4 * C::N3 + N * q + c * V, g5);
                ld_chunk<TV, V>(gst + 5 * C::N3 + N * q + c * V, g6);
            } else {
            ld_chunk<TV, V>(ge + 0 * C::N3 + c * V, g1);
            ld_chunk<TV, V>(ge + 1 * C::N3 + c * V, g2);
            ld_chunk<TV, V>(ge + 2 * C::N3 + c * V, g3);
            ld_chunk<TV, V>(ge + 3 * C::N3 + c * V, g4);
            ld_chunk<TV, V>(ge + 4 * C::N3 + c * V, g5);
            ld_chunk<TV, V>(ge + 5 * C::N3 + c * V, g6);
            }
            ld_chunk<TV, V>(S0 + rp + c * V, ur);
            ld_chunk<TV, V>(A1 + rp + c * V, us);
            ld_chunk<TV, V>(A2 + rp + c * V, ut);
#pragma unroll
            for (int t = 0; t < V; t++) {
                wr[t] = fma(g3[t], ut[t], fma(g2[t], us[t], g1[t] * ur[t]));
                ws[t] = fma(g5[t], ut[t], fma(g4[t], us[t], g2[t] * ur[t]));
                wt[t] = fma(g6[t], ut[t], fma(g5[t], us[t], g3[t] * ur[t]));
                if (MODE == 1) acc.add_sum(((TS)ur[t] * (TS)wr[t] + (TS)us[t] * (TS)ws[t]) + (TS)ut[t] * (TS)wt[t]);
            }
            st_chunk<TV, V>(S0 + rp + c * V, wr);
            st_chunk<TV, V>(A1 + rp + c * V, ws);
            st_chunk<TV, V>(A2 + rp + c * V, wt);
        }
        {
            TV v[N], o[N];
            ld_pencil<TV, N>(S0 + rp, v);
            contract_t<TV, N>(D, v, o);
            st_pencil<TV, N>(S0 + rp, o);
        }
    }
    elem_sync<C::N2P, C::EPB>();
    if constexpr (GS) {   // the element's threads are done with the stage: flip its parity, fetch the next group's
        if (active && q == 0) {
            gsh->par[el] ^= 1u;
            if (e_next >= 0) gstage_issue<TV, N>(g, e_next, gst, &gsh->bar[el]);
        }
    }
    // ---- 4. s- and t-parts of local_grad3_t, in place on the owner's pencils
    if (active) {
        TV v[N], o[N];
#pragma unroll
        for (int j = 0; j < N; j++) v[j] = A1[sp + C::R * j];
        contract_t<TV, N>(D, v, o);
#pragma unroll
        for (int j = 0; j < N; j++) A1[sp + C::R * j] = o[j];
#pragma unroll
        for (int k = 0; k < N; k++) v[k] = A2[tp + C::P * k];
        contract_t<TV, N>(D, v, o);
#pragma unroll
        for (int k = 0; k < N; k++) A2[tp + C::P * k] = o[k];
    }
    elem_sync<C::N2P, C::EPB>();
    // ---- 5. w = (w_r + w_s) + w_t, Dirichlet mask, store
    if (active) {
        TV out[N];
        {
            TV t0[N], t1[N], t2[N];
            ld_pencil<TV, N>(S0 + rp, t0);
            ld_pencil<TV, N>(A1 + rp, t1);
            ld_pencil<TV, N>(A2 + rp, t2);
#pragma unroll
            for (int i = 0; i < N; i++) out[i] = (t0[i] + t1[i]) + t2[i];
        }
        if (MODE != 0 || apply_mask) {
            const ElemPos P = elem_pos<SLAB>(m, e);
            const bool mjk = axis_bnd(a, N, P.ey, m.nely) || axis_bnd(b, N, P.ez, m.nelz);
#pragma unroll
            for (int i = 0; i < N; i++)
                if (mjk || axis_bnd(i, N, P.ex, m.nelx)) out[i] = TV(0);
            if (MODE == 2) {   // unshared nodes only (c = 1); the CSR phase adds the shared ones
                const bool sjk = axis_mult(a, N, P.ey, m.nely) * axis_mult(b, N, P.ez, m.nelz) > 1;
                TV pp[N];
                ldg_pencil<TV, N>(pv + gbase, pp);   // written by this thread in step 1
#pragma unroll
                for (int i = 0; i < N; i++)
                    if (!sjk && axis_mult(i, N, P.ex, m.nelx) == 1) acc.add((TS)out[i], (TS)pp[i]);
            }
        }
        stg_pencil<TV, N>(w + gbase, out);
    }
    }
    return acc;
}

// o[i'] = sum_l M[I0 + i'][l] v[l] for NO consecutive output rows starting at the compile-time row
// I0 (M column-pair-adjacent as in contract_pairs): the partial contraction of a half pencil.
template <typename T, int N, int I0, int NO>
__device__ __forceinline__ void contract_rows(const T *__restrict__ mt, const T (&v)[N], T (&o)[NO])
{
#pragma unroll
    for (int i = 0; i < NO; i++) {
        T s = mt[I0 + i] * v[0];
#pragma unroll
        for (int l = 1; l < N; l++) s = fma(mt[l * N + I0 + i], v[l], s);
        o[i] = s;
    }
}

// ax_group with TWO threads per r-pencil (AxCfg::HALF, fp64): the element's 2 N^2 threads are
// two warp-aligned halves -- half h owns nodes [h N/2, (h+1) N/2) of its pencil for the pointwise
// work (operand, geometric factors, output) and does the s-contractions (h = 0) or the
// t-contractions (h = 1) of its pencil index.  Half the pencil registers per thread lets fp64
// run twice the warps per SM (16 instead of 8).  h is warp-uniform, so the row split of the
// r-contractions keeps D in constant-bank operands without divergence.  Arrays: S0 = u, then
// w_r^T; A1 = us, ws, then w_s^T; A2 = ut, wt, then w_t^T; A3 = wr.
template <int PREC, int N, int MODE, bool SLAB = false>
__device__ __forceinline__ Acc<PREC>
ax_group_half(const MeshDev &m, const DMat<typename Pol<PREC>::TV, N> &D, const typename Pol<PREC>::TV *__restrict__ in,
              typename Pol<PREC>::TV *__restrict__ pv, typename Pol<PREC>::TV *__restrict__ xv,
              const typename Pol<PREC>::TV *__restrict__ g, typename Pol<PREC>::TV *__restrict__ w, bool apply_mask,
              typename Pol<PREC>::TV beta, typename Pol<PREC>::TV alpha, int e, bool active, int a, int b, int h,
              typename Pol<PREC>::TV *__restrict__ S0)
{
    using TV = typename Pol<PREC>::TV;
    using TS = typename Pol<PREC>::TS;
    using C = AxCfg<TV, N>;
    constexpr int H = N / 2;
    static_assert(N % 2 == 0 && (H * sizeof(TV)) % 16 == 0 || H % 2 == 0, "half pencils of whole 16-byte chunks");
    TV *A1 = S0 + C::ESZ;
    TV *A2 = A1 + C::ESZ;
    TV *A3 = A2 + C::ESZ;
    const int q = a + N * b;
    const int i0 = h * H;
    const int rp = C::R * a + C::P * b;
    const int sp = a + C::P * b;
    const int tp = C::TT ? b + C::R * a : a + C::R * b;
    const size_t gbase = (size_t)e * C::N3 + (size_t)N * q + i0;
    Acc<PREC> acc;

    // ---- 1. operand half: u, or p = z + beta p_old with the deferred x update
    if (active) {
        TV u[H];
        if (MODE == 0) {
            ld_pencil<TV, H>(in + gbase, u);
        } else {
            TV zz[H], po[H], xx[H];
            ld_pencil<TV, H, LD_CS>(in + gbase, zz);
            ld_pencil<TV, H>(pv + gbase, po);
            ld_pencil<TV, H, LD_CS>(xv + gbase, xx);
#pragma unroll
            for (int i = 0; i < H; i++) {
                u[i] = fma(beta, po[i], zz[i]);      // add2s1
                xx[i] = fma(alpha, po[i], xx[i]);    // add2s2(x, p_old, alpha_prev)
            }
            st_pencil<TV, H>(pv + gbase, u);
            st_pencil<TV, H, LD_CS>(xv + gbase, xx);
        }
        st_pencil<TV, H>(S0 + rp + i0, u);
    }
    elem_sync<C::N2P, C::EPB>();
    // ---- 2. us (h = 0) or ut (h = 1) of pencil index (a, b)
    if (active) {
        TV v[N], o[N];
        if (h == 0) {
#pragma unroll
            for (int j = 0; j < N; j++) v[j] = S0[sp + C::R * j];
            contract<TV, N>(D, v, o);
#pragma unroll
            for (int j = 0; j < N; j++) A1[sp + C::R * j] = o[j];
        } else {
#pragma unroll
            for (int k = 0; k < N; k++) v[k] = S0[tp + C::P * k];
            contract<TV, N>(D, v, o);
#pragma unroll
            for (int k = 0; k < N; k++) A2[tp + C::P * k] = o[k];
        }
    }
    elem_sync<C::N2P, C::EPB>();
    // ---- 3. ur of the owned rows from the full u pencil; geometric factors; wr -> A3, ws/wt in place
    if (active) {
        TV ur[H];
        {
            TV v[N];
            ld_pencil<TV, N>(S0 + rp, v);
            if (h == 0) contract_rows<TV, N, 0, H>(D.dt, v, ur);
            else contract_rows<TV, N, H, H>(D.dt, v, ur);
        }
        const TV *ge = g + (size_t)e * 6 * C::N3 + (size_t)N * q + i0;
        TV g1[H], g2[H], g3[H], g4[H], g5[H], g6[H], us[H], ut[H], wr[H], ws[H], wt[H];
        ld_pencil<TV, H, LD_CS>(ge + 0 * C::N3, g1);
        ld_pencil<TV, H, LD_CS>(ge + 1 * C::N3, g2);
        ld_pencil<TV, H, LD_CS>(ge + 2 * C::N3, g3);
        ld_pencil<TV, H, LD_CS>(ge + 3 * C::N3, g4);
        ld_pencil<TV, H, LD_CS>(ge + 4 * C::N3, g5);
        ld_pencil<TV, H, LD_CS>(ge + 5 * C::N3, g6);
        ld_pencil<TV, H>(A1 + rp + i0, us);
        ld_pencil<TV, H>(A2 + rp + i0, ut);
#pragma unroll
        for (int t = 0; t < H; t++) {
            wr[t] = fma(g3[t], ut[t], fma(g2[t], us[t], g1[t] * ur[t]));
            ws[t] = fma(g5[t], ut[t], fma(g4[t], us[t], g2[t] * ur[t]));
            wt[t] = fma(g6[t], ut[t], fma(g5[t], us[t], g3[t] * ur[t]));
            if (MODE == 1) acc.add_sum(((TS)ur[t] * (TS)wr[t] + (TS)us[t] * (TS)ws[t]) + (TS)ut[t] * (TS)wt[t]);
        }
        st_pencil<TV, H>(A3 + rp + i0, wr);
        st_pencil<TV, H>(A1 + rp + i0, ws);
        st_pencil<TV, H>(A2 + rp + i0, wt);
    }
    elem_sync<C::N2P, C::EPB>();
    // ---- 3b. r-part of local_grad3_t for the owned rows (S0's u is no longer read);
    // ---- 4. s- (h = 0) or t-part (h = 1) of local_grad3_t, in place
    if (active) {
        {
            TV v[N], o[H];
            ld_pencil<TV, N>(A3 + rp, v);
            if (h == 0) contract_rows<TV, N, 0, H>(D.d, v, o);
            else contract_rows<TV, N, H, H>(D.d, v, o);
            st_pencil<TV, H>(S0 + rp + i0, o);
        }
        TV v[N], o[N];
        if (h == 0) {
#pragma unroll
            for (int j = 0; j < N; j++) v[j] = A1[sp + C::R * j];
            contract_t<TV, N>(D, v, o);
#pragma unroll
            for (int j = 0; j < N; j++) A1[sp + C::R * j] = o[j];
        } else {
#pragma unroll
            for (int k = 0; k < N; k++) v[k] = A2[tp + C::P * k];
            contract_t<TV, N>(D, v, o);
#pragma unroll
            for (int k = 0; k < N; k++) A2[tp + C::P * k] = o[k];
        }
    }
    elem_sync<C::N2P, C::EPB>();
    // ---- 5. w = (w_r + w_s) + w_t on the owned nodes, Dirichlet mask, store
    if (active) {
        TV out[H];
        {
            TV t0[H], t1[H], t2[H];
            ld_pencil<TV, H>(S0 + rp + i0, t0);
            ld_pencil<TV, H>(A1 + rp + i0, t1);
            ld_pencil<TV, H>(A2 + rp + i0, t2);
#pragma unroll
            for (int i = 0; i < H; i++) out[i] = (t0[i] + t1[i]) + t2[i];
        }
        if (MODE != 0 || apply_mask) {
            const ElemPos P = elem_pos<SLAB>(m, e);
            const bool mjk = axis_bnd(a, N, P.ey, m.nely) || axis_bnd(b, N, P.ez, m.nelz);
#pragma unroll
            for (int i = 0; i < H; i++)
                if (mjk || axis_bnd(i0 + i, N, P.ex, m.nelx)) out[i] = TV(0);
            if (MODE == 2) {   // unshared nodes only (c = 1); the CSR phase adds the shared ones
                const bool sjk = axis_mult(a, N, P.ey, m.nely) * axis_mult(b, N, P.ez, m.nelz) > 1;
                TV pp[H];
                ld_pencil<TV, H>(pv + gbase, pp);   // written by this thread in step 1
#pragma unroll
                for (int i = 0; i < H; i++)
                    if (!sjk && axis_mult(i0 + i, N, P.ex, m.nelx) == 1) acc.add((TS)out[i], (TS)pp[i]);
            }
        }
        st_pencil<TV, H>(w + gbase, out);
    }
    return acc;
}

// ===========================================================================
// phase B: (gather QQ^T) + add2s2(r) + solveM + glsc3 x2, one r-pencil per call
// ===========================================================================
// Consistent-order assembled value of the pencil (a, b) of element e (C-8): for each node
// the copies are summed in ascending element order (= ascending local index), i.e.
// lexicographic in (dz, dy, dx), in the gather-scatter precision TG, and rounded once.
// Neighbour values are read through L2 (ld.cg): other blocks wrote them in this kernel.
template <int PREC, int N>
__device__ __forceinline__ void gather_pencil(const MeshDev &m, const typename Pol<PREC>::TV *__restrict__ w,
                                              int e, const ElemPos &P, int a, int b,
                                              typename Pol<PREC>::TV (&ww)[N], typename Pol<PREC>::TV own_l,
                                              typename Pol<PREC>::TV own_r,
                                              const typename Pol<PREC>::TV *wlo = nullptr,
                                              const typename Pol<PREC>::TV *whi = nullptr)
{
    using TV = typename Pol<PREC>::TV;
    using TG = typename Pol<PREC>::TG;
    constexpr int N2 = N * N, N3 = N * N * N;
    const int ys = (a == 0 && P.ey > 0) ? -1 : ((a == N - 1 && P.ey < m.nely - 1) ? 1 : 0);
    const int zs = (b == 0 && P.ez > 0) ? -1 : ((b == N - 1 && P.ez < m.nelz - 1) ? 1 : 0);
    const bool xl = P.ex > 0, xr = P.ex < m.nelx - 1;
    if (ys == 0 && zs == 0 && !xl && !xr) return;
    // Issue every neighbour load first (one L2 round trip), then sum in the fixed order.
    // Copies of the pencil's nodes: own (0,0), y-neighbour (0,1), z-neighbour (1,0) and the
    // yz-diagonal neighbour (1,1); each with its x-partners for the end nodes.
    TV vy[N], vz[N], vyz[N];
    TV ly = 0, ry = 0, lz = 0, rz = 0, lyz = 0, ryz = 0;
    const size_t base = ((size_t)e * N2 + (size_t)(a + N * b)) * N;
    const int64_t sy = (int64_t)ys * (m.nelx * (int64_t)N3) + (int64_t)(ys ? (N - 1 - 2 * a) : 0) * N;
    const int64_t sz = (int64_t)zs * ((int64_t)m.nelx * m.nely * N3) + (int64_t)(zs ? (N - 1 - 2 * b) : 0) * N2;
    // z-neighbour layer: this slab's own w, or a neighbour slab's (multi-rank; rebased pointers)
    const TV *wz = w;
    if (wlo && zs < 0 && P.ez == m.ez0) wz = wlo;
    if (whi && zs > 0 && P.ez == m.ez0 + m.nelzl - 1) wz = whi;
    if (ys) {
        ld_pencil<TV, N, NB_WLD>(w + base + sy, vy);
        if (xl) ly = ldv<NB_WLD>(w + base + sy - N3 + (N - 1));
        if (xr) ry = ldv<NB_WLD>(w + base + sy + N3);
    }
    if (zs) {
        ld_pencil<TV, N, NB_WLD>(wz + base + sz, vz);
        if (xl) lz = ldv<NB_WLD>(wz + base + sz - N3 + (N - 1));
        if (xr) rz = ldv<NB_WLD>(wz + base + sz + N3);
    }
    if (ys && zs) {
        ld_pencil<TV, N, NB_WLD>(wz + base + sy + sz, vyz);
        if (xl) lyz = ldv<NB_WLD>(wz + base + sy + sz - N3 + (N - 1));
        if (xr) ryz = ldv<NB_WLD>(wz + base + sy + sz + N3);
    }
    // ascending element order: lexicographic (dz, dy, dx); a negative offset comes first
    TG s[N];
#pragma unroll
    for (int iz = 0; iz < 2; iz++) {
#pragma unroll
        for (int iy = 0; iy < 2; iy++) {
            if (iz == 1 && !zs) continue;
            if (iy == 1 && !ys) continue;
            const bool zf = zs ? ((zs < 0) == (iz == 0)) : false;   // this combo uses the z-neighbour
            const bool yf = ys ? ((ys < 0) == (iy == 0)) : false;
            const bool first = (iz == 0 && iy == 0);
#pragma unroll
            for (int i = 0; i < N; i++) {
                const TV v = zf ? (yf ? vyz[i] : vz[i]) : (yf ? vy[i] : ww[i]);
                if (i == 0 && xl) {
                    const TV l = zf ? (yf ? lyz : lz) : (yf ? ly : own_l);
                    s[0] = first ? (TG)l : s[0] + (TG)l;
                    s[0] += (TG)v;
                } else {
                    s[i] = first ? (TG)v : s[i] + (TG)v;
                }
                if (i == N - 1 && xr) {
                    const TV rr = zf ? (yf ? ryz : rz) : (yf ? ry : own_r);
                    s[N - 1] += (TG)rr;
                }
            }
        }
    }
    const bool yz = ys != 0 || zs != 0;
#pragma unroll
    for (int i = 0; i < N; i++)
        if (yz || (i == 0 && xl) || (i == N - 1 && xr)) ww[i] = (TV)s[i];
}

// z = M^-1 r of the preconditioner variant (nb.h nb_precond, uniform runtime pc): the dinv
// pencil as TJ -- the policy's diagonal, or under mixed the fp32 copy (NB_PC_JACOBI_F32) widened
// exactly; the identity loads nothing (d = 1, so z = r exactly, and z aliases r).
template <typename TJ, int N>
__device__ __forceinline__ void ld_dinv(const void *__restrict__ dinv, size_t base, int pc, TJ (&dd)[N])
{
    if (pc == NB_PC_IDENTITY) {
#pragma unroll
        for (int i = 0; i < N; i++) dd[i] = TJ(1);
    } else if (sizeof(TJ) == 8 && pc == NB_PC_JACOBI_F32) {
        float f[N];
        ld_pencil<float, N, LD_NC>((const float *)dinv + base, f);
#pragma unroll
        for (int i = 0; i < N; i++) dd[i] = (TJ)f[i];
    } else {
        ld_pencil<TJ, N, LD_NC>((const TJ *)dinv + base, dd);
    }
}
template <int PREC>
__device__ __forceinline__ typename Pol<PREC>::TV solve_m(typename Pol<PREC>::TV r, typename Pol<PREC>::TJ d, int pc)
{
    using TV = typename Pol<PREC>::TV;
    if (PREC == NB_MIXED && pc == NB_PC_JACOBI_F32) return (TV)((float)r * (float)d);   // Neko's fp32 copy
    return (TV)((typename Pol<PREC>::TJ)r * d);
}

template <int PREC, int N, int GATHER, bool SLAB = false, bool SW = false>
__device__ __forceinline__ void upd_pencil(const MeshDev &m, const typename Pol<PREC>::TV *__restrict__ w,
                                           typename Pol<PREC>::TV *__restrict__ r, typename Pol<PREC>::TV *__restrict__ z,
                                           const void *__restrict__ dinv,
                                           typename Pol<PREC>::TV alpha, int64_t pid, Acc<PREC> &rtr, Acc<PREC> &rho,
                                           int pc = NB_PC_JACOBI, const typename Pol<PREC>::TV *wlo = nullptr,
                                           const typename Pol<PREC>::TV *whi = nullptr)
{
    using TV = typename Pol<PREC>::TV;
    using TJ = typename Pol<PREC>::TJ;
    using TS = typename Pol<PREC>::TS;
    constexpr int N2 = N * N;
    const int e = (int)(pid / N2);
    const int q = (int)(pid - (int64_t)e * N2);
    const int a = q % N, b = q / N;
    const size_t base = (size_t)pid * N;
    TV ww[N], rr[N], zz[N];
    TJ dd[N];
    const ElemPos P = elem_pos<SLAB>(m, e);
    ld_pencil<TV, N, NB_WLD>(w + base, ww);
    ld_pencil<TV, N>(r + base, rr);
    if (!SW) ld_dinv<TJ, N>(dinv, base, pc, dd);
    if (GATHER) {
        constexpr int N3 = N * N * N;
        const TV ol = P.ex > 0 ? ldv<NB_WLD>(w + base - N3 + (N - 1)) : TV(0);
        const TV orr = P.ex < m.nelx - 1 ? ldv<NB_WLD>(w + base + N3) : TV(0);
        gather_pencil<PREC, N>(m, w, e, P, a, b, ww, ol, orr, wlo, whi);
    }
    const int mjk = axis_mult(a, N, P.ey, m.nely) * axis_mult(b, N, P.ez, m.nelz);
#pragma unroll
    for (int i = 0; i < N; i++) {
        rr[i] = fma(-alpha, ww[i], rr[i]);                   // add2s2(r, w, -alpha)
        const TS c = (TS)1 / (TS)(mjk * axis_mult(i, N, P.ex, m.nelx));
        const TS rs = (TS)rr[i];
        rtr.add(rs * c, rs);                                 // glsc3(r, c, r)
        if (!SW) {                                           // (Schwarz: solveM is its own phase)
            zz[i] = solve_m<PREC>(rr[i], dd[i], pc);          // solveM
            rho.add(rs * c, (TS)zz[i]);                      // glsc3(r, c, z)
        }
    }
    st_pencil<TV, N>(r + base, rr);
    if (!SW && pc != NB_PC_IDENTITY) st_pencil<TV, N>(z + base, zz);
}

// CG prologue for one pencil: r = b, x = 0, p = 0, z = M^-1 r; rtr0 and rho_1 partials.
template <int PREC, int N, bool SLAB = false, bool SW = false>
__device__ __forceinline__ void init_pencil(const MeshDev &m, const typename Pol<PREC>::TV *__restrict__ bvec,
                                            typename Pol<PREC>::TV *__restrict__ x, typename Pol<PREC>::TV *__restrict__ pv,
                                            typename Pol<PREC>::TV *__restrict__ r, typename Pol<PREC>::TV *__restrict__ z,
                                            const void *__restrict__ dinv, int64_t pid,
                                            Acc<PREC> &rtr, Acc<PREC> &rho, bool x64 = false, int pc = NB_PC_JACOBI)
{
    using TV = typename Pol<PREC>::TV;
    using TS = typename Pol<PREC>::TS;
    using TD = typename Pol<PREC>::TJ;
    constexpr int N2 = N * N;
    const int e = (int)(pid / N2);
    const int q = (int)(pid - (int64_t)e * N2);
    const int a = q % N, b = q / N;
    const size_t base = (size_t)pid * N;
    const ElemPos P = elem_pos<SLAB>(m, e);
    TV rr[N], zz[N], zero[N];
    TD dd[N];
    ld_pencil<TV, N>(bvec + base, rr);
    if (!SW) ld_dinv<TD, N>(dinv, base, pc, dd);
    const int mjk = axis_mult(a, N, P.ey, m.nely) * axis_mult(b, N, P.ez, m.nelz);
#pragma unroll
    for (int i = 0; i < N; i++) {
        zero[i] = TV(0);
        const TS c = (TS)1 / (TS)(mjk * axis_mult(i, N, P.ex, m.nelx));
        const TS rs = (TS)rr[i];
        rtr.add(rs * c, rs);
        if (!SW) {
            zz[i] = solve_m<PREC>(rr[i], dd[i], pc);
            rho.add(rs * c, (TS)zz[i]);
        }
    }
    st_pencil<TV, N>(r + base, rr);
    if (!SW && pc != NB_PC_IDENTITY) st_pencil<TV, N>(z + base, zz);
    if (PREC == NB_MIXED && x64) {
        double zd[N];
#pragma unroll
        for (int i = 0; i < N; i++) zd[i] = 0.0;
        st_pencil<double, N>((double *)x + base, zd);
    } else {
        st_pencil<TV, N>(x + base, zero);
    }
    st_pencil<TV, N>(pv + base, zero);
}

// contiguous even split of [0, n) over `parts`
__device__ __forceinline__ int64_t split(int64_t n, int parts, int i) { return n * i / parts; }

// Element groups [lo, hi) of (virtual) block i of G.  S = 0: the contiguous even split over the
// blocks.  S > 0 (a full persistent grid of G = occ * S blocks, block i = the k-th resident block of
// the s-th SM, i = s occ + k): the groups are split evenly over the S SMs first and each SM's
// contiguous share over its occ blocks, so the busiest SM holds ceil(ng / S) groups instead of
// occ * ceil(ng / G) (configs[1]: 1024 groups, 148 SMs, occ 2: 7 instead of 8).
__device__ __forceinline__ void grp_range(int64_t ng, int G, int S, int i, int64_t &lo, int64_t &hi)
{
    if (S > 0 && G > S && G % S == 0) {
        const int occ = G / S, s = i / occ, k = i % occ;
        const int64_t a = split(ng, S, s), b = split(ng, S, s + 1);
        lo = a + split(b - a, occ, k);
        hi = a + split(b - a, occ, k + 1);
    } else {
        lo = split(ng, G, i);
        hi = split(ng, G, i + 1);
    }
}

// ---------------------------------------------------------------------------
// L2 prefetch distances (l2_prefetch, nb_common.cuh): phase A prefetches the operands of the
// element group NB_L2PF_A groups ahead (g, z, p_old, x: one contiguous range each), phase B the
// w, r, dinv ranges of the pencil trip NB_L2PF_B trips ahead; each phase's first ranges are
// prefetched before the grid barrier that precedes it (they are the block's own data, final
// before that barrier).  0 = off.
// ---------------------------------------------------------------------------
#ifndef NB_L2PF_A
#define NB_L2PF_A 0
#endif
#ifndef NB_L2PF_B
#define NB_L2PF_B 0
#endif
#ifndef NB_L2PF_N8ONLY
#define NB_L2PF_N8ONLY 0
#endif
#ifndef NB_L2PF_LEAD
#define NB_L2PF_LEAD 1
#endif
// which phase-A ranges (bits: 1 g, 2 z, 4 p_old, 8 x)
#ifndef NB_L2PF_MASK
#define NB_L2PF_MASK 15
#endif
// the standalone operator k_ax (u and g, one group ahead)
#ifndef NB_L2PF_AX
#define NB_L2PF_AX 1
#endif
// group grp (EPB elements from grp*EPB, clipped to E): threads 0, 32, 64, 96 issue one range each
template <typename TV, int N, int EPB, int MASK = NB_L2PF_MASK>
__device__ __forceinline__ void pf_group(int64_t grp, int64_t gend, int E, const TV *g, const void *z, const void *p,
                                         const void *x, int xsz)
{
    constexpr int64_t N3 = N * N * N;
    const int t = threadIdx.x;
    if ((t & 31) || t >= 128 || grp >= gend) return;
    const int64_t e0 = grp * EPB;
    if (e0 >= E) return;
    const int64_t ne = min((int64_t)EPB, (int64_t)E - e0);
    if (t == 0 && (MASK & 1)) l2_prefetch(g + e0 * 6 * N3, (size_t)(ne * 6 * N3) * sizeof(TV));
    else if (t == 32 && z && (MASK & 2)) l2_prefetch((const TV *)z + e0 * N3, (size_t)(ne * N3) * sizeof(TV));
    else if (t == 64 && p && (MASK & 4)) l2_prefetch((const TV *)p + e0 * N3, (size_t)(ne * N3) * sizeof(TV));
    else if (t == 96 && x && (MASK & 8)) l2_prefetch((const char *)x + e0 * N3 * xsz, (size_t)(ne * N3) * xsz);
}
// phase-B pencils [pb, min(pb + blockDim, pend)): w, r and the diagonal (dsz bytes per value, 0: none)
template <typename TV, int N>
__device__ __forceinline__ void pf_trip(int64_t pb, int64_t pend, const void *w, const void *r, const void *dinv,
                                        int dsz)
{
    const int t = threadIdx.x;
    if ((t & 31) || t >= 96 || pb >= pend) return;
    const int64_t np = min((int64_t)blockDim.x, pend - pb);
    if (t == 0) l2_prefetch((const TV *)w + pb * N, (size_t)(np * N) * sizeof(TV));
    else if (t == 32) l2_prefetch((const TV *)r + pb * N, (size_t)(np * N) * sizeof(TV));
    else if (dsz) l2_prefetch((const char *)dinv + pb * N * dsz, (size_t)(np * N) * dsz);
}

// ===========================================================================
// persistent cooperative megakernel: the whole solve in one launch
// ===========================================================================
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int *p)
{
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int *p, unsigned int v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Grid-wide barrier of a cooperative launch (all blocks co-resident): arrival counter +
// generation word with release/acquire ordering.  The gpu-scope fences make every block's
// global writes before the barrier visible to every block after it.
__device__ __forceinline__ void grid_barrier(unsigned int *bar)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int gen = ld_acquire_u32(bar + 1);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");   // this block's writes before the arrival
        const unsigned int prev = atomicAdd(bar, 1u);
        if (prev == gridDim.x - 1) {
            bar[0] = 0;
            st_release_u32(bar + 1, gen + 1);              // orders the reset before the release
        } else {
            while (ld_acquire_u32(bar + 1) == gen) __nanosleep(20);
        }
    }
    __syncthreads();
}

// Megakernel grid barrier, thread 0 of each block, after a __syncthreads that ordered the
// block's writes before it: one fire-and-forget release-add on a monotone arrival counter
// (zeroed before the launch), then acquire-polls until all blocks of this epoch arrived.
__device__ __forceinline__ void grid_arrive_wait(unsigned int *cnt, unsigned int target)
{
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    while ((int)(ld_acquire_u32(cnt) - target) < 0) {
#if NB_POLL_NS
        __nanosleep(NB_POLL_NS);
#endif
    }
}

// K values summed over the block in a fixed tree; result valid in thread 0 (sh: >= 32*K)
template <typename TS, int K>
__device__ __forceinline__ void block_reduce(TS (&v)[K], TS *sh)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int k = 0; k < K; k++) v[k] = warp_sum(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) sh[wid * K + k] = v[k];
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) v[k] = warp_sum(lane < nw ? sh[lane * K + k] : TS(0));
    }
}

// every block: sum part[i*K + k] over all G blocks in a fixed order (bit-identical in every
// block), one pass over the partials; result in every thread
template <typename TS, int K>
__device__ __forceinline__ void all_blocks_reduce(const double *part, int G, TS (&out)[K], TS *sh)
{
    __shared__ TS bc[K];
    TS s[K];
#pragma unroll
    for (int k = 0; k < K; k++) s[k] = 0;
    for (int i = threadIdx.x; i < G; i += blockDim.x) {
#pragma unroll
        for (int k = 0; k < K; k++) s[k] += (TS)__ldcg(part + (size_t)i * K + k);
    }
    block_reduce<TS, K>(s, sh);   // caller: sh free (a __syncthreads since its last use)
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) bc[k] = s[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; k++) out[k] = bc[k];
}

// Acc versions (dot-product accumulators, plain or Dot2 expansions): block tree, then every
// block merges all blocks' stored partials in a fixed order; TOT = merged values (TS)
template <int PREC, int K>
__device__ __forceinline__ void block_reduce_acc(Acc<PREC> (&v)[K], Acc<PREC> *sh)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int k = 0; k < K; k++)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k].merge(v[k].shfl_down(o));
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) sh[wid * K + k] = v[k];
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) {
            Acc<PREC> t = lane < nw ? sh[lane * K + k] : Acc<PREC>();
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t.merge(t.shfl_down(o));
            v[k] = t;
        }
    }
}
template <int PREC, int K>
__device__ __forceinline__ void all_blocks_reduce_acc(const double *part, int G, typename Pol<PREC>::TS (&out)[K],
                                                      Acc<PREC> *sh)
{
    using TS = typename Pol<PREC>::TS;
    __shared__ TS bc[K];
    Acc<PREC> s[K];
    // 16-byte loads (L2): one block's K*W doubles per thread, or two blocks' single values
    constexpr int W = Acc<PREC>::W, KW = K * W;
    if constexpr (KW % 2 == 0) {
        for (int i = threadIdx.x; i < G; i += blockDim.x) {
            double d[KW];
#pragma unroll
            for (int j = 0; j < KW / 2; j++) {
                const double2 t = __ldcg(reinterpret_cast<const double2 *>(part + (size_t)i * KW) + j);
                d[2 * j] = t.x;
                d[2 * j + 1] = t.y;
            }
#pragma unroll
            for (int k = 0; k < K; k++) s[k].merge(Acc<PREC>::from(d + k * W));
        }
    } else {
        for (int i2 = threadIdx.x; 2 * i2 < G; i2 += blockDim.x) {
            if (2 * i2 + 1 < G) {
                const double2 t = __ldcg(reinterpret_cast<const double2 *>(part) + i2);
                s[0].merge(Acc<PREC>::from(&t.x));
                s[0].merge(Acc<PREC>::from(&t.y));
            } else {
                s[0].merge(Acc<PREC>::load(part + 2 * (size_t)i2));
            }
        }
    }
    block_reduce_acc<PREC, K>(s, sh);   // caller: sh free (a __syncthreads since its last use)
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) bc[k] = s[k].value();
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; k++) out[k] = bc[k];
}

// every block: sum part[i*K + k] over all G blocks in a fixed order (same result everywhere);
// K values per block are summed in one pass (one L2 round trip)
template <typename TS, int K>
__device__ __forceinline__ void all_blocks_sum(const double *part, int G, TS (&out)[K], TS *sh)
{
    __syncthreads();
    all_blocks_reduce<TS, K>(part, G, out, sh);
    __syncthreads();
}
template <typename TS>
__device__ __forceinline__ TS all_blocks_sum1(const double *part, int G, TS *sh)
{
    TS o[1];
    all_blocks_sum<TS, 1>(part, G, o, sh);
    return o[0];
}

__device__ __forceinline__ unsigned int ld_acquire_sys_u32(const unsigned int *p)
{
    unsigned int v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Multi-rank reduction + barrier (VAR = 2), after block_reduce_acc left this block's K values
// in thread 0 of VALS: block partials -> rank-local grid barrier -> every block sums its rank's
// partials (fixed order, the same value in every block) -> block 0 pushes that rank partial into
// every rank's slot array and bumps every rank's flag -> every block waits until its rank's flag
// counts all R pushes and merges the R rank partials in rank order (bit-identical in every block
// of every rank).  One local barrier, one push, one flag wait per reduction.
// Every wait of the multi-rank solve is bounded: it gives up when its rank's abort word is set
// (another block or rank gave up) or after mr.timeout_ns, and then sets every rank's abort word.
// A dead or mismatched peer (not launched, other options) thus ends the solve with the
// `aborted` status instead of hanging every GPU (the host then requires a re-attach).
__device__ __forceinline__ bool mr_give_up(const MrArgs &mr, int me, unsigned long long t0)
{
    const unsigned int ab = mr.sys ? ld_acquire_sys_u32(mr.abrt[me]) : ld_acquire_u32(mr.abrt[me]);
    if (ab) return true;
    if (globaltimer() - t0 < mr.timeout_ns) return false;
    for (int q = 0; q < mr.nrank; q++) {
        if (mr.sys) asm volatile("st.release.sys.global.u32 [%0], 1;" ::"l"(mr.abrt[q]) : "memory");
        else asm volatile("st.release.gpu.global.u32 [%0], 1;" ::"l"(mr.abrt[q]) : "memory");
    }
    return true;
}

template <int PREC, int K>
__device__ __forceinline__ bool mr_reduce(const MegaArgs &A, const MrArgs &mr, int vr, int bid, int G,
                                          Acc<PREC> (&vals)[K], double *part, unsigned int &tgt, unsigned int ep,
                                          typename Pol<PREC>::TS (&tot)[K], Acc<PREC> *acc_sh)
{
    using TS = typename Pol<PREC>::TS;
    constexpr int W = Acc<PREC>::W;
    const int tid = threadIdx.x;
    const int R = mr.nrank, me = mr.rank0 + vr, par = ep & 1;
    __shared__ TS bc[K];
    __shared__ int gave_up;
    if (tid < 32) {
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < K; k++) vals[k].store(part + ((size_t)bid * K + k) * W);
            tgt += G;
            gave_up = 0;
            // rank-local grid barrier, bounded
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(A.bar) : "memory");
            const unsigned long long t0 = globaltimer();
            while ((int)(ld_acquire_u32(A.bar) - tgt) < 0) {
                if (mr_give_up(mr, me, t0)) { gave_up = 1; break; }
                __nanosleep(NB_POLL_NS);
            }
        }
        __syncwarp();
        // warp 0: the rank partial (fixed order, the same value in every block of the rank)
        Acc<PREC> s[K];
        for (int i = tid; i < G; i += 32) {
#pragma unroll
            for (int k = 0; k < K; k++) s[k].merge(Acc<PREC>::load(part + ((size_t)i * K + k) * W));
        }
#pragma unroll
        for (int k = 0; k < K; k++)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s[k].merge(s[k].shfl_down(o));
        if (tid == 0) {
            const unsigned int want = (unsigned int)R * ep;
            if (bid == 0) {
                for (int q = 0; q < R; q++) {
                    double *dst = mr.slot[q] + ((size_t)par * NB_MAX_RANKS + me) * 4;
#pragma unroll
                    for (int k = 0; k < K; k++) s[k].store(dst + k * W);
                }
            }
            // the release orders the slot stores before the flag bumps; system scope only when
            // ranks live on other GPUs (peer memory), GPU scope when they share this launch
            const unsigned long long t0 = globaltimer();
            if (mr.sys) {
                if (bid == 0)
                    for (int q = 0; q < R; q++)
                        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(mr.flag[q]) : "memory");
                while (!gave_up && (int)(ld_acquire_sys_u32(mr.flag[me]) - want) < 0)
                    if (mr_give_up(mr, me, t0)) gave_up = 1;
            } else {
                if (bid == 0)
                    for (int q = 0; q < R; q++)
                        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(mr.flag[q]) : "memory");
                while (!gave_up && (int)(ld_acquire_u32(mr.flag[me]) - want) < 0)
                    if (mr_give_up(mr, me, t0)) gave_up = 1;
            }
            Acc<PREC> t[K];
            const double *src = mr.slot[me] + (size_t)par * NB_MAX_RANKS * 4;
            for (int q = 0; q < R; q++) {
#pragma unroll
                for (int k = 0; k < K; k++)
                    t[k].merge(q == me ? s[k] : Acc<PREC>::load(src + (size_t)q * 4 + k * W));
            }
#pragma unroll
            for (int k = 0; k < K; k++) bc[k] = t[k].value();
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; k++) tot[k] = bc[k];
    return gave_up != 0;
}


// The solve of one slab (or the whole box) by the blocks [0, G) of its rank (bid = block index
// within the rank).  VAR = 0: the default options (Jacobi, x in the policy precision) folded at
// compile time; VAR = 1: the NEXT-3 variants (nb_cg_opts.precond / .x_fp64) as uniform runtime
// selects; VAR = 2: VAR 1 as one rank of a multi-rank z-slab solve (mr, vr: slab in the launch).
template <int PREC, int N, int FUSED, int VAR>
__global__ void NB_KERNEL_BOUNDS(AxCfg<typename Pol<PREC>::TV, N>)
k_cg_mega(const __grid_constant__ MegaArgs A, const __grid_constant__ DMat<typename Pol<PREC>::TV, N> D)
{
    static_assert(VAR == 0 || VAR == 1, "k_cg_mega: VAR 0 or 1 (VAR 2 is k_cg_mega_mr)");
    const MrArgs *const mr = nullptr;
    const int vr = 0, bid = 0, G = 0;
#include "nb_mega_body.inc"
}

// Multi-rank solve: nloc slabs in this launch, Gr blocks each (cooperative launch, so the
// slabs of one GPU that wait on one another are co-resident).
template <int PREC, int N>
__global__ void NB_KERNEL_BOUNDS(AxCfg<typename Pol<PREC>::TV, N>)
k_cg_mega_mr(const __grid_constant__ MultiArgs M, const __grid_constant__ DMat<typename Pol<PREC>::TV, N> D)
{
    constexpr int FUSED = 1, VAR = 2;
    const int vr = blockIdx.x / M.mr.Gr;
    if (vr >= M.mr.nloc) return;
    const MegaArgs &A = M.a[vr];
    const MrArgs *const mr = &M.mr;
    const int bid = blockIdx.x - vr * M.mr.Gr, G = M.mr.Gr;
#include "nb_mega_body.inc"
}

// Schwarz-preconditioned solve (NB_PC_SCHWARZ): the same body with the
// preconditioner phases of nb_schwarz.cuh between phase B and the next phase A (VAR = 3).
// FUSED = 0: the per-copy / ranked gather-scatter orders (CSR phase for Ax, ordered overlap sum).
template <int PREC, int N, int FUSED>
__global__ void NB_KERNEL_BOUNDS(AxCfg<typename Pol<PREC>::TV, N>)
k_cg_sw(const __grid_constant__ MegaArgs A, const __grid_constant__ DMat<typename Pol<PREC>::TV, N> D)
{
    constexpr int VAR = 3;
    const MrArgs *const mr = nullptr;
    const int vr = 0, bid = 0, G = 0;
    (void)vr; (void)bid; (void)G; (void)mr;
#include "nb_mega_body.inc"
}

// solveM alone (nb_precond_apply): z = M^-1 r with the Schwarz phases, one cooperative launch
template <int PREC, int N>
__global__ void NB_KERNEL_BOUNDS(AxCfg<typename Pol<PREC>::TV, N>)
k_sw_apply(const __grid_constant__ MegaArgs A)
{
    using TV = typename Pol<PREC>::TV;
    using TG = typename Pol<PREC>::TG;
    using C = AxCfg<TV, N>;
    extern __shared__ __align__(16) unsigned char smraw[];
    constexpr int EB = SwCfg<TV, N>::EB;
    __shared__ TG sw_red[8 * EB * 8], sw_w[28];
    sw_weights_init(sw_w);
    const int tid = threadIdx.x;
    unsigned int tgt = 0;

    const int64_t ng = ((int64_t)A.m.E + C::EPB - 1) / C::EPB;
    const int64_t g0 = split(ng, gridDim.x, blockIdx.x), g1 = split(ng, gridDim.x, blockIdx.x + 1);
    const int e0 = (int)min((int64_t)A.m.E, g0 * C::EPB), e1 = (int)min((int64_t)A.m.E, g1 * C::EPB);
    sw_local_range<PREC, N>(A.m, A.sw, (const TV *)A.r, e0, e1, smraw, sw_red, sw_w);
    __syncthreads();
    if (tid == 0) { tgt += gridDim.x; grid_arrive_wait(A.bar, tgt); }
    __syncthreads();
    if (A.sw.nv[0] > 0 && A.sw.nv[1] > 0 && A.sw.nv[2] > 0) {
        for (int pass = 0; pass <= 6; pass++) {
            sw_coarse<PREC>(A.m, A.sw, pass, (int64_t)blockIdx.x * blockDim.x + tid, (int64_t)gridDim.x * blockDim.x);
            __syncthreads();
            if (tid == 0) { tgt += gridDim.x; grid_arrive_wait(A.bar, tgt); }
            __syncthreads();
        }
    }
    Acc<PREC> rho;
    for (int64_t pid = (int64_t)e0 * C::N2 + tid; pid < (int64_t)e1 * C::N2; pid += blockDim.x)
        sw_gather_pencil<PREC, N>(A.m, A.sw, (const TV *)A.r, (TV *)A.z, pid, rho, sw_w);
}

// ===========================================================================
// standalone operator (nb_ax): w = A_L u (+ dssum-free mask), one persistent kernel
// ===========================================================================
template <int PREC, int N>
__global__ void NB_KERNEL_BOUNDS(AxCfg<typename Pol<PREC>::TV, N>)
k_ax(const MeshDev m, const __grid_constant__ DMat<typename Pol<PREC>::TV, N> D,
     const typename Pol<PREC>::TV *__restrict__ in, const typename Pol<PREC>::TV *__restrict__ g,
     typename Pol<PREC>::TV *__restrict__ w, int apply_mask)
{
    using TV = typename Pol<PREC>::TV;
    using C = AxCfg<TV, N>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int tid = threadIdx.x;
    const int el = tid / C::N2P;
    const int q = tid - el * C::N2P;
    const int qp = C::HALF ? q % C::N2 : q;   // pencil index (two threads per pencil: HALF)
    const int h = C::HALF ? q / C::N2 : 0;
    const int a = qp % N, b = qp / N;
    TV *S0 = reinterpret_cast<TV *>(smraw) + (el < C::EPB ? el : 0) * C::NARR * C::ESZ;
    const int64_t ngroups = ((int64_t)m.E + C::EPB - 1) / C::EPB;
    const int64_t g0 = split(ngroups, gridDim.x, blockIdx.x), g1 = split(ngroups, gridDim.x, blockIdx.x + 1);
    // u and g of the next group into L2 (measured at 32^3: mixed p9 323 -> 270 us, p11 587 -> 406 us,
    // fp64 p9 721 -> 634 us; fp64 p7 slower, 226 -> 240 us, so not there); with the staged geometric
    // factors (AxCfg::GSTAGE_AX: one TMA bulk copy per element, as in the solve's phase A) only u
    constexpr bool GS = C::GSTAGE_AX;
    constexpr bool PF = NB_L2PF_AX && !(sizeof(TV) == 8 && N == 8);
    constexpr int PFM = GS ? 2 : 3;
    __shared__ GStage gsh;
    TV *const gst = GS ? reinterpret_cast<TV *>(smraw + C::SMEM + (el < C::EPB ? el : 0) * C::GSB_AX) : nullptr;
    if constexpr (GS) {
        if (tid < 4) {
            mbar_init(&gsh.bar[tid], 1);
            gsh.par[tid] = 0;
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        const int e0 = (int)(g0 * C::EPB) + el;
        if (g0 < g1 && el < C::EPB && q == 0 && e0 < m.E) gstage_issue<TV, N>(g, e0, gst, &gsh.bar[el]);
    }
    if (PF) pf_group<TV, N, C::EPB, PFM>(g0, g1, m.E, g, in, nullptr, nullptr, 0);
#pragma unroll 1
    for (int64_t gr = g0; gr < g1; gr++) {
        if (PF) pf_group<TV, N, C::EPB, PFM>(gr + 1, g1, m.E, g, in, nullptr, nullptr, 0);
        const int e = (int)(gr * C::EPB) + el;
        const bool active = el < C::EPB && (C::N2P == C::N2 || C::HALF || q < C::N2) && e < m.E;
        const int en = (GS && gr + 1 < g1 && e + C::EPB < m.E) ? e + C::EPB : -1;
        // the handle may be a z-slab (global mask layers): SLAB = true
        if constexpr (C::HALF)
            ax_group_half<PREC, N, 0, true>(m, D, in, nullptr, nullptr, g, w, apply_mask != 0, TV(0), TV(0), e, active,
                                            a, b, h, S0);
        else
            ax_group<PREC, N, 0, true, GS>(m, D, in, nullptr, nullptr, g, w, apply_mask != 0, TV(0), TV(0), e, active, a, b,
                                           S0, nullptr, 0.0, gst, en, &gsh, el < C::EPB ? el : 0);
    }
}

// ===========================================================================
// launchers
// ===========================================================================
// Per-device cache of a kernel's residency (the function attributes it depends on are
// per device: set them and query once on every device that launches the kernel).
struct DevCache {
    int v[NB_MAX_DEVICES];
    DevCache() { for (int i = 0; i < NB_MAX_DEVICES; i++) v[i] = -1; }
    int &here()
    {
        int d = 0;
        cudaGetDevice(&d);
        return v[(d >= 0 && d < NB_MAX_DEVICES) ? d : 0];
    }
};

template <int PREC, int N>
static int ax_grid_t(const nb_handle *h)
{
    using TV = typename Pol<PREC>::TV;
    using C = AxCfg<TV, N>;
    static DevCache cache;
    int &occ = cache.here();
    if (occ < 0) {
        cudaFuncSetAttribute(k_ax<PREC, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_AX);
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_ax<PREC, N>, C::NT, C::SMEM_AX);
        occ = o > 0 ? o : 1;
    }
    const int64_t ngroups = (h->E + C::EPB - 1) / C::EPB;
    int64_t grid = (int64_t)h->sm_count * occ;
    if (grid > ngroups) grid = ngroups;
    return (int)(grid < 1 ? 1 : grid);
}

template <int PREC, int N>
static cudaError_t ax_launch_t(const nb_handle *h, const void *in, void *w, int apply_mask, cudaStream_t st)
{
    using TV = typename Pol<PREC>::TV;
    using C = AxCfg<TV, N>;
    const int grid = ax_grid_t<PREC, N>(h);
    const TV *g = (const TV *)(sizeof(TV) == 8 ? (const void *)h->g64 : (const void *)h->g32);
    k_ax<PREC, N><<<grid, C::NT, C::SMEM_AX, st>>>(h->md(), make_dmat<TV, N>(h->D), (const TV *)in, g, (TV *)w,
                                                apply_mask);
    return cudaGetLastError();
}

template <int PREC>
cudaError_t launch_ax_local(const nb_handle *h, const void *u, void *w, bool mask, cudaStream_t st)
{
    NB_DISPATCH_N(h->n, return (ax_launch_t<PREC, NN>(h, u, w, mask ? 1 : 0, st)))
}

#define NB_INSTANTIATE_CG(P)                                                                                  \
    extern template int grid_mega_var<P, 1>(const nb_handle *);                                               \
    extern template cudaError_t launch_cg_mega_var<P, 1>(const nb_handle *, const MegaArgs &, bool, cudaStream_t); \
    template cudaError_t launch_ax_local<P>(const nb_handle *, const void *, void *, bool, cudaStream_t);      \
    template int grid_mega<P>(const nb_handle *);                                                             \
    template int grid_mega_var<P, 0>(const nb_handle *);                                                      \
    template cudaError_t launch_cg_mega<P>(const nb_handle *, Workspace &, const void *, int, int, double,    \
                                           int, int, unsigned long long *, cudaStream_t, RankPart);           \
    template cudaError_t launch_cg_mega_var<P, 0>(const nb_handle *, const MegaArgs &, bool, cudaStream_t);
#define NB_INSTANTIATE_CG_SW(P) \
    template cudaError_t launch_cg_sw<P>(const nb_handle *, const MegaArgs &, int, bool, cudaStream_t);
// the variant (VAR = 1) megakernels: their own translation units (parallel build)
#define NB_INSTANTIATE_CG_VAR(P)                                                                              \
    template int grid_mega_var<P, 1>(const nb_handle *);                                                      \
    template cudaError_t launch_cg_mega_var<P, 1>(const nb_handle *, const MegaArgs &, bool, cudaStream_t);   \
    template void fill_mega_args<P>(const nb_handle *, Workspace &, const void *, int, int, double, int, int, \
                                    unsigned long long *, MegaArgs &);                                        \
    template int grid_mega_mr<P>(const nb_handle *);                                                          \
    template cudaError_t launch_cg_mr<P>(const nb_handle *, const MultiArgs &, cudaStream_t);

}  // namespace nb
