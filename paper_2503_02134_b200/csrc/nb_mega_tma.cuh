// nb_mega_tma.cuh -- the CG megakernel with every element-group operand streamed into shared
// memory by 1-D TMA bulk copies (cp.async.bulk + mbarrier, S-stage ring), the B200-native
// data path for even N (the bulk copies need 16-byte multiples: N^3 * sizeof(T) % 16 == 0).
//
// Same mathematics, same phases and same grid-barrier/redundant-reduction protocol as
// k_cg_mega (nb_cg.cuh); the difference is only where operands come from:
//   phase A: z, p_old, x and the six geometric factors of the group (one contiguous block per
//            array: the element-interleaved g layout makes a group's g one 6*EPB*N^3 run)
//            arrive in shared memory while the previous group is computed;
//   phase B: the group's w, r and dinv likewise; the x-neighbour copies inside the group come
//            from the staged w, y/z-neighbour copies from L2 (ld.global.cg).
// No global load is held in registers, so the register budget is set by the contractions.
#pragma once
#include "nb_cg.cuh"
#include "nb_tma.cuh"

#include <cstdlib>

namespace nb {

template <int PREC, int N> struct TmaCfg {
    using TV = typename Pol<PREC>::TV;
    using TJ = typename Pol<PREC>::TJ;
    using A = AxCfg<TV, N>;
    static constexpr int N2 = N * N, N3 = N * N * N;
    static constexpr int EPB = (128 / N2) >= 1 ? (128 / N2) : 1;   // elements per group
    static constexpr int NT = ((EPB * N2 + 31) / 32) * 32;
    static constexpr int S = 2;                                      // ring stages
    static constexpr int VB = EPB * N3 * (int)sizeof(TV);             // one vector, one group (bytes)
    static constexpr int STAGE = 9 * VB;                             // z, p, x, 6 g  (>= w, r, dinv)
    static constexpr int WORK = 3 * EPB * A::ESZ * (int)sizeof(TV);
    static constexpr int SMEM = S * STAGE + WORK;
    static constexpr bool OK = ((N3 * (int)sizeof(TV)) % 16 == 0) && (SMEM <= 200 * 1024) &&
                               (2 * VB + EPB * N3 * (int)sizeof(TJ) <= STAGE);
};

// phase A on one staged group (all threads).  sz/sp/sx/sg: this element slot in the stage.
// `release` runs in all threads right after the last read of the stage (post step-3 barrier).
template <int PREC, int N, int MODE, typename Rel>
__device__ __forceinline__ typename Pol<PREC>::TS
ax_group_tma(const MeshDev &m, const DMat<typename Pol<PREC>::TV, N> &D, const typename Pol<PREC>::TV *sz,
             const typename Pol<PREC>::TV *sp, const typename Pol<PREC>::TV *sx, const typename Pol<PREC>::TV *sg,
             typename Pol<PREC>::TV *__restrict__ pv, typename Pol<PREC>::TV *__restrict__ xv,
             typename Pol<PREC>::TV *__restrict__ w, typename Pol<PREC>::TV beta, typename Pol<PREC>::TV alpha,
             int e, bool active, int a, int b, typename Pol<PREC>::TV *__restrict__ S0, Rel release)
{
    using TV = typename Pol<PREC>::TV;
    using TS = typename Pol<PREC>::TS;
    using C = AxCfg<TV, N>;
    constexpr int V = VecW<TV, N>::V;
    TV *A1 = S0 + C::ESZ;
    TV *A2 = A1 + C::ESZ;
    const int q = a + N * b;
    const int rp = N * a + C::P * b;
    const int sp_ = a + C::P * b;
    const int tp = a + N * b;
    const size_t gbase = (size_t)e * C::N3 + (size_t)N * q;

    // ---- 1. p = z + beta p_old (add2s1), x += alpha_prev p_old (deferred add2s2)
    if (active) {
        TV u[N], xx[N];
        {
            TV zz[N], po[N];
            ld_pencil<TV, N>(sz + N * q, zz);
            ld_pencil<TV, N>(sp + N * q, po);
            ld_pencil<TV, N>(sx + N * q, xx);
#pragma unroll
            for (int i = 0; i < N; i++) {
                u[i] = fma(beta, po[i], zz[i]);
                xx[i] = fma(alpha, po[i], xx[i]);
            }
        }
        st_pencil<TV, N>(pv + gbase, u);
        st_pencil<TV, N, LD_CS>(xv + gbase, xx);
        st_pencil<TV, N>(S0 + rp, u);
    }
    __syncthreads();
    // ---- 2. us, ut
    if (active) {
        TV v[N], o[N];
#pragma unroll
        for (int j = 0; j < N; j++) v[j] = S0[sp_ + N * j];
        contract<TV, N>(D, v, o);
#pragma unroll
        for (int j = 0; j < N; j++) A1[sp_ + N * j] = o[j];
#pragma unroll
        for (int k = 0; k < N; k++) v[k] = S0[tp + C::P * k];
        contract<TV, N>(D, v, o);
#pragma unroll
        for (int k = 0; k < N; k++) A2[tp + C::P * k] = o[k];
    }
    __syncthreads();
    // ---- 3. ur; geometric factors; r-part of local_grad3_t; pap in energy form (MODE 1)
    TS acc = 0;
    if (active) {
        TV wr[N];
        {
            TV v[N];
            ld_pencil<TV, N>(S0 + rp, v);
            contract<TV, N>(D, v, wr);   // ur, overwritten by wr
        }
        const TV *ge = sg + N * q;
#pragma unroll
        for (int c = 0; c < N / V; c++) {
            TV g1[V], g2[V], g3[V], g4[V], g5[V], g6[V], us[V], ut[V], ws[V], wt[V];
            ld_chunk<TV, V>(ge + 0 * C::N3 + c * V, g1);
            ld_chunk<TV, V>(ge + 1 * C::N3 + c * V, g2);
            ld_chunk<TV, V>(ge + 2 * C::N3 + c * V, g3);
            ld_chunk<TV, V>(ge + 3 * C::N3 + c * V, g4);
            ld_chunk<TV, V>(ge + 4 * C::N3 + c * V, g5);
            ld_chunk<TV, V>(ge + 5 * C::N3 + c * V, g6);
            ld_chunk<TV, V>(A1 + rp + c * V, us);
            ld_chunk<TV, V>(A2 + rp + c * V, ut);
#pragma unroll
            for (int t = 0; t < V; t++) {
                const TV r_ = wr[c * V + t];
                const TV wr_ = fma(g3[t], ut[t], fma(g2[t], us[t], g1[t] * r_));
                ws[t] = fma(g5[t], ut[t], fma(g4[t], us[t], g2[t] * r_));
                wt[t] = fma(g6[t], ut[t], fma(g5[t], us[t], g3[t] * r_));
                if (MODE == 1) acc += ((TS)r_ * (TS)wr_ + (TS)us[t] * (TS)ws[t]) + (TS)ut[t] * (TS)wt[t];
                wr[c * V + t] = wr_;
            }
            st_chunk<TV, V>(A1 + rp + c * V, ws);
            st_chunk<TV, V>(A2 + rp + c * V, wt);
        }
        TV o[N];
        contract_t<TV, N>(D, wr, o);
        st_pencil<TV, N>(S0 + rp, o);
    }
    __syncthreads();
    release();   // the stage is no longer read: refill it
    // ---- 4. s- and t-parts of local_grad3_t
    if (active) {
        TV v[N], o[N];
#pragma unroll
        for (int j = 0; j < N; j++) v[j] = A1[sp_ + N * j];
        contract_t<TV, N>(D, v, o);
#pragma unroll
        for (int j = 0; j < N; j++) A1[sp_ + N * j] = o[j];
#pragma unroll
        for (int k = 0; k < N; k++) v[k] = A2[tp + C::P * k];
        contract_t<TV, N>(D, v, o);
#pragma unroll
        for (int k = 0; k < N; k++) A2[tp + C::P * k] = o[k];
    }
    __syncthreads();
    // ---- 5. w = (w_r + w_s) + w_t, mask, store; MODE 2: unshared part of pap
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
        const ElemPos P = elem_pos<false>(m, e);
        const bool mjk = axis_bnd(a, N, P.ey, m.nely) || axis_bnd(b, N, P.ez, m.nelz);
#pragma unroll
        for (int i = 0; i < N; i++)
            if (mjk || axis_bnd(i, N, P.ex, m.nelx)) out[i] = TV(0);
        if (MODE == 2) {
            const bool sjk = axis_mult(a, N, P.ey, m.nely) * axis_mult(b, N, P.ez, m.nelz) > 1;
            TV pp[N];
            ld_pencil<TV, N>(pv + gbase, pp);   // written by this thread in step 1
#pragma unroll
            for (int i = 0; i < N; i++)
                if (!sjk && axis_mult(i, N, P.ex, m.nelx) == 1) acc += (TS)out[i] * (TS)pp[i];
        }
        st_pencil<TV, N>(w + gbase, out);
    }
    return acc;
}

// phase B on one staged group (all threads): sw/sr/sd are the group's w, r, dinv in the stage.
template <int PREC, int N, int GATHER, typename Rel>
__device__ __forceinline__ void upd_group_tma(const MeshDev &m, const typename Pol<PREC>::TV *__restrict__ w,
                                              typename Pol<PREC>::TV *__restrict__ r,
                                              typename Pol<PREC>::TV *__restrict__ z, typename Pol<PREC>::TV alpha,
                                              int e, bool active, int el, int a, int b, int e_end,
                                              const typename Pol<PREC>::TV *sw, const typename Pol<PREC>::TV *sr,
                                              const typename Pol<PREC>::TJ *sd, typename Pol<PREC>::TS &rtr,
                                              typename Pol<PREC>::TS &rho, Rel release)
{
    using TV = typename Pol<PREC>::TV;
    using TJ = typename Pol<PREC>::TJ;
    using TS = typename Pol<PREC>::TS;
    using T = TmaCfg<PREC, N>;
    constexpr int N2 = N * N, N3 = N * N * N;
    const int q = a + N * b;
    const int off = el * N3 + q * N;
    if (active) {
        const size_t base = ((size_t)e * N2 + q) * N;
        const ElemPos P = elem_pos<false>(m, e);
        TV ww[N];
        ld_pencil<TV, N>(sw + off, ww);
        if (GATHER) {
            TV ol = 0, orr = 0;
            if (P.ex > 0) ol = el > 0 ? sw[off - N3 + (N - 1)] : __ldcg(w + base - N3 + (N - 1));
            if (P.ex < m.nelx - 1) orr = (el + 1 < T::EPB && e + 1 < e_end) ? sw[off + N3] : __ldcg(w + base + N3);
            gather_pencil<PREC, N>(m, w, e, P, a, b, ww, ol, orr);
        }
        TV rr[N], zz[N];
        TJ dd[N];
        ld_pencil<TV, N>(sr + off, rr);
        ld_pencil<TJ, N>(sd + off, dd);
        const int mjk = axis_mult(a, N, P.ey, m.nely) * axis_mult(b, N, P.ez, m.nelz);
#pragma unroll
        for (int i = 0; i < N; i++) {
            rr[i] = fma(-alpha, ww[i], rr[i]);                   // add2s2(r, w, -alpha)
            zz[i] = (TV)((TJ)rr[i] * dd[i]);                     // solveM
            const TS c = (TS)1 / (TS)(mjk * axis_mult(i, N, P.ex, m.nelx));
            const TS rs = (TS)rr[i];
            rtr += (rs * c) * rs;                                // glsc3(r, c, r)
            rho += (rs * c) * (TS)zz[i];                         // glsc3(r, c, z)
        }
        st_pencil<TV, N>(r + base, rr);
        st_pencil<TV, N>(z + base, zz);
    }
    __syncthreads();
    release();
}

template <int PREC, int N, int FUSED>
__global__ void __launch_bounds__(TmaCfg<PREC, N>::NT)
k_cg_mega_tma(const __grid_constant__ MegaArgs A, const __grid_constant__ DMat<typename Pol<PREC>::TV, N> D)
{
    using TV = typename Pol<PREC>::TV;
    using TJ = typename Pol<PREC>::TJ;
    using TS = typename Pol<PREC>::TS;
    using T = TmaCfg<PREC, N>;
    using C = AxCfg<TV, N>;
    extern __shared__ __align__(16) unsigned char smraw[];
    __shared__ TS sh[32];
    __shared__ __align__(8) uint64_t bars[T::S];
    struct State {
        TS rtr0, rho, rtr, beta, alpha, pap;
        int it, status, pending, done;
    };
    __shared__ State st;
    const int tid = threadIdx.x;
    const bool t0 = (blockIdx.x == 0 && tid == 0);
    const int64_t ngroups = ((int64_t)A.m.E + T::EPB - 1) / T::EPB;
    const int64_t g0 = split(ngroups, gridDim.x, blockIdx.x), g1 = split(ngroups, gridDim.x, blockIdx.x + 1);
    const int ngr = (int)(g1 - g0);
    const int el = tid / T::N2;
    const int qq = tid - el * T::N2;
    const int a = qq % N, b = qq / N;
    unsigned char *stage0 = smraw;
    TV *S0 = reinterpret_cast<TV *>(smraw + T::S * T::STAGE) + (el < T::EPB ? el : 0) * 3 * C::ESZ;
    uint32_t ph = 0;   // per-stage mbarrier parity bits (every thread waits on every group)

    if (tid == 0) {
        for (int s = 0; s < T::S; s++) mbar_init(&bars[s], 1);
        mbar_fence_init();
    }
    __syncthreads();

    // producers (thread 0): all operands of one group into stage s
    auto issueA = [&](int k) {
        const int s = k % T::S;
        const int64_t e0 = (g0 + k) * T::EPB;
        const int ne = (int)min((int64_t)T::EPB, (int64_t)A.m.E - e0);
        const uint32_t vb = (uint32_t)ne * T::N3 * sizeof(TV);
        unsigned char *stg = stage0 + (size_t)s * T::STAGE;
        fence_proxy_async();
        mbar_arrive_expect_tx(&bars[s], 9 * vb);
        bulk_g2s(stg, (const TV *)A.z + e0 * T::N3, vb, &bars[s]);
        bulk_g2s(stg + T::VB, (const TV *)A.p + e0 * T::N3, vb, &bars[s]);
        bulk_g2s(stg + 2 * T::VB, (const TV *)A.x + e0 * T::N3, vb, &bars[s]);
        bulk_g2s(stg + 3 * T::VB, (const TV *)A.g + e0 * 6 * T::N3, 6 * vb, &bars[s]);
    };
    auto issueB = [&](int k) {
        const int s = k % T::S;
        const int64_t e0 = (g0 + k) * T::EPB;
        const int ne = (int)min((int64_t)T::EPB, (int64_t)A.m.E - e0);
        const uint32_t vb = (uint32_t)ne * T::N3 * sizeof(TV);
        const uint32_t jb = (uint32_t)ne * T::N3 * sizeof(TJ);
        unsigned char *stg = stage0 + (size_t)s * T::STAGE;
        fence_proxy_async();
        mbar_arrive_expect_tx(&bars[s], 2 * vb + jb);
        bulk_g2s(stg, (const TV *)A.w + e0 * T::N3, vb, &bars[s]);
        bulk_g2s(stg + T::VB, (const TV *)A.r + e0 * T::N3, vb, &bars[s]);
        bulk_g2s(stg + 2 * T::VB, (const TJ *)A.dinv + e0 * T::N3, jb, &bars[s]);
    };
    auto wait_stage = [&](int k) {
        const int s = k % T::S;
        mbar_wait(&bars[s], (ph >> s) & 1u);
        ph ^= 1u << s;
    };

    // ---- prologue: r = b, x = p = 0, z = M^-1 r; rtr0, rho_1 (plain loads, once per solve)
    {
        const int64_t p0 = min((int64_t)A.m.E, g0 * T::EPB) * T::N2;
        const int64_t p1 = min((int64_t)A.m.E, g1 * T::EPB) * T::N2;
        Acc<PREC> artr, arho;
#pragma unroll 1
        for (int64_t pid = p0 + tid; pid < p1; pid += blockDim.x)
            init_pencil<PREC, N>(A.m, (const TV *)A.b, (TV *)A.x, (TV *)A.p, (TV *)A.r, (TV *)A.z,
                                 (const TJ *)A.dinv, pid, artr, arho);
        fence_proxy_async();   // these writes are read by bulk copies after the barrier
        const TS rtr = block_sum<TS>(artr.value(), sh);
        const TS rho = block_sum<TS>(arho.value(), sh);
        if (tid == 0) { A.partB[2 * blockIdx.x] = (double)rtr; A.partB[2 * blockIdx.x + 1] = (double)rho; }
    }
    grid_barrier(A.bar);
    if (t0 && A.tim) A.tim[0] = globaltimer();
    {
        TS tot2[2];
        all_blocks_sum<TS, 2>(A.partB, gridDim.x, tot2, sh);
        const TS rtr0 = tot2[0], rho = tot2[1];
        if (tid == 0) {
            st.rtr0 = rtr0; st.rho = rho; st.rtr = rtr0; st.beta = 0; st.alpha = 0; st.pap = 0;
            st.it = 0; st.status = NB_MAXITER; st.pending = 0; st.done = 0;
            if (rtr0 == (TS)0) { st.status = NB_CONVERGED; st.done = 1; }
            else if (!isfinite((double)rtr0)) { st.status = NB_BROKEDOWN; st.done = 1; }
            else if (A.max_iter <= 0) { st.status = NB_MAXITER; st.done = 1; }
            if (blockIdx.x == 0) A.hist[0] = rtr0 == (TS)0 ? 0.0 : 1.0;
        }
        __syncthreads();
    }

#pragma unroll 1
    while (!st.done) {
        // ---- phase A
        {
            if (tid == 0)
                for (int k = 0; k < T::S && k < ngr; k++) issueA(k);
            TS acc = 0;
            const TV bv = (TV)st.beta, av = st.pending ? (TV)st.alpha : TV(0);
#pragma unroll 1
            for (int k = 0; k < ngr; k++) {
                wait_stage(k);
                const TV *stg = reinterpret_cast<const TV *>(stage0 + (size_t)(k % T::S) * T::STAGE);
                const int slot = el < T::EPB ? el : 0;
                const int e = (int)((g0 + k) * T::EPB) + el;
                const bool active = el < T::EPB && e < A.m.E;
                acc += ax_group_tma<PREC, N, FUSED ? 1 : 2>(
                    A.m, D, stg + slot * T::N3, stg + T::EPB * T::N3 + slot * T::N3,
                    stg + 2 * T::EPB * T::N3 + slot * T::N3, stg + 3 * T::EPB * T::N3 + slot * 6 * T::N3,
                    (TV *)A.p, (TV *)A.x, (TV *)A.w, bv, av, e, active, a, b, S0, [&]() {
                        if (tid == 0 && k + T::S < ngr) issueA(k + T::S);
                    });
            }
            fence_proxy_async();   // p, x, w are read by bulk copies after the barrier
            acc = block_sum<TS>(acc, sh);
            if (tid == 0) A.partA[blockIdx.x] = (double)acc;
        }
        grid_barrier(A.bar);
        if (t0 && A.tim) A.tim[3 * st.it + 1] = globaltimer();
        TS pap = all_blocks_sum1<TS>(A.partA, gridDim.x, sh);
        if (!FUSED) {
            const int64_t s0 = split(A.nseg, gridDim.x, blockIdx.x), s1 = split(A.nseg, gridDim.x, blockIdx.x + 1);
            TS acc2 = 0;
            for (int64_t s = s0 + tid; s < s1; s += blockDim.x) {
                if (A.order == NB_GS_CONSISTENT)
                    acc2 += gs_segment<PREC, NB_GS_CONSISTENT, 1, TV, typename Pol<PREC>::TG, LD_CG>(
                        (int32_t)s, A.gs_off, A.gs_idx, (TV *)A.w, (const TV *)A.p).value();
                else
                    acc2 += gs_segment<PREC, NB_GS_PER_COPY, 1, TV, typename Pol<PREC>::TG, LD_CG>(
                        (int32_t)s, A.gs_off, A.gs_idx, (TV *)A.w, (const TV *)A.p).value();
            }
            fence_proxy_async();   // w is read by bulk copies after the barrier
            acc2 = block_sum<TS>(acc2, sh);
            if (tid == 0) A.partS[blockIdx.x] = (double)acc2;
            grid_barrier(A.bar);
            pap = pap + all_blocks_sum1<TS>(A.partS, gridDim.x, sh);
        }
        if (t0 && A.tim) A.tim[3 * st.it + 2] = globaltimer();
        if (tid == 0) {
            st.pap = pap;
            if (!(pap > (TS)0) || !isfinite((double)pap) || !isfinite((double)st.rho)) {
                st.status = NB_BROKEDOWN;
                st.pending = 0;
                st.done = 2;
            } else {
                st.alpha = st.rho / pap;
                st.pending = 1;
            }
        }
        __syncthreads();
        if (st.done) break;
        // ---- phase B
        {
            if (tid == 0)
                for (int k = 0; k < T::S && k < ngr; k++) issueB(k);
            TS prtr = 0, prho = 0;
            const TV av = (TV)st.alpha;
            const int e_end = (int)min((int64_t)A.m.E, g1 * T::EPB);
#pragma unroll 1
            for (int k = 0; k < ngr; k++) {
                wait_stage(k);
                const unsigned char *stg = stage0 + (size_t)(k % T::S) * T::STAGE;
                const int e = (int)((g0 + k) * T::EPB) + el;
                const bool active = el < T::EPB && e < e_end;
                upd_group_tma<PREC, N, FUSED>(
                    A.m, (const TV *)A.w, (TV *)A.r, (TV *)A.z, av, e, active, el, a, b, e_end,
                    reinterpret_cast<const TV *>(stg), reinterpret_cast<const TV *>(stg + T::VB),
                    reinterpret_cast<const TJ *>(stg + 2 * T::VB), prtr, prho, [&]() {
                        if (tid == 0 && k + T::S < ngr) issueB(k + T::S);
                    });
            }
            fence_proxy_async();   // r, z are read by bulk copies after the barrier
            prtr = block_sum<TS>(prtr, sh);
            prho = block_sum<TS>(prho, sh);
            if (tid == 0) { A.partB[2 * blockIdx.x] = (double)prtr; A.partB[2 * blockIdx.x + 1] = (double)prho; }
        }
        grid_barrier(A.bar);
        {
            TS tot2[2];
            all_blocks_sum<TS, 2>(A.partB, gridDim.x, tot2, sh);
            const TS rtr = tot2[0], rho_new = tot2[1];
            if (tid == 0) {
                const int it = st.it + 1;
                const double res = sqrt((double)rtr / (double)st.rtr0);
                if (blockIdx.x == 0) {
                    A.hist[it] = res;
                    if (A.tim) A.tim[3 * it] = globaltimer();
                }
                if (!isfinite((double)rtr) || !isfinite((double)rho_new)) { st.status = NB_BROKEDOWN; st.done = 1; }
                else if (res <= A.rtol || rtr == (TS)0) { st.status = NB_CONVERGED; st.done = 1; }
                else if (it >= A.max_iter) { st.status = NB_MAXITER; st.done = 1; }
                st.beta = rho_new / st.rho;
                st.rho = rho_new;
                st.rtr = rtr;
                st.it = it;
            }
            __syncthreads();
        }
    }
    // ---- epilogue: the deferred x += alpha p of the last iteration (own elements)
    if (st.pending) {
        const TV av = (TV)st.alpha;
        const int64_t l0 = min((int64_t)A.m.E, g0 * T::EPB) * T::N3;
        const int64_t l1 = min((int64_t)A.m.E, g1 * T::EPB) * T::N3;
        TV *x = (TV *)A.x;
        const TV *pv = (const TV *)A.p;
        for (int64_t l = l0 + tid; l < l1; l += blockDim.x) x[l] = fma(av, pv[l], x[l]);
    }
    if (t0) {
        Scal *s = A.scal;
        s->rho = (double)st.rho; s->beta = (double)st.beta; s->alpha = (double)st.alpha; s->pap = (double)st.pap;
        s->rtr = (double)st.rtr; s->rtr0 = (double)st.rtr0; s->iter = st.it; s->status = st.status; s->done = 1;
        s->pending = 0;
    }
}

// ---- megakernel launchers: the TMA-staged variant where its bulk copies apply (even N and
// the 2-stage ring fits in shared memory), the register-staged one otherwise ----
template <int PREC, int N, int FUSED, bool TMA, int VAR>
struct MegaSel {
    static const void *fn()
    {
        if constexpr (TMA) return (const void *)k_cg_mega_tma<PREC, N, FUSED>;
        else return (const void *)k_cg_mega<PREC, N, FUSED, VAR>;
    }
    static int nt() { return TMA ? TmaCfg<PREC, N>::NT : AxCfg<typename Pol<PREC>::TV, N>::NT; }
    static int smem() { return TMA ? TmaCfg<PREC, N>::SMEM : AxCfg<typename Pol<PREC>::TV, N>::SMEM; }
};

// The TMA-staged variant measured slower than the register-streamed one on B200 (DESIGN.md
// §6): compiled only with -DNB_WITH_TMA=1 and then selected by NB_MEGA_TMA=1 (default options).
#ifndef NB_WITH_TMA
#define NB_WITH_TMA 0
#endif
template <int PREC, int N, int VAR>
constexpr bool use_tma()
{
    return NB_WITH_TMA && VAR == 0 && PREC != NB_FP32_DOT2 && TmaCfg<PREC, N>::OK;
}

static bool env_no_tma()
{
    static int v = -1;
    if (v < 0) {
        const char *s = std::getenv("NB_MEGA_TMA");
        v = (s && s[0] == '1') ? 0 : 1;
    }
    return v == 1;
}

// Shared-memory carve-out: just what the resident blocks need, the rest of the 256 KB stays L1
// (phase B's neighbour-copy loads hit in L1).  NB_CARVEOUT=0 leaves the driver's choice.
static void set_carveout(const void *fn, int occ, int smem)
{
    static int mode = -1;
    if (mode < 0) {
        const char *s = std::getenv("NB_CARVEOUT");
        mode = (s && s[0] == '0') ? 0 : 1;
    }
    if (!mode) return;
    const int need = occ * (smem + 1024) + 1024;                   // + per-block reservation
    int pct = (int)((100LL * need + 228 * 1024 - 1) / (228 * 1024));
    if (pct > 100) pct = 100;
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

template <int PREC, int N, int FUSED, bool TMA, int VAR>
static int mega_grid_t(const nb_handle *h)
{
    using Sel = MegaSel<PREC, N, FUSED, TMA, VAR>;
    static int occ = -1;
    if (occ < 0) {
        cudaFuncSetAttribute(Sel::fn(), cudaFuncAttributeMaxDynamicSharedMemorySize, Sel::smem());
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, Sel::fn(), Sel::nt(), Sel::smem());
        occ = o > 0 ? o : 1;
        set_carveout(Sel::fn(), occ, Sel::smem());
    }
    return h->sm_count * occ;
}

template <int PREC, int N, int FUSED, int VAR>
static int mega_grid_sel(const nb_handle *h)
{
    if (use_tma<PREC, N, VAR>() && !env_no_tma()) return mega_grid_t<PREC, N, FUSED, use_tma<PREC, N, VAR>(), VAR>(h);
    return mega_grid_t<PREC, N, FUSED, false, VAR>(h);
}

template <int PREC, int VAR>
int grid_mega_var(const nb_handle *h)
{
    NB_DISPATCH_N(h->n, return (mega_grid_sel<PREC, NN, 1, VAR>(h) > mega_grid_sel<PREC, NN, 0, VAR>(h)
                                    ? mega_grid_sel<PREC, NN, 1, VAR>(h)
                                    : mega_grid_sel<PREC, NN, 0, VAR>(h)))
}

// grid size of every megakernel of the policy (sizes the per-block partials)
template <int PREC>
int grid_mega(const nb_handle *h)
{
    const int g0 = grid_mega_var<PREC, 0>(h), g1 = grid_mega_var<PREC, 1>(h);
    return g0 > g1 ? g0 : g1;
}

template <int PREC, int N, int FUSED, int VAR>
static cudaError_t mega_launch_t(const nb_handle *h, const MegaArgs &args, cudaStream_t st)
{
    using TV = typename Pol<PREC>::TV;
    const bool tma = use_tma<PREC, N, VAR>() && !env_no_tma();
    DMat<TV, N> D = make_dmat<TV, N>(h->D);
    void *params[2] = {(void *)&args, (void *)&D};
    if (tma) {
        using Sel = MegaSel<PREC, N, FUSED, use_tma<PREC, N, VAR>(), VAR>;
        const int grid = mega_grid_t<PREC, N, FUSED, use_tma<PREC, N, VAR>(), VAR>(h);
        return cudaLaunchCooperativeKernel(Sel::fn(), dim3(grid), dim3(Sel::nt()), params, (size_t)Sel::smem(), st);
    }
    using Sel = MegaSel<PREC, N, FUSED, false, VAR>;
    const int grid = mega_grid_t<PREC, N, FUSED, false, VAR>(h);
    return cudaLaunchCooperativeKernel(Sel::fn(), dim3(grid), dim3(Sel::nt()), params, (size_t)Sel::smem(), st);
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
    A.x = A.x64 ? (void *)ws.xd : ws.x; A.p = ws.p; A.r = ws.r; A.w = ws.w;
    A.z = precond == NB_PC_IDENTITY ? ws.r : ws.z;   // identity: z aliases r (never stored)
    A.g = (sizeof(typename Pol<PREC>::TV) == 8) ? (const void *)h->g64 : (const void *)h->g32;
    A.dinv = (sizeof(typename Pol<PREC>::TJ) == 4 || precond == NB_PC_JACOBI_F32) ? (const void *)h->dinv32
                                                                                  : (const void *)h->dinv64;
    A.gs_off = h->gs_off; A.gs_idx = h->gs_idx; A.nseg = (int32_t)h->nseg;
    A.order = order; A.max_iter = max_iter; A.rtol = rtol;
    A.hist = ws.hist; A.tim = tim;
    // per-block partials: W doubles per accumulator (2 for the Dot2 expansions)
    const size_t W = (size_t)Acc<PREC>::W;
    A.partA = ws.red.part; A.partS = ws.red.part + W * ws.mega_G; A.partB = ws.red.part + 2 * W * ws.mega_G;
    A.bar = ws.bar;
    A.scal = ws.scal;
    A.wlo = ws.peer.wlo;
    A.whi = ws.peer.whi;
}

template <int PREC>
cudaError_t launch_cg_mega(const nb_handle *h, Workspace &ws, const void *b, int order, int max_iter, double rtol,
                           int precond, int x64, unsigned long long *tim, cudaStream_t st)
{
    MegaArgs A;
    fill_mega_args<PREC>(h, ws, b, order, max_iter, rtol, precond, x64, tim, A);
    A.wlo = A.whi = nullptr;
    const bool fused = order == NB_GS_CONSISTENT && !h->cg_csr;
    cudaError_t e = cudaMemsetAsync(ws.bar, 0, 2 * sizeof(unsigned int), st);   // barrier epoch 0
    if (e != cudaSuccess) return e;
    const bool var = precond != NB_PC_JACOBI || A.x64;
    return var ? launch_cg_mega_var<PREC, 1>(h, A, fused, st) : launch_cg_mega_var<PREC, 0>(h, A, fused, st);
}

// ---- multi-rank (z-slab) megakernel: consistent order, runtime options ----
template <int PREC, int N>
static int mr_occupancy()
{
    using C = AxCfg<typename Pol<PREC>::TV, N>;
    static int occ = -1;
    if (occ < 0) {
        const void *fn = (const void *)k_cg_mega_mr<PREC, N>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, C::NT, C::SMEM);
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
    DMat<TV, N> D = make_dmat<TV, N>(h->D);
    void *params[2] = {(void *)&M, (void *)&D};
    (void)mr_occupancy<PREC, N>();
    return cudaLaunchCooperativeKernel((const void *)k_cg_mega_mr<PREC, N>, dim3(M.mr.nloc * M.mr.Gr), dim3(C::NT),
                                       params, (size_t)C::SMEM, st);
}

template <int PREC>
cudaError_t launch_cg_mr(const nb_handle *h0, const MultiArgs &M, cudaStream_t st)
{
    NB_DISPATCH_N(h0->n, return (mr_launch_t<PREC, NN>(h0, M, st)))
}

}  // namespace nb
