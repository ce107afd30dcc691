// nb_sw_setup.cu -- host setup of the two-level Schwarz preconditioner (NB_PC_SCHWARZ, SURVEY.md
// §8(f) NEXT-4; reading 28): the 1-D fast-diagonalisation tables of the element boxes
// extended by one GLL layer, the overlap counts behind the weights 1/sqrt(count), the coarse
// (interior element vertex) tables, and the per-policy scratch.
//
// Per axis a with nel elements of length h = 1/nel and lattice points I = 0 .. nel p:
//   the assembled 1-D GLL stiffness A1 = sum_e (2/h) Ahat_e and mass B1 = sum_e (h/2) w_e
//   (Ahat[i][j] = sum_q w_q D[q][i] D[q][j]); the extended index set of element position ex is
//   [ex p - 1, ex p + p + 1] clipped to the unknowns [1, nel p - 1]; its principal blocks of A1, B1
//   give the generalised eigenproblem A S = B S Lambda (S^T B S = I), solved by cuSOLVER's
//   sygvd (setup only).  The blocks depend on the set's offsets relative to the element only, so
//   element positions share "cases".  Coarse: the trilinear hats of the interior vertices,
//   A0 = Phi^T A1 Phi and B0 = Phi^T B1 Phi assembled from element 2 x 2 blocks, same solver.
// Tables are stored in the extended-box frame t = lattice - (ex p - 1), t in [0, p + 3): rows of
// points outside the set are zero, padded modes have lambda = 1 (their coefficients are zero).
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cmath>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "nb.h"
#include "nb_internal.h"

namespace nb {

struct SwState {
    bool tables = false;
    int nv[3] = {0, 0, 0};
    uint8_t *cs[3] = {}, *cnt[3] = {};
    double *S64[3] = {}, *lam[3] = {}, *S064[3] = {}, *lam0[3] = {};
    float *S32[3] = {}, *S032[3] = {};
    double *phL = nullptr, *phR = nullptr;
    void *zext[4] = {}, *cpart[4] = {}, *c0[4] = {}, *c1[4] = {};
};

namespace {

// generalised symmetric-definite eigenproblems A_k x = lambda B_k x (n_k x n_k, row-major and
// symmetric) on the device with cuSOLVER: eigenvectors (column k = mode k, B-orthonormal) and
// eigenvalues (ascending) returned in S (row-major: S[i n + k] = component i of mode k), lam.
bool gen_eig_batch(std::vector<std::vector<double>> &A, std::vector<std::vector<double>> &B, const std::vector<int> &n,
                   std::vector<std::vector<double>> &S, std::vector<std::vector<double>> &lam)
{
    cusolverDnHandle_t hs = nullptr;
    if (cusolverDnCreate(&hs) != CUSOLVER_STATUS_SUCCESS) return false;
    bool ok = true;
    int nmax = 1;
    for (int v : n) nmax = v > nmax ? v : nmax;
    double *dA = nullptr, *dB = nullptr, *dW = nullptr, *work = nullptr;
    int *info = nullptr;
    int lwork = 0;
    ok = cudaMalloc(&dA, sizeof(double) * nmax * nmax) == cudaSuccess && cudaMalloc(&dB, sizeof(double) * nmax * nmax) == cudaSuccess &&
         cudaMalloc(&dW, sizeof(double) * nmax) == cudaSuccess && cudaMalloc(&info, sizeof(int)) == cudaSuccess;
    if (ok && cusolverDnDsygvd_bufferSize(hs, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, nmax,
                                          dA, nmax, dB, nmax, dW, &lwork) != CUSOLVER_STATUS_SUCCESS)
        ok = false;
    if (ok && cudaMalloc(&work, sizeof(double) * (lwork > 0 ? lwork : 1)) != cudaSuccess) ok = false;
    S.assign(n.size(), {});
    lam.assign(n.size(), {});
    for (size_t c = 0; ok && c < n.size(); c++) {
        const int m = n[c];
        if (m <= 0) continue;
        int lw = 0;
        ok = cudaMemcpy(dA, A[c].data(), sizeof(double) * m * m, cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(dB, B[c].data(), sizeof(double) * m * m, cudaMemcpyHostToDevice) == cudaSuccess &&
             cusolverDnDsygvd_bufferSize(hs, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, dA,
                                         m, dB, m, dW, &lw) == CUSOLVER_STATUS_SUCCESS &&
             lw <= lwork &&
             cusolverDnDsygvd(hs, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, dA, m, dB, m, dW,
                              work, lwork, info) == CUSOLVER_STATUS_SUCCESS;
        int hinfo = 1;
        std::vector<double> z((size_t)m * m), w(m);
        ok = ok && cudaMemcpy(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess && hinfo == 0 &&
             cudaMemcpy(z.data(), dA, sizeof(double) * m * m, cudaMemcpyDeviceToHost) == cudaSuccess &&
             cudaMemcpy(w.data(), dW, sizeof(double) * m, cudaMemcpyDeviceToHost) == cudaSuccess;
        if (!ok) break;
        S[c].assign((size_t)m * m, 0.0);
        for (int i = 0; i < m; i++)
            for (int k = 0; k < m; k++) S[c][(size_t)i * m + k] = z[i + (size_t)k * m];   // column-major -> row-major
        lam[c] = w;
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dW); cudaFree(work); cudaFree(info);
    cusolverDnDestroy(hs);
    return ok;
}

template <typename T>
bool upload(T **dst, const std::vector<T> &v)
{
    if (cudaMalloc(dst, sizeof(T) * (v.empty() ? 1 : v.size())) != cudaSuccess) return false;
    return v.empty() || cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) == cudaSuccess;
}

bool build_tables(const nb_handle *h, SwState &s)
{
    const int p = h->p, n = h->n, P3 = p + 3;
    // Ahat[i][j] = sum_q w_q D[q][i] D[q][j] (D[q*n + i] = l_i'(x_q))
    std::vector<double> Ah((size_t)n * n, 0.0);
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) {
            double v = 0.0;
            for (int q = 0; q < n; q++) v += h->weights[q] * h->D[q * n + i] * h->D[q * n + j];
            Ah[(size_t)i * n + j] = v;
        }
    std::vector<double> phl(n), phr(n);
    for (int i = 0; i < n; i++) { phl[i] = 0.5 * (1.0 - h->nodes[i]); phr[i] = 0.5 * (1.0 + h->nodes[i]); }
    const int nels[3] = {h->nelx, h->nely, h->nelz};
    for (int a = 0; a < 3; a++) {
        const int nel = nels[a], last = nel * p;   // lattice 0 .. last; unknowns 1 .. last - 1
        const double hl = 1.0 / nel;
        // assembled 1-D entries on the lattice
        auto A1 = [&](int I, int J) {
            double v = 0.0;
            for (int e = (I / p) - 1; e <= I / p; e++) {
                if (e < 0 || e >= nel) continue;
                const int i = I - e * p, j = J - e * p;
                if (i >= 0 && i <= p && j >= 0 && j <= p) v += (2.0 / hl) * Ah[(size_t)i * n + j];
            }
            return v;
        };
        auto B1 = [&](int I) {
            double v = 0.0;
            for (int e = (I / p) - 1; e <= I / p; e++) {
                if (e < 0 || e >= nel) continue;
                const int i = I - e * p;
                if (i >= 0 && i <= p) v += (hl / 2.0) * h->weights[i];
            }
            return v;
        };
        std::map<std::pair<int, int>, int> cases;
        std::vector<uint8_t> cs(nel), cnt((size_t)nel * P3, 0);
        std::vector<std::vector<double>> cA, cB;
        std::vector<int> cn, coff;
        for (int ex = 0; ex < nel; ex++) {
            const int lo = std::max(ex * p - 1, 1), hi = std::min(ex * p + p + 1, last - 1);
            for (int t = 0; t < P3; t++) {   // overlap count of the extended point (0: not an unknown)
                const int I = ex * p - 1 + t;
                if (I < 1 || I > last - 1) continue;
                int c = 0;
                for (int e2 = 0; e2 < nel; e2++)
                    if (I >= e2 * p - 1 && I <= e2 * p + p + 1) c++;
                cnt[(size_t)ex * P3 + t] = (uint8_t)c;
            }
            const std::pair<int, int> key(lo - ex * p, hi - ex * p);
            auto it = cases.find(key);
            if (it == cases.end()) {
                const int m = hi - lo + 1, id = (int)cn.size();
                if (id > 255) return false;
                it = cases.emplace(key, id).first;
                std::vector<double> A((size_t)(m > 0 ? m * m : 0)), B((size_t)(m > 0 ? m * m : 0), 0.0);
                for (int i = 0; i < m; i++) {
                    for (int j = 0; j < m; j++) A[(size_t)i * m + j] = A1(lo + i, lo + j);
                    B[(size_t)i * m + i] = B1(lo + i);
                }
                cA.push_back(A);
                cB.push_back(B);
                cn.push_back(m);
                coff.push_back(lo - (ex * p - 1));
            }
            cs[ex] = (uint8_t)it->second;
        }
        std::vector<std::vector<double>> cS, cL;
        if (!gen_eig_batch(cA, cB, cn, cS, cL)) return false;
        const int nc = (int)cn.size();
        std::vector<double> S((size_t)nc * P3 * P3, 0.0), L((size_t)nc * P3, 1.0);
        for (int c = 0; c < nc; c++)
            for (int i = 0; i < cn[c]; i++) {
                for (int k = 0; k < cn[c]; k++) S[((size_t)c * P3 + coff[c] + i) * P3 + k] = cS[c][(size_t)i * cn[c] + k];
                L[(size_t)c * P3 + i] = cL[c][i];
            }
        std::vector<float> Sf(S.begin(), S.end());
        // coarse level: interior vertices 1 .. nel - 1 (index v - 1)
        const int nv = nel - 1;
        s.nv[a] = nv;
        std::vector<double> S0, L0;
        if (nv > 0) {
            std::vector<std::vector<double>> A0(1, std::vector<double>((size_t)nv * nv, 0.0)), B0 = A0;
            for (int e = 0; e < nel; e++) {   // element e: vertices e (phl) and e + 1 (phr)
                double ae[2][2] = {{0, 0}, {0, 0}}, be[2][2] = {{0, 0}, {0, 0}};
                for (int u = 0; u < 2; u++)
                    for (int v = 0; v < 2; v++)
                        for (int i = 0; i < n; i++) {
                            const double fu = u ? phr[i] : phl[i];
                            be[u][v] += fu * (hl / 2.0) * h->weights[i] * (v ? phr[i] : phl[i]);
                            for (int j = 0; j < n; j++) ae[u][v] += fu * (2.0 / hl) * Ah[(size_t)i * n + j] * (v ? phr[j] : phl[j]);
                        }
                for (int u = 0; u < 2; u++)
                    for (int v = 0; v < 2; v++) {
                        const int gu = e + u - 1, gv = e + v - 1;   // interior index of vertex e + u
                        if (gu < 0 || gu >= nv || gv < 0 || gv >= nv) continue;
                        A0[0][(size_t)gu * nv + gv] += ae[u][v];
                        B0[0][(size_t)gu * nv + gv] += be[u][v];
                    }
            }
            std::vector<std::vector<double>> s0, l0;
            if (!gen_eig_batch(A0, B0, std::vector<int>{nv}, s0, l0)) return false;
            S0 = s0[0];
            L0 = l0[0];
        }
        std::vector<float> S0f(S0.begin(), S0.end());
        if (!upload(&s.cs[a], cs) || !upload(&s.cnt[a], cnt) || !upload(&s.S64[a], S) || !upload(&s.S32[a], Sf) ||
            !upload(&s.lam[a], L) || !upload(&s.S064[a], S0) || !upload(&s.S032[a], S0f) || !upload(&s.lam0[a], L0))
            return false;
    }
    if (!upload(&s.phL, phl) || !upload(&s.phR, phr)) return false;
    s.tables = true;
    return true;
}

}  // namespace

int sw_ensure(nb_handle *h, int prec, const char **msg)
{
    if (h->nelzl != h->nelz) { *msg = "NB_PC_SCHWARZ needs a whole-box handle (not a z-slab)"; return NB_EINVAL; }
    if (!h->sw) h->sw = new (std::nothrow) SwState();
    if (!h->sw) { *msg = "host allocation failed"; return NB_ENOMEM; }
    SwState &s = *h->sw;
    if (!s.tables && !build_tables(h, s)) {
        cudaGetLastError();
        *msg = "Schwarz table setup (cuSOLVER sygvd) failed";
        return NB_ECUDA;
    }
    const size_t vs = prec == NB_FP64 ? 8 : 4;                                  // TV
    const size_t gs = (prec == NB_FP64 || prec == NB_MIXED) ? 8 : 4;            // TG
    const size_t P3 = (size_t)h->p + 3;
    const size_t V = (size_t)(s.nv[0] > 0 ? s.nv[0] : 0) * (s.nv[1] > 0 ? s.nv[1] : 0) * (s.nv[2] > 0 ? s.nv[2] : 0);
    if (!s.zext[prec]) {
        if (cudaMalloc(&s.zext[prec], vs * (size_t)h->E * P3 * P3 * P3) != cudaSuccess ||
            cudaMalloc(&s.cpart[prec], gs * (size_t)h->E * 8) != cudaSuccess ||
            cudaMalloc(&s.c0[prec], vs * (V > 0 ? V : 1)) != cudaSuccess ||
            cudaMalloc(&s.c1[prec], vs * (V > 0 ? V : 1)) != cudaSuccess) {
            cudaGetLastError();
            cudaFree(s.zext[prec]); cudaFree(s.cpart[prec]); cudaFree(s.c0[prec]); cudaFree(s.c1[prec]);
            s.zext[prec] = s.cpart[prec] = s.c0[prec] = s.c1[prec] = nullptr;
            *msg = "cudaMalloc Schwarz scratch";
            return NB_ENOMEM;
        }
    }
    return NB_OK;
}

void sw_fill(const nb_handle *h, int prec, SwArgs &a)
{
    memset(&a, 0, sizeof(a));
    if (!h->sw || !h->sw->tables) return;
    const SwState &s = *h->sw;
    const bool d = prec == NB_FP64;
    a.on = 1;
    for (int k = 0; k < 3; k++) {
        a.nv[k] = s.nv[k];
        a.cs[k] = s.cs[k];
        a.cnt[k] = s.cnt[k];
        a.S[k] = d ? (const void *)s.S64[k] : (const void *)s.S32[k];
        a.lam[k] = s.lam[k];
        a.S0[k] = d ? (const void *)s.S064[k] : (const void *)s.S032[k];
        a.lam0[k] = s.lam0[k];
    }
    a.phL = s.phL;
    a.phR = s.phR;
    a.zext = s.zext[prec];
    a.cpart = s.cpart[prec];
    a.c0 = s.c0[prec];
    a.c1 = s.c1[prec];
}

void sw_free(nb_handle *h)
{
    if (!h->sw) return;
    SwState &s = *h->sw;
    for (int k = 0; k < 3; k++) {
        cudaFree(s.cs[k]); cudaFree(s.cnt[k]); cudaFree(s.S64[k]); cudaFree(s.S32[k]); cudaFree(s.lam[k]);
        cudaFree(s.S064[k]); cudaFree(s.S032[k]); cudaFree(s.lam0[k]);
    }
    cudaFree(s.phL); cudaFree(s.phR);
    for (int k = 0; k < 4; k++) { cudaFree(s.zext[k]); cudaFree(s.cpart[k]); cudaFree(s.c0[k]); cudaFree(s.c1[k]); }
    delete h->sw;
    h->sw = nullptr;
}

}  // namespace nb
