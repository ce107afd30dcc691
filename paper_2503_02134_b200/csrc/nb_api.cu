// nb_api.cu -- the C ABI (include/nb.h): argument checking, setup orchestration,
// GLL basis on the host, CG driver (one persistent megakernel per solve: device-resident
// scalars, the whole iteration loop without host round trips).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <unistd.h>

#include "nb.h"
#include "nb_internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg)
{
    g_err = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char *where)
{
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return NB_ECUDA;
}
#define NB_CU(call, where)                                     \
    do {                                                       \
        cudaError_t _e = (call);                               \
        if (_e != cudaSuccess) return cuda_fail(_e, where);    \
    } while (0)

// ---------------------------------------------------------------------------
// GLL basis, computed independently of the oracle: Newton on
// q(x) = L_{N+1}(x) - L_{N-1}(x) (roots: +-1 and the zeros of L_N'),
// q'(x) = (2N+1) L_N(x); derivative matrix from barycentric weights, diagonal
// by the negative-sum rule.
// ---------------------------------------------------------------------------
void legendre3(int N, double x, double &LNm1, double &LN, double &LNp1)
{
    double a = 1.0, b = x;   // L_0, L_1
    if (N == 0) { LNm1 = 0.0; LN = 1.0; LNp1 = x; return; }
    for (int k = 1; k < N; k++) {
        double c = ((2.0 * k + 1.0) * x * b - k * a) / (k + 1.0);
        a = b;
        b = c;
    }
    LNm1 = a;
    LN = b;
    LNp1 = ((2.0 * N + 1.0) * x * b - N * a) / (N + 1.0);
}

bool gll_basis(int N, double *x, double *w, double *D)
{
    const double pi = 3.14159265358979323846;
    const int n = N + 1;
    x[0] = -1.0;
    x[N] = 1.0;
    for (int j = 1; j <= (N - 1) / 2; j++) {
        double t = -std::cos(pi * j / N);
        bool ok = false;
        for (int it = 0; it < 200; it++) {
            double a, b, c;
            legendre3(N, t, a, b, c);
            const double dt = -(c - a) / ((2.0 * N + 1.0) * b);
            t += dt;
            if (std::fabs(dt) <= 1e-16) { ok = true; break; }
        }
        if (!ok) {
            double a, b, c;
            legendre3(N, t, a, b, c);
            if (std::fabs(c - a) > 1e-13) return false;
        }
        x[j] = t;
        x[N - j] = -t;
    }
    if (N % 2 == 0) x[N / 2] = 0.0;
    for (int j = 0; j < n; j++) {
        double a, b, c;
        legendre3(N, x[j], a, b, c);
        w[j] = 2.0 / (N * (N + 1.0) * b * b);
    }
    double lam[16];
    for (int j = 0; j < n; j++) {
        double prod = 1.0;
        for (int k = 0; k < n; k++)
            if (k != j) prod *= (x[j] - x[k]);
        lam[j] = 1.0 / prod;
    }
    for (int i = 0; i < n; i++) {
        double s = 0.0;
        for (int j = 0; j < n; j++) {
            if (j == i) continue;
            const double v = (lam[j] / lam[i]) / (x[i] - x[j]);
            D[i * n + j] = v;
            s += v;
        }
        D[i * n + i] = -s;
    }
    return true;
}

bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

int check_dev_ptr(const nb_handle *h, const void *p, const char *name)
{
    if (!p) return fail(NB_EINVAL, std::string(name) + " is NULL");
    if (!aligned16(p)) return fail(NB_EINVAL, std::string(name) + " is not 16-byte aligned");
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return fail(NB_EINVAL, std::string(name) + " is not a CUDA pointer");
    }
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
        return fail(NB_EINVAL, std::string(name) + " is not device memory");
    if (at.device != h->device) return fail(NB_EINVAL, std::string(name) + " lives on another device");
    return NB_OK;
}

size_t vsize(int prec) { return prec == NB_FP64 ? sizeof(double) : sizeof(float); }

int ensure_f32(nb_handle *h)
{
    // one-time casts (first single-precision call only; no synchronisation afterwards)
    if (h->g32 && h->dinv32) return NB_OK;
    if (!h->g32) {
        NB_CU(cudaMalloc(&h->g32, sizeof(float) * 6 * h->NL), "cudaMalloc g32");
        NB_CU(nb::launch_cast(h->g64, h->g32, 6 * h->NL, 0), "cast g");
    }
    if (!h->dinv32) {
        NB_CU(cudaMalloc(&h->dinv32, sizeof(float) * h->NL), "cudaMalloc dinv32");
        NB_CU(nb::launch_cast(h->dinv64, h->dinv32, h->NL, 0), "cast dinv");
    }
    NB_CU(cudaStreamSynchronize(0), "cast sync");
    return NB_OK;
}

// policy dispatch of the per-policy kernel templates
#define NB_POL(prec, F, ...)                                                                       \
    ((prec) == NB_FP64 ? F<NB_FP64>(__VA_ARGS__)                                                   \
     : (prec) == NB_FP32 ? F<NB_FP32>(__VA_ARGS__)                                                 \
     : (prec) == NB_MIXED ? F<NB_MIXED>(__VA_ARGS__) : F<NB_FP32_DOT2>(__VA_ARGS__))

void free_ws(nb::Workspace &ws);

static int alloc_ws(nb_handle *h, int prec, int32_t max_iter)
{
    nb::Workspace &ws = h->ws[prec];
    if (!ws.ctl) {
        // multi-rank control block (small; allocated first so later allocations keep their layout)
        NB_CU(cudaMalloc(&ws.ctl, nb::NB_CTL_BYTES), "cudaMalloc ctl");
        NB_CU(cudaMemset(ws.ctl, 0, nb::NB_CTL_BYTES), "memset ctl");
    }
    if (!ws.ready) {
        const size_t vs = vsize(prec) * h->NL;
        NB_CU(cudaMalloc(&ws.r, vs), "cudaMalloc r");
        NB_CU(cudaMalloc(&ws.p, vs), "cudaMalloc p");
        NB_CU(cudaMalloc(&ws.w, vs), "cudaMalloc w");
        NB_CU(cudaMalloc(&ws.x, vs), "cudaMalloc x");
        NB_CU(cudaMalloc(&ws.z, vs), "cudaMalloc z");
        ws.mega_G = NB_POL(prec, nb::grid_mega, h);
        // megakernel partials: 4 accumulators per block (pap, shared pap, rtr, rho), 2 doubles
        // each for the Dot2 expansions (nb_mega_launch.cuh: launch_cg_mega)
        const int mslots = (prec == NB_FP32_DOT2 ? 8 : 4) * ws.mega_G;
        NB_CU(cudaMalloc(&ws.part, sizeof(double) * mslots), "cudaMalloc part");
        NB_CU(cudaMalloc(&ws.bar, sizeof(unsigned int) * nb::BAR_WORDS), "cudaMalloc bar");
        NB_CU(cudaMemset(ws.bar, 0, sizeof(unsigned int) * nb::BAR_WORDS), "memset bar");
        NB_CU(cudaMalloc(&ws.scal, sizeof(nb::Scal)), "cudaMalloc scal");
        NB_CU(cudaMallocHost(&ws.scal_host, sizeof(nb::Scal)), "cudaMallocHost scal");
        NB_CU(cudaMemset(ws.scal, 0, sizeof(nb::Scal)), "memset scal");
        NB_CU(cudaDeviceSynchronize(), "ws sync");
        ws.ready = true;
    }
    if (ws.hist_cap < max_iter + 1) {
        if (ws.hist) cudaFree(ws.hist);
        if (ws.shist) cudaFree(ws.shist);
        if (ws.tim) cudaFree(ws.tim);
        ws.hist = nullptr;
        ws.shist = nullptr;
        ws.tim = nullptr;
        ws.hist_cap = 0;
        const int cap = max_iter + 1 < 1024 ? 1024 : max_iter + 1;
        NB_CU(cudaMalloc(&ws.hist, sizeof(double) * cap), "cudaMalloc hist");
        NB_CU(cudaMalloc(&ws.shist, sizeof(double) * 3 * cap), "cudaMalloc shist");
        NB_CU(cudaMalloc(&ws.tim, sizeof(unsigned long long) * 3 * cap), "cudaMalloc tim");
        ws.hist_cap = cap;
    }
    return NB_OK;
}

// The policy's CG workspace, allocated on first use; a failed allocation releases everything
// allocated so far (the next call starts clean).
int ensure_ws(nb_handle *h, int prec, int32_t max_iter)
{
    const int rc = alloc_ws(h, prec, max_iter);
    if (rc != NB_OK) {
        const std::string msg = g_err;   // keep the failing call's message
        free_ws(h->ws[prec]);
        g_err = msg;
    }
    return rc;
}

void free_ws(nb::Workspace &ws)
{
    for (int i = 0; i < ws.peer.nopened; i++) cudaIpcCloseMemHandle(ws.peer.opened[i]);
    cudaFree(ws.r); cudaFree(ws.p); cudaFree(ws.w); cudaFree(ws.x); cudaFree(ws.z); cudaFree(ws.xd); cudaFree(ws.ctl);
    cudaFree(ws.part);
    cudaFree(ws.scal); cudaFree(ws.hist); cudaFree(ws.shist); cudaFree(ws.tim); cudaFree(ws.bar);
    if (ws.scal_host) cudaFreeHost(ws.scal_host);
    ws = nb::Workspace();
}

// C-11 stagnation rule on the host history (only for runs that did not converge)
int classify(const std::vector<double> &res, int k, int W)
{
    double mk = res[0];
    for (int i = 1; i <= k; i++) mk = res[i] < mk ? res[i] : mk;
    if (res[k] > 100.0 * mk) return NB_STAGNATED;
    if (W > 0 && k >= W) {
        double mkw = res[0];
        for (int i = 1; i <= k - W; i++) mkw = res[i] < mkw ? res[i] : mkw;
        if (mk > 0.1 * mkw) return NB_STAGNATED;
    }
    return NB_MAXITER;
}

}  // namespace

namespace nb {
void deform_phases(uint64_t seed, double ph[3])
{
    for (int a = 0; a < 3; a++) {
        uint64_t z = (seed ^ (3ull * 0xD1B54A32D192ED03ull)) + ((uint64_t)a + 1ull) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        ph[a] = 3.14159265358979323846 * (1.0 + ((double)(z >> 11) * 0x1.0p-52 - 1.0));
    }
}
}  // namespace nb

extern "C" {

const char *nb_last_error(void) { return g_err.c_str(); }
const char *nb_version(void) { return "nb-b200 0.1 (sm_100a)"; }

// Build the data of one handle's slab [ez0, ez0 + nelzl) of the box (every field of h set by
// make_handle): geometry, GS segments and (when `jacobi`) the Jacobi diagonal.
static int setup_box(nb_handle *h, bool jacobi)
{
    const int64_t NL = h->NL;
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e, "stream");
    {
        const char *gs = std::getenv("NB_CG_GS");
        h->cg_csr = (gs && std::strcmp(gs, "csr") == 0) ? 1 : 0;
        const char *po = std::getenv("NB_PHASE_ONLY");   // measurement knob (tools/ncu_phases.sh)
        h->phase_only = po ? (po[0] == 'A' ? 1 : po[0] == 'B' ? 2 : 0) : 0;
        const char *dc = std::getenv("NB_DSSUM");         // consistent nb_dssum: structured (default) or CSR
        h->dssum_csr = (dc && std::strcmp(dc, "csr") == 0) ? 1 : 0;
    }
    if ((e = cudaMalloc(&h->g64, sizeof(double) * 6 * NL)) != cudaSuccess) return fail(NB_ENOMEM, "cudaMalloc g64");
    if ((e = cudaMalloc(&h->B, sizeof(double) * NL)) != cudaSuccess) return fail(NB_ENOMEM, "cudaMalloc B");
    if ((e = cudaMalloc(&h->dinv64, sizeof(double) * NL)) != cudaSuccess) return fail(NB_ENOMEM, "cudaMalloc dinv");
    if ((e = cudaMalloc(&h->flag, sizeof(int32_t))) != cudaSuccess) return fail(NB_ENOMEM, "cudaMalloc flag");
    cudaStream_t st = h->cap_stream;
    if ((e = cudaMemsetAsync(h->flag, 0, sizeof(int32_t), st)) != cudaSuccess) return cuda_fail(e, "memset");
    double ph[3];
    nb::deform_phases(h->seed, ph);
    if ((e = nb::launch_geometry(h, ph, st)) != cudaSuccess) return cuda_fail(e, "geometry");
    if ((e = nb::build_gs(h, st)) != cudaSuccess) return cuda_fail(e, "gs segments");
    double *diag = nullptr;
    if (jacobi) {
        if ((e = cudaMalloc(&diag, sizeof(double) * NL)) != cudaSuccess) return fail(NB_ENOMEM, "cudaMalloc diag");
        e = nb::launch_jacobi(h, diag, st);
    }
    int32_t flag = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&flag, h->flag, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(diag);
    if (e != cudaSuccess) return cuda_fail(e, "jacobi");
    if (flag & 1) return fail(NB_EGEOM, "non-positive Jacobian");
    if (flag & 2) return fail(NB_EGEOM, "non-positive Jacobi diagonal");
    return NB_OK;
}

static nb_handle *make_handle(int32_t nelx, int32_t nely, int32_t nelz, int32_t ez0, int32_t ez1, int32_t p,
                              double deform_amp, uint64_t seed, int32_t device, int sm_count)
{
    nb_handle *h = new (std::nothrow) nb_handle();
    if (!h) return nullptr;
    const int n = p + 1;
    h->device = device;
    h->nelx = nelx; h->nely = nely; h->nelz = nelz; h->p = p; h->n = n;
    h->ez0 = ez0; h->nelzl = ez1 - ez0;
    h->E = (int64_t)nelx * nely * h->nelzl;
    h->NL = h->E * n * n * n;
    h->NX = (int64_t)nelx * p + 1; h->NY = (int64_t)nely * p + 1; h->NZ = (int64_t)nelz * p + 1;
    h->NG = h->NX * h->NY * h->NZ;
    h->NZl = (int64_t)h->nelzl * p + 1;
    h->NGl = h->NX * h->NY * h->NZl;
    h->n_unmasked = ((int64_t)nelx * p - 1) * ((int64_t)nely * p - 1) * ((int64_t)nelz * p - 1);
    h->deform = deform_amp;
    h->seed = seed;
    h->sm_count = sm_count;
    if (!gll_basis(p, h->nodes, h->weights, h->D)) { delete h; return nullptr; }
    return h;
}

int nb_setup_slab(int32_t nelx, int32_t nely, int32_t nelz, int32_t ez0, int32_t ez1, int32_t p, double deform_amp,
                  uint64_t seed, int32_t device, nb_handle **out)
{
    if (!out) return fail(NB_EINVAL, "out is NULL");
    *out = nullptr;
    if (p < 1 || p > 15) return fail(NB_EINVAL, "p must be in [1,15]");
    if (nelx < 1 || nely < 1 || nelz < 1) return fail(NB_EINVAL, "element counts must be >= 1");
    if (ez0 < 0 || ez1 > nelz || ez0 >= ez1) return fail(NB_EINVAL, "slab must satisfy 0 <= ez0 < ez1 <= nelz");
    if (!(deform_amp >= 0.0) || deform_amp > 0.25) return fail(NB_EINVAL, "deform_amp must be in [0, 0.25]");
    const int n = p + 1;
    // the slab (and its ghost-extended twin) must fit the int32 local indexing
    const int32_t ghosts = (ez0 > 0) + (ez1 < nelz);
    if ((int64_t)nelx * nely * (int64_t)(ez1 - ez0 + ghosts) * n * n * n >= 2147483647LL)
        return fail(NB_EINVAL, "n_local must be < 2^31 (int32 GS indices)");
    int ndev = 0;
    NB_CU(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) return fail(NB_EINVAL, "bad device ordinal");
    NB_CU(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    NB_CU(cudaGetDeviceProperties(&prop, device), "props");
    const int64_t NX = (int64_t)nelx * p + 1, NY = (int64_t)nely * p + 1, NZ = (int64_t)nelz * p + 1;
    if (NX * NY * NZ >= 2147483647LL) return fail(NB_EINVAL, "global node count must be < 2^31");

    nb_handle *h = make_handle(nelx, nely, nelz, ez0, ez1, p, deform_amp, seed, device, prop.multiProcessorCount);
    if (!h) return fail(NB_ENOMEM, "host allocation or GLL Newton failed");
    const bool whole = ez0 == 0 && ez1 == nelz;
    int rc;
    if (whole) {
        if ((rc = setup_box(h, true))) { nb_destroy(h); return rc; }
    } else {
        // The Jacobi diagonal (and the manufactured RHS) of the slab's interface nodes need the
        // neighbour slabs' element contributions: computed redundantly on a twin slab with one
        // ghost layer per side (closed-form geometry), so setup needs no communication.  Same
        // elements, same ascending-element summation order: bit-identical to the whole box.
        const int32_t x0 = ez0 > 0 ? ez0 - 1 : 0, x1 = ez1 < nelz ? ez1 + 1 : nelz;
        nb_handle *x = make_handle(nelx, nely, nelz, x0, x1, p, deform_amp, seed, device, prop.multiProcessorCount);
        if (!x) { delete h; return fail(NB_ENOMEM, "host allocation failed"); }
        h->ext = x;
        h->ext_off = (int64_t)(ez0 - x0) * nelx * nely;
        if ((rc = setup_box(x, true)) || (rc = setup_box(h, false))) { nb_destroy(h); return rc; }
        const size_t n3 = (size_t)n * n * n;
        cudaError_t e = cudaMemcpy(h->dinv64, x->dinv64 + h->ext_off * n3, sizeof(double) * h->NL, cudaMemcpyDeviceToDevice);
        if (e != cudaSuccess) { nb_destroy(h); return cuda_fail(e, "slab dinv"); }
    }
    *out = h;
    return NB_OK;
}

int nb_setup(int32_t nelx, int32_t nely, int32_t nelz, int32_t p, double deform_amp, uint64_t seed, int32_t device,
             nb_handle **out)
{
    if (nelz < 1) {
        if (out) *out = nullptr;
        return fail(NB_EINVAL, "element counts must be >= 1");
    }
    return nb_setup_slab(nelx, nely, nelz, 0, nelz, p, deform_amp, seed, device, out);
}

int nb_destroy(nb_handle *h)
{
    if (!h) return NB_OK;
    cudaSetDevice(h->device);
    if (h->ext) nb_destroy(h->ext);
    for (auto &ws : h->ws) free_ws(ws);
    nb::sw_free(h);
    cudaFree(h->g64); cudaFree(h->g32); cudaFree(h->B); cudaFree(h->dinv64); cudaFree(h->dinv32);
    cudaFree(h->gs_off); cudaFree(h->gs_idx); cudaFree(h->flag);
    if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
    delete h;
    return NB_OK;
}

int nb_query(const nb_handle *h, nb_info *o)
{
    if (!h || !o) return fail(NB_EINVAL, "NULL argument");
    o->E = h->E; o->n_local = h->NL; o->n_global = h->NG; o->n_unmasked = h->n_unmasked;
    o->n_shared_global = h->nseg; o->n_shared_copies = h->ncopies;
    o->p = h->p; o->nelx = h->nelx; o->nely = h->nely; o->nelz = h->nelz;
    o->ez0 = h->ez0; o->nelz_local = h->nelzl;
    return NB_OK;
}

int nb_rhs(nb_handle *h, nb_rhs_kind kind, double noise_amp, uint64_t seed, nb_policy prec, void *b, void *stream)
{
    if (!h) return fail(NB_EINVAL, "NULL handle");
    if (prec < NB_FP64 || prec > NB_FP32_DOT2) return fail(NB_EINVAL, "bad policy");
    if (prec == NB_FP32_DOT2) prec = NB_FP32;   // same vectors and arithmetic outside the dots
    if (kind != NB_RHS_UNIFORM && kind != NB_RHS_MANUFACTURED) return fail(NB_EINVAL, "bad rhs kind");
    NB_CU(cudaSetDevice(h->device), "cudaSetDevice");
    int rc = check_dev_ptr(h, b, "b");
    if (rc) return rc;
    if (kind == NB_RHS_MANUFACTURED && h->ext) {
        // QQ^T (B f) on the slab's interface nodes needs the neighbours' B f: computed on the
        // ghost-extended twin, then the owned elements sliced out (stream-ordered)
        const size_t es = prec == NB_FP64 ? sizeof(double) : sizeof(float);
        const size_t n3 = (size_t)h->n * h->n * h->n;
        cudaStream_t st = (cudaStream_t)stream;
        void *tmp = nullptr;
        NB_CU(cudaMallocAsync(&tmp, es * h->ext->NL, st), "rhs tmp");
        cudaError_t e = nb::launch_rhs(h->ext, kind, noise_amp, seed, prec, tmp, st);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(b, (char *)tmp + es * h->ext_off * n3, es * h->NL, cudaMemcpyDeviceToDevice, st);
        cudaError_t e2 = cudaFreeAsync(tmp, st);
        NB_CU(e != cudaSuccess ? e : e2, "slab rhs");
        return NB_OK;
    }
    NB_CU(nb::launch_rhs(h, kind, noise_amp, seed, prec, b, (cudaStream_t)stream), "rhs");
    return NB_OK;
}

int nb_ax(nb_handle *h, nb_policy prec, const void *u, void *w, uint32_t flags, void *stream)
{
    if (!h) return fail(NB_EINVAL, "NULL handle");
    if (prec < NB_FP64 || prec > NB_FP32_DOT2) return fail(NB_EINVAL, "bad policy");
    if (prec == NB_FP32_DOT2) prec = NB_FP32;
    if (flags & ~NB_AX_LOCAL) return fail(NB_EINVAL, "unknown flags");
    NB_CU(cudaSetDevice(h->device), "cudaSetDevice");
    int rc = check_dev_ptr(h, u, "u");
    if (!rc) rc = check_dev_ptr(h, w, "w");
    if (rc) return rc;
    if (u == w) return fail(NB_EINVAL, "u and w must be distinct");
    if (prec != NB_FP64 && (rc = ensure_f32(h))) return rc;
    const bool local = (flags & NB_AX_LOCAL) != 0;
    NB_CU(NB_POL(prec, nb::launch_ax_local, h, u, w, !local, (cudaStream_t)stream), "ax");
    if (!local) NB_CU(nb::launch_dssum(h, prec, NB_GS_CONSISTENT, w, (cudaStream_t)stream), "ax dssum");
    return NB_OK;
}

int nb_dssum_ranked(nb_handle *h, nb_policy prec, nb_gs_order order, int32_t px, int32_t py, int32_t pz, void *u,
                    void *stream)
{
    if (!h) return fail(NB_EINVAL, "NULL handle");
    if (prec < NB_FP64 || prec > NB_FP32_DOT2) return fail(NB_EINVAL, "bad policy");
    if (prec == NB_FP32_DOT2) prec = NB_FP32;
    if (order < NB_GS_CONSISTENT || order > NB_GS_ALLREDUCE) return fail(NB_EINVAL, "bad gs order");
    if (px < 1 || py < 1 || pz < 1 || px > h->nelx || py > h->nely || pz > h->nelz)
        return fail(NB_EINVAL, "rank partition must satisfy 1 <= p_a <= nel_a");
    if ((order == NB_GS_PAIRWISE || order == NB_GS_ALLREDUCE) && h->nelzl != h->nelz)
        return fail(NB_EINVAL, "ranked gather-scatter orders need the whole box");
    NB_CU(cudaSetDevice(h->device), "cudaSetDevice");
    int rc = check_dev_ptr(h, u, "u");
    if (rc) return rc;
    NB_CU(nb::launch_dssum(h, prec, order, u, (cudaStream_t)stream, nb::RankPart{px, py, pz}), "dssum");
    return NB_OK;
}

int nb_dssum(nb_handle *h, nb_policy prec, nb_gs_order order, void *u, void *stream)
{
    if (h && (order == NB_GS_PAIRWISE || order == NB_GS_ALLREDUCE))
        return fail(NB_EINVAL, "NB_GS_PAIRWISE / NB_GS_ALLREDUCE need a partition: nb_dssum_ranked");
    return nb_dssum_ranked(h, prec, order, 1, 1, 1, u, stream);
}

// CUDA events released on every return path
struct EventSet {
    std::vector<cudaEvent_t> ev;
    cudaError_t create(size_t n)
    {
        ev.assign(n, nullptr);
        for (auto &e : ev) {
            const cudaError_t r = cudaEventCreate(&e);
            if (r != cudaSuccess) return r;
        }
        return cudaSuccess;
    }
    ~EventSet()
    {
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
    }
};

// One solve over nh handles: nh = 1 -> the handle's own solve (whole box, or one slab of a
// multi-rank solve when nb_peer_attach'ed); nh > 1 -> slabs of one box sharing this GPU, one
// cooperative launch (nb_cg_group).  b, x: per handle.
static int cg_run(nb_handle *const *hs, int nh, const nb_cg_opts *o, const void *const *b, bool b_host, void *const *x,
                  bool x_host, nb_cg_report *reps, cudaStream_t st)
{
    const int prec = o->policy;
    const int order = o->gs_order;
    int rc;
    for (int r = 0; r < nh; r++) {
        nb_handle *h = hs[r];
        if (prec != NB_FP64 && (rc = ensure_f32(h))) return rc;
        if ((rc = ensure_ws(h, prec, o->max_iter))) return rc;
        const char *swm = "";
        if (o->precond == NB_PC_SCHWARZ && (rc = nb::sw_ensure(h, prec, &swm))) return fail(rc, swm);
        nb::Workspace &ws = h->ws[prec];
        if (o->x_fp64 && !ws.xd) NB_CU(cudaMalloc(&ws.xd, sizeof(double) * h->NL), "cudaMalloc xd");
    }
    nb_handle *h0 = hs[0];
    nb::Workspace &ws0 = h0->ws[prec];
    const bool multi = nh > 1 || ws0.peer.nrank > 0;

    EventSet tev;
    NB_CU(tev.create(2), "event");
    cudaEvent_t t0 = tev.ev[0], t1 = tev.ev[1];
    nb::Scal s0;
    memset(&s0, 0, sizeof(s0));
    s0.rtol = o->rtol;
    s0.max_iter = o->max_iter;
    NB_CU(cudaEventRecord(t0, st), "event record");
    std::vector<const void *> bdev(nh);
    for (int r = 0; r < nh; r++) {
        nb::Workspace &ws = hs[r]->ws[prec];
        *ws.scal_host = s0;
        // host b is staged in w (the only H2D copy of the solve); the prologue reads it
        bdev[r] = b[r];
        if (b_host) {
            NB_CU(cudaMemcpyAsync(ws.w, b[r], vsize(prec) * hs[r]->NL, cudaMemcpyHostToDevice, st), "copy b");
            bdev[r] = ws.w;
        }
        NB_CU(cudaMemcpyAsync(ws.scal, ws.scal_host, sizeof(nb::Scal), cudaMemcpyHostToDevice, st), "copy scal");
    }
    int64_t launches = 0;
    if (multi) {
        // z-slab solve: one MR megakernel for this GPU's slabs
        nb::MultiArgs M;
        memset(&M, 0, sizeof(M));
        const size_t es = vsize(prec);
        for (int r = 0; r < nh; r++) {
            nb_handle *h = hs[r];
            nb::Workspace &ws = h->ws[prec];
            NB_POL(prec, nb::fill_mega_args, h, ws, bdev[r], order, o->max_iter, o->rtol, (int)o->precond,
                   (int)o->x_fp64, ws.tim, M.a[r]);
            NB_CU(cudaMemsetAsync(ws.bar, 0, nb::BAR_WORDS * sizeof(unsigned int), st), "memset bar");
        }
        if (nh > 1) {
            // slabs sharing this launch: neighbours' w and control blocks are plain device pointers
            const size_t n3 = (size_t)h0->n * h0->n * h0->n;
            for (int r = 0; r < nh; r++) {
                nb::Workspace &ws = hs[r]->ws[prec];
                M.a[r].wlo = r > 0 ? (const void *)((const char *)hs[r - 1]->ws[prec].w + es * hs[r - 1]->E * n3) : nullptr;
                M.a[r].whi = r + 1 < nh ? (const void *)((const char *)hs[r + 1]->ws[prec].w - es * hs[r]->E * n3) : nullptr;
                M.mr.flag[r] = (unsigned int *)ws.ctl;
                M.mr.abrt[r] = (unsigned int *)(ws.ctl + nb::NB_CTL_ABORT_OFF);
                M.mr.slot[r] = (double *)(ws.ctl + nb::NB_CTL_FLAG_BYTES);
                NB_CU(cudaMemsetAsync(ws.ctl, 0, nb::NB_CTL_BYTES, st), "memset ctl");
            }
            M.mr.nrank = nh; M.mr.rank0 = 0; M.mr.nloc = nh; M.mr.epoch0 = 0; M.mr.sys = 0;
            // fault injection (tests only): a phantom extra rank that never arrives -- every
            // cross-rank wait must give up after NB_PEER_TIMEOUT_MS and end the solve (no hang)
            const char *ph = std::getenv("NB_FAULT_PHANTOM_RANK");
            if (ph && ph[0] == '1' && nh < nb::NB_MAX_RANKS) {
                unsigned char *c0 = hs[0]->ws[prec].ctl;
                M.mr.flag[nh] = (unsigned int *)(c0 + 96);
                M.mr.abrt[nh] = (unsigned int *)(c0 + 100);
                M.mr.slot[nh] = (double *)(c0 + nb::NB_CTL_FLAG_BYTES);   // same values as rank 0's slots
                M.mr.nrank = nh + 1;
            }
        } else {
            const nb::PeerState &ps = ws0.peer;
            for (int q = 0; q < ps.nrank; q++) {
                M.mr.flag[q] = ps.flag[q];
                M.mr.abrt[q] = ps.abrt[q];
                M.mr.slot[q] = ps.slot[q];
            }
            M.mr.nrank = ps.nrank; M.mr.rank0 = ps.rank; M.mr.nloc = 1; M.mr.epoch0 = ps.epoch;
            M.mr.sys = ps.nrank > 1 ? 1 : 0;
        }
        {
            const char *tm = std::getenv("NB_PEER_TIMEOUT_MS");
            const double ms_to = tm ? std::atof(tm) : 20000.0;
            M.mr.timeout_ns = (unsigned long long)((ms_to > 0 ? ms_to : 20000.0) * 1e6);
        }
        M.mr.Gr = NB_POL(prec, nb::grid_mega_mr, h0) / nh;
        if (M.mr.Gr < 1) return fail(NB_EINVAL, "too many slabs for one launch");
        NB_CU(NB_POL(prec, nb::launch_cg_mr, h0, M, st), "cg multi-rank megakernel");
        launches = 1;
    } else if (o->precond == NB_PC_SCHWARZ) {
        // NEXT-4: the Schwarz-preconditioned megakernel (k_cg_sw)
        nb::MegaArgs A;
        memset(&A, 0, sizeof(A));
        NB_POL(prec, nb::fill_mega_args, h0, ws0, bdev[0], order, o->max_iter, o->rtol, (int)o->precond,
               (int)o->x_fp64, ws0.tim, A);
        A.wlo = A.whi = nullptr;
        nb::sw_fill(h0, prec, A.sw);
        A.rp = nb::RankPart{o->ranks[0] > 0 ? o->ranks[0] : 1, o->ranks[1] > 0 ? o->ranks[1] : 1,
                            o->ranks[2] > 0 ? o->ranks[2] : 1};
        NB_CU(cudaMemsetAsync(ws0.bar, 0, nb::BAR_WORDS * sizeof(unsigned int), st), "memset bar");
        NB_CU(NB_POL(prec, nb::launch_cg_sw, h0, A, ws0.mega_G, false, st), "cg Schwarz megakernel");
        launches = 1;
    } else {
        const nb::RankPart rp{o->ranks[0] > 0 ? o->ranks[0] : 1, o->ranks[1] > 0 ? o->ranks[1] : 1,
                              o->ranks[2] > 0 ? o->ranks[2] : 1};
        NB_CU(NB_POL(prec, nb::launch_cg_mega, h0, ws0, bdev[0], order, o->max_iter, o->rtol, (int)o->precond,
                     (int)o->x_fp64, ws0.tim, st, rp),
              "cg megakernel");
        launches = 1;
    }
    for (int r = 0; r < nh; r++) {
        nb_handle *h = hs[r];
        nb::Workspace &ws = h->ws[prec];
        NB_CU(cudaMemcpyAsync(ws.scal_host, ws.scal, sizeof(nb::Scal), cudaMemcpyDeviceToHost, st), "copy scal back");
        const cudaMemcpyKind kind = x_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
        if (o->x_fp64) NB_CU(cudaMemcpyAsync(x[r], ws.xd, sizeof(double) * h->NL, kind, st), "copy x");
        else NB_CU(cudaMemcpyAsync(x[r], ws.x, vsize(prec) * h->NL, kind, st), "copy x");
    }
    NB_CU(cudaEventRecord(t1, st), "event record");
    NB_CU(cudaStreamSynchronize(st), "solve sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    int ret = NB_OK;
    for (int r = 0; r < nh; r++) {
        nb_handle *h = hs[r];
        nb::Workspace &ws = h->ws[prec];
        const nb::Scal s = *ws.scal_host;
        if (multi) {
            // a bounded cross-rank wait gave up somewhere (this rank's abort word, or block 0's report)
            uint32_t ab = 0;
            NB_CU(cudaMemcpy(&ab, ws.ctl + nb::NB_CTL_ABORT_OFF, sizeof(ab), cudaMemcpyDeviceToHost), "copy abort");
            if (ab || s.aborted) {
                if (nh == 1) ws.peer.broken = true;   // flags and epochs are out of step: re-attach
                ret = NB_ETIMEOUT;
            } else if (nh == 1) {
                ws.peer.epoch += (uint32_t)s.epochs;   // flags are never reset
            }
        }
        const int k = s.iter;
        std::vector<double> res(k + 1, 0.0);
        NB_CU(cudaMemcpy(res.data(), ws.hist, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost), "copy hist");
        double km[3] = {0.0, 0.0, 0.0};
        const int64_t nl = launches;
        {
            // phase durations from the block-0 globaltimer stamps taken after each grid barrier
            std::vector<unsigned long long> tm(3 * (size_t)(k + 1), 0ull);
            NB_CU(cudaMemcpy(tm.data(), ws.tim, sizeof(unsigned long long) * 3 * (k + 1), cudaMemcpyDeviceToHost),
                  "copy tim");
            for (int i = 1; i <= k; i++) {
                const double tA = (double)tm[3 * (i - 1) + 1] - (double)tm[3 * (i - 1)];
                const double tS = (double)tm[3 * (i - 1) + 2] - (double)tm[3 * (i - 1) + 1];
                const double tB = (double)tm[3 * i] - (double)tm[3 * (i - 1) + 2];
                km[0] += 1e-6 * tA; km[1] += 1e-6 * tS; km[2] += 1e-6 * tB;
            }
        }
        if (o->scal_history && r == 0 && k > 0)
            NB_CU(cudaMemcpy(o->scal_history, ws.shist, sizeof(double) * 3 * k, cudaMemcpyDeviceToHost), "copy shist");
        int status = s.status;
        if (status == NB_MAXITER && o->rtol > 0.0) status = classify(res, k, o->stag_window > 0 ? o->stag_window : 200);
        if (o->rel_res_history && r == 0) memcpy(o->rel_res_history, res.data(), sizeof(double) * (k + 1));
        if (reps) {
            nb_cg_report *rep = reps + r;
            rep->iterations = k;
            rep->status = status;
            rep->rtr0 = s.rtr0;
            rep->rtr_final = s.rtr;
            rep->rel_res_final = res[k];
            double mn = res[0];
            for (int i = 1; i <= k; i++) mn = res[i] < mn ? res[i] : mn;
            rep->rel_res_min = mn;
            rep->solve_ms = ms;
            rep->kernel_launches = nl;
            rep->k_ax_ms = km[0];
            rep->k_gs_ms = km[1];
            rep->k_upd_ms = km[2];
        }
        if (status == NB_BROKEDOWN && ret == NB_OK) ret = NB_EBREAKDOWN;
    }
    if (ret == NB_ETIMEOUT)
        return fail(NB_ETIMEOUT, "multi-rank solve aborted: a peer rank did not arrive in time (re-attach before the next solve)");
    if (ret == NB_EBREAKDOWN) return fail(NB_EBREAKDOWN, "CG breakdown (pap <= 0 or non-finite scalar)");
    return NB_OK;
}

static int cg_impl(nb_handle *h, const nb_cg_opts *o, const void *b, bool b_host, void *x, bool x_host,
                   nb_cg_report *rep, cudaStream_t st)
{
    nb_handle *hs[1] = {h};
    const void *bs[1] = {b};
    void *xs[1] = {x};
    return cg_run(hs, 1, o, bs, b_host, xs, x_host, rep, st);
}

static int cg_args(nb_handle *h, const nb_cg_opts *o)
{
    if (!h || !o) return fail(NB_EINVAL, "NULL argument");
    if (o->policy < NB_FP64 || o->policy > NB_FP32_DOT2) return fail(NB_EINVAL, "bad policy");
    if (o->precond < NB_PC_JACOBI || o->precond > NB_PC_SCHWARZ) return fail(NB_EINVAL, "bad precond");
    if (o->precond == NB_PC_SCHWARZ) {
        if (h->nelzl != h->nelz || h->ws[o->policy].peer.nrank > 0)
            return fail(NB_EINVAL, "NB_PC_SCHWARZ needs a whole-box handle (no slabs, no peers)");
    }
    if (o->precond == NB_PC_JACOBI_F32 && o->policy == NB_FP64)
        return fail(NB_EINVAL, "NB_PC_JACOBI_F32 is a single-precision variant (not for NB_FP64)");
    if (o->x_fp64 != 0 && o->x_fp64 != 1) return fail(NB_EINVAL, "x_fp64 must be 0 or 1");
    if (o->reserved0 != 0) return fail(NB_EINVAL, "nb_cg_opts.reserved0 must be 0");
    if (o->x_fp64 && o->policy != NB_MIXED) return fail(NB_EINVAL, "x_fp64 applies to NB_MIXED only");
    if (o->gs_order < NB_GS_CONSISTENT || o->gs_order > NB_GS_ALLREDUCE) return fail(NB_EINVAL, "bad gs order");
    if (o->gs_order == NB_GS_PAIRWISE || o->gs_order == NB_GS_ALLREDUCE) {
        const int32_t nel[3] = {h->nelx, h->nely, h->nelz};
        for (int a = 0; a < 3; a++)
            if (o->ranks[a] < 0 || o->ranks[a] > nel[a])
                return fail(NB_EINVAL, "ranks[a] must be in [1, nel_a] (0 = 1)");
        if (h->nelzl != h->nelz) return fail(NB_EINVAL, "ranked gather-scatter orders need the whole box");
    }
    if (o->max_iter < 0 || !(o->rtol >= 0.0)) return fail(NB_EINVAL, "bad max_iter/rtol");
    if (h->n_unmasked == 0) return fail(NB_EINVAL, "the mesh has no unknowns (every node is on the Dirichlet boundary)");
    NB_CU(cudaSetDevice(h->device), "cudaSetDevice");
    return NB_OK;
}

// a slab solve (group or attached): the fused consistent-order megakernel only
static int mr_args(const nb_handle *h, const nb_cg_opts *o)
{
    if (o->gs_order != NB_GS_CONSISTENT) return fail(NB_EINVAL, "multi-rank solves use the consistent GS order");
    if (h->ws[o->policy].peer.broken)
        return fail(NB_ESTATE, "the last multi-rank solve aborted: nb_peer_detach and nb_peer_attach again");
    if (h->cg_csr) return fail(NB_EINVAL, "multi-rank solves run on the fused megakernel only");
    return NB_OK;
}

int nb_cg(nb_handle *h, const nb_cg_opts *o, const void *b, void *x, nb_cg_report *rep, void *stream)
{
    int rc = cg_args(h, o);
    if (rc) return rc;
    const bool slab = h->nelzl != h->nelz;
    if (slab && h->ws[o->policy].peer.nrank == 0)
        return fail(NB_EINVAL, "a slab handle solves with nb_cg_group or after nb_peer_attach");
    if (h->ws[o->policy].peer.nrank > 0 && (rc = mr_args(h, o))) return rc;
    if ((rc = check_dev_ptr(h, b, "b")) || (rc = check_dev_ptr(h, x, "x"))) return rc;
    return cg_impl(h, o, b, false, x, false, rep, (cudaStream_t)stream);
}

int nb_precond_apply(nb_handle *h, nb_policy prec, nb_precond pc, const void *r, void *z, void *stream)
{
    if (!h) return fail(NB_EINVAL, "NULL handle");
    if (prec < NB_FP64 || prec > NB_FP32_DOT2) return fail(NB_EINVAL, "bad policy");
    if (pc != NB_PC_SCHWARZ) return fail(NB_EINVAL, "nb_precond_apply: only NB_PC_SCHWARZ has a standalone apply");
    if (r == z) return fail(NB_EINVAL, "r and z must be distinct");
    NB_CU(cudaSetDevice(h->device), "cudaSetDevice");
    int rc;
    if ((rc = check_dev_ptr(h, r, "r")) || (rc = check_dev_ptr(h, z, "z"))) return rc;
    if (prec != NB_FP64 && (rc = ensure_f32(h))) return rc;
    if ((rc = ensure_ws(h, prec, 0))) return rc;
    const char *swm = "";
    if ((rc = nb::sw_ensure(h, prec, &swm))) return fail(rc, swm);
    nb::Workspace &ws = h->ws[prec];
    nb::MegaArgs A;
    memset(&A, 0, sizeof(A));
    A.m = h->md();
    A.r = const_cast<void *>(r);
    A.z = z;
    A.bar = ws.bar;
    nb::sw_fill(h, prec, A.sw);
    cudaStream_t st = (cudaStream_t)stream;
    NB_CU(cudaMemsetAsync(ws.bar, 0, nb::BAR_WORDS * sizeof(unsigned int), st), "memset bar");
    NB_CU(NB_POL(prec, nb::launch_cg_sw, h, A, ws.mega_G, true, st), "Schwarz apply");
    return NB_OK;
}

int nb_cg_host(nb_handle *h, const nb_cg_opts *o, const void *b_host, void *x_host, nb_cg_report *rep, void *stream)
{
    if (h && o && o->policy >= NB_FP64 && o->policy <= NB_FP32_DOT2) {
        if (h->nelzl != h->nelz && h->ws[o->policy].peer.nrank == 0)
            return fail(NB_EINVAL, "a slab handle solves with nb_cg_group or after nb_peer_attach");
        int rc0;
        if (h->ws[o->policy].peer.nrank > 0 && (rc0 = mr_args(h, o))) return rc0;
    }
    int rc = cg_args(h, o);
    if (rc) return rc;
    if (!b_host || !x_host) return fail(NB_EINVAL, "NULL host buffer");
    return cg_impl(h, o, b_host, true, x_host, true, rep, (cudaStream_t)stream);
}

int nb_export_maps(const nb_handle *h, int64_t *gid, uint8_t *mask, int32_t *gs_off, int32_t *gs_idx)
{
    if (!h) return fail(NB_EINVAL, "NULL handle");
    NB_CU(cudaSetDevice(h->device), "cudaSetDevice");
    if (gid || mask) {
        int64_t *dg = nullptr;
        uint8_t *dm = nullptr;
        if (gid) NB_CU(cudaMalloc(&dg, sizeof(int64_t) * h->NL), "cudaMalloc");
        if (mask) NB_CU(cudaMalloc(&dm, h->NL), "cudaMalloc");
        NB_CU(nb::launch_maps(h, dg, dm, 0), "maps");
        if (gid) NB_CU(cudaMemcpy(gid, dg, sizeof(int64_t) * h->NL, cudaMemcpyDeviceToHost), "copy gid");
        if (mask) NB_CU(cudaMemcpy(mask, dm, h->NL, cudaMemcpyDeviceToHost), "copy mask");
        cudaFree(dg);
        cudaFree(dm);
    }
    if (gs_off) NB_CU(cudaMemcpy(gs_off, h->gs_off, sizeof(int32_t) * (h->nseg + 1), cudaMemcpyDeviceToHost), "copy off");
    if (gs_idx && h->ncopies)
        NB_CU(cudaMemcpy(gs_idx, h->gs_idx, sizeof(int32_t) * h->ncopies, cudaMemcpyDeviceToHost), "copy idx");
    return NB_OK;
}

int nb_export_geom(const nb_handle *h, double *g6, double *B, double *dinv)
{
    if (!h) return fail(NB_EINVAL, "NULL handle");
    NB_CU(cudaSetDevice(h->device), "cudaSetDevice");
    if (g6) {
        // device layout [e][c][n^3] -> factor-major [c][NL]
        const int64_t n3 = (int64_t)h->n * h->n * h->n;
        std::vector<double> tmp(6 * h->NL);
        NB_CU(cudaMemcpy(tmp.data(), h->g64, sizeof(double) * 6 * h->NL, cudaMemcpyDeviceToHost), "copy g");
        for (int64_t e = 0; e < h->E; e++)
            for (int c = 0; c < 6; c++)
                memcpy(g6 + c * h->NL + e * n3, tmp.data() + (e * 6 + c) * n3, sizeof(double) * n3);
    }
    if (B) NB_CU(cudaMemcpy(B, h->B, sizeof(double) * h->NL, cudaMemcpyDeviceToHost), "copy B");
    if (dinv) NB_CU(cudaMemcpy(dinv, h->dinv64, sizeof(double) * h->NL, cudaMemcpyDeviceToHost), "copy dinv");
    return NB_OK;
}

int nb_export_basis(const nb_handle *h, double *nodes, double *weights, double *D)
{
    if (!h) return fail(NB_EINVAL, "NULL handle");
    const int n = h->n;
    if (nodes) memcpy(nodes, h->nodes, sizeof(double) * n);
    if (weights) memcpy(weights, h->weights, sizeof(double) * n);
    if (D) memcpy(D, h->D, sizeof(double) * n * n);
    return NB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// multi-rank z-slab solves
// ---------------------------------------------------------------------------
int nb_cg_group(nb_handle *const *hs, int32_t nslab, const nb_cg_opts *o, const void *const *b, void *const *x,
                nb_cg_report *reps, void *stream)
{
    if (!hs || !b || !x) return fail(NB_EINVAL, "NULL argument");
    if (nslab < 1 || nslab > nb::NB_MAX_LOCAL) return fail(NB_EINVAL, "nslab must be in [1, 4]");
    int rc;
    for (int r = 0; r < nslab; r++) {
        if ((rc = cg_args(hs[r], o))) return rc;
        if ((rc = mr_args(hs[r], o))) return rc;
        const nb_handle *h = hs[r], *a = hs[0];
        if (h->device != a->device || h->nelx != a->nelx || h->nely != a->nely || h->nelz != a->nelz || h->p != a->p ||
            h->deform != a->deform || h->seed != a->seed)
            return fail(NB_EINVAL, "slabs must be of the same box on the same device");
        if (h->ez0 != (r == 0 ? 0 : hs[r - 1]->ez0 + hs[r - 1]->nelzl))
            return fail(NB_EINVAL, "slabs must be given bottom to top and tile the box");
        if (h->ws[o->policy].peer.nrank > 0) return fail(NB_EINVAL, "a peer-attached slab cannot join a group");
        if ((rc = check_dev_ptr(h, b[r], "b")) || (rc = check_dev_ptr(h, x[r], "x"))) return rc;
    }
    if (hs[nslab - 1]->ez0 + hs[nslab - 1]->nelzl != hs[0]->nelz)
        return fail(NB_EINVAL, "slabs must tile the box");
    if (nslab == 1) return cg_run(hs, 1, o, b, false, x, false, reps, (cudaStream_t)stream);
    return cg_run(hs, nslab, o, b, false, x, false, reps, (cudaStream_t)stream);
}

namespace {
struct PeerBlob {                 // NB_PEER_BLOB_BYTES, one per rank
    cudaIpcMemHandle_t w, ctl;    // 64 + 64 bytes
    int32_t magic, policy, nelx, nely, nelz, p, ez0, nelzl;
    int64_t E;
    int32_t pid, device;
    unsigned char pad[NB_PEER_BLOB_BYTES - 2 * sizeof(cudaIpcMemHandle_t) - 8 * 4 - 8 - 2 * 4];
};
static_assert(sizeof(PeerBlob) == NB_PEER_BLOB_BYTES, "peer blob size");
constexpr int32_t kPeerMagic = 0x6e62706b;
}  // namespace

int nb_peer_export(nb_handle *h, nb_policy policy, void *blob)
{
    if (!h || !blob) return fail(NB_EINVAL, "NULL argument");
    if (policy < NB_FP64 || policy > NB_FP32_DOT2) return fail(NB_EINVAL, "bad policy");
    NB_CU(cudaSetDevice(h->device), "cudaSetDevice");
    int rc;
    if ((rc = ensure_ws(h, policy, 1))) return rc;
    nb::Workspace &ws = h->ws[policy];
    PeerBlob pb;
    memset(&pb, 0, sizeof(pb));
    NB_CU(cudaIpcGetMemHandle(&pb.w, ws.w), "cudaIpcGetMemHandle w");
    NB_CU(cudaIpcGetMemHandle(&pb.ctl, ws.ctl), "cudaIpcGetMemHandle ctl");
    pb.magic = kPeerMagic; pb.policy = policy;
    pb.nelx = h->nelx; pb.nely = h->nely; pb.nelz = h->nelz; pb.p = h->p; pb.ez0 = h->ez0; pb.nelzl = h->nelzl;
    pb.E = h->E;
    pb.pid = (int32_t)getpid();
    pb.device = h->device;
    memcpy(blob, &pb, sizeof(pb));
    return NB_OK;
}

int nb_peer_attach(nb_handle *h, nb_policy policy, int32_t nrank, int32_t rank, const void *blobs)
{
    if (!h || !blobs) return fail(NB_EINVAL, "NULL argument");
    if (policy < NB_FP64 || policy > NB_FP32_DOT2) return fail(NB_EINVAL, "bad policy");
    if (nrank < 1 || nrank > nb::NB_MAX_RANKS || rank < 0 || rank >= nrank) return fail(NB_EINVAL, "bad nrank/rank");
    NB_CU(cudaSetDevice(h->device), "cudaSetDevice");
    int rc;
    if ((rc = ensure_ws(h, policy, 1))) return rc;
    nb::Workspace &ws = h->ws[policy];
    if (ws.peer.nrank > 0) return fail(NB_ESTATE, "already attached (nb_peer_detach first)");
    const PeerBlob *pb = (const PeerBlob *)blobs;
    int32_t z = 0;
    for (int q = 0; q < nrank; q++) {
        if (pb[q].magic != kPeerMagic || pb[q].policy != policy) return fail(NB_EINVAL, "bad peer blob");
        if (pb[q].nelx != h->nelx || pb[q].nely != h->nely || pb[q].nelz != h->nelz || pb[q].p != h->p)
            return fail(NB_EINVAL, "peers hold slabs of another box");
        if (pb[q].ez0 != z) return fail(NB_EINVAL, "peer slabs must be ordered by rank and tile the box");
        z += pb[q].nelzl;
    }
    if (z != h->nelz) return fail(NB_EINVAL, "peer slabs must tile the box");
    if (pb[rank].ez0 != h->ez0 || pb[rank].nelzl != h->nelzl) return fail(NB_EINVAL, "this rank's blob is not this slab");
    nb::PeerState ps;
    auto open = [&](const cudaIpcMemHandle_t &hd, void **out) -> int {
        cudaError_t e = cudaIpcOpenMemHandle(out, hd, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
        ps.opened[ps.nopened++] = *out;
        return NB_OK;
    };
    auto fail_close = [&](int code) {
        for (int i = 0; i < ps.nopened; i++) cudaIpcCloseMemHandle(ps.opened[i]);
        return code;
    };
    const size_t es = vsize(policy), n3 = (size_t)h->n * h->n * h->n;
    for (int q = 0; q < nrank; q++) {
        unsigned char *ctl = nullptr;
        if (q == rank) ctl = ws.ctl;
        else if ((rc = open(pb[q].ctl, (void **)&ctl))) return fail_close(rc);
        ps.flag[q] = (unsigned int *)ctl;
        ps.abrt[q] = (unsigned int *)(ctl + nb::NB_CTL_ABORT_OFF);
        ps.slot[q] = (double *)(ctl + nb::NB_CTL_FLAG_BYTES);
    }
    if (rank > 0) {
        void *w = nullptr;
        if ((rc = open(pb[rank - 1].w, &w))) return fail_close(rc);
        ps.wlo = (const char *)w + es * (size_t)pb[rank - 1].E * n3;
    }
    if (rank + 1 < nrank) {
        void *w = nullptr;
        if ((rc = open(pb[rank + 1].w, &w))) return fail_close(rc);
        ps.whi = (const char *)w - es * (size_t)h->E * n3;
    }
    ps.nrank = nrank;
    ps.rank = rank;
    // flags count from 0: every rank must attach before any rank solves
    NB_CU(cudaMemset(ws.ctl, 0, nb::NB_CTL_BYTES), "memset ctl");
    ps.epoch = 0;
    ws.peer = ps;
    return NB_OK;
}

int nb_peer_detach(nb_handle *h, nb_policy policy)
{
    if (!h) return fail(NB_EINVAL, "NULL handle");
    if (policy < NB_FP64 || policy > NB_FP32_DOT2) return fail(NB_EINVAL, "bad policy");
    NB_CU(cudaSetDevice(h->device), "cudaSetDevice");
    nb::Workspace &ws = h->ws[policy];
    for (int i = 0; i < ws.peer.nopened; i++) cudaIpcCloseMemHandle(ws.peer.opened[i]);
    ws.peer = nb::PeerState();
    return NB_OK;
}
