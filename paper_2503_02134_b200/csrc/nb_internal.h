// nb_internal.h -- private declarations shared by the host layer (nb_api.cu) and the
// kernel translation unit (nb_kernels.cu).  No torch, no oracle.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "nb.h"

namespace nb {

// Device-resident CG scalars.  Values of the policy's scalar
// precision (float under NB_FP32, double otherwise) are stored widened to double.
struct Scal {
    double rho;        // rho_k = glsc3(r, c, z) of the current iteration
    double beta;       // beta_k used by the p update of the current iteration
    double alpha;      // alpha_k
    double pap;        // pap_k
    double rtr;        // rtr_k after the update
    double rtr0;
    double rtol;
    int32_t iter;      // completed iterations
    int32_t max_iter;
    int32_t done;      // 1: no further updates
    int32_t status;    // NB_CONVERGED / NB_MAXITER / NB_BROKEDOWN (stagnation decided on host)
    uint32_t cnt_gs;   // last-block-done counters
    uint32_t cnt_upd;
    uint32_t cnt_init;
    uint32_t pad;
};

// Geometry/maps needed by kernels, passed by value.
struct MeshDev {
    int32_t nelx, nely, nelz, p, n;
    int64_t E, NL, NX, NY, NZ, NG;
    int32_t nseg;
};

struct Workspace {          // per-policy CG workspace (lazily allocated)
    bool ready = false;
    void *r = nullptr, *p = nullptr, *w = nullptr, *x = nullptr;
    double *part = nullptr;     // per-block partials (2 slots per block)
    Scal *scal = nullptr;       // device scalars
    Scal *scal_host = nullptr;  // pinned mirror
    double *hist = nullptr;     // device history, capacity hist_cap
    int32_t hist_cap = 0;
    // conditional-while graph cache
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int32_t graph_order = -1;
};

}  // namespace nb

struct nb_handle {
    int32_t device;
    int32_t nelx, nely, nelz, p, n;
    int64_t E, NL, NX, NY, NZ, NG;
    int64_t n_unmasked, nseg, ncopies;
    double deform;
    uint64_t seed;
    double nodes[16], weights[16], D[256];
    int sm_count;
    // device data owned by the handle
    double *g64 = nullptr;      // [E][6][n^3]
    float *g32 = nullptr;       // one-time cast, lazily
    double *B = nullptr;        // [NL]
    double *dinv64 = nullptr;   // [NL]
    float *dinv32 = nullptr;    // lazily
    int32_t *gs_off = nullptr;  // [nseg+1]
    int32_t *gs_idx = nullptr;  // [ncopies]
    int32_t *flag = nullptr;    // device error flags for setup checks
    cudaStream_t cap_stream = nullptr;   // private stream used for graph capture
    nb::Workspace ws[3];
    nb::MeshDev md() const {
        nb::MeshDev m;
        m.nelx = nelx; m.nely = nely; m.nelz = nelz; m.p = p; m.n = n;
        m.E = E; m.NL = NL; m.NX = NX; m.NY = NY; m.NZ = NZ; m.NG = NG;
        m.nseg = (int32_t)nseg;
        return m;
    }
};

namespace nb {

// C-3 deformation phases phi_a = pi (1 + U(seed, 3, a)) (host, nb_api.cu)
void deform_phases(uint64_t seed, double ph[3]);

// ---- launchers implemented in nb_kernels.cu (all asynchronous on `st`) ----
cudaError_t upload_basis(int n, const double *D);
cudaError_t launch_geometry(const nb_handle *h, const double phi[3], cudaStream_t st);
cudaError_t launch_jacobi(nb_handle *h, double *diag_scratch, cudaStream_t st);
cudaError_t build_gs(nb_handle *h, cudaStream_t st);   // allocates gs_off/gs_idx (synchronizes)
cudaError_t launch_cast(const double *src, float *dst, int64_t n, cudaStream_t st);
cudaError_t launch_maps(const nb_handle *h, int64_t *gid, uint8_t *mask, cudaStream_t st);
cudaError_t launch_rhs(const nb_handle *h, int kind, double noise, uint64_t seed, int prec,
                       void *b, cudaStream_t st);
cudaError_t launch_ax(const nb_handle *h, int prec, const void *u, void *w, bool local, cudaStream_t st);
cudaError_t launch_dssum(const nb_handle *h, int prec, int order, void *u, cudaStream_t st);

// CG pieces
int grid_ax(const nb_handle *h, int prec);
int grid_gs(const nb_handle *h);
int grid_upd(const nb_handle *h, int prec);
cudaError_t launch_cg_init(const nb_handle *h, int prec, Workspace &ws, const void *b, cudaStream_t st);
cudaError_t launch_cg_ax(const nb_handle *h, int prec, Workspace &ws, cudaStream_t st);
cudaError_t launch_cg_gs(const nb_handle *h, int prec, int order, Workspace &ws, cudaStream_t st,
                         cudaGraphConditionalHandle cond, bool use_cond);
cudaError_t launch_cg_upd(const nb_handle *h, int prec, Workspace &ws, cudaStream_t st,
                          cudaGraphConditionalHandle cond, bool use_cond);

}  // namespace nb
