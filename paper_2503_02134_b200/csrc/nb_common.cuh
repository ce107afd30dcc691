// nb_common.cuh -- device-side building blocks for the sm_100a kernels.
//
// Precision policies:
//   TV: vector storage and local-Ax arithmetic   TG: gather-scatter accumulation
//   TS: glsc3 accumulation and CG scalars        TJ: Jacobi inverse diagonal
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "nb.h"
#include "nb_internal.h"

namespace nb {

template <int PREC> struct Pol;
template <> struct Pol<NB_FP64> { using TV = double; using TG = double; using TS = double; using TJ = double; };
template <> struct Pol<NB_FP32> { using TV = float;  using TG = float;  using TS = float;  using TJ = float; };
template <> struct Pol<NB_MIXED> { using TV = float; using TG = double; using TS = double; using TJ = double; };

// ---------------------------------------------------------------------------
// GLL derivative matrix in constant memory, one n*n block per order (n = 2..16).
// Indices are compile-time constants after unrolling, so every D entry is a
// constant-bank operand of the FMA (no register or shared-memory traffic).
// ---------------------------------------------------------------------------
// (defined here: this header is included by exactly one translation unit, nb_kernels.cu)
__constant__ double c_D64[17 * 256];
__constant__ float c_D32[17 * 256];

template <typename T> __device__ __forceinline__ T cD(int i);
template <> __device__ __forceinline__ double cD<double>(int i) { return c_D64[i]; }
template <> __device__ __forceinline__ float cD<float>(int i) { return c_D32[i]; }

// D[row][col] for order N (D[i][j] = l_j'(x_i))
template <typename T, int N> __device__ __forceinline__ T Dm(int row, int col) { return cD<T>(N * 256 + row * N + col); }

// o[i] = sum_l D[i][l] v[l]  (local_grad3 direction)
template <typename T, int N>
__device__ __forceinline__ void contract(const T (&v)[N], T (&o)[N])
{
#pragma unroll
    for (int i = 0; i < N; i++) {
        T s = Dm<T, N>(i, 0) * v[0];
#pragma unroll
        for (int l = 1; l < N; l++) s = fma(Dm<T, N>(i, l), v[l], s);
        o[i] = s;
    }
}
// o[i] = sum_l D[l][i] v[l]  (local_grad3_t direction)
template <typename T, int N>
__device__ __forceinline__ void contract_t(const T (&v)[N], T (&o)[N])
{
#pragma unroll
    for (int i = 0; i < N; i++) {
        T s = Dm<T, N>(0, i) * v[0];
#pragma unroll
        for (int l = 1; l < N; l++) s = fma(Dm<T, N>(l, i), v[l], s);
        o[i] = s;
    }
}

// ---------------------------------------------------------------------------
// pencil (N contiguous values) loads/stores with the widest aligned vector type
// ---------------------------------------------------------------------------
template <typename T, int N> struct VecW {
    static constexpr int bytes = (int)sizeof(T);
    static constexpr int V = (bytes == 4) ? ((N % 4 == 0) ? 4 : (N % 2 == 0 ? 2 : 1)) : ((N % 2 == 0) ? 2 : 1);
};
template <typename T, int V> struct VT { using type = T; };
template <> struct VT<float, 4> { using type = float4; };
template <> struct VT<float, 2> { using type = float2; };
template <> struct VT<double, 2> { using type = double2; };

template <typename T, int V> struct VAcc;
template <typename T> struct VAcc<T, 1> {
    static __device__ __forceinline__ void get(const T &s, T *d) { d[0] = s; }
    static __device__ __forceinline__ T put(const T *d) { return d[0]; }
};
template <> struct VAcc<float, 2> {
    static __device__ __forceinline__ void get(const float2 &s, float *d) { d[0] = s.x; d[1] = s.y; }
    static __device__ __forceinline__ float2 put(const float *d) { return make_float2(d[0], d[1]); }
};
template <> struct VAcc<float, 4> {
    static __device__ __forceinline__ void get(const float4 &s, float *d) { d[0] = s.x; d[1] = s.y; d[2] = s.z; d[3] = s.w; }
    static __device__ __forceinline__ float4 put(const float *d) { return make_float4(d[0], d[1], d[2], d[3]); }
};
template <> struct VAcc<double, 2> {
    static __device__ __forceinline__ void get(const double2 &s, double *d) { d[0] = s.x; d[1] = s.y; }
    static __device__ __forceinline__ double2 put(const double *d) { return make_double2(d[0], d[1]); }
};

template <typename T, int N>
__device__ __forceinline__ void ld_pencil(const T *__restrict__ src, T (&v)[N])
{
    constexpr int V = VecW<T, N>::V;
    using W = typename VT<T, V>::type;
    const W *s = reinterpret_cast<const W *>(src);
#pragma unroll
    for (int c = 0; c < N / V; c++) {
        W t = s[c];
        VAcc<T, V>::get(t, &v[c * V]);
    }
}
template <typename T, int N>
__device__ __forceinline__ void ld_pencil_stream(const T *__restrict__ src, T (&v)[N])
{
    constexpr int V = VecW<T, N>::V;
    using W = typename VT<T, V>::type;
    const W *s = reinterpret_cast<const W *>(src);
#pragma unroll
    for (int c = 0; c < N / V; c++) {
        W t = __ldcs(s + c);
        VAcc<T, V>::get(t, &v[c * V]);
    }
}
template <typename T, int N>
__device__ __forceinline__ void st_pencil(T *__restrict__ dst, const T (&v)[N])
{
    constexpr int V = VecW<T, N>::V;
    using W = typename VT<T, V>::type;
    W *d = reinterpret_cast<W *>(dst);
#pragma unroll
    for (int c = 0; c < N / V; c++) d[c] = VAcc<T, V>::put(&v[c * V]);
}

// ---------------------------------------------------------------------------
// lattice helpers: multiplicity and mask are analytic on the box
// ---------------------------------------------------------------------------
struct ElemPos {
    int32_t ex, ey, ez;
};
__device__ __forceinline__ ElemPos elem_pos(const MeshDev &m, int64_t e)
{
    ElemPos r;
    int64_t t = e / m.nelx;
    r.ex = (int32_t)(e - t * m.nelx);
    r.ey = (int32_t)(t % m.nely);
    r.ez = (int32_t)(t / m.nely);
    return r;
}
// multiplicity factor along one axis for local index i of element coordinate ex (nel elements)
__device__ __forceinline__ int axis_mult(int i, int n, int ex, int nel)
{
    return ((i == 0 && ex > 0) || (i == n - 1 && ex < nel - 1)) ? 2 : 1;
}
__device__ __forceinline__ bool axis_bnd(int i, int n, int ex, int nel)
{
    return (i == 0 && ex == 0) || (i == n - 1 && ex == nel - 1);
}

// ---------------------------------------------------------------------------
// deterministic reductions: warp shuffle tree -> shared -> one value per block
// (blockDim.x must be a multiple of 32)
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_sum(T v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}
template <typename T>
__device__ __forceinline__ T block_sum(T v, T *sh)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    T r = 0;
    if (wid == 0) {
        r = (lane < nw) ? sh[lane] : T(0);
        r = warp_sum(r);
    }
    return r;  // valid in thread 0
}
// sum of n values (fixed order: thread-strided sequential, then tree), all threads of the block
template <typename T>
__device__ __forceinline__ T block_sum_array(const double *src, int n, int stride, T *sh)
{
    T v = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) v += (T)__ldcg(src + (int64_t)i * stride);
    return block_sum<T>(v, sh);
}

// last-block-done election: returns true in every thread of the last block to finish
__device__ __forceinline__ bool last_block(uint32_t *cnt)
{
    __shared__ bool am_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t prev = atomicAdd(cnt, 1u);
        am_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (am_last) __threadfence();
    return am_last;
}

// ---------------------------------------------------------------------------
// counter-based SplitMix64; the CUDA path's own implementation
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix(uint64_t seed, uint64_t stream, uint64_t i)
{
    uint64_t z = (seed ^ (stream * 0xD1B54A32D192ED03ull)) + (i + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double unif(uint64_t seed, uint64_t stream, uint64_t i)
{
    return (double)(splitmix(seed, stream, i) >> 11) * 0x1.0p-52 - 1.0;
}

}  // namespace nb
