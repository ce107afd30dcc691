// Microbenchmark: achievable HBM throughput for phase-B-shaped streaming traffic on this GPU
// (read w f32, r f32, dinv f64; write r f32, z f32: 24 B/DOF), persistent grid like the
// megakernel (2 x 256-thread blocks per SM), 8-value pencils per thread, no gather.
// Also the phase-A operand pattern (read 9 f32 streams, write 3).  nvcc -arch=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 2) phase_b_like(const float4 *__restrict__ w, float4 *__restrict__ r,
                                                     float4 *__restrict__ z, const double2 *__restrict__ d,
                                                     long npen, float alpha, double *out)
{
    double acc = 0;
    for (long p = blockIdx.x * 256L + threadIdx.x; p < npen; p += (long)gridDim.x * 256) {
        float4 w0 = __ldcg(w + 2 * p), w1 = __ldcg(w + 2 * p + 1);
        float4 r0 = r[2 * p], r1 = r[2 * p + 1];
        double2 d0 = __ldg(d + 4 * p), d1 = __ldg(d + 4 * p + 1), d2 = __ldg(d + 4 * p + 2), d3 = __ldg(d + 4 * p + 3);
        r0.x -= alpha * w0.x; r0.y -= alpha * w0.y; r0.z -= alpha * w0.z; r0.w -= alpha * w0.w;
        r1.x -= alpha * w1.x; r1.y -= alpha * w1.y; r1.z -= alpha * w1.z; r1.w -= alpha * w1.w;
        float4 z0 = make_float4(r0.x * d0.x, r0.y * d0.y, r0.z * d1.x, r0.w * d1.y);
        float4 z1 = make_float4(r1.x * d2.x, r1.y * d2.y, r1.z * d3.x, r1.w * d3.y);
        acc += (double)r0.x * z0.x + (double)r1.w * z1.w;
        r[2 * p] = r0; r[2 * p + 1] = r1;
        z[2 * p] = z0; z[2 * p + 1] = z1;
    }
    if (acc == 12345.0) out[0] = acc;
}

__global__ void copy_like(const float4 *__restrict__ a, float4 *__restrict__ b, long n)
{
    for (long i = blockIdx.x * 256L + threadIdx.x; i < n; i += (long)gridDim.x * 256) b[i] = a[i];
}

int main()
{
    const long NL = 16777216;   // 32^3 p=7
    const long npen = NL / 8;
    float4 *w, *r, *z, *a, *b;
    double2 *d;
    double *out;
    cudaMalloc(&w, NL * 4); cudaMalloc(&r, NL * 4); cudaMalloc(&z, NL * 4); cudaMalloc(&d, NL * 8);
    cudaMalloc(&a, NL * 16); cudaMalloc(&b, NL * 16); cudaMalloc(&out, 8);
    cudaMemset(w, 0, NL * 4); cudaMemset(r, 0, NL * 4); cudaMemset(d, 0, NL * 8); cudaMemset(a, 0, NL * 16);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int grid_mult : {2, 4, 8}) {
        for (int it = 0; it < 3; it++) phase_b_like<<<sms * grid_mult, 256>>>((float4 *)w, r, z, d, npen, 0.5f, out);
        cudaEventRecord(e0);
        for (int it = 0; it < 20; it++) phase_b_like<<<sms * grid_mult, 256>>>((float4 *)w, r, z, d, npen, 0.5f, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("phase-B-like grid=%d x 256: %.1f us/launch, %.0f GB/s (24 B/DOF)\n", sms * grid_mult, 1e3 * ms / 20,
               24.0 * NL / (ms * 1e-3 / 20) / 1e9);
    }
    for (int it = 0; it < 3; it++) copy_like<<<sms * 8, 256>>>(a, b, NL);
    cudaEventRecord(e0);
    for (int it = 0; it < 20; it++) copy_like<<<sms * 8, 256>>>(a, b, NL);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 256 MB: %.1f us, %.0f GB/s (read+write)\n", 1e3 * ms / 20, 2.0 * 16 * NL / (ms * 1e-3 / 20) / 1e9);
    return 0;
}
