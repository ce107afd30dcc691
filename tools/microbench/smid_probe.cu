// smid_probe.cu -- which SM each block of a full cooperative grid lands on (the per-SM split of
// the megakernel, grp_range in nb_cg.cuh, assumes block i and block i + #SMs share an SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o smid_probe smid_probe.cu && ./smid_probe
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 2) k(int *smid)
{
    extern __shared__ char sm[];
    if (threadIdx.x == 0) {
        unsigned s;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        smid[blockIdx.x] = (int)s;
    }
}
int main()
{
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int S = p.multiProcessorCount, smem = 40 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, smem);
    const int G = S * occ;
    int *d, *h = new int[G];
    cudaMalloc(&d, G * sizeof(int));
    void *args[1] = {&d};
    for (int rep = 0; rep < 3; rep++) {
        cudaLaunchCooperativeKernel((void *)k, dim3(G), dim3(256), args, smem, 0);
        cudaMemcpy(h, d, G * sizeof(int), cudaMemcpyDeviceToHost);
        int same = 0, adj = 0, mx = 0;
        for (int i = 0; i + S < G; i++) same += h[i] == h[i + S];
        for (int i = 0; i + 1 < G; i += 2) adj += h[i] == h[i + 1];
        for (int i = 0; i < G; i++) mx = h[i] > mx ? h[i] : mx;
        printf("rep %d: SMs %d occ %d grid %d: blocks i and i+S on one SM: %d of %d; blocks 2j and 2j+1 on one SM: %d of %d; max smid %d\n",
               rep, S, occ, G, same, G - S, adj, G / 2, mx);
    }
    printf("first 16 smids:");
    for (int i = 0; i < 16; i++) printf(" %d", h[i]);
    printf("\nsmids of blocks S..S+15:");
    for (int i = S; i < S + 16 && i < G; i++) printf(" %d", h[i]);
    printf("\n");
    return 0;
}
