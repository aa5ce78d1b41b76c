// host->device bandwidth: DMA (cudaMemcpyAsync from pinned memory) vs zero-copy SM reads (mapped pinned)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_read(const float4 *__restrict__ src, float4 *__restrict__ dst, long long n)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
}
int main()
{
    const size_t bytes = 256ull << 20;
    float *h, *d, *hd;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaMalloc(&d, bytes);
    cudaHostGetDevicePointer(&hd, h, 0);
    for (size_t i = 0; i < bytes / 4; i++) h[i] = 1.0f;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(a);
        cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("DMA memcpy H2D: %.1f GB/s\n", bytes / ms / 1e6);
        for (int g : {148 * 4, 148 * 16, 148 * 64}) {
            cudaEventRecord(a);
            k_read<<<g, 256>>>((const float4 *)hd, (float4 *)d, bytes / 16);
            cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
            printf("zero-copy SM reads (grid %d): %.1f GB/s\n", g, bytes / ms / 1e6);
        }
    }
    return 0;
}
