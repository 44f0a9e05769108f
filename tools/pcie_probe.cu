// PCIe device-to-host probe (tools/pcie_probe.cu): DMA copies of 276 MB (one C3 frame's planes) to
// pinned memory, split copies, two streams, SM stores into mapped memory, DMA under HBM load.
// nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o pcie_probe tools/pcie_probe.cu; e2e tracks this rate.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__global__ void store_kernel(float4* __restrict__ dst, const float4* __restrict__ src, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) dst[i] = src[i];
}
int main() {
  const size_t bytes = 276480000;
  void *d, *h, *hm;
  CK(cudaMalloc(&d, bytes));
  CK(cudaMemset(d, 1, bytes));
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocDefault));
  CK(cudaHostAlloc(&hm, bytes, cudaHostAllocMapped));
  memset(h, 0, bytes); memset(hm, 0, bytes);
  void* hmd; CK(cudaHostGetDevicePointer(&hmd, hm, 0));
  cudaStream_t s1, s2; CK(cudaStreamCreate(&s1)); CK(cudaStreamCreate(&s2));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a, s1);
    CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s1));
    cudaEventRecord(b, s1); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("dma 1 copy: %.3f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
  }
  for (int nb : {2, 4, 8, 32}) {
    cudaEventRecord(a, s1);
    for (int i = 0; i < nb; ++i) CK(cudaMemcpyAsync((char*)h + bytes / nb * i, (char*)d + bytes / nb * i, bytes / nb, cudaMemcpyDeviceToHost, s1));
    cudaEventRecord(b, s1); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("dma %d copies 1 stream: %.3f ms %.1f GB/s\n", nb, ms, bytes / ms / 1e6);
  }
  {  // two streams, halves
    cudaEventRecord(a, s1); cudaStreamWaitEvent(s2, a, 0);
    CK(cudaMemcpyAsync(h, d, bytes / 2, cudaMemcpyDeviceToHost, s1));
    CK(cudaMemcpyAsync((char*)h + bytes / 2, (char*)d + bytes / 2, bytes / 2, cudaMemcpyDeviceToHost, s2));
    cudaEvent_t c; cudaEventCreate(&c); cudaEventRecord(c, s2); cudaStreamWaitEvent(s1, c, 0);
    cudaEventRecord(b, s1); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("dma 2 streams: %.3f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
  }
  for (int grid : {148, 296, 592, 1184}) for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a, s1);
    store_kernel<<<grid, 256, 0, s1>>>((float4*)hmd, (const float4*)d, bytes / 16);
    cudaEventRecord(b, s1); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    printf("sm stores grid %d: %.3f ms %.1f GB/s\n", grid, ms, bytes / ms / 1e6);
  }
  {  // dma with compute running concurrently
    float4* d2; CK(cudaMalloc(&d2, bytes));
    cudaEventRecord(a, s1);
    CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s1));
    cudaEventRecord(b, s1);
    for (int i = 0; i < 20; ++i) store_kernel<<<1184, 256, 0, s2>>>(d2, (const float4*)d, bytes / 16);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("dma under HBM load: %.3f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
    cudaDeviceSynchronize();
  }
  return 0;
}
