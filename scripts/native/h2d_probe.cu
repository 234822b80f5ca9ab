// H2D ingress probe (development aid): DMA copy rate vs chunk size, and zero-copy kernel reads of
// mapped pinned memory (the "fused ingress" alternative).  nvcc -O2 -arch=sm_100a h2d_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__global__ void zc_read(const float4* __restrict__ src, __nv_bfloat162* __restrict__ dst, long n4) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    float4 v = src[i];
    dst[2 * i] = __floats2bfloat162_rn(v.x, v.y);
    dst[2 * i + 1] = __floats2bfloat162_rn(v.z, v.w);
  }
}

int main() {
  const size_t maxb = 64ull << 20;
  float* h;
  cudaHostAlloc(&h, maxb * 4, cudaHostAllocMapped);
  for (size_t i = 0; i < maxb; ++i) h[i] = 1.0f;
  float* d;
  cudaMalloc(&d, maxb * 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double mbs[] = {0.2, 0.6, 1.6, 3.2, 16};
  for (double mb : mbs) {
    size_t bytes = ((size_t)(mb * (1 << 20))) & ~(size_t)255;
    int iters = 400;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a, s);
      for (int i = 0; i < iters; ++i)
        cudaMemcpyAsync((char*)d + (i % 8) * bytes, (char*)h + (i % 8) * bytes, bytes, cudaMemcpyHostToDevice, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("DMA  chunk %5.1f MB: %6.1f GB/s  %7.1f us/copy\n", mb, bytes * (double)iters / ms / 1e6, ms * 1000 / iters);
  }
  float* hd;
  cudaHostGetDevicePointer(&hd, h, 0);
  for (double mb : mbs) {
    size_t bytes = ((size_t)(mb * (1 << 20))) & ~(size_t)255;
    long n4 = bytes / 16;
    for (int grid : {16, 64, 148, 592}) {
      int iters = 100;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a, s);
        for (int i = 0; i < iters; ++i)
          zc_read<<<grid, 256, 0, s>>>((const float4*)((char*)hd + (i % 8) * bytes), (__nv_bfloat162*)d, n4);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("ZC   chunk %5.1f MB grid %3d: %6.1f GB/s  %7.1f us/read\n", mb, grid, bytes * (double)iters / ms / 1e6,
             ms * 1000 / iters);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
