// tcgen05.mma issue-rate probe (development aid): cycles per M=128 x N x K=16 bf16 MMA issued
// back to back by one thread from shared-memory operands (SS mode), for N = 16..256, with the A
// descriptor 1024-byte aligned (a normal k-block) or starting at a 128-byte row inside a swizzle
// atom (the halo conv's shifted taps).  No loads, no epilogue: the tensor pipe alone.  One CTA per
// SM on `nsm` SMs; operands are zeros (timing does not depend on values).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2312_10636_b200/csrc -o mma_probe mma_probe.cu
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "gx_ptx.cuh"

using namespace gx;

constexpr int kABytes = 9 * 128 * 128;  // room for 128 rows + shifted starts (halo-like region)
constexpr int kBBytes = 256 * 128;

__global__ void __launch_bounds__(128, 1) mma_probe(int N, int iters, int row_shift, int kslices,
                                                   unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kABytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + kBBytes);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (kABytes + kBBytes) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(tslot, 256);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = *tslot;
  if (warp == 0) {
    const bool issuer = elect_one();
    const uint32_t idesc = umma_idesc_bf16(128, N);
    const uint32_t abase = smem_u32(sA);
    const uint64_t bd = umma_desc_sw128(sB);
    uint32_t ph = 0;
    unsigned long long t0 = 0, t1 = 0;
    for (int rep = 0; rep < 2; ++rep) {  // rep 0 warms up
      if (issuer) {
        t0 = clock64();
        for (int i = 0; i < iters; ++i) {
          // a "tap": the A tile at row offset (i % 9) * row_shift rows, K slices of 16
          const uint32_t a_addr = abase + static_cast<uint32_t>((i % 9) * row_shift) * 128u;
          const uint64_t ad = ((static_cast<uint64_t>(a_addr) >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) |
                              (1ull << 46) | (2ull << 61);
          for (int kk = 0; kk < kslices; ++kk) umma_bf16(d, ad + 2 * kk, bd + 2 * kk, idesc, (i | kk) != 0);
        }
        umma_commit(bar);
      }
      __syncwarp();
      mbar_wait(bar, ph);
      ph ^= 1;
      tc_fence_after();
      if (issuer) t1 = clock64();
      __syncwarp();
    }
    if (issuer) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(d, 256);
}

int main(int argc, char** argv) {
  const int nsm = argc > 1 ? atoi(argv[1]) : 1;
  const int iters = argc > 2 ? atoi(argv[2]) : 2048;
  const int smem = kABytes + kBBytes + 1024 + 64;
  cudaFuncSetAttribute(mma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* dout = nullptr;
  cudaMalloc(&dout, nsm * sizeof(unsigned long long));
  unsigned long long* hout = static_cast<unsigned long long*>(malloc(nsm * sizeof(unsigned long long)));
  printf("# M=128 x N x K=16 bf16 tcgen05.mma (SS mode), %d MMA groups per run, %d CTA(s) (1 per SM)\n", iters, nsm);
  printf("# floor (guide): 128*N/256 cycles per MMA\n");
  printf("%6s %9s %7s %14s %10s\n", "N", "row_shift", "kslices", "cycles/MMA", "floor");
  const int Ns[] = {16, 32, 64, 128, 256};
  for (int shift = 0; shift <= 1; ++shift)
    for (int ks : {4, 1})
      for (int N : Ns) {
        mma_probe<<<nsm, 128, smem>>>(N, iters, shift, ks, dout);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(hout, dout, nsm * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < nsm; ++i) mx = hout[i] > mx ? hout[i] : mx;
        printf("%6d %9d %7d %14.1f %10.1f\n", N, shift, ks, static_cast<double>(mx) / (iters * ks), 128.0 * N / 256);
      }
  return 0;
}
