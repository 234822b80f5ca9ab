// Per-SM memory feed probe (development aid): how many bytes/clock one SM can read from / write to
// L2-resident data with plain 16-byte loads/stores and with TMA bulk copies, when `nsm` SMs run
// the same loop.  This is the per-SM roofline that bounds kernels running on a few-SM budget.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sm_feed_probe sm_feed_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__global__ void rd(const uint4* __restrict__ src, size_t n_per_block, int reps, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const uint4* p = src + blockIdx.x * n_per_block;
  for (int r = 0; r < reps; ++r)
    for (size_t i = threadIdx.x; i < n_per_block; i += blockDim.x * 4) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = (i + u * blockDim.x < n_per_block) ? p[i + u * blockDim.x] : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc.x ^= v[u].x, acc.y ^= v[u].y, acc.z ^= v[u].z, acc.w ^= v[u].w;
    }
  if (acc.x == 0x12345678) sink[threadIdx.x] = acc;
}

__global__ void wr(uint4* __restrict__ dst, size_t n_per_block, int reps) {
  uint4* p = dst + blockIdx.x * n_per_block;
  for (int r = 0; r < reps; ++r)
    for (size_t i = threadIdx.x; i < n_per_block; i += blockDim.x) p[i] = make_uint4(r, i, 0, 0);
}

__global__ void bulk_rd(const char* __restrict__ src, size_t bytes_per_block, int reps, unsigned chunk, int infl) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    unsigned phase = 0;
    const char* p = src + blockIdx.x * bytes_per_block;
    for (int r = 0; r < reps; ++r)
      for (size_t off = 0; off + infl * chunk <= bytes_per_block; off += infl * chunk) {
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(infl * chunk));
        for (int j = 0; j < infl; ++j)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  static_cast<unsigned>(__cvta_generic_to_shared(sm + j * chunk))),
              "l"(p + off + j * chunk), "r"(chunk), "r"(b)
              : "memory");
        unsigned done = 0;
        while (!done)
          asm volatile(
              "{ .reg .pred q; mbarrier.try_wait.parity.shared.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
              : "=r"(done)
              : "r"(b), "r"(phase));
        phase ^= 1;
      }
  }
}

// TMA bulk stores (smem -> global), `infl` groups of `chunk` bytes in flight; with `rd_too` a second
// warp streams bulk reads at the same time (the read+write mix of a conv epilogue).
__global__ void bulk_wr(char* __restrict__ dst, const char* __restrict__ src, size_t bytes_per_block, int reps,
                        unsigned chunk, int infl, int rd_too) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    char* p = dst + blockIdx.x * bytes_per_block;
    for (int r = 0; r < reps; ++r)
      for (size_t off = 0; off + infl * chunk <= bytes_per_block; off += infl * chunk) {
        for (int j = 0; j < infl; ++j)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + off + j * chunk),
                       "r"(static_cast<unsigned>(__cvta_generic_to_shared(sm + j * chunk))), "r"(chunk)
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  if (warp == 1 && lane == 0 && rd_too) {
    char* rbuf = sm + 4 * 32768;
    unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    unsigned phase = 0;
    const char* p = src + blockIdx.x * bytes_per_block;
    for (int r = 0; r < reps; ++r)
      for (size_t off = 0; off + 2 * 32768 <= bytes_per_block; off += 2 * 32768) {
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(2 * 32768));
        for (int j = 0; j < 2; ++j)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  static_cast<unsigned>(__cvta_generic_to_shared(rbuf + j * 32768))),
              "l"(p + off + j * 32768), "r"(32768u), "r"(b)
              : "memory");
        unsigned done = 0;
        while (!done)
          asm volatile(
              "{ .reg .pred q; mbarrier.try_wait.parity.shared.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
              : "=r"(done)
              : "r"(b), "r"(phase));
        phase ^= 1;
      }
  }
}

int main(int argc, char** argv) {
  const int nsm_list[] = {1, 3, 8, 148};
  const size_t per_block = 8u << 20;  // 8 MB per block, L2-resident after the first rep for small nsm
  char* buf;
  cudaMalloc(&buf, per_block * 148 + (1 << 20));
  cudaMemset(buf, 1, per_block * 148);
  uint4* sink;
  cudaMalloc(&sink, 4096 * sizeof(uint4));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  cudaFuncSetAttribute(bulk_rd, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int nsm : nsm_list) {
    const int reps = nsm <= 8 ? 8 : 2;
    for (int kind = 0; kind < 3; ++kind) {
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(e0);
        if (kind == 0) rd<<<nsm, 1024>>>(reinterpret_cast<uint4*>(buf), per_block / 16, reps, sink);
        if (kind == 1) wr<<<nsm, 1024>>>(reinterpret_cast<uint4*>(buf), per_block / 16, reps);
        if (kind == 2) bulk_rd<<<nsm, 32, 4 * 32768>>>(buf, per_block, reps, 32768, 4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it == 1) {
          const double bytes = static_cast<double>(per_block) * reps * nsm;
          const double gbs = bytes / (ms * 1e-3) / 1e9;
          printf("nsm=%3d %-10s %8.1f GB/s total  %7.1f GB/s/SM  %5.1f B/clk/SM (@%d MHz)\n", nsm,
                 kind == 0 ? "ld.v4" : kind == 1 ? "st.v4" : "bulk-copy", gbs, gbs / nsm,
                 gbs * 1e9 / nsm / (1965e6), clk_khz / 1000);
        }
      }
    }
  }
  // request-size / in-flight sweep on 1 and 3 SMs: is a bulk copy's cost per byte or per request?
  cudaFuncSetAttribute(bulk_rd, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int nsm : {1, 3}) {
    for (unsigned chunk : {4096u, 8192u, 16384u, 32768u, 65536u}) {
      for (int infl : {1, 2, 4, 8}) {
        if (chunk * infl > 196608u) continue;
        float ms = 0;
        for (int it = 0; it < 2; ++it) {
          cudaEventRecord(e0);
          bulk_rd<<<nsm, 32, 200 * 1024>>>(buf, per_block, 4, chunk, infl);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms, e0, e1);
        }
        const double bytes = static_cast<double>(per_block / (chunk * infl) * (chunk * infl)) * 4 * nsm;
        const double gbs = bytes / (ms * 1e-3) / 1e9;
        printf("bulk nsm=%d chunk=%6u inflight=%d: %6.1f GB/s/SM %5.1f B/clk/SM  %6.0f clk/request\n", nsm, chunk, infl,
               gbs / nsm, gbs * 1e9 / nsm / 1965e6, chunk * infl / (gbs * 1e9 / nsm / 1965e6) / infl);
      }
    }
  }
  // TMA bulk stores per SM, alone and with a concurrent bulk-read stream
  cudaFuncSetAttribute(bulk_wr, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
  char* buf2;
  cudaMalloc(&buf2, per_block * 148 + (1 << 20));
  for (int nsm : {1, 2, 3}) {
    for (int rd_too : {0, 1}) {
      for (unsigned chunk : {4096u, 16384u, 32768u}) {
        for (int infl : {1, 2, 4}) {
          if (chunk * infl > 131072u) continue;
          float ms = 0;
          for (int it = 0; it < 2; ++it) {
            cudaEventRecord(e0);
            bulk_wr<<<nsm, 64, 6 * 32768>>>(buf2, buf, per_block, 4, chunk, infl, rd_too);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
          }
          const double wbytes = static_cast<double>(per_block / (chunk * infl) * (chunk * infl)) * 4 * nsm;
          const double gbs = wbytes / (ms * 1e-3) / 1e9;
          const double rgbs = rd_too ? static_cast<double>(per_block) * 4 * nsm / (ms * 1e-3) / 1e9 : 0.0;
          printf("bulk-store nsm=%d chunk=%6u inflight=%d %s: write %6.1f GB/s/SM %5.1f B/clk/SM  (read stream bound: "
                 "%5.1f B/clk/SM)\n", nsm, chunk, infl, rd_too ? "+read " : "alone", gbs / nsm, gbs * 1e9 / nsm / 1965e6,
                 rgbs * 1e9 / nsm / 1965e6);
        }
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
