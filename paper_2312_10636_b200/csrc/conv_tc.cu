// K2/K3: implicit-GEMM convolution (and token-wise linear) on 5th-gen tensor cores.
//
//   D[M, N] = im2col(X)[M, K] * W[N, K]^T  (+ bias, + residual, act)   M = k*Ho*Wo, N = Cout
//
// Warp-specialised persistent kernel, one CTA per SM, grid bounded by the stage's SM budget:
//   warps 0-3  A producers: im2col rows gathered with cp.async (16 B, zero-fill for padding)
//              straight into the 128B-swizzled K-major layout UMMA expects;
//   warp 4     B producer: TMA 2D tile loads of the packed weights (SWIZZLE_128B) + TMEM owner;
//   warp 5     MMA issuer: one thread issues tcgen05.mma (M=128, N=BN, K=16) into TMEM;
//   warps 6-9  epilogue: tcgen05.ld -> bias/residual/activation -> bf16 (or fp32) stores.
// Smem ring of `stages` (A,B) slots with full/empty mbarriers; two TMEM accumulators so the
// epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda_bf16.h>

#include "gx_internal.h"
#include "gx_ptx.cuh"

namespace gx {

namespace {
constexpr int kLag = 2;  // cp.async groups in flight per producer thread before signalling
constexpr int kATileBytes = kBM * kBK * 2;

__device__ __forceinline__ float gelu_erf(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

__global__ void __launch_bounds__(kConvThreads, 1) conv_tc_kernel(const __grid_constant__ CUtensorMap wmap,
                                                                   const ConvArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S_ = a.stages;
  const int BN = a.BN;
  const uint32_t b_bytes = static_cast<uint32_t>(BN) * 128u;
  uint8_t* sA = smem;
  uint8_t* sB = sA + static_cast<size_t>(S_) * kATileBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + static_cast<size_t>(S_) * b_bytes);
  uint64_t* empty = full + S_;
  uint64_t* tfull = empty + S_;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  int2* ktab = reinterpret_cast<int2*>(tslot + 4);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  // K-chunk table: chunk q = K elements [8q, 8q+8) -> (filter row r, filter col s, channel c).
  const int nq = a.num_kb * 8;
  for (int q = tid; q < nq; q += blockDim.x) {
    const int kk = q * 8;
    int2 e;
    if (kk < a.K) {
      const int tap = kk / a.Cin;
      const int c = kk - tap * a.Cin;
      const int r = tap / a.S;
      const int s = tap - r * a.S;
      e.x = (r << 16) | s;
      e.y = c;
    } else {
      e.x = 0;
      e.y = -1;
    }
    ktab[q] = e;
  }
  if (warp == 4) {
    if (lane == 0) {
      for (int i = 0; i < S_; ++i) {
        mbar_init(&full[i], 128 + 1);
        mbar_init(&empty[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&tfull[i], 1);
        mbar_init(&tempty[i], 128);
      }
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(tslot, a.tmem_cols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tslot;
  const uint32_t acc_stride = a.tmem_cols >> 1;

  // Programmatic dependent launch: everything above overlapped the previous kernel's tail.
  pdl_wait();

  if (warp < 4) {
    // ------------------------------------------------------------ A producer (im2col)
    const int row = tid;
    const int HoWo = a.Ho * a.Wo;
    int it = 0;
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
      const int m_blk = tile / a.n_tiles;
      const int m = m_blk * kBM + row;
      const bool row_ok = m < a.M;
      int n = 0, ho = 0, wo = 0;
      if (row_ok) {
        n = m / HoWo;
        const int rem = m - n * HoWo;
        ho = rem / a.Wo;
        wo = rem - ho * a.Wo;
      }
      const int hi0 = ho * a.sh - a.ph;
      const int wi0 = wo * a.sw - a.pw;
      const __nv_bfloat16* xn = a.x + static_cast<size_t>(n) * a.H * a.W * a.x_ld;
      for (int kb = 0; kb < a.num_kb; ++kb, ++it) {
        const int st = it % S_;
        const uint32_t ph = (it / S_) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        const uint32_t dst = smem_u32(sA + st * kATileBytes + row * 128);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int2 e = ktab[kb * 8 + j];
          const int hi = hi0 + (e.x >> 16);
          const int wi = wi0 + (e.x & 0xffff);
          const bool ok = row_ok && e.y >= 0 && static_cast<unsigned>(hi) < static_cast<unsigned>(a.H) &&
                          static_cast<unsigned>(wi) < static_cast<unsigned>(a.W);
          const __nv_bfloat16* src = ok ? xn + (static_cast<size_t>(hi) * a.W + wi) * a.x_ld + e.y : a.x;
          cp_async16_zfill(dst + ((j ^ (row & 7)) << 4), src, ok ? 16u : 0u);
        }
        cp_async_commit();
        if (it >= kLag) {
          cp_async_wait<kLag>();
          fence_proxy_async_smem();
          mbar_arrive(&full[(it - kLag) % S_]);
        }
      }
    }
    cp_async_wait<0>();
    fence_proxy_async_smem();
    for (int j = (it > kLag ? it - kLag : 0); j < it; ++j) mbar_arrive(&full[j % S_]);
  } else if (warp == 4) {
    // ------------------------------------------------------------ B producer (TMA)
    if (lane == 0) {
      tma_prefetch_desc(&wmap);
      int it = 0;
      for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
        const int n_blk = tile % a.n_tiles;
        for (int kb = 0; kb < a.num_kb; ++kb, ++it) {
          const int st = it % S_;
          const uint32_t ph = (it / S_) & 1;
          mbar_wait(&empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&full[st], b_bytes);
          tma_load_2d(sB + static_cast<size_t>(st) * b_bytes, &wmap, &full[st], kb * kBK, n_blk * BN);
        }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int it = 0, t = 0;
      for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++t) {
        const int acc = t & 1;
        const uint32_t aph = (t >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * acc_stride;
        for (int kb = 0; kb < a.num_kb; ++kb, ++it) {
          const int st = it % S_;
          const uint32_t ph = (it / S_) & 1;
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(sA + st * kATileBytes);
          const uint64_t bd = umma_desc_sw128(sB + static_cast<size_t>(st) * b_bytes);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            umma_bf16(d, ad + 2 * kk, bd + 2 * kk, a.idesc, (kb | kk) != 0);
          }
          umma_commit(&empty[st]);
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    int t = 0;
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++t) {
      const int m_blk = tile / a.n_tiles;
      const int n_blk = tile % a.n_tiles;
      const int acc = t & 1;
      const uint32_t aph = (t >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int m = m_blk * kBM + row;
      const bool row_ok = m < a.M;
      const uint32_t tbase = tmem_base + acc * acc_stride + (static_cast<uint32_t>(q * 32) << 16);
      for (int c = 0; c < BN; c += 16) {
        uint32_t v[16];
        tmem_ld16(tbase + c, v);
        tmem_ld_wait();
        const int n0 = n_blk * BN + c;
        if (row_ok && n0 < a.Cout) {
          float f[16];
          const float4* b4 = reinterpret_cast<const float4*>(a.bias + n0);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 bb = __ldg(b4 + i);
            f[4 * i + 0] = __uint_as_float(v[4 * i + 0]) + bb.x;
            f[4 * i + 1] = __uint_as_float(v[4 * i + 1]) + bb.y;
            f[4 * i + 2] = __uint_as_float(v[4 * i + 2]) + bb.z;
            f[4 * i + 3] = __uint_as_float(v[4 * i + 3]) + bb.w;
          }
          if (a.res != nullptr) {
            const uint4* r4 = reinterpret_cast<const uint4*>(a.res + static_cast<size_t>(m) * a.res_ld + n0);
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const uint4 rr = __ldg(r4 + i);
              const uint32_t w[4] = {rr.x, rr.y, rr.z, rr.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float2 p = unpack_bf16x2(w[j]);
                f[8 * i + 2 * j] += p.x;
                f[8 * i + 2 * j + 1] += p.y;
              }
            }
          }
          if (a.act == GX_ACT_RELU) {
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = fmaxf(f[i], 0.0f);
          } else if (a.act == GX_ACT_GELU) {
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = gelu_erf(f[i]);
          }
          if (a.y_f32) {
            float4* y4 = reinterpret_cast<float4*>(static_cast<float*>(a.y) + static_cast<size_t>(m) * a.y_ld +
                                                   a.y_coff + n0);
#pragma unroll
            for (int i = 0; i < 4; ++i) y4[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
          } else {
            uint4* y4 = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.y) + static_cast<size_t>(m) * a.y_ld +
                                                 a.y_coff + n0);
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              uint4 o;
              o.x = pack_bf16x2(f[8 * i + 0], f[8 * i + 1]);
              o.y = pack_bf16x2(f[8 * i + 2], f[8 * i + 3]);
              o.z = pack_bf16x2(f[8 * i + 4], f[8 * i + 5]);
              o.w = pack_bf16x2(f[8 * i + 6], f[8 * i + 7]);
              y4[i] = o;
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  // Let the next kernel in the stream start its prologue.
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem_base, a.tmem_cols);
  }
}
}  // namespace

size_t conv_smem_bytes(int BN, int stages, int num_kb) {
  return 1024 + static_cast<size_t>(stages) * (kATileBytes + BN * 128) + (2 * stages + 4) * 8 + 16 +
         static_cast<size_t>(num_kb) * 8 * sizeof(int2);
}

int conv_pick_stages(int BN, int num_kb) {
  const size_t budget = 200 * 1024 - static_cast<size_t>(num_kb) * 8 * sizeof(int2);
  int s = static_cast<int>(budget / (kATileBytes + BN * 128));
  if (s > 8) s = 8;
  if (s < 2) s = 2;
  return s;
}

cudaError_t launch_conv(const CUtensorMap& wmap, const ConvArgs& a, int grid, cudaStream_t s, bool pdl) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(conv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kConvThreads, 1, 1);
  cfg.dynamicSmemBytes = conv_smem_bytes(a.BN, a.stages, a.num_kb);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, conv_tc_kernel, wmap, a);
}

}  // namespace gx
