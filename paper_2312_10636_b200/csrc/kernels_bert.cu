// BERT encoder pieces (configs[4]): LayerNorm (K7) and self-attention (K6).  The four linears of
// a layer (QKV, output + residual, FFN1 + GELU, FFN2 + residual) run on the tcgen05 GEMM path
// (GX_OP_LINEAR through conv_tc_kernel), so only these two bandwidth/latency-bound ops live here.
#include <cuda_bf16.h>

#include "gx_internal.h"
#include "gx_ptx.cuh"

namespace gx {

namespace {

// One warp per row of C (C % 256 == 0 for the vector path): mean / biased variance in fp32,
// y = (x - mean) * rsqrt(var + eps) * gamma + beta  (torch.nn.LayerNorm semantics).
template <int VPL>  // 16-byte vectors per lane
__global__ void layernorm_kernel(const __nv_bfloat16* __restrict__ x, int rows, int C, const float* __restrict__ g,
                                 const float* __restrict__ b, float eps, __nv_bfloat16* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(r) * C);
    float v[VPL * 8];
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const uint4 q = __ldcg(xr + lane + 32 * i);
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack_bf16x2(w[j]);
        v[8 * i + 2 * j] = f.x;
        v[8 * i + 2 * j + 1] = f.y;
        s += f.x + f.y;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    const float mean = s / C;
    float ss = 0.0f;
#pragma unroll
    for (int i = 0; i < VPL * 8; ++i) {
      const float d = v[i] - mean;
      ss += d * d;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const float inv = rsqrtf(ss / C + eps);
    uint4* yr = reinterpret_cast<uint4*>(y + static_cast<int64_t>(r) * C);
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c0 = (lane + 32 * i) * 8;
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(g + c0)), g1 = __ldg(reinterpret_cast<const float4*>(g + c0 + 4));
      const float4 b0 = __ldg(reinterpret_cast<const float4*>(b + c0)), b1 = __ldg(reinterpret_cast<const float4*>(b + c0 + 4));
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = (v[8 * i + j] - mean) * inv * gg[j] + bb[j];
      uint4 q;
      q.x = pack_bf16x2(o[0], o[1]);
      q.y = pack_bf16x2(o[2], o[3]);
      q.z = pack_bf16x2(o[4], o[5]);
      q.w = pack_bf16x2(o[6], o[7]);
      yr[lane + 32 * i] = q;
    }
  }
}

// Self-attention of one (request, head) per CTA iteration: K and V of the head staged in shared
// memory, one thread per query row with an online (streaming) softmax in fp32, so the S x S score
// matrix never materialises.  qkv rows are [q | k | v] (3 x hidden), heads are D-wide slices.
template <int D>
__global__ void __launch_bounds__(128) attention_kernel(const __nv_bfloat16* __restrict__ qkv, int N, int S, int heads,
                                                        int hidden, float scale, __nv_bfloat16* __restrict__ out) {
  extern __shared__ uint4 smem_kv[];
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smem_kv);
  __nv_bfloat16* Vs = Ks + static_cast<size_t>(S) * D;
  const int pairs = N * heads;
  for (int pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
    const int n = pr / heads, h = pr - n * heads;
    const __nv_bfloat16* base = qkv + static_cast<int64_t>(n) * S * 3 * hidden;
    __syncthreads();
    for (int i = threadIdx.x; i < S * (D / 8); i += blockDim.x) {
      const int j = i / (D / 8), c = i - j * (D / 8);
      const __nv_bfloat16* row = base + static_cast<int64_t>(j) * 3 * hidden + h * D + c * 8;
      reinterpret_cast<uint4*>(Ks + j * D)[c] = __ldcg(reinterpret_cast<const uint4*>(row + hidden));
      reinterpret_cast<uint4*>(Vs + j * D)[c] = __ldcg(reinterpret_cast<const uint4*>(row + 2 * hidden));
    }
    __syncthreads();
    for (int qi = threadIdx.x; qi < S; qi += blockDim.x) {
      float q[D], o[D];
      const uint4* qr = reinterpret_cast<const uint4*>(base + static_cast<int64_t>(qi) * 3 * hidden + h * D);
#pragma unroll
      for (int c = 0; c < D / 8; ++c) {
        const uint4 t = __ldcg(qr + c);
        const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack_bf16x2(w[j]);
          q[8 * c + 2 * j] = f.x * scale;
          q[8 * c + 2 * j + 1] = f.y * scale;
        }
      }
#pragma unroll
      for (int d = 0; d < D; ++d) o[d] = 0.0f;
      float m = -INFINITY, l = 0.0f;
      for (int j = 0; j < S; ++j) {
        const uint4* kr = reinterpret_cast<const uint4*>(Ks + j * D);
        float sp[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // 4 independent FMA chains
#pragma unroll
        for (int c = 0; c < D / 8; ++c) {
          const uint4 t = kr[c];
          const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const float2 f = unpack_bf16x2(w[jj]);
            sp[jj] = fmaf(q[8 * c + 2 * jj], f.x, sp[jj]);
            sp[jj] = fmaf(q[8 * c + 2 * jj + 1], f.y, sp[jj]);
          }
        }
        const float s = (sp[0] + sp[1]) + (sp[2] + sp[3]);
        const float mn = fmaxf(m, s);
        const float corr = __expf(m - mn);
        const float p = __expf(s - mn);
        l = l * corr + p;
        m = mn;
        const uint4* vr = reinterpret_cast<const uint4*>(Vs + j * D);
#pragma unroll
        for (int c = 0; c < D / 8; ++c) {
          const uint4 t = vr[c];
          const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const float2 f = unpack_bf16x2(w[jj]);
            o[8 * c + 2 * jj] = fmaf(o[8 * c + 2 * jj], corr, p * f.x);
            o[8 * c + 2 * jj + 1] = fmaf(o[8 * c + 2 * jj + 1], corr, p * f.y);
          }
        }
      }
      const float il = 1.0f / l;
      uint4* orow = reinterpret_cast<uint4*>(out + (static_cast<int64_t>(n) * S + qi) * hidden + h * D);
#pragma unroll
      for (int c = 0; c < D / 8; ++c) {
        uint4 t;
        t.x = pack_bf16x2(o[8 * c + 0] * il, o[8 * c + 1] * il);
        t.y = pack_bf16x2(o[8 * c + 2] * il, o[8 * c + 3] * il);
        t.z = pack_bf16x2(o[8 * c + 4] * il, o[8 * c + 5] * il);
        t.w = pack_bf16x2(o[8 * c + 6] * il, o[8 * c + 7] * il);
        orow[c] = t;
      }
    }
  }
}

}  // namespace

cudaError_t launch_layernorm(const __nv_bfloat16* x, const __nv_bfloat16* res, int rows, int C, const float* gamma,
                             const float* beta, float eps, __nv_bfloat16* y, int grid, cudaStream_t s) {
  (void)res;
  if (C % 256 != 0 || C > 1024) return cudaErrorInvalidValue;
  const int warps_per_block = 8;
  int blocks = (rows + warps_per_block - 1) / warps_per_block;
  if (blocks > grid) blocks = grid;
  if (blocks < 1) blocks = 1;
  switch (C / 256) {
    case 1:
      layernorm_kernel<1><<<blocks, 32 * warps_per_block, 0, s>>>(x, rows, C, gamma, beta, eps, y);
      break;
    case 2:
      layernorm_kernel<2><<<blocks, 32 * warps_per_block, 0, s>>>(x, rows, C, gamma, beta, eps, y);
      break;
    case 3:
      layernorm_kernel<3><<<blocks, 32 * warps_per_block, 0, s>>>(x, rows, C, gamma, beta, eps, y);
      break;
    default:
      layernorm_kernel<4><<<blocks, 32 * warps_per_block, 0, s>>>(x, rows, C, gamma, beta, eps, y);
      break;
  }
  return cudaGetLastError();
}

cudaError_t launch_attention(const __nv_bfloat16* qkv, int N, int S, int heads, int dh, __nv_bfloat16* out, int grid,
                             cudaStream_t s) {
  if (dh != 64 || S > 512) return cudaErrorInvalidValue;
  const size_t smem = static_cast<size_t>(S) * dh * 2 * 2;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(attention_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    configured = true;
  }
  int blocks = N * heads;
  if (blocks > grid) blocks = grid;
  if (blocks < 1) blocks = 1;
  attention_kernel<64><<<blocks, 128, smem, s>>>(qkv, N, S, heads, heads * dh, 1.0f / sqrtf(static_cast<float>(dh)),
                                                 out);
  return cudaGetLastError();
}

}  // namespace gx
