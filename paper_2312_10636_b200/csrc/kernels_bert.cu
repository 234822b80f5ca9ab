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

// K8: BERT embeddings for fragments entering at boundary 0 (BertEmbeddings: word[id] + pos[s] +
// type[0], then LayerNorm).  One warp per token row; the row's C values stay in registers between
// the mean, variance and normalise passes (C % 256 == 0, C <= 1024; 8 elements per lane-vector).
// Tables are in the chain's element type T (bf16 or fp32), sums and LayerNorm in fp32.  Token ids
// outside [0, V) are clamped (torch raises; the executor never reads outside the table).
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* v) {
  const uint4 q = __ldg(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = unpack_bf16x2(w[j]);
    v[2 * j] = f.x;
    v[2 * j + 1] = f.y;
  }
}
__device__ __forceinline__ void load8(const float* p, float* v) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float* o) {
  uint4 q;
  q.x = pack_bf16x2(o[0], o[1]);
  q.y = pack_bf16x2(o[2], o[3]);
  q.z = pack_bf16x2(o[4], o[5]);
  q.w = pack_bf16x2(o[6], o[7]);
  *reinterpret_cast<uint4*>(p) = q;
}
__device__ __forceinline__ void store8(float* p, const float* o) {
  reinterpret_cast<float4*>(p)[0] = make_float4(o[0], o[1], o[2], o[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(o[4], o[5], o[6], o[7]);
}

template <typename T, int VPL>
__global__ void embed_ln_kernel(const int32_t* __restrict__ ids, int rows, int S, int C, const T* __restrict__ word,
                                int V, const T* __restrict__ pos, const T* __restrict__ type0,
                                const float* __restrict__ g, const float* __restrict__ b, float eps,
                                T* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const int id = min(max(__ldg(ids + r), 0), V - 1);
    const int sp = r % S;
    const T* wr = word + static_cast<int64_t>(id) * C;
    const T* pr = pos + static_cast<int64_t>(sp) * C;
    float v[VPL * 8];
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c0 = (lane + 32 * i) * 8;
      float a[8], p8[8], t8[8];
      load8(wr + c0, a);
      load8(pr + c0, p8);
      load8(type0 + c0, t8);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v[8 * i + j] = a[j] + t8[j] + p8[j];  // torch: (inputs_embeds + token_type) + position
        s += v[8 * i + j];
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
    T* yr = y + static_cast<int64_t>(r) * C;
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
      store8(yr + c0, o);
    }
  }
}

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t ld_b32(const __nv_bfloat16* p) { return *reinterpret_cast<const uint32_t*>(p); }

constexpr int kAttnQ = 64;  // query rows per CTA (4 warps x 16)

// Self-attention of one (request, head, 64-query block) per CTA iteration.  The per-head products
// are tiny (S x S x 64): QK^T and PV run on warp-level bf16 MMA (m16n8k16) with fp32
// accumulators, each warp owning 16 query rows; K and V^T of the head are staged in shared memory
// (row strides padded so the fragment loads are bank-conflict free) and keys are consumed in
// 64-wide chunks with an online softmax, so the S x S score matrix never leaves registers.
// qkv rows are [q | k | v] (3 x hidden); heads are D-wide slices; no mask.
template <int D>
__global__ void __launch_bounds__(128) attention_kernel(const __nv_bfloat16* __restrict__ qkv, int N, int S, int heads,
                                                        int hidden, float scale_log2, __nv_bfloat16* __restrict__ out) {
  extern __shared__ uint4 smem_kv[];
  const int SP = (S + 63) & ~63;
  constexpr int KST = D + 8;
  const int VST = SP + 8;
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smem_kv);  // [SP][KST]
  __nv_bfloat16* Vt = Ks + static_cast<size_t>(SP) * KST;         // [D][VST]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int qblocks = (S + kAttnQ - 1) / kAttnQ;
  const int items = N * heads * qblocks;
  const int64_t row_ld = 3 * static_cast<int64_t>(hidden);
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int qb = it % qblocks, nh = it / qblocks;
    const int n = nh / heads, h = nh - n * heads;
    const __nv_bfloat16* base = qkv + static_cast<int64_t>(n) * S * row_ld + h * D;
    __syncthreads();  // the previous item is done with K / V^T
    for (int i = threadIdx.x; i < SP * (D / 8); i += blockDim.x) {
      const int j = i / (D / 8), c = i - j * (D / 8);
      uint4 kv = make_uint4(0, 0, 0, 0), vv = kv;
      if (j < S) {
        const __nv_bfloat16* row = base + j * row_ld + c * 8;
        kv = __ldcg(reinterpret_cast<const uint4*>(row + hidden));
        vv = __ldcg(reinterpret_cast<const uint4*>(row + 2 * hidden));
      }
      *reinterpret_cast<uint4*>(Ks + j * KST + c * 8) = kv;
      const __nv_bfloat16* v8 = reinterpret_cast<const __nv_bfloat16*>(&vv);
#pragma unroll
      for (int e = 0; e < 8; ++e) Vt[(c * 8 + e) * VST + j] = v8[e];
    }
    __syncthreads();
    const int q0 = qb * kAttnQ + warp * 16;
    if (q0 >= S) continue;  // warp-uniform; the loop-top barrier is reached by every warp
    const int r0 = min(q0 + g, S - 1), r1 = min(q0 + g + 8, S - 1);
    uint32_t qa[D / 16][4];
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      qa[kk][0] = __ldcg(reinterpret_cast<const unsigned int*>(base + r0 * row_ld + 16 * kk + 2 * t));
      qa[kk][1] = __ldcg(reinterpret_cast<const unsigned int*>(base + r1 * row_ld + 16 * kk + 2 * t));
      qa[kk][2] = __ldcg(reinterpret_cast<const unsigned int*>(base + r0 * row_ld + 16 * kk + 8 + 2 * t));
      qa[kk][3] = __ldcg(reinterpret_cast<const unsigned int*>(base + r1 * row_ld + 16 * kk + 8 + 2 * t));
    }
    float o[D / 8][4];
#pragma unroll
    for (int j = 0; j < D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.0f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.0f, l1 = 0.0f;
    for (int kc = 0; kc < SP; kc += 64) {
      float sc[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.0f;
        const __nv_bfloat16* kr = Ks + (kc + 8 * j + g) * KST + 2 * t;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) mma_bf16_16816(sc[j], qa[kk], ld_b32(kr + 16 * kk), ld_b32(kr + 16 * kk + 8));
      }
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = kc + 8 * j + 2 * t + (e & 1);
          sc[j][e] = key < S ? sc[j][e] * scale_log2 : -INFINITY;
        }
        mx0 = fmaxf(mx0, fmaxf(sc[j][0], sc[j][1]));
        mx1 = fmaxf(mx1, fmaxf(sc[j][2], sc[j][3]));
      }
#pragma unroll
      for (int off = 1; off <= 2; off <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
      }
      const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);  // finite: key kc < S is always valid
      const float c0 = exp2f(m0 - n0), c1 = exp2f(m1 - n1);
      m0 = n0;
      m1 = n1;
      l0 *= c0;
      l1 *= c1;
#pragma unroll
      for (int j = 0; j < D / 8; ++j) {
        o[j][0] *= c0;
        o[j][1] *= c0;
        o[j][2] *= c1;
        o[j][3] *= c1;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        sc[j][0] = exp2f(sc[j][0] - n0);
        sc[j][1] = exp2f(sc[j][1] - n0);
        sc[j][2] = exp2f(sc[j][2] - n1);
        sc[j][3] = exp2f(sc[j][3] - n1);
        l0 += sc[j][0] + sc[j][1];
        l1 += sc[j][2] + sc[j][3];
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {  // P (16 x 64 keys) as the A operand, straight from registers
        const uint32_t pa[4] = {pack_bf16x2(sc[2 * kk][0], sc[2 * kk][1]), pack_bf16x2(sc[2 * kk][2], sc[2 * kk][3]),
                                pack_bf16x2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]),
                                pack_bf16x2(sc[2 * kk + 1][2], sc[2 * kk + 1][3])};
#pragma unroll
        for (int j = 0; j < D / 8; ++j) {
          const __nv_bfloat16* vr = Vt + (8 * j + g) * VST + kc + 16 * kk + 2 * t;
          mma_bf16_16816(o[j], pa, ld_b32(vr), ld_b32(vr + 8));
        }
      }
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    const float i0 = 1.0f / l0, i1 = 1.0f / l1;
    __nv_bfloat16* o0 = out + (static_cast<int64_t>(n) * S + q0 + g) * hidden + h * D + 2 * t;
    __nv_bfloat16* o1 = o0 + 8 * static_cast<int64_t>(hidden);
#pragma unroll
    for (int j = 0; j < D / 8; ++j) {
      if (q0 + g < S) *reinterpret_cast<uint32_t*>(o0 + 8 * j) = pack_bf16x2(o[j][0] * i0, o[j][1] * i0);
      if (q0 + g + 8 < S) *reinterpret_cast<uint32_t*>(o1 + 8 * j) = pack_bf16x2(o[j][2] * i1, o[j][3] * i1);
    }
  }
}

}  // namespace

template <typename T>
static cudaError_t launch_embed_t(const int32_t* ids, int rows, int S, int C, const T* word, int V, const T* pos,
                                  const T* type0, const float* gamma, const float* beta, float eps, T* y, int grid,
                                  cudaStream_t s) {
  if (C % 256 != 0 || C > 1024 || V < 1 || S < 1) return cudaErrorInvalidValue;
  const int wpb = 8;
  int blocks = (rows + wpb - 1) / wpb;
  if (blocks > grid) blocks = grid;
  if (blocks < 1) blocks = 1;
  switch (C / 256) {
    case 1: embed_ln_kernel<T, 1><<<blocks, 32 * wpb, 0, s>>>(ids, rows, S, C, word, V, pos, type0, gamma, beta, eps, y); break;
    case 2: embed_ln_kernel<T, 2><<<blocks, 32 * wpb, 0, s>>>(ids, rows, S, C, word, V, pos, type0, gamma, beta, eps, y); break;
    case 3: embed_ln_kernel<T, 3><<<blocks, 32 * wpb, 0, s>>>(ids, rows, S, C, word, V, pos, type0, gamma, beta, eps, y); break;
    default: embed_ln_kernel<T, 4><<<blocks, 32 * wpb, 0, s>>>(ids, rows, S, C, word, V, pos, type0, gamma, beta, eps, y); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_embed(const int32_t* ids, int rows, int S, int C, const void* word, int V, const void* pos,
                         const void* type0, const float* gamma, const float* beta, float eps, void* y, int f32,
                         int grid, cudaStream_t s) {
  if (f32)
    return launch_embed_t<float>(ids, rows, S, C, static_cast<const float*>(word), V, static_cast<const float*>(pos),
                                 static_cast<const float*>(type0), gamma, beta, eps, static_cast<float*>(y), grid, s);
  return launch_embed_t<__nv_bfloat16>(ids, rows, S, C, static_cast<const __nv_bfloat16*>(word), V,
                                       static_cast<const __nv_bfloat16*>(pos), static_cast<const __nv_bfloat16*>(type0),
                                       gamma, beta, eps, static_cast<__nv_bfloat16*>(y), grid, s);
}

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

// K6 on the 5th-gen tensor cores (S <= 128, head dim 64: BERT-base).  One CTA of 4 warps owns one
// (request, head) item at a time, persistent over the items:
//   TMA     Q and K tiles ([128 rows][64] bf16, 128-byte swizzle) straight into the MMA layout;
//           V is transposed by the threads into V^T ([2 key blocks][64 d][64 keys], same swizzle);
//   MMA 1   S = Q K^T : M=128 queries, N=128 keys, K=64  (4 x tcgen05.mma, fp32 in TMEM cols 0-127);
//           the softmax reads S out completely before MMA 2 writes O over its first 64 columns, and P
//           takes the shared memory of Q and K: 48 KB and 128 TMEM columns per CTA, 4 items per SM;
//   softmax thread q = TMEM lane q owns query row q: two passes over its 128 scores (row max, then
//           exp2 / row sum), P = bf16 probabilities written to shared memory as the next A operand;
//   MMA 2   O = P V   : M=128, N=64, K=128 keys  (8 x tcgen05.mma, TMEM cols 0-63);
//   epilogue O / rowsum -> bf16 -> out.  Keys >= S are masked; queries >= S are not stored.
// One elected thread issues each MMA group and commits it to an mbarrier the 128 threads wait on.
constexpr int kAttnTcThreads = 128;
constexpr uint32_t kAttnTcSmem = 1024 + 16384 * 3 + 64;  // Q|K (then P) + V^T + barriers: 4 CTAs per SM

__device__ __forceinline__ void tma_load_2d_attn(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// byte offset of element (row, col) of a [rows][64] bf16 tile with the 128-byte swizzle
__device__ __forceinline__ uint32_t sw128_off(int row, int col) {
  return static_cast<uint32_t>(row) * 128u + ((((col >> 3) ^ (row & 7)) & 7) << 4) + (col & 7) * 2;
}

__global__ void __launch_bounds__(kAttnTcThreads, 4)
    attention_tc_kernel(const __grid_constant__ CUtensorMap qkmap, const __nv_bfloat16* __restrict__ qkv, int N, int S,
                        int heads, int hidden, float scale_log2, __nv_bfloat16* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;               // [128][64]
  uint8_t* sK = sQ + 16384;         // [128][64]
  uint8_t* sP = smem;               // [2][128][64]: P overwrites Q and K once S = Q K^T is in TMEM
  uint8_t* sVt = sK + 16384;        // [2][64][64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sVt + 16384);  // qk_full, s_full, o_full
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 3);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < 3; ++i) mbar_init(&bars[i], 1);
      fence_barrier_init();
      tma_prefetch_desc(&qkmap);
    }
    __syncwarp();
    tmem_alloc(tslot, 128);  // S (128 columns), then O (64) over it
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
  const int64_t row_ld = 3 * static_cast<int64_t>(hidden);
  const uint32_t idesc_s = umma_idesc_bf16(128, 128), idesc_o = umma_idesc_bf16(128, 64);
  pdl_wait();
  uint32_t ph = 0;
  for (int it = blockIdx.x; it < N * heads; it += gridDim.x, ph ^= 1) {
    const int n = it / heads, h = it - n * heads;
    if (tid == 0) {
      mbar_arrive_expect_tx(&bars[0], 32768u);
      tma_load_2d_attn(sQ, &qkmap, &bars[0], h * 64, n * S);
      tma_load_2d_attn(sK, &qkmap, &bars[0], hidden + h * 64, n * S);
    }
    {  // V^T: thread t transposes key t's 64 values (zero rows past S)
      const int key = tid;
      uint4 v[8];
      const uint4* src = reinterpret_cast<const uint4*>(qkv + (static_cast<int64_t>(n) * S + key) * row_ld + 2 * hidden +
                                                        h * 64);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = key < S ? __ldcg(src + j) : make_uint4(0, 0, 0, 0);
      uint8_t* vt = sVt + (key >> 6) * 8192;
      const int kc = key & 63;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v[j]);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<__nv_bfloat16*>(vt + sw128_off(j * 8 + q, kc)) = e[q];
      }
    }
    fence_async_shared();
    __syncthreads();
    if (tid == 0) {  // S = Q K^T
      mbar_wait(&bars[0], ph);
      tc_fence_after();
      const uint64_t qd = umma_desc_sw128(sQ), kd = umma_desc_sw128(sK);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) umma_bf16(tmem, qd + 2 * kk, kd + 2 * kk, idesc_s, kk != 0);
      umma_commit(&bars[1]);
    }
    mbar_wait(&bars[1], ph);
    tc_fence_after();
    // softmax of row q over the valid keys: pass 1 max, pass 2 exp2 + sum + P (bf16) to smem
    const int q = tid;
    float mx = -INFINITY;
    for (int c = 0; c < 128; c += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + lane_base + c, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (c + j < S) mx = fmaxf(mx, __uint_as_float(r[j]));
    }
    const float mscaled = mx * scale_log2;
    float sum = 0.0f;
    for (int c = 0; c < 128; c += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + lane_base + c, r);
      tmem_ld_wait();
      float pr[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        pr[j] = c + j < S ? exp2f(__uint_as_float(r[j]) * scale_log2 - mscaled) : 0.0f;
        sum += pr[j];
      }
      uint8_t* pt = sP + (c >> 6) * 16384;
      const int cc = c & 63;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint4 o;
        o.x = pack_bf16x2(pr[8 * hh + 0], pr[8 * hh + 1]);
        o.y = pack_bf16x2(pr[8 * hh + 2], pr[8 * hh + 3]);
        o.z = pack_bf16x2(pr[8 * hh + 4], pr[8 * hh + 5]);
        o.w = pack_bf16x2(pr[8 * hh + 6], pr[8 * hh + 7]);
        *reinterpret_cast<uint4*>(pt + sw128_off(q, cc + 8 * hh)) = o;
      }
    }
    fence_async_shared();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {  // O = P V
      tc_fence_after();
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        const uint64_t pd = umma_desc_sw128(sP + kb * 16384), vd = umma_desc_sw128(sVt + kb * 8192);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_bf16(tmem, pd + 2 * kk, vd + 2 * kk, idesc_o, (kb | kk) != 0);
      }
      umma_commit(&bars[2]);
    }
    mbar_wait(&bars[2], ph);
    tc_fence_after();
    {  // tcgen05.ld is warp-collective: every lane loads, only rows q < S are stored
      const float inv = 1.0f / sum;
      uint4* dst = reinterpret_cast<uint4*>(out + (static_cast<int64_t>(n) * S + q) * hidden + h * 64);
#pragma unroll
      for (int c = 0; c < 64; c += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + lane_base + c, r);
        tmem_ld_wait();
        if (q >= S) continue;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint4 o;
          o.x = pack_bf16x2(__uint_as_float(r[8 * hh + 0]) * inv, __uint_as_float(r[8 * hh + 1]) * inv);
          o.y = pack_bf16x2(__uint_as_float(r[8 * hh + 2]) * inv, __uint_as_float(r[8 * hh + 3]) * inv);
          o.z = pack_bf16x2(__uint_as_float(r[8 * hh + 4]) * inv, __uint_as_float(r[8 * hh + 5]) * inv);
          o.w = pack_bf16x2(__uint_as_float(r[8 * hh + 6]) * inv, __uint_as_float(r[8 * hh + 7]) * inv);
          dst[(c >> 3) + hh] = o;
        }
      }
    }
    tc_fence_before();
    __syncthreads();  // TMEM and the smem tiles are reused by the next item
  }
  pdl_launch_dependents();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

cudaError_t launch_attention(const __nv_bfloat16* qkv, int N, int S, int heads, int dh, __nv_bfloat16* out, int grid,
                             cudaStream_t s) {
  if (dh != 64 || S < 1 || S > 512) return cudaErrorInvalidValue;
  if (S <= 128) {  // tcgen05 path (BERT-base: S = 128)
    static bool tc_configured = false;
    if (!tc_configured) {
      cudaFuncSetAttribute(attention_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnTcSmem);
      tc_configured = true;
    }
    CUtensorMap map;
    if (!encode_tmap_2d_bf16(&map, qkv, 3ull * heads * dh, static_cast<uint64_t>(N) * S, 3ull * heads * dh * 2, 64,
                             128))
      return cudaErrorInvalidValue;
    int blocks = N * heads;
    if (blocks > grid / 2) blocks = std::max(1, grid / 2);  // grid = budget x 8: <= 4 CTAs per budget SM
    const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(dh));
    attention_tc_kernel<<<blocks, kAttnTcThreads, kAttnTcSmem, s>>>(map, qkv, N, S, heads, heads * dh, scale_log2,
                                                                    out);
    return cudaGetLastError();
  }
  const int SP = (S + 63) & ~63;
  const size_t smem = (static_cast<size_t>(SP) * (dh + 8) + static_cast<size_t>(dh) * (SP + 8)) * 2;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(attention_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    configured = true;
  }
  int blocks = N * heads * ((S + kAttnQ - 1) / kAttnQ);
  if (blocks > grid) blocks = grid;
  if (blocks < 1) blocks = 1;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(dh));
  attention_kernel<64><<<blocks, 128, smem, s>>>(qkv, N, S, heads, heads * dh, scale_log2, out);
  return cudaGetLastError();
}

}  // namespace gx
