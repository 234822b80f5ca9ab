// Bandwidth-bound kernels: ragged batch assembly (K1 gather/scatter), pooling (K4), the skinny
// FC layer at small batch, and channel-slice copies.  All are grid-stride loops over 16-byte
// vectors so one launch can be bounded to the stage's SM budget (grid = budget * blocks/SM).
#include <cuda_bf16.h>

#include "gx_internal.h"
#include "gx_ptx.cuh"

namespace gx {

namespace {
constexpr int kMaxRows = 64;  // max requests in one dispatched batch (profiles.py:200 caps at 127;
                              // fixtures use 16-32)
struct RowPtrs {
  const void* p[kMaxRows];
  int32_t dt[kMaxRows];
};
struct RowDst {
  void* p[kMaxRows];
};

// Read-once weight stream: non-coherent, no L1 allocation.
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ uint4 f32x8_to_bf16x8(float4 a, float4 b) {
  uint4 o;
  o.x = pack_bf16x2(a.x, a.y);
  o.y = pack_bf16x2(a.z, a.w);
  o.z = pack_bf16x2(b.x, b.y);
  o.w = pack_bf16x2(b.z, b.w);
  return o;
}

// K1 gather: k entry activations (each fp32 from ingress or bf16 from an alignment stage) ->
// one contiguous bf16 NHWC batch.  c_src == c_dst: 8-element vectors; otherwise per-element
// with zero padding of the extra channels (the 3-channel image into the 8-channel stem input).
// K1 gather into a space-to-depth boundary: client image [Ho*f, Wo*f, c_src] (fp32 or bf16) ->
// [Ho, Wo, c_dst] with channel (dy*f + dx)*c_src + c = pixel (f*h + dy, f*w + dx), zero above.
__global__ void gather_s2d_kernel(RowPtrs src, int k, int Ho, int Wo, int f, int c_src, int c_dst,
                                  __nv_bfloat16* __restrict__ dst) {
  const int64_t per_row = static_cast<int64_t>(Ho) * Wo * c_dst;
  const int64_t total = per_row * k;
  const int Wi = Wo * f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(i / per_row);
    const int64_t e = i - r * per_row;
    const int64_t px = e / c_dst;
    const int cd = static_cast<int>(e - px * c_dst);
    float val = 0.0f;
    if (cd < f * f * c_src) {
      const int blk = cd / c_src, c = cd - blk * c_src;
      const int h = static_cast<int>(px / Wo) * f + blk / f;
      const int w = static_cast<int>(px % Wo) * f + blk % f;
      const int64_t si = (static_cast<int64_t>(h) * Wi + w) * c_src + c;
      val = src.dt[r] == GX_F32 ? __ldg(reinterpret_cast<const float*>(src.p[r]) + si)
                                : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(src.p[r])[si]);
    }
    dst[i] = __float2bfloat16_rn(val);
  }
}

// The stem's case (2x2 blocks of a 3-channel image into 16 channels, 12 used): a thread owns one
// output pixel, reads its two 6-value input row segments as 8-byte vectors (the pixel pair starts
// at an even column: 24-byte aligned) and writes the 32-byte output pixel as two 16-byte stores.
// (The per-element kernel above did a 64-bit div/mod chain and a 2-byte store per element.)
__global__ void gather_s2d_rgb2_kernel(RowPtrs src, int k, int Ho, int Wo, __nv_bfloat16* __restrict__ dst) {
  const int per_row = Ho * Wo;
  const int total = per_row * k;  // < 2^31: k <= 64 rows of <= 112x112 pixels
  const int Wi = Wo * 2;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int r = i / per_row;
    const int px = i - r * per_row;
    const int ho = px / Wo, wo = px - (px / Wo) * Wo;
    float v[12];  // channel (dy*2 + dx)*3 + c
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const int64_t e0 = (static_cast<int64_t>(2 * ho + dy) * Wi + 2 * wo) * 3;  // 6 values: (dx, c)
      if (src.dt[r] == GX_F32) {
        const float2* p = reinterpret_cast<const float2*>(static_cast<const float*>(src.p[r]) + e0);
        const float2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
        v[dy * 6 + 0] = a.x, v[dy * 6 + 1] = a.y, v[dy * 6 + 2] = b.x;
        v[dy * 6 + 3] = b.y, v[dy * 6 + 4] = c.x, v[dy * 6 + 5] = c.y;
      } else {
        const __nv_bfloat16* p = static_cast<const __nv_bfloat16*>(src.p[r]) + e0;
#pragma unroll
        for (int j = 0; j < 6; ++j) v[dy * 6 + j] = __bfloat162float(p[j]);
      }
    }
    uint4 o0, o1;
    o0.x = pack_bf16x2(v[0], v[1]);
    o0.y = pack_bf16x2(v[2], v[3]);
    o0.z = pack_bf16x2(v[4], v[5]);
    o0.w = pack_bf16x2(v[6], v[7]);
    o1.x = pack_bf16x2(v[8], v[9]);
    o1.y = pack_bf16x2(v[10], v[11]);
    o1.z = 0u;
    o1.w = 0u;
    uint4* d = reinterpret_cast<uint4*>(dst + static_cast<int64_t>(i) * 16);
    d[0] = o0;
    d[1] = o1;
  }
}

__global__ void gather_kernel(RowPtrs src, int k, int64_t pixels, int c_src, int c_dst,
                              __nv_bfloat16* __restrict__ dst) {
  if (c_src == c_dst && (c_dst & 7) == 0) {
    const int64_t vec_per_row = pixels * c_dst / 8;
    const int64_t total = vec_per_row * k;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
      const int r = static_cast<int>(i / vec_per_row);
      const int64_t v = i - r * vec_per_row;
      uint4 o;
      if (src.dt[r] == GX_F32) {
        const float4* s = reinterpret_cast<const float4*>(src.p[r]) + 2 * v;
        o = f32x8_to_bf16x8(__ldg(s), __ldg(s + 1));
      } else {
        o = __ldg(reinterpret_cast<const uint4*>(src.p[r]) + v);
      }
      reinterpret_cast<uint4*>(dst)[i] = o;
    }
  } else {
    const int64_t per_row = pixels * c_dst;
    const int64_t total = per_row * k;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
      const int r = static_cast<int>(i / per_row);
      const int64_t e = i - r * per_row;
      const int64_t px = e / c_dst;
      const int c = static_cast<int>(e - px * c_dst);
      float val = 0.0f;
      if (c < c_src) {
        const int64_t si = px * c_src + c;
        val = src.dt[r] == GX_F32 ? __ldg(reinterpret_cast<const float*>(src.p[r]) + si)
                                  : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(src.p[r])[si]);
      }
      dst[i] = __float2bfloat16_rn(val);
    }
  }
}

// K1 gather of 4-byte words (token ids at a K8 embedding boundary): k rows of `words` each.
__global__ void gather_words_kernel(RowPtrs src, int k, int64_t words, uint32_t* __restrict__ dst) {
  const int64_t total = words * k;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / words);
    dst[i] = __ldg(static_cast<const uint32_t*>(src.p[r]) + (i - r * words));
  }
}

// K1 scatter: batch rows -> per-request destinations (bf16 activations or fp32 logits).
__global__ void scatter_kernel(const void* __restrict__ src, int src_f32, int k, int64_t row_elems, RowDst dst,
                               int dst_f32) {
  const int64_t vec_per_row = row_elems / 8;
  const int64_t total = vec_per_row * k;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (!src_f32 && !dst_f32) {
    // bf16 rows -> bf16 slots: 4 independent 16-byte loads in flight per thread before any store
    // (one per thread leaves too few bytes in flight to cover HBM latency at full occupancy)
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < total; i0 += 4 * stride) {
      uint4 val[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u * stride < total) val[u] = ldg_stream(reinterpret_cast<const uint4*>(src) + i0 + u * stride);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * stride;
        if (i < total) {
          const int r = static_cast<int>(i / vec_per_row);
          reinterpret_cast<uint4*>(dst.p[r])[i - r * vec_per_row] = val[u];
        }
      }
    }
    return;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
    const int r = static_cast<int>(i / vec_per_row);
    const int64_t v = i - r * vec_per_row;
    if (src_f32) {
      const float4* s = reinterpret_cast<const float4*>(src) + 2 * i;
      const float4 a = __ldg(s), b = __ldg(s + 1);
      if (dst_f32) {
        float4* d = reinterpret_cast<float4*>(dst.p[r]) + 2 * v;
        d[0] = a;
        d[1] = b;
      } else {
        reinterpret_cast<uint4*>(dst.p[r])[v] = f32x8_to_bf16x8(a, b);
      }
      continue;
    }
    const uint4 val = __ldg(reinterpret_cast<const uint4*>(src) + i);
    if (dst_f32) {
      float4* d = reinterpret_cast<float4*>(dst.p[r]) + 2 * v;
      const float2 a = unpack_bf16x2(val.x), b = unpack_bf16x2(val.y), c = unpack_bf16x2(val.z),
                   e = unpack_bf16x2(val.w);
      d[0] = make_float4(a.x, a.y, b.x, b.y);
      d[1] = make_float4(c.x, c.y, e.x, e.y);
    } else {
      reinterpret_cast<uint4*>(dst.p[r])[v] = val;
    }
  }
}

// K1 scatter of the chain output fused with K9 (head / top-1): one block per request row of fp32
// logits; the row is copied to dst[r] (when non-null) while the block reduces (value, index) to the
// first maximal index (torch.argmax's tie rule), written to top1[r].
struct RowTop1 {
  int32_t* p[kMaxRows];
};
__global__ void __launch_bounds__(256) scatter_top1_kernel(const float* __restrict__ src, int64_t row_elems,
                                                           RowDst dst, RowTop1 top1) {
  __shared__ float sv[8];
  __shared__ int si[8];
  const int r = blockIdx.x;
  const float* row = src + static_cast<int64_t>(r) * row_elems;
  float* out = static_cast<float*>(dst.p[r]);
  float best = -INFINITY;
  int bi = 0x7fffffff;
  const int64_t nv = row_elems / 4;
  for (int64_t v = threadIdx.x; v < nv; v += blockDim.x) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(row) + v);
    if (out) reinterpret_cast<float4*>(out)[v] = x;
    const float e[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int idx = static_cast<int>(4 * v + j);
      if (e[j] > best || (e[j] == best && idx < bi)) {
        best = e[j];
        bi = idx;
      }
    }
  }
  for (int64_t i = nv * 4 + threadIdx.x; i < row_elems; i += blockDim.x) {  // row_elems % 4 tail
    const float e = row[i];
    if (out) out[i] = e;
    if (e > best || (e == best && static_cast<int>(i) < bi)) {
      best = e;
      bi = static_cast<int>(i);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sv[warp] = best;
    si[warp] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) {
        best = sv[w];
        bi = si[w];
      }
    // a row of NaNs (no value compares greater than -inf) reports index 0
    *top1.p[r] = bi == 0x7fffffff ? 0 : bi;
  }
}

// K4 pooling over NHWC, 8 channels per thread (C % 8 == 0).  mode 0 = max, 1 = average.
// KR > 0: the window is KR x KR at compile time, so the taps unroll into independent (predicated)
// 16-byte loads that are all in flight before the reduction; KR = 0 is the generic window.
template <int KR>
__global__ void pool_kernel(int mode, const __nv_bfloat16* __restrict__ x, int N, int H, int W, int C, int x_ld,
                            __nv_bfloat16* __restrict__ y, int Ho, int Wo, int y_ld, int y_coff, int R, int S,
                            int sh, int sw, int ph, int pw, int count_include_pad) {
  const int cv = C / 8;
  const int64_t total = static_cast<int64_t>(N) * Ho * Wo * cv;
  // 32-bit index decomposition (the launcher guarantees total < 2^31): three 64-bit div/mod
  // sequences per 16-byte output cost more issue slots than the nine loads
  const int total32 = static_cast<int>(total);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total32; i += gridDim.x * blockDim.x) {
    const int c8 = i % cv;
    int p = i / cv;
    const int wo = p % Wo;
    p /= Wo;
    const int ho = p % Ho;
    const int n = p / Ho;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = mode == 0 ? -INFINITY : 0.0f;
    int cnt = 0;
    auto tap = [&](const uint4 v) {
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack_bf16x2(w[j]);
        if (mode == 0) {
          acc[2 * j] = fmaxf(acc[2 * j], f.x);
          acc[2 * j + 1] = fmaxf(acc[2 * j + 1], f.y);
        } else {
          acc[2 * j] += f.x;
          acc[2 * j + 1] += f.y;
        }
      }
      ++cnt;
    };
    if constexpr (KR > 0) {
      // all KR*KR taps are loaded first, from clamped in-bounds addresses, so they are independent
      // loads in flight together (SASS: 9 LDG.128 before the first FMNMX); padding taps are then
      // skipped in the reduction
      uint4 v[KR * KR];
#pragma unroll
      for (int r = 0; r < KR; ++r)
#pragma unroll
        for (int s = 0; s < KR; ++s) {
          const int hc = min(max(ho * sh - ph + r, 0), H - 1), wc = min(max(wo * sw - pw + s, 0), W - 1);
          v[r * KR + s] =
              __ldg(reinterpret_cast<const uint4*>(x + ((static_cast<int64_t>(n) * H + hc) * W + wc) * x_ld) + c8);
        }
#pragma unroll
      for (int r = 0; r < KR; ++r) {
        const int hi = ho * sh - ph + r;
#pragma unroll
        for (int s = 0; s < KR; ++s) {
          const int wi = wo * sw - pw + s;
          if (hi >= 0 && hi < H && wi >= 0 && wi < W) tap(v[r * KR + s]);
        }
      }
    } else {
      for (int r = 0; r < R; ++r) {
        const int hi = ho * sh - ph + r;
        if (hi < 0 || hi >= H) continue;
        for (int s = 0; s < S; ++s) {
          const int wi = wo * sw - pw + s;
          if (wi < 0 || wi >= W) continue;
          tap(__ldg(reinterpret_cast<const uint4*>(x + ((static_cast<int64_t>(n) * H + hi) * W + wi) * x_ld) + c8));
        }
      }
    }
    if (mode == 1) {
      // count_include_pad: divisor is the window clipped to the padded extent (PyTorch semantics)
      int div = cnt;
      if (count_include_pad) {
        const int h0 = ho * sh - ph, w0 = wo * sw - pw;
        const int h1 = min(h0 + R, H + ph), w1 = min(w0 + S, W + pw);
        div = (h1 - h0) * (w1 - w0);
      }
      const float inv = 1.0f / static_cast<float>(div);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] *= inv;
    }
    uint4 o;
    o.x = pack_bf16x2(acc[0], acc[1]);
    o.y = pack_bf16x2(acc[2], acc[3]);
    o.z = pack_bf16x2(acc[4], acc[5]);
    o.w = pack_bf16x2(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(y + ((static_cast<int64_t>(n) * Ho + ho) * Wo + wo) * y_ld + y_coff + 8 * c8) = o;
  }
}

// 3x3 / stride-1 pooling (Inception's branch_pool avg pools, and max): a thread owns a vertical
// strip of kPoolStrip outputs at one (column, 8 channels) and slides down it, combining each input
// row's three taps once into a row value (max or sum) and each output from three row values:
// 3*(T+2) loads for T outputs instead of 9*T.  Rows stream through a register ring with the loads
// of row j+1 issued before row j is combined (6 loads in flight, <= 85 registers: 3 blocks of 256
// per SM), and every address is one 32-bit offset from a per-thread base (round 1 held all 24
// taps and did the 64-bit index math per tap: 127 registers, 2 blocks per SM, issue-bound at 0.41
// of HBM).  The combine order is unchanged: row = ((id + t0) + t1) + t2, out = ((id + r0) + r1) + r2.
constexpr int kPoolStrip = 6;
__global__ void __launch_bounds__(256, 3) pool3s1_kernel(int mode, const __nv_bfloat16* __restrict__ x, int N, int H,
                                                        int W, int C, int x_ld, __nv_bfloat16* __restrict__ y,
                                                        int Ho, int Wo, int y_ld, int y_coff, int ph, int pw,
                                                        int count_include_pad) {
  constexpr int T = kPoolStrip;
  const int cv = C / 8;
  const int ldv = x_ld / 8;  // pixel pitch in 16-byte vectors
  const int strips = (Ho + T - 1) / T;
  const int total = N * strips * Wo * cv;  // < 2^31 (launcher)
  const float ident = mode == 0 ? -INFINITY : 0.0f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c8 = i % cv;
    int p = i / cv;
    const int wo = p % Wo;
    p /= Wo;
    const int st = p % strips;
    const int n = p / strips;
    const int ho0 = st * T;
    const int w0 = wo - pw;
    const uint4* base = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(n) * H * W * x_ld) + c8;
    int co[3];
    bool cok[3];
    int ncols = 0;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      cok[s] = w0 + s >= 0 && w0 + s < W;
      ncols += cok[s] ? 1 : 0;
      co[s] = min(max(w0 + s, 0), W - 1) * ldv;
    }
    const int rstep = W * ldv;
    uint4 raw[2][3];
    float rv[3][8];
    auto load_row = [&](int j) {
      const int ro = min(max(ho0 - ph + j, 0), H - 1) * rstep;
#pragma unroll
      for (int s = 0; s < 3; ++s) raw[j % 2][s] = __ldg(base + ro + co[s]);
    };
    load_row(0);
#pragma unroll
    for (int j = 0; j < T + 2; ++j) {
      if (j + 1 < T + 2) load_row(j + 1);
      float* r = rv[j % 3];
#pragma unroll
      for (int e = 0; e < 8; ++e) r[e] = ident;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        if (!cok[s]) continue;
        const uint4 v = raw[j % 2][s];
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = unpack_bf16x2(w[q]);
          if (mode == 0) {
            r[2 * q] = fmaxf(r[2 * q], f.x);
            r[2 * q + 1] = fmaxf(r[2 * q + 1], f.y);
          } else {
            r[2 * q] += f.x;
            r[2 * q + 1] += f.y;
          }
        }
      }
      const int t = j - 2;
      const int ho = ho0 + t;
      if (j < 2 || ho >= Ho) continue;
      float acc[8];
      int nrows = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = ident;
#pragma unroll
      for (int rr = 0; rr < 3; ++rr) {
        const int hi = ho - ph + rr;
        if (hi < 0 || hi >= H) continue;
        ++nrows;
        const float* rw = rv[(t + rr) % 3];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = mode == 0 ? fmaxf(acc[e], rw[e]) : acc[e] + rw[e];
      }
      if (mode == 1) {
        int div = nrows * ncols;
        if (count_include_pad) {
          const int h0 = ho - ph, ww0 = wo - pw;
          div = (min(h0 + 3, H + ph) - h0) * (min(ww0 + 3, W + pw) - ww0);
        }
        const float inv = 1.0f / static_cast<float>(div);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] *= inv;
      }
      uint4 o;
      o.x = pack_bf16x2(acc[0], acc[1]);
      o.y = pack_bf16x2(acc[2], acc[3]);
      o.z = pack_bf16x2(acc[4], acc[5]);
      o.w = pack_bf16x2(acc[6], acc[7]);
      *reinterpret_cast<uint4*>(y + (static_cast<int64_t>(n) * Ho + ho) * Wo * y_ld + wo * y_ld + y_coff + 8 * c8) = o;
    }
  }
}

// 3x3 max pool at any stride (the ResNet stem 3x3/2, Inception's 3x3/2 reductions): the nine taps
// are loaded from clamped coordinates (a clamped tap is another pixel of the same window, and max
// is idempotent, so no tap needs a predicate) and combined as packed bf16x2 maxima (exact: the
// result is one of the inputs), 4 HMNMX2 per tap instead of 8 unpacks + 8 FMNMX; addresses are
// 32-bit offsets from a per-sample base.  Round 1's generic kernel was issue-bound at 0.61 of HBM.
__global__ void __launch_bounds__(256) maxpool3_kernel(const __nv_bfloat16* __restrict__ x, int N, int H, int W,
                                                       int C, int x_ld, __nv_bfloat16* __restrict__ y, int Ho, int Wo,
                                                       int y_ld, int y_coff, int sh, int sw, int ph, int pw) {
  const int cv = C / 8;
  const int ldv = x_ld / 8;
  const int total = N * Ho * Wo * cv;  // < 2^31 (launcher)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c8 = i % cv;
    int p = i / cv;
    const int wo = p % Wo;
    p /= Wo;
    const int ho = p % Ho;
    const int n = p / Ho;
    const uint4* base = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(n) * H * W * x_ld) + c8;
    int ro[3], co[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      ro[t] = min(max(ho * sh - ph + t, 0), H - 1) * W * ldv;
      co[t] = min(max(wo * sw - pw + t, 0), W - 1) * ldv;
    }
    uint4 v[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) v[t] = __ldg(base + ro[t / 3] + co[t % 3]);
    __nv_bfloat162 m[4];
    m[0] = *reinterpret_cast<const __nv_bfloat162*>(&v[0].x);
    m[1] = *reinterpret_cast<const __nv_bfloat162*>(&v[0].y);
    m[2] = *reinterpret_cast<const __nv_bfloat162*>(&v[0].z);
    m[3] = *reinterpret_cast<const __nv_bfloat162*>(&v[0].w);
#pragma unroll
    for (int t = 1; t < 9; ++t) {
      m[0] = __hmax2(m[0], *reinterpret_cast<const __nv_bfloat162*>(&v[t].x));
      m[1] = __hmax2(m[1], *reinterpret_cast<const __nv_bfloat162*>(&v[t].y));
      m[2] = __hmax2(m[2], *reinterpret_cast<const __nv_bfloat162*>(&v[t].z));
      m[3] = __hmax2(m[3], *reinterpret_cast<const __nv_bfloat162*>(&v[t].w));
    }
    uint4 o;
    o.x = *reinterpret_cast<const uint32_t*>(&m[0]);
    o.y = *reinterpret_cast<const uint32_t*>(&m[1]);
    o.z = *reinterpret_cast<const uint32_t*>(&m[2]);
    o.w = *reinterpret_cast<const uint32_t*>(&m[3]);
    *reinterpret_cast<uint4*>(y + (static_cast<int64_t>(n) * Ho + ho) * Wo * y_ld + wo * y_ld + y_coff + 8 * c8) = o;
  }
}

// Global average pool: [N, HW, C] -> [N, C].  A warp owns one (sample, 256 channels) item: lane =
// 8 channels (the warp reads 512 contiguous bytes of one pixel) and walks the HW pixels with 4
// independent 16-byte loads in flight per lane, accumulating in fp32 registers; no shared memory
// and no block barriers, so the 8 warps of a block stream 8 items concurrently.  At <= 32
// registers 8 blocks fit per SM, so a 1024-sample batch (8192 items) is resident in one wave; with
// 8 loads in flight (40 registers, 6 blocks per SM) 15% of the items ran as a second, near-empty
// wave (0.62 of HBM).  (Round 1 split one item over the 8 warps through shared memory: 0.55.)
constexpr int kGapWarps = 8;
__global__ void __launch_bounds__(kGapWarps * 32, 8) gap_kernel(const __nv_bfloat16* __restrict__ x, int N, int HW,
                                                            int C, __nv_bfloat16* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int cv = C / 8;
  const int groups = (cv + 31) / 32;
  const float inv = 1.0f / HW;
  const int64_t items = static_cast<int64_t>(N) * groups;
  const int64_t wstride = static_cast<int64_t>(gridDim.x) * kGapWarps;
  for (int64_t item = static_cast<int64_t>(blockIdx.x) * kGapWarps + (threadIdx.x >> 5); item < items;
       item += wstride) {
    const int n = static_cast<int>(item / groups);
    const int c8 = static_cast<int>(item % groups) * 32 + lane;
    if (c8 >= cv) continue;
    const uint4* base = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(n) * HW * C) + c8;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    constexpr int U = 4;  // <= 32 registers: 8 blocks (64 warps) per SM, every item resident in one wave
    for (int p0 = 0; p0 < HW; p0 += U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        v[u] = p0 + u < HW ? ldg_stream(base + static_cast<int64_t>(p0 + u) * cv) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack_bf16x2(w[j]);
          acc[2 * j] += f.x;
          acc[2 * j + 1] += f.y;
        }
      }
    }
    uint4 o;
    o.x = pack_bf16x2(acc[0] * inv, acc[1] * inv);
    o.y = pack_bf16x2(acc[2] * inv, acc[3] * inv);
    o.z = pack_bf16x2(acc[4] * inv, acc[5] * inv);
    o.w = pack_bf16x2(acc[6] * inv, acc[7] * inv);
    reinterpret_cast<uint4*>(y + static_cast<int64_t>(n) * C)[c8] = o;
  }
}

// GAP for few items (the batch-1..4 tails of a serving plan): one item per block, its 8 warps split
// the HW pixels (one load per warp per pixel row of the walk, all in flight) and reduce through
// shared memory; the per-warp kernel above would leave all but a handful of warps idle and walk 49
// pixels in 7 dependent rounds.
__global__ void __launch_bounds__(kGapWarps * 32) gap_split_kernel(const __nv_bfloat16* __restrict__ x, int N, int HW,
                                                                  int C, __nv_bfloat16* __restrict__ y) {
  __shared__ float part[kGapWarps][32][9];  // +1 pad: lane-strided rows hit distinct banks
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cv = C / 8;
  const int groups = (cv + 31) / 32;
  const float inv = 1.0f / HW;
  for (int64_t item = blockIdx.x; item < static_cast<int64_t>(N) * groups; item += gridDim.x) {
    const int n = static_cast<int>(item / groups);
    const int c8 = static_cast<int>(item % groups) * 32 + lane;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (c8 < cv) {
      const uint4* base = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(n) * HW * C) + c8;
      constexpr int U = 8;
      for (int p0 = warp; p0 < HW; p0 += kGapWarps * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int pp = p0 + u * kGapWarps;
          v[u] = pp < HW ? ldg_stream(base + static_cast<int64_t>(pp) * cv) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = unpack_bf16x2(w[j]);
            acc[2 * j] += f.x;
            acc[2 * j + 1] += f.y;
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) part[warp][lane][j] = acc[j];
    __syncthreads();
    if (warp == 0 && c8 < cv) {
      float t[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        t[j] = 0.0f;
#pragma unroll
        for (int w = 0; w < kGapWarps; ++w) t[j] += part[w][lane][j];
      }
      uint4 o;
      o.x = pack_bf16x2(t[0] * inv, t[1] * inv);
      o.y = pack_bf16x2(t[2] * inv, t[3] * inv);
      o.z = pack_bf16x2(t[4] * inv, t[5] * inv);
      o.w = pack_bf16x2(t[6] * inv, t[7] * inv);
      reinterpret_cast<uint4*>(y + static_cast<int64_t>(n) * C)[c8] = o;
    }
    __syncthreads();
  }
}

// Skinny FC at small batch (weight-streaming, HBM-bound): y[n][o] = x[n] . w[o] + b[o].
// Block = 8 warps; warp w owns OPW consecutive output features; lanes stride K in 16-byte
// vectors.  The batch rows are staged in shared memory one K-chunk at a time (each weight byte is
// read from HBM exactly once, x comes from smem), 16 rows per accumulator pass.
constexpr int kFcWarps = 8;
constexpr int kFcRows = 16;
constexpr int kFcKChunk = 2048;
template <int OPW, int ROWS>
__global__ void __launch_bounds__(256, 2) fc_kernel(const __nv_bfloat16* __restrict__ x, int N, int K,
                                                 const __nv_bfloat16* __restrict__ w, const float* __restrict__ b,
                                                 void* __restrict__ y, int Nout, int y_f32, int act) {
  extern __shared__ uint4 xs[];  // [ROWS][kFcKChunk / 8]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int groups = (Nout + kFcWarps * OPW - 1) / (kFcWarps * OPW);
  int64_t staged = -1;
  for (int g = blockIdx.x; g < groups; g += gridDim.x) {
    const int o0 = (g * kFcWarps + warp) * OPW;
    for (int n0 = 0; n0 < N; n0 += ROWS) {
      const int rows = min(ROWS, N - n0);
      float acc[OPW][ROWS];
#pragma unroll
      for (int a = 0; a < OPW; ++a)
#pragma unroll
        for (int r = 0; r < ROWS; ++r) acc[a][r] = 0.0f;
      for (int k0 = 0; k0 < K; k0 += kFcKChunk) {
        const int kc = min(kFcKChunk, K - k0) / 8;  // 16-byte vectors in this chunk
        const int64_t key = static_cast<int64_t>(n0) * K + k0;
        if (key != staged) {  // block-uniform: re-stage only when the (rows, K-chunk) changes
          __syncthreads();
          for (int i = threadIdx.x; i < rows * kc; i += blockDim.x) {
            const int r = i / kc, v = i - r * kc;
            xs[r * (kFcKChunk / 8) + v] =
                __ldg(reinterpret_cast<const uint4*>(x + static_cast<int64_t>(n0 + r) * K + k0) + v);
          }
          __syncthreads();
          staged = key;
        }
        // 8 independent 16-byte weight loads in flight per lane (U vectors x OPW outputs) before
        // any FMA: at a few-SM budget the kernel is latency-bound on L2/HBM, not FMA-bound
        constexpr int U = OPW >= 4 ? 1 : 8 / OPW;
        for (int v0 = lane; v0 < kc; v0 += 32 * U) {
          uint4 wv[U][OPW];
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int a = 0; a < OPW; ++a) {
              const int v = v0 + 32 * u;
              wv[u][a] = (v < kc && o0 + a < Nout)
                             ? ldg_stream(reinterpret_cast<const uint4*>(w + static_cast<int64_t>(o0 + a) * K + k0) + v)
                             : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int v = v0 + 32 * u;
            if (v >= kc) break;
            float wf[OPW][8];
#pragma unroll
            for (int a = 0; a < OPW; ++a) {
              const uint32_t ww[4] = {wv[u][a].x, wv[u][a].y, wv[u][a].z, wv[u][a].w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float2 f = unpack_bf16x2(ww[j]);
                wf[a][2 * j] = f.x;
                wf[a][2 * j + 1] = f.y;
              }
            }
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
              if (r < rows) {
                const uint4 xv = xs[r * (kFcKChunk / 8) + v];
                const uint32_t xx[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float2 f = unpack_bf16x2(xx[j]);
#pragma unroll
                  for (int a = 0; a < OPW; ++a) {
                    acc[a][r] = fmaf(wf[a][2 * j], f.x, acc[a][r]);
                    acc[a][r] = fmaf(wf[a][2 * j + 1], f.y, acc[a][r]);
                  }
                }
              }
            }
          }
        }
      }
      // warm L2 with the next group's weight rows while this group reduces and stores
      {
        const int gn = g + gridDim.x;
        if (gn < groups && n0 + ROWS >= N) {
#pragma unroll
          for (int a = 0; a < OPW; ++a) {
            const int on = (gn * kFcWarps + warp) * OPW + a;
            if (on < Nout) {
              const char* rowp = reinterpret_cast<const char*>(w + static_cast<int64_t>(on) * K);
              for (int64_t off = static_cast<int64_t>(lane) * 128; off < static_cast<int64_t>(K) * 2; off += 32 * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(rowp + off));
            }
          }
        }
      }
      // butterfly-reduce the rows this pass holds (ROWS = batch rounded up to a power of two)
#pragma unroll
      for (int a = 0; a < OPW; ++a)
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          if (r < rows) {
            float v = acc[a][r];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            acc[a][r] = v;
          }
        }
      // lane r writes row r (r < 16) for each of the warp's outputs
#pragma unroll
      for (int a = 0; a < OPW; ++a) {
        const int o = o0 + a;
        float mine = 0.0f;
#pragma unroll
        for (int r = 0; r < ROWS; ++r)
          if (lane == r) mine = acc[a][r];
        if (o < Nout && lane < rows) {
          float v = mine + (b ? b[o] : 0.0f);
          if (act == GX_ACT_RELU) v = fmaxf(v, 0.0f);
          const int64_t idx = static_cast<int64_t>(n0 + lane) * Nout + o;
          if (y_f32)
            static_cast<float*>(y)[idx] = v;
          else
            static_cast<__nv_bfloat16*>(y)[idx] = __float2bfloat16_rn(v);
        }
      }
    }
  }
}

__global__ void copy_channels_kernel(const __nv_bfloat16* __restrict__ x, int64_t pixels, int C, int x_ld,
                                     int x_coff, __nv_bfloat16* __restrict__ y, int y_ld, int y_coff) {
  const int cv = C / 8;
  const int total = static_cast<int>(pixels * cv);  // < 2^31 (launcher)
  const int stride = gridDim.x * blockDim.x;
  // (pixel, vector) of the thread's element advanced incrementally: one division per thread, none
  // per element (a 32-bit division by the runtime vector count per 16-byte element made the copy
  // issue-bound at 0.62 of HBM)
  const int dp = stride / cv, dr = stride - dp * cv;
  int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  int p0 = i0 / cv, r0 = i0 - p0 * cv;
  // 4 independent 16-byte loads in flight per thread, then the 4 stores
  for (; i0 < total; i0 += 4 * stride) {
    uint4 v[4];
    int pp[4], rr[4];
    int p = p0, r = r0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      pp[u] = p;
      rr[u] = r;
      if (i0 + u * stride < total)
        v[u] = ldg_stream(reinterpret_cast<const uint4*>(x + static_cast<int64_t>(p) * x_ld + x_coff) + r);
      p += dp;
      r += dr;
      if (r >= cv) {
        r -= cv;
        ++p;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * stride < total)
        reinterpret_cast<uint4*>(y + static_cast<int64_t>(pp[u]) * y_ld + y_coff)[rr[u]] = v[u];
    p0 = p;
    r0 = r;
  }
}

inline int grid_for(int64_t work_items, int threads, int grid_cap) {
  int64_t g = (work_items + threads - 1) / threads;
  if (g > grid_cap) g = grid_cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}
}  // namespace

cudaError_t launch_gather(int k, const void* const* src, const int32_t* src_dtype, int64_t pixels, int c_src,
                          int c_dst, __nv_bfloat16* dst, int grid, cudaStream_t s) {
  if (k > kMaxRows) return cudaErrorInvalidValue;
  RowPtrs rp;
  for (int i = 0; i < k; ++i) {
    rp.p[i] = src[i];
    rp.dt[i] = src_dtype[i];
  }
  const int64_t work = (c_src == c_dst && (c_dst & 7) == 0) ? pixels * c_dst / 8 * k : pixels * c_dst * k;
  gather_kernel<<<grid_for(work, 256, grid), 256, 0, s>>>(rp, k, pixels, c_src, c_dst, dst);
  return cudaGetLastError();
}

cudaError_t launch_gather_s2d(int k, const void* const* src, const int32_t* src_dtype, int Ho, int Wo, int f,
                              int c_src, int c_dst, __nv_bfloat16* dst, int grid, cudaStream_t s) {
  if (k > kMaxRows || f * f * c_src > c_dst) return cudaErrorInvalidValue;
  RowPtrs rp;
  for (int i = 0; i < k; ++i) {
    rp.p[i] = src[i];
    rp.dt[i] = src_dtype[i];
  }
  if (f == 2 && c_src == 3 && c_dst == 16 && (Wo & 1) == 0) {  // the ResNet stems: one thread per output pixel
    const int64_t work = static_cast<int64_t>(Ho) * Wo * k;
    gather_s2d_rgb2_kernel<<<grid_for(work, 256, grid), 256, 0, s>>>(rp, k, Ho, Wo, dst);
    return cudaGetLastError();
  }
  const int64_t work = static_cast<int64_t>(Ho) * Wo * c_dst * k;
  gather_s2d_kernel<<<grid_for(work, 256, grid), 256, 0, s>>>(rp, k, Ho, Wo, f, c_src, c_dst, dst);
  return cudaGetLastError();
}

cudaError_t launch_gather_words(int k, const void* const* src, int64_t words, uint32_t* dst, int grid,
                                cudaStream_t s) {
  if (k > kMaxRows) return cudaErrorInvalidValue;
  RowPtrs rp;
  for (int i = 0; i < k; ++i) rp.p[i] = src[i];
  gather_words_kernel<<<grid_for(words * k, 256, grid), 256, 0, s>>>(rp, k, words, dst);
  return cudaGetLastError();
}

cudaError_t launch_scatter(int k, const void* src, int src_dtype, int64_t row_elems, void* const* dst,
                           int dst_dtype, int grid, cudaStream_t s) {
  if (k > kMaxRows || (row_elems & 7)) return cudaErrorInvalidValue;
  RowDst rd;
  for (int i = 0; i < k; ++i) rd.p[i] = dst[i];
  scatter_kernel<<<grid_for(row_elems / 8 * k, 256, grid), 256, 0, s>>>(src, src_dtype == GX_F32, k, row_elems, rd,
                                                                     dst_dtype == GX_F32);
  return cudaGetLastError();
}

cudaError_t launch_scatter_top1(int k, const float* src, int64_t row_elems, void* const* dst, int32_t* const* top1,
                                cudaStream_t s) {
  if (k > kMaxRows || (row_elems & 3) || (reinterpret_cast<uintptr_t>(src) & 15)) return cudaErrorInvalidValue;
  RowDst rd;
  RowTop1 rt;
  for (int i = 0; i < k; ++i) {
    rd.p[i] = dst ? dst[i] : nullptr;
    rt.p[i] = top1[i];
    if (!rt.p[i]) return cudaErrorInvalidValue;
  }
  scatter_top1_kernel<<<k, 256, 0, s>>>(src, row_elems, rd, rt);
  return cudaGetLastError();
}

cudaError_t launch_pool(int mode, const __nv_bfloat16* x, int N, int H, int W, int C, int x_ld, __nv_bfloat16* y,
                        int Ho, int Wo, int y_ld, int y_coff, int R, int S, int sh, int sw, int ph, int pw,
                        int count_include_pad, int grid, cudaStream_t s) {
  if (C & 7) return cudaErrorInvalidValue;
  const int64_t work = static_cast<int64_t>(N) * Ho * Wo * (C / 8);
  if (work >= (int64_t{1} << 31)) return cudaErrorInvalidValue;
  if (R == 3 && S == 3 && sh == 1 && sw == 1 && ph <= 2 && pw <= 2 && !dev().pool_nostrip) {
    const int64_t strips = static_cast<int64_t>(N) * ((Ho + kPoolStrip - 1) / kPoolStrip) * Wo * (C / 8);
    pool3s1_kernel<<<grid_for(strips, 256, grid), 256, 0, s>>>(mode, x, N, H, W, C, x_ld, y, Ho, Wo, y_ld, y_coff, ph,
                                                               pw, count_include_pad);
  } else if (R == 3 && S == 3 && mode == 0 && (x_ld & 7) == 0)
    maxpool3_kernel<<<grid_for(work, 256, grid), 256, 0, s>>>(x, N, H, W, C, x_ld, y, Ho, Wo, y_ld, y_coff, sh, sw, ph,
                                                              pw);
  else if (R == 3 && S == 3)
    pool_kernel<3><<<grid_for(work, 256, grid), 256, 0, s>>>(mode, x, N, H, W, C, x_ld, y, Ho, Wo, y_ld, y_coff, R, S,
                                                             sh, sw, ph, pw, count_include_pad);
  else
    pool_kernel<0><<<grid_for(work, 256, grid), 256, 0, s>>>(mode, x, N, H, W, C, x_ld, y, Ho, Wo, y_ld, y_coff, R, S,
                                                             sh, sw, ph, pw, count_include_pad);
  return cudaGetLastError();
}

cudaError_t launch_gap(const __nv_bfloat16* x, int N, int HW, int C, __nv_bfloat16* y, int grid, cudaStream_t s) {
  if (C & 7) return cudaErrorInvalidValue;
  const int64_t items = static_cast<int64_t>(N) * ((C / 8 + 31) / 32);
  if (items < 4 * static_cast<int64_t>(grid))  // few items: one block per item, warps split the pixels
    gap_split_kernel<<<grid_for(items, 1, grid), kGapWarps * 32, 0, s>>>(x, N, HW, C, y);
  else
    gap_kernel<<<grid_for(items, kGapWarps, grid), kGapWarps * 32, 0, s>>>(x, N, HW, C, y);
  return cudaGetLastError();
}

cudaError_t launch_fc(const __nv_bfloat16* x, int N, int K, const __nv_bfloat16* w, const float* b, void* y, int Nout,
                      int y_f32, int act, int grid, cudaStream_t s) {
  if (K & 7) return cudaErrorInvalidValue;
  // rows per accumulator pass = the batch rounded up to a power of two (<= 16): the unrolled
  // per-row FMA / reduction work matches k instead of a fixed 16-row capacity
  const int rows = N >= 16 ? 16 : N > 4 ? 8 : N > 2 ? 4 : N;
  const size_t smem = static_cast<size_t>(rows) * kFcKChunk * 2;
  static bool configured = false;
  if (!configured) {
    const int mx = static_cast<int>(static_cast<size_t>(kFcRows) * kFcKChunk * 2);
#define GX_FC_ATTR(O, R) cudaFuncSetAttribute(fc_kernel<O, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    GX_FC_ATTR(1, 1) GX_FC_ATTR(1, 2) GX_FC_ATTR(1, 4) GX_FC_ATTR(1, 8) GX_FC_ATTR(1, 16)
    GX_FC_ATTR(2, 1) GX_FC_ATTR(2, 2) GX_FC_ATTR(2, 4) GX_FC_ATTR(2, 8) GX_FC_ATTR(2, 16)
    GX_FC_ATTR(4, 1) GX_FC_ATTR(4, 2) GX_FC_ATTR(4, 4) GX_FC_ATTR(4, 8) GX_FC_ATTR(4, 16)
#undef GX_FC_ATTR
    configured = true;
  }
  const int opw = Nout >= 4096 ? 4 : Nout >= 2048 ? 2 : 1;
  const int groups = (Nout + kFcWarps * opw - 1) / (kFcWarps * opw);
  // up to 3 blocks per SM of the budget: weight streaming needs many loads in flight
  const int g = grid_for(groups, 1, grid / 8 > 0 ? 3 * (grid / 8) : 1);
#define GX_FC_LAUNCH(O, R) fc_kernel<O, R><<<g, 256, smem, s>>>(x, N, K, w, b, y, Nout, y_f32, act)
#define GX_FC_ROWS(O)               \
  switch (rows) {                   \
    case 1: GX_FC_LAUNCH(O, 1); break; \
    case 2: GX_FC_LAUNCH(O, 2); break; \
    case 4: GX_FC_LAUNCH(O, 4); break; \
    case 8: GX_FC_LAUNCH(O, 8); break; \
    default: GX_FC_LAUNCH(O, 16); break; \
  }
  if (opw == 4) {
    GX_FC_ROWS(4)
  } else if (opw == 2) {
    GX_FC_ROWS(2)
  } else {
    GX_FC_ROWS(1)
  }
#undef GX_FC_ROWS
#undef GX_FC_LAUNCH
  return cudaGetLastError();
}

cudaError_t launch_copy_channels(const __nv_bfloat16* x, int64_t pixels, int C, int x_ld, int x_coff,
                                 __nv_bfloat16* y, int y_ld, int y_coff, int grid, cudaStream_t s) {
  if ((C | x_ld | x_coff | y_ld | y_coff) & 7) return cudaErrorInvalidValue;
  if (pixels * (C / 8) >= (int64_t{1} << 31)) return cudaErrorInvalidValue;
  copy_channels_kernel<<<grid_for(pixels * (C / 8), 256, grid), 256, 0, s>>>(x, pixels, C, x_ld, x_coff, y, y_ld,
                                                                             y_coff);
  return cudaGetLastError();
}

}  // namespace gx
