// Device bodies of the bandwidth-bound ops, shared by the standalone kernels and the persistent
// span kernel.  Every body is a strided loop over work items [i0, total) step `stride`.
#pragma once
#include <cuda_bf16.h>

#include "gx_ptx.cuh"

namespace gx {

// NHWC pooling, 8 channels per work item.  mode 0 = max, 1 = average (PyTorch divisor rules).
__device__ __forceinline__ void pool_body(int mode, const __nv_bfloat16* __restrict__ x, int N, int H, int W, int C,
                                          int x_ld, __nv_bfloat16* __restrict__ y, int Ho, int Wo, int y_ld,
                                          int y_coff, int R, int S, int sh, int sw, int ph, int pw,
                                          int count_include_pad, int64_t i0, int64_t stride) {
  const int cv = C / 8;
  const int64_t total = static_cast<int64_t>(N) * Ho * Wo * cv;
  for (int64_t i = i0; i < total; i += stride) {
    const int c8 = static_cast<int>(i % cv);
    int64_t p = i / cv;
    const int wo = static_cast<int>(p % Wo);
    p /= Wo;
    const int ho = static_cast<int>(p % Ho);
    const int n = static_cast<int>(p / Ho);
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = mode == 0 ? -INFINITY : 0.0f;
    int cnt = 0;
    if (R == 3 && S == 3) {
      // all nine window loads in flight at once (latency-bound otherwise)
      uint4 v[9];
      bool ok[9];
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        const int hi = ho * sh - ph + t / 3, wi = wo * sw - pw + t % 3;
        ok[t] = hi >= 0 && hi < H && wi >= 0 && wi < W;
        v[t] = ok[t] ? __ldcg(reinterpret_cast<const uint4*>(x + ((static_cast<int64_t>(n) * H + hi) * W + wi) * x_ld) +
                              c8)
                     : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        if (!ok[t]) continue;
        const uint32_t w[4] = {v[t].x, v[t].y, v[t].z, v[t].w};
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
      }
    }
    for (int r = 0; r < R && !(R == 3 && S == 3); ++r) {
      const int hi = ho * sh - ph + r;
      if (hi < 0 || hi >= H) continue;
      for (int s = 0; s < S; ++s) {
        const int wi = wo * sw - pw + s;
        if (wi < 0 || wi >= W) continue;
        const uint4 v =
            __ldcg(reinterpret_cast<const uint4*>(x + ((static_cast<int64_t>(n) * H + hi) * W + wi) * x_ld) + c8);
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
      }
    }
    if (mode == 1) {
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

// Global average pool [N, HW, C] -> [N, C], 8 channels per work item.
__device__ __forceinline__ void gap_body(const __nv_bfloat16* __restrict__ x, int N, int HW, int C,
                                         __nv_bfloat16* __restrict__ y, int64_t i0, int64_t stride) {
  const int cv = C / 8;
  const int64_t total = static_cast<int64_t>(N) * cv;
  const float inv = 1.0f / HW;
  for (int64_t i = i0; i < total; i += stride) {
    const int n = static_cast<int>(i / cv);
    const int c8 = static_cast<int>(i % cv);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const uint4* base = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(n) * HW * C) + c8;
#pragma unroll 7
    for (int p = 0; p < HW; ++p) {
      const uint4 v = __ldcg(base + static_cast<int64_t>(p) * cv);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack_bf16x2(w[j]);
        acc[2 * j] += f.x;
        acc[2 * j + 1] += f.y;
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

// Small-batch FC, one warp per output feature (no shared memory): weights streamed once,
// activations re-read through L1/L2.  Work item = output feature; lane strides K by 8.
__device__ __forceinline__ void fc_warp_body(const __nv_bfloat16* __restrict__ x, int N, int K,
                                             const __nv_bfloat16* __restrict__ w, const float* __restrict__ b,
                                             void* __restrict__ y, int Nout, int y_f32, int act, int warp0,
                                             int nwarps, int lane) {
  constexpr int kRows = 16;
  const int kv = K / 8;
  for (int o = warp0; o < Nout; o += nwarps) {
    for (int n0 = 0; n0 < N; n0 += kRows) {
      const int rows = min(kRows, N - n0);
      float acc[kRows];
#pragma unroll
      for (int r = 0; r < kRows; ++r) acc[r] = 0.0f;
      for (int v = lane; v < kv; v += 32) {
        const uint4 wv = __ldg(reinterpret_cast<const uint4*>(w + static_cast<int64_t>(o) * K) + v);
        const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
        float wf[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack_bf16x2(ww[j]);
          wf[2 * j] = f.x;
          wf[2 * j + 1] = f.y;
        }
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          if (r < rows) {
            const uint4 xv = __ldcg(reinterpret_cast<const uint4*>(x + static_cast<int64_t>(n0 + r) * K) + v);
            const uint32_t xx[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 f = unpack_bf16x2(xx[j]);
              acc[r] = fmaf(wf[2 * j], f.x, acc[r]);
              acc[r] = fmaf(wf[2 * j + 1], f.y, acc[r]);
            }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        float v = acc[r];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        acc[r] = v;
      }
      float mine = 0.0f;
#pragma unroll
      for (int r = 0; r < kRows; ++r)
        if (lane == r) mine = acc[r];
      if (lane < rows) {
        float v = mine + (b ? b[o] : 0.0f);
        if (act == 1) v = fmaxf(v, 0.0f);
        const int64_t idx = static_cast<int64_t>(n0 + lane) * Nout + o;
        if (y_f32)
          static_cast<float*>(y)[idx] = v;
        else
          static_cast<__nv_bfloat16*>(y)[idx] = __float2bfloat16_rn(v);
      }
    }
  }
}

// Small-batch FC, one warp per group of 4 output features: the 4 weight rows stream together (4
// independent 16 B loads per lane per step), activations come through L2.  Work item = group.
__device__ __forceinline__ void fc_warp4_body(const __nv_bfloat16* __restrict__ x, int N, int K,
                                              const __nv_bfloat16* __restrict__ w, const float* __restrict__ b,
                                              void* __restrict__ y, int Nout, int y_f32, int act, int warp0,
                                              int nwarps, int lane) {
  constexpr int kRows = 8;
  constexpr int kO = 4;
  const int kv = K / 8;
  const int groups = (Nout + kO - 1) / kO;
  for (int g = warp0; g < groups; g += nwarps) {
    const int o0 = g * kO;
    for (int n0 = 0; n0 < N; n0 += kRows) {
      const int rows = min(kRows, N - n0);
      float acc[kO][kRows];
#pragma unroll
      for (int a = 0; a < kO; ++a)
#pragma unroll
        for (int r = 0; r < kRows; ++r) acc[a][r] = 0.0f;
#pragma unroll 2
      for (int v = lane; v < kv; v += 32) {
        uint4 wv[kO];
#pragma unroll
        for (int a = 0; a < kO; ++a)
          wv[a] = o0 + a < Nout ? __ldg(reinterpret_cast<const uint4*>(w + static_cast<int64_t>(o0 + a) * K) + v)
                                : make_uint4(0, 0, 0, 0);
        uint4 xv[kRows];
#pragma unroll
        for (int r = 0; r < kRows; ++r)
          xv[r] = r < rows ? __ldcg(reinterpret_cast<const uint4*>(x + static_cast<int64_t>(n0 + r) * K) + v)
                           : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int a = 0; a < kO; ++a) {
          const uint32_t ww[4] = {wv[a].x, wv[a].y, wv[a].z, wv[a].w};
#pragma unroll
          for (int r = 0; r < kRows; ++r) {
            const uint32_t xx[4] = {xv[r].x, xv[r].y, xv[r].z, xv[r].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 fw = unpack_bf16x2(ww[j]);
              const float2 fx = unpack_bf16x2(xx[j]);
              acc[a][r] = fmaf(fw.x, fx.x, acc[a][r]);
              acc[a][r] = fmaf(fw.y, fx.y, acc[a][r]);
            }
          }
        }
      }
#pragma unroll
      for (int a = 0; a < kO; ++a)
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          float v = acc[a][r];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
          acc[a][r] = v;
        }
      // lane (a * kRows + r) writes output o0 + a of row n0 + r
      float mine = 0.0f;
#pragma unroll
      for (int a = 0; a < kO; ++a)
#pragma unroll
        for (int r = 0; r < kRows; ++r)
          if (lane == a * kRows + r) mine = acc[a][r];
      const int a = lane / kRows, r = lane % kRows;
      const int o = o0 + a;
      if (o < Nout && r < rows) {
        float v = mine + (b ? b[o] : 0.0f);
        if (act == 1) v = fmaxf(v, 0.0f);
        const int64_t idx = static_cast<int64_t>(n0 + r) * Nout + o;
        if (y_f32)
          static_cast<float*>(y)[idx] = v;
        else
          static_cast<__nv_bfloat16*>(y)[idx] = __float2bfloat16_rn(v);
      }
    }
  }
}

// Channel-slice copy, 8 channels per work item.
__device__ __forceinline__ void copy_body(const __nv_bfloat16* __restrict__ x, int64_t pixels, int C, int x_ld,
                                          int x_coff, __nv_bfloat16* __restrict__ y, int y_ld, int y_coff,
                                          int64_t i0, int64_t stride) {
  const int cv = C / 8;
  const int64_t total = pixels * cv;
  for (int64_t i = i0; i < total; i += stride) {
    const int64_t p = i / cv;
    const int c8 = static_cast<int>(i - p * cv);
    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(x + p * x_ld + x_coff) + c8);
    reinterpret_cast<uint4*>(y + p * y_ld + y_coff)[c8] = v;
  }
}

}  // namespace gx
