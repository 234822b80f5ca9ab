// fp32 execution mode (north star: outputs within 1e-3 of the fp32 forward): every op of a chain
// whose tensors are GX_F32, in fp32 end to end on the CUDA cores.
//
//   conv_f32_kernel       implicit-GEMM conv / token-wise linear / FC (a 1x1 conv on a 1x1 image):
//                         64x64 output tiles, K in steps of 16 staged through shared memory
//                         (register-prefetched double buffer), 4x4 outputs per thread, fused bias /
//                         residual / ReLU / GELU epilogue writing a channel slice (concat).  Each
//                         output sums its K terms in one fixed order (k = (r, s, cin) ascending),
//                         independent of batch, tile and SM budget, so a request's bits do not
//                         depend on the batch it rides in (split-vs-whole bit-exactness).
//   pool / gap / copy     NHWC, 4-channel vectors when aligned;
//   layernorm             one warp per row, two-pass mean / variance;
//   attention             one CTA per (request, head): K and V of the head staged in shared memory,
//                         one warp per query row, exact softmax (max-subtracted, fp32);
//   gather                k entry activations (fp32 ingress / fp32 alignment outputs) -> one fp32
//                         batch, channel padding and the space-to-depth stem rearrangement fused.
// Persistent grid-stride loops bounded by the stage's SM budget like the bf16 kernels.
#include <cuda_bf16.h>

#include <cmath>

#include "gx_internal.h"

namespace gx {

namespace {
constexpr int kMaxRows = 64;
struct RowPtrs {
  const void* p[kMaxRows];
  int32_t dt[kMaxRows];
};

__device__ __forceinline__ float load_any(const void* p, int dt, int64_t i) {
  return dt == GX_F32 ? __ldg(static_cast<const float*>(p) + i)
                      : __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}

__device__ __forceinline__ float act_f32(float v, int act) {
  if (act == GX_ACT_RELU) return fmaxf(v, 0.0f);
  if (act == GX_ACT_GELU) return 0.5f * v * (1.0f + erff(v * 0.70710678118654752f));
  return v;
}

// ------------------------------------------------------------------ implicit-GEMM conv (fp32)
constexpr int kTM = 64, kTN = 64, kTK = 16, kF32Threads = 256;

__global__ void __launch_bounds__(kF32Threads) conv_f32_kernel(const ConvF32Args a) {
  __shared__ __align__(16) float As[2][kTK][kTM + 4];
  __shared__ __align__(16) float Bs[2][kTK][kTN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // compute: 4 output channels x 4 output pixels
  const int lk = tid & 15, lr = tid >> 4;  // loads: k column lk, rows lr + 16*i
  const int HoWo = a.Ho * a.Wo;
  const int m_tiles = (a.M + kTM - 1) / kTM, n_tiles = (a.Cout + kTN - 1) / kTN;
  const int k_steps = (a.K + kTK - 1) / kTK;
  for (int tile = blockIdx.x; tile < m_tiles * n_tiles; tile += gridDim.x) {
    const int m0 = (tile / n_tiles) * kTM, n0 = (tile % n_tiles) * kTN;
    // per loaded row: image, top-left input coordinate (or invalid)
    int img[4], hb[4], wb[4];
    bool mok[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + lr + 16 * i;
      mok[i] = m < a.M;
      const int mm = mok[i] ? m : 0;
      img[i] = mm / HoWo;
      const int rem = mm - img[i] * HoWo;
      const int ho = rem / a.Wo, wo = rem - (rem / a.Wo) * a.Wo;
      hb[i] = ho * a.sh - a.ph;
      wb[i] = wo * a.sw - a.pw;
    }
    float ra[4], rb[4];
    auto fetch = [&](int ks) {
      const int k = ks * kTK + lk;
      const bool kok = k < a.K;
      int r = 0, s = 0, c = 0;
      if (kok) {
        const int tap = k / a.Cin;
        c = k - tap * a.Cin;
        r = tap / a.S;
        s = tap - r * a.S;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int hi = hb[i] + r, wi = wb[i] + s;
        const bool ok = kok && mok[i] && static_cast<unsigned>(hi) < static_cast<unsigned>(a.H) &&
                        static_cast<unsigned>(wi) < static_cast<unsigned>(a.W);
        ra[i] = ok ? __ldg(a.x + ((static_cast<int64_t>(img[i]) * a.H + hi) * a.W + wi) * a.x_ld + c) : 0.0f;
        const int co = n0 + lr + 16 * i;
        rb[i] = (kok && co < a.Cout) ? __ldg(a.w + static_cast<int64_t>(co) * a.w_ld + k) : 0.0f;
      }
    };
    auto stash = [&](int buf) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        As[buf][lk][lr + 16 * i] = ra[i];
        Bs[buf][lk][lr + 16 * i] = rb[i];
      }
    };
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    fetch(0);
    stash(0);
    __syncthreads();
    for (int ks = 0; ks < k_steps; ++ks) {
      const int buf = ks & 1;
      if (ks + 1 < k_steps) fetch(ks + 1);  // next tile's loads in flight during the math
#pragma unroll
      for (int kk = 0; kk < kTK; ++kk) {
        const float4 av = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
        const float4 bv = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
        const float am[4] = {av.x, av.y, av.z, av.w}, bn[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(am[i], bn[j], acc[i][j]);
      }
      if (ks + 1 < k_steps) stash(buf ^ 1);
      __syncthreads();
    }
    // epilogue: + bias (+ residual) -> act -> y[m][y_coff + co]
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + ty * 4 + i;
      if (m >= a.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int co = n0 + tx * 4 + j;
        if (co >= a.Cout) continue;
        float v = acc[i][j] + (a.bias ? __ldg(a.bias + co) : 0.0f);
        if (a.res) v += __ldg(a.res + static_cast<int64_t>(m) * a.res_ld + co);
        a.y[static_cast<int64_t>(m) * a.y_ld + a.y_coff + co] = act_f32(v, a.act);
      }
    }
  }
}

// ------------------------------------------------------------------ pooling / GAP / copy
__global__ void pool_f32_kernel(int mode, const float* __restrict__ x, int N, int H, int W, int C, float* __restrict__ y,
                                int Ho, int Wo, int y_ld, int y_coff, int R, int S, int sh, int sw, int ph, int pw,
                                int count_include_pad) {
  const int64_t total = static_cast<int64_t>(N) * Ho * Wo * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    int64_t p = i / C;
    const int wo = static_cast<int>(p % Wo);
    p /= Wo;
    const int ho = static_cast<int>(p % Ho);
    const int n = static_cast<int>(p / Ho);
    float acc = mode == 0 ? -INFINITY : 0.0f;
    int cnt = 0;
    for (int r = 0; r < R; ++r) {
      const int hi = ho * sh - ph + r;
      if (hi < 0 || hi >= H) continue;
      for (int s = 0; s < S; ++s) {
        const int wi = wo * sw - pw + s;
        if (wi < 0 || wi >= W) continue;
        const float v = __ldg(x + ((static_cast<int64_t>(n) * H + hi) * W + wi) * C + c);
        acc = mode == 0 ? fmaxf(acc, v) : acc + v;
        ++cnt;
      }
    }
    if (mode == 1) {
      int div = cnt;
      if (count_include_pad) {
        const int h0 = ho * sh - ph, w0 = wo * sw - pw;
        div = (min(h0 + R, H + ph) - h0) * (min(w0 + S, W + pw) - w0);
      }
      acc /= static_cast<float>(div);
    }
    y[((static_cast<int64_t>(n) * Ho + ho) * Wo + wo) * y_ld + y_coff + c] = acc;
  }
}

// one thread per (sample, channel): pixels summed in order (fixed order, batch-independent)
__global__ void gap_f32_kernel(const float* __restrict__ x, int N, int HW, int C, float* __restrict__ y) {
  const int64_t total = static_cast<int64_t>(N) * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(i / C), c = static_cast<int>(i % C);
    const float* xp = x + static_cast<int64_t>(n) * HW * C + c;
    float s = 0.0f;
    for (int p = 0; p < HW; ++p) s += __ldg(xp + static_cast<int64_t>(p) * C);
    y[i] = s / static_cast<float>(HW);
  }
}

__global__ void copy_channels_f32_kernel(const float* __restrict__ x, int64_t pixels, int C, int x_ld, int x_coff,
                                         float* __restrict__ y, int y_ld, int y_coff) {
  const int64_t total = pixels * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = i / C;
    const int c = static_cast<int>(i - p * C);
    y[p * y_ld + y_coff + c] = __ldg(x + p * x_ld + x_coff + c);
  }
}

// ------------------------------------------------------------------ LayerNorm (warp per row)
__global__ void layernorm_f32_kernel(const float* __restrict__ x, int rows, int C, const float* __restrict__ g,
                                     const float* __restrict__ b, float eps, float* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const float* xr = x + static_cast<int64_t>(r) * C;
    float s = 0.0f;
    for (int c = lane; c < C; c += 32) s += xr[c];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    const float mean = s / C;
    float ss = 0.0f;
    for (int c = lane; c < C; c += 32) {
      const float d = xr[c] - mean;
      ss += d * d;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const float inv = 1.0f / sqrtf(ss / C + eps);
    float* yr = y + static_cast<int64_t>(r) * C;
    for (int c = lane; c < C; c += 32) yr[c] = (xr[c] - mean) * inv * __ldg(g + c) + __ldg(b + c);
  }
}

// ------------------------------------------------------------------ attention (CTA per head)
// qkv: [N, S, 3*hidden] rows [q | k | v], head h = columns [h*dh, (h+1)*dh) of each; out [N, S, hidden].
constexpr int kAttnF32Warps = 8;
__global__ void __launch_bounds__(kAttnF32Warps * 32)
    attention_f32_kernel(const float* __restrict__ qkv, int N, int S, int heads, int dh, float scale,
                         float* __restrict__ out) {
  extern __shared__ float sm[];
  const int hidden = heads * dh;
  const int ld = dh + 1;  // padded rows: lane-strided key reads hit distinct banks
  float* Ks = sm;
  float* Vs = Ks + static_cast<size_t>(S) * ld;
  float* P = Vs + static_cast<size_t>(S) * ld;  // [warps][S] probabilities
  float* Q = P + static_cast<size_t>(kAttnF32Warps) * S;  // [warps][dh]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int item = blockIdx.x; item < N * heads; item += gridDim.x) {
    const int n = item / heads, h = item - (item / heads) * heads;
    const float* base = qkv + static_cast<int64_t>(n) * S * 3 * hidden;
    __syncthreads();
    for (int i = threadIdx.x; i < S * dh; i += blockDim.x) {
      const int j = i / dh, d = i - (i / dh) * dh;
      Ks[j * ld + d] = base[static_cast<int64_t>(j) * 3 * hidden + hidden + h * dh + d];
      Vs[j * ld + d] = base[static_cast<int64_t>(j) * 3 * hidden + 2 * hidden + h * dh + d];
    }
    __syncthreads();
    float* p = P + warp * S;
    float* q = Q + warp * dh;
    for (int row = warp; row < S; row += kAttnF32Warps) {
      for (int d = lane; d < dh; d += 32) q[d] = base[static_cast<int64_t>(row) * 3 * hidden + h * dh + d];
      __syncwarp();
      float mx = -INFINITY;
      for (int j = lane; j < S; j += 32) {
        float sc = 0.0f;
        for (int d = 0; d < dh; ++d) sc = fmaf(q[d], Ks[j * ld + d], sc);
        sc *= scale;
        p[j] = sc;
        mx = fmaxf(mx, sc);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      float sum = 0.0f;
      for (int j = lane; j < S; j += 32) {
        const float e = expf(p[j] - mx);
        p[j] = e;
        sum += e;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
      __syncwarp();
      const float inv = 1.0f / sum;
      float* o = out + (static_cast<int64_t>(n) * S + row) * hidden + h * dh;
      for (int d = lane; d < dh; d += 32) {
        float acc = 0.0f;
        for (int j = 0; j < S; ++j) acc = fmaf(p[j], Vs[j * ld + d], acc);
        o[d] = acc * inv;
      }
      __syncwarp();
    }
  }
}

// ------------------------------------------------------------------ K1 gather into an fp32 batch
__global__ void gather_f32_kernel(RowPtrs src, int k, int64_t pixels, int c_src, int c_dst, float* __restrict__ dst) {
  const int64_t per_row = pixels * c_dst;
  const int64_t total = per_row * k;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / per_row);
    const int64_t e = i - r * per_row;
    const int64_t px = e / c_dst;
    const int c = static_cast<int>(e - px * c_dst);
    dst[i] = c < c_src ? load_any(src.p[r], src.dt[r], px * c_src + c) : 0.0f;
  }
}

// client image [Ho*f, Wo*f, c_src] -> [Ho, Wo, c_dst], channel (dy*f + dx)*c_src + c
__global__ void gather_s2d_f32_kernel(RowPtrs src, int k, int Ho, int Wo, int f, int c_src, int c_dst,
                                      float* __restrict__ dst) {
  const int64_t per_row = static_cast<int64_t>(Ho) * Wo * c_dst;
  const int64_t total = per_row * k;
  const int Wi = Wo * f;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / per_row);
    const int64_t e = i - r * per_row;
    const int64_t px = e / c_dst;
    const int cd = static_cast<int>(e - px * c_dst);
    float v = 0.0f;
    if (cd < f * f * c_src) {
      const int blk = cd / c_src, c = cd - blk * c_src;
      const int h = static_cast<int>(px / Wo) * f + blk / f;
      const int w = static_cast<int>(px % Wo) * f + blk % f;
      v = load_any(src.p[r], src.dt[r], (static_cast<int64_t>(h) * Wi + w) * c_src + c);
    }
    dst[i] = v;
  }
}

inline int grid_for(int64_t items, int threads, int cap) {
  int64_t g = (items + threads - 1) / threads;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}
}  // namespace

cudaError_t launch_conv_f32(const ConvF32Args& a, int grid, cudaStream_t s) {
  const int tiles = ((a.M + kTM - 1) / kTM) * ((a.Cout + kTN - 1) / kTN);
  conv_f32_kernel<<<grid_for(tiles, 1, grid), kF32Threads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pool_f32(int mode, const float* x, int N, int H, int W, int C, float* y, int Ho, int Wo, int y_ld,
                            int y_coff, int R, int S, int sh, int sw, int ph, int pw, int count_include_pad, int grid,
                            cudaStream_t s) {
  pool_f32_kernel<<<grid_for(static_cast<int64_t>(N) * Ho * Wo * C, 256, grid), 256, 0, s>>>(
      mode, x, N, H, W, C, y, Ho, Wo, y_ld, y_coff, R, S, sh, sw, ph, pw, count_include_pad);
  return cudaGetLastError();
}

cudaError_t launch_gap_f32(const float* x, int N, int HW, int C, float* y, int grid, cudaStream_t s) {
  gap_f32_kernel<<<grid_for(static_cast<int64_t>(N) * C, 128, grid), 128, 0, s>>>(x, N, HW, C, y);
  return cudaGetLastError();
}

cudaError_t launch_copy_channels_f32(const float* x, int64_t pixels, int C, int x_ld, int x_coff, float* y, int y_ld,
                                     int y_coff, int grid, cudaStream_t s) {
  copy_channels_f32_kernel<<<grid_for(pixels * C, 256, grid), 256, 0, s>>>(x, pixels, C, x_ld, x_coff, y, y_ld, y_coff);
  return cudaGetLastError();
}

cudaError_t launch_layernorm_f32(const float* x, int rows, int C, const float* gamma, const float* beta, float eps,
                                 float* y, int grid, cudaStream_t s) {
  layernorm_f32_kernel<<<grid_for(rows, 8, grid), 256, 0, s>>>(x, rows, C, gamma, beta, eps, y);
  return cudaGetLastError();
}

cudaError_t launch_attention_f32(const float* qkv, int N, int S, int heads, int dh, float* out, int grid,
                                 cudaStream_t s) {
  const size_t smem = (2 * static_cast<size_t>(S) * (dh + 1) + kAttnF32Warps * (static_cast<size_t>(S) + dh)) * 4;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  static bool configured = false;
  if (!configured) {
    const cudaError_t e =
        cudaFuncSetAttribute(attention_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  attention_f32_kernel<<<grid_for(static_cast<int64_t>(N) * heads, 1, grid), kAttnF32Warps * 32, smem, s>>>(
      qkv, N, S, heads, dh, 1.0f / sqrtf(static_cast<float>(dh)), out);
  return cudaGetLastError();
}

cudaError_t launch_gather_f32(int k, const void* const* src, const int32_t* src_dtype, int64_t pixels, int c_src,
                              int c_dst, float* dst, int grid, cudaStream_t s) {
  if (k > kMaxRows) return cudaErrorInvalidValue;
  RowPtrs rp;
  for (int i = 0; i < k; ++i) {
    rp.p[i] = src[i];
    rp.dt[i] = src_dtype[i];
  }
  gather_f32_kernel<<<grid_for(pixels * c_dst * k, 256, grid), 256, 0, s>>>(rp, k, pixels, c_src, c_dst, dst);
  return cudaGetLastError();
}

cudaError_t launch_gather_s2d_f32(int k, const void* const* src, const int32_t* src_dtype, int Ho, int Wo, int f,
                                  int c_src, int c_dst, float* dst, int grid, cudaStream_t s) {
  if (k > kMaxRows || f * f * c_src > c_dst) return cudaErrorInvalidValue;
  RowPtrs rp;
  for (int i = 0; i < k; ++i) {
    rp.p[i] = src[i];
    rp.dt[i] = src_dtype[i];
  }
  gather_s2d_f32_kernel<<<grid_for(static_cast<int64_t>(Ho) * Wo * c_dst * k, 256, grid), 256, 0, s>>>(
      rp, k, Ho, Wo, f, c_src, c_dst, dst);
  return cudaGetLastError();
}

}  // namespace gx
