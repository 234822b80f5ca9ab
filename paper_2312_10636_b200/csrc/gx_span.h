// Device-side op program of the persistent span kernel (span_kernel.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace gx {

// One op of a span, resolved for a fixed stage (buffers) and batch size k.  Conv/linear fields
// mirror ConvArgs; the bandwidth ops reuse the shape fields.  Lives in device memory.
struct alignas(16) SpanOp {
  int kind;
  int tmap;  // conv: index of the weight map in SpanMaps; the activation map is tmap+1
  int rmap;  // conv with residual: index of the residual map, else -1
  // conv / linear
  int BN, n_tiles, num_tiles, num_kb, Cin, cpl, a2d, HoWo, M, Cout, act, y_ld, y_coff, y_f32;
  uint32_t idesc;
  // shared shape fields (conv: filter R,S / strides / pads / output Wo; pool: window)
  int N, H, W, C, x_ld, Ho, Wo, R, S, sh, sw, ph, pw, flags, K, x_coff;
  int64_t pixels;
  const __nv_bfloat16* x;
  const __nv_bfloat16* res;  // conv residual (null if none)
  const __nv_bfloat16* w;    // FC weights
  const float* bias;
  void* y;
};

struct SpanSmem {
  int stages;
  int bn_max;
  int has_res;
  int bias_bytes;
};

// Tensor maps travel as a __grid_constant__ kernel parameter: TMA through param-space descriptors
// is ~1.5x faster than through descriptors in global memory (measured, scripts/bench_conv.py).
constexpr int kMaxSpanMaps = 236;  // 236 x 128 B + the other params stay under the 32 KB limit
struct SpanMaps {
  CUtensorMap m[kMaxSpanMaps];
};

size_t span_smem_bytes(const SpanSmem& L);
cudaError_t launch_span(const SpanOp* ops, int n_ops, const SpanMaps& maps, unsigned long long* bar,
                        unsigned long long bar_base, const SpanSmem& L, int grid, cudaStream_t s,
                        unsigned long long* trace = nullptr);

}  // namespace gx
