// Runtime objects behind the opaque C handles.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "gx_internal.h"

struct gx_ctx {
  int device = 0;
  int sm_count = 0;
};

namespace gx {
struct SpanMaps;
struct ConvLaunch {
  CUtensorMap wmap;
  CUtensorMap amap;  // im2col map of the input (args.tma_a)
  CUtensorMap rmap;  // residual tile map (args.res)
  CUtensorMap ymap;  // output tile map (args.ystore)
  ConvArgs args;
  int grid;
};

int elem_size(int dtype);
int64_t tensor_elems(const gx_tensor& t);
// wsw: the op's weights pre-tiled and pre-swizzled for bulk copies ([kb][Cout][64] bf16, 128B
// swizzle), or null to load them with a tiled TMA from the [Cout][Kpad] blob.
// for_span: plan for the persistent span kernel (span_kernel.cu), which loads 128-row residual
// boxes and stores outputs itself: no per-warp epilogue I/O.
int plan_conv(const gx_op& op, const gx_tensor* T, void* const* ptrs, const uint8_t* wbase, int k, int sm_budget,
              ConvLaunch* out, int bn_cap = 256, const uint8_t* wsw = nullptr, bool for_span = false);
int launch_op(const gx_op& op, const gx_tensor* T, void* const* ptrs, const uint8_t* wbase, int k, int sm_budget,
              cudaStream_t s, bool pdl, const ConvLaunch* pre, int* kernels);
unsigned long long* debug_trace_buffer();
// 1x1 / stride-1 / unpadded convs with a residual: the residual is added by the tensor core through
// identity k-blocks appended to the op's pre-swizzled weights (the epilogue then has no residual
// traffic), when the op's planning confirms the 2D A path (plan_conv).
inline bool res_through_mma(const gx_op& op) {
  return op.kind == GX_OP_CONV && op.in2 >= 0 && !(op.flags & GX_OPF_DS) && op.R == 1 && op.S == 1 && op.sh == 1 &&
         op.sw == 1 && op.ph == 0 && op.pw == 0 && op.Cout % 64 == 0 && op.Cin % 64 == 0;
}
// FC (GX_OP_FC) on the tcgen05 GEMM path: the flattened per-sample input is a [k, K] row-major A
// operand (1x1 conv on a 1x1 image with Cin = K), the [Cout][K] weights the B operand.  Needs whole
// 64-wide k-blocks and 8-aligned outputs; GX_FC_SIMT keeps the CUDA-core weight-streaming kernel.
// The choice must not depend on the batch or the SM budget: a request's bits may not depend on
// which instance serves it (split-vs-whole bit-exactness, test_models_gpu.py), and the two paths
// sum K in different orders.  (The CUDA-core kernel is faster only for batch-1 heads spread over
// a whole GPU, which serving never runs.)
inline bool fc_on_tc(const gx_op& op) {
  return op.kind == GX_OP_FC && op.Cin % 64 == 0 && op.Cout % 8 == 0 && op.b_off >= 0 && !gx::dev().fc_simt &&
         !(op.flags & GX_OPF_FC_SIMT);
}
// ops executed by conv_tc_kernel / conv_halo_kernel (planned with plan_conv)
inline bool is_gemm_op(const gx_op& op) { return op.kind == GX_OP_CONV || op.kind == GX_OP_LINEAR || fc_on_tc(op); }
// ... in a bf16 chain (fp32 chains run every op on the fp32 kernels, kernels_f32.cu)
inline bool is_tc_op(const gx_op& op, const gx_tensor* T) { return is_gemm_op(op) && T[op.in].dtype == GX_BF16; }
int launch_op_f32(const gx_op& op, const gx_tensor* T, void* const* ptrs, const uint8_t* wbase, int k, int sm_budget,
                  cudaStream_t s);
void op_work(const gx_op& op, const gx_tensor* T, int k, double* flops, double* bytes);
}  // namespace gx

struct gx_model {
  gx_ctx* ctx = nullptr;
  std::string id;
  std::vector<gx_tensor> tensors;
  std::vector<gx_op> ops;
  std::vector<int32_t> unit_first_op;  // n_units + 1
  std::vector<int32_t> boundary;       // n_units + 1
  int32_t dtype = GX_BF16;             // compute element type (gx_model_dtype)
  void* wdev = nullptr;
  size_t wbytes = 0;
  void* wsw = nullptr;                // conv/linear weights re-laid for bulk copies (see plan_conv)
  std::vector<int64_t> wsw_off;       // per op: byte offset into wsw, -1 if none
  const uint8_t* op_wsw(int op) const {
    return wsw && wsw_off[op] >= 0 ? static_cast<const uint8_t*>(wsw) + wsw_off[op] : nullptr;
  }
  int n_units() const { return static_cast<int>(boundary.size()) - 1; }
};

struct gx_stage {
  gx_model* m = nullptr;
  int start = 0, end = 0, max_batch = 0, sm_budget = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::vector<int> ops;         // op indices of the span, in order
  std::vector<void*> tptr;      // device pointer per tensor id (workspace), nullptr if unused
  void* ws = nullptr;
  size_t ws_bytes = 0;
  int in_tid = -1, out_tid = -1;
  struct SpanChunk {
    void* d_ops = nullptr;  // SpanOp[n_ops] (device)
    int n_ops = 0;
    std::shared_ptr<gx::SpanMaps> maps;  // tensor maps, passed by value as a kernel parameter
  };
  struct PerK {
    cudaGraphExec_t exec = nullptr;
    int kernels = 0;
    // persistent span program (span_kernel.cu): consecutive launches, one per chunk
    std::vector<SpanChunk> chunks;
    int n_ops = 0;
    int span_stages = 0, bn_max = 0, has_res = 0, bias_bytes = 0;
  };
  std::map<int, PerK> graphs;
  bool span_mode = true;                 // one persistent launch per batch (else per-op CUDA graph)
  unsigned long long* bar = nullptr;     // grid-barrier arrival counter (device)
  unsigned long long arrivals = 0;       // barrier arrivals so far (base of the next launch)
  // profiling scratch
  void* prof_src = nullptr;
  void* prof_dst = nullptr;
};

namespace gx {
// gx_stage_run on an explicit stream (gx_stage.cu); used by the serving loop's stream pool.
// top1 (optional): per-row int32 destinations of the output's argmax (K9, fp32 chain outputs
// only); dst may then be null (top-1 only, no logits written).
int stage_run_on(gx_stage* st, cudaStream_t stream, int k, const void* const* src, const int32_t* src_dtype,
                 int32_t src_channels, void* const* dst, int32_t dst_dtype, int32_t* const* top1 = nullptr);
}  // namespace gx
