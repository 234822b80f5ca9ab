// Unit chains (gx_model) and stage instances (gx_stage): workspace planning, CUDA-graph capture of
// a span per batch size k, and the gather -> span -> scatter dispatch that replaces
// _StageRT.latency_for (simulator.py:95-100).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "gx_internal.h"
#include "gx_runtime.h"
#include "gx_span.h"

using namespace gx;

namespace {

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Greedy liveness-based workspace assignment for the tensors a span touches.
int plan_workspace(gx_stage* st) {
  gx_model* m = st->m;
  const int nt = static_cast<int>(m->tensors.size());
  std::vector<int> first(nt, INT32_MAX), last(nt, -2);
  auto use = [&](int t, int pos) {
    if (t < 0) return;
    if (t >= nt) return;
    last[t] = std::max(last[t], pos);
  };
  auto def = [&](int t, int pos) {
    if (t < 0 || t >= nt) return;
    first[t] = std::min(first[t], pos);
    last[t] = std::max(last[t], pos);
  };
  def(st->in_tid, -1);
  const int n = static_cast<int>(st->ops.size());
  for (int i = 0; i < n; ++i) {
    const gx_op& op = m->ops[st->ops[i]];
    use(op.in, i);
    use(op.in2, i);
    def(op.out, i);
  }
  last[st->out_tid] = n;  // the span output lives until the scatter
  for (int i = 0; i < n; ++i) {
    const gx_op& op = m->ops[st->ops[i]];
    if ((op.in >= 0 && first[op.in] == INT32_MAX) || (op.in2 >= 0 && first[op.in2] == INT32_MAX))
      return fail(GX_EINVAL, "span reads a tensor no earlier op of the span produces");
  }
  struct Buf {
    size_t bytes;
    int free_at;  // position after which the buffer is free again
  };
  std::vector<Buf> bufs;
  std::vector<int> assign(nt, -1);
  for (int pos = -1; pos < n; ++pos) {
    for (int t = 0; t < nt; ++t) {
      if (first[t] != pos || assign[t] >= 0) continue;
      const size_t need =
          round_up(static_cast<size_t>(st->max_batch) * tensor_elems(m->tensors[t]) * elem_size(m->tensors[t].dtype), 256);
      int best = -1;
      for (int b = 0; b < static_cast<int>(bufs.size()); ++b)
        if (bufs[b].free_at < pos && bufs[b].bytes >= need && (best < 0 || bufs[b].bytes < bufs[best].bytes)) best = b;
      if (best < 0) {
        bufs.push_back({need, INT32_MAX});
        best = static_cast<int>(bufs.size()) - 1;
      }
      bufs[best].free_at = last[t];
      assign[t] = best;
    }
  }
  std::vector<size_t> off(bufs.size());
  size_t total = 0;
  for (size_t b = 0; b < bufs.size(); ++b) {
    off[b] = total;
    total += bufs[b].bytes;
  }
  GX_CUDA(cudaMalloc(&st->ws, std::max<size_t>(total, 256)));
  st->ws_bytes = total;
  st->tptr.assign(nt, nullptr);
  for (int t = 0; t < nt; ++t)
    if (assign[t] >= 0) st->tptr[t] = static_cast<uint8_t*>(st->ws) + off[assign[t]];
  return GX_OK;
}

int capture_span(gx_stage* st, int k, gx_stage::PerK* out) {
  gx_model* m = st->m;
  const uint8_t* wbase = static_cast<const uint8_t*>(m->wdev);
  // Plan every conv first so capture only records launches.
  std::vector<ConvLaunch> plans(st->ops.size());
  for (size_t i = 0; i < st->ops.size(); ++i) {
    const gx_op& op = m->ops[st->ops[i]];
    if (is_tc_op(op, m->tensors.data())) {
      int rc = plan_conv(op, m->tensors.data(), st->tptr.data(), wbase, k, st->sm_budget, &plans[i], 256,
                         m->op_wsw(st->ops[i]));
      if (rc != GX_OK) return rc;
    }
  }
  cudaGraph_t graph = nullptr;
  GX_CUDA(cudaStreamBeginCapture(st->stream, cudaStreamCaptureModeThreadLocal));
  int kernels = 0;
  int rc = GX_OK;
  const bool use_pdl = !dev().no_pdl;
  for (size_t i = 0; i < st->ops.size() && rc == GX_OK; ++i) {
    const gx_op& op = m->ops[st->ops[i]];
    const bool is_conv = is_tc_op(op, m->tensors.data());
    rc = launch_op(op, m->tensors.data(), st->tptr.data(), wbase, k, st->sm_budget, st->stream, use_pdl,
                   is_conv ? &plans[i] : nullptr, &kernels);
  }
  cudaError_t e = cudaStreamEndCapture(st->stream, &graph);
  if (rc != GX_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
  e = cudaGraphInstantiate(&out->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
  out->kernels = kernels;
  return GX_OK;
}

// Resolve the span's ops for batch k into the persistent kernel's device program: one SpanOp per
// op, three tensor maps (weights, activation, residual) per conv, BN capped at 128 so the smem
// ring, two residual slots and the bias vector fit next to each other.
int build_span_program(gx_stage* st, int k, gx_stage::PerK* out) {
  gx_model* m = st->m;
  const uint8_t* wbase = static_cast<const uint8_t*>(m->wdev);
  const gx_tensor* T = m->tensors.data();
  std::vector<SpanOp> ops(st->ops.size());
  // chunks of consecutive ops whose tensor maps fit one kernel parameter block
  std::vector<std::shared_ptr<SpanMaps>> chunk_maps(1, std::make_shared<SpanMaps>());
  std::vector<int> chunk_first(1, 0), chunk_used(1, 0);
  int bn_max = 16, has_res = 0, cout_max = 16;
  for (size_t i = 0; i < st->ops.size(); ++i) {
    const gx_op& op = m->ops[st->ops[i]];
    SpanOp& s = ops[i];
    memset(&s, 0, sizeof(s));
    s.kind = op.kind;
    const gx_tensor& ti = T[op.in];
    const gx_tensor& to = T[op.out];
    s.x = static_cast<const __nv_bfloat16*>(st->tptr[op.in]);
    s.y = st->tptr[op.out];
    s.N = k;
    s.H = ti.H;
    s.W = ti.W;
    s.C = ti.C;
    s.x_ld = ti.C;
    s.Ho = to.H;
    s.Wo = to.W;
    s.y_ld = to.C;
    s.y_coff = op.out_coff;
    s.y_f32 = to.dtype == GX_F32;
    s.act = op.act;
    switch (op.kind) {
      case GX_OP_CONV:
      case GX_OP_LINEAR: {
        ConvLaunch cl;
        int rc = plan_conv(op, T, st->tptr.data(), wbase, k, st->sm_budget, &cl, 256, nullptr, true);
        if (rc != GX_OK) return rc;
        const ConvArgs& a = cl.args;
        if (!a.tma_a) return fail(GX_EINVAL, "span kernel needs the TMA im2col path");
        const int need = a.res ? 3 : 2;
        if (chunk_used.back() + need > kMaxSpanMaps) {
          chunk_maps.push_back(std::make_shared<SpanMaps>());
          chunk_first.push_back(static_cast<int>(i));
          chunk_used.push_back(0);
        }
        SpanMaps& cm = *chunk_maps.back();
        int& used = chunk_used.back();
        s.tmap = used;
        cm.m[used++] = cl.wmap;
        cm.m[used++] = cl.amap;
        s.rmap = -1;
        if (a.res) {
          s.rmap = used;
          cm.m[used++] = cl.rmap;
        }
        s.BN = a.BN;
        s.n_tiles = a.n_tiles;
        s.num_tiles = a.num_tiles;
        s.num_kb = a.num_kb;
        s.Cin = a.Cin;
        s.cpl = a.cpl;
        s.a2d = a.a2d;
        s.HoWo = a.Ho * a.Wo;
        s.M = a.M;
        s.Cout = a.Cout;
        s.idesc = a.idesc;
        s.R = a.R;
        s.S = a.S;
        s.sh = a.sh;
        s.sw = a.sw;
        s.ph = a.ph;
        s.pw = a.pw;
        s.res = a.res;
        s.bias = a.bias;
        bn_max = std::max(bn_max, a.BN);
        cout_max = std::max(cout_max, a.Cout);
        has_res |= a.res != nullptr;
        break;
      }
      case GX_OP_MAXPOOL:
      case GX_OP_AVGPOOL:
        s.R = op.R;
        s.S = op.S;
        s.sh = op.sh;
        s.sw = op.sw;
        s.ph = op.ph;
        s.pw = op.pw;
        s.flags = op.flags;
        if (ti.C & 7) return fail(GX_EINVAL, "pool channels must be a multiple of 8");
        break;
      case GX_OP_GAP:
        break;
      case GX_OP_FC:
        s.K = static_cast<int>(tensor_elems(ti));
        s.Cout = op.Cout;
        s.w = reinterpret_cast<const __nv_bfloat16*>(wbase + op.w_off);
        s.bias = op.b_off >= 0 ? reinterpret_cast<const float*>(wbase + op.b_off) : nullptr;
        if (s.K & 7) return fail(GX_EINVAL, "FC input must be a multiple of 8");
        break;
      case GX_OP_COPY:
        s.pixels = static_cast<int64_t>(k) * ti.H * ti.W;
        s.C = op.Cin;
        s.x_coff = op.ph;
        break;
      default:
        return fail(GX_EINVAL, "op kind " + std::to_string(op.kind) + " not supported by the span kernel");
    }
  }
  SpanSmem L;
  L.bn_max = bn_max;
  L.bias_bytes = (cout_max * 4 + 15) & ~15;
  // residual slots: two (prefetch one tile ahead) unless that squeezes the ring below 3 stages
  for (int nres = has_res ? 2 : 0; nres >= (has_res ? 1 : 0); --nres) {
    L.has_res = nres;
    L.stages = 8;
    while (L.stages > 2 && span_smem_bytes(L) > 225 * 1024) --L.stages;
    if (L.stages >= 3) break;
  }
  if (span_smem_bytes(L) > 227 * 1024) return fail(GX_EINVAL, "span kernel shared memory does not fit");
  out->span_stages = L.stages;
  out->bn_max = L.bn_max;
  out->has_res = L.has_res;
  out->bias_bytes = L.bias_bytes;
  out->n_ops = static_cast<int>(ops.size());
  chunk_first.push_back(static_cast<int>(ops.size()));
  for (size_t c = 0; c + 1 < chunk_first.size(); ++c) {
    gx_stage::SpanChunk ch;
    ch.n_ops = chunk_first[c + 1] - chunk_first[c];
    ch.maps = chunk_maps[c];
    GX_CUDA(cudaMalloc(&ch.d_ops, std::max(1, ch.n_ops) * sizeof(SpanOp)));
    GX_CUDA(cudaMemcpy(ch.d_ops, ops.data() + chunk_first[c], ch.n_ops * sizeof(SpanOp), cudaMemcpyHostToDevice));
    out->chunks.push_back(ch);
  }
  out->kernels = static_cast<int>(out->chunks.size());
  return GX_OK;
}

// Conv / linear weights re-laid for the conv kernel's B operand: [kb][Cout][64] bf16 with the
// 128-byte swizzle already applied (16-byte chunk j of row n stored at chunk j ^ (n & 7)), so a
// BN x 64 tile of k-block kb is one contiguous BN*128-byte run that a plain bulk copy drops into
// shared memory exactly as a SWIZZLE_128B tensor-map load would (tiles start at multiples of 16
// rows).  One extra k-block of slack lets a partial last N tile over-read harmlessly.
cudaError_t build_bulk_weights(gx_model* m, const uint8_t* blob) {
  // (res_through_mma: see gx_runtime.h)
  const int n = static_cast<int>(m->ops.size());
  m->wsw_off.assign(n, -1);
  size_t total = 0;
  for (int i = 0; i < n; ++i) {
    const gx_op& op = m->ops[i];
    if (!is_tc_op(op, m->tensors.data())) continue;
    const int R = op.kind != GX_OP_CONV ? 1 : op.R, S = op.kind != GX_OP_CONV ? 1 : op.S;
    const size_t kpad = (static_cast<size_t>(R) * S * op.Cin + 63) / 64 * 64 +
                        ((op.flags & GX_OPF_DS) ? static_cast<size_t>(m->tensors[op.in2].C) : 0);
    m->wsw_off[i] = static_cast<int64_t>(total);
    total += (kpad + (res_through_mma(op) ? op.Cout : 0)) * op.Cout * 2;
  }
  if (total == 0) return cudaSuccess;
  total += 256 * 128;
  std::vector<uint8_t> h(total, 0);
  for (int i = 0; i < n; ++i) {
    if (m->wsw_off[i] < 0) continue;
    const gx_op& op = m->ops[i];
    const int R = op.kind != GX_OP_CONV ? 1 : op.R, S = op.kind != GX_OP_CONV ? 1 : op.S;
    const size_t kpad = (static_cast<size_t>(R) * S * op.Cin + 63) / 64 * 64 +
                        ((op.flags & GX_OPF_DS) ? static_cast<size_t>(m->tensors[op.in2].C) : 0);
    const size_t nkb = kpad / 64;
    const uint8_t* src = blob + op.w_off;  // [Cout][kpad] bf16
    uint8_t* dst = h.data() + m->wsw_off[i];
    for (size_t kb = 0; kb < nkb; ++kb)
      for (int row = 0; row < op.Cout; ++row)
        for (int j = 0; j < 8; ++j)
          std::memcpy(dst + ((kb * op.Cout + row) * 8 + (j ^ (row & 7))) * 16,
                      src + (static_cast<size_t>(row) * kpad + kb * 64 + j * 8) * 2, 16);
    if (res_through_mma(op)) {
      // identity k-blocks kb = nkb + c/64: B[row][c] = (row == c), so the residual tile fed as the
      // A operand of those k-blocks is added by the tensor core in fp32
      const uint16_t one = 0x3F80;  // bf16 1.0
      for (int row = 0; row < op.Cout; ++row) {
        const size_t kb = nkb + row / 64;
        const int c = row % 64, j = c / 8, e = c % 8;
        std::memcpy(dst + ((kb * op.Cout + row) * 8 + (j ^ (row & 7))) * 16 + e * 2, &one, 2);
      }
    }
  }
  cudaError_t e = cudaMalloc(&m->wsw, total);
  if (e == cudaSuccess) e = cudaMemcpy(m->wsw, h.data(), total, cudaMemcpyHostToDevice);
  return e;
}

}  // namespace

extern "C" {

int gx_model_create(gx_ctx* ctx, const char* model_id, int n_tensors, const gx_tensor* tensors, int n_ops,
                    const gx_op* ops, int n_units, const int32_t* unit_first_op, const int32_t* boundary,
                    const void* weight_blob, size_t blob_bytes, gx_model** out) {
  if (!ctx || !out || !tensors || !ops || !unit_first_op || !boundary) return fail(GX_EINVAL, "null arg");
  if (n_units < 1 || n_tensors < 1 || n_ops < 1) return fail(GX_EINVAL, "empty unit chain");
  if (int rc = bind_device(ctx->device)) return rc;
  if (unit_first_op[0] != 0 || unit_first_op[n_units] != n_ops) return fail(GX_EINVAL, "bad unit op ranges");
  for (int u = 0; u < n_units; ++u)
    if (unit_first_op[u + 1] < unit_first_op[u]) return fail(GX_EINVAL, "unit op ranges must be non-decreasing");
  for (int u = 0; u <= n_units; ++u)
    if (boundary[u] < 0 || boundary[u] >= n_tensors) return fail(GX_EINVAL, "bad boundary tensor id");
  for (int i = 0; i < n_ops; ++i) {
    const gx_op& op = ops[i];
    if (op.in < 0 || op.in >= n_tensors || op.out < 0 || op.out >= n_tensors || op.in2 >= n_tensors)
      return fail(GX_EINVAL, "op " + std::to_string(i) + " has a bad tensor id");
    if ((op.w_off >= 0 && static_cast<size_t>(op.w_off) >= blob_bytes) ||
        (op.b_off >= 0 && static_cast<size_t>(op.b_off) >= blob_bytes))
      return fail(GX_EINVAL, "op " + std::to_string(i) + " weight offset outside the blob");
  }
  // one compute element type per chain (the boundary-0 tensor's); only the chain output may differ
  // (fp32 logits of a bf16 chain)
  // (fp32 logits of a bf16 chain) and the int32 token ids a K8 embedding reads
  std::vector<char> ids_tensor(n_tensors, 0);
  int32_t mdt = -1;
  for (int i = 0; i < n_ops; ++i)
    if (ops[i].kind == GX_OP_EMBED) {
      ids_tensor[ops[i].in] = 1;
      if (ops[i].in == boundary[0]) mdt = tensors[ops[i].out].dtype;
      if ((ops[i].w2_off >= 0 && static_cast<size_t>(ops[i].w2_off) >= blob_bytes) ||
          (ops[i].w3_off >= 0 && static_cast<size_t>(ops[i].w3_off) >= blob_bytes) || ops[i].w_off < 0 ||
          ops[i].w2_off < 0 || ops[i].w3_off < 0 || ops[i].b_off < 0 || ops[i].Cin < 1 || ops[i].R < 1)
        return fail(GX_EINVAL, "op " + std::to_string(i) + ": embed needs word/pos/type tables, LayerNorm "
                               "parameters, the vocabulary size (Cin) and max positions (R)");
    }
  if (mdt < 0) mdt = tensors[boundary[0]].dtype;
  if (mdt != GX_BF16 && mdt != GX_F32) return fail(GX_EINVAL, "tensor dtype must be GX_BF16 or GX_F32");
  for (int t = 0; t < n_tensors; ++t) {
    if (ids_tensor[t]) {
      if (tensors[t].dtype != GX_I32) return fail(GX_EINVAL, "embed input must be GX_I32 token ids");
      continue;
    }
    if (tensors[t].dtype != mdt && !(t == boundary[n_units] && tensors[t].dtype == GX_F32))
      return fail(GX_EINVAL, "tensor " + std::to_string(t) + " mixes element types within one chain");
  }
  GX_CUDA(cudaSetDevice(ctx->device));
  gx_model* m = new gx_model();
  m->dtype = mdt;
  m->ctx = ctx;
  m->id = model_id ? model_id : "";
  m->tensors.assign(tensors, tensors + n_tensors);
  m->ops.assign(ops, ops + n_ops);
  m->unit_first_op.assign(unit_first_op, unit_first_op + n_units + 1);
  m->boundary.assign(boundary, boundary + n_units + 1);
  m->wbytes = blob_bytes;
  cudaError_t e = cudaMalloc(&m->wdev, std::max<size_t>(blob_bytes, 256));
  if (e == cudaSuccess && blob_bytes) e = cudaMemcpy(m->wdev, weight_blob, blob_bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = build_bulk_weights(m, static_cast<const uint8_t*>(weight_blob));
  if (e != cudaSuccess) {
    if (m->wdev) cudaFree(m->wdev);
    if (m->wsw) cudaFree(m->wsw);
    delete m;
    return cuda_fail(e, "weight upload");
  }
  *out = m;
  return GX_OK;
}

int gx_model_destroy(gx_model* m) {
  if (!m) return GX_OK;
  cudaSetDevice(m->ctx->device);
  if (m->wdev) cudaFree(m->wdev);
  if (m->wsw) cudaFree(m->wsw);
  delete m;
  return GX_OK;
}

int gx_model_dtype(gx_model* m, int32_t* dtype_out) {
  if (!m || !dtype_out) return fail(GX_EINVAL, "null arg");
  *dtype_out = m->dtype;
  return GX_OK;
}

int gx_model_tensor_elems(gx_model* m, int tid, int64_t* out) {
  if (!m || !out || tid < 0 || tid >= static_cast<int>(m->tensors.size())) return fail(GX_EINVAL, "bad tensor id");
  *out = tensor_elems(m->tensors[tid]);
  return GX_OK;
}

int gx_stage_create(gx_model* m, int start, int end, int max_batch, int sm_budget, int32_t dtype, void* stream,
                    gx_stage** out) {
  if (!m || !out) return fail(GX_EINVAL, "null arg");
  if (dtype != m->dtype)
    return fail(GX_EINVAL, std::string("stage dtype ") + (dtype == GX_F32 ? "fp32" : dtype == GX_BF16 ? "bf16" : "?") +
                               " does not match model " + m->id + "'s " + (m->dtype == GX_F32 ? "fp32" : "bf16"));
  if (!(0 <= start && start < end && end <= m->n_units()))
    return fail(GX_EINVAL, "bad span [" + std::to_string(start) + ", " + std::to_string(end) + ") for model " + m->id);
  if (max_batch < 1 || max_batch > 64) return fail(GX_EINVAL, "max_batch must be in 1..64");
  if (int rc = bind_device(m->ctx->device)) return rc;
  if (sm_budget < 1 || sm_budget > m->ctx->sm_count)
    return fail(GX_EINFEASIBLE, "SM budget " + std::to_string(sm_budget) + " outside 1.." +
                                    std::to_string(m->ctx->sm_count));
  GX_CUDA(cudaSetDevice(m->ctx->device));
  gx_stage* st = new gx_stage();
  st->m = m;
  st->start = start;
  st->end = end;
  st->max_batch = max_batch;
  st->sm_budget = sm_budget;
  for (int i = m->unit_first_op[start]; i < m->unit_first_op[end]; ++i) st->ops.push_back(i);
  st->in_tid = m->boundary[start];
  st->out_tid = m->boundary[end];
  int rc = plan_workspace(st);
  if (rc != GX_OK) {
    delete st;
    return rc;
  }
  if (stream) {
    st->stream = static_cast<cudaStream_t>(stream);
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      cudaFree(st->ws);
      delete st;
      return cuda_fail(e, "cudaStreamCreate");
    }
    st->own_stream = true;
  }
  // default: per-op persistent kernels in a CUDA graph with PDL (measured faster at the serving
  // operating point); gx_stage_set_exec(GX_EXEC_SPAN) selects the single-launch span kernel
  st->span_mode = false;
  cudaError_t e = cudaMalloc(&st->bar, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(st->bar, 0, sizeof(unsigned long long));
  if (e != cudaSuccess) {
    gx_stage_destroy(st);
    return cuda_fail(e, "grid barrier counter");
  }
  *out = st;
  return GX_OK;
}

int gx_stage_destroy(gx_stage* st) {
  if (!st) return GX_OK;
  cudaSetDevice(st->m->ctx->device);
  cudaStreamSynchronize(st->stream);
  for (auto& kv : st->graphs) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    for (auto& ch : kv.second.chunks)
      if (ch.d_ops) cudaFree(ch.d_ops);
  }
  if (st->bar) cudaFree(st->bar);
  if (st->ws) cudaFree(st->ws);
  if (st->prof_src) cudaFree(st->prof_src);
  if (st->prof_dst) cudaFree(st->prof_dst);
  if (st->own_stream) cudaStreamDestroy(st->stream);
  delete st;
  return GX_OK;
}

int gx_stage_set_exec(gx_stage* st, int32_t mode) {
  if (!st) return fail(GX_EINVAL, "null arg");
  if (mode != GX_EXEC_GRAPH && mode != GX_EXEC_SPAN) return fail(GX_EINVAL, "unknown execution mode");
  if (mode == GX_EXEC_SPAN && st->m->dtype != GX_BF16) return fail(GX_EINVAL, "the span kernel is bf16-only");
  const bool span = mode == GX_EXEC_SPAN;
  if (span != st->span_mode) {
    if (int rc = bind_device(st->m->ctx->device)) return rc;
    GX_CUDA(cudaStreamSynchronize(st->stream));
    for (auto& kv : st->graphs) {  // programs of the other mode are rebuilt on demand
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      for (auto& ch : kv.second.chunks)
        if (ch.d_ops) cudaFree(ch.d_ops);
    }
    st->graphs.clear();
    st->span_mode = span;
  }
  return GX_OK;
}

int gx_stage_stream(gx_stage* st, void** stream_out) {
  if (!st || !stream_out) return fail(GX_EINVAL, "null arg");
  *stream_out = st->stream;
  return GX_OK;
}

static int stage_graph(gx_stage* st, int k, gx_stage::PerK** out) {
  auto it = st->graphs.find(k);
  if (it == st->graphs.end()) {
    gx_stage::PerK pk;
    int rc = st->span_mode ? build_span_program(st, k, &pk) : capture_span(st, k, &pk);
    if (rc != GX_OK) return rc;
    it = st->graphs.emplace(k, pk).first;
  }
  *out = &it->second;
  return GX_OK;
}

int gx_stage_run(gx_stage* st, int k, const void* const* src, const int32_t* src_dtype, int32_t src_channels,
                 void* const* dst, int32_t dst_dtype) {
  if (!st || !src || !src_dtype || !dst) return fail(GX_EINVAL, "null arg");
  if (k < 1 || k > st->max_batch) return fail(GX_EINVAL, "batch k outside 1..max_batch");
  if (int rc = bind_device(st->m->ctx->device)) return rc;
  return gx::stage_run_on(st, st->stream, k, src, src_dtype, src_channels, dst, dst_dtype);
}

int gx_stage_run_async(gx_stage* st, void* stream, int k, const void* const* src, const int32_t* src_dtype,
                       int32_t src_channels, void* const* dst, int32_t dst_dtype, void* done_event) {
  if (!st || !src || !src_dtype || !dst) return fail(GX_EINVAL, "null arg");
  if (k < 1 || k > st->max_batch) return fail(GX_EINVAL, "batch k outside 1..max_batch");
  if (int rc = bind_device(st->m->ctx->device)) return rc;
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : st->stream;
  if (int rc = gx::stage_run_on(st, s, k, src, src_dtype, src_channels, dst, dst_dtype)) return rc;
  if (done_event) GX_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(done_event), s));
  return GX_OK;
}

int gx_stage_run_top1(gx_stage* st, void* stream, int k, const void* const* src, const int32_t* src_dtype,
                      int32_t src_channels, void* const* dst, int32_t* const* top1, void* done_event) {
  if (!st || !src || !src_dtype || !top1) return fail(GX_EINVAL, "null arg");
  if (k < 1 || k > st->max_batch) return fail(GX_EINVAL, "batch k outside 1..max_batch");
  if (int rc = bind_device(st->m->ctx->device)) return rc;
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : st->stream;
  if (int rc = gx::stage_run_on(st, s, k, src, src_dtype, src_channels, dst, GX_F32, top1)) return rc;
  if (done_event) GX_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(done_event), s));
  return GX_OK;
}

}  // extern "C"

namespace gx {
// The body of gx_stage_run on an explicit stream: the serving loop runs batches of any instance on
// a pooled stream (an instance never has two batches in flight, so its workspace is never shared).
int stage_run_on(gx_stage* st, cudaStream_t stream, int k, const void* const* src, const int32_t* src_dtype,
                 int32_t src_channels, void* const* dst, int32_t dst_dtype, int32_t* const* top1) {
  gx_model* m = st->m;
  if (k < 1 || k > st->max_batch) return fail(GX_EINVAL, "batch k outside 1..max_batch");
  const gx_tensor& tin = m->tensors[st->in_tid];
  const gx_tensor& tout = m->tensors[st->out_tid];
  const int c_src = src_channels > 0 ? src_channels : tin.C;
  if (c_src > tin.C) return fail(GX_EINVAL, "source has more channels than the boundary tensor");
  if (top1 && (tout.dtype != GX_F32 || (dst && dst_dtype != GX_F32)))
    return fail(GX_EINVAL, "top-1 needs the fp32 chain output (logits)");
  for (int i = 0; i < k; ++i) {
    const void* d = dst ? dst[i] : nullptr;
    if (!src[i] || (!d && !top1) || ((reinterpret_cast<uintptr_t>(src[i]) | reinterpret_cast<uintptr_t>(d)) & 15u))
      return fail(GX_EINVAL, "batch row " + std::to_string(i) + ": null or not 16-byte aligned source/destination");
    if (top1 && !top1[i]) return fail(GX_EINVAL, "batch row " + std::to_string(i) + ": null top-1 destination");
  }
  gx_stage::PerK* pk = nullptr;
  int rc = stage_graph(st, k, &pk);
  if (rc != GX_OK) return rc;
  const int bw_grid = st->sm_budget * 8;
  if (tin.s2d > 1 && src_channels <= 0)
    return fail(GX_EINVAL, "space-to-depth boundary needs the client's channel count");
  if (tin.dtype == GX_I32) {  // token ids (K8 embedding input): a plain 4-byte word gather
    for (int i = 0; i < k; ++i)
      if (src_dtype[i] != GX_I32) return fail(GX_EINVAL, "a token-id boundary takes GX_I32 sources");
    GX_CUDA(launch_gather_words(k, src, tensor_elems(tin), static_cast<uint32_t*>(st->tptr[st->in_tid]), bw_grid,
                                stream));
  } else if (tin.dtype == GX_F32) {  // fp32 chain: the batch is assembled in fp32
    float* bt = static_cast<float*>(st->tptr[st->in_tid]);
    if (tin.s2d > 1)
      GX_CUDA(launch_gather_s2d_f32(k, src, src_dtype, tin.H, tin.W, tin.s2d, src_channels, tin.C, bt, bw_grid,
                                    stream));
    else
      GX_CUDA(launch_gather_f32(k, src, src_dtype, static_cast<int64_t>(tin.H) * tin.W, c_src, tin.C, bt, bw_grid,
                                stream));
  } else if (tin.s2d > 1) {
    GX_CUDA(launch_gather_s2d(k, src, src_dtype, tin.H, tin.W, tin.s2d, src_channels, tin.C,
                              static_cast<__nv_bfloat16*>(st->tptr[st->in_tid]), bw_grid, stream));
  } else {
    GX_CUDA(launch_gather(k, src, src_dtype, static_cast<int64_t>(tin.H) * tin.W, c_src, tin.C,
                          static_cast<__nv_bfloat16*>(st->tptr[st->in_tid]), bw_grid, stream));
  }
  if (st->span_mode) {
    SpanSmem L;
    L.stages = pk->span_stages;
    L.bn_max = pk->bn_max;
    L.has_res = pk->has_res;
    L.bias_bytes = pk->bias_bytes;
    for (const auto& ch : pk->chunks) {
      GX_CUDA(launch_span(static_cast<const SpanOp*>(ch.d_ops), ch.n_ops, *ch.maps, st->bar, st->arrivals, L,
                          st->sm_budget, stream));
      st->arrivals += static_cast<unsigned long long>(ch.n_ops) * st->sm_budget;
    }
  } else {
    GX_CUDA(cudaGraphLaunch(pk->exec, stream));
  }
  if (top1)
    GX_CUDA(launch_scatter_top1(k, static_cast<const float*>(st->tptr[st->out_tid]), tensor_elems(tout), dst, top1,
                                stream));
  else
    GX_CUDA(launch_scatter(k, st->tptr[st->out_tid], tout.dtype, tensor_elems(tout), dst, dst_dtype, bw_grid,
                           stream));
  return GX_OK;
}
}  // namespace gx

extern "C" {

int gx_stage_span_trace(gx_stage* st, int k, int64_t* out, int64_t cap, int* n_ops_out) {
  if (!st || !out || !n_ops_out) return fail(GX_EINVAL, "null arg");
  if (!st->span_mode) return fail(GX_EINVAL, "stage is not in span mode");
  if (k < 1 || k > st->max_batch) return fail(GX_EINVAL, "bad k");
  if (int rc = bind_device(st->m->ctx->device)) return rc;
  gx_stage::PerK* pk = nullptr;
  int rc = stage_graph(st, k, &pk);
  if (rc != GX_OK) return rc;
  const int64_t n = static_cast<int64_t>(st->sm_budget) * pk->n_ops * 4;
  if (cap < n) return fail(GX_EINVAL, "trace buffer too small");
  unsigned long long* d = nullptr;
  GX_CUDA(cudaMalloc(&d, n * sizeof(unsigned long long)));
  GX_CUDA(cudaMemset(d, 0, n * sizeof(unsigned long long)));
  SpanSmem L;
  L.stages = pk->span_stages;
  L.bn_max = pk->bn_max;
  L.has_res = pk->has_res;
  L.bias_bytes = pk->bias_bytes;
  if (pk->chunks.size() != 1) return fail(GX_EINVAL, "trace supports single-chunk spans");
  const gx_stage::SpanChunk& ch = pk->chunks[0];
  GX_CUDA(launch_span(static_cast<const SpanOp*>(ch.d_ops), ch.n_ops, *ch.maps, st->bar, st->arrivals, L,
                      st->sm_budget, st->stream, d));
  st->arrivals += static_cast<unsigned long long>(ch.n_ops) * st->sm_budget;
  GX_CUDA(cudaStreamSynchronize(st->stream));
  GX_CUDA(cudaMemcpy(out, d, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  cudaFree(d);
  *n_ops_out = pk->n_ops;
  return GX_OK;
}

int gx_stage_kernel_count(gx_stage* st, int k, int* out) {
  if (!st || !out) return fail(GX_EINVAL, "null arg");
  if (int rc = bind_device(st->m->ctx->device)) return rc;
  gx_stage::PerK* pk = nullptr;
  int rc = stage_graph(st, k, &pk);
  if (rc != GX_OK) return rc;
  *out = pk->kernels + 2;
  return GX_OK;
}

int gx_stage_profile(gx_stage* st, int k, int iters, float* ms_out) {
  if (!st || !ms_out) return fail(GX_EINVAL, "null arg");
  if (k < 1 || k > st->max_batch || iters < 1) return fail(GX_EINVAL, "bad profile arguments");
  if (int rc = bind_device(st->m->ctx->device)) return rc;
  gx_model* m = st->m;
  const gx_tensor& tin = m->tensors[st->in_tid];
  const gx_tensor& tout = m->tensors[st->out_tid];
  const size_t in_bytes = static_cast<size_t>(tensor_elems(tin)) * 4;
  const size_t out_bytes = static_cast<size_t>(tensor_elems(tout)) * 4;
  GX_CUDA(cudaSetDevice(m->ctx->device));
  if (!st->prof_src) {
    GX_CUDA(cudaMalloc(&st->prof_src, in_bytes * st->max_batch));
    GX_CUDA(cudaMemset(st->prof_src, 0, in_bytes * st->max_batch));
    GX_CUDA(cudaMalloc(&st->prof_dst, out_bytes * st->max_batch));
  }
  std::vector<const void*> src(k);
  std::vector<int32_t> dt(k, tin.dtype == GX_I32 ? GX_I32 : GX_F32);
  std::vector<void*> dst(k);
  for (int i = 0; i < k; ++i) {
    src[i] = static_cast<uint8_t*>(st->prof_src) + i * in_bytes;
    dst[i] = static_cast<uint8_t*>(st->prof_dst) + i * out_bytes;
  }
  const int32_t dst_dtype = st->end == m->n_units() ? GX_F32 : GX_BF16;
  // a space-to-depth boundary takes the client image (same byte count, C / s2d^2 channels)
  const int c_src = tin.s2d > 1 ? tin.C / (tin.s2d * tin.s2d) : tin.C;
  // warm-up (also captures the graph)
  for (int w = 0; w < 3; ++w) {
    int rc = gx_stage_run(st, k, src.data(), dt.data(), c_src, dst.data(), dst_dtype);
    if (rc != GX_OK) return rc;
  }
  cudaEvent_t e0, e1;
  GX_CUDA(cudaEventCreate(&e0));
  GX_CUDA(cudaEventCreate(&e1));
  std::vector<float> t(iters);
  for (int i = 0; i < iters; ++i) {
    GX_CUDA(cudaEventRecord(e0, st->stream));
    int rc = gx_stage_run(st, k, src.data(), dt.data(), c_src, dst.data(), dst_dtype);
    if (rc != GX_OK) return rc;
    GX_CUDA(cudaEventRecord(e1, st->stream));
    GX_CUDA(cudaEventSynchronize(e1));
    GX_CUDA(cudaEventElapsedTime(&t[i], e0, e1));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  std::sort(t.begin(), t.end());
  *ms_out = t[iters / 2];
  return GX_OK;
}

int gx_stage_op_count(gx_stage* st, int* out) {
  if (!st || !out) return fail(GX_EINVAL, "null arg");
  *out = static_cast<int>(st->ops.size());
  return GX_OK;
}

int gx_stage_profile_ops(gx_stage* st, int k, int iters, int cap, float* ms, double* flops, double* bytes,
                         int32_t* kind) {
  if (!st || !ms || !flops || !bytes || !kind) return fail(GX_EINVAL, "null arg");
  if (k < 1 || k > st->max_batch || iters < 1) return fail(GX_EINVAL, "bad profile arguments");
  if (cap < static_cast<int>(st->ops.size())) return fail(GX_EINVAL, "output arrays smaller than the span");
  float whole = 0.0f;
  // one full batch first: captures the graph and leaves real activations in every workspace tensor
  if (int rc = gx_stage_profile(st, k, 3, &whole)) return rc;
  gx_model* m = st->m;
  const gx_tensor* T = m->tensors.data();
  const uint8_t* wbase = static_cast<const uint8_t*>(m->wdev);
  cudaEvent_t e0, e1;
  GX_CUDA(cudaEventCreate(&e0));
  GX_CUDA(cudaEventCreate(&e1));
  std::vector<float> t(iters);
  for (size_t i = 0; i < st->ops.size(); ++i) {
    const gx_op& op = m->ops[st->ops[i]];
    ConvLaunch cl;
    const bool is_conv = is_tc_op(op, T);
    if (is_conv) {
      if (int rc = plan_conv(op, T, st->tptr.data(), wbase, k, st->sm_budget, &cl, 256, m->op_wsw(st->ops[i])))
        return rc;
    }
    for (int w = 0; w < 2; ++w)
      if (int rc = launch_op(op, T, st->tptr.data(), wbase, k, st->sm_budget, st->stream, false,
                             is_conv ? &cl : nullptr, nullptr))
        return rc;
    for (int it = 0; it < iters; ++it) {
      GX_CUDA(cudaEventRecord(e0, st->stream));
      if (int rc = launch_op(op, T, st->tptr.data(), wbase, k, st->sm_budget, st->stream, false,
                             is_conv ? &cl : nullptr, nullptr))
        return rc;
      GX_CUDA(cudaEventRecord(e1, st->stream));
      GX_CUDA(cudaEventSynchronize(e1));
      GX_CUDA(cudaEventElapsedTime(&t[it], e0, e1));
    }
    std::sort(t.begin(), t.end());
    ms[i] = t[iters / 2];
    op_work(op, T, k, &flops[i], &bytes[i]);
    kind[i] = op.kind;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return GX_OK;
}

}  // extern "C"
