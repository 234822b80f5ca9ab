// libgx C ABI: contexts, unit chains (models), stage instances, and the debug op entry.
// See include/graft_exec.h for the mapping onto the reference's interfaces.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "gx_internal.h"
#include "gx_ptx.cuh"
#include "gx_runtime.h"

namespace gx {

static thread_local std::string g_last_error;
static thread_local std::string g_last_encode;  // detail of the last failed tensor-map encode

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int bind_device(int device) {
  static thread_local bool bound = false;
  int cur = -1;
  if (!bound || cudaGetDevice(&cur) != cudaSuccess || cur != device) {
    const cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    bound = true;
  }
  return GX_OK;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return GX_ECUDA;
}

// Development switches: read from the environment only in builds compiled with -DGX_DEV_KNOBS
// (scripts/ experiments); the shipped library always takes the defaults.
const DevKnobs& dev() {
  static const DevKnobs knobs = [] {
    DevKnobs d;
#ifdef GX_DEV_KNOBS
    auto flag = [](const char* n) { return getenv(n) != nullptr; };
    auto num = [](const char* n, int def) {
      const char* v = getenv(n);
      return v ? atoi(v) : def;
    };
    d.no_halo = flag("GX_NO_HALO");
    d.no_halo32 = flag("GX_NO_HALO32");
    d.no_wbulk = flag("GX_NO_WBULK");
    d.no_ystore = flag("GX_NO_YSTORE");
    d.gmaps = flag("GX_GMAPS");
    d.no_res_mma = flag("GX_NO_RES_MMA");
    d.no_tma_im2col = flag("GX_NO_TMA_IM2COL");
    d.no_a2d = flag("GX_NO_A2D");
    d.no_wres = flag("GX_NO_WRES");
    d.no_wstore = flag("GX_NO_WSTORE");
    d.fc_simt = flag("GX_FC_SIMT");
    d.no_pdl = flag("GX_NO_PDL");
    d.pool_nostrip = flag("GX_POOL_NOSTRIP");
    d.no_bres = flag("GX_NO_BRES");
    d.conv_dbg = num("GX_CONV_DBG", 0);
    d.bn = num("GX_BN", 0);
    d.kps = num("GX_KPS", 0);
    d.stages = num("GX_STAGES", 0);
    d.res2_kb = num("GX_RES2_KB", 0);
    d.serve_streams = num("GX_SERVE_STREAMS", d.serve_streams);
    d.copy_streams = num("GX_COPY_STREAMS", d.copy_streams);
#endif
    return d;
  }();
  return knobs;
}

// ---------------------------------------------------------------- tensor maps
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  }
  return fn;
}

bool encode_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                         uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  PFN_encodeTiled_t fn = encode_fn();
  if (fn == nullptr) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  const CUresult rc = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) {
    char b[256];
    snprintf(b, sizeof b, "CUresult %d: base=%p dims=(%llu,%llu) stride=%llu box=(%u,%u)", static_cast<int>(rc), base,
             static_cast<unsigned long long>(inner), static_cast<unsigned long long>(outer),
             static_cast<unsigned long long>(row_stride_bytes), box_inner, box_outer);
    g_last_encode = b;
  }
  return rc == CUDA_SUCCESS;
}

typedef CUresult (*PFN_encodeIm2col_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                       const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                       CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeIm2col_t im2col_fn() {
  static PFN_encodeIm2col_t fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeIm2col_t>(p);
  }
  return fn;
}

// NHWC input as a rank-4 (C, W, H, N) im2col map: 128 output pixels x 64 channels per load.
// Box corners follow the fprop convention: lower = -pad, upper = pad - (filter - 1).
bool encode_tmap_im2col_bf16(CUtensorMap* map, const void* base, int C, int W, int H, int N, int lower_w,
                             int lower_h, int upper_w, int upper_h, int stride_w, int stride_h, int cpl) {
  PFN_encodeIm2col_t fn = im2col_fn();
  if (fn == nullptr) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(N)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(C) * 2, static_cast<cuuint64_t>(C) * 2 * W,
                           static_cast<cuuint64_t>(C) * 2 * W * H};
  int lower[2] = {lower_w, lower_h};
  int upper[2] = {upper_w, upper_h};
  cuuint32_t es[4] = {1, static_cast<cuuint32_t>(stride_w), static_cast<cuuint32_t>(stride_h), 1};
  const CUtensorMapSwizzle sw = cpl == 64   ? CU_TENSOR_MAP_SWIZZLE_128B
                                : cpl == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : cpl == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                            : CU_TENSOR_MAP_SWIZZLE_NONE;
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, lower, upper,
            static_cast<cuuint32_t>(cpl), kBM, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---------------------------------------------------------------- development trace buffer
static unsigned long long* g_trace = nullptr;
constexpr int kTraceEntries = 1 << 20;  // >= 8*8192 + 4096 (conv_tc layout)
unsigned long long* debug_trace_buffer() {
  if (!g_trace) {
    cudaMalloc(&g_trace, kTraceEntries * sizeof(unsigned long long));
    cudaMemset(g_trace, 0, kTraceEntries * sizeof(unsigned long long));
  }
  return g_trace;
}

// NHWC input as a rank-4 (C, W, H, N) tiled map with a [64, box_w, box_h, 1] box (the halo of a
// conv_halo_kernel M tile; negative / past-the-edge coordinates are zero-filled = padding).
bool encode_tmap_halo_bf16(CUtensorMap* map, const void* base, int C, int W, int H, int N, int box_w, int box_h,
                           int box_c) {
  PFN_encodeTiled_t fn = encode_fn();
  if (fn == nullptr) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(N)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(C) * 2, static_cast<cuuint64_t>(C) * 2 * W,
                           static_cast<cuuint64_t>(C) * 2 * W * H};
  cuuint32_t box[4] = {static_cast<cuuint32_t>(box_c), static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_h),
                       1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE,
            box_c == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : box_c == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---------------------------------------------------------------- op planning
int elem_size(int dtype) { return dtype == GX_BF16 ? 2 : 4; }  // GX_F32, GX_I32: 4 bytes
int64_t tensor_elems(const gx_tensor& t) { return static_cast<int64_t>(t.H) * t.W * t.C; }

// N tile width: the persistent grid runs min(tiles, budget) CTAs, so the makespan of the busiest
// CTA is ceil(tiles / grid) tiles of (BN + a fixed per-tile cost of ~64 accumulator columns: the A
// operand fetch and the epilogue start).  Candidates: multiples of 64 (the fast epilogue paths)
// and divisors of Cout that are multiples of 16 (Inception 320 / 384 / 448 -> 160 / 192 / 224,
// the 1000-way FC); the cheapest makespan wins, wider tiles on ties.  (A pure halving rule left
// the ResNet head at 5 tiles on 2 or 4 SMs: 3 / 2 waves.)
static int pick_bn(int Cout, int m_tiles, int sm_budget, int cap) {
  const int budget = std::max(1, sm_budget);
  int best = 0;
  int64_t best_t = 0;
  auto consider = [&](int bn) {
    if (bn < 16 || bn > cap || bn > ((Cout + 15) / 16) * 16) return;
    const int64_t tiles = static_cast<int64_t>(m_tiles) * ((Cout + bn - 1) / bn);
    const int64_t grid = std::min<int64_t>(tiles, budget);
    const int64_t t = (tiles + grid - 1) / grid * (bn + 64);
    if (best == 0 || t < best_t || (t == best_t && bn > best)) {
      best = bn;
      best_t = t;
    }
  };
  for (int bn = 64; bn <= cap; bn += 64) consider(bn);
  for (int bn = 16; bn <= cap; bn += 16)
    if (Cout % bn == 0) consider(bn);
  if (Cout < 64) consider(((Cout + 15) / 16) * 16);
  return best > 0 ? best : std::min(cap, ((Cout + 15) / 16) * 16);
}

static uint32_t tmem_cols_for(int bn) {
  uint32_t need = 2u * static_cast<uint32_t>(bn);
  uint32_t c = 32;
  while (c < need) c <<= 1;
  return c;
}

int plan_conv(const gx_op& op, const gx_tensor* T, void* const* ptrs, const uint8_t* wbase, int k, int sm_budget,
              ConvLaunch* out, int bn_cap, const uint8_t* wsw, bool for_span) {
  const bool fc = op.kind == GX_OP_FC;
  if (fc && (for_span || !fc_on_tc(op) || op.Cin != tensor_elems(T[op.in])))
    return fail(GX_EINVAL, "FC not eligible for the tensor-core path");
  // an FC sees its flattened per-sample input as a 1x1 image with K channels (NHWC flatten order,
  // which is how the weights are laid out) and writes a 1x1 output with Cout channels
  const gx_tensor ti = fc ? gx_tensor{1, 1, op.Cin, T[op.in].dtype} : T[op.in];
  const gx_tensor to = fc ? gx_tensor{1, 1, op.Cout, T[op.out].dtype} : T[op.out];
  const bool gemm1x1 = op.kind != GX_OP_CONV;
  const int R = gemm1x1 ? 1 : op.R;
  const int S = gemm1x1 ? 1 : op.S;
  if (ti.dtype != GX_BF16) return fail(GX_EINVAL, "conv input must be bf16");
  if ((op.Cin & 7) || (ti.C & 7) || op.Cin > ti.C) return fail(GX_EINVAL, "conv Cin must be a multiple of 8");
  if (op.Cout & (fc ? 7 : 15)) return fail(GX_EINVAL, "conv Cout must be a multiple of 16");
  if ((to.C & 7) || (op.out_coff & 7)) return fail(GX_EINVAL, "conv output pitch/offset must be multiples of 8");
  ConvArgs& a = out->args;
  memset(&a, 0, sizeof(a));
  a.x = static_cast<const __nv_bfloat16*>(ptrs[op.in]);
  a.N = k;
  a.H = ti.H;
  a.W = ti.W;
  a.x_ld = ti.C;
  a.Cin = op.Cin;
  a.Ho = to.H;
  a.Wo = to.W;
  a.R = R;
  a.S = S;
  a.sh = gemm1x1 ? 1 : op.sh;
  a.sw = gemm1x1 ? 1 : op.sw;
  a.ph = gemm1x1 ? 0 : op.ph;
  a.pw = gemm1x1 ? 0 : op.pw;
  a.K = R * S * op.Cin;
  a.num_kb = (a.K + kBK - 1) / kBK;
  const bool ds = (op.flags & GX_OPF_DS) != 0;
  if (ds) {
    // the expand 1x1 and the block's 1x1 downsample as one GEMM: K = [in's channels | in2's]
    if (op.kind != GX_OP_CONV || R != 1 || S != 1 || op.sh != 1 || op.sw != 1 || op.ph != 0 || op.pw != 0 ||
        op.in2 < 0 || op.Cin % 64 != 0 || op.Cin != ti.C || T[op.in2].C % 64 != 0 || T[op.in2].dtype != GX_BF16 ||
        op.reserved < 1 || T[op.in2].H != to.H * op.reserved || T[op.in2].W != to.W * op.reserved || for_span)
      return fail(GX_EINVAL, "fused downsample needs a 1x1/1 conv and a 1x1 downsample over 64-channel blocks");
    a.K = op.Cin + T[op.in2].C;
    a.num_kb = a.K / kBK;
    a.ds = 1;
    a.kb_split = op.Cin / kBK;
    a.ds_stride = op.reserved;
  }
  a.M = k * a.Ho * a.Wo;
  a.Cout = op.Cout;
  a.m_tiles = (a.M + kBM - 1) / kBM;
  // 3x3 / stride 1 / pad 1 on wide images: one halo tile per 64-channel block (conv_halo.cu)
  const bool pad1 = a.ph == 1 && a.pw == 1 && (op.ph_hi < 0 || op.ph_hi == 1) && (op.pw_hi < 0 || op.pw_hi == 1);
  const bool halo128 = R == 3 && S == 3 && pad1 && op.Cin % 64 == 0 && ti.W >= 28 && ti.W + 2 <= 64;
  // the space-to-depth stem (4x4 / s1 / pad 2,2,1,1 over 16 channels): 32-byte halo rows, one K=16
  // MMA per tap, 128 // (W + 3) output rows per tile
  const bool halo32 = R == 4 && S == 4 && a.ph == 2 && a.pw == 2 && op.ph_hi == 1 && op.pw_hi == 1 && op.Cin == 16 &&
                      ti.W + 3 <= kBM && !dev().no_halo32;
  // 3x3 / stride 1 / pad 0 or 1 on images wider than a tile row (Inception's 147x147 stem convs) or
  // over 32 channels: column tiles of WT output columns, 64-byte halo rows for 32 channels
  const bool sym01 = a.ph == a.pw && a.ph <= 1 && (op.ph_hi < 0 || op.ph_hi == a.ph) && (op.pw_hi < 0 || op.pw_hi == a.pw);
  const bool halo_wide = !halo128 && R == 3 && S == 3 && sym01 && (op.Cin % 64 == 0 || op.Cin == 32) && ti.W >= 28 &&
                         a.Wo >= 28;
  if (!for_span && op.kind == GX_OP_CONV && (halo128 || halo32 || halo_wide) && a.sh == 1 && a.sw == 1 &&
      op.Cin == ti.C && (halo_wide || (a.Ho == ti.H && a.Wo == ti.W)) && op.in2 < 0 && to.dtype == GX_BF16 &&
      !dev().no_halo && !(op.flags & GX_OPF_NO_HALO)) {
    int WT = a.Wo, Wp = ti.W + (halo32 ? 3 : 2), BH = std::min(ti.H, kBM / Wp);
    if (halo_wide) {
      // the column-tile width with the fewest tiles: BH = 128 / (WT + 2) rows per tile, the halo
      // ((BH + 2) x (WT + 2) pixels) within one 256-row halo buffer
      int64_t best = INT64_MAX;
      for (int wt = 16; wt <= std::min(62, a.Wo); ++wt) {
        const int bh = std::min(a.Ho, kBM / (wt + 2));
        if (bh < 1 || (bh + 2) * (wt + 2) > 256) continue;
        const int64_t tiles = static_cast<int64_t>((a.Ho + bh - 1) / bh) * ((a.Wo + wt - 1) / wt);
        if (tiles < best) {
          best = tiles;
          WT = wt;
          BH = bh;
        }
      }
      Wp = WT + 2;
    }
    a.halo = 1;
    a.hWp = Wp;
    a.hRB = halo32 ? 32 : op.Cin == 32 ? 64 : 128;
    a.hBH = BH;
    a.hWT = halo_wide ? WT : a.Wo;
    a.hCT = (a.Wo + a.hWT - 1) / a.hWT;
    a.hTPI = (a.Ho + a.hBH - 1) / a.hBH;
    a.m_tiles = k * a.hTPI * a.hCT;
    a.BN = pick_bn(op.Cout, a.m_tiles, sm_budget, bn_cap);
    a.n_tiles = (a.Cout + a.BN - 1) / a.BN;
    a.num_tiles = a.m_tiles * a.n_tiles;
    a.bias = reinterpret_cast<const float*>(wbase + op.b_off);
    a.y = ptrs[op.out];
    a.y_ld = to.C;
    a.y_coff = op.out_coff;
    a.act = op.act;
    a.idesc = umma_idesc_bf16(kBM, a.BN);
    a.stages = conv_halo_pick_stages(a.BN, a.Cout);
    a.tmem_cols = tmem_cols_for(a.BN);
    a.wsw = dev().no_wbulk ? nullptr : wsw;
    a.dbg = dev().conv_dbg;
    a.tma_a = 1;
    const int kpad = a.num_kb * kBK;
    memset(&out->amap, 0, sizeof(out->amap));
    memset(&out->rmap, 0, sizeof(out->rmap));
    memset(&out->ymap, 0, sizeof(out->ymap));
    if (!encode_tmap_2d_bf16(&out->wmap, wbase + op.w_off, kpad, op.Cout, static_cast<uint64_t>(kpad) * 2, kBK, a.BN))
      return fail(GX_ECUDA, "cuTensorMapEncodeTiled failed for conv weights: " + g_last_encode);
    if (!encode_tmap_halo_bf16(&out->amap, a.x, ti.C, ti.W, ti.H, k, Wp, a.hBH + R - 1, halo32 ? 16 : a.hRB / 2))
      return fail(GX_ECUDA, "cuTensorMapEncodeTiled failed for the conv halo");
    if (a.stages < 2) return fail(GX_EINVAL, "halo conv: shared memory too small for the weight ring");
    out->grid = std::min(a.num_tiles, std::max(1, sm_budget));
    return GX_OK;
  }
  a.BN = pick_bn(op.Cout, a.m_tiles, sm_budget, bn_cap);
  if (const int bn = dev().bn) {  // tuning override (development builds only)
    if (bn >= 16 && bn <= 256 && bn % 16 == 0) a.BN = bn;
  }
  a.n_tiles = (a.Cout + a.BN - 1) / a.BN;
  a.num_tiles = a.m_tiles * a.n_tiles;
  a.bias = reinterpret_cast<const float*>(wbase + op.b_off);
  a.res = op.in2 >= 0 && !ds ? static_cast<const __nv_bfloat16*>(ptrs[op.in2]) : nullptr;
  a.res_ld = op.in2 >= 0 && !ds ? T[op.in2].C : 0;
  a.y = ptrs[op.out];
  a.y_ld = to.C;
  a.y_coff = op.out_coff;
  a.y_f32 = to.dtype == GX_F32;
  a.act = op.act;
  a.idesc = umma_idesc_bf16(kBM, a.BN);
  // bf16 output through smem + TMA store when every 64-column group of a tile is whole (a tile
  // never writes past its own channel slice of a concat tensor)
  a.ystore = !a.y_f32 && a.BN % 64 == 0 && a.Cout % 64 == 0 && to.C >= 64 && !dev().no_ystore && !dev().gmaps;
  // residual through the tensor core (identity k-blocks): needs the bulk-weight layout, the 2D A
  // path and whole 64-column groups; the epilogue then runs residual-free
  // only where the epilogue dominates (K <= 128: layer1/2 expands); for K >= 256 the extra BN/64
  // identity k-blocks cost more MMA time than the epilogue add they remove (measured)
  a.res_mma = !for_span && a.res && wsw && !dev().no_wbulk && res_through_mma(op) && a.BN % 64 == 0 &&
              a.num_kb <= 2 &&
              a.Cin == ti.C && !dev().no_tma_im2col && !dev().no_a2d && !dev().no_res_mma;
  const bool epi_res = a.res != nullptr && !a.res_mma;  // residual handled by the epilogue
  // Resident weights: when every tile a CTA runs shares one N tile and its weight k-blocks fit,
  // they are bulk-loaded once per CTA instead of once per tile.  At BN=256 the per-tile weight
  // stream is twice the A operand's bytes, through an L2 feed of ~86 B/clk per SM on the serving
  // budgets (the layer1/2 1x1 convs); with res_mma the BN/64 full-width identity k-blocks per tile
  // (128 KB at BN=256) become N=64 MMAs against one resident 8 KB identity block.
  {
    const int grid = std::min(a.num_tiles, std::max(1, sm_budget));
    const size_t bytes = static_cast<size_t>(a.num_kb) * a.BN * 128 + (a.res_mma ? 8192 : 0);
    a.bres = !for_span && wsw && !dev().no_wbulk && !dev().no_tma_im2col && !dev().no_bres &&
             (a.n_tiles == 1 || grid % a.n_tiles == 0 || grid >= a.num_tiles) && bytes <= 72 * 1024;
    a.idesc64 = umma_idesc_bf16(kBM, 64);
  }
  const size_t bres_bytes = a.bres ? static_cast<size_t>(a.num_kb) * a.BN * 128 + (a.res_mma ? 8192 : 0) : 0;
  // two k-blocks per pipeline stage halve the barrier round trips per unit of K; worth it when the
  // per-k-block MMA time (2*BN cycles) is below the ~500-cycle stage round trip and >= 3 stages fit
  a.cpl = (op.Cin % 64 == 0) ? 64 : (op.Cin % 32 == 0) ? 32 : (op.Cin % 16 == 0) ? 16 : 8;
  a.tma_a = !dev().no_tma_im2col;
  a.a2d = a.tma_a && a.R == 1 && a.S == 1 && a.sh == 1 && a.sw == 1 && a.ph == 0 && a.pw == 0 && a.cpl == 64 &&
          a.Cin == ti.C && !dev().no_a2d;
  // one M tile with fewer than 128 live rows (batch-1..2 FC and layer4 1x1 convs): the A box holds
  // only those rows and the pipeline stages are packed at that stride (the MMA's other rows read
  // whatever follows in smem; their outputs are never stored), so a weight-streaming GEMM keeps up
  // to 32 stages of B in flight instead of 8 stages of mostly zero-filled 16 KB A tiles (a batch-1
  // FC streamed weights at 0.22 of HBM)
  a.a_rows = (a.a2d && !ds && !for_span && !a.res_mma && a.m_tiles == 1 && a.M < kBM) ? (a.M + 7) & ~7 : kBM;
  a.kps = 1;
  {
    const bool tma = !dev().no_tma_im2col;
    const int want = dev().kps ? dev().kps : (a.BN <= 64 ? 2 : 1);
    for (int kk = want; kk >= 2 && a.kps == 1 && !a.res_mma; --kk) {
      int nres2 = 0;
      if (tma && kk <= 3 && a.num_kb >= kk &&
          conv_pick_stages(a.BN, a.num_kb, epi_res || a.ystore, a.Cout, &nres2, kk, bres_bytes, a.a_rows) >=
              (a.m_tiles == 1 ? 2 : 3))
        a.kps = kk;
    }
  }
  a.stages = conv_pick_stages(a.BN, a.num_kb + (a.res_mma ? a.BN / 64 : 0), epi_res || a.ystore, a.Cout, &a.nres,
                              a.kps, bres_bytes, a.a_rows);
  if (const int st = dev().stages) {
    if (st >= 1 && st <= a.stages) a.stages = st;
  }
  a.tmem_cols = tmem_cols_for(a.BN);
  a.wsw = dev().no_wbulk ? nullptr : wsw;
  a.dbg = dev().conv_dbg;
  a.trace = (a.dbg & 16) ? debug_trace_buffer() : nullptr;
  if (a.res && (T[op.in2].dtype != GX_BF16 || (a.res_ld & 7))) return fail(GX_EINVAL, "bad residual tensor");
  const int kpad = a.num_kb * kBK;
  memset(&out->amap, 0, sizeof(out->amap));
  memset(&out->rmap, 0, sizeof(out->rmap));
  memset(&out->ymap, 0, sizeof(out->ymap));
  a.wstore = !for_span && a.ystore && (!epi_res || !dev().no_wres) && !dev().no_tma_im2col &&
             a.BN % 128 == 0 && !dev().no_wstore;
  if (a.ystore && !encode_tmap_2d_bf16(&out->ymap, a.y, to.C, a.M, static_cast<uint64_t>(to.C) * 2, 64,
                                       a.wstore ? 32 : kBM))
    return fail(GX_ECUDA, "cuTensorMapEncodeTiled failed for the conv output: " + g_last_encode);
  if (!encode_tmap_2d_bf16(&out->wmap, wbase + op.w_off, kpad, op.Cout, static_cast<uint64_t>(kpad) * 2, kBK, a.BN))
    return fail(GX_ECUDA, "cuTensorMapEncodeTiled failed for conv weights: " + g_last_encode);
  if (a.a2d) {
    if (!encode_tmap_2d_bf16(&out->amap, a.x, ti.C, a.M, static_cast<uint64_t>(ti.C) * 2, kBK, a.a_rows))
      return fail(GX_ECUDA, "cuTensorMapEncodeTiled failed for conv input: " + g_last_encode);
  } else if (a.tma_a && !encode_tmap_im2col_bf16(&out->amap, a.x, ti.C, ti.W, ti.H, k, -a.pw, -a.ph,
                                                 (op.pw_hi >= 0 ? op.pw_hi : a.pw) - (a.S - 1),
                                                 (op.ph_hi >= 0 ? op.ph_hi : a.ph) - (a.R - 1), a.sw, a.sh, a.cpl))
    return fail(GX_ECUDA, "cuTensorMapEncodeIm2col failed for conv input");
  if (a.res && !encode_tmap_2d_bf16(&out->rmap, a.res, a.res_ld, a.M, static_cast<uint64_t>(a.res_ld) * 2, 64,
                                    (a.wstore && !a.res_mma) ? 32 : kBM))
    return fail(GX_ECUDA, "cuTensorMapEncodeTiled failed for the residual: " + g_last_encode);
  if (ds) {  // rmap = the downsample's A operand: in2 at the output pixels (x stride)
    const gx_tensor& tx = T[op.in2];
    const void* xb = ptrs[op.in2];
    const bool ok = a.ds_stride == 1
                        ? encode_tmap_2d_bf16(&out->rmap, xb, tx.C, a.M, static_cast<uint64_t>(tx.C) * 2, kBK, kBM)
                        : encode_tmap_im2col_bf16(&out->rmap, xb, tx.C, tx.W, tx.H, k, 0, 0, 0, 0, a.ds_stride,
                                                  a.ds_stride, 64);
    if (!ok) return fail(GX_ECUDA, "tensor map encode failed for the fused downsample input: " + g_last_encode);
    if (!a.tma_a || !a.a2d) return fail(GX_EINVAL, "fused downsample needs the 2D TMA A path");
  }
  out->grid = std::min(a.num_tiles, std::max(1, sm_budget));
  a.gmaps = nullptr;
  if (dev().gmaps) {  // experiment: maps in global memory (leaks one small buffer per plan)
    CUtensorMap* d = nullptr;
    CUtensorMap h[3] = {out->wmap, out->amap, out->rmap};
    if (cudaMalloc(&d, sizeof(h)) == cudaSuccess && cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice) == cudaSuccess)
      a.gmaps = d;
  }
  return GX_OK;
}

// Algorithmic work of one op at batch k: FLOPs of the unpadded math and the bytes a perfect kernel
// moves (every logical input, weight, bias, residual and output byte exactly once).
void op_work(const gx_op& op, const gx_tensor* T, int k, double* flops, double* bytes) {
  const gx_tensor& ti = T[op.in];
  const gx_tensor& to = T[op.out];
  const double es_in = elem_size(ti.dtype), es_out = elem_size(to.dtype);
  const double in_px = static_cast<double>(k) * ti.H * ti.W;
  const double out_px = static_cast<double>(k) * to.H * to.W;
  double f = 0.0, b = 0.0;
  switch (op.kind) {
    case GX_OP_CONV:
    case GX_OP_LINEAR: {
      const int R = op.kind == GX_OP_LINEAR ? 1 : op.R, S = op.kind == GX_OP_LINEAR ? 1 : op.S;
      double K = static_cast<double>(R) * S * op.Cin;
      if (op.flags & GX_OPF_DS) {  // + the fused downsample: in2 read once at the output pixels
        K += T[op.in2].C;
        b = out_px * T[op.in2].C * es_in;
      }
      f = 2.0 * out_px * op.Cout * K;
      b += in_px * op.Cin * es_in + static_cast<double>(op.Cout) * K * es_in + op.Cout * 4.0 +
           out_px * op.Cout * es_out;
      if (op.in2 >= 0 && !(op.flags & GX_OPF_DS)) b += out_px * op.Cout * es_in;
      break;
    }
    case GX_OP_MAXPOOL:
    case GX_OP_AVGPOOL:
      f = out_px * ti.C * op.R * op.S;
      b = in_px * ti.C * es_in + out_px * ti.C * es_out;
      break;
    case GX_OP_GAP:
      f = in_px * ti.C;
      b = in_px * ti.C * es_in + static_cast<double>(k) * to.C * es_out;
      break;
    case GX_OP_FC: {
      const double K = static_cast<double>(tensor_elems(ti));
      f = 2.0 * k * K * op.Cout;
      b = K * op.Cout * es_in + op.Cout * 4.0 + k * K * es_in + static_cast<double>(k) * op.Cout * es_out;
      break;
    }
    case GX_OP_COPY:
      b = 2.0 * in_px * op.Cin * es_in;
      break;
    case GX_OP_LAYERNORM:
      f = 8.0 * in_px * ti.C;
      b = in_px * ti.C * (es_in + es_out) + ti.C * 8.0;
      break;
    case GX_OP_EMBED:  // ids in; three table rows per token; LayerNorm (~8 flops per element)
      f = 10.0 * out_px * to.C;
      b = in_px * 4.0 + out_px * to.C * (3.0 * es_out + es_out) + to.C * 8.0;
      break;
    case GX_OP_ATTENTION: {
      const double S = ti.H, D = to.C;  // D = heads * head_dim
      f = 4.0 * k * S * S * D;
      b = in_px * ti.C * es_in + out_px * to.C * es_out;
      break;
    }
    default:
      b = in_px * ti.C * es_in + out_px * to.C * es_out;
  }
  *flops = f;
  *bytes = b;
}

// fp32 chains: every op on the fp32 kernels (kernels_f32.cu), same op semantics and weight layout
// as the bf16 path with fp32 elements (conv / linear weights [Cout][Kpad], FC [Cout][K]).
int launch_op_f32(const gx_op& op, const gx_tensor* T, void* const* ptrs, const uint8_t* wbase, int k, int sm_budget,
                  cudaStream_t s) {
  const int grid = std::max(1, sm_budget) * 8;
  const gx_tensor& ti = T[op.in];
  const gx_tensor& to = T[op.out];
  if (to.dtype != GX_F32) return fail(GX_EINVAL, "fp32 op writes a non-fp32 tensor");
  if (op.flags & GX_OPF_DS) return fail(GX_EINVAL, "fp32 chains take the unfused downsample");
  const float* x = static_cast<const float*>(ptrs[op.in]);
  float* y = static_cast<float*>(ptrs[op.out]);
  switch (op.kind) {
    case GX_OP_CONV:
    case GX_OP_LINEAR:
    case GX_OP_FC: {
      const bool fc = op.kind == GX_OP_FC;
      const bool conv = op.kind == GX_OP_CONV;
      ConvF32Args a;
      memset(&a, 0, sizeof(a));
      a.x = x;
      a.H = fc ? 1 : ti.H;
      a.W = fc ? 1 : ti.W;
      a.x_ld = fc ? static_cast<int>(tensor_elems(ti)) : ti.C;
      a.Cin = op.Cin;
      a.Ho = fc ? 1 : to.H;
      a.Wo = fc ? 1 : to.W;
      a.R = conv ? op.R : 1;
      a.S = conv ? op.S : 1;
      a.sh = conv ? op.sh : 1;
      a.sw = conv ? op.sw : 1;
      a.ph = conv ? op.ph : 0;
      a.pw = conv ? op.pw : 0;
      a.K = a.R * a.S * op.Cin;
      a.M = k * a.Ho * a.Wo;
      a.Cout = op.Cout;
      if (fc && op.Cin != tensor_elems(ti)) return fail(GX_EINVAL, "FC Cin must equal the flattened input size");
      if (op.Cin > (fc ? a.x_ld : ti.C)) return fail(GX_EINVAL, "conv Cin exceeds the input pitch");
      a.w = reinterpret_cast<const float*>(wbase + op.w_off);
      a.w_ld = fc ? op.Cin : (a.K + 63) / 64 * 64;
      a.bias = op.b_off >= 0 ? reinterpret_cast<const float*>(wbase + op.b_off) : nullptr;
      a.res = op.in2 >= 0 ? static_cast<const float*>(ptrs[op.in2]) : nullptr;
      a.res_ld = op.in2 >= 0 ? T[op.in2].C : 0;
      a.y = y;
      a.y_ld = fc ? op.Cout : to.C;
      a.y_coff = op.out_coff;
      a.act = op.act;
      GX_CUDA(launch_conv_f32(a, std::max(1, sm_budget) * 4, s));
      break;
    }
    case GX_OP_MAXPOOL:
    case GX_OP_AVGPOOL:
      GX_CUDA(launch_pool_f32(op.kind == GX_OP_MAXPOOL ? 0 : 1, x, k, ti.H, ti.W, ti.C, y, to.H, to.W, to.C,
                              op.out_coff, op.R, op.S, op.sh, op.sw, op.ph, op.pw, op.flags & 1, grid, s));
      break;
    case GX_OP_GAP:
      GX_CUDA(launch_gap_f32(x, k, ti.H * ti.W, ti.C, y, grid, s));
      break;
    case GX_OP_COPY:
      GX_CUDA(launch_copy_channels_f32(x, static_cast<int64_t>(k) * ti.H * ti.W, op.Cin, ti.C, op.ph, y, to.C,
                                       op.out_coff, grid, s));
      break;
    case GX_OP_LAYERNORM:
      GX_CUDA(launch_layernorm_f32(x, k * ti.H * ti.W, ti.C, reinterpret_cast<const float*>(wbase + op.w_off),
                                   reinterpret_cast<const float*>(wbase + op.b_off), op.eps, y, grid, s));
      break;
    case GX_OP_ATTENTION:
      if (op.heads < 1 || to.C % op.heads || ti.C != 3 * to.C) return fail(GX_EINVAL, "bad attention shapes");
      GX_CUDA(launch_attention_f32(x, k, ti.H, op.heads, to.C / op.heads, y, grid, s));
      break;
    default:
      return fail(GX_EINVAL, "op kind " + std::to_string(op.kind) + " has no fp32 kernel");
  }
  return GX_OK;
}

int launch_op(const gx_op& op, const gx_tensor* T, void* const* ptrs, const uint8_t* wbase, int k, int sm_budget,
              cudaStream_t s, bool pdl, const ConvLaunch* pre, int* kernels) {
  const int bw_grid = std::max(1, sm_budget) * 8;
  if (op.kind == GX_OP_EMBED) {
    // K8: token ids (int32 [S]) -> LayerNorm(word[id] + pos[s] + type[0]) in the chain's type
    const gx_tensor& ti = T[op.in];
    const gx_tensor& to = T[op.out];
    if (ti.dtype != GX_I32 || ti.C != 1 || ti.W != 1 || to.H != ti.H || to.W != 1 || ti.H > op.R)
      return fail(GX_EINVAL, "embed: int32 ids [S,1,1] -> [S,1,C] with S <= max positions");
    GX_CUDA(launch_embed(static_cast<const int32_t*>(ptrs[op.in]), k * ti.H, ti.H, to.C, wbase + op.w_off, op.Cin,
                         wbase + op.w2_off, wbase + op.w3_off, reinterpret_cast<const float*>(wbase + op.b_off),
                         reinterpret_cast<const float*>(wbase + op.b_off) + to.C, op.eps, ptrs[op.out],
                         to.dtype == GX_F32, bw_grid, s));
    if (kernels) ++*kernels;
    return GX_OK;
  }
  if (T[op.in].dtype == GX_F32) {
    const int rc = launch_op_f32(op, T, ptrs, wbase, k, sm_budget, s);
    if (rc == GX_OK && kernels) ++*kernels;
    return rc;
  }
  switch (op.kind) {
    case GX_OP_CONV:
    case GX_OP_LINEAR: {
      ConvLaunch cl;
      if (pre == nullptr) {
        int rc = plan_conv(op, T, ptrs, wbase, k, sm_budget, &cl);
        if (rc != GX_OK) return rc;
        pre = &cl;
      }
      if (pre->args.halo)
        GX_CUDA(launch_conv_halo(pre->wmap, pre->amap, pre->args, pre->grid, s, pdl));
      else
        GX_CUDA(launch_conv(pre->wmap, pre->amap, pre->rmap, pre->ymap, pre->args, pre->grid, s, pdl));
      break;
    }
    case GX_OP_MAXPOOL:
    case GX_OP_AVGPOOL: {
      const gx_tensor& ti = T[op.in];
      const gx_tensor& to = T[op.out];
      GX_CUDA(launch_pool(op.kind == GX_OP_MAXPOOL ? 0 : 1, static_cast<const __nv_bfloat16*>(ptrs[op.in]), k, ti.H,
                          ti.W, ti.C, ti.C, static_cast<__nv_bfloat16*>(ptrs[op.out]), to.H, to.W, to.C, op.out_coff,
                          op.R, op.S, op.sh, op.sw, op.ph, op.pw, op.flags & 1, bw_grid, s));
      break;
    }
    case GX_OP_GAP: {
      const gx_tensor& ti = T[op.in];
      GX_CUDA(launch_gap(static_cast<const __nv_bfloat16*>(ptrs[op.in]), k, ti.H * ti.W, ti.C,
                         static_cast<__nv_bfloat16*>(ptrs[op.out]), bw_grid, s));
      break;
    }
    case GX_OP_FC: {
      if (fc_on_tc(op)) {
        ConvLaunch cl;
        if (pre == nullptr) {
          int rc = plan_conv(op, T, ptrs, wbase, k, sm_budget, &cl);
          if (rc != GX_OK) return rc;
          pre = &cl;
        }
        GX_CUDA(launch_conv(pre->wmap, pre->amap, pre->rmap, pre->ymap, pre->args, pre->grid, s, pdl));
        break;
      }
      const gx_tensor& ti = T[op.in];
      const gx_tensor& to = T[op.out];
      const int K = static_cast<int>(tensor_elems(ti));
      if (op.Cin != K) return fail(GX_EINVAL, "FC Cin must equal the flattened input size");
      GX_CUDA(launch_fc(static_cast<const __nv_bfloat16*>(ptrs[op.in]), k, K,
                        reinterpret_cast<const __nv_bfloat16*>(wbase + op.w_off),
                        op.b_off >= 0 ? reinterpret_cast<const float*>(wbase + op.b_off) : nullptr, ptrs[op.out],
                        op.Cout, to.dtype == GX_F32, op.act, bw_grid, s));
      break;
    }
    case GX_OP_COPY: {
      const gx_tensor& ti = T[op.in];
      const gx_tensor& to = T[op.out];
      GX_CUDA(launch_copy_channels(static_cast<const __nv_bfloat16*>(ptrs[op.in]),
                                   static_cast<int64_t>(k) * ti.H * ti.W, op.Cin, ti.C, op.ph,
                                   static_cast<__nv_bfloat16*>(ptrs[op.out]), to.C, op.out_coff, bw_grid, s));
      break;
    }
    case GX_OP_LAYERNORM: {
      const gx_tensor& ti = T[op.in];
      const int rows = k * ti.H * ti.W;
      GX_CUDA(launch_layernorm(static_cast<const __nv_bfloat16*>(ptrs[op.in]), nullptr, rows, ti.C,
                               reinterpret_cast<const float*>(wbase + op.w_off),
                               reinterpret_cast<const float*>(wbase + op.b_off), op.eps,
                               static_cast<__nv_bfloat16*>(ptrs[op.out]), bw_grid, s));
      break;
    }
    case GX_OP_ATTENTION: {
      const gx_tensor& ti = T[op.in];
      const gx_tensor& to = T[op.out];
      if (op.heads < 1 || to.C % op.heads || ti.C != 3 * to.C) return fail(GX_EINVAL, "bad attention shapes");
      GX_CUDA(launch_attention(static_cast<const __nv_bfloat16*>(ptrs[op.in]), k, ti.H, op.heads, to.C / op.heads,
                               static_cast<__nv_bfloat16*>(ptrs[op.out]), bw_grid, s));
      break;
    }
    default:
      return fail(GX_EINVAL, "unsupported op kind " + std::to_string(op.kind));
  }
  if (kernels) ++*kernels;
  return GX_OK;
}

}  // namespace gx

using namespace gx;

// ==================================================================== C ABI
extern "C" {

int gx_abi_version(void) { return GX_ABI_VERSION; }

// Development: copy the conv kernel's clock64 trace (GX_CONV_DBG & 16) to the host and clear it.
int gx_debug_trace(int64_t* out, int64_t n) {
  if (!g_trace || !out || n <= 0) return fail(GX_EINVAL, "no trace");
  if (n > kTraceEntries) n = kTraceEntries;
  GX_CUDA(cudaDeviceSynchronize());
  GX_CUDA(cudaMemcpy(out, g_trace, n * sizeof(int64_t), cudaMemcpyDeviceToHost));
  GX_CUDA(cudaMemset(g_trace, 0, kTraceEntries * sizeof(unsigned long long)));
  return GX_OK;
}

int gx_last_error(char* buf, size_t n) {
  if (buf && n) {
    std::strncpy(buf, g_last_error.c_str(), n - 1);
    buf[n - 1] = 0;
  }
  return static_cast<int>(g_last_error.size());
}

int gx_init(int device, gx_ctx** out) {
  if (!out) return fail(GX_EINVAL, "null out");
  GX_CUDA(cudaSetDevice(device));
  int sms = 0;
  GX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  int major = 0, minor = 0;
  GX_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  GX_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
  if (major != 10 || minor != 0)
    return fail(GX_EINFEASIBLE, "libgx is built for sm_100a (B200); device is sm_" + std::to_string(major) +
                                    std::to_string(minor));
  if (encode_fn() == nullptr) return fail(GX_ECUDA, "driver entry point cuTensorMapEncodeTiled unavailable");
  gx_ctx* c = new gx_ctx();
  c->device = device;
  c->sm_count = sms;
  *out = c;
  return GX_OK;
}

int gx_destroy(gx_ctx* ctx) {
  delete ctx;
  return GX_OK;
}

int gx_sm_count(gx_ctx* ctx, int* out) {
  if (!ctx || !out) return fail(GX_EINVAL, "null arg");
  *out = ctx->sm_count;
  return GX_OK;
}

int gx_run_op(gx_ctx* ctx, const gx_op* op, const gx_tensor* tensors, void* const* tensor_ptrs, const void* weights,
              int k, int sm_budget, void* stream) {
  if (!ctx || !op || !tensors || !tensor_ptrs) return fail(GX_EINVAL, "null arg");
  if (k < 1) return fail(GX_EINVAL, "batch must be >= 1");
  if (int rc = bind_device(ctx->device)) return rc;
  if (sm_budget <= 0 || sm_budget > ctx->sm_count) sm_budget = ctx->sm_count;
  return launch_op(*op, tensors, tensor_ptrs, static_cast<const uint8_t*>(weights), k, sm_budget,
                   static_cast<cudaStream_t>(stream), false, nullptr, nullptr);
}

int gx_gather(gx_ctx* ctx, int k, const void* const* src, const int32_t* src_dtype, int64_t pixels, int32_t c_src,
              int32_t c_dst, void* dst, int sm_budget, void* stream) {
  if (!ctx) return fail(GX_EINVAL, "null ctx");
  if (k < 1 || k > 64) return fail(GX_EINVAL, "gather batch must be in 1..64");
  if (int rc = bind_device(ctx->device)) return rc;
  if (sm_budget <= 0 || sm_budget > ctx->sm_count) sm_budget = ctx->sm_count;
  GX_CUDA(launch_gather(k, src, src_dtype, pixels, c_src, c_dst, static_cast<__nv_bfloat16*>(dst), sm_budget * 8,
                        static_cast<cudaStream_t>(stream)));
  return GX_OK;
}

int gx_gather_ex(gx_ctx* ctx, int k, const void* const* src, const int32_t* src_dtype, int32_t Ho, int32_t Wo,
                 int32_t f, int32_t c_src, int32_t c_dst, void* dst, int32_t dst_dtype, int sm_budget, void* stream) {
  if (!ctx || !src || !src_dtype || !dst) return fail(GX_EINVAL, "null arg");
  if (k < 1 || k > 64) return fail(GX_EINVAL, "gather batch must be in 1..64");
  if (f < 1 || Ho < 1 || Wo < 1 || c_src < 1 || c_dst < 1 || f * f * c_src > c_dst)
    return fail(GX_EINVAL, "bad gather shape");
  if (int rc = bind_device(ctx->device)) return rc;
  if (sm_budget <= 0 || sm_budget > ctx->sm_count) sm_budget = ctx->sm_count;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = sm_budget * 8;
  if (dst_dtype == GX_F32) {
    if (f > 1)
      GX_CUDA(launch_gather_s2d_f32(k, src, src_dtype, Ho, Wo, f, c_src, c_dst, static_cast<float*>(dst), grid, s));
    else
      GX_CUDA(launch_gather_f32(k, src, src_dtype, static_cast<int64_t>(Ho) * Wo, c_src, c_dst,
                                static_cast<float*>(dst), grid, s));
  } else if (f > 1) {
    GX_CUDA(launch_gather_s2d(k, src, src_dtype, Ho, Wo, f, c_src, c_dst, static_cast<__nv_bfloat16*>(dst), grid, s));
  } else {
    GX_CUDA(launch_gather(k, src, src_dtype, static_cast<int64_t>(Ho) * Wo, c_src, c_dst,
                          static_cast<__nv_bfloat16*>(dst), grid, s));
  }
  return GX_OK;
}

int gx_scatter(gx_ctx* ctx, int k, const void* src, int32_t src_dtype, int64_t row_elems, void* const* dst,
               int32_t dst_dtype, int sm_budget, void* stream) {
  if (!ctx) return fail(GX_EINVAL, "null ctx");
  if (k < 1 || k > 64) return fail(GX_EINVAL, "scatter batch must be in 1..64");
  if (int rc = bind_device(ctx->device)) return rc;
  if (sm_budget <= 0 || sm_budget > ctx->sm_count) sm_budget = ctx->sm_count;
  GX_CUDA(launch_scatter(k, src, src_dtype, row_elems, dst, dst_dtype, sm_budget * 8,
                         static_cast<cudaStream_t>(stream)));
  return GX_OK;
}

}  // extern "C"
