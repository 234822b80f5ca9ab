// Internal declarations shared by the libgx translation units.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "graft_exec.h"

namespace gx {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
// Make `device`'s primary context current on the calling thread (tensor-map encoding and graph
// capture need one; a caller thread that never touched CUDA has none).  Cheap when already bound.
int bind_device(int device);

// Kernel-selection experiments of development builds (-DGX_DEV_KNOBS reads them from GX_*
// environment variables once); the product library always runs the defaults below.
struct DevKnobs {
  bool no_halo = false, no_halo32 = false, no_wbulk = false, no_ystore = false, gmaps = false, no_res_mma = false,
       no_tma_im2col = false, no_a2d = false, no_wres = false, no_wstore = false, fc_simt = false, no_pdl = false,
       pool_nostrip = false, no_bres = false;
  int conv_dbg = 0, bn = 0, kps = 0, stages = 0, res2_kb = 0;
  int serve_streams = 64;  // serving stream-pool lanes
  int copy_streams = 1;    // DMA-ingress copy streams
};
const DevKnobs& dev();

#define GX_CUDA(call)                                   \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return ::gx::cuda_fail(_e, #call); \
  } while (0)

// Driver entry point for cuTensorMapEncodeTiled (resolved once through the runtime).
bool encode_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                         uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);

// ------------------------------------------------------------------ implicit-GEMM conv (K2)
// GEMM view: M = k*Ho*Wo output pixels, N = Cout, K = R*S*Cin (ordered r, s, cin).
struct ConvArgs {
  const __nv_bfloat16* x;  // input NHWC, pixel pitch x_ld elements
  int N, H, W, x_ld, Cin;
  int Ho, Wo, R, S, sh, sw, ph, pw;
  int K, num_kb;  // num_kb = ceil(K / 64)
  int M, Cout, BN, m_tiles, n_tiles, num_tiles;
  const float* bias;
  const __nv_bfloat16* res;  // residual [M][res_ld] or null
  int res_ld;
  void* y;  // output [M][y_ld] at column offset y_coff (bf16, or fp32 if y_f32)
  int y_ld, y_coff, y_f32;
  int act;
  uint32_t idesc;
  int stages;
  uint32_t tmem_cols;
  int tma_a;  // A operand via im2col TMA, else cp.async im2col producers
  int cpl;    // channels per im2col TMA load (8/16/32/64): Cin % cpl == 0, cpl | 64
  int nres;   // residual smem slots (0 without residual, else 1 or 2)
  int a2d;    // A via a plain 2D tiled map over [M, C] (1x1, stride 1, no padding)
  const CUtensorMap* gmaps;  // experiment: tensor maps read from global memory instead of params
  int ystore;  // bf16 output staged in the smem slots and written by TMA stores (ymap), else st.global
  int wstore;  // ystore without residual: each epilogue warp TMA-stores its own 32-row box (ymap box 64x32)
  int dbg;  // GX_CONV_DBG timing attribution (results invalid): 1 skip A loads, 2 skip B loads,
            // 4 skip MMAs, 8 skip the epilogue's TMEM reads and stores
  int kps;  // k-blocks per pipeline stage (1 or 2; 2 only with TMA-built A)
  unsigned long long* trace;  // dbg & 16: per-iteration clock64 stamps of CTA 0 (development)
  const uint8_t* wsw;  // B tiles by plain bulk copy from the pre-swizzled [kb][Cout][64] layout (or null)
  int res_mma;         // residual added by the MMA: BN/64 extra k-blocks per tile, A = residual tile
                       // (rmap, box 64 x 128), B = identity blocks at kb = num_kb + col/64 (wsw)
  int halo;            // 3x3/s1/p1 wide-image conv on conv_halo_kernel (amap = the 4D halo map)
  int hBH, hTPI;       // halo: output rows per M tile, M tiles per image
  int hWp, hRB;        // halo: row pitch of a tile's halo (WT + S - 1), bytes per halo pixel row (128 | 64 | 32)
  int hWT, hCT;        // halo: output columns per tile, column tiles per image row
  int bres;            // B resident: the CTA's num_kb weight k-blocks (its N tile is fixed) are bulk-loaded
                       // once and stay in smem; with res_mma the residual is added by N=64 MMAs into
                       // the accumulator's 64-column slices against one resident 64x64 identity block
  uint32_t idesc64;    // instruction descriptor of those M=128, N=64 MMAs
  int ds;              // GX_OPF_DS: k-blocks >= kb_split take A from the block input (rmap): a 2D map
  int kb_split;        // over [M][Cx] (ds_stride 1) or a 1x1 im2col map at the downsample stride
  int ds_stride;
  int a_rows;  // a2d: rows per A load; a single M tile with M < 128 (FC / 1x1 convs at batch 1-2)
               // loads only its live rows, the MMA's other rows read stale smem whose outputs are
               // never stored (row i of the product depends on row i of A only)
};
constexpr int kConvThreads = 320;  // span kernel: 4 A-producer warps, TMA warp, MMA warp, 4 epilogue warps
// conv_tc: warps 0-3 cp.async A producers (or epilogue when TMA builds A), 4 A/B TMA, 5 MMA,
// 6-9 epilogue, 10 B TMA (TMA mode)
constexpr int kConvTcThreads = 352;
constexpr int kBM = 128;
constexpr int kBK = 64;
// bres_bytes: resident weight (+ identity) bytes; stages then hold only the A operand
// a_rows < kBM: A tiles packed at a_rows x 128 bytes per k-block (ConvArgs::a_rows)
size_t conv_smem_bytes(int BN, int stages, int num_kb, int nres, int Cout, int kps = 1, size_t bres_bytes = 0,
                       int a_rows = kBM);
int conv_pick_stages(int BN, int num_kb, bool res, int Cout, int* nres_out, int kps = 1, size_t bres_bytes = 0,
                     int a_rows = kBM);
// wmap: weights [Cout][Kpad]; amap: im2col map of the input (tma_a); rmap: residual [M][res_ld];
// ymap: output [M][y_ld] (ystore).
cudaError_t launch_conv(const CUtensorMap& wmap, const CUtensorMap& amap, const CUtensorMap& rmap,
                        const CUtensorMap& ymap, const ConvArgs& a, int grid, cudaStream_t s, bool pdl);
size_t conv_halo_smem_bytes(int BN, int stages, int Cout);
int conv_halo_pick_stages(int BN, int Cout);
cudaError_t launch_conv_halo(const CUtensorMap& wmap, const CUtensorMap& hmap, const ConvArgs& a, int grid,
                             cudaStream_t s, bool pdl);
bool encode_tmap_halo_bf16(CUtensorMap* map, const void* base, int C, int W, int H, int N, int box_w, int box_h,
                           int box_c = 64);
bool encode_tmap_im2col_bf16(CUtensorMap* map, const void* base, int C, int W, int H, int N, int lower_w,
                             int lower_h, int upper_w, int upper_h, int stride_w, int stride_h, int cpl);

// ------------------------------------------------------------------ bandwidth-bound kernels
cudaError_t launch_gather(int k, const void* const* src, const int32_t* src_dtype, int64_t pixels,
                          int c_src, int c_dst, __nv_bfloat16* dst, int grid, cudaStream_t s);
cudaError_t launch_gather_s2d(int k, const void* const* src, const int32_t* src_dtype, int Ho, int Wo, int f,
                              int c_src, int c_dst, __nv_bfloat16* dst, int grid, cudaStream_t s);
cudaError_t launch_scatter(int k, const void* src, int src_dtype, int64_t row_elems, void* const* dst,
                           int dst_dtype, int grid, cudaStream_t s);
cudaError_t launch_gather_words(int k, const void* const* src, int64_t words, uint32_t* dst, int grid,
                                cudaStream_t s);
// K1 scatter of fp32 chain outputs fused with K9 top-1 (argmax, first maximal index) per row;
// dst may be null (or hold null rows): top-1 only
cudaError_t launch_scatter_top1(int k, const float* src, int64_t row_elems, void* const* dst, int32_t* const* top1,
                                cudaStream_t s);
cudaError_t launch_pool(int mode, const __nv_bfloat16* x, int N, int H, int W, int C, int x_ld,
                        __nv_bfloat16* y, int Ho, int Wo, int y_ld, int y_coff, int R, int S, int sh,
                        int sw, int ph, int pw, int count_include_pad, int grid, cudaStream_t s);
cudaError_t launch_gap(const __nv_bfloat16* x, int N, int HW, int C, __nv_bfloat16* y, int grid,
                       cudaStream_t s);
cudaError_t launch_fc(const __nv_bfloat16* x, int N, int K, const __nv_bfloat16* w, const float* b,
                      void* y, int Nout, int y_f32, int act, int grid, cudaStream_t s);
cudaError_t launch_copy_channels(const __nv_bfloat16* x, int64_t pixels, int C, int x_ld, int x_coff,
                                 __nv_bfloat16* y, int y_ld, int y_coff, int grid, cudaStream_t s);
cudaError_t launch_flatten_nchw(const __nv_bfloat16* x, int N, int HW, int C, __nv_bfloat16* y, int grid,
                                cudaStream_t s);
// K8 BERT embeddings + LayerNorm: ids int32 [rows], token s = row % S; tables in bf16 (f32 = 0)
// or fp32 (f32 = 1), output in the same type
cudaError_t launch_embed(const int32_t* ids, int rows, int S, int C, const void* word, int V, const void* pos,
                         const void* type0, const float* gamma, const float* beta, float eps, void* y, int f32,
                         int grid, cudaStream_t s);
cudaError_t launch_layernorm(const __nv_bfloat16* x, const __nv_bfloat16* res, int rows, int C,
                             const float* gamma, const float* beta, float eps, __nv_bfloat16* y, int grid,
                             cudaStream_t s);
cudaError_t launch_attention(const __nv_bfloat16* qkv, int N, int S, int heads, int dh,
                             __nv_bfloat16* out, int grid, cudaStream_t s);

// ------------------------------------------------------------------ fp32 execution mode (kernels_f32.cu)
struct ConvF32Args {
  const float* x;  // input NHWC, pixel pitch x_ld
  int H, W, x_ld, Cin;
  int Ho, Wo, R, S, sh, sw, ph, pw;
  int K, M, Cout;  // K = R*S*Cin (ordered r, s, cin), M = k*Ho*Wo
  const float* w;  // [Cout][w_ld] fp32
  int w_ld;
  const float* bias;  // [Cout] or null
  const float* res;   // residual [M][res_ld] or null
  int res_ld;
  float* y;  // [M][y_ld] at column offset y_coff
  int y_ld, y_coff, act;
};
cudaError_t launch_conv_f32(const ConvF32Args& a, int grid, cudaStream_t s);
cudaError_t launch_pool_f32(int mode, const float* x, int N, int H, int W, int C, float* y, int Ho, int Wo, int y_ld,
                            int y_coff, int R, int S, int sh, int sw, int ph, int pw, int count_include_pad, int grid,
                            cudaStream_t s);
cudaError_t launch_gap_f32(const float* x, int N, int HW, int C, float* y, int grid, cudaStream_t s);
cudaError_t launch_copy_channels_f32(const float* x, int64_t pixels, int C, int x_ld, int x_coff, float* y, int y_ld,
                                     int y_coff, int grid, cudaStream_t s);
cudaError_t launch_layernorm_f32(const float* x, int rows, int C, const float* gamma, const float* beta, float eps,
                                 float* y, int grid, cudaStream_t s);
cudaError_t launch_attention_f32(const float* qkv, int N, int S, int heads, int dh, float* out, int grid,
                                 cudaStream_t s);
cudaError_t launch_gather_f32(int k, const void* const* src, const int32_t* src_dtype, int64_t pixels, int c_src,
                              int c_dst, float* dst, int grid, cudaStream_t s);
cudaError_t launch_gather_s2d_f32(int k, const void* const* src, const int32_t* src_dtype, int Ho, int Wo, int f,
                                  int c_src, int c_dst, float* dst, int grid, cudaStream_t s);

}  // namespace gx
