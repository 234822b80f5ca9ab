// K2/K3: implicit-GEMM convolution (and token-wise linear) on 5th-gen tensor cores.
//
//   D[M, N] = im2col(X)[M, K] * W[N, K]^T  (+ bias, + residual, act)   M = k*Ho*Wo, N = Cout
//
// Warp-specialised persistent kernel, one CTA per SM, grid bounded by the stage's SM budget:
//   warp 4     producer: per smem stage one im2col-mode TMA for the A tile (128 output pixels x
//              64 channels of one filter tap; padding and image edges are TMA zero-fill) and one
//              tiled TMA for the B (weight) tile, both on the stage's full barrier.  When
//              Cin % 64 != 0 (3-channel stem, Inception's 288/48/80-channel tensors) warps 0-3
//              build A with cp.async im2col instead (16 B chunks, zero-fill for padding);
//   warp 4     also owns TMEM (alloc/dealloc);
//   warp 5     MMA issuer: one thread issues tcgen05.mma (M=128, N=BN, K=16) into TMEM;
//   warps 6-9  epilogue: bias (bulk copy) and the residual tile (TMA) are staged in smem at
//              tile start, then tcgen05.ld -> +bias +residual -> act -> bf16/fp32 stores.
// Smem ring of `stages` (A,B) slots with full/empty mbarriers; two TMEM accumulators so the
// epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda_bf16.h>

#include <cstdlib>

#include "gx_internal.h"
#include "gx_ptx.cuh"

namespace gx {

namespace {
constexpr int kATileBytes = kBM * kBK * 2;
constexpr int kMaxStages = 32;  // pipeline stages of a short-A (a_rows < 128) weight-streaming GEMM
constexpr int kResGroupBytes = kBM * 64 * 2;  // one 128 x 64 bf16 residual box

__device__ __forceinline__ float gelu_erf(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

struct SmemPlan {
  uint8_t* sA;
  uint8_t* sB;
  uint8_t* sRes;
  float* sBias;
  uint64_t* full;
  uint64_t* empty;
  uint64_t* tfull;
  uint64_t* tempty;
  uint64_t* rfull;  // [2] residual slot filled
  uint64_t* rfw;    // [8 epilogue warps][2 slots] per-warp residual boxes filled (WST)
  uint64_t* bfull;  // bias vector staged
  uint64_t* bresbar;  // resident weights (and identity block) landed
  uint8_t* sBres;     // bres: [num_kb][BN*128] resident weight k-blocks of the CTA's N tile
  uint8_t* sIdent;    // bres + res_mma: one 64x64 identity block (swizzled, 8 KB)
  uint32_t* tslot;
  int2* ktab;
};

__host__ __device__ inline uint32_t bres_alloc(int bres, int num_kb, int BN, int res_mma) {
  return bres ? static_cast<uint32_t>(num_kb) * BN * 128u + (res_mma ? 8192u : 0u) : 0u;
}

__host__ __device__ inline int res_groups(int BN) { return (BN + 63) / 64; }
__host__ __device__ inline uint32_t bias_alloc(int Cout) { return (static_cast<uint32_t>(Cout) * 4u + 1023u) & ~1023u; }

// How the many epilogue threads wait for the accumulator / residual / bias (development knob;
// default: every thread polls with a short back-off).
__device__ __forceinline__ void epi_wait(uint64_t* bar, uint32_t parity) {
#if defined(GX_EPI_WAIT) && GX_EPI_WAIT == 0
  mbar_wait(bar, parity);
#elif defined(GX_EPI_WAIT) && GX_EPI_WAIT == 2
  if ((threadIdx.x & 31) == 0) mbar_wait(bar, parity);
  __syncwarp();
  mbar_wait(bar, parity);  // completed phase: returns at once, gives every lane the acquire
#else
  mbar_wait_sleepy(bar, parity);
#endif
}

// Producer / MMA warps: how the warp waits on a pipeline barrier (development knob).
__device__ __forceinline__ void pipe_wait(uint64_t* bar, uint32_t parity, bool issuer) {
#if defined(GX_WAIT1)
  if (issuer) mbar_wait(bar, parity);
  __syncwarp();
#else
  (void)issuer;
  mbar_wait(bar, parity);
#endif
}

template <bool kTmaA, int KPS, bool WST>
__global__ void __launch_bounds__(kConvTcThreads, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap amap,
                   const __grid_constant__ CUtensorMap rmap, const __grid_constant__ CUtensorMap ymap,
                   const ConvArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const CUtensorMap* WM = a.gmaps ? a.gmaps : &wmap;
  const CUtensorMap* AM = a.gmaps ? a.gmaps + 1 : &amap;
  const CUtensorMap* RM = a.gmaps ? a.gmaps + 2 : &rmap;
  const CUtensorMap* YM = &ymap;
  const int S_ = a.stages;
  const int BN = a.BN;
  const bool has_res = a.res != nullptr && !a.res_mma;  // residual added in the epilogue
  const bool ystore = a.ystore != 0;
  // k-blocks per tile: the conv's K, plus (res_mma) BN/64 residual x identity blocks
  const int nkb_tile = a.num_kb + (a.res_mma ? BN / 64 : 0);
  const uint32_t b_bytes = static_cast<uint32_t>(BN) * 128u;
  SmemPlan sp;
  sp.sA = smem;
  // KPS: k-blocks per pipeline stage (TMA mode): one barrier round trip per KPS*64 of K
  const bool bres = a.bres != 0;
  // A tile stride: 128 rows, or a single short M tile's live rows (a.a_rows); the region keeps a
  // full tile's worth past the last stage so the MMA's 128-row reads stay inside the allocation
  const uint32_t a_tile = static_cast<uint32_t>(a.a_rows) * 128u;
  const uint32_t sa_bytes = KPS * a_tile, sb_bytes = bres ? 0u : KPS * b_bytes;
  sp.sB = sp.sA + static_cast<size_t>(S_) * sa_bytes + (kATileBytes - a_tile);
  sp.sBres = sp.sB + static_cast<size_t>(S_) * sb_bytes;
  sp.sIdent = sp.sBres + static_cast<size_t>(a.num_kb) * b_bytes;
  sp.sRes = sp.sBres + bres_alloc(a.bres, a.num_kb, BN, a.res_mma);
  // slots: the residual tile (TMA-loaded) and/or the staged output tile (TMA-stored), in place
  const uint32_t res_slot_bytes = (has_res || ystore) ? res_groups(BN) * kResGroupBytes : 0u;
  sp.sBias = reinterpret_cast<float*>(sp.sRes + a.nres * res_slot_bytes);
  sp.full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sp.sBias) + bias_alloc(a.Cout));
  sp.empty = sp.full + S_;
  sp.tfull = sp.empty + S_;
  sp.tempty = sp.tfull + 2;
  sp.rfull = sp.tempty + 2;
  sp.bfull = sp.rfull + 2;
  sp.rfw = sp.bfull + 1;
  sp.bresbar = sp.rfw + 16;
  sp.tslot = reinterpret_cast<uint32_t*>(sp.bresbar + 1);
  sp.ktab = reinterpret_cast<int2*>(sp.tslot + 4);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  if (!kTmaA) {
    // K-chunk table: chunk q = K elements [8q, 8q+8) -> (filter row r, filter col s, channel c).
    const int nq = a.num_kb * 8;
    for (int q = tid; q < nq; q += blockDim.x) {
      const int kk = q * 8;
      int2 e;
      if (kk < a.K) {
        const int tap = kk / a.Cin;
        const int c = kk - tap * a.Cin;
        const int r = tap / a.S;
        const int s = tap - r * a.S;
        e.x = (r << 16) | s;
        e.y = c;
      } else {
        e.x = 0;
        e.y = -1;
      }
      sp.ktab[q] = e;
    }
  }
  if (warp == 4) {
    if (lane == 0) {
      for (int i = 0; i < S_; ++i) {
        mbar_init(&sp.full[i], kTmaA ? 2 : 128 + 1);
        mbar_init(&sp.empty[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&sp.tfull[i], 1);
        mbar_init(&sp.tempty[i], kTmaA ? 8 : 4);  // one arrival per epilogue warp
      }
      mbar_init(&sp.rfull[0], 1);
      mbar_init(&sp.rfull[1], 1);
      for (int i = 0; i < 16; ++i) mbar_init(&sp.rfw[i], 1);
      mbar_init(sp.bfull, 1);
      mbar_init(sp.bresbar, 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(sp.tslot, a.tmem_cols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *sp.tslot;
  const uint32_t acc_stride = a.tmem_cols >> 1;

  // Programmatic dependent launch: everything above overlapped the previous kernel's tail.
  pdl_wait();

  const int HoWo = a.Ho * a.Wo;
  if (warp < 4 && !kTmaA) {
    {
      // ---------------------------------------------------------- A producers (cp.async im2col)
      const int row = tid;
      int it = 0;
      for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
        const int m_blk = tile / a.n_tiles;
        const int m = m_blk * kBM + row;
        const bool row_ok = m < a.M;
        int n = 0, ho = 0, wo = 0;
        if (row_ok) {
          n = m / HoWo;
          const int rem = m - n * HoWo;
          ho = rem / a.Wo;
          wo = rem - ho * a.Wo;
        }
        const int hi0 = ho * a.sh - a.ph;
        const int wi0 = wo * a.sw - a.pw;
        const __nv_bfloat16* xn = a.x + static_cast<size_t>(n) * a.H * a.W * a.x_ld;
        for (int kb = 0; kb < a.num_kb; ++kb, ++it) {
          const int st = it % S_;
          const uint32_t ph = (it / S_) & 1;
          mbar_wait(&sp.empty[st], ph ^ 1);
          const uint32_t dst = smem_u32(sp.sA + st * kATileBytes + row * 128);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int2 e = sp.ktab[kb * 8 + j];
            const int hi = hi0 + (e.x >> 16);
            const int wi = wi0 + (e.x & 0xffff);
            const bool ok = row_ok && e.y >= 0 && static_cast<unsigned>(hi) < static_cast<unsigned>(a.H) &&
                            static_cast<unsigned>(wi) < static_cast<unsigned>(a.W);
            const __nv_bfloat16* src = ok ? xn + (static_cast<size_t>(hi) * a.W + wi) * a.x_ld + e.y : a.x;
            cp_async16_zfill(dst + ((j ^ (row & 7)) << 4), src, ok ? 16u : 0u);
          }
          // non-blocking: the mbarrier counts this thread's arrival when its copies land
          cp_async_arrive_noinc(&sp.full[st]);
        }
      }
    }
  } else if (warp == 4 || warp == 10) {
    // ------------------------------------------------------------ TMA producers
    // Warp 4 issues the A operand (im2col / 2D TMA), warp 10 the B operand (weights), each on its
    // own arrival of the stage's full barrier, so the two request streams overlap instead of
    // queueing behind one issuing thread.  (cp.async mode: warps 0-3 build A, warp 4 loads B.)
    // The whole warp walks the loop (waits, coordinates: warp-uniform values the compiler keeps in
    // uniform registers); one elected lane issues each copy.
    const bool issuer = elect_one();
    const bool do_a = kTmaA && warp == 4;
    const bool do_b = kTmaA ? warp == 10 : warp == 4;
    const bool skipA = a.dbg & 1, skipB = a.dbg & 2;
    if (issuer) {
      if (do_b && !a.wsw) tma_prefetch_desc(WM);
      if (do_a) tma_prefetch_desc(AM);
      if (do_a && a.ds) tma_prefetch_desc(RM);
    }
    const bool loadB = do_b && !skipB && !bres;  // bres: the weights were loaded once, below
    const uint32_t tx = (do_a && !skipA ? a_tile : 0u) + (loadB ? b_bytes : 0u);
    if (do_b && bres && issuer) {
      // every tile of this CTA has the same N tile (planned so): its num_kb weight k-blocks, and
      // with res_mma the 64x64 identity block (rows 0..63 of identity k-block num_kb), once
      const int n_fix = blockIdx.x % a.n_tiles;
      mbar_arrive_expect_tx(sp.bresbar, bres_alloc(1, a.num_kb, BN, a.res_mma));
      for (int kb = 0; kb < a.num_kb; ++kb)
        bulk_load(sp.sBres + static_cast<size_t>(kb) * b_bytes,
                  a.wsw + (static_cast<size_t>(kb) * a.Cout + static_cast<size_t>(n_fix) * BN) * 128u, b_bytes,
                  sp.bresbar);
      if (a.res_mma) bulk_load(sp.sIdent, a.wsw + static_cast<size_t>(a.num_kb) * a.Cout * 128u, 8192u, sp.bresbar);
    }
    const int cpl = a.cpl;
    const int nl = kBK / cpl;
    const uint32_t region = static_cast<uint32_t>(kBM * cpl * 2);
    int st = 0, it = 0;
    uint32_t ph = 0;
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
      const int m_blk = tile / a.n_tiles;
      const int n_blk = tile % a.n_tiles;
      int wc = 0, hc = 0, nimg = 0;
      if (do_a) {
        const int m0 = m_blk * kBM;
        nimg = m0 / HoWo;
        const int rem = m0 - nimg * HoWo;
        const int ho0 = rem / a.Wo;
        wc = (rem - ho0 * a.Wo) * a.sw - a.pw;
        hc = ho0 * a.sh - a.ph;
      }
      // (filter row r, filter col s, channel block c0) of the next im2col load; K is ordered
      // (r, s, c).  Loads past the last tap (K padding) read real pixels, but the matching
      // packed weights are zero, so they contribute nothing.
      int c0 = 0, r = 0, s = 0;
      const uint8_t* wsrc = a.wsw ? a.wsw + static_cast<size_t>(n_blk) * BN * 128u : nullptr;
      for (int kb0 = 0; kb0 < nkb_tile; kb0 += KPS, ++it) {
        pipe_wait(&sp.empty[st], ph ^ 1, issuer);
        if (issuer && warp == 4 && a.trace && blockIdx.x == 0 && it < 8192) a.trace[it * 4 + 0] = clock64();
        const int nk = min(KPS, nkb_tile - kb0);
        if (issuer) {
          if (tx)
            mbar_arrive_expect_tx(&sp.full[st], tx * nk);
          else
            mbar_arrive(&sp.full[st]);
        }
        for (int j = 0; j < nk; ++j) {
        const int kb = kb0 + j;
        uint8_t* const sa = sp.sA + st * sa_bytes + j * a_tile;
        uint8_t* const sb = sp.sB + static_cast<size_t>(st) * sb_bytes + j * b_bytes;
        if (do_a && kb >= a.num_kb) {
          // residual x identity block: A = residual columns [nb0 + 64*(kb - num_kb), +64)
          if (issuer && !skipA) tma_load_2d(sa, RM, &sp.full[st], n_blk * BN + (kb - a.num_kb) * 64, m_blk * kBM);
        } else if (do_a) {
          if (a.ds && kb >= a.kb_split) {
            // fused downsample (GX_OPF_DS): these k-blocks are the block input's channels at the
            // output pixels (2D map at stride 1, 1x1 im2col map at the downsample stride)
            const int cds = (kb - a.kb_split) * kBK;
            if (issuer && !skipA) {
              if (a.ds_stride == 1)
                tma_load_2d(sa, RM, &sp.full[st], cds, m_blk * kBM);
              else
                tma_load_im2col_4d(sa, RM, &sp.full[st], cds, wc * a.ds_stride, hc * a.ds_stride, nimg, 0, 0);
            }
          } else if (a.a2d) {
            // 1x1 / stride 1 / no padding: A is the plain [M, C] activation matrix
            if (issuer && !skipA) tma_load_2d(sa, AM, &sp.full[st], kb * kBK, m_blk * kBM);
          } else {
            for (int l = 0; l < nl; ++l) {
              if (issuer && !skipA)
                tma_load_im2col_4d(sa + l * region, AM, &sp.full[st], c0, wc, hc, nimg, static_cast<uint16_t>(s),
                                   static_cast<uint16_t>(r));
              c0 += cpl;
              if (c0 == a.Cin) {
                c0 = 0;
                if (++s == a.S) {
                  s = 0;
                  ++r;
                }
              }
            }
          }
        }
        if (loadB && issuer) {
          // identity blocks sit at kb = num_kb + column/64: this tile's are num_kb + nb0/64 + j
          const int kbw = kb < a.num_kb ? kb : kb + n_blk * BN / 64;
          if (wsrc)  // pre-swizzled tile: one contiguous bulk copy (no tensor-map walk)
            bulk_load(sb, wsrc + static_cast<size_t>(kbw) * a.Cout * 128u, b_bytes, &sp.full[st]);
          else
            tma_load_2d(sb, WM, &sp.full[st], kb * kBK, n_blk * BN);
        }
        }
        __syncwarp();
        if (++st == S_) {
          st = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer (warp-uniform loop)
    const bool issuer = elect_one();
    int it = 0, t = 0, st = 0;
    uint32_t ph = 0;
    if (bres) {  // resident weights (completed phase 0 once, never re-armed)
      pipe_wait(sp.bresbar, 0, issuer);
      tc_fence_after();
    }
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++t) {
      const int acc = t & 1;
      const uint32_t aph = (t >> 1) & 1;
      pipe_wait(&sp.tempty[acc], aph ^ 1, issuer);
      if (issuer && a.trace && blockIdx.x == 0 && t < 4096) a.trace[8 * 8192 + t] = clock64();
      tc_fence_after();
      const uint32_t d = tmem_base + acc * acc_stride;
      for (int kb0 = 0; kb0 < nkb_tile; kb0 += KPS, ++it, st = (st + 1 == S_) ? 0 : st + 1, ph ^= (st == 0)) {
        pipe_wait(&sp.full[st], ph, issuer);
        if (issuer && a.trace && blockIdx.x == 0 && it < 8192) a.trace[it * 4 + 1] = clock64();
        tc_fence_after();
        if (a.dbg & 4) {
          if (issuer) umma_commit(&sp.empty[st]);
          __syncwarp();
          continue;
        }
        const int nk = min(KPS, nkb_tile - kb0);
        for (int jj = 0; jj < nk; ++jj) {
        const int kb = kb0 + jj;
        const uint32_t abase = smem_u32(sp.sA + st * sa_bytes + jj * a_tile);
        const uint64_t bd = bres ? umma_desc_sw128(sp.sBres + static_cast<size_t>(min(kb, a.num_kb - 1)) * b_bytes)
                                 : umma_desc_sw128(sp.sB + static_cast<size_t>(st) * sb_bytes + jj * b_bytes);
        if (bres && kb >= a.num_kb) {
          // residual columns [64j, 64j+64) x identity: four M=128 N=64 K=16 MMAs into that 64-column
          // slice of the accumulator (a quarter of the work of a full-width identity k-block, and
          // no identity weights streamed per tile)
          const uint32_t dj = d + 64u * static_cast<uint32_t>(kb - a.num_kb);
          const uint64_t ad = umma_desc_kmajor(abase, 64, 0);
          const uint64_t idd = umma_desc_sw128(sp.sIdent);
          if (issuer) {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) umma_bf16(dj, ad + 2 * kk, idd + 2 * kk, a.idesc64, 1);
          }
        } else if (!kTmaA || a.cpl == 64) {
          const uint64_t ad = umma_desc_kmajor(abase, 64, 0);
          if (issuer) {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) umma_bf16(d, ad + 2 * kk, bd + 2 * kk, a.idesc, (kb | kk) != 0);
          }
        } else {
          // A stage = 64/cpl regions of 128 rows x cpl channels; MMA kk covers K [16kk, 16kk+16)
          const uint32_t region = static_cast<uint32_t>(kBM * a.cpl * 2);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const int e0 = kk * 16;
            const uint32_t addr = abase + (e0 / a.cpl) * region + (e0 % a.cpl) * 2;
            const uint64_t adk = umma_desc_kmajor(addr, a.cpl, region);
            if (issuer) umma_bf16(d, adk, bd + 2 * kk, a.idesc, (kb | kk) != 0);
          }
        }
        }
        if (issuer) {
          umma_commit(&sp.empty[st]);
          if (a.trace && blockIdx.x == 0 && it < 8192) a.trace[it * 4 + 2] = clock64();
        }
        __syncwarp();
      }
      if (issuer) umma_commit(&sp.tfull[acc]);
      __syncwarp();
    }
  } else if ((warp >= 6 && warp <= 9) || (kTmaA && warp < 4)) {
    // ------------------------------------------------------------ epilogue
    // warps 6-9, plus warps 0-3 when TMA builds A (they have no producer work): two warps per
    // TMEM lane quarter split the tile's 16-column chunks, two tcgen05.ld in flight per wait
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    const int nepi = kTmaA ? 256 : 128;
    const int half = (kTmaA && warp < 4) ? 1 : 0;
    // column split between the two warps of a lane quarter: contiguous halves with per-warp stores
    // (each warp owns whole 64-column groups and stores them itself), else interleaved 16-column
    // chunks (measured 7% faster for the residual epilogue)
    const bool halves = kTmaA && WST;
    const int cbase = !kTmaA ? 0 : halves ? half * (BN / 2) : half * 16;
    const int cstep = (!kTmaA || halves) ? 16 : 32;
    const int cend = halves ? cbase + BN / 2 : BN;
    // per-warp TMA stores (no residual): a warp overwrites only the smem rows/columns it stored
    // itself, so no cross-warp barrier is needed around the output staging slot
    constexpr bool wstore = WST;  // compile-time: the residual / shared-store paths keep their code
    const bool wissuer = wstore && elect_one();
    const bool leader = warp == 6 && lane == 0;
    const int nres = a.nres;
    const int nslot = (has_res || ystore) ? nres : 1;
    // residual tile of the t-th tile this CTA processes -> slot t % nres
    auto issue_res = [&](int t_idx) {
      const int tile = blockIdx.x + t_idx * gridDim.x;
      if (tile >= a.num_tiles) return;
      const int slot = t_idx % nres;
      mbar_arrive_expect_tx(&sp.rfull[slot], res_slot_bytes);
      for (int g = 0; g < res_groups(BN); ++g)
        tma_load_2d(sp.sRes + slot * res_slot_bytes + g * kResGroupBytes, RM, &sp.rfull[slot],
                    (tile % a.n_tiles) * BN + g * 64, (tile / a.n_tiles) * kBM);
    };
    // WST + residual: each epilogue warp TMA-loads its own 32-row x (BN/2)-column residual box
    const int ew = warp >= 6 ? warp - 6 : 4 + warp;  // epilogue warp index 0..7
    auto issue_res_w = [&](int t_idx) {
      const int tile = blockIdx.x + t_idx * gridDim.x;
      if (tile >= a.num_tiles) return;
      const int slot = t_idx % nres;
      uint64_t* bar = &sp.rfw[ew * 2 + slot];
      mbar_arrive_expect_tx(bar, static_cast<uint32_t>((cend - cbase) / 64) * 32u * 128u);
      for (int g = cbase / 64; g < cend / 64; ++g)
        tma_load_2d(sp.sRes + slot * res_slot_bytes + g * kResGroupBytes + q * 32 * 128, RM, bar,
                    (tile % a.n_tiles) * BN + g * 64, (tile / a.n_tiles) * kBM + q * 32);
    };
    if (leader) {
      // the whole bias vector once per CTA; residual tiles run ahead by `nres` tiles
      mbar_arrive_expect_tx(sp.bfull, static_cast<uint32_t>(a.Cout) * 4u);
      bulk_load(sp.sBias, a.bias, static_cast<uint32_t>(a.Cout) * 4u, sp.bfull);
      if (has_res && !WST) {
        tma_prefetch_desc(RM);
        for (int i = 0; i < nres; ++i) issue_res(i);
      }
    }
    if (WST && has_res) {
      if (wissuer)
        for (int i = 0; i < nres; ++i) issue_res_w(i);
      __syncwarp();
    }
    epi_wait(sp.bfull, 0);
    int t = 0;
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++t) {
      const int m_blk = tile / a.n_tiles;
      const int n_blk = tile % a.n_tiles;
      const int m0 = m_blk * kBM;
      const int nb0 = n_blk * BN;
      const int ncols = min(BN, a.Cout - nb0);
      const int slot = t % nslot;
      const uint32_t bias_s = smem_u32(sp.sBias + nb0);
      const uint8_t* res_base = sp.sRes + slot * res_slot_bytes;
      const int acc = t & 1;
      const uint32_t aph = (t >> 1) & 1;
      epi_wait(&sp.tfull[acc], aph);
      const bool tr = a.trace && leader && blockIdx.x == 0 && t < 4096;
      if (tr) a.trace[4 * 8192 + t * 4 + 0] = clock64();
      tc_fence_after();
      if (WST && has_res) {
        epi_wait(&sp.rfw[ew * 2 + slot], (t / nres) & 1);
      } else if (has_res) {
        epi_wait(&sp.rfull[slot], (t / nres) & 1);
      } else if (wstore) {
        // this warp's own previous store from this slot has finished reading it
        if (wissuer) {
          if (nres == 1)
            bulk_wait_read<0>();
          else
            bulk_wait_read<1>();
        }
        __syncwarp();
      } else if (ystore) {
        // the TMA store that last used this slot (tile t - nres) has finished reading it
        if (leader) {
          if (nres == 1)
            bulk_wait_read<0>();
          else
            bulk_wait_read<1>();
        }
        named_bar_sync(1, nepi);
      }
      const int m = m0 + row;
      const bool row_ok = m < a.M;
      const uint32_t tbase = tmem_base + acc * acc_stride + (static_cast<uint32_t>(q * 32) << 16);
      auto emit = [&](const int c, const uint32_t (&v)[16]) {
        if ((row_ok || ystore) && c < ncols) {
          const int n0 = nb0 + c;
          float f[16];
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {  // bias: 4 x ld.shared.v4 (a generic pointer made 16 LD.E)
            const float4 bb = lds_f4(bias_s + static_cast<uint32_t>(c + 4 * q4) * 4u);
            f[4 * q4 + 0] = __uint_as_float(v[4 * q4 + 0]) + bb.x;
            f[4 * q4 + 1] = __uint_as_float(v[4 * q4 + 1]) + bb.y;
            f[4 * q4 + 2] = __uint_as_float(v[4 * q4 + 2]) + bb.z;
            f[4 * q4 + 3] = __uint_as_float(v[4 * q4 + 3]) + bb.w;
          }
          if (has_res) {
            const uint8_t* rrow = res_base + (c >> 6) * kResGroupBytes + row * 128;
            const int j0 = (c & 63) >> 3;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const uint4 rr = *reinterpret_cast<const uint4*>(rrow + (((j0 + i) ^ (row & 7)) << 4));
              const uint32_t w[4] = {rr.x, rr.y, rr.z, rr.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float2 p = unpack_bf16x2(w[j]);
                f[8 * i + 2 * j] += p.x;
                f[8 * i + 2 * j + 1] += p.y;
              }
            }
          }
          if (a.act == GX_ACT_RELU) {
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = fmaxf(f[i], 0.0f);
          } else if (a.act == GX_ACT_GELU) {
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = gelu_erf(f[i]);
          }
          if (ystore) {
            // back into the slot, same swizzled position the residual came from
            uint8_t* srow = const_cast<uint8_t*>(res_base) + (c >> 6) * kResGroupBytes + row * 128;
            const int j0 = (c & 63) >> 3;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              uint4 o;
              o.x = pack_bf16x2(f[8 * i + 0], f[8 * i + 1]);
              o.y = pack_bf16x2(f[8 * i + 2], f[8 * i + 3]);
              o.z = pack_bf16x2(f[8 * i + 4], f[8 * i + 5]);
              o.w = pack_bf16x2(f[8 * i + 6], f[8 * i + 7]);
              *reinterpret_cast<uint4*>(srow + (((j0 + i) ^ (row & 7)) << 4)) = o;
            }
          } else if (a.y_f32) {
            float4* y4 = reinterpret_cast<float4*>(static_cast<float*>(a.y) + static_cast<size_t>(m) * a.y_ld +
                                                   a.y_coff + n0);
#pragma unroll
            for (int i = 0; i < 4; ++i)  // Cout % 4 tails (FC 1000)
              if (c + 4 * i < ncols) y4[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
          } else {
            uint4* y4 = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.y) + static_cast<size_t>(m) * a.y_ld +
                                                 a.y_coff + n0);
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              uint4 o;
              o.x = pack_bf16x2(f[8 * i + 0], f[8 * i + 1]);
              o.y = pack_bf16x2(f[8 * i + 2], f[8 * i + 3]);
              o.z = pack_bf16x2(f[8 * i + 4], f[8 * i + 5]);
              o.w = pack_bf16x2(f[8 * i + 6], f[8 * i + 7]);
              if (c + 8 * i < ncols) y4[i] = o;
            }
          }
        }
      };
      // this warp's 16-column chunks: c_j = half*16 + j*cstep.  Software-pipelined: the TMEM load
      // of chunk j+1 is in flight while chunk j is converted and stored (tcgen05.wait::ld waits
      // for all of the warp's loads, so the next load is issued before the math, waited after).
      const int nch = (a.dbg & 8) ? 0 : (cend - cbase + cstep - 1) / cstep;
      if (nch > 0) {
        uint32_t va[16], vb[16];
        tmem_ld16(tbase + cbase, va);
        tmem_ld_wait();
        for (int j = 0; j < nch; j += 2) {
          const int ca = cbase + j * cstep, cb = ca + cstep;
          if (j + 1 < nch) tmem_ld16(tbase + cb, vb);
          emit(ca, va);
          tmem_ld_wait();
          if (j + 1 >= nch) break;
          if (j + 2 < nch) tmem_ld16(tbase + cb + cstep, va);
          emit(cb, vb);
          tmem_ld_wait();
        }
      }
      if (tr) a.trace[4 * 8192 + t * 4 + 1] = clock64();
      // one arrival per warp: 256 same-word smem arrives serialise (~2k cycles per tile, measured)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sp.tempty[acc]);
      if (wstore) {
        fence_proxy_async_smem();
        __syncwarp();
        if (wissuer) {
          for (int g = cbase / 64; g < cend / 64; ++g)
            if (g * 64 < ncols)
              tma_store_2d(YM, res_base + g * kResGroupBytes + q * 32 * 128, a.y_coff + nb0 + g * 64, m0 + q * 32);
          bulk_commit();
          if (has_res) {
            bulk_wait_read<0>();  // this warp's region is refilled with its next residual box
            issue_res_w(t + nres);
          }
        }
        __syncwarp();
      } else if (ystore) {
        fence_proxy_async_smem();  // make the slot's generic-proxy writes visible to the TMA store
        named_bar_sync(1, nepi);
        if (leader) {
          for (int g = 0; g < (ncols + 63) / 64; ++g)
            tma_store_2d(YM, res_base + g * kResGroupBytes, a.y_coff + nb0 + g * 64, m0);
          bulk_commit();
          if (has_res) {
            bulk_wait_read<0>();  // the slot is refilled by the next residual load
            issue_res(t + nres);
          }
          if (tr) a.trace[4 * 8192 + t * 4 + 2] = clock64();
        }
      } else if (has_res) {
        named_bar_sync(1, nepi);  // every epilogue thread is done with this residual slot
        if (leader) issue_res(t + nres);
      }
    }
  }
  if (ystore && !WST && warp == 6 && lane == 0) bulk_wait<0>();  // output stores complete before exit
  if (WST && ((warp >= 6 && warp <= 9) || (kTmaA && warp < 4))) {
    if (elect_one()) bulk_wait<0>();
    __syncwarp();
  }
  // Let the next kernel in the stream start its prologue.
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem_base, a.tmem_cols);
  }
}
}  // namespace

size_t conv_smem_bytes(int BN, int stages, int num_kb, int nres, int Cout, int kps, size_t bres_bytes, int a_rows) {
  const size_t a_tile = static_cast<size_t>(a_rows) * 128;
  return 1024 + static_cast<size_t>(stages) * kps * (a_tile + (bres_bytes ? 0 : BN * 128)) + (kATileBytes - a_tile) +
         bres_bytes +
         static_cast<size_t>(nres) * res_groups(BN) * kResGroupBytes + bias_alloc(Cout) + (2 * stages + 26) * 8 + 16 +
         static_cast<size_t>(num_kb) * 8 * sizeof(int2);
}

// Pipeline depth and residual slots that fit in ~220 KB: prefer >= 3 stages with a double-
// buffered residual, else a single residual slot.
int conv_pick_stages(int BN, int num_kb, bool res, int Cout, int* nres_out, int kps, size_t bres_bytes, int a_rows) {
  const size_t budget = 220 * 1024;
  const size_t per_stage = static_cast<size_t>(kps) * (static_cast<size_t>(a_rows) * 128 + (bres_bytes ? 0 : BN * 128)) +
                           16;
  int best_s = 2, best_r = res ? 1 : 0;
  for (int nres = res ? 2 : 0; nres >= (res ? 1 : 0); --nres) {
    const size_t fixed = conv_smem_bytes(BN, 0, num_kb, nres, Cout, kps, bres_bytes, a_rows);
    int s = budget > fixed ? static_cast<int>((budget - fixed) / per_stage) : 0;
    const int cap = a_rows < kBM ? kMaxStages : 8;  // short A tiles: weight streaming wants depth
    if (s > cap) s = cap;
    // short-K convs (the bottleneck expand 1x1s) are epilogue-bound: with the per-warp epilogue the next tile's residual/staging slot must be free while this
    // tile's epilogue runs; for K <= 128 one operand stage keeps the MMA ahead of the epilogue
    const int kb_short = dev().res2_kb;  // measured neutral: off
    if (s >= 3 || nres <= 1 || (s >= 1 && num_kb <= kb_short)) {
      best_s = s < 1 ? 1 : (s < 2 && num_kb > kb_short) ? 2 : s;
      best_r = nres;
      break;
    }
  }
  *nres_out = best_r;
  return best_s;
}

cudaError_t launch_conv(const CUtensorMap& wmap, const CUtensorMap& amap, const CUtensorMap& rmap,
                        const CUtensorMap& ymap, const ConvArgs& a, int grid, cudaStream_t s, bool pdl) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaSuccess;
    for (auto fn : {conv_tc_kernel<true, 1, false>, conv_tc_kernel<true, 2, false>, conv_tc_kernel<true, 3, false>,
                    conv_tc_kernel<false, 1, false>, conv_tc_kernel<true, 1, true>, conv_tc_kernel<true, 2, true>,
                    conv_tc_kernel<true, 3, true>})
      if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kConvTcThreads, 1, 1);
  cfg.dynamicSmemBytes = conv_smem_bytes(a.BN, a.stages, a.num_kb, a.nres, a.Cout, a.kps,
                                         bres_alloc(a.bres, a.num_kb, a.BN, a.res_mma), a.a_rows);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (a.tma_a && a.wstore)
    return a.kps == 3   ? cudaLaunchKernelEx(&cfg, conv_tc_kernel<true, 3, true>, wmap, amap, rmap, ymap, a)
           : a.kps == 2 ? cudaLaunchKernelEx(&cfg, conv_tc_kernel<true, 2, true>, wmap, amap, rmap, ymap, a)
                        : cudaLaunchKernelEx(&cfg, conv_tc_kernel<true, 1, true>, wmap, amap, rmap, ymap, a);
  if (a.tma_a && a.kps == 3) return cudaLaunchKernelEx(&cfg, conv_tc_kernel<true, 3, false>, wmap, amap, rmap, ymap, a);
  if (a.tma_a && a.kps == 2) return cudaLaunchKernelEx(&cfg, conv_tc_kernel<true, 2, false>, wmap, amap, rmap, ymap, a);
  if (a.tma_a) return cudaLaunchKernelEx(&cfg, conv_tc_kernel<true, 1, false>, wmap, amap, rmap, ymap, a);
  return cudaLaunchKernelEx(&cfg, conv_tc_kernel<false, 1, false>, wmap, amap, rmap, ymap, a);
}

}  // namespace gx
