// K2 variant for 3x3 / stride-1 / pad-1 convolutions on wide images (ResNet layer1/layer2): the
// A operand comes from ONE halo tile per 64-channel block instead of one im2col load per filter tap.
//
// An M tile covers BH whole output rows of one image laid out with a padded pitch Wp = W + 2:
// virtual row u = i*Wp + j (i < BH output row, j < Wp; j >= W is a discarded column).  The halo
// is the input rows h0-1 .. h0+BH, columns -1 .. W, fetched by one 4D tiled TMA with zero fill
// for the padding, stored as [(BH+2)*Wp pixels][64 channels] with the 128-byte swizzle.  Tap
// (r, s) of virtual row u reads halo pixel u + r*Wp + s, so the A operand of tap (r, s) is the
// halo itself started (r*Wp + s) rows later: the nine MMAs of a channel block read one smem tile
// at nine row offsets, and each input pixel crosses L2->SM
// once per M tile instead of nine times.
//
// Images wider than a tile (Inception's 147x147 stem convs) are cut into column tiles: an M tile is
// BH output rows x WT output columns of one image, its halo (BH + R - 1) x (WT + S - 1) input pixels
// with pitch Wp = WT + S - 1, and the same row-offset trick holds inside the tile.  RB = 64: the
// 32-channel inputs (SWIZZLE_64B rows), two taps per weight k-block, two K=16 MMAs per tap.
//
// Roles (352 threads): warp 4 halo producer, warp 10 weight producer (bulk copies of the
// pre-swizzled [kb][Cout][64] tiles, kb = tap*Cin/64 + cb), one elected lane of warp 5 issues the
// MMAs, warps 0-3 and 6-9 run the epilogue (bias, ReLU, bf16, row-remapped stores).
#include <cuda_bf16.h>

#include "gx_internal.h"
#include "gx_ptx.cuh"

namespace gx {

namespace {
constexpr int kHaloRows = 256;                  // smem rows per halo buffer (>= 128 + 2*Wp + 2)
constexpr int kHaloBytes = kHaloRows * 128;     // 32 KB

struct HaloSmem {
  uint8_t* halo;   // [NH][HB]: 2 x 32 KB (128-byte rows) or 4 x 16 KB (32-byte rows)
  uint8_t* sB;     // [S][BN*128]
  float* bias;
  uint64_t *hfull, *hempty, *bfull, *bempty, *tfull, *tempty, *biasbar;
  uint32_t* tslot;
};

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// K-major SW128 descriptor whose start may sit at any 128-byte row of a 1024-aligned atom: the
// tensor core applies the 128-byte swizzle on absolute shared-memory address bits (as the TMA
// wrote it), so the base-offset field stays 0 (measured: setting it to (addr >> 7) & 7 breaks
// every tap but (0, 0); scripts/debug_halo.py).
__device__ __forceinline__ uint64_t desc_sw128_row(uint32_t saddr) {
  return ((static_cast<uint64_t>(saddr) >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}

// RB = bytes per halo pixel row: 128 (64-channel blocks, SWIZZLE_128B, 3x3 taps, four K=16 MMAs per
// tap) or 32 (the 16-channel s2d stem, SWIZZLE_32B, 4x4 taps, one K=16 MMA per tap; the four taps
// of filter row r are the four 32-byte K slices of weight k-block r)
template <int RB>
__global__ void __launch_bounds__(kConvTcThreads, 1)
    conv_halo_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap hmap,
                     const ConvArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S_ = a.stages;
  const int BN = a.BN;
  const uint32_t b_bytes = static_cast<uint32_t>(BN) * 128u;
  const int Wp = a.hWp, BH = a.hBH, TPI = a.hTPI, WT = a.hWT, CT = a.hCT;
  const int CB = RB == 128 ? a.Cin / 64 : 1;
  // weight k-blocks per channel block: one per tap (128-byte rows), per filter row (the 32-byte
  // s2d stem), per pair of taps (64-byte rows: 32 channels)
  const int NKB = RB == 128 ? 9 : RB == 32 ? a.R : (a.R * a.S + 1) / 2;
  const uint32_t hbytes = static_cast<uint32_t>(Wp * (BH + a.R - 1) * RB);
  // one N tile and one channel block (the stem; layer1's 56x56x64 3x3): the NKB weight k-blocks
  // are loaded once into ring slots 0..NKB-1 and stay resident.  Every tile would otherwise
  // re-load the same weights: 32 KB per stem tile (60% of its TMA bytes), 72 KB per layer1 tile
  // (2.4x its halo bytes) through a few-SM budget's L2 feed.
  const bool resident = a.n_tiles == 1 && S_ >= NKB && CB == 1 && !(a.dbg & 32);  // GX_CONV_DBG=32: ring as before
  // the stem's halo is ~15 KB and one tile's MMAs take ~0.3 us: four buffers keep enough TMA loads
  // in flight to cover their latency
  constexpr int NH = RB == 128 ? 2 : 4;
  constexpr uint32_t HB = 2u * kHaloBytes / NH;
  HaloSmem sp;
  sp.halo = smem;
  sp.sB = sp.halo + 2 * kHaloBytes;
  sp.bias = reinterpret_cast<float*>(sp.sB + static_cast<size_t>(S_) * b_bytes);
  sp.hfull = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sp.bias) + ((a.Cout * 4 + 1023) & ~1023));
  sp.hempty = sp.hfull + NH;
  sp.bfull = sp.hempty + NH;
  sp.bempty = sp.bfull + S_;
  sp.tfull = sp.bempty + S_;
  sp.tempty = sp.tfull + 2;
  sp.biasbar = sp.tempty + 2;
  sp.tslot = reinterpret_cast<uint32_t*>(sp.biasbar + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 4) {
    if (lane == 0) {
      for (int i = 0; i < NH; ++i) {
        mbar_init(&sp.hfull[i], 1);
        mbar_init(&sp.hempty[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&sp.tfull[i], 1);
        mbar_init(&sp.tempty[i], 8);  // one arrival per epilogue warp
      }
      for (int i = 0; i < S_; ++i) {
        mbar_init(&sp.bfull[i], 1);
        mbar_init(&sp.bempty[i], 1);
      }
      mbar_init(sp.biasbar, 1);
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
  pdl_wait();

  if (warp == 4) {
    // ------------------------------------------------------------ halo producer
    const bool issuer = elect_one();
    if (issuer) tma_prefetch_desc(&hmap);
    int hs = 0;
    uint32_t hph = 0;
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
      const int m_blk = tile / a.n_tiles;
      const int n = m_blk / (TPI * CT), rc = m_blk % (TPI * CT);
      const int h0 = (rc / CT) * BH, c0 = (rc % CT) * WT;
      for (int cb = 0; cb < CB; ++cb) {
        mbar_wait(&sp.hempty[hs], hph ^ 1);
        if (issuer) {
          mbar_arrive_expect_tx(&sp.hfull[hs], hbytes);
          tma_load_4d(sp.halo + hs * HB, &hmap, &sp.hfull[hs], cb * 64, c0 - a.pw, h0 - a.ph, n);
        }
        __syncwarp();
        if (++hs == NH) {
          hs = 0;
          hph ^= 1;
        }
      }
    }
  } else if (warp == 10) {
    // ------------------------------------------------------------ weight producer
    const bool issuer = elect_one();
    if (issuer && !a.wsw) tma_prefetch_desc(&wmap);
    int bs = 0;
    uint32_t bph = 0;
    if (resident) {
      if (issuer)
        for (int kb = 0; kb < NKB; ++kb) {
          uint8_t* dst = sp.sB + static_cast<size_t>(kb) * b_bytes;
          mbar_arrive_expect_tx(&sp.bfull[kb], b_bytes);
          if (a.wsw)
            bulk_load(dst, a.wsw + static_cast<size_t>(kb) * a.Cout * 128u, b_bytes, &sp.bfull[kb]);
          else
            tma_load_2d(dst, &wmap, &sp.bfull[kb], kb * kBK, 0);
        }
      __syncwarp();
    }
    for (int tile = resident ? a.num_tiles : blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
      const int n_blk = tile % a.n_tiles;
      for (int cb = 0; cb < CB; ++cb) {
        for (int tap = 0; tap < NKB; ++tap) {
          const int kb = tap * CB + cb;
          mbar_wait(&sp.bempty[bs], bph ^ 1);
          if (issuer) {
            uint8_t* dst = sp.sB + static_cast<size_t>(bs) * b_bytes;
            mbar_arrive_expect_tx(&sp.bfull[bs], b_bytes);
            if (a.wsw)
              bulk_load(dst, a.wsw + (static_cast<size_t>(kb) * a.Cout + static_cast<size_t>(n_blk) * BN) * 128u,
                        b_bytes, &sp.bfull[bs]);
            else
              tma_load_2d(dst, &wmap, &sp.bfull[bs], kb * kBK, n_blk * BN);
          }
          __syncwarp();
          if (++bs == S_) {
            bs = 0;
            bph ^= 1;
          }
        }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    const bool issuer = elect_one();
    int hs = 0, bs = 0, t = 0;
    uint32_t hph = 0, bph = 0;
    // descriptor bases: a tap's A / B descriptor is the base plus a 16-byte-unit offset (the start
    // field is addr >> 4 in 14 bits, smem < 256 KB, so the add never carries out of it)
    const uint64_t b0 = umma_desc_sw128(sp.sB);
    const uint32_t b_step = b_bytes >> 4, row_step = static_cast<uint32_t>(Wp) * 8u;
    if (resident) {
      // resident weights: each slot completed phase 0 once and is never re-armed, so the NKB waits
      // happen once here instead of once per tap of every tile
      for (int tap = 0; tap < NKB; ++tap) mbar_wait(&sp.bfull[tap], 0u);
      tc_fence_after();
    }
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++t) {
      const int acc = t & 1;
      mbar_wait(&sp.tempty[acc], ((t >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + acc * acc_stride;
      for (int cb = 0; cb < CB; ++cb) {
        mbar_wait(&sp.hfull[hs], hph);
        tc_fence_after();
        const uint32_t hbase = smem_u32(sp.halo + hs * HB);
        if (RB == 128 && resident) {
          // resident weights: the nine taps unrolled with (r, s) compile-time, each descriptor one
          // 64-bit add and no barrier between taps, so the issuing thread keeps the tensor pipe fed
          // (scripts/native/mma_probe.cu: back-to-back M128 N64 K16 MMAs run at 48 cycles; the
          // rolled loop's per-tap division, R2UR moves and barrier wait cost ~115 per MMA).  Layer1's
          // 56x56x64 3x3: 440 -> 284 us at k=16 on 2 SMs.  (Unrolling the weight-ring case as well
          // measured slower: 28x28x128 3x3 286 -> 349 us; it keeps the rolled loop below.)
          const uint64_t a0 = desc_sw128_row(hbase);
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const int r = tap / 3, s = tap - r * 3;
            const uint64_t bd = b0 + static_cast<uint64_t>(static_cast<uint32_t>(tap) * b_step);
            const uint64_t ad = a0 + static_cast<uint64_t>(static_cast<uint32_t>(r) * row_step + s * 8u);
            if (issuer) {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) umma_bf16(d, ad + 2 * kk, bd + 2 * kk, a.idesc, (cb | tap | kk) != 0);
            }
          }
        } else if (RB == 32 && resident) {
          // the s2d stem (4x4 taps over 32-byte rows), same unrolled issue: k-block r holds filter
          // row r, its four 32-byte K slices are taps (r, 0..3)
          const uint64_t a0 = umma_desc_kmajor(hbase, 16, 0);
#pragma unroll
          for (int tap = 0; tap < 4; ++tap) {
            const uint64_t bd = b0 + static_cast<uint64_t>(static_cast<uint32_t>(tap) * b_step);
            if (issuer) {
#pragma unroll
              for (int s = 0; s < 4; ++s)
                umma_bf16(d, a0 + static_cast<uint64_t>((static_cast<uint32_t>(tap) * Wp + s) * 2u), bd + 2 * s,
                          a.idesc, (tap | s) != 0);
            }
          }
        } else if (RB == 64 && resident) {
          // 32-channel 3x3 (64-byte rows): k-block kb holds taps 2kb and 2kb + 1, two K=16 MMAs each
          const uint64_t a0 = umma_desc_kmajor(hbase, 32, 0);
#pragma unroll
          for (int t9 = 0; t9 < 9; ++t9) {
            const int r = t9 / 3, s = t9 - r * 3, kb = t9 / 2, h = t9 & 1;
            const uint64_t bd = b0 + static_cast<uint64_t>(static_cast<uint32_t>(kb) * b_step);
            const uint64_t ad = a0 + static_cast<uint64_t>((static_cast<uint32_t>(r) * Wp + s) * 4u);
            if (issuer) {
#pragma unroll
              for (int kk = 0; kk < 2; ++kk) umma_bf16(d, ad + 2 * kk, bd + 2 * (2 * h + kk), a.idesc, (t9 | kk) != 0);
            }
          }
        } else
        for (int tap = 0; tap < NKB; ++tap) {
          const int slot = resident ? tap : bs;
          // resident slots completed phase 0 once and are never re-armed: parity-0 waits pass
          mbar_wait(&sp.bfull[slot], resident ? 0u : bph);
          tc_fence_after();
          const uint64_t bd = umma_desc_sw128(sp.sB + static_cast<size_t>(slot) * b_bytes);
          if (RB == 128) {
            const int r = tap / 3, s = tap - r * 3;
            const uint64_t ad = desc_sw128_row(hbase + static_cast<uint32_t>(r * Wp + s) * 128u);
            if (issuer) {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                umma_bf16(d, ad + 2 * kk, bd + 2 * kk, a.idesc, (cb | tap | kk) != 0);
            }
          } else if (RB == 64) {
            // k-block `tap` holds taps 2*tap and 2*tap+1 (32 channels each): two K=16 MMAs per tap,
            // A = the halo started r*Wp + s pixel rows later (64-byte rows, SWIZZLE_64B)
            if (issuer) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int t9 = 2 * tap + h;
                if (t9 >= a.R * a.S) break;
                const int r = t9 / a.S, s = t9 - r * a.S;
#pragma unroll
                for (int kk = 0; kk < 2; ++kk)
                  umma_bf16(d, umma_desc_kmajor(hbase + static_cast<uint32_t>(r * Wp + s) * 64u, 32, 0) + 2 * kk,
                            bd + 2 * (2 * h + kk), a.idesc, (tap | h | kk) != 0);
              }
            }
          } else if (issuer) {
            // k-block `tap` = filter row r; its K slice s (32 bytes) is tap (r, s), whose A operand
            // is the halo started r*Wp + s pixel rows later (SWIZZLE_32B on absolute address bits,
            // like the 128-byte case: base-offset field 0)
#pragma unroll
            for (int s = 0; s < 4; ++s)
              umma_bf16(d, umma_desc_kmajor(hbase + static_cast<uint32_t>(tap * Wp + s) * 32u, 16, 0), bd + 2 * s,
                        a.idesc, (tap | s) != 0);
          }
          if (!resident) {
            if (issuer) umma_commit(&sp.bempty[bs]);
            if (++bs == S_) {
              bs = 0;
              bph ^= 1;
            }
          }
          __syncwarp();
        }
        if (issuer) umma_commit(&sp.hempty[hs]);
        __syncwarp();
        if (++hs == NH) {
          hs = 0;
          hph ^= 1;
        }
      }
      if (issuer) umma_commit(&sp.tfull[acc]);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 0-3, 6-9)
    const int q = warp & 3;
    const int half = warp < 4 ? 1 : 0;
    const int row = q * 32 + lane;  // virtual row u of the tile
    const int i = row / Wp, j = row - (row / Wp) * Wp;  // output (h0 + i, c0 + j) of the tile
    if (warp == 6 && lane == 0) {
      mbar_arrive_expect_tx(sp.biasbar, static_cast<uint32_t>(a.Cout) * 4u);
      bulk_load(sp.bias, a.bias, static_cast<uint32_t>(a.Cout) * 4u, sp.biasbar);
    }
    mbar_wait_sleepy(sp.biasbar, 0);
    int t = 0;
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++t) {
      const int m_blk = tile / a.n_tiles, n_blk = tile % a.n_tiles;
      const int n = m_blk / (TPI * CT), rc = m_blk % (TPI * CT);
      const int h = (rc / CT) * BH + i, w = (rc % CT) * WT + j;
      const bool row_ok = i < BH && j < WT && h < a.Ho && w < a.Wo;
      const int nb0 = n_blk * BN;
      const int ncols = min(BN, a.Cout - nb0);
      const int acc = t & 1;
      mbar_wait_sleepy(&sp.tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * acc_stride + (static_cast<uint32_t>(q * 32) << 16);
      const uint32_t bias_s = smem_u32(sp.bias + nb0);
      __nv_bfloat16* yrow = static_cast<__nv_bfloat16*>(a.y) +
                            ((static_cast<size_t>(n) * a.Ho + h) * a.Wo + w) * a.y_ld + a.y_coff + nb0;
      for (int c = half * 16; c < BN; c += 32) {
        uint32_t v[16];
        tmem_ld16(tbase + c, v);
        tmem_ld_wait();
        if (row_ok && c < ncols) {
          float f[16];
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const float4 bb = lds_f4(bias_s + static_cast<uint32_t>(c + 4 * q4) * 4u);
            f[4 * q4 + 0] = __uint_as_float(v[4 * q4 + 0]) + bb.x;
            f[4 * q4 + 1] = __uint_as_float(v[4 * q4 + 1]) + bb.y;
            f[4 * q4 + 2] = __uint_as_float(v[4 * q4 + 2]) + bb.z;
            f[4 * q4 + 3] = __uint_as_float(v[4 * q4 + 3]) + bb.w;
          }
          if (a.act == GX_ACT_RELU) {
#pragma unroll
            for (int e = 0; e < 16; ++e) f[e] = fmaxf(f[e], 0.0f);
          }
          uint4* y4 = reinterpret_cast<uint4*>(yrow + c);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            uint4 o;
            o.x = pack_bf16x2(f[8 * e + 0], f[8 * e + 1]);
            o.y = pack_bf16x2(f[8 * e + 2], f[8 * e + 3]);
            o.z = pack_bf16x2(f[8 * e + 4], f[8 * e + 5]);
            o.w = pack_bf16x2(f[8 * e + 6], f[8 * e + 7]);
            y4[e] = o;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&sp.tempty[acc]);  // one arrival per warp
    }
  }
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem_base, a.tmem_cols);
  }
}
}  // namespace

size_t conv_halo_smem_bytes(int BN, int stages, int Cout) {
  return 1024 + 2 * static_cast<size_t>(kHaloBytes) + static_cast<size_t>(stages) * BN * 128 +
         ((static_cast<size_t>(Cout) * 4 + 1023) & ~size_t(1023)) + (2 * stages + 13) * 8 + 16;
}

int conv_halo_pick_stages(int BN, int Cout) {
  const size_t budget = 220 * 1024;
  const size_t fixed = conv_halo_smem_bytes(BN, 0, Cout);
  int s = budget > fixed ? static_cast<int>((budget - fixed) / (static_cast<size_t>(BN) * 128 + 16)) : 0;
  return s > 9 ? 9 : s;
}

cudaError_t launch_conv_halo(const CUtensorMap& wmap, const CUtensorMap& hmap, const ConvArgs& a, int grid,
                             cudaStream_t s, bool pdl) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(conv_halo_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(conv_halo_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(conv_halo_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kConvTcThreads, 1, 1);
  cfg.dynamicSmemBytes = conv_halo_smem_bytes(a.BN, a.stages, a.Cout);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (a.hRB == 32) return cudaLaunchKernelEx(&cfg, conv_halo_kernel<32>, wmap, hmap, a);
  if (a.hRB == 64) return cudaLaunchKernelEx(&cfg, conv_halo_kernel<64>, wmap, hmap, a);
  return cudaLaunchKernelEx(&cfg, conv_halo_kernel<128>, wmap, hmap, a);
}

}  // namespace gx
