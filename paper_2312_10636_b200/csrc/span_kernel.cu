// R1: the bounded-SM persistent span kernel.  ONE launch per dispatched batch executes every op
// of a stage's span [start, end) on exactly `sm_budget` CTAs (one per SM), with a grid-wide
// barrier between ops — the B200 replacement for Graft's MPS-percentage GPU sharing
// and for the per-layer launch train.
//
// Roles per CTA (320 threads):
//   warp 4 lane 0   TMA producer for conv ops.  For op j it first streams the WEIGHT tiles of its
//                   first `stages` k-blocks (they do not depend on op j-1), then waits for the
//                   grid barrier of op j-1 and issues the im2col activation tiles;
//   warp 5 lane 0   tcgen05.mma issuer (M=128, N=BN<=128, K=16), TMEM double buffer;
//   warps 6-9       conv epilogue (bias staged per op, residual tiles TMA-prefetched 2 ahead);
//   warps 0-3, 6-9  workers for the bandwidth ops (pool, GAP, FC, channel copy).
// Grid barrier: a 64-bit arrival counter per stage instance; CTA c arrives once per op after its
// writers finished (generic stores + fence.proxy.async, then release); waiting for op j means
// counter >= base + (j + 1) * gridDim.x.  Every arrival for op j is preceded by observing the
// barrier of op j-1, so the count can only reach that value once all CTAs finished op j.
// All CTAs must be co-resident: the deployment keeps the sum of SM budgets <= SM count.
#include <cuda_bf16.h>

#include "bw_ops.cuh"
#include "gx_internal.h"
#include "gx_ptx.cuh"
#include "gx_span.h"

namespace gx {

namespace {
constexpr int kATile = kBM * kBK * 2;
constexpr int kResGroup = kBM * 64 * 2;

__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_wait(const unsigned long long* bar, unsigned long long target) {
  while (ld_acquire_u64(bar) < target) __nanosleep(40);
}
__device__ __forceinline__ void grid_arrive(unsigned long long* bar) {
  asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx_arrive(uint64_t* bar, uint32_t tx) { mbar_arrive_expect_tx(bar, tx); }

__device__ __forceinline__ int cta_tiles(int num_tiles) {
  return num_tiles > static_cast<int>(blockIdx.x) ? (num_tiles - 1 - static_cast<int>(blockIdx.x)) / gridDim.x + 1 : 0;
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// trace (optional): [gridDim.x][n_ops][4] ns stamps: 0 producer passed the barrier of op j-1,
// 1 producer issued its last activation load of op j, 2 worker/epilogue leader started op j,
// 3 worker/epilogue leader arrived for op j.
__global__ void __launch_bounds__(kConvThreads, 1)
    span_kernel(const SpanOp* __restrict__ ops, int n_ops, const __grid_constant__ SpanMaps P,
                unsigned long long* __restrict__ bar, unsigned long long bar_base, SpanSmem L,
                unsigned long long* __restrict__ trace) {
  auto stamp = [&](int j, int slot) {
    if (trace) trace[(static_cast<size_t>(blockIdx.x) * n_ops + j) * 4 + slot] = gtime();
  };
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S_ = L.stages;
  const uint32_t b_stage = static_cast<uint32_t>(L.bn_max) * 128u;
  uint8_t* sA = smem;
  uint8_t* sB = sA + static_cast<size_t>(S_) * kATile;
  uint8_t* sRes = sB + static_cast<size_t>(S_) * b_stage;
  const uint32_t res_slot = static_cast<uint32_t>((L.bn_max + 63) / 64) * kResGroup;
  float* sBias = reinterpret_cast<float*>(sRes + L.has_res * res_slot);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sBias) + L.bias_bytes);
  uint64_t* empty = full + S_;
  uint64_t* tfull = empty + S_;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;
  uint64_t* bfull = rfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const unsigned long long grid = gridDim.x;

  if (warp == 4) {
    if (lane == 0) {
      for (int i = 0; i < S_; ++i) {
        mbar_init(&full[i], 2);  // weights arrival + activation arrival
        mbar_init(&empty[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&tfull[i], 1);
        mbar_init(&tempty[i], 8);  // one arrival per epilogue warp
        mbar_init(&rfull[i], 1);
      }
      mbar_init(bfull, 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(tslot, 2 * L.bn_max <= 128 ? 128 : (2 * L.bn_max <= 256 ? 256 : 512));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tslot;
  const uint32_t acc_stride = static_cast<uint32_t>(L.bn_max);

  if (warp == 4) {
    // ================================================================ TMA producer
    // Incremental walkers: no divisions per k-block (a single thread issues every load).
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;  // ring position of the next stage to fill
      for (int j = 0; j < n_ops; ++j) {
        const SpanOp& op = ops[j];
        if (op.kind != GX_OP_CONV && op.kind != GX_OP_LINEAR) continue;
        const CUtensorMap* wmap = &P.m[op.tmap];
        const CUtensorMap* amap = &P.m[op.tmap + 1];
        tma_prefetch_desc(wmap);
        tma_prefetch_desc(amap);
        const int num_kb = op.num_kb, n_tiles = op.n_tiles, cpl = op.cpl, Cin = op.Cin, Sf = op.S;
        const uint32_t b_bytes = static_cast<uint32_t>(op.BN) * 128u;
        const int n_iter = cta_tiles(op.num_tiles) * num_kb;
        const int npre = n_iter < S_ ? n_iter : S_;
        const uint32_t region = static_cast<uint32_t>(kBM * cpl * 2);
        const int nloads = kBK / cpl;
        // B walker: tile, k-block, weight row offset of the tile
        int b_tile = blockIdx.x, b_kb = 0, b_row = (b_tile % n_tiles) * op.BN;
        int b_st = st;
        uint32_t b_ph = ph;
        auto issue_b = [&](int stage) {
          mbar_expect_tx_arrive(&full[stage], b_bytes);
          tma_load_2d(sB + static_cast<size_t>(stage) * b_stage, wmap, &full[stage], b_kb * kBK, b_row);
          if (++b_kb == num_kb) {
            b_kb = 0;
            b_tile += gridDim.x;
            b_row = (b_tile % n_tiles) * op.BN;
          }
        };
        // 1) weights of the first `npre` k-blocks: independent of the previous op
        for (int i = 0; i < npre; ++i) {
          mbar_wait(&empty[b_st], b_ph ^ 1);
          issue_b(b_st);
          if (++b_st == S_) {
            b_st = 0;
            b_ph ^= 1;
          }
        }
        // 2) activations only once every CTA finished op j-1
        if (n_iter > 0) {
          grid_wait(bar, bar_base + static_cast<unsigned long long>(j) * grid);
          fence_proxy_async_global();
        }
        stamp(j, 0);
        // A walker: per tile (image, output row/col origin), per load (filter tap r, s, channel c0)
        int a_tile = blockIdx.x, a_kb = 0, m0 = 0, nimg = 0, wc = 0, hc = 0, c0 = 0, r = 0, s = 0;
        auto tile_origin = [&]() {
          m0 = (a_tile / n_tiles) * kBM;
          nimg = m0 / op.HoWo;
          const int rem = m0 - nimg * op.HoWo;
          const int ho0 = rem / op.Wo;
          wc = (rem - ho0 * op.Wo) * op.sw - op.pw;
          hc = ho0 * op.sh - op.ph;
          c0 = r = s = 0;
        };
        if (n_iter > 0) tile_origin();
        for (int i = 0; i < n_iter; ++i) {
          if (i >= npre) {  // 3) steady state: both operands of this stage
            mbar_wait(&empty[st], ph ^ 1);
            issue_b(st);
          }
          mbar_expect_tx_arrive(&full[st], kATile);
          uint8_t* dst = sA + static_cast<size_t>(st) * kATile;
          if (op.a2d) {
            tma_load_2d(dst, amap, &full[st], a_kb * kBK, m0);
          } else {
            for (int l = 0; l < nloads; ++l) {
              tma_load_im2col_4d(dst + l * region, amap, &full[st], c0, wc, hc, nimg, static_cast<uint16_t>(s),
                                 static_cast<uint16_t>(r));
              c0 += cpl;  // K order (r, s, c); loads past the last tap hit zero weights
              if (c0 == Cin) {
                c0 = 0;
                if (++s == Sf) {
                  s = 0;
                  ++r;
                }
              }
            }
          }
          if (++a_kb == num_kb) {
            a_kb = 0;
            a_tile += gridDim.x;
            if (i + 1 < n_iter) tile_origin();
          }
          if (++st == S_) {
            st = 0;
            ph ^= 1;
          }
        }
        stamp(j, 1);
      }
    }
  } else if (warp == 5) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      int st = 0, t = 0;
      uint32_t ph = 0;
      for (int j = 0; j < n_ops; ++j) {
        const SpanOp& op = ops[j];
        if (op.kind != GX_OP_CONV && op.kind != GX_OP_LINEAR) continue;
        const int cpl = op.cpl, num_kb = op.num_kb;
        const uint32_t idesc = op.idesc;
        const uint32_t region = static_cast<uint32_t>(kBM * cpl * 2);
        // per-op descriptor template and the A offset of each K=16 step inside a stage
        const uint64_t dbits = umma_desc_kmajor(0, cpl, region);
        uint32_t offs[kBK / 16];
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk) offs[kk] = (kk * 16 / cpl) * region + (kk * 16 % cpl) * 2;
        const int ntile = cta_tiles(op.num_tiles);
        for (int tt = 0; tt < ntile; ++tt, ++t) {
          const int acc = t & 1;
          mbar_wait(&tempty[acc], ((t >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem_base + acc * acc_stride;
          for (int kb = 0; kb < num_kb; ++kb) {
            mbar_wait(&full[st], ph);
            tc_fence_after();
            const uint32_t abase = smem_u32(sA + static_cast<size_t>(st) * kATile);
            const uint64_t bd = umma_desc_sw128(sB + static_cast<size_t>(st) * b_stage);
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              umma_bf16(d, dbits | (((abase + offs[kk]) >> 4) & 0x3FFFull), bd + 2 * kk, idesc, (kb | kk) != 0);
            umma_commit(&empty[st]);
            if (++st == S_) {
              st = 0;
              ph ^= 1;
            }
          }
          umma_commit(&tfull[acc]);
        }
      }
    }
  } else {
    // ================================================================ epilogue + bandwidth workers
    const bool epi = warp >= 6;
    const bool leader = warp == 6 && lane == 0;
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int wtid = epi ? 128 + (warp - 6) * 32 + lane : tid;  // 0..255 over warps 0-3, 6-9
    int t = 0;          // tiles processed (TMEM accumulator sequence)
    int conv_seen = 0;  // conv ops processed (bias barrier phase)
    int r_issued = 0, r_waited = 0;
    for (int j = 0; j < n_ops; ++j) {
      const SpanOp& op = ops[j];
      const bool conv = op.kind == GX_OP_CONV || op.kind == GX_OP_LINEAR;
      const unsigned long long prev_done = bar_base + static_cast<unsigned long long>(j) * grid;
      if (!conv) {
        // ---------------------------------------------------------- bandwidth op
        if (leader) {
          grid_wait(bar, prev_done);
          stamp(j, 2);
        }
        named_bar_sync(2, 256);
        const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 256 + wtid;
        const int64_t stride = static_cast<int64_t>(gridDim.x) * 256;
        switch (op.kind) {
          case GX_OP_MAXPOOL:
          case GX_OP_AVGPOOL:
            pool_body(op.kind == GX_OP_MAXPOOL ? 0 : 1, op.x, op.N, op.H, op.W, op.C, op.x_ld,
                      static_cast<__nv_bfloat16*>(op.y), op.Ho, op.Wo, op.y_ld, op.y_coff, op.R, op.S, op.sh, op.sw,
                      op.ph, op.pw, op.flags & 1, i0, stride);
            break;
          case GX_OP_GAP:
            gap_body(op.x, op.N, op.H * op.W, op.C, static_cast<__nv_bfloat16*>(op.y), i0, stride);
            break;
          case GX_OP_FC:
            fc_warp4_body(op.x, op.N, op.K, op.w, op.bias, op.y, op.Cout, op.y_f32, op.act,
                          static_cast<int>(blockIdx.x) * 8 + (wtid >> 5), static_cast<int>(gridDim.x) * 8, lane);
            break;
          case GX_OP_COPY:
            copy_body(op.x, op.pixels, op.C, op.x_ld, op.x_coff, static_cast<__nv_bfloat16*>(op.y), op.y_ld,
                      op.y_coff, i0, stride);
            break;
          default:
            break;
        }
        fence_proxy_async_global();
        named_bar_sync(2, 256);
        if (leader) {
          __threadfence();
          grid_arrive(bar);
          stamp(j, 3);
        }
        continue;
      }
      // ------------------------------------------------------------ conv epilogue
      // 8 warps: warp w reads TMEM lane quarter w % 4; warps 6-9 take the even 16-column chunks,
      // warps 0-3 the odd ones, so small-K convs are not bound by one warp group's epilogue.
      const int ntile = cta_tiles(op.num_tiles);
      const bool has_res = op.res != nullptr;
      const CUtensorMap* rmap = &P.m[op.rmap >= 0 ? op.rmap : 0];
      auto issue_res = [&](int tt) {
        const int tile = static_cast<int>(blockIdx.x) + tt * static_cast<int>(gridDim.x);
        const int slot = L.has_res == 2 ? (r_issued & 1) : 0;
        const int groups = (op.BN + 63) / 64;
        mbar_arrive_expect_tx(&rfull[slot], static_cast<uint32_t>(groups) * kResGroup);
        for (int g = 0; g < groups; ++g)
          tma_load_2d(sRes + slot * res_slot + g * kResGroup, rmap, &rfull[slot], (tile % op.n_tiles) * op.BN + g * 64,
                      (tile / op.n_tiles) * kBM);
        ++r_issued;
      };
      if (leader) {
        mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(op.Cout) * 4u);
        bulk_load(sBias, op.bias, static_cast<uint32_t>(op.Cout) * 4u, bfull);
        if (has_res && ntile > 0) {
          tma_prefetch_desc(rmap);
          grid_wait(bar, prev_done);  // the residual may be the previous op's output
          fence_proxy_async_global();
          for (int tt = 0; tt < ntile && tt < L.has_res; ++tt) issue_res(tt);
        }
      }
      mbar_wait_sleepy(bfull, conv_seen & 1);
      ++conv_seen;
      if (leader) stamp(j, 2);
      for (int tt = 0; tt < ntile; ++tt, ++t) {
        const int tile = static_cast<int>(blockIdx.x) + tt * static_cast<int>(gridDim.x);
        const int m0 = (tile / op.n_tiles) * kBM;
        const int nb0 = (tile % op.n_tiles) * op.BN;
        const int ncols = min(op.BN, op.Cout - nb0);
        const int acc = t & 1;
        mbar_wait_sleepy(&tfull[acc], (t >> 1) & 1);
        tc_fence_after();
        int slot = 0;
        if (has_res) {
          slot = L.has_res == 2 ? (r_waited & 1) : 0;
          mbar_wait_sleepy(&rfull[slot], (L.has_res == 2 ? (r_waited >> 1) : r_waited) & 1);
          ++r_waited;
        }
        const uint8_t* res_base = sRes + slot * res_slot;
        const float* bias = sBias + nb0;
        const int m = m0 + row;
        const bool row_ok = m < op.M;
        const uint32_t tbase = tmem_base + acc * acc_stride + (static_cast<uint32_t>(q * 32) << 16);
        for (int c = epi ? 0 : 16; c < op.BN; c += 32) {
          uint32_t v[16];
          tmem_ld16(tbase + c, v);
          tmem_ld_wait();
          if (row_ok && c < ncols) {
            const int n0 = nb0 + c;
            float f[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]) + bias[c + i];
            if (has_res) {
              const uint8_t* rrow = res_base + (c >> 6) * kResGroup + row * 128;
              const int j0 = (c & 63) >> 3;
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const uint4 rr = *reinterpret_cast<const uint4*>(rrow + (((j0 + i) ^ (row & 7)) << 4));
                const uint32_t w[4] = {rr.x, rr.y, rr.z, rr.w};
#pragma unroll
                for (int k2 = 0; k2 < 4; ++k2) {
                  const float2 p = unpack_bf16x2(w[k2]);
                  f[8 * i + 2 * k2] += p.x;
                  f[8 * i + 2 * k2 + 1] += p.y;
                }
              }
            }
            if (op.act == GX_ACT_RELU) {
#pragma unroll
              for (int i = 0; i < 16; ++i) f[i] = fmaxf(f[i], 0.0f);
            } else if (op.act == GX_ACT_GELU) {
#pragma unroll
              for (int i = 0; i < 16; ++i) f[i] = gelu_f(f[i]);
            }
            if (op.y_f32) {
              float4* y4 = reinterpret_cast<float4*>(static_cast<float*>(op.y) + static_cast<size_t>(m) * op.y_ld +
                                                     op.y_coff + n0);
#pragma unroll
              for (int i = 0; i < 4; ++i) y4[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
            } else {
              uint4* y4 = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(op.y) + static_cast<size_t>(m) * op.y_ld +
                                                   op.y_coff + n0);
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                uint4 o;
                o.x = pack_bf16x2(f[8 * i + 0], f[8 * i + 1]);
                o.y = pack_bf16x2(f[8 * i + 2], f[8 * i + 3]);
                o.z = pack_bf16x2(f[8 * i + 4], f[8 * i + 5]);
                o.w = pack_bf16x2(f[8 * i + 6], f[8 * i + 7]);
                y4[i] = o;
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&tempty[acc]);  // one arrival per warp
        if (has_res) {
          named_bar_sync(1, 256);  // all epilogue threads are done with this residual slot
          if (leader && tt + L.has_res < ntile) issue_res(tt + L.has_res);
        }
      }
      // op done on this CTA: publish to the grid
      fence_proxy_async_global();
      named_bar_sync(1, 256);
      if (leader) {
        grid_wait(bar, prev_done);  // keeps arrivals in op order (see header)
        __threadfence();
        grid_arrive(bar);
        stamp(j, 3);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * L.bn_max <= 128 ? 128 : (2 * L.bn_max <= 256 ? 256 : 512));
  }
}
}  // namespace

size_t span_smem_bytes(const SpanSmem& L) {
  const size_t res_slot = static_cast<size_t>((L.bn_max + 63) / 64) * kResGroup;
  return 1024 + static_cast<size_t>(L.stages) * (kATile + L.bn_max * 128) + L.has_res * res_slot +
         L.bias_bytes + (2 * L.stages + 9) * 8 + 16;
}

cudaError_t launch_span(const SpanOp* ops, int n_ops, const SpanMaps& maps, unsigned long long* bar,
                        unsigned long long bar_base, const SpanSmem& L, int grid, cudaStream_t s,
                        unsigned long long* trace) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(span_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  span_kernel<<<grid, kConvThreads, span_smem_bytes(L), s>>>(ops, n_ops, maps, bar, bar_base, L, trace);
  return cudaGetLastError();
}

}  // namespace gx
