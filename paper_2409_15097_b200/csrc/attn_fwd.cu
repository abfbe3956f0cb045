// attn_fwd.cu — block-sparse masked flash-attention forward for sm_100a (TMA + tcgen05 + TMEM).
//
// Replaces the reference's blocked_forward (engine.hpp:282-341): for every (slot, query row
// tile p) it walks only the KV tiles its variant processes — the compacted occupied-tile list
// built by prep.cu for binblk / dense_binblk, all tiles for dense / naive — in ascending order
// (engine.hpp:311), with an online softmax whose fully-masked rows are exact no-ops
// (engine.hpp:206-235) and fully-masked output rows written as zeros (engine.hpp:330-332).
//
// CTA = one 128-row query tile at a time, persistent over a static slot-major / LPT work list,
// 2 CTAs per SM so one CTA's MMAs overlap the other's softmax. 256 threads:
//   warp 0      TMA producer: Q tile, then K_j / V_j per listed tile (128B-swizzled boxes)
//   warp 1      MMA issuer (one thread): S = Q K^T (SS, K-major) into TMEM, then
//               O += P V (TS: P read from TMEM, V MN-major) — tcgen05.commit -> mbarriers
//   warp 2      TMEM allocator (256 columns: S/P at [0,128), O at [128,128+D))
//   warps 4-7   softmax + correction + epilogue, one query row per thread (TMEM lane = row)
// Numerics: S is scaled into the log2 domain; the running max is only raised when it grows by
// more than 2^8 (stale-max trick, exact after the final O/l), P is rounded to bf16 for the MMA,
// l accumulates in fp32. Partial tiles read 16 B of mask bits per row (coalesced, tile-major);
// full tiles read none.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "bbm_internal.h"
#include "bbm_ptx.cuh"
#include "bbm_tmap.h"

namespace bbm {
namespace {

using namespace ptx;

enum Mode : int { kModeBinblk = 0, kModeDenseBinblk = 1, kModeDense = 2, kModeNaive = 3 };

struct FwdParams {
  uint64_t n;
  uint32_t slots;
  uint32_t krows, kcols;
  uint32_t total_items;
  float sl2;  // scale * log2(e)
  const uint32_t* list;
  const uint32_t* row_cnt;
  const uint32_t* order;
  const uint4* bitmaps;
  const uint4* mask;  // padded packed mask, kcols uint4 per row
  __nv_bfloat16* out;
  float* row_max;
  float* row_sum;
};

constexpr uint32_t kThreads = 256;
constexpr uint32_t kBoxBytes = 128 * 64 * 2;  // 128 rows x 64 bf16, one 128B-swizzle box
constexpr float kRescaleThreshold = 8.0f;     // log2 units
constexpr float kLn2 = 0.69314718055994530942f;

template <int D>
struct Cfg {
  static constexpr uint32_t kBoxes = D / 64;
  static constexpr uint32_t kTileBytes = kBoxes * kBoxBytes;  // one 128 x D bf16 tile
  static constexpr uint32_t kStages = (D == 64) ? 2 : 1;
  static constexpr uint32_t kSmem = kTileBytes * (1 + 2 * kStages) + 1024;  // + align slack
  static constexpr uint32_t kTmemCols = 256;
  static constexpr uint32_t kOCol = 128;
};

__device__ __forceinline__ void decode_item(const FwdParams& p, uint32_t item, uint32_t& slot,
                                            uint32_t& row_tile) {
  slot = item / p.krows;
  row_tile = p.order[item % p.krows];
}

template <int MODE>
__device__ __forceinline__ uint32_t tiles_of(const FwdParams& p, uint32_t row_tile) {
  if constexpr (MODE == kModeDense || MODE == kModeNaive) return p.kcols;
  else return p.row_cnt[row_tile];
}

template <int MODE>
__device__ __forceinline__ uint32_t entry_of(const FwdParams& p, uint32_t row_tile, uint32_t j) {
  if constexpr (MODE == kModeDense || MODE == kModeNaive) return j;
  else return p.list[static_cast<uint64_t>(row_tile) * p.kcols + j];
}

template <int D, int MODE>
__global__ void __launch_bounds__(kThreads, 2)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const FwdParams p) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sq = smem;
  uint8_t* sk = sq + C::kTileBytes;
  uint8_t* sv = sk + C::kStages * C::kTileBytes;

  __shared__ uint64_t bar_q_full, bar_q_empty, bar_s_full, bar_p_full, bar_o_full, bar_o_empty;
  __shared__ uint64_t bar_k_full[C::kStages], bar_k_empty[C::kStages];
  __shared__ uint64_t bar_v_full[C::kStages], bar_v_empty[C::kStages];
  __shared__ uint32_t tmem_base_sh;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(&bar_q_full, 1);
    mbar_init(&bar_q_empty, 1);
    mbar_init(&bar_s_full, 1);
    mbar_init(&bar_p_full, 128);
    mbar_init(&bar_o_full, 1);
    mbar_init(&bar_o_empty, 128);
    for (uint32_t s = 0; s < C::kStages; ++s) {
      mbar_init(&bar_k_full[s], 1);
      mbar_init(&bar_k_empty[s], 1);
      mbar_init(&bar_v_full[s], 1);
      mbar_init(&bar_v_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  if (warp == 2) {
    tmem_alloc<C::kTmemCols>(&tmem_base_sh);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t tmem_s = tmem;
  const uint32_t tmem_o = tmem + C::kOCol;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      uint32_t q_phase = 1, ks = 0, k_phase = 1, vs = 0, v_phase = 1;
      for (uint32_t item = blockIdx.x; item < p.total_items; item += gridDim.x) {
        uint32_t slot, rt;
        decode_item(p, item, slot, rt);
        const uint32_t nt = tiles_of<MODE>(p, rt);
        if (nt == 0) continue;
        mbar_wait(&bar_q_empty, q_phase);
        q_phase ^= 1;
        mbar_arrive_expect_tx(&bar_q_full, C::kTileBytes);
        for (uint32_t b = 0; b < C::kBoxes; ++b)
          tma_load_3d(sq + b * kBoxBytes, &tm_q, &bar_q_full, b * 64, rt * 128, slot, pol_q);
        for (uint32_t j = 0; j < nt; ++j) {
          const uint32_t q = entry_of<MODE>(p, rt, j) & 0x7FFFFFFFu;
          mbar_wait(&bar_k_empty[ks], k_phase);
          mbar_arrive_expect_tx(&bar_k_full[ks], C::kTileBytes);
          for (uint32_t b = 0; b < C::kBoxes; ++b)
            tma_load_3d(sk + ks * C::kTileBytes + b * kBoxBytes, &tm_k, &bar_k_full[ks], b * 64,
                        q * 128, slot, pol_kv);
          if (++ks == C::kStages) { ks = 0; k_phase ^= 1; }
          mbar_wait(&bar_v_empty[vs], v_phase);
          mbar_arrive_expect_tx(&bar_v_full[vs], C::kTileBytes);
          for (uint32_t b = 0; b < C::kBoxes; ++b)
            tma_load_3d(sv + vs * C::kTileBytes + b * kBoxBytes, &tm_v, &bar_v_full[vs], b * 64,
                        q * 128, slot, pol_kv);
          if (++vs == C::kStages) { vs = 0; v_phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, D, false, true);
      const uint32_t sq_addr = smem_u32(sq), sk_addr = smem_u32(sk), sv_addr = smem_u32(sv);
      uint32_t q_phase = 0, ks = 0, k_phase = 0, vs = 0, v_phase = 0;
      uint32_t p_phase = 0, oe_phase = 1;

      auto issue_s = [&](bool last_s) {
        mbar_wait(&bar_k_full[ks], k_phase);
        tc_fence_after();
        const uint32_t kbase = sk_addr + ks * C::kTileBytes;
#pragma unroll
        for (uint32_t kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * kBoxBytes + (kk % 4) * 32;
          umma_ss(tmem_s, make_sdesc_sw128(sq_addr + off, 16, 1024),
                  make_sdesc_sw128(kbase + off, 16, 1024), idesc_s, kk > 0);
        }
        tc_commit(&bar_k_empty[ks]);
        if (last_s) tc_commit(&bar_q_empty);
        tc_commit(&bar_s_full);
        if (++ks == C::kStages) { ks = 0; k_phase ^= 1; }
      };
      auto issue_pv = [&](bool first) {
        mbar_wait(&bar_p_full, p_phase);
        p_phase ^= 1;
        mbar_wait(&bar_v_full[vs], v_phase);
        if (first) {
          mbar_wait(&bar_o_empty, oe_phase);
          oe_phase ^= 1;
        }
        tc_fence_after();
        const uint32_t vbase = sv_addr + vs * C::kTileBytes;
#pragma unroll
        for (uint32_t kk = 0; kk < 128 / 16; ++kk)
          umma_ts(tmem_o, tmem_s + kk * 8, make_sdesc_sw128(vbase + kk * 2048, kBoxBytes, 1024),
                  idesc_o, (!first || kk > 0) ? 1u : 0u);
        tc_commit(&bar_v_empty[vs]);
        if (++vs == C::kStages) { vs = 0; v_phase ^= 1; }
      };

      for (uint32_t item = blockIdx.x; item < p.total_items; item += gridDim.x) {
        uint32_t slot, rt;
        decode_item(p, item, slot, rt);
        const uint32_t nt = tiles_of<MODE>(p, rt);
        if (nt == 0) continue;
        mbar_wait(&bar_q_full, q_phase);
        q_phase ^= 1;
        issue_s(nt == 1);
        for (uint32_t j = 1; j <= nt; ++j) {
          issue_pv(j == 1);
          if (j < nt) issue_s(j == nt - 1);
        }
        tc_commit(&bar_o_full);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ softmax / epilogue
    const uint32_t quad = warp & 3;
    const uint32_t row = quad * 32 + lane;
    const uint32_t lane_off = (quad * 32) << 16;
    const uint32_t ts = tmem_s + lane_off, to = tmem_o + lane_off;
    const bool ragged = (p.n % 128) != 0;
    const uint32_t last_q = p.kcols - 1;
    const uint32_t kv_valid_last = static_cast<uint32_t>(p.n - static_cast<uint64_t>(last_q) * 128);
    uint32_t s_phase = 0, o_phase = 0;

    for (uint32_t item = blockIdx.x; item < p.total_items; item += gridDim.x) {
      uint32_t slot, rt;
      decode_item(p, item, slot, rt);
      const uint32_t nt = tiles_of<MODE>(p, rt);
      const uint64_t grow = static_cast<uint64_t>(rt) * 128 + row;
      const bool row_ok = grow < p.n;
      float m_run = -INFINITY, m_true = -INFINITY, l = 0.0f;

      uint32_t entry = nt ? entry_of<MODE>(p, rt, 0) : 0;
      for (uint32_t j = 0; j < nt; ++j) {
        const uint32_t q = entry & 0x7FFFFFFFu;
        const bool full = (entry & 0x80000000u) != 0;
        bool masked;
        if constexpr (MODE == kModeDense) masked = false;
        else if constexpr (MODE == kModeDenseBinblk) masked = !full;
        else masked = true;
        uint4 bits = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
        if (masked) {
          if constexpr (MODE == kModeNaive)
            bits = __ldg(p.mask + grow * p.kcols + q);
          else
            bits = __ldg(p.bitmaps + (static_cast<uint64_t>(rt) * p.kcols + q) * 128 + row);
        }
        if (ragged && q == last_q) {
          // columns >= n do not exist (TMA zero-filled rows of K/V): never visible
          const uint32_t v = kv_valid_last;
          const uint32_t w0 = v >= 32 ? 0xFFFFFFFFu : ((1u << v) - 1u);
          const uint32_t w1 = v >= 64 ? 0xFFFFFFFFu : (v <= 32 ? 0u : ((1u << (v - 32)) - 1u));
          const uint32_t w2 = v >= 96 ? 0xFFFFFFFFu : (v <= 64 ? 0u : ((1u << (v - 64)) - 1u));
          const uint32_t w3 = v >= 128 ? 0xFFFFFFFFu : (v <= 96 ? 0u : ((1u << (v - 96)) - 1u));
          bits.x &= w0; bits.y &= w1; bits.z &= w2; bits.w &= w3;
        }
        if (j + 1 < nt) entry = entry_of<MODE>(p, rt, j + 1);

        mbar_wait(&bar_s_full, s_phase);
        s_phase ^= 1;
        tc_fence_after();

        // pass 1: masked, scaled row max over the tile
        float tmax = -INFINITY;
#pragma unroll 1
        for (uint32_t c = 0; c < 4; ++c) {
          uint32_t r[32];
          tmem_ld32(ts + c * 32, r);
          tmem_ld_wait();
          const uint32_t mw = c == 0 ? bits.x : c == 1 ? bits.y : c == 2 ? bits.z : bits.w;
#pragma unroll
          for (uint32_t i = 0; i < 32; ++i) {
            const float x = ((mw >> i) & 1u) ? __uint_as_float(r[i]) * p.sl2 : -INFINITY;
            tmax = fmaxf(tmax, x);
          }
        }
        m_true = fmaxf(m_true, tmax);
        const bool need = tmax > m_run + kRescaleThreshold || (m_run == -INFINITY && tmax > -INFINITY);
        const bool rescale_o = need && j > 0 && m_run > -INFINITY;
        float factor = 1.0f;
        if (need) {
          if (m_run > -INFINITY) factor = fast_exp2(m_run - tmax);
          m_run = tmax;
        }
        if (__any_sync(0xffffffffu, rescale_o)) {
          const float f = rescale_o ? factor : 1.0f;
#pragma unroll
          for (uint32_t c = 0; c < D / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(to + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (uint32_t i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
            tmem_st32(to + c * 32, r);
          }
        }
        l *= factor;
        const float m_use = m_run == -INFINITY ? 0.0f : m_run;

        // pass 2: P = exp2(s - m) as bf16, written over S columns [0,64) chunk by chunk
#pragma unroll 1
        for (uint32_t c = 0; c < 4; ++c) {
          uint32_t r[32];
          tmem_ld32(ts + c * 32, r);
          tmem_ld_wait();
          const uint32_t mw = c == 0 ? bits.x : c == 1 ? bits.y : c == 2 ? bits.z : bits.w;
          uint32_t pk[16];
#pragma unroll
          for (uint32_t i = 0; i < 32; i += 2) {
            const float x0 = ((mw >> i) & 1u) ? __uint_as_float(r[i]) * p.sl2 - m_use : -INFINITY;
            const float x1 =
                ((mw >> (i + 1)) & 1u) ? __uint_as_float(r[i + 1]) * p.sl2 - m_use : -INFINITY;
            const float e0 = fast_exp2(x0), e1 = fast_exp2(x1);
            l += e0 + e1;
            pk[i / 2] = pack_bf16x2(e0, e1);
          }
          // chunk c of P (16 packed columns) lands on S columns [16c, 16c+16): S chunk c/2,
          // which has already been read, so the in-place overwrite is safe.
          tmem_st16(ts + c * 16, pk);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bar_p_full);
      }

      // ---------------------------------------------------------------- epilogue
      __nv_bfloat16* orow = p.out + (static_cast<uint64_t>(slot) * p.n + grow) * D;
      if (nt > 0) {
        mbar_wait(&bar_o_full, o_phase);
        o_phase ^= 1;
        tc_fence_after();
        const float inv = l > 0.0f ? 1.0f / l : 0.0f;
#pragma unroll 1
        for (uint32_t c = 0; c < D / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(to + c * 32, r);
          tmem_ld_wait();
          if (row_ok) {
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
            for (uint32_t v = 0; v < 4; ++v) {
              uint4 w;
              w.x = pack_bf16x2(__uint_as_float(r[v * 8 + 0]) * inv, __uint_as_float(r[v * 8 + 1]) * inv);
              w.y = pack_bf16x2(__uint_as_float(r[v * 8 + 2]) * inv, __uint_as_float(r[v * 8 + 3]) * inv);
              w.z = pack_bf16x2(__uint_as_float(r[v * 8 + 4]) * inv, __uint_as_float(r[v * 8 + 5]) * inv);
              w.w = pack_bf16x2(__uint_as_float(r[v * 8 + 6]) * inv, __uint_as_float(r[v * 8 + 7]) * inv);
              dst[v] = w;
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&bar_o_empty);
      } else if (row_ok) {
        uint4* dst = reinterpret_cast<uint4*>(orow);
        for (uint32_t v = 0; v < D / 8; ++v) dst[v] = make_uint4(0, 0, 0, 0);
      }
      if (row_ok) {
        const uint64_t si = static_cast<uint64_t>(slot) * p.n + grow;
        if (p.row_max) p.row_max[si] = m_true == -INFINITY ? -INFINITY : m_true * kLn2;
        if (p.row_sum) p.row_sum[si] = l > 0.0f ? l * fast_exp2(m_run - m_true) : 0.0f;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<C::kTmemCols>(tmem);
}

}  // namespace
}  // namespace bbm

namespace bbm {
namespace {

template <int D, int MODE>
void launch_impl(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms) {
  using C = Cfg<D>;
  const KernelMeta& km = prep.kmeta;
  const CUtensorMap tq = make_tmap_bf16_3d(a.q, D, a.n, a.slots, 64, 128);
  const CUtensorMap tk = make_tmap_bf16_3d(a.k, D, a.n, a.slots, 64, 128);
  const CUtensorMap tv = make_tmap_bf16_3d(a.v, D, a.n, a.slots, 64, 128);
  FwdParams p{};
  p.n = a.n;
  p.slots = static_cast<uint32_t>(a.slots);
  p.krows = km.krows;
  p.kcols = km.kcols;
  p.total_items = static_cast<uint32_t>(a.slots * km.krows);
  p.sl2 = a.scale * 1.4426950408889634f;
  p.list = km.list;
  p.row_cnt = km.row_cnt;
  p.order = km.order;
  p.bitmaps = km.bitmaps;
  p.mask = reinterpret_cast<const uint4*>(km.mask);
  p.out = static_cast<__nv_bfloat16*>(a.o);
  p.row_max = a.row_max;
  p.row_sum = a.row_sum;
  static bool attr_set = false;  // per (D, MODE) instantiation
  if (!attr_set) {
    BBM_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<D, MODE>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr_set = true;
  }
  const uint32_t grid = std::min<uint32_t>(p.total_items, 2u * static_cast<uint32_t>(num_sms));
  attn_fwd_kernel<D, MODE><<<grid, kThreads, C::kSmem, s>>>(tq, tk, tv, p);
  BBM_CUDA(cudaGetLastError());
}

template <int D>
void launch_d(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms) {
  switch (a.variant) {
    case 0: launch_impl<D, kModeDense>(prep, a, s, num_sms); break;
    case 1: launch_impl<D, kModeNaive>(prep, a, s, num_sms); break;
    case 2: launch_impl<D, kModeBinblk>(prep, a, s, num_sms); break;
    case 3: launch_impl<D, kModeDenseBinblk>(prep, a, s, num_sms); break;
    default: throw ArgError("unknown variant");
  }
}

}  // namespace

void launch_attn_fwd(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms) {
  require(a.slots >= 1, "need at least one batch/head slot");
  require(a.n == prep.n, "mask preprocessing does not match this problem");
  if (a.slots * prep.kmeta.krows == 0) return;
  if (a.d == 64) launch_d<64>(prep, a, s, num_sms);
  else if (a.d == 128) launch_d<128>(prep, a, s, num_sms);
  else throw ArgError("head dim must be 64 or 128 on the sm_100a kernel");
}

int attn_fwd_kernel_launches_per_call() { return 1; }

}  // namespace bbm
