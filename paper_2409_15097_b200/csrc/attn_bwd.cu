// attn_bwd.cu — block-sparse masked flash-attention backward for sm_100a (TMA + tcgen05 + TMEM).
//
// Replaces the reference's blocked_backward (engine.hpp:346-471): gradients of
// L = sum(out * d_out) from the forward's saved row statistics, over the same tiles the forward
// processed (so the counters equal the forward's). Two deterministic kernels, no atomics on
// gradients (engine.hpp:379-389 merges dK/dV in a fixed order for the same reason):
//
//   dkdv  one item per (slot, key tile j): walks the COLUMN list of j (query row tiles i whose
//         tile (i, j) is occupied, ascending) and accumulates in TMEM
//             S^T  = K_j Q_i^T          dP^T = V_j dO_i^T         (SS MMAs, M = keys)
//             P^T  = exp2(S^T sl2 - lse2_i)   dS^T = P^T (dP^T - delta_i)   (registers)
//             dV_j += P^T dO_i          dK_j += dS^T Q_i           (TS MMAs, A = P^T / dS^T in TMEM)
//         then writes dK_j * scale and dV_j.
//   dq    one item per (slot, query row tile i): walks the ROW list of i (the forward's list) with
//             S = Q_i K_j^T   dP = dO_i V_j^T   P, dS as above   dQ_i += dS K_j
//         then writes dQ_i * scale.
// delta_i = rowsum(dO_i * O_i) (engine.hpp:366-372) and lse2 = (row_max + ln row_sum) log2 e come
// from a small row pass (rowstats_kernel). Fully masked rows (row_sum = 0) and rows past n get
// lse2 = +inf, so every P of theirs is exactly 0.
//
// Both kernels share one structure (the template parameter SIDE picks the operand roles):
//   warp 0      producer: claims items, loads the item's two fixed tiles (K_j, V_j | Q_i, dO_i)
//               and streams the partner tiles (Q_i, dO_i | K_j, V_j) through a ring (TMA, 128B
//               swizzle); for dkdv the partner's lse2 / delta vectors ride along (bulk copy).
//   warp 1      MMA issuer (one thread).
//   warp 2      TMEM allocator: S at [0,128), dP at [128,256), accumulators at 256 (+D); when a
//               second accumulator set fits (dq; dkdv at d=64) items alternate between the two
//               sets and an item's epilogue is deferred until the next item's first tile.
//   warps 4-11  elementwise engine: warp w owns TMEM lanes 32*(w%4).. and column half w/8;
//               epilogue: accumulators -> bf16 -> 128B-swizzled staging -> TMA store.
//               P and dS are written back as packed bf16 into their own half's columns
//               ([64h, 64h+32) of S / dP), which the TS MMAs read as the A operand.
// Mask bits: partial tiles only (full tiles skip them), 8 B per row and half from tile-major
// bitmaps — the forward's row bitmaps for dq, the transposed column bitmaps for dkdv.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <numeric>
#include <vector>

#include "bbm_internal.h"
#include "bbm_ptx.cuh"
#include "bbm_tmap.h"

namespace bbm {
namespace {

using namespace ptx;

enum Side : int { kSideDQ = 0, kSideDKDV = 1 };

constexpr uint32_t kThreads = 384;
constexpr uint32_t kQueue = 4;
constexpr uint32_t kEnd = 0xFFFFFFFFu;  // kNoSplit: bbm_internal.h
constexpr uint32_t kBoxBytes = 128 * 64 * 2;
constexpr float kLog2e = 1.4426950408889634f;

struct BwdParams {
  uint64_t n;
  uint32_t slots;
  float sl2, scale;
  bool all_tiles;             // dense variant: every partner, no mask
  const PlanHdr* hdr;         // device-built plan (plan.cu): units per slot, split rows / chunks
  const uint4* unit_desc;     // [units] {tile, j0, partners walked, split | kNoSplit}, longest first
  const uint2* split_info;    // [split tiles] {chunks, first workspace chunk}
  float* ws;                  // split partials: [slots][split_chunks][128][accumulator columns]
  uint32_t* split_ctr;        // [slots][split rows] finished chunks (reset by the combiner)
  const uint32_t* list;       // [tiles][stride] partner entries, bit 31 = full
  uint32_t list_stride;
  const uint4* bitmaps;       // list-position tile-major bits (row bitmaps | transposed)
  const uint8_t* halves;      // per list position: the tile's empty 64-row partner halves (dq: keys,
                              // dkdv: queries; nullptr = multiply whole tiles)
  const float* lse2;          // [slots][rows_pad], NEGATED (-lse2, rowstats_kernel)
  const float* delta;         // [slots][rows_pad], NEGATED (-delta)
  uint32_t rows_pad;          // krows * 128
  uint32_t* ctr;              // [2] next item, finished CTAs
  __nv_bfloat16* out0;        // dq | dk
  __nv_bfloat16* out1;        // -  | dv
  uint64_t* trace;            // optional event trace (bbm_set_trace), nullptr = off
  uint32_t trace_ctas;
};

// Trace event: [63:24] clock64 low 40 bits | [23:16] code | [15] stream (= half) | [14:0] aux.
// Codes: MMA 40 S/dP of half issued (aux = tile), 41 accumulate of half issued, 42 P/dS of half
// seen, 43 item start (fixed tiles landed); engine 50 s_full wait begin, 51 s_full wait end,
// 52 p_full arrive, 53 acc_full wait end, 54 epilogue done, 55 item descriptor read.
constexpr uint32_t kTraceCap = 8192;
template <bool kTrace>
__device__ __forceinline__ void trace_ev(bool on, const BwdParams& p, uint32_t* counter, uint32_t code,
                                         uint32_t stream, uint32_t aux) {
  if constexpr (!kTrace) return;
  if (!on) return;
  const uint32_t i = atomicAdd(counter, 1u);
  if (i >= kTraceCap) return;
  const uint64_t t = static_cast<uint64_t>(clock64()) & ((1ull << 40) - 1);
  p.trace[static_cast<uint64_t>(blockIdx.x) * kTraceCap + i] =
      (t << 24) | (static_cast<uint64_t>(code & 0xFF) << 16) | ((stream & 1u) << 15) | (aux & 0x7FFF);
}

struct ItemDesc {
  uint32_t t, slot, tile, j0, nt, split;
};

template <int D, int SIDE>
struct BCfg {
  static constexpr uint32_t kBoxes = D / 64;
  static constexpr uint32_t kTileBytes = kBoxes * kBoxBytes;
  static constexpr uint32_t kVecBytes = SIDE == kSideDKDV ? 1024 : 0;  // lse2 | delta of 128 rows
  static constexpr uint32_t kStageBytes = 2 * kTileBytes + (SIDE == kSideDKDV ? 1024 : 0);
  static constexpr uint32_t kStageAlloc = (kStageBytes + 1023) / 1024 * 1024;
  static constexpr uint32_t kStages = D == 64 ? 4 : 2;
  static constexpr uint32_t kOutStage = (D / 64) * kBoxBytes;  // epilogue staging: one 128 x D bf16 tile
  static constexpr uint32_t kAcc0 = 256;      // dQ | dK
  static constexpr uint32_t kAcc1 = 256 + D;  // dV
  // Two accumulator sets when TMEM has room (dq; dkdv at d=64): items alternate between them and
  // an item's epilogue is deferred until the next item's first tile is with the tensor core.
  static constexpr uint32_t kAccSet = SIDE == kSideDQ ? D : 2 * D;  // columns per set
  static constexpr bool kDefer = 256 + 2 * kAccSet <= 512;
};

struct BwdCtl {
  uint64_t fixed_full, fixed_empty, s_full[2], p_full[2], acc_full[2], acc_empty[2];
  uint64_t ring_full[4], ring_empty[4];
  uint64_t item_full[kQueue], item_empty[kQueue];
  ItemDesc items[kQueue];
  uint32_t stage_halves[4];  // per ring stage: the streamed tile's empty partner halves (bit h)
  uint32_t tmem_base;
  uint32_t units, total_items, split_rows, split_chunks;  // this launch's plan
  uint32_t bcast;
  uint32_t trace_count;
};

template <int D, int SIDE>
constexpr uint32_t bwd_smem_bytes() {
  using C = BCfg<D, SIDE>;
  return 2 * C::kTileBytes + C::kStages * C::kStageAlloc + C::kOutStage + sizeof(BwdCtl);
}

__device__ __forceinline__ ItemDesc bwd_decode(const BwdParams& p, uint32_t units, uint32_t total, uint32_t t) {
  ItemDesc d{};
  if (t >= total) {
    d.t = kEnd;
    return d;
  }
  d.t = t;
  d.slot = t / units;
  const uint4 u = p.unit_desc[t - d.slot * units];
  d.tile = u.x;
  d.j0 = u.y;
  d.nt = u.z;
  d.split = u.w;
  return d;
}

__device__ __forceinline__ uint32_t bwd_entry(const BwdParams& p, uint32_t tile, uint32_t j) {
  return p.all_tiles ? j : p.list[static_cast<uint64_t>(tile) * p.list_stride + j];
}

// 1-D bulk copy global -> shared, completion on an mbarrier (16-byte aligned, multiple of 16 B)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// kHalves: this launch skips empty 64-row partner halves (p.halves set). A separate build, so the
// launches without it run exactly the plain issue loop (at d = 64 its issue rate bounds the kernel).
template <int D, int SIDE, bool kTrace, bool kHalves>
__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_f0, const __grid_constant__ CUtensorMap tm_f1,
                    const __grid_constant__ CUtensorMap tm_s0, const __grid_constant__ CUtensorMap tm_s1,
                    const __grid_constant__ CUtensorMap tm_o0, const __grid_constant__ CUtensorMap tm_o1,
                    const __grid_constant__ CUtensorMap tm_s0h, const __grid_constant__ CUtensorMap tm_s1h,
                    const BwdParams p) {
  // fixed tiles f0, f1: (Q_i, dO_i) for dq, (K_j, V_j) for dkdv; streamed s0, s1: the partner's
  // (K_j, V_j) for dq, (Q_i, dO_i) for dkdv.
  using C = BCfg<D, SIDE>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* fixed = smem;                       // [2][tile]
  uint8_t* ring = smem + 2 * C::kTileBytes;    // [kStages][stage]
  uint8_t* ostage = ring + C::kStages * C::kStageAlloc;  // [D/64][128 x 64 bf16] epilogue staging
  auto* ctl = reinterpret_cast<BwdCtl*>(ostage + C::kOutStage);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if ((smem_u32(smem) & 1023u) != 0) __trap();

  const bool tracing = kTrace && blockIdx.x < p.trace_ctas;
  if (threadIdx.x == 0) {
    ctl->trace_count = 0;
    const PlanHdr h = *p.hdr;
    ctl->units = h.units;
    ctl->total_items = h.units * p.slots;
    ctl->split_rows = h.split_rows;
    ctl->split_chunks = h.split_chunks;
    mbar_init(&ctl->fixed_full, 1);
    mbar_init(&ctl->fixed_empty, 1);
    for (int h = 0; h < 2; ++h) {
      mbar_init(&ctl->s_full[h], 1);
      mbar_init(&ctl->p_full[h], 128);  // the four softmax warps of half h
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ctl->acc_full[b], 1);
      mbar_init(&ctl->acc_empty[b], 256);
    }
    for (uint32_t r = 0; r < C::kStages; ++r) {
      mbar_init(&ctl->ring_full[r], 1);
      mbar_init(&ctl->ring_empty[r], 1);
    }
    for (uint32_t r = 0; r < kQueue; ++r) {
      mbar_init(&ctl->item_full[r], 1);
      mbar_init(&ctl->item_empty[r], 1 + 8);  // MMA issuer + the 8 engine warps
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_f0);
    tma_prefetch_desc(&tm_f1);
    tma_prefetch_desc(&tm_s0);
    tma_prefetch_desc(&tm_s1);
  }
  if (warp == 2) {
    tmem_alloc<512>(&ctl->tmem_base);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol_fixed = policy_evict_first();
      const uint64_t pol_stream = policy_evict_last();
      uint32_t r = 0, rph = 1, qi = 0, qiph = 1, fph = 1;
      for (;;) {
        const ItemDesc d = bwd_decode(p, ctl->units, ctl->total_items, atomicAdd(&p.ctr[0], 1u));
        mbar_wait(&ctl->item_empty[qi], qiph);
        ctl->items[qi] = d;
        mbar_arrive(&ctl->item_full[qi]);
        if (++qi == kQueue) { qi = 0; qiph ^= 1; }
        if (d.t == kEnd) break;
        if (d.nt == 0) continue;
        mbar_wait(&ctl->fixed_empty, fph);
        fph ^= 1;
        mbar_arrive_expect_tx(&ctl->fixed_full, 2 * C::kTileBytes);
        for (uint32_t b = 0; b < C::kBoxes; ++b) {
          tma_load_3d(fixed + b * kBoxBytes, &tm_f0, &ctl->fixed_full, b * 64, d.tile * 128, d.slot, pol_fixed);
          tma_load_3d(fixed + C::kTileBytes + b * kBoxBytes, &tm_f1, &ctl->fixed_full, b * 64,
                      d.tile * 128, d.slot, pol_fixed);
        }
        for (uint32_t j = 0; j < d.nt; ++j) {
          const uint32_t u = bwd_entry(p, d.tile, d.j0 + j) & 0x7FFFFFFFu;
          uint32_t hv = 0;
          if constexpr (kHalves) hv = __ldg(p.halves + static_cast<uint64_t>(d.tile) * p.list_stride + d.j0 + j);
          mbar_wait(&ctl->ring_empty[r], rph);
          uint64_t* full = &ctl->ring_full[r];
          uint8_t* st = ring + r * C::kStageAlloc;
          if constexpr (kHalves) ctl->stage_halves[r] = hv;  // published by the arrive below
          if (!kHalves || hv == 0) {
            mbar_arrive_expect_tx(full, C::kStageBytes);
            for (uint32_t b = 0; b < C::kBoxes; ++b) {
              tma_load_3d(st + b * kBoxBytes, &tm_s0, full, b * 64, u * 128, d.slot, pol_stream);
              tma_load_3d(st + C::kTileBytes + b * kBoxBytes, &tm_s1, full, b * 64, u * 128, d.slot,
                          pol_stream);
            }
          } else {
            // one partner half is never paired: only the other half's 64 rows are loaded (64-row boxes)
            const uint32_t hh = (hv & 1u) ? 1u : 0u;
            mbar_arrive_expect_tx(full, C::kStageBytes - C::kTileBytes);
            for (uint32_t b = 0; b < C::kBoxes; ++b) {
              tma_load_3d(st + b * kBoxBytes + hh * (kBoxBytes / 2), &tm_s0h, full, b * 64, u * 128 + hh * 64,
                          d.slot, pol_stream);
              tma_load_3d(st + C::kTileBytes + b * kBoxBytes + hh * (kBoxBytes / 2), &tm_s1h, full, b * 64,
                          u * 128 + hh * 64, d.slot, pol_stream);
            }
          }
          if constexpr (SIDE == kSideDKDV) {
            const uint64_t off = static_cast<uint64_t>(d.slot) * p.rows_pad + u * 128;
            bulk_load(st + 2 * C::kTileBytes, p.lse2 + off, 512, full);
            bulk_load(st + 2 * C::kTileBytes + 512, p.delta + off, 512, full);
          }
          if (++r == C::kStages) { r = 0; rph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    // Each tile's work is split by partner-row halves h (TMEM columns [64h, 64h+64) of S and dP,
    // owned by softmax warps 4-7 / 8-11): S_h, dP_h (N = 64) and the accumulate MMAs over K-steps
    // of half h. Issue order  SdP_0(j) SdP_1(j) | acc_0(j) SdP_0(j+1) | acc_1(j) SdP_1(j+1) | ...
    // so one half's elementwise pass overlaps the other half's MMAs, and a half's next scores
    // overwrite its P / dS columns only after its accumulate MMAs (in-order execution).
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, false, false);
      constexpr uint32_t idesc_acc = make_idesc_bf16(128, D, false, true);
      const uint32_t faddr = smem_u32(fixed), raddr = smem_u32(ring);
      const uint64_t f0 = make_sdesc_sw128(faddr, 16, 1024), f1 = make_sdesc_sw128(faddr + C::kTileBytes, 16, 1024);
      uint32_t qi = 0, qiph = 0, r = 0, rph = 0, fph = 0, items = 0;
      PhaseBits aph{0x3u};  // acc_empty phases (both sets start free)
      PhaseBits pph{0u};
      // S_h = f0 s0[64h..]^T, dP_h = f1 s1[64h..]^T: both K-major, K = D, N = 64 partner rows
      // a partner half that no row of the tile sees (dq: an empty 64-key half) is not multiplied:
      // its S / dP columns keep stale values whose P / dS no accumulate MMA reads
      // (the stage's flags are read once per tile, and only when the launch skips halves: at
      // d = 64 this thread's issue rate bounds the kernel)
      constexpr bool skips = kHalves;
      auto issue_sdp = [&](uint32_t h, uint32_t stage, uint32_t hv) {
        if (kHalves && ((hv >> h) & 1u)) {
          tc_commit(&ctl->s_full[h]);
          return;
        }
        const uint32_t sbase = raddr + stage * C::kStageAlloc + h * 8192;
        const uint64_t s0 = make_sdesc_sw128(sbase, 16, 1024), s1 = make_sdesc_sw128(sbase + C::kTileBytes, 16, 1024);
#pragma unroll
        for (uint32_t kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * kBoxBytes + (kk % 4) * 32;
          umma_ss(tmem + h * 64, sdesc_advance(f0, off), sdesc_advance(s0, off), idesc_s, kk > 0);
        }
#pragma unroll
        for (uint32_t kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * kBoxBytes + (kk % 4) * 32;
          umma_ss(tmem + 128 + h * 64, sdesc_advance(f1, off), sdesc_advance(s1, off), idesc_s, kk > 0);
        }
        tc_commit(&ctl->s_full[h]);
      };
      // accumulate MMAs of half h: K steps 4h..4h+3 (partner rows 64h..64h+63). Packed bf16 A
      // operand: half h's 32 columns at [64h, 64h+32) of its region -> column (kk/4)*64 + (kk%4)*8
      // the item's first accumulate MMA overwrites, the others accumulate: the first is K step 0 of
      // tile 0's first non-empty half h0 (no mutable state in this loop: at d = 64 the issue rate
      // bounds the kernel)
      auto issue_acc = [&](uint32_t h, uint32_t stage, uint32_t j, uint32_t h0, uint32_t acc0, uint32_t hv) {
        if (kHalves && ((hv >> h) & 1u)) return;
        const uint32_t sbase = raddr + stage * C::kStageAlloc;
        const uint64_t b0 = make_sdesc_sw128(sbase, kBoxBytes, 1024);
        const uint64_t b1 = make_sdesc_sw128(sbase + C::kTileBytes, kBoxBytes, 1024);
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
          const uint32_t kk = 4 * h + q;
          const uint32_t acol = (kk / 4) * 64 + (kk % 4) * 8;
          const uint32_t acc = (j > 0 || h != h0 || q > 0) ? 1u : 0u;
          // dQ += dS K_j  |  dK += dS^T Q_i   (B = streamed tile 0, MN-major)
          umma_ts(tmem + acc0, tmem + 128 + acol, sdesc_advance(b0, kk * 2048), idesc_acc, acc);
          if constexpr (SIDE == kSideDKDV)  // dV += P^T dO_i   (B = streamed tile 1)
            umma_ts(tmem + acc0 + D, tmem + acol, sdesc_advance(b1, kk * 2048), idesc_acc, acc);
        }
      };
      for (;;) {
        mbar_wait(&ctl->item_full[qi], qiph);
        const ItemDesc it = ctl->items[qi];
        mbar_arrive(&ctl->item_empty[qi]);
        if (++qi == kQueue) { qi = 0; qiph ^= 1; }
        if (it.t == kEnd) break;
        if (it.nt == 0) continue;
        mbar_wait(&ctl->fixed_full, fph);
        fph ^= 1;
        mbar_wait(&ctl->ring_full[r], rph);
        tc_fence_after();
        trace_ev<kTrace>(tracing, p, &ctl->trace_count, 43, 0, it.t);
        uint32_t hv_cur = skips ? ctl->stage_halves[r] : 0u;
        issue_sdp(0, r, hv_cur);
        trace_ev<kTrace>(tracing, p, &ctl->trace_count, 40, 0, 0);
        issue_sdp(1, r, hv_cur);
        trace_ev<kTrace>(tracing, p, &ctl->trace_count, 40, 1, 0);
        if (it.nt == 1) tc_commit(&ctl->fixed_empty);
        const uint32_t ab = C::kDefer ? (items++ & 1u) : 0u;  // this item's accumulator set
        const uint32_t h0 = (hv_cur & 1u) ? 1u : 0u;  // tile 0's first non-empty half
        const uint32_t acc0 = C::kAcc0 + ab * C::kAccSet;
        for (uint32_t j = 0; j < it.nt; ++j) {
          const uint32_t rn = r + 1 == C::kStages ? 0 : r + 1;
          const uint32_t rnph = r + 1 == C::kStages ? rph ^ 1 : rph;
          uint32_t hv_next = 0;
          for (uint32_t h = 0; h < 2; ++h) {
            mbar_wait(&ctl->p_full[h], pph[h]);
            pph.flip(h);
            trace_ev<kTrace>(tracing, p, &ctl->trace_count, 42, h, j);
            if (j == 0 && h == 0) {
              mbar_wait(&ctl->acc_empty[ab], aph[ab]);  // this set's last epilogue has read it
              aph.flip(ab);
            }
            tc_fence_after();
            issue_acc(h, r, j, h0, acc0, hv_cur);
            trace_ev<kTrace>(tracing, p, &ctl->trace_count, 41, h, j);
            if (h == 1) tc_commit(&ctl->ring_empty[r]);  // both halves of tile j consumed
            if (j + 1 < it.nt) {
              if (h == 0) {
                mbar_wait(&ctl->ring_full[rn], rnph);
                tc_fence_after();
                hv_next = skips ? ctl->stage_halves[rn] : 0u;
              }
              issue_sdp(h, rn, hv_next);
              trace_ev<kTrace>(tracing, p, &ctl->trace_count, 40, h, j + 1);
              if (h == 1 && j + 2 == it.nt) tc_commit(&ctl->fixed_empty);
            }
          }
          r = rn;
          rph = rnph;
          hv_cur = hv_next;
        }
        tc_commit(&ctl->acc_full[ab]);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ elementwise engine
    const uint32_t half = warp >= 8 ? 1u : 0u;
    const uint32_t quad = warp & 3;
    const uint32_t row = quad * 32 + lane;  // TMEM lane: key (dkdv) or query (dq) in the tile
    const uint32_t lane_off = (quad * 32) << 16;
    const bool tracer = quad == 0 && lane == 0;  // one per half
    const bool leader = warp == 4 && lane == 0;
    const float sl2 = p.sl2;
    uint32_t qi = 0, qiph = 0, sph = 0, r = 0;
    const uint32_t last = (static_cast<uint32_t>(p.n) + 127) / 128 - 1;
    const int valid_last = static_cast<int>(p.n - static_cast<uint64_t>(last) * 128) - static_cast<int>(half * 64);
    // Epilogue of item `it` (accumulator set ab; has_acc = false writes zero rows for an item
    // without partners): waits for the item's last accumulate MMAs, then accumulator -> bf16 ->
    // staging -> TMA store and releases the set. Called by all 256 engine threads together.
    PhaseBits afph{0u};
    auto finish = [&](const ItemDesc& it, uint32_t ab, bool has_acc) {
      const uint32_t acc0 = C::kAcc0 + ab * C::kAccSet;
      if (has_acc) {
        mbar_wait(&ctl->acc_full[ab], afph[ab]);
        afph.flip(ab);
        tc_fence_after();
        if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 53, half, it.t);
      }
      constexpr uint32_t kHalf = D / 2;
      constexpr uint32_t kAccs = SIDE == kSideDKDV ? 2u : 1u;
      constexpr uint32_t kBlk = 128 * kAccs * D;  // floats per split-chunk partial block
      // Split tile (a long list cut into chunks by the plan): publish this chunk's fp32 partial
      // accumulators; the last chunk to finish adds every chunk's partial IN CHUNK ORDER
      // (deterministic, no atomics on gradients) and writes the gradients.
      const float* sum_base = nullptr;
      uint32_t sum_chunks = 0;
      if (it.split != kNoSplit) {
        const uint32_t srow = it.split >> 8, chunk = it.split & 0xFF;
        const uint2 si = p.split_info[srow];  // {chunks, first workspace chunk}
        float* wsb = p.ws + (static_cast<uint64_t>(it.slot) * ctl->split_chunks + si.y + chunk) * kBlk;
#pragma unroll
        for (uint32_t a = 0; a < kAccs; ++a)
#pragma unroll
          for (uint32_t c32 = 0; c32 < kHalf / 32; ++c32) {
            uint32_t v[32];
            tmem_ld32(tmem + lane_off + acc0 + a * D + half * kHalf + c32 * 32, v);
            tmem_ld_wait();
            uint4* dst = reinterpret_cast<uint4*>(wsb + row * (kAccs * D) + a * D + half * kHalf + c32 * 32);
#pragma unroll
            for (uint32_t q = 0; q < 8; ++q) dst[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
        tc_fence_before();
        mbar_arrive(&ctl->acc_empty[ab]);
        __threadfence();
        named_bar_sync(1, 256);
        uint32_t* ctr = p.split_ctr + static_cast<uint64_t>(it.slot) * ctl->split_rows + srow;
        if (leader) ctl->bcast = atomicAdd(ctr, 1u);
        named_bar_sync(1, 256);
        const bool last = ctl->bcast + 1 == si.x;
        named_bar_sync(1, 256);  // every thread has read the count
        if (!last) return;
        __threadfence();
        if (leader) *ctr = 0;  // ready for the next launch
        sum_base = p.ws + (static_cast<uint64_t>(it.slot) * ctl->split_chunks + si.y) * kBlk;
        sum_chunks = si.x;
      }
      // accumulator (TMEM, or the chunks' sum) -> bf16 (x scale for dq / dk) -> 128B-swizzled
      // staging -> TMA store (rows past n are clipped by the tensor map). Half h stages output
      // columns [D/2 h, D/2 (h+1)).
#pragma unroll
      for (uint32_t a = 0; a < kAccs; ++a) {
        const float mul = a == 0 ? p.scale : 1.0f;
        if (leader) bulk_wait_group_read<0>();  // the previous store has read the staging tile
        named_bar_sync(1, 256);
#pragma unroll
        for (uint32_t c32 = 0; c32 < kHalf / 32; ++c32) {
          uint32_t v[32];
          const uint32_t col = half * kHalf + c32 * 32;  // output column of v[0]
          if (sum_base) {
            float acc[32];
#pragma unroll
            for (uint32_t i2 = 0; i2 < 32; ++i2) acc[i2] = 0.0f;
            for (uint32_t c = 0; c < sum_chunks; ++c) {
              const float4* src = reinterpret_cast<const float4*>(sum_base + c * kBlk + row * (kAccs * D) + a * D + col);
#pragma unroll
              for (uint32_t q = 0; q < 8; ++q) {
                const float4 f = __ldcg(src + q);
                acc[4 * q] += f.x;
                acc[4 * q + 1] += f.y;
                acc[4 * q + 2] += f.z;
                acc[4 * q + 3] += f.w;
              }
            }
#pragma unroll
            for (uint32_t i2 = 0; i2 < 32; ++i2) v[i2] = __float_as_uint(acc[i2]);
          } else if (has_acc) {
            tmem_ld32(tmem + lane_off + acc0 + a * D + col, v);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (uint32_t i2 = 0; i2 < 32; ++i2) v[i2] = 0u;
          }
          uint8_t* rowp = ostage + (col / 64) * kBoxBytes + row * 128;
#pragma unroll
          for (uint32_t c = 0; c < 4; ++c) {
            uint4 w;
            w.x = pack_bf16x2(__uint_as_float(v[c * 8 + 0]) * mul, __uint_as_float(v[c * 8 + 1]) * mul);
            w.y = pack_bf16x2(__uint_as_float(v[c * 8 + 2]) * mul, __uint_as_float(v[c * 8 + 3]) * mul);
            w.z = pack_bf16x2(__uint_as_float(v[c * 8 + 4]) * mul, __uint_as_float(v[c * 8 + 5]) * mul);
            w.w = pack_bf16x2(__uint_as_float(v[c * 8 + 6]) * mul, __uint_as_float(v[c * 8 + 7]) * mul);
            *reinterpret_cast<uint4*>(rowp + ((((col % 64) / 8 + c) ^ (row & 7)) << 4)) = w;
          }
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 256);
        if (leader) {
#pragma unroll
          for (uint32_t b = 0; b < D / 64; ++b)
            tma_store_3d(a == 0 ? &tm_o0 : &tm_o1, ostage + b * kBoxBytes, b * 64, it.tile * 128, it.slot);
          bulk_commit_group();
        }
      }
      if (has_acc && !sum_base) {
        tc_fence_before();
        mbar_arrive(&ctl->acc_empty[ab]);
      }
      if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 54, half, it.t);
    };
    struct Pending {
      ItemDesc it;
      uint32_t ab;
      bool valid;
    };
    Pending pend{};
    uint32_t items = 0;
    for (;;) {
      mbar_wait(&ctl->item_full[qi], qiph);
      const ItemDesc it = ctl->items[qi];
      if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 55, half, it.t);
      __syncwarp();  // every lane of this warp has read the descriptor
      if (lane == 0) mbar_arrive(&ctl->item_empty[qi]);
      if (++qi == kQueue) { qi = 0; qiph ^= 1; }
      if (it.t == kEnd) break;
      const uint64_t grow = static_cast<uint64_t>(it.tile) * 128 + row;
      if (it.nt > 0) {
        uint64_t my_nl = 0, my_nd = 0;  // (-lse2, -delta) of this thread's query row, both lanes
        if constexpr (SIDE == kSideDQ) {
          const uint64_t o = static_cast<uint64_t>(it.slot) * p.rows_pad + grow;
          const float nl = p.lse2[o], nd = p.delta[o];
          my_nl = f2_pack(nl, nl);
          my_nd = f2_pack(nd, nd);
        }
        const uint64_t sl2x2 = f2_pack(sl2, sl2);
        const uint32_t ab = C::kDefer ? (items++ & 1u) : 0u;  // same sequence as the MMA issuer
        for (uint32_t j = 0; j < it.nt; ++j) {
          const uint32_t e = bwd_entry(p, it.tile, it.j0 + j);
          const uint32_t u = e & 0x7FFFFFFFu;
          bool masked;
          uint2 bits = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
          if (p.all_tiles) {
            // dense: only the dq side has a ragged key edge (its columns are keys); rows past n
            // on the dkdv side carry lse2 = +inf
            masked = SIDE == kSideDQ && u == last && valid_last < 64;
            if (masked) {
              const int v = valid_last;
              bits.x = v >= 32 ? 0xFFFFFFFFu : (v <= 0 ? 0u : ((1u << v) - 1u));
              bits.y = v >= 64 ? 0xFFFFFFFFu : (v <= 32 ? 0u : ((1u << (v - 32)) - 1u));
            }
          } else {
            masked = (e & 0x80000000u) == 0;
            if (masked)
              bits = __ldg(reinterpret_cast<const uint2*>(
                                p.bitmaps + (static_cast<uint64_t>(it.tile) * p.list_stride + it.j0 + j) * 128 + row) +
                            half);
          }
          if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 50, half, j);
          mbar_wait(&ctl->s_full[half], sph);
          sph ^= 1;
          tc_fence_after();
          if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 51, half, j);
          const uint32_t ts = tmem + lane_off + half * 64;
          const float* vec = nullptr;
          if constexpr (SIDE == kSideDKDV)
            vec = reinterpret_cast<const float*>(ring + r * C::kStageAlloc + 2 * C::kTileBytes) + half * 64;
          // a warp whose 32 rows pair with none of this half's 64 partners: P = dS = 0 without
          // loading S / dP or computing anything (exactly what the masked path writes)
          const bool empty = masked && __all_sync(0xffffffffu, (bits.x | bits.y) == 0u);
#pragma unroll
          for (uint32_t c32 = 0; c32 < 2; ++c32) {
            if (empty) {
              uint32_t z[16];
#pragma unroll
              for (uint32_t i = 0; i < 16; ++i) z[i] = 0u;
              tmem_st16(ts + c32 * 16, z);
              tmem_st16(ts + 128 + c32 * 16, z);
              continue;
            }
            uint32_t s[32], dp[32];
            tmem_ld32(ts + c32 * 32, s);
            tmem_ld32(ts + 128 + c32 * 32, dp);
            tmem_ld_wait();
            const uint32_t mw = c32 ? bits.y : bits.x;
            uint32_t pk[16], dk[16];
#pragma unroll
            for (uint32_t i = 0; i < 32; i += 2) {
              uint64_t nl = my_nl, nd = my_nd;
              if constexpr (SIDE == kSideDKDV) {  // per key pair: the partner query rows' values
                nl = *reinterpret_cast<const uint64_t*>(vec + c32 * 32 + i);
                nd = *reinterpret_cast<const uint64_t*>(vec + 128 + c32 * 32 + i);
              }
              // x = S sl2 - lse2, two lanes per instruction
              const uint64_t x = ffma2(f2_pack(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), sl2x2, nl);
              float p0 = fast_exp2(f2_lo(x));
              float p1 = fast_exp2(f2_hi(x));
              if (masked) {
                p0 = ((mw >> i) & 1u) ? p0 : 0.0f;
                p1 = ((mw >> (i + 1)) & 1u) ? p1 : 0.0f;
              }
              // dS = P (dP - delta)
              const uint64_t g = fmul2(f2_pack(p0, p1),
                                       fadd2(f2_pack(__uint_as_float(dp[i]), __uint_as_float(dp[i + 1])), nd));
              pk[i / 2] = pack_bf16x2(p0, p1);
              dk[i / 2] = pack_bf16x2(f2_lo(g), f2_hi(g));
            }
            tmem_st16(ts + c32 * 16, pk);        // P over this half's own S columns
            tmem_st16(ts + 128 + c32 * 16, dk);  // dS over this half's own dP columns
          }
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&ctl->p_full[half]);
          if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 52, half, j);
          if (++r == C::kStages) r = 0;
          if (C::kDefer && j == 0 && pend.valid) {  // the previous item's accumulate MMAs drained meanwhile
            finish(pend.it, pend.ab, true);
            pend.valid = false;
          }
        }
        if constexpr (C::kDefer) {
          pend = Pending{it, ab, true};  // written after the next item's first tile
        } else {
          finish(it, 0, true);
        }
      } else {
        finish(it, 0, false);  // no partner: zero rows
      }
      if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 54, half, it.t);
    }
    if (pend.valid) finish(pend.it, pend.ab, true);
    if (leader) bulk_wait_group<0>();  // gradient stores landed
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&p.ctr[1], 1u) == gridDim.x - 1) {
      p.ctr[0] = 0;
      p.ctr[1] = 0;
      __threadfence();
    }
  }
}

// delta = rowsum(dO * O) (engine.hpp:366-372), lse2 = (row_max + ln row_sum) * log2(e); rows with
// row_sum == 0 (fully masked) and rows past n: lse2 = +inf (their P is 0), delta = 0. Both are
// stored NEGATED (nlse2, ndelta) so the engine adds them with packed FFMA2 / FADD2.
// One warp per row.
template <typename OT>
__global__ void rowstats_kernel(const OT* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                const float* __restrict__ row_max, const float* __restrict__ row_sum,
                                uint64_t slots, uint64_t n, uint32_t d, uint32_t rows_pad,
                                float* __restrict__ nlse2, float* __restrict__ ndelta) {
  const uint64_t total = slots * rows_pad;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; w < total;
       w += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
    const uint64_t slot = w / rows_pad, r = w % rows_pad;
    float acc = 0.0f, l = INFINITY;
    if (r < n) {
      const uint64_t base = (slot * n + r) * d;
      for (uint32_t c = lane; c < d; c += 32) {
        float ov;
        if constexpr (sizeof(OT) == 4) ov = o[base + c];
        else ov = __bfloat162float(o[base + c]);
        acc += ov * __bfloat162float(dout[base + c]);
      }
      const float rs = row_sum[slot * n + r];
      if (rs > 0.0f) l = (row_max[slot * n + r] + logf(rs)) * kLog2e;
    }
#pragma unroll
    for (uint32_t m = 16; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (lane == 0) {
      nlse2[w] = -l;
      ndelta[w] = r < n ? -acc : 0.0f;
    }
  }
}

// Column lists: for key tile q, the ascending occupied query row tiles (bit 31 = full, never on
// a ragged tile). One CTA (256 threads) per column tile.
__global__ void __launch_bounds__(256) collist_kernel(const uint32_t* __restrict__ sums, uint64_t n,
                                                      uint32_t krows, uint32_t kcols,
                                                      uint32_t* __restrict__ col_list,
                                                      uint32_t* __restrict__ col_cnt) {
  __shared__ uint32_t warp_cnt[8];
  const uint32_t q = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t base = 0;
  for (uint32_t p0 = 0; p0 < krows; p0 += 256) {
    const uint32_t pr = p0 + threadIdx.x;
    const uint32_t s = pr < krows ? sums[static_cast<uint64_t>(pr) * kcols + q] : 0u;
    const bool o = s > 0;
    const uint32_t ballot = __ballot_sync(0xffffffffu, o);
    if (lane == 0) warp_cnt[warp] = __popc(ballot);
    __syncthreads();
    uint32_t before = base;
    for (uint32_t w = 0; w < warp; ++w) before += warp_cnt[w];
    before += __popc(ballot & ((1u << lane) - 1u));
    const bool full = s == 128u * 128u && (static_cast<uint64_t>(pr) + 1) * 128 <= n &&
                      (static_cast<uint64_t>(q) + 1) * 128 <= n;
    if (o) col_list[static_cast<uint64_t>(q) * krows + before] = pr | (full ? 0x80000000u : 0u);
    for (uint32_t w = 0; w < 8; ++w) base += warp_cnt[w];
    __syncthreads();
  }
  if (threadIdx.x == 0) col_cnt[q] = base;
}

// Transposed bits of every occupied tile at its column-list position: CTA (q, k), 4 warps; warp w
// holds query rows 32w..32w+31 of the tile and emits, per key c, the ballot of their bit c.
__global__ void __launch_bounds__(128) transpose_bitmaps_kernel(const uint4* __restrict__ mask,
                                                                uint32_t krows, uint32_t kcols,
                                                                const uint32_t* __restrict__ col_list,
                                                                const uint32_t* __restrict__ col_cnt,
                                                                uint4* __restrict__ tbits,
                                                                uint8_t* __restrict__ col_halves) {
  const uint32_t q = blockIdx.y, k = blockIdx.x;
  if (k >= col_cnt[q]) return;
  const uint32_t pr = col_list[static_cast<uint64_t>(q) * krows + k] & 0x7FFFFFFFu;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint4 rowbits = mask[(static_cast<uint64_t>(pr) * 128 + warp * 32 + lane) * kcols + q];
  // query halves of the tile that see no key of it
  const bool seen = (rowbits.x | rowbits.y | rowbits.z | rowbits.w) != 0u;
  const int lo = __syncthreads_or(warp < 2 && seen), hi = __syncthreads_or(warp >= 2 && seen);
  if (threadIdx.x == 0)
    col_halves[static_cast<uint64_t>(q) * krows + k] = static_cast<uint8_t>((lo ? 0 : 1) | (hi ? 0 : 2));
  uint32_t* out = reinterpret_cast<uint32_t*>(tbits + (static_cast<uint64_t>(q) * krows + k) * 128);
  const uint32_t words[4] = {rowbits.x, rowbits.y, rowbits.z, rowbits.w};
#pragma unroll
  for (uint32_t wd = 0; wd < 4; ++wd)
#pragma unroll 8
    for (uint32_t b = 0; b < 32; ++b) {
      const uint32_t col = __ballot_sync(0xffffffffu, (words[wd] >> b) & 1u);
      if (lane == 0) out[(wd * 32 + b) * 4 + warp] = col;
    }
}

template <int D, int SIDE>
void launch_side(const Prep& prep, StreamCtx& ctx, const BwdArgs& a, const float* lse2, const float* delta,
                 uint32_t rows_pad, cudaStream_t s, int num_sms) {
  static_assert(bwd_smem_bytes<D, SIDE>() <= 232448, "exceeds the 227 KB opt-in shared memory");
  const KernelMeta& km = prep.kmeta;
  const BwdMeta& bm = prep.bwd;
  BwdParams p{};
  p.n = a.n;
  p.slots = static_cast<uint32_t>(a.slots);
  p.all_tiles = a.variant == 0;
  p.sl2 = a.scale * kLog2e;
  p.scale = a.scale;
  p.lse2 = lse2;
  p.delta = delta;
  p.rows_pad = rows_pad;
  // work units from the device-built plan over the row view (dq) or the column view (dkdv):
  // whole tiles, or balanced chunks of long lists (global tokens) combined deterministically
  const TileView view =
      SIDE == kSideDQ ? row_view(km) : TileView{bm.col_cnt, bm.col_list, km.kcols, km.krows, 1, bm.col_halves};
  const uint32_t workers = static_cast<uint32_t>(num_sms);
  const DevPlan& plan = plan_for(prep, ctx, view, p.all_tiles ? kPlanDense : kPlanList, a.slots, workers, s);
  const bool can_split = plan.cap_units > view.tiles;
  p.hdr = plan.hdr;
  p.unit_desc = plan.unit_desc;
  p.split_info = plan.split_info;
  p.ws = can_split ? ctx_workspace(ctx, plan_cap_chunks(a.slots, workers) * 128 * 256, s) : nullptr;
  p.split_ctr = can_split ? ctx_split_ctr(ctx, plan_cap_chunks(a.slots, workers) + a.slots, s) : nullptr;
  if (SIDE == kSideDQ) {
    p.list = km.list;
    p.list_stride = km.kcols;
    p.bitmaps = km.bitmaps;
#ifdef BBM_NO_HALF_SKIP  // A/B builds: whole tiles always
    p.halves = nullptr;
#else
    p.halves = plan.half_heavy ? km.halves : nullptr;  // known one launch after a new mask version
#endif
    p.ctr = ctx.ctr + 2;
    p.out0 = static_cast<__nv_bfloat16*>(a.dq);
  } else {
    p.list = bm.col_list;
    p.list_stride = km.krows;
    p.bitmaps = bm.tbitmaps;
#ifdef BBM_NO_HALF_SKIP  // A/B builds: whole tiles always
    p.halves = nullptr;
#else
    p.halves = plan.half_heavy ? bm.col_halves : nullptr;  // partner (query) halves of the column view
#endif
    p.ctr = ctx.ctr + 4;
    p.out0 = static_cast<__nv_bfloat16*>(a.dk);
    p.out1 = static_cast<__nv_bfloat16*>(a.dv);
  }
  const CUtensorMap tq = cached_tmap_bf16_3d(a.q, D, a.n, a.slots, 64, 128);
  const CUtensorMap tk = cached_tmap_bf16_3d(a.k, D, a.n, a.slots, 64, 128);
  const CUtensorMap tv = cached_tmap_bf16_3d(a.v, D, a.n, a.slots, 64, 128);
  const CUtensorMap tdo = cached_tmap_bf16_3d(a.d_out, D, a.n, a.slots, 64, 128);
  const CUtensorMap to0 = cached_tmap_bf16_3d(p.out0, D, a.n, a.slots, 64, 128);
  const CUtensorMap to1 = SIDE == kSideDKDV ? cached_tmap_bf16_3d(p.out1, D, a.n, a.slots, 64, 128) : to0;
  // streamed tiles with an empty partner half: 64-row boxes of the other half
  const CUtensorMap tk64 = cached_tmap_bf16_3d(a.k, D, a.n, a.slots, 64, 64);
  const CUtensorMap tv64 = cached_tmap_bf16_3d(a.v, D, a.n, a.slots, 64, 64);
  const CUtensorMap tq64 = cached_tmap_bf16_3d(a.q, D, a.n, a.slots, 64, 64);
  const CUtensorMap tdo64 = cached_tmap_bf16_3d(a.d_out, D, a.n, a.slots, 64, 64);
  static std::atomic<uint64_t> attr_devices{0};
  once_per_device(attr_devices, [] {
    BBM_CUDA(cudaFuncSetAttribute(attn_bwd_kernel<D, SIDE, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  bwd_smem_bytes<D, SIDE>()));
    BBM_CUDA(cudaFuncSetAttribute(attn_bwd_kernel<D, SIDE, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  bwd_smem_bytes<D, SIDE>()));
    BBM_CUDA(cudaFuncSetAttribute(attn_bwd_kernel<D, SIDE, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  bwd_smem_bytes<D, SIDE>()));
  });
  const uint32_t grid = static_cast<uint32_t>(
      std::max<uint64_t>(1, std::min<uint64_t>(a.slots * plan.cap_units, static_cast<uint64_t>(num_sms))));
  // event trace (bbm_set_trace) of one side only, chosen by BBM_TRACE_BWD_SIDE (0 dq, 1 dkdv):
  // both kernels would otherwise write the same buffer
  const char* tside = std::getenv("BBM_TRACE_BWD_SIDE");
  if (g_trace.buffer && tside && std::atoi(tside) == SIDE) {
    p.trace = static_cast<uint64_t*>(g_trace.buffer);
    p.trace_ctas = g_trace.ctas;
  }
  auto go = [&](auto kernel) {
    if (SIDE == kSideDQ)
      kernel<<<grid, kThreads, bwd_smem_bytes<D, SIDE>(), s>>>(tq, tdo, tk, tv, to0, to1, tk64, tv64, p);
    else
      kernel<<<grid, kThreads, bwd_smem_bytes<D, SIDE>(), s>>>(tk, tv, tq, tdo, to0, to1, tq64, tdo64, p);
  };
  if (p.trace)
    go(attn_bwd_kernel<D, SIDE, true, false>);
  else if (p.halves)
    go(attn_bwd_kernel<D, SIDE, false, true>);
  else
    go(attn_bwd_kernel<D, SIDE, false, false>);
  BBM_CUDA(cudaGetLastError());
}

template <class T>
T* bwd_alloc(uint64_t count) {
  void* ptr = nullptr;
  BBM_CUDA(cudaMalloc(&ptr, std::max<uint64_t>(1, count) * sizeof(T)));
  return static_cast<T*>(ptr);
}


}  // namespace

void free_bwd_meta(BwdMeta& b) {
  cudaFree(b.col_cnt);
  cudaFree(b.col_list);
  cudaFree(b.tbitmaps);
  cudaFree(b.col_halves);
  cudaFree(b.scratch);
  if (b.ready) cudaEventDestroy(b.ready);
  b = BwdMeta{};
}

// Column view of the current mask version, built on stream s by kernels only (called with
// prep.mu held). Streams that did not build it wait for `ready`.
void ensure_bwd_meta(const Prep& prep, cudaStream_t s) {
  BwdMeta& b = prep.bwd;
  const KernelMeta& km = prep.kmeta;
  const uint32_t kr = km.krows, kc = km.kcols;
  if (b.version != prep.version) {
    if (!b.col_cnt) {
      b.col_cnt = bwd_alloc<uint32_t>(kc);
      b.col_list = bwd_alloc<uint32_t>(static_cast<uint64_t>(kc) * kr);
      b.tbitmaps = bwd_alloc<uint4>(static_cast<uint64_t>(kc) * kr * 128);
      b.col_halves = bwd_alloc<uint8_t>(static_cast<uint64_t>(kc) * kr);
      b.scratch = bwd_alloc<uint32_t>(static_cast<uint64_t>(kr) + kc + 2);
      BBM_CUDA(cudaEventCreateWithFlags(&b.ready, cudaEventDisableTiming));
    }
    collist_kernel<<<kc, 256, 0, s>>>(km.sums, prep.n, kr, kc, b.col_list, b.col_cnt);
    BBM_CUDA(cudaGetLastError());
    transpose_bitmaps_kernel<<<dim3(kr, kc), 128, 0, s>>>(reinterpret_cast<const uint4*>(km.mask), kr, kc,
                                                           b.col_list, b.col_cnt, b.tbitmaps, b.col_halves);
    BBM_CUDA(cudaGetLastError());
    BBM_CUDA(cudaEventRecord(b.ready, s));
    b.version = prep.version;
  } else {
    BBM_CUDA(cudaStreamWaitEvent(s, b.ready, 0));
  }
}

void launch_attn_bwd(const Prep& prep, const BwdArgs& a, cudaStream_t s, int num_sms) {
  require(a.slots >= 1, "need at least one batch/head slot");
  require(a.n == prep.n, "mask preprocessing does not match this problem");
  if (a.d != 64 && a.d != 128) throw ArgError("head dim must be 64 or 128 on the sm_100a kernel");
  std::lock_guard<std::recursive_mutex> lk(prep.mu);
  StreamCtx& ctx = prep.ctx_for(s);
  ensure_bwd_meta(prep, s);
  const uint32_t rows_pad = prep.kmeta.krows * 128;
  const size_t need = 2 * static_cast<size_t>(a.slots) * rows_pad;
  if (need > ctx.rowws_floats) {
    if (ctx.rowws) {
      BBM_CUDA(cudaStreamSynchronize(s));
      cudaFree(ctx.rowws);
    }
    ctx.rowws = nullptr;
    ctx.rowws_floats = 0;
    BBM_CUDA(cudaMalloc(&ctx.rowws, need * sizeof(float)));
    ctx.rowws_floats = need;
  }
  float* lse2 = ctx.rowws;
  float* delta = ctx.rowws + static_cast<size_t>(a.slots) * rows_pad;
  const uint64_t warps = a.slots * rows_pad;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((warps + 7) / 8, 148ull * 64));
  if (a.o_f32)
    rowstats_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(a.o),
                                                static_cast<const __nv_bfloat16*>(a.d_out), a.row_max,
                                                a.row_sum, a.slots, a.n, a.d, rows_pad, lse2, delta);
  else
    rowstats_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(a.o), static_cast<const __nv_bfloat16*>(a.d_out), a.row_max,
        a.row_sum, a.slots, a.n, a.d, rows_pad, lse2, delta);
  BBM_CUDA(cudaGetLastError());
  if (a.d == 64) {
    launch_side<64, kSideDKDV>(prep, ctx, a, lse2, delta, rows_pad, s, num_sms);
    launch_side<64, kSideDQ>(prep, ctx, a, lse2, delta, rows_pad, s, num_sms);
  } else {
    launch_side<128, kSideDKDV>(prep, ctx, a, lse2, delta, rows_pad, s, num_sms);
    launch_side<128, kSideDQ>(prep, ctx, a, lse2, delta, rows_pad, s, num_sms);
  }
  mark_launch_done(ctx, s);
}

}  // namespace bbm
