// attn_fwd_pair.cu — the block-sparse masked forward as two query-tile streams per CTA (sm_100a).
//
// Same contract and arithmetic as attn_fwd.cu (blocked_forward, engine.hpp:282-341; the softmax
// math of bbm_softmax.cuh in the same per-row order, so outputs and statistics are bit-identical
// to the single-stream kernel whenever that kernel splits no row), organised for more overlap:
//
// Work item = (slot, row-tile pair r): stream 0 walks row tile 2r's occupied-tile list, stream 1
// row tile 2r+1's. Each stream owns one Q tile, one S/P buffer and one O accumulator in TMEM
// (D = 128: S0 0, S1 128, O0 256, O1 384), and one softmax warpgroup with ONE THREAD PER ROW: no
// cross-warp max exchange, and the two warpgroups run decoupled, so one computes exponentials
// while the other reduces maxima (FA4-style ping-pong).
//
// Status: selected only on request (bbm_set_fwd_kernel(2)). Measured on B200 it is 15-25 % slower
// than attn_fwd.cu, its MMA side alone included: one thread issues every MMA of
// both streams (tcgen05 issue takes ~56 cycles per 128x128x16 MMA, so S + PV of a tile are ~900
// issue cycles for 1024 tensor cycles) and S_s(t+1) waits for PV_s(t) to complete.
//
// K/V sharing: the producer merges the two lists into one load schedule. A tile both rows visit
// is loaded once and feeds both streams' MMAs (adjacent row tiles of banded, causal and packed
// masks share most of their tiles); a stream whose next tile the other stream reaches within two
// steps waits for it instead of loading it separately. Every K/V load carries a meta word
// (consumers, first/last-of-item flags) in shared memory, so the MMA issuer needs no list.
//
// MMA issue (one thread): per stream the ops alternate S_s = Q_s K^T, then O_s += P_s V once the
// softmax has written P_s over S_s; S_s(t+1) is issued only after PV_s(t) has completed (P lives in
// S's columns). The issuer polls both streams and issues whichever op is ready, so the tensor pipe
// works on one stream while the other stream's softmax runs.
//
// Roles (512 threads): warp 0 producer (TMA; claims items), warp 1 MMA issuer, warp 2 TMEM
// allocator, warps 4-7 / 8-11 softmax of stream 0 / 1 (176 registers), warps 12-15 epilogue:
// O / l -> bf16 rows stored straight from registers. Shared memory: the two Q tiles and a K/V ring
// of 5 tiles at D = 128 (the ring depth, not Q double-buffering, is what hides the L2 -> shared
// latency of the next shared K tile: its slot frees only when both streams are past the slot
// five loads back). The next item's Q_s loads as soon as the stream's last S MMA has completed.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "bbm_internal.h"
#include "bbm_ptx.cuh"
#include "bbm_softmax.cuh"
#include "bbm_tmap.h"

namespace bbm {
namespace {

using namespace ptx;
using namespace softmax;

enum PairMode : int { kPModeBinblk = 0, kPModeDenseBinblk = 1, kPModeDense = 2, kPModeNaive = 3 };

constexpr uint32_t kPEnd = 0xFFFFFFFFu;
constexpr uint32_t kPQueue = 4;  // item queue depth
constexpr uint32_t kPBox = 128 * 64 * 2;
constexpr uint32_t kSmemMax = 232448;

// meta word of one K/V load
enum : uint32_t {
  kMetaV = 1u,         // V tile (else K)
  kMetaS0 = 2u,        // consumed by stream 0 (stream s: kMetaS0 << s)
  kMetaFirst0 = 8u,    // first S (K load) / first PV (V load) of the item for stream 0
  kMetaLast0 = 32u,    // last S (K load) / last PV (V load) of the item for stream 0
  kMetaEnd = 128u,     // no more work
};

struct PairParams {
  uint64_t n;
  uint32_t slots, krows, kcols, npairs;
  float sl2;  // scale * log2(e)
  const uint32_t* list;
  const uint32_t* row_cnt;
  const uint4* bitmaps;
  const uint4* mask;  // padded packed mask (naive)
  uint32_t* work_ctr;
  __nv_bfloat16* out;
  float* row_max;
  float* row_sum;
};

struct PairItem {
  uint32_t t, slot, pair, n0, n1;
};

template <int D>
struct PCfg {
  static constexpr uint32_t kBoxes = D / 64;
  static constexpr uint32_t kTile = kBoxes * kPBox;
  static constexpr uint32_t kCtlReserve = 2048;
  static constexpr uint32_t kRingFit = (kSmemMax - 2 * kTile - kCtlReserve) / kTile;
  static constexpr uint32_t kRing = kRingFit > 8 ? 8 : kRingFit;
  static constexpr uint32_t kSCol = 0;      // S_s at s * 128
  static constexpr uint32_t kOCol = 256;    // O_s at 256 + s * D
};

template <uint32_t kRing>
struct PairCtl {
  uint64_t q_full[2], q_empty[2];
  uint64_t s_full[2], p_full[2], pv_done[2], o_full[2], o_empty[2];
  uint64_t stats_full[2], stats_empty[2];
  uint64_t ring_full[kRing], ring_empty[kRing];
  uint64_t item_full[kPQueue], item_empty[kPQueue];
  PairItem items[kPQueue];
  uint32_t meta[kRing];
  uint32_t tmem_base;
  float l[2][128];  // row sums handed from the softmax to the epilogue, per stream
};

template <int D>
constexpr uint32_t pair_smem_bytes() {
  return PCfg<D>::kTile * (2 + PCfg<D>::kRing) + sizeof(PairCtl<PCfg<D>::kRing>);
}

template <int MODE>
__device__ __forceinline__ uint32_t pentry(const PairParams& p, uint32_t rt, uint32_t j) {
  if constexpr (MODE == kPModeDense || MODE == kPModeNaive) return j;
  else return __ldg(p.list + static_cast<uint64_t>(rt) * p.kcols + j);
}

template <int D, int MODE>
__global__ void __launch_bounds__(512, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                     const PairParams p) {
  using C = PCfg<D>;
  constexpr uint32_t kRing = C::kRing;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sq = smem;                        // [stream][tile] Q
  uint8_t* ring = smem + 2 * C::kTile;       // [kRing][tile] K / V
  auto* ctl = reinterpret_cast<PairCtl<kRing>*>(ring + kRing * C::kTile);

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if ((smem_u32(smem) & 1023u) != 0) __trap();

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&ctl->q_full[i], 1);
      mbar_init(&ctl->q_empty[i], 1);  // the issuer's commit after the stream's last S of an item
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&ctl->s_full[s], 1);
      mbar_init(&ctl->p_full[s], 128);
      mbar_init(&ctl->pv_done[s], 1);
      mbar_init(&ctl->o_full[s], 1);
      mbar_init(&ctl->o_empty[s], 128);
      mbar_init(&ctl->stats_full[s], 128);
      mbar_init(&ctl->stats_empty[s], 128);
    }
    for (uint32_t r = 0; r < kRing; ++r) {
      mbar_init(&ctl->ring_full[r], 1);
      mbar_init(&ctl->ring_empty[r], 1);
    }
    for (uint32_t r = 0; r < kPQueue; ++r) {
      mbar_init(&ctl->item_full[r], 1);
      mbar_init(&ctl->item_empty[r], 12);  // 8 softmax warps + 4 epilogue warps
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_o);
  }
  if (warp == 2) {
    tmem_alloc<512>(&ctl->tmem_base);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl->tmem_base;
  const uint32_t total = p.slots * p.npairs;

  if (warp < 4) {
    setmaxnreg_dec<80>();
    if (warp == 0) {
      // ------------------------------------------------------------------ producer
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      uint32_t qi = 0, qiph = 1, lpos = 0;
      PhaseBits qe{0x3u};  // q_empty phases per stream, first use passes
      uint32_t slot = 0;
      auto load = [&](const CUtensorMap* tm, uint32_t col, uint32_t meta) {
        const uint32_t r = lpos % kRing;
        mbar_wait(&ctl->ring_empty[r], ((lpos / kRing) & 1) ^ 1);
        if (lane == 0) {
          ctl->meta[r] = meta;
          if (meta & kMetaEnd) {
            mbar_arrive(&ctl->ring_full[r]);
          } else {
            mbar_arrive_expect_tx(&ctl->ring_full[r], C::kTile);
            for (uint32_t b = 0; b < C::kBoxes; ++b)
              tma_load_3d(ring + r * C::kTile + b * kPBox, tm, &ctl->ring_full[r], b * 64, col * 128, slot,
                          pol_kv);
          }
        }
        __syncwarp();
        ++lpos;
      };
      // list windows: lane i holds entry base + i of the row's list (one coalesced load per 32)
      uint32_t w0base = 0, w0 = 0, w1base = 0, w1 = 0;
      for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(&p.work_ctr[0], 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        PairItem it{kPEnd, 0, 0, 0, 0};
        if (t < total) {
          it.t = t;
          it.slot = t / p.npairs;
          it.pair = t - it.slot * p.npairs;
          const uint32_t rt0 = 2 * it.pair, rt1 = rt0 + 1;
          if constexpr (MODE == kPModeDense || MODE == kPModeNaive) {
            it.n0 = p.kcols;
            it.n1 = rt1 < p.krows ? p.kcols : 0u;
          } else {
            it.n0 = __ldg(p.row_cnt + rt0);
            it.n1 = rt1 < p.krows ? __ldg(p.row_cnt + rt1) : 0u;
          }
        }
        mbar_wait(&ctl->item_empty[qi], qiph);
        if (lane == 0) {
          ctl->items[qi] = it;
          mbar_arrive(&ctl->item_full[qi]);
        }
        if (++qi == kPQueue) { qi = 0; qiph ^= 1; }
        if (it.t == kPEnd) {
          load(nullptr, 0, kMetaEnd);
          break;
        }
        slot = it.slot;
        const uint32_t rt0 = 2 * it.pair, rt1 = rt0 + 1;
        // Q tiles of both streams (each once the stream's last S of its previous item completed)
#pragma unroll
        for (uint32_t st = 0; st < 2; ++st) {
          if (st ? it.n1 : it.n0) {
            mbar_wait(&ctl->q_empty[st], qe[st]);
            qe.flip(st);
            if (lane == 0) {
              mbar_arrive_expect_tx(&ctl->q_full[st], C::kTile);
              for (uint32_t b = 0; b < C::kBoxes; ++b)
                tma_load_3d(sq + st * C::kTile + b * kPBox, &tm_q, &ctl->q_full[st], b * 64, (rt0 + st) * 128, slot,
                            pol_q);
            }
            __syncwarp();
          }
        }
        // merged K/V schedule of the two lists
        w0base = w1base = 0xFFFFFFFFu;
        auto col_of = [&](uint32_t rt, uint32_t i, uint32_t nlist, uint32_t& wbase, uint32_t& wv) -> uint32_t {
          if constexpr (MODE == kPModeDense || MODE == kPModeNaive) {
            return i;
          } else {
            const uint32_t base = i & ~31u;
            if (base != wbase) {
              wbase = base;
              wv = base + lane < nlist ? __ldg(p.list + static_cast<uint64_t>(rt) * p.kcols + base + lane) : 0u;
            }
            return __shfl_sync(0xffffffffu, wv, i - base) & 0x7FFFFFFFu;
          }
        };
        // does list (rt, n) hold `c` at positions i+1 or i+2 inside the current window?
        auto soon = [&](uint32_t rt, uint32_t i, uint32_t nlist, uint32_t& wbase, uint32_t& wv, uint32_t c) -> bool {
          bool hit = false;
#pragma unroll
          for (uint32_t d = 1; d <= 2; ++d) {
            const uint32_t j = i + d;
            if (j < nlist && (j & ~31u) == wbase) hit |= col_of(rt, j, nlist, wbase, wv) == c;
          }
          return hit;
        };
        uint32_t i0 = 0, i1 = 0;
        const uint32_t n0 = it.n0, n1 = it.n1;
        while (i0 < n0 || i1 < n1) {
          const uint32_t a = i0 < n0 ? col_of(rt0, i0, n0, w0base, w0) : 0xFFFFFFFFu;
          const uint32_t b = i1 < n1 ? col_of(rt1, i1, n1, w1base, w1) : 0xFFFFFFFFu;
          bool use0, use1;
          if (a == b) {
            use0 = use1 = true;
          } else if (a < b) {
            use0 = true;
            use1 = i1 < n1 && !soon(rt0, i0, n0, w0base, w0, b);
          } else {
            use1 = true;
            use0 = i0 < n0 && !soon(rt1, i1, n1, w1base, w1, a);
          }
          const bool shared = use0 && use1 && a == b;
          const uint32_t f0 = (use0 && i0 == 0) ? kMetaFirst0 : 0u, f1 = (use1 && i1 == 0) ? (kMetaFirst0 << 1) : 0u;
          const uint32_t l0 = (use0 && i0 + 1 == n0) ? kMetaLast0 : 0u, l1 = (use1 && i1 + 1 == n1) ? (kMetaLast0 << 1) : 0u;
          if (shared) {
            load(&tm_k, a, kMetaS0 | (kMetaS0 << 1) | f0 | f1 | l0 | l1);
            load(&tm_v, a, kMetaV | kMetaS0 | (kMetaS0 << 1) | f0 | f1 | l0 | l1);
          } else {
            if (use0) load(&tm_k, a, kMetaS0 | f0 | l0);
            if (use1) load(&tm_k, b, (kMetaS0 << 1) | f1 | l1);
            if (use0) load(&tm_v, a, kMetaV | kMetaS0 | f0 | l0);
            if (use1) load(&tm_v, b, kMetaV | (kMetaS0 << 1) | f1 | l1);
          }
          if (use0) ++i0;
          if (use1) ++i1;
        }
      }
    } else if (warp == 1) {
      // ------------------------------------------------------------------ MMA issuer
      if (lane == 0) {
        constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
        constexpr uint32_t idesc_o = make_idesc_bf16(128, D, false, true);
        const uint32_t qaddr = smem_u32(sq), raddr = smem_u32(ring);
        uint32_t pos[2] = {0, 0}, ppos[2] = {0, 0}, pmeta[2] = {0, 0};
        bool pend[2] = {false, false}, done[2] = {false, false}, pv_out[2] = {false, false};
        PhaseBits qf{0u}, pf{0u}, pvd{0u}, oe{0x3u};
        uint32_t cons = 0;  // consumptions so far per ring slot, 4 bits each
        while (!(done[0] && done[1])) {
#pragma unroll
          for (uint32_t s = 0; s < 2; ++s) {
            if (done[s]) continue;
            if (!pend[s]) {
              const uint32_t r = pos[s] % kRing;
              if (!mbar_test(&ctl->ring_full[r], (pos[s] / kRing) & 1)) continue;
              const uint32_t m = ctl->meta[r];
              if (m & kMetaEnd) {
                done[s] = true;
                continue;
              }
              if (!(m & (kMetaS0 << s))) {
                // not this stream's load: pass it (a slot is reused only after BOTH streams have
                // passed its position, or a lagging stream could miss the meta word)
                const uint32_t c = ((cons >> (4 * r)) & 15u) + 1;
                if (c == 2) {
                  tc_commit(&ctl->ring_empty[r]);
                  cons &= ~(15u << (4 * r));
                } else {
                  cons = (cons & ~(15u << (4 * r))) | (c << (4 * r));
                }
                ++pos[s];
                continue;
              }
              pend[s] = true;
              pmeta[s] = m;
              ppos[s] = pos[s]++;
            }
            const uint32_t m = pmeta[s];
            const uint32_t r = ppos[s] % kRing;
            const bool first = m & (kMetaFirst0 << s);
            if (!(m & kMetaV)) {
              // S_s = Q_s K^T: the Q tile has landed (first of item) and PV_s(prev) has completed
              if (first && !mbar_test(&ctl->q_full[s], qf[s])) continue;
              if (pv_out[s] && !mbar_test(&ctl->pv_done[s], pvd[s])) continue;
              if (first) qf.flip(s);
              if (pv_out[s]) {
                pvd.flip(s);
                pv_out[s] = false;
              }
              tc_fence_after();
              const uint64_t qdesc = make_sdesc_sw128(qaddr + s * C::kTile, 16, 1024);
              const uint64_t kdesc = make_sdesc_sw128(raddr + r * C::kTile, 16, 1024);
#pragma unroll
              for (uint32_t kk = 0; kk < D / 16; ++kk) {
                const uint32_t off = (kk / 4) * kPBox + (kk % 4) * 32;
                umma_ss(tmem + s * 128, sdesc_advance(qdesc, off), sdesc_advance(kdesc, off), idesc_s, kk > 0);
              }
              tc_commit(&ctl->s_full[s]);
              if (m & (kMetaLast0 << s)) tc_commit(&ctl->q_empty[s]);  // Q_s free for the next item
            } else {
              // O_s += P_s V: the softmax has written P_s; the epilogue has drained O_s (first)
              if (!mbar_test(&ctl->p_full[s], pf[s])) continue;
              if (first && !mbar_test(&ctl->o_empty[s], oe[s])) continue;
              pf.flip(s);
              if (first) oe.flip(s);
              tc_fence_after();
              const uint64_t vdesc = make_sdesc_sw128(raddr + r * C::kTile, kPBox, 1024);
              const uint32_t to = tmem + C::kOCol + s * D, pc = tmem + s * 128;
#pragma unroll
              for (uint32_t kk = 0; kk < 128 / 16; ++kk)
                umma_ts(to, pc + kk * 8, sdesc_advance(vdesc, kk * 2048), idesc_o, (!first || kk > 0) ? 1u : 0u);
              tc_commit(&ctl->pv_done[s]);
              pv_out[s] = true;
              if (m & (kMetaLast0 << s)) tc_commit(&ctl->o_full[s]);
            }
            // the ring slot is free once both streams have passed its position (consumed or not)
            const uint32_t c = ((cons >> (4 * r)) & 15u) + 1;
            if (c == 2) {
              tc_commit(&ctl->ring_empty[r]);
              cons &= ~(15u << (4 * r));
            } else {
              cons = (cons & ~(15u << (4 * r))) | (c << (4 * r));
            }
            pend[s] = false;
          }
        }
      }
    }
  } else if (warp < 12) {
    setmaxnreg_inc<176>();
    // ------------------------------------------------------------------ softmax (one thread per row)
    const uint32_t s = (warp - 4) >> 2;
    const uint32_t quad = warp & 3;
    const uint32_t row = quad * 32 + lane;
    const uint32_t lane_off = (quad * 32) << 16;
    const bool neg = p.sl2 < 0.0f;
    const float abs_sl2 = fabsf(p.sl2);
    const bool ragged = (p.n % 128) != 0;
    const uint32_t last_q = p.kcols - 1;
    const uint32_t kv_valid_last = static_cast<uint32_t>(p.n - static_cast<uint64_t>(last_q) * 128);
    const uint32_t sentinel = neg ? 0x7F800000u : 0xFF800000u;
    const uint32_t ts = tmem + s * 128 + lane_off;
    const uint32_t to = tmem + C::kOCol + s * D + lane_off;
    uint32_t qi = 0, qiph = 0;
    uint32_t ntile = 0;  // this stream's tiles so far (phase of s_full / pv_done)
    PhaseBits se{1u};
    auto write_stats = [&](uint32_t slot, uint64_t grow, float m_true2, float m_run2, float l_tot) {
      if (grow < p.n) {
        const uint64_t si = static_cast<uint64_t>(slot) * p.n + grow;
        if (p.row_max) p.row_max[si] = m_true2 == -INFINITY ? -INFINITY : m_true2 * kLn2;
        if (p.row_sum) p.row_sum[si] = l_tot > 0.0f ? l_tot * exp2f(m_run2 - m_true2) : 0.0f;
      }
    };
    auto load_bits = [&](uint32_t rt, uint32_t jj, uint4& bits, uint32_t& entry) {
      const uint64_t grow = static_cast<uint64_t>(rt) * 128 + row;
      if constexpr (MODE == kPModeNaive) bits = __ldg(p.mask + grow * p.kcols + jj);
      else if constexpr (MODE != kPModeDense) bits = __ldg(p.bitmaps + (static_cast<uint64_t>(rt) * p.kcols + jj) * 128 + row);
      if constexpr (MODE == kPModeDenseBinblk) entry = pentry<MODE>(p, rt, jj);
    };
    for (;;) {
      mbar_wait(&ctl->item_full[qi], qiph);
      const PairItem it = ctl->items[qi];
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl->item_empty[qi]);
      if (++qi == kPQueue) { qi = 0; qiph ^= 1; }
      if (it.t == kPEnd) break;
      const uint32_t rt = 2 * it.pair + s;
      const uint32_t nt = s ? it.n1 : it.n0;
      if (rt >= p.krows) continue;
      const uint64_t grow = static_cast<uint64_t>(rt) * 128 + row;
      if (nt == 0) {  // fully masked row tile (engine.hpp:330-332)
        if (grow < p.n) {
          uint4* dst = reinterpret_cast<uint4*>(p.out + (static_cast<uint64_t>(it.slot) * p.n + grow) * D);
          for (uint32_t v = 0; v < D / 8; ++v) dst[v] = make_uint4(0, 0, 0, 0);
          write_stats(it.slot, grow, -INFINITY, -INFINITY, 0.0f);
        }
        continue;
      }
      float m_run = -INFINITY, m_true = -INFINITY, l0 = 0.0f, l1 = 0.0f;
      uint4 nbits = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
      uint32_t nentry = 0;
      load_bits(rt, 0, nbits, nentry);
      for (uint32_t j = 0; j < nt; ++j, ++ntile) {
        uint4 bits = nbits;
        bool masked;
        if constexpr (MODE == kPModeDense) {
          masked = ragged && j == last_q;
          if (masked) {
            uint32_t w[4];
#pragma unroll
            for (uint32_t c = 0; c < 4; ++c) {
              const int v = static_cast<int>(kv_valid_last) - static_cast<int>(c * 32);
              w[c] = v >= 32 ? 0xFFFFFFFFu : (v <= 0 ? 0u : ((1u << v) - 1u));
            }
            bits = make_uint4(w[0], w[1], w[2], w[3]);
          }
        } else if constexpr (MODE == kPModeDenseBinblk) {
          masked = (nentry & 0x80000000u) == 0;
        } else {
          masked = true;
        }
        if (j + 1 < nt) load_bits(rt, j + 1, nbits, nentry);

        mbar_wait(&ctl->s_full[s], ntile & 1);
        tc_fence_after();
#ifdef BBM_ABLATE_FAST_ENGINE  // timing experiments only: P = 0, no softmax work (MMA-side ceiling)
        if (true) {
          uint32_t z[16];
#pragma unroll
          for (uint32_t i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll
          for (uint32_t c = 0; c < 4; ++c) tmem_st16(ts + c * 16, z);
          l0 = l1 = 1.0f;
          m_run = m_true = 0.0f;
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&ctl->p_full[s]);
          continue;
        }
#endif
        uint32_t a0[32], a1[32], a2[32], a3[32];
        tmem_ld32(ts, a0);
        tmem_ld32(ts + 32, a1);
        tmem_ld32(ts + 64, a2);
        tmem_ld32(ts + 96, a3);
        tmem_ld_wait();
        if (masked) {
          if (!__all_sync(0xffffffffu, (bits.x & bits.y) == 0xFFFFFFFFu)) {
            apply_mask(a0, bits.x, sentinel);
            apply_mask(a1, bits.y, sentinel);
          }
          if (!__all_sync(0xffffffffu, (bits.z & bits.w) == 0xFFFFFFFFu)) {
            apply_mask(a2, bits.z, sentinel);
            apply_mask(a3, bits.w, sentinel);
          }
        }
        float pm0, pm1;
        if (neg) {
          pm0 = fmaxf(chunk_max<true>(a0), chunk_max<true>(a1));
          pm1 = fmaxf(chunk_max<true>(a2), chunk_max<true>(a3));
        } else {
          pm0 = fmaxf(chunk_max<false>(a0), chunk_max<false>(a1));
          pm1 = fmaxf(chunk_max<false>(a2), chunk_max<false>(a3));
        }
        float tmax = fmaxf(pm0, pm1);
        tmax = tmax == -INFINITY ? -INFINITY : tmax * abs_sl2;
        m_true = fmaxf(m_true, tmax);
        const bool need = tmax > m_run + kRescaleThreshold || (m_run == -INFINITY && tmax > -INFINITY);
        const bool rescale_o = need && j > 0 && m_run > -INFINITY;
        float factor = 1.0f;
        if (need) {
          if (m_run > -INFINITY) factor = fast_exp2(m_run - tmax);
          m_run = tmax;
        }
        if (__any_sync(0xffffffffu, rescale_o)) {
          // O_s must be quiescent: this stream's previous PV has to complete first
          mbar_wait(&ctl->pv_done[s], (ntile - 1) & 1);
          tc_fence_after();
          const float f = rescale_o ? factor : 1.0f;
#pragma unroll 1
          for (uint32_t c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(to + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (uint32_t i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
            tmem_st32(to + c * 32, o);
          }
        }
        l0 *= factor;
        l1 *= factor;
        const float m_use = m_run == -INFINITY ? 0.0f : m_run;
        const uint64_t sl2x2 = f2_pack(p.sl2, p.sl2), nm2 = f2_pack(-m_use, -m_use);
        uint32_t pk[16];
        uint64_t lacc0 = 0, lacc1 = 0;
        chunk_exp(a0, sl2x2, nm2, pk, lacc0);
        tmem_st16(ts, pk);
        chunk_exp(a1, sl2x2, nm2, pk, lacc0);
        tmem_st16(ts + 16, pk);
        chunk_exp(a2, sl2x2, nm2, pk, lacc1);
        tmem_st16(ts + 32, pk);
        chunk_exp(a3, sl2x2, nm2, pk, lacc1);
        tmem_st16(ts + 48, pk);
        l0 += f2_lo(lacc0) + f2_hi(lacc0);
        l1 += f2_lo(lacc1) + f2_hi(lacc1);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&ctl->p_full[s]);
      }
      // item end: the row statistics go out here, the row sum to the epilogue
      write_stats(it.slot, grow, m_true, m_run, l0 + l1);
      mbar_wait(&ctl->stats_empty[s], se[0]);
      se.flip(0);
      ctl->l[s][row] = l0 + l1;
      mbar_arrive(&ctl->stats_full[s]);
    }
  } else {
    setmaxnreg_dec<80>();
    // ------------------------------------------------------------------ epilogue
    const uint32_t quad = warp & 3;
    const uint32_t row = quad * 32 + lane;
    const uint32_t lane_off = (quad * 32) << 16;
    uint32_t qi = 0, qiph = 0;
    PhaseBits sf{0u}, of{0u};
    for (;;) {
      mbar_wait(&ctl->item_full[qi], qiph);
      const PairItem it = ctl->items[qi];
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl->item_empty[qi]);
      if (++qi == kPQueue) { qi = 0; qiph ^= 1; }
      if (it.t == kPEnd) break;
#pragma unroll 1
      for (uint32_t s = 0; s < 2; ++s) {
        const uint32_t rt = 2 * it.pair + s;
        const uint32_t nt = s ? it.n1 : it.n0;
        if (rt >= p.krows || nt == 0) continue;
        mbar_wait(&ctl->stats_full[s], sf[s]);
        sf.flip(s);
        const float l = ctl->l[s][row];
        mbar_arrive(&ctl->stats_empty[s]);
        mbar_wait(&ctl->o_full[s], of[s]);
        of.flip(s);
        tc_fence_after();
        const float inv = l > 0.0f ? 1.0f / l : 0.0f;
        const uint32_t to = tmem + C::kOCol + s * D + lane_off;
        const uint64_t grow = static_cast<uint64_t>(rt) * 128 + row;
        uint4* dst = reinterpret_cast<uint4*>(p.out + (static_cast<uint64_t>(it.slot) * p.n + grow) * D);
#pragma unroll
        for (uint32_t c = 0; c < D / 32; ++c) {
          uint32_t o[32];
          tmem_ld32(to + c * 32, o);
          tmem_ld_wait();
          if (c + 1 == D / 32) {
            tc_fence_before();
            mbar_arrive(&ctl->o_empty[s]);
          }
          if (grow < p.n) {
            const float* f = reinterpret_cast<const float*>(o);
#pragma unroll
            for (uint32_t v = 0; v < 4; ++v)
              dst[c * 4 + v] = make_uint4(pack_bf16x2(f[v * 8 + 0] * inv, f[v * 8 + 1] * inv),
                                          pack_bf16x2(f[v * 8 + 2] * inv, f[v * 8 + 3] * inv),
                                          pack_bf16x2(f[v * 8 + 4] * inv, f[v * 8 + 5] * inv),
                                          pack_bf16x2(f[v * 8 + 6] * inv, f[v * 8 + 7] * inv));
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&p.work_ctr[1], 1u) == gridDim.x - 1) {
      p.work_ctr[0] = 0;
      p.work_ctr[1] = 0;
      __threadfence();
    }
  }
}

template <int D, int MODE>
void launch_pair_impl(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms) {
  static_assert(pair_smem_bytes<D>() <= kSmemMax, "exceeds the 227 KB opt-in shared memory");
  const KernelMeta& km = prep.kmeta;
  std::lock_guard<std::recursive_mutex> lk(prep.mu);
  StreamCtx& ctx = prep.ctx_for(s);
  PairParams p{};
  p.n = a.n;
  p.slots = static_cast<uint32_t>(a.slots);
  p.krows = km.krows;
  p.kcols = km.kcols;
  p.npairs = (km.krows + 1) / 2;
  p.sl2 = a.scale * 1.4426950408889634f;
  if (p.sl2 == 0.0f) p.sl2 = 7.8886090522101181e-31f;  // as attn_fwd.cu: uniform weights, masked stay -inf
  p.list = km.list;
  p.row_cnt = km.row_cnt;
  p.bitmaps = km.bitmaps;
  p.mask = reinterpret_cast<const uint4*>(km.mask);
  p.work_ctr = ctx.ctr;
  p.out = static_cast<__nv_bfloat16*>(a.o);
  p.row_max = a.row_max;
  p.row_sum = a.row_sum;
  const CUtensorMap tq = cached_tmap_bf16_3d(a.q, D, a.n, a.slots, 64, 128);
  const CUtensorMap tk = cached_tmap_bf16_3d(a.k, D, a.n, a.slots, 64, 128);
  const CUtensorMap tv = cached_tmap_bf16_3d(a.v, D, a.n, a.slots, 64, 128);
  const CUtensorMap to = cached_tmap_bf16_3d(a.o, D, a.n, a.slots, 64, 128);
  static std::atomic<uint64_t> attr_devices{0};
  once_per_device(attr_devices, [] {
    BBM_CUDA(cudaFuncSetAttribute(attn_pair_kernel<D, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  pair_smem_bytes<D>()));
  });
  const uint64_t items = static_cast<uint64_t>(p.slots) * p.npairs;
  const uint32_t grid = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(items, num_sms)));
  attn_pair_kernel<D, MODE><<<grid, 512, pair_smem_bytes<D>(), s>>>(tq, tk, tv, to, p);
  BBM_CUDA(cudaGetLastError());
  mark_launch_done(ctx, s);
}

// BBM_FWD_KERNEL=single|pair (or bbm_set_fwd_kernel): which forward kernel runs (measurement,
// tests); the default is the single-stream kernel
std::atomic<int> g_fwd_kernel{-1};
int fwd_kernel_override() {
  int v = g_fwd_kernel.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = std::getenv("BBM_FWD_KERNEL");
    v = (e && std::string(e) == "single") ? 1 : ((e && std::string(e) == "pair") ? 2 : 0);
    g_fwd_kernel.store(v, std::memory_order_relaxed);
  }
  return v;
}

}  // namespace

void set_fwd_kernel(int mode) { g_fwd_kernel.store(mode, std::memory_order_relaxed); }

bool launch_attn_fwd_pair(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms) {
  // Selected explicitly only (bbm_set_fwd_kernel(2) / BBM_FWD_KERNEL=pair): measured slower than
  // attn_fwd.cu on B200.
  if (fwd_kernel_override() != 2 || a.rows) return false;
  if (a.d != 128 && a.d != 64) return false;
  const KernelMeta& km = prep.kmeta;
  if (km.kcols > 0xFFFFu || km.krows < 2) return false;
  auto go = [&](auto dtag) {
    constexpr int D = decltype(dtag)::value;
    switch (a.variant) {
      case 0: launch_pair_impl<D, kPModeDense>(prep, a, s, num_sms); break;
      case 1: launch_pair_impl<D, kPModeNaive>(prep, a, s, num_sms); break;
      case 2: launch_pair_impl<D, kPModeBinblk>(prep, a, s, num_sms); break;
      case 3: launch_pair_impl<D, kPModeDenseBinblk>(prep, a, s, num_sms); break;
      default: throw ArgError("unknown variant");
    }
  };
  if (a.d == 128) go(std::integral_constant<int, 128>{});
  else go(std::integral_constant<int, 64>{});
  return true;
}

}  // namespace bbm
