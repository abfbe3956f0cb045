// attn_fwd.cu — block-sparse masked flash-attention forward for sm_100a (TMA + tcgen05 + TMEM).
//
// Replaces the reference's blocked_forward (engine.hpp:282-341): for every (slot, query row
// tile p) it walks only the KV tiles its variant processes — the compacted occupied-tile list
// built by prep.cu for binblk / dense_binblk, all tiles for dense / naive — in ascending order
// (engine.hpp:311), with an online softmax whose fully-masked rows are exact no-ops
// (engine.hpp:206-235) and fully-masked output rows written as zeros (engine.hpp:330-332).
//
// Structure: one persistent CTA per SM (384 threads) running TWO fully independent query-tile
// streams that share the tensor core — while softmax warpgroup A turns S_A into P_A, the tensor
// core runs stream B's MMAs, and vice versa. Each stream walks its own work items (slot, row
// tile), so row tiles with different KV lists pair up freely (block-sparse masks give every row
// its own list; FA-style shared KV loops do not apply). Every role blocks in hardware
// (mbarrier try_wait) on exactly the event it needs; nothing polls.
//   warps 0, 1   TMA producer of stream A / B: Q tile per item, then K_j, V_j into the stream's
//                K/V ring (128B-swizzled 64-column boxes).
//   warps 2, 3   MMA issuer of stream A / B (one thread each; tcgen05.commit tracks the issuing
//                thread's ops, so the two streams never wait on each other's MMAs):
//                S = Q K^T (SS, both K-major) into TMEM, O += P V (TS: P read straight from
//                TMEM, V MN-major). Warp 2 also owns the TMEM allocation (512 columns:
//                S_A, S_B at [0,256), O_A, O_B at [256,512)).
//   warps 4-7    softmax + correction + epilogue of stream A (TMEM lane = query row); the
//                epilogue stages bf16 O in swizzled shared memory and writes it with TMA stores
//   warps 8-11   same for stream B
// Numerics: scores are scaled into the log2 domain; the running max is only raised when it grows
// by more than 2^8 (stale-max trick; exact after the final O/l), P is rounded to bf16 for the
// MMA and written over S in TMEM, l accumulates in fp32. Partial tiles read 16 B of mask bits
// per row (coalesced, tile-major); full tiles read none.
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
  uint64_t* trace;       // optional event trace (bbm_set_trace), nullptr = off
  uint32_t trace_ctas;   // CTAs that record
};

constexpr uint32_t kThreads = 384;
constexpr uint32_t kTraceCap = 8192;  // events per traced CTA

// Trace event: [63:24] clock64 low 40 bits | [23:16] code | [15] stream | [14:0] aux.
// Codes: producer 1 Q issued (aux = item), 2 K_j issued, 3 V_j issued;
//        MMA 10 S_j issued, 11 PV_j issued;
//        softmax 20 s_full wait begin, 21 s_full wait end, 22 p_full arrive, 23 o_full wait end,
//        24 epilogue done.
__device__ __forceinline__ void trace_ev(bool on, const FwdParams& p, uint32_t* counter,
                                         uint32_t code, uint32_t stream, uint32_t aux) {
  if (!on) return;
  const uint32_t i = atomicAdd(counter, 1u);
  if (i >= kTraceCap) return;
  const uint64_t t = static_cast<uint64_t>(clock64()) & ((1ull << 40) - 1);
  p.trace[static_cast<uint64_t>(blockIdx.x) * kTraceCap + i] =
      (t << 24) | (static_cast<uint64_t>(code & 0xFF) << 16) | ((stream & 1u) << 15) | (aux & 0x7FFF);
}
constexpr uint32_t kBoxBytes = 128 * 64 * 2;  // 128 rows x 64 bf16, one 128B-swizzle box
constexpr float kRescaleThreshold = 8.0f;     // log2 units
constexpr float kLn2 = 0.69314718055994530942f;

constexpr uint32_t kMetaRows = 256;  // row tiles whose order / count are staged in smem

template <int D>
struct Cfg {
  static constexpr uint32_t kBoxes = D / 64;
  static constexpr uint32_t kTileBytes = kBoxes * kBoxBytes;  // one 128 x D bf16 tile
  static constexpr uint32_t kRing = (D == 64) ? 5 : 2;        // K/V ring slots per stream
  static constexpr uint32_t kStageBytes = kBoxBytes;          // epilogue staging per stream
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kOCol = 256;
};

// Everything that is not a tile lives behind the tiles in the same dynamic allocation (no static
// smem, so the dynamic base is the 1024-byte aligned start of the CTA's window).
template <uint32_t kRing>
struct SmemCtl {
  uint64_t q_full[2], q_empty[2], s_full[2], p_full[2], o_full[2];
  uint64_t ring_full[2][kRing], ring_empty[2][kRing];
  uint32_t tmem_base;
  uint32_t trace_count;
  float xchg[2][2][128];  // [exchange parity][half][row]: partial row max / row sum
  uint16_t cnt[kMetaRows];   // row_cnt, staged when krows <= kMetaRows
  uint8_t order[kMetaRows];  // LPT order (row tile < 256), staged likewise
};

template <int D>
constexpr uint32_t smem_bytes() {
  return Cfg<D>::kTileBytes * (2 + 2 * Cfg<D>::kRing) + 2 * Cfg<D>::kStageBytes +
         sizeof(SmemCtl<Cfg<D>::kRing>);
}

template <int MODE>
__device__ __forceinline__ uint32_t tiles_of(const FwdParams& p, const uint32_t* cnt,
                                             uint32_t row_tile) {
  if constexpr (MODE == kModeDense || MODE == kModeNaive) return p.kcols;
  else return cnt[row_tile];
}

template <int MODE>
__device__ __forceinline__ uint32_t entry_of(const FwdParams& p, uint32_t row_tile, uint32_t j) {
  if constexpr (MODE == kModeDense || MODE == kModeNaive) return j;
  else return p.list[static_cast<uint64_t>(row_tile) * p.kcols + j];
}

// Work item t -> (slot, row tile): slot-major (K/V reuse across a slot's row tiles stays in L2),
// row tiles in LPT order inside a slot.
struct Item {
  uint32_t t, slot, rt, nt;
};

// Row order / counts come from the smem copies when krows <= kMetaRows, else from global.
struct MetaView {
  const uint8_t* order_s;
  const uint16_t* cnt_s;
  const uint32_t* order_g;
  const uint32_t* cnt_g;
  bool staged;
};

template <int MODE>
__device__ __forceinline__ Item make_item(const FwdParams& p, const MetaView& mv, uint32_t t) {
  Item it;
  it.t = t;
  it.slot = t / p.krows;
  const uint32_t k = t - it.slot * p.krows;
  it.rt = mv.staged ? mv.order_s[k] : mv.order_g[k];
  if constexpr (MODE == kModeDense || MODE == kModeNaive) it.nt = p.kcols;
  else it.nt = mv.staged ? mv.cnt_s[it.rt] : mv.cnt_g[it.rt];
  return it;
}

// Next item with work (nt > 0) of a stream whose items are t0, t0 + stride, ...
template <int MODE>
__device__ __forceinline__ bool next_busy_item(const FwdParams& p, const MetaView& mv, uint32_t& t,
                                               uint32_t stride, Item& it) {
  for (; t < p.total_items; t += stride) {
    it = make_item<MODE>(p, mv, t);
    if (it.nt > 0) return true;
  }
  return false;
}

// Masked max of 32 raw scores of one row chunk (negated first when the scale is negative).
template <bool kMasked, bool kNeg>
__device__ __forceinline__ float chunk_max(const uint32_t (&r)[32], uint32_t mw) {
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (uint32_t i = 0; i < 32; i += 4) {
    float a = __uint_as_float(r[i]), b = __uint_as_float(r[i + 1]);
    float c = __uint_as_float(r[i + 2]), d = __uint_as_float(r[i + 3]);
    if constexpr (kNeg) { a = -a; b = -b; c = -c; d = -d; }
    if constexpr (kMasked) {
      a = ((mw >> i) & 1u) ? a : -INFINITY;
      b = ((mw >> (i + 1)) & 1u) ? b : -INFINITY;
      c = ((mw >> (i + 2)) & 1u) ? c : -INFINITY;
      d = ((mw >> (i + 3)) & 1u) ? d : -INFINITY;
    }
    m0 = fmax3(m0, a, b);
    m1 = fmax3(m1, c, d);
  }
  return fmaxf(m0, m1);
}

// P chunk: 32 scores -> 16 packed bf16x2; accumulates the fp32 sum of the unrounded
// exponentials into the packed pair `lacc`. Scale/shift and the sum run two lanes per
// instruction (FFMA2 / FADD2).
template <bool kMasked>
__device__ __forceinline__ void chunk_exp(const uint32_t (&r)[32], uint32_t mw, uint64_t sl2x2,
                                          uint64_t neg_m_x2, uint32_t (&pk)[16], uint64_t& lacc) {
#pragma unroll
  for (uint32_t i = 0; i < 32; i += 2) {
    const uint64_t x = ffma2(f2_pack(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sl2x2,
                             neg_m_x2);
    float x0 = f2_lo(x), x1 = f2_hi(x);
    if constexpr (kMasked) {
      x0 = ((mw >> i) & 1u) ? x0 : -INFINITY;
      x1 = ((mw >> (i + 1)) & 1u) ? x1 : -INFINITY;
    }
    const float e0 = fast_exp2(x0), e1 = fast_exp2(x1);
    lacc = fadd2(lacc, f2_pack(e0, e1));
    pk[i / 2] = pack_bf16x2(e0, e1);
  }
}

template <int D, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                    const FwdParams p) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sq = smem;                      // [2][tile]     Q of each stream
  uint8_t* ring = sq + 2 * C::kTileBytes;  // [2][kRing][tile] K/V ring of each stream
  uint8_t* stage = ring + 2 * C::kRing * C::kTileBytes;  // [2][128 x 64 bf16] epilogue staging
  auto* ctl = reinterpret_cast<SmemCtl<C::kRing>*>(stage + 2 * C::kStageBytes);
  uint64_t* bar_q_full = ctl->q_full;
  uint64_t* bar_q_empty = ctl->q_empty;
  uint64_t* bar_s_full = ctl->s_full;
  uint64_t* bar_p_full = ctl->p_full;
  uint64_t* bar_o_full = ctl->o_full;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t stride = 2 * gridDim.x;  // items of stream s: 2*blockIdx.x + s + k*stride
  if ((smem_u32(smem) & 1023u) != 0) __trap();  // 128B-swizzle atoms need 1024-byte alignment

  const bool staged = p.krows <= kMetaRows;
  if (staged) {
    for (uint32_t i = threadIdx.x; i < p.krows; i += blockDim.x) {
      ctl->order[i] = static_cast<uint8_t>(p.order[i]);
      ctl->cnt[i] = static_cast<uint16_t>(p.row_cnt[i]);
    }
  }
  const MetaView mv{ctl->order, ctl->cnt, p.order, p.row_cnt, staged};
  const bool tracing = p.trace != nullptr && blockIdx.x < p.trace_ctas;

  if (threadIdx.x == 0) {
    ctl->trace_count = 0;
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_q_full[s], 1);
      mbar_init(&bar_q_empty[s], 1);
      mbar_init(&bar_s_full[s], 1);
      mbar_init(&bar_p_full[s], 256);
      mbar_init(&bar_o_full[s], 1);
    }
    for (int s = 0; s < 2; ++s)
      for (uint32_t r = 0; r < C::kRing; ++r) {
        mbar_init(&ctl->ring_full[s][r], 1);
        mbar_init(&ctl->ring_empty[s][r], 1);
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
    tmem_alloc<C::kTmemCols>(&ctl->tmem_base);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl->tmem_base;

  if (warp < 2) {
    // ------------------------------------------------------------------ TMA producer (stream = warp)
    if (lane == 0) {
      const int s = static_cast<int>(warp);
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      uint32_t r = 0, rph = 1, qph = 1;
      uint8_t* myring = ring + s * C::kRing * C::kTileBytes;
      auto load_tile = [&](const CUtensorMap* tm, uint32_t q, uint32_t slot, uint32_t code,
                           uint32_t j) {
        mbar_wait(&ctl->ring_empty[s][r], rph);
        uint64_t* full = &ctl->ring_full[s][r];
        mbar_arrive_expect_tx(full, C::kTileBytes);
        for (uint32_t b = 0; b < C::kBoxes; ++b)
          tma_load_3d(myring + r * C::kTileBytes + b * kBoxBytes, tm, full, b * 64, q * 128, slot,
                      pol_kv);
        trace_ev(tracing, p, &ctl->trace_count, code, s, j);
        if (++r == C::kRing) { r = 0; rph ^= 1; }
      };
      Item it;
      for (uint32_t t = 2 * blockIdx.x + s; next_busy_item<MODE>(p, mv, t, stride, it); t += stride) {
        // list entries one tile ahead so the TMA issue never waits on an L2 load
        uint32_t cur = entry_of<MODE>(p, it.rt, 0);
        mbar_wait(&bar_q_empty[s], qph);
        qph ^= 1;
        mbar_arrive_expect_tx(&bar_q_full[s], C::kTileBytes);
        for (uint32_t b = 0; b < C::kBoxes; ++b)
          tma_load_3d(sq + s * C::kTileBytes + b * kBoxBytes, &tm_q, &bar_q_full[s], b * 64,
                      it.rt * 128, it.slot, pol_q);
        trace_ev(tracing, p, &ctl->trace_count, 1, s, t);
        for (uint32_t j = 0; j < it.nt; ++j) {
          const uint32_t nxt = (j + 1 < it.nt) ? entry_of<MODE>(p, it.rt, j + 1) : 0;
          const uint32_t q = cur & 0x7FFFFFFFu;
          load_tile(&tm_k, q, it.slot, 2, j);
          load_tile(&tm_v, q, it.slot, 3, j);
          cur = nxt;
        }
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------------ MMA issuer (stream = warp-2)
    // Op sequence S_0, PV_0, S_1, PV_1, ...: S_{j+1} overwrites the TMEM columns P_j lives in,
    // so it is issued after PV_j (tcgen05.mma executes in issue order).
    if (lane == 0) {
      const int s = static_cast<int>(warp) - 2;
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, D, false, true);
      const uint32_t qbase = smem_u32(sq) + s * C::kTileBytes;
      const uint32_t rbase = smem_u32(ring) + s * C::kRing * C::kTileBytes;
      const uint32_t tmem_s = tmem + s * 128, tmem_o = tmem + C::kOCol + s * 128;
      uint32_t r = 0, rph = 0, qph = 0, pph = 0;
      Item it;
      for (uint32_t t = 2 * blockIdx.x + s; next_busy_item<MODE>(p, mv, t, stride, it); t += stride) {
        mbar_wait(&bar_q_full[s], qph);
        qph ^= 1;
        for (uint32_t j = 0; j < it.nt; ++j) {
          // S_j = Q K_j^T
          mbar_wait(&ctl->ring_full[s][r], rph);
          tc_fence_after();
          const uint32_t kbase = rbase + r * C::kTileBytes;
#pragma unroll
          for (uint32_t kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk / 4) * kBoxBytes + (kk % 4) * 32;
            umma_ss(tmem_s, make_sdesc_sw128(qbase + off, 16, 1024),
                    make_sdesc_sw128(kbase + off, 16, 1024), idesc_s, kk > 0);
          }
          tc_commit(&ctl->ring_empty[s][r]);
          if (++r == C::kRing) { r = 0; rph ^= 1; }
          if (j + 1 == it.nt) tc_commit(&bar_q_empty[s]);
          tc_commit(&bar_s_full[s]);
          trace_ev(tracing, p, &ctl->trace_count, 10, s, j);
          // O += P_j V_j
          mbar_wait(&bar_p_full[s], pph);
          pph ^= 1;
          mbar_wait(&ctl->ring_full[s][r], rph);
          tc_fence_after();
          const uint32_t vbase = rbase + r * C::kTileBytes;
#pragma unroll
          for (uint32_t kk = 0; kk < 128 / 16; ++kk)
            umma_ts(tmem_o, tmem_s + kk * 8, make_sdesc_sw128(vbase + kk * 2048, kBoxBytes, 1024),
                    idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          tc_commit(&ctl->ring_empty[s][r]);
          if (++r == C::kRing) { r = 0; rph ^= 1; }
          if (j + 1 == it.nt) tc_commit(&bar_o_full[s]);
          trace_ev(tracing, p, &ctl->trace_count, 11, s, j);
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ softmax engine
    // ONE engine of 8 warps serves both streams in turn (A, B, A, B, ...): while it turns S_A
    // into P_A the tensor core runs stream B's MMAs, and vice versa. Warps 4-7 own S/O columns
    // [0, 64) / [0, D/2), warps 8-11 the other half; the two halves exchange their partial row
    // max through shared memory once per tile, so both hold identical softmax state.
    const uint32_t half = (warp >= 8) ? 1u : 0u;
    const uint32_t quad = warp & 3;
    const uint32_t row = quad * 32 + lane;
    const uint32_t lane_off = (quad * 32) << 16;
    const bool leader = (warp == 4 && lane == 0);
    const bool tracer = (quad == 0 && lane == 0 && half == 0);
    const bool ragged = (p.n % 128) != 0;
    const uint32_t last_q = p.kcols - 1;
    const uint32_t kv_valid_last = static_cast<uint32_t>(p.n - static_cast<uint64_t>(last_q) * 128);
    const bool neg = p.sl2 < 0.0f;
    const float abs_sl2 = fabsf(p.sl2);
    constexpr uint32_t kHalfO = D / 2;  // O columns per half

    struct Stream {
      uint32_t t, j, s_phase, o_phase;
      Item it;
      float m_run, m_true, l;
      bool live;  // has an item with tiles in progress
      bool pend;  // finished item waiting for its epilogue
      Item eit;   // item of the pending epilogue
      float e_m_run, e_m_true, e_l;
      uint2 nbits;      // this half's mask bits of tile j, loaded a turn ahead
      uint32_t nentry;  // list entry of tile j (dense_binblk: the full flag), a turn ahead
    } st[2];

    // loads for tile j of the current item, issued one engine turn before they are needed; the
    // bitmap address depends only on (row tile, list position), never on a loaded value
    auto prefetch = [&](Stream& x) {
      if (!x.live) return;
      const uint64_t grow = static_cast<uint64_t>(x.it.rt) * 128 + row;
      if constexpr (MODE == kModeNaive)
        x.nbits = __ldg(reinterpret_cast<const uint2*>(p.mask + grow * p.kcols + x.j) + half);
      else if constexpr (MODE != kModeDense)
        x.nbits = __ldg(reinterpret_cast<const uint2*>(
                            p.bitmaps + (static_cast<uint64_t>(x.it.rt) * p.kcols + x.j) * 128 + row) +
                        half);
      if constexpr (MODE == kModeDenseBinblk) x.nentry = entry_of<MODE>(p, x.it.rt, x.j);
    };

    // zero rows / stats for items without any tile (fully masked row tiles)
    auto zero_item = [&](const Item& it) {
      const uint64_t grow = static_cast<uint64_t>(it.rt) * 128 + row;
      if (grow >= p.n) return;
      uint4* dst = reinterpret_cast<uint4*>(p.out + (static_cast<uint64_t>(it.slot) * p.n + grow) * D +
                                            half * kHalfO);
      for (uint32_t v = 0; v < kHalfO / 8; ++v) dst[v] = make_uint4(0, 0, 0, 0);
      if (half == 0) {
        const uint64_t si = static_cast<uint64_t>(it.slot) * p.n + grow;
        if (p.row_max) p.row_max[si] = -INFINITY;
        if (p.row_sum) p.row_sum[si] = 0.0f;
      }
    };
    // advance stream x to its next item that has tiles (writing zero items on the way)
    auto next_item = [&](Stream& x) {
      x.live = false;
      for (; x.t < p.total_items; x.t += stride) {
        const Item it = make_item<MODE>(p, mv, x.t);
        if (it.nt == 0) {
          zero_item(it);
          continue;
        }
        x.it = it;
        x.j = 0;
        x.m_run = -INFINITY;
        x.m_true = -INFINITY;
        x.l = 0.0f;
        x.live = true;
        x.t += stride;
        break;
      }
    };
    for (int s = 0; s < 2; ++s) {
      st[s].t = 2 * blockIdx.x + s;
      st[s].s_phase = st[s].o_phase = 0;
      st[s].pend = false;
      next_item(st[s]);
      prefetch(st[s]);
    }
    uint32_t step = 0;  // parity selects the max-exchange buffer

    while (st[0].live || st[0].pend || st[1].live || st[1].pend) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        Stream& x = st[s];
        const uint32_t ts = tmem + s * 128 + lane_off;
        const uint32_t to = tmem + C::kOCol + s * 128 + lane_off;
        // ---------------- deferred epilogue of this stream's previous item (its last PV ran
        // while the engine served the other stream)
        if (x.pend) {
          x.pend = false;
          mbar_wait(&bar_o_full[s], x.o_phase);
          x.o_phase ^= 1;
          tc_fence_after();
          if (tracer) trace_ev(tracing, p, &ctl->trace_count, 23, s, x.eit.t);
          // total row sum = both halves' partial sums
          ctl->xchg[step & 1][half][row] = x.e_l;
          named_bar_sync(1, 256);
          const float l_tot = x.e_l + ctl->xchg[step & 1][half ^ 1][row];
          ++step;
          const float inv = l_tot > 0.0f ? 1.0f / l_tot : 0.0f;
          if (leader) bulk_wait_group_read<0>();  // staging buffers free again
          named_bar_sync(1, 256);
          // D=128: half h stages columns [64h, 64h+64) in buffer h; D=64: both halves share
          // buffer 0, 32 columns (4 chunks) each
          uint8_t* stg = stage + (D == 128 ? half * C::kStageBytes : 0);
          uint8_t* rowp = stg + row * 128;
#pragma unroll
          for (uint32_t c32 = 0; c32 < kHalfO / 32; ++c32) {
            uint32_t o[32];
            tmem_ld32(to + half * kHalfO + c32 * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (uint32_t c = 0; c < 4; ++c) {
              const uint32_t chunk = (D == 128 ? c32 * 4 : half * 4) + c;
              uint4 w;
              w.x = pack_bf16x2(__uint_as_float(o[c * 8 + 0]) * inv, __uint_as_float(o[c * 8 + 1]) * inv);
              w.y = pack_bf16x2(__uint_as_float(o[c * 8 + 2]) * inv, __uint_as_float(o[c * 8 + 3]) * inv);
              w.z = pack_bf16x2(__uint_as_float(o[c * 8 + 4]) * inv, __uint_as_float(o[c * 8 + 5]) * inv);
              w.w = pack_bf16x2(__uint_as_float(o[c * 8 + 6]) * inv, __uint_as_float(o[c * 8 + 7]) * inv);
              *reinterpret_cast<uint4*>(rowp + ((chunk ^ (row & 7)) << 4)) = w;
            }
          }
          // O TMEM of this stream may now be overwritten (its next first PV waits for this
          // engine's next p_full arrival on this stream, which comes later)
          tc_fence_before();
          fence_proxy_async_smem();
          named_bar_sync(1, 256);
          if (leader) {
            tma_store_3d(&tm_o, stage, 0, x.eit.rt * 128, x.eit.slot);
            if (D == 128) tma_store_3d(&tm_o, stage + C::kStageBytes, 64, x.eit.rt * 128, x.eit.slot);
            bulk_commit_group();
          }
          const uint64_t grow = static_cast<uint64_t>(x.eit.rt) * 128 + row;
          if (half == 0 && grow < p.n) {
            const uint64_t si = static_cast<uint64_t>(x.eit.slot) * p.n + grow;
            if (p.row_max) p.row_max[si] = x.e_m_true == -INFINITY ? -INFINITY : x.e_m_true * kLn2;
            if (p.row_sum)
              p.row_sum[si] = l_tot > 0.0f ? l_tot * fast_exp2(x.e_m_run - x.e_m_true) : 0.0f;
          }
          if (tracer) trace_ev(tracing, p, &ctl->trace_count, 24, s, x.eit.t);
        }
        if (!x.live) continue;

        // ---------------- one tile of this stream
        const uint32_t j = x.j;
        bool masked;
        uint2 bits = x.nbits;
        if constexpr (MODE == kModeDense) {
          // only the ragged right edge needs a column bound (no bitmap in this mode)
          masked = ragged && j == last_q;
          if (masked) {
            const int v = static_cast<int>(kv_valid_last) - static_cast<int>(half * 64);
            bits.x = v >= 32 ? 0xFFFFFFFFu : (v <= 0 ? 0u : ((1u << v) - 1u));
            bits.y = v >= 64 ? 0xFFFFFFFFu : (v <= 32 ? 0u : ((1u << (v - 32)) - 1u));
          }
        } else if constexpr (MODE == kModeDenseBinblk) {
          masked = (x.nentry & 0x80000000u) == 0;  // full tiles skip the mask bits
        } else {
          masked = true;  // bitmaps carry zeros beyond n, so ragged edges need nothing extra
        }

        if (tracer) trace_ev(tracing, p, &ctl->trace_count, 20, s, j);
        mbar_wait(&bar_s_full[s], x.s_phase);
        x.s_phase ^= 1;
        tc_fence_after();
        if (tracer) trace_ev(tracing, p, &ctl->trace_count, 21, s, j);

        uint32_t a0[32], a1[32];
        tmem_ld32(ts + half * 64, a0);
        tmem_ld32(ts + half * 64 + 32, a1);
        tmem_ld_wait();
        float pmax;
        if (masked) {
          pmax = neg ? fmaxf(chunk_max<true, true>(a0, bits.x), chunk_max<true, true>(a1, bits.y))
                     : fmaxf(chunk_max<true, false>(a0, bits.x), chunk_max<true, false>(a1, bits.y));
        } else {
          pmax = neg ? fmaxf(chunk_max<false, true>(a0, 0), chunk_max<false, true>(a1, 0))
                     : fmaxf(chunk_max<false, false>(a0, 0), chunk_max<false, false>(a1, 0));
        }
        // exchange with the other half (double-buffered by step parity); after this barrier
        // every S read of this tile has completed, so P may overwrite S columns [0, 64)
        ctl->xchg[step & 1][half][row] = pmax;
        named_bar_sync(1, 256);
        float tmax = fmaxf(pmax, ctl->xchg[step & 1][half ^ 1][row]);
        ++step;
        tmax = tmax == -INFINITY ? -INFINITY : tmax * abs_sl2;  // log2 domain
        x.m_true = fmaxf(x.m_true, tmax);
        const bool need = tmax > x.m_run + kRescaleThreshold || (x.m_run == -INFINITY && tmax > -INFINITY);
        const bool rescale_o = need && j > 0 && x.m_run > -INFINITY;
        float factor = 1.0f;
        if (need) {
          if (x.m_run > -INFINITY) factor = fast_exp2(x.m_run - tmax);
          x.m_run = tmax;
        }
        if (__any_sync(0xffffffffu, rescale_o)) {
          const float f = rescale_o ? factor : 1.0f;
#pragma unroll 1
          for (uint32_t c = 0; c < kHalfO / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(to + half * kHalfO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (uint32_t i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
            tmem_st32(to + half * kHalfO + c * 32, o);
          }
        }
        x.l *= factor;
        const float m_use = x.m_run == -INFINITY ? 0.0f : x.m_run;
        uint32_t pk[16];
        uint64_t lacc = 0;
        const uint64_t sl2x2 = f2_pack(p.sl2, p.sl2), nm2 = f2_pack(-m_use, -m_use);
        // this half's 64 columns -> 32 packed P columns at [32 * half, 32 * half + 32)
        if (masked) {
          chunk_exp<true>(a0, bits.x, sl2x2, nm2, pk, lacc);
          tmem_st16(ts + half * 32, pk);
          chunk_exp<true>(a1, bits.y, sl2x2, nm2, pk, lacc);
          tmem_st16(ts + half * 32 + 16, pk);
        } else {
          chunk_exp<false>(a0, 0, sl2x2, nm2, pk, lacc);
          tmem_st16(ts + half * 32, pk);
          chunk_exp<false>(a1, 0, sl2x2, nm2, pk, lacc);
          tmem_st16(ts + half * 32 + 16, pk);
        }
        x.l += f2_lo(lacc) + f2_hi(lacc);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bar_p_full[s]);
        if (tracer) trace_ev(tracing, p, &ctl->trace_count, 22, s, j);

        if (++x.j == x.it.nt) {  // item done: epilogue on this stream's next turn
          x.pend = true;
          x.eit = x.it;
          x.e_m_run = x.m_run;
          x.e_m_true = x.m_true;
          x.e_l = x.l;
          next_item(x);
        }
        prefetch(x);
      }
    }
  }

  if (warp == 4 && lane == 0) bulk_wait_group<0>();  // O stores landed
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<C::kTmemCols>(tmem);
}

template <int D, int MODE>
void launch_impl(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms) {
  static_assert(smem_bytes<D>() <= 232448, "exceeds the 227 KB opt-in shared memory");
  const KernelMeta& km = prep.kmeta;
  const CUtensorMap tq = make_tmap_bf16_3d(a.q, D, a.n, a.slots, 64, 128);
  const CUtensorMap tk = make_tmap_bf16_3d(a.k, D, a.n, a.slots, 64, 128);
  const CUtensorMap tv = make_tmap_bf16_3d(a.v, D, a.n, a.slots, 64, 128);
  const CUtensorMap to = make_tmap_bf16_3d(a.o, D, a.n, a.slots, 64, 128);
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
  p.trace = static_cast<uint64_t*>(g_trace.buffer);
  p.trace_ctas = g_trace.ctas;
  static bool attr_set = false;  // per (D, MODE) instantiation
  if (!attr_set) {
    BBM_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<D, MODE>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<D>()));
    attr_set = true;
  }
  // two item streams per CTA, at most one CTA per SM (the kernel owns the SM's whole TMEM)
  const uint32_t grid =
      std::min<uint32_t>((p.total_items + 1) / 2, static_cast<uint32_t>(num_sms));
  attn_fwd_kernel<D, MODE><<<grid, kThreads, smem_bytes<D>(), s>>>(tq, tk, tv, to, p);
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
