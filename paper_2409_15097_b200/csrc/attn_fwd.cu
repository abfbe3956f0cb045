// attn_fwd.cu — block-sparse masked flash-attention forward for sm_100a (TMA + tcgen05 + TMEM).
//
// Replaces the reference's blocked_forward (engine.hpp:282-341): for every (slot, query row
// tile p) it walks only the KV tiles its variant processes — the compacted occupied-tile list
// built by prep.cu for binblk / dense_binblk, all tiles for dense / naive — in ascending order
// (engine.hpp:311), with an online softmax whose fully-masked rows are exact no-ops
// (engine.hpp:206-235) and fully-masked output rows written as zeros (engine.hpp:330-332).
//
// Work: a (slot, row unit) item, where a row unit is a row tile's whole KV list or — for rows
// longer than the launch's unit length L — one balanced chunk of it (split-KV). Chunks write
// unnormalized partials (O, running max, sum) to a workspace and the last chunk to finish
// combines them. Items are claimed dynamically (one global atomic per item) in slot-major order,
// longest units first inside a slot.
//
// Structure: one persistent CTA per SM (512 threads = four warpgroups, registers rebalanced with
// setmaxnreg), one stream of items (the tile sequence of consecutive items is treated as one
// sequence k = 0, 1, 2, ...). The score accumulator is triple-buffered in TMEM, so S_{k+1} and
// S_{k+2} are computed while the softmax engine turns S_k into P_k.
//   warp 0       producer: claims items, publishes them through a shared-memory item queue,
//                loads Q (double-buffered across items) and K_k, V_k into a K/V ring (TMA,
//                128B-swizzled 64-column boxes).
//   warps 1, 3   MMA issuers (one thread each): warp 1 S_k = Q K_k^T (SS, both K-major) into
//                TMEM buffer k % 3 once PV_{k-3} has completed (S_{k+3} reuses P_k's columns);
//                warp 3 O += P_k V_k (TS: P read from TMEM, V MN-major).
//   warp 2       TMEM allocator (512 columns: S buffers at 0, 128, 256; O at 384 — at d=64 two O
//                accumulators at 384 and 448, alternating between items).
//   warps 4-11   softmax engine (168 registers): warps 4-7 own S columns [0,64), warps 8-11 the
//                other half; the halves exchange their partial row max through shared memory
//                once per tile. At an item's end the engine hands its row statistics to the
//                epilogue warpgroup through shared memory (ItemStats) and moves on.
//   warps 12-15  epilogue (88 registers): waits for an item's last PV, reads O out of TMEM and
//                releases the accumulator, then writes O / l as bf16 one 64-column box at a time
//                through a 128B-swizzled staging box and TMA stores (or a split-KV partial).
// Numerics: scores are scaled into the log2 domain; the running max is only raised when it grows
// by more than 2^8 (stale-max trick; exact after the final O/l), P is rounded to bf16 for the
// MMA and written over S in TMEM, l accumulates in fp32. Partial tiles read 8 B of mask bits per
// row and half (coalesced, list-position tile-major, prefetched a tile ahead); full tiles read
// none under dense_binblk.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "bbm_internal.h"
#include "bbm_ptx.cuh"
#include "bbm_softmax.cuh"
#include "bbm_tmap.h"

namespace bbm {
namespace {

using namespace ptx;
using namespace softmax;

enum Mode : int { kModeBinblk = 0, kModeDenseBinblk = 1, kModeDense = 2, kModeNaive = 3 };

constexpr uint32_t kEnd = 0xFFFFFFFFu;

struct FwdParams {
  uint64_t n;
  uint32_t slots;
  uint32_t krows, kcols;
  const PlanHdr* hdr;    // device plan header: row units per slot, split rows / chunks
  float sl2;             // scale * log2(e)
  const uint32_t* list;
  const uint8_t* halves;   // per list position: key half 0 / 1 empty for the whole tile (bit 0 / 1),
                           // nullptr = load and multiply whole tiles
  const uint4* bitmaps;
  const uint4* mask;        // padded packed mask, kcols uint4 per row
  const uint4* unit_desc;   // [units] {row tile, j0, tiles, split (kNoSplit | row << 8 | chunk)}
  const uint2* split_info;  // [split rows] {chunks, first workspace chunk}
  float* ws;             // [slots][split_chunks][128 * (D + 3)] partial O | m_run | m_true | l
  uint32_t* split_ctr;   // [slots][split_rows] finished chunks (reset by the combiner)
  uint32_t* work_ctr;    // [2] next item, finished CTAs (reset by the last CTA; per stream)
  __nv_bfloat16* out;
  float* row_max;
  float* row_sum;
  const uint32_t* rows;  // gather mode: token of each (permuted) row position, new -> old [n]
  const __nv_bfloat16* qg;  // LSU gather mode (kGather == 3): Q / K / V in the caller's token order
  const __nv_bfloat16* kg;
  const __nv_bfloat16* vg;
  uint64_t* trace;       // optional event trace (bbm_set_trace), nullptr = off
  uint32_t trace_ctas;   // CTAs that record
};

// Softmax engine split: kParts warps per TMEM lane quadrant, each owning 128/kParts score
// columns and D/kParts output columns of its 32 rows.
#ifndef BBM_PARTS128
#define BBM_PARTS128 2
#endif
template <int D>
constexpr uint32_t kParts = D == 128 ? BBM_PARTS128 : 2;
// warpgroup 0: producer / MMA issuers / TMEM allocator; 1..kParts: softmax engine; last: epilogue
template <int D>
constexpr uint32_t kThreadsOf = 256 + 128 * kParts<D>;
#ifndef BBM_ENGINE_REGS
#define BBM_ENGINE_REGS 168
#endif
// setmaxnreg moves registers between the warpgroups of the CTA's launch allocation (the launch
// register count x threads): 2 parts: 512 threads x 128 = 2 x 128 x 168 (engine) + 2 x 128 x 88;
// 4 parts: 768 threads x 80 = 4 x 128 x 88 + 2 x 128 x 64.
template <int D>
constexpr uint32_t kLaunchRegs = (65536 / kThreadsOf<D>) / 8 * 8;
template <int D>
constexpr uint32_t kEngineRegs = kParts<D> == 2 ? BBM_ENGINE_REGS : 88;
template <int D>
constexpr uint32_t kOtherRegs = (kLaunchRegs<D> * (2 + kParts<D>) - kParts<D> * kEngineRegs<D>) / 2;
static_assert(kOtherRegs<128> % 8 == 0 && kOtherRegs<128> >= 56, "register split");
constexpr uint32_t kTraceCap = 8192;  // events per traced CTA
constexpr uint32_t kQueue = 8;        // item queue depth (items open between the producer and the PV issuer)

// Trace event: [63:24] clock64 low 40 bits | [23:16] code | [15] stream | [14:0] aux.
// Codes: producer 1 Q issued (aux = item), 2 K_k issued, 3 V_k issued;
//        MMA 10 S_k issued, 11 PV_k issued, 12 V_k landed, 13 K_k landed, 14 P_k seen;
//        softmax 20 s_full wait begin, 21 s_full wait end, 22 p_full arrive, 23 o_full wait end,
//        24 epilogue done, 25 S in registers, 26 row max exchanged, 27 P computed,
//        28 item statistics handed over, 29 next item's descriptor read.
template <bool kTrace>
__device__ __forceinline__ void trace_ev(bool on, const FwdParams& p, uint32_t* counter,
                                         uint32_t code, uint32_t stream, uint32_t aux) {
  if constexpr (!kTrace) return;
  if (!on) return;
  const uint32_t i = atomicAdd(counter, 1u);
  if (i >= kTraceCap) return;
  const uint64_t t = static_cast<uint64_t>(clock64()) & ((1ull << 40) - 1);
  p.trace[static_cast<uint64_t>(blockIdx.x) * kTraceCap + i] =
      (t << 24) | (static_cast<uint64_t>(code & 0xFF) << 16) | ((stream & 1u) << 15) | (aux & 0x7FFF);
}

constexpr uint32_t kBoxBytes = 128 * 64 * 2;  // 128 rows x 64 bf16, one 128B-swizzle box

// S buffers in TMEM: S_{k+kSBufs} is issued once PV_k (the last reader of P_k, written over S_k)
// has completed, so the S issuer runs kSBufs tiles ahead of the PV issuer. TMEM at D = 128:
// S at 0, 128 and 256, one O accumulator at 384 (the whole 512-column allocation; the epilogue
// warpgroup releases it as soon as it has read it out); at D = 64 two O accumulators.
#ifndef BBM_SBUFS
#define BBM_SBUFS 3
#endif
constexpr uint32_t kSBufs = BBM_SBUFS;
// O accumulators behind the S buffers: two (items alternate) when they fit, else one
template <int D>
constexpr uint32_t kOBufs = 512 - kSBufs * 128 >= 2 * D ? 2 : 1;
// Ring positions in the load order K_0 .. K_{kSBufs-1}, V_0, K_kSBufs, V_1, ...: the order the
// two MMA issuers consume them in, so a load only waits for the slot freed kRing positions
// earlier in that same order.
__host__ __device__ constexpr uint32_t kseq_of(uint32_t k) {
  return k < kSBufs ? k : 2 * k - (kSBufs - 1);
}
__host__ __device__ constexpr uint32_t vseq_of(uint32_t k) { return 2 * k + kSBufs; }
static_assert(kseq_of(kSBufs) == vseq_of(0) + 1 && vseq_of(1) == kseq_of(kSBufs) + 1, "interleave");

template <int D>
struct Cfg {
  static constexpr uint32_t kBoxes = D / 64;
  static constexpr uint32_t kTileBytes = kBoxes * kBoxBytes;  // one 128 x D bf16 tile
  // K/V ring slots: the K cursor runs kSBufs tiles ahead of the V cursor
#ifndef BBM_RING128
#define BBM_RING128 (BBM_SBUFS + 1)
#endif
  static constexpr uint32_t kRing = (D == 64) ? 9 : BBM_RING128;
  static constexpr uint32_t kStageBytes = kBoxBytes;          // epilogue staging: one 128 x 64 box
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kOCol = kSBufs * 128;
};

struct ItemDesc {
  uint32_t t, slot, rt, j0, nt, split;
};

// Everything that is not a tile lives behind the tiles in the same dynamic allocation (no static
// smem, so the dynamic base is the 1024-byte aligned start of the CTA's window).
// Row statistics of a finished item, handed from the softmax engine to the epilogue warpgroup
// (one per O accumulator).
template <uint32_t kXP>
struct ItemStats {
  ItemDesc item;
  float l[kXP][128];  // per-part row sums
  float m_run[128], m_true[128];
};

template <uint32_t kRing, uint32_t kXP>
struct SmemCtl {
  uint64_t q_full[2], q_empty[2], s_full[kSBufs], p_full[kSBufs], o_full[2], o_empty[2], pv_done[kSBufs];
  uint64_t stats_full[2], stats_empty[2];
  uint64_t ring_full[kRing], ring_empty[kRing];
  uint64_t item_full[kQueue], item_empty[kQueue];
  ItemDesc items[kQueue];
  uint32_t ring_meta[kRing];  // per loaded K / V tile: its empty key half (bit 0 / 1), 0 = none
  uint32_t tmem_base;
  uint32_t units, total_items, split_rows, split_chunks;  // this launch's plan (device-built)
  uint32_t trace_count;
  uint32_t bcast;
  float xchg[2][kXP][128];  // [exchange parity][part][row]: partial row max
  ItemStats<kXP> stats[2];
  // LSU gather: the row tokens of the last 8 K tiles, per producer warp (64 rows each), so the V
  // load of the same key tile (kSBufs tiles later) needs no second lookup
  int32_t lsu_tok[2][8][64];
};
static_assert(kSBufs < 8, "the V cursor trails the K cursor by kSBufs tiles: lsu_tok keeps 8");

template <int D>
constexpr uint32_t smem_bytes() {
  return Cfg<D>::kTileBytes * (2 + Cfg<D>::kRing) + Cfg<D>::kStageBytes +
         sizeof(SmemCtl<Cfg<D>::kRing, kParts<D>>);
}

template <int MODE>
__device__ __forceinline__ uint32_t entry_of(const FwdParams& p, uint32_t row_tile, uint32_t j) {
  if constexpr (MODE == kModeDense || MODE == kModeNaive) return j;
  else return p.list[static_cast<uint64_t>(row_tile) * p.kcols + j];
}

// Empty key halves of list entry j of row tile `row_tile` (list modes; the other modes and the
// in-kernel gather always load and multiply whole tiles)
// Only the engine build for partial-heavy masks (kSkip) carries the half-skipping code, so the
// plain build's issue loops are exactly those without it.
template <int MODE, bool kGather, bool kSkip>
__device__ __forceinline__ uint32_t half_of(const FwdParams& p, uint32_t row_tile, uint32_t j) {
#ifdef BBM_NO_HALF_SKIP  // A/B builds: whole tiles always
  return 0u;
#else
  if constexpr (MODE == kModeDense || MODE == kModeNaive || kGather || !kSkip) return 0u;
  else return p.halves ? __ldg(p.halves + static_cast<uint64_t>(row_tile) * p.kcols + j) : 0u;
#endif
}

__device__ __forceinline__ ItemDesc decode_item(const FwdParams& p, uint32_t units, uint32_t total,
                                                uint32_t t) {
  ItemDesc d;
  d.t = t;
  if (t >= total) {
    d.t = kEnd;
    d.slot = d.rt = d.j0 = d.nt = 0;
    d.split = kNoSplit;
    return d;
  }
  d.slot = t / units;
  const uint4 u = p.unit_desc[t - d.slot * units];
  d.rt = u.x;
  d.j0 = u.y;
  d.nt = u.z;
  d.split = u.w;
  return d;
}

// Gather mode: the 2-D [slots * n][D] row of (permuted) position a of `slot`, or a coordinate past
// the tensor (zero-filled loads, skipped stores) for the padding rows a >= n.
__device__ __forceinline__ int32_t gather_row(const FwdParams& p, uint32_t slot, uint32_t a) {
  return a < p.n ? static_cast<int32_t>(static_cast<uint64_t>(slot) * p.n + __ldg(p.rows + a)) : INT32_MAX;
}
// Output row of (permuted) row `grow` of `slot` in the caller's [slots][n] layout
template <bool kGather>
__device__ __forceinline__ uint64_t out_row(const FwdParams& p, uint32_t slot, uint64_t grow) {
  return static_cast<uint64_t>(slot) * p.n + (kGather ? __ldg(p.rows + grow) : grow);
}

template <int D, int MODE, bool kTrace, int kGather, bool kSkip>
__global__ void __launch_bounds__(kThreadsOf<D>, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                    const __grid_constant__ CUtensorMap tm_k64, const __grid_constant__ CUtensorMap tm_v64,
                    const FwdParams p) {
  // kGather: 0 plain tiles; 1 every Q / K / V row gathered and O scattered in the kernel
  // (tile::gather4 / scatter4); 2 only Q gathered and O scattered, K / V from permuted copies;
  // 3 Q / K / V rows gathered by LSU cp.async (16 B per lane, the TMA unit left to the O scatter)
  constexpr bool kGQ = kGather != 0, kGKV = kGather == 1 || kGather == 3, kLsu = kGather == 3;
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sq = smem;                              // [2][tile]          Q, double-buffered
  uint8_t* ring = sq + 2 * C::kTileBytes;          // [kRing][tile]      K/V ring
  uint8_t* stage = ring + C::kRing * C::kTileBytes;  // [128 x 64 bf16] epilogue staging box
  auto* ctl = reinterpret_cast<SmemCtl<C::kRing, kParts<D>>*>(stage + C::kStageBytes);

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if ((smem_u32(smem) & 1023u) != 0) __trap();  // 128B-swizzle atoms need 1024-byte alignment
  const bool tracing = kTrace && blockIdx.x < p.trace_ctas;

  if (threadIdx.x == 0) {
    ctl->trace_count = 0;
    const PlanHdr h = *p.hdr;
    ctl->units = h.units;
    ctl->total_items = h.units * p.slots;
    ctl->split_rows = h.split_rows;
    ctl->split_chunks = h.split_chunks;
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ctl->q_full[b], kLsu ? 64 : 1);  // LSU gather: every producer lane's cp.async arrive
      mbar_init(&ctl->q_empty[b], 1);
    }
    for (uint32_t b = 0; b < kSBufs; ++b) {
      mbar_init(&ctl->s_full[b], 1);
      mbar_init(&ctl->p_full[b], 128 * kParts<D>);
      mbar_init(&ctl->pv_done[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ctl->o_full[b], 1);
      mbar_init(&ctl->o_empty[b], 128);                 // the epilogue warpgroup's threads
      // every thread of the handing-over side arrives, releasing its own writes
      mbar_init(&ctl->stats_full[b], 128 * kParts<D>);  // engine threads
      mbar_init(&ctl->stats_empty[b], 128);             // epilogue threads
    }
    for (uint32_t r = 0; r < C::kRing; ++r) {
      mbar_init(&ctl->ring_full[r], kLsu ? 64 : 1);
      mbar_init(&ctl->ring_empty[r], 1);
    }
    for (uint32_t r = 0; r < kQueue; ++r) {
      mbar_init(&ctl->item_full[r], 1);
      // S issuer + PV issuer + engine warps (+ the V-cursor warp of the LSU gather mode)
      mbar_init(&ctl->item_empty[r], 2 + kParts<D> * 4 + (kLsu ? 1 : 0));
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
  const bool engine_wg = warp >= 4 && warp < 4 + 4 * kParts<D>;

  if (warp < 4) {
  setmaxnreg_dec<kOtherRegs<D>>();
  if (warp == 0 || (kLsu && warp == 2)) {
    // ------------------------------------------------------------------ producer
    // (LSU gather mode: the cp.async gathers cost a warp instruction per 512 bytes, so warps 0
    // and 2 both run the producer, each copying 64 rows of every tile; warp 2 takes the items
    // warp 0 claims from the item queue, as one more consumer)
    // Loads follow the MMA issuers' consumption order (kseq_of / vseq_of): a K cursor runs kSBufs
    // tiles ahead of a V cursor, so a load only ever waits for the ring slot freed kRing
    // positions earlier in that same order.
    // The whole warp runs the loop (warp-uniform state; lane 0 owns the side effects: the work
    // counter, the item queue, the expect-tx arrivals). Plain mode: lane 0 issues the tiled TMA
    // loads. Gather mode (kGather): every lane gathers 4 rows of each 128-row tile
    // (tile::gather4), so a tile costs 32 instructions per 64-column box spread over the warp.
    {
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      uint32_t qi = 0, qiph = 1, qb = 0;
      PhaseBits qph{0x3u};
      ItemDesc pit[kQueue];  // items claimed by the K cursor, replayed by the V cursor
      uint32_t pw = 0, pr = 0;
      // one 128 x D tile (row tile `tile` of `slot`) into dst, completing on `bar` (expect-tx
      // already posted by lane 0)
      // `pre` / `save` (LSU gather only): take this lane's row tokens from / leave them in shared
      // memory (slot [ii * 32 + lane] of a 64-entry row of lsu_tok)
      auto issue_tile = [&](uint8_t* dst, const CUtensorMap* tm, uint64_t* bar, uint32_t tile, uint32_t slot,
                            uint64_t pol, auto gather, const int32_t* pre = nullptr, int32_t* save = nullptr) {
        if constexpr (kLsu) {
          // Coalesced: lane l copies 16-byte chunk l % 8 of rows 4g + l / 8, g = 0..31, so one warp
          // instruction moves four whole 128-byte box rows. The chunk lands where TMA's 128B
          // swizzle puts it (chunk c of row r at ((c ^ (r % 8)) * 16) within the row's 128 bytes).
          // Row tokens: lane l looks up rows l, l + 32, l + 64, l + 96; the others come by shuffle.
          const __nv_bfloat16* base = tm == &tm_q ? p.qg : (tm == &tm_k ? p.kg : p.vg);
          const uint32_t d0 = smem_u32(dst), c = lane & 7, rr = lane >> 3, i0 = warp == 0 ? 0u : 2u;
          int32_t tok[2];
#pragma unroll
          for (uint32_t ii = 0; ii < 2; ++ii)
            tok[ii] = pre ? pre[ii * 32 + lane] : gather_row(p, slot, tile * 128 + (i0 + ii) * 32 + lane);
          if (save) {
            save[lane] = tok[0];
            save[32 + lane] = tok[1];
          }
#pragma unroll
          for (uint32_t ii = 0; ii < 2; ++ii) {
            const uint32_t i = i0 + ii;
#pragma unroll
            for (uint32_t g8 = 0; g8 < 8; ++g8) {
              const uint32_t r = i * 32 + g8 * 4 + rr;  // row of the tile; its token is in lane r % 32
              const int32_t gr = __shfl_sync(0xffffffffu, tok[ii], g8 * 4 + rr);
              const bool in = gr != INT32_MAX;
              const __nv_bfloat16* src = base + (in ? static_cast<uint64_t>(gr) * D : 0) + c * 8;
#pragma unroll
              for (uint32_t b = 0; b < C::kBoxes; ++b)
                cp_async16(d0 + b * kBoxBytes + r * 128 + ((c ^ (r & 7)) << 4), src + b * 64, in ? 16 : 0);
            }
          }
          cp_async_mbar_arrive(bar);
          (void)pol;
        } else if constexpr (decltype(gather)::value) {
          int32_t r[4];
#pragma unroll
          for (uint32_t i = 0; i < 4; ++i) r[i] = gather_row(p, slot, tile * 128 + lane * 4 + i);
#pragma unroll
          for (uint32_t b = 0; b < C::kBoxes; ++b)
            tma_gather4(dst + b * kBoxBytes + lane * 512, tm, bar, b * 64, r[0], r[1], r[2], r[3], pol);
        } else {
          if (lane == 0)
            for (uint32_t b = 0; b < C::kBoxes; ++b)
              tma_load_3d(dst + b * kBoxBytes, tm, bar, b * 64, tile * 128, slot, pol);
        }
      };
      // K / V tile q into the ring; a key half that no row of the tile sees (`half`, bit 0 / 1) is
      // not loaded (64-row boxes for the other half); the MMA issuers read `half` from ring_meta
      auto load_tile = [&](const CUtensorMap* tm, const CUtensorMap* tm64, uint32_t seq, uint32_t q, uint32_t slot,
                           uint32_t code, uint32_t j, uint32_t half, const int32_t* pre, int32_t* save) {
        const uint32_t r = seq % C::kRing;
        mbar_wait(&ctl->ring_empty[r], ((seq / C::kRing) & 1) ^ 1);
        uint64_t* full = &ctl->ring_full[r];
#if defined(BBM_ABLATE_NO_KVLOAD) || defined(BBM_ABLATE_HALF_KVLOAD)
        // timing experiments only (wrong results): the ring keeps stale tiles after its first
        // fill (NO_KVLOAD) or every second K/V pair reuses them (HALF_KVLOAD)
#ifdef BBM_ABLATE_NO_KVLOAD
        const bool skip_load = seq >= C::kRing;
#else
        const bool skip_load = seq >= C::kRing && ((seq / 2) & 1);
#endif
        if (skip_load) {
          __syncwarp();
          if (lane == 0) {
            ctl->ring_meta[r] = half;
            mbar_arrive(full);
          }
          return;
        }
#endif
        if (lane == 0) {
          ctl->ring_meta[r] = half;  // published by the arrive below
          if (!kLsu) mbar_arrive_expect_tx(full, half ? C::kTileBytes / 2 : C::kTileBytes);
        }
        __syncwarp();
        if (half == 0) {
          issue_tile(ring + r * C::kTileBytes, tm, full, q, slot, pol_kv, std::bool_constant<kGKV>{}, pre, save);
        } else if (lane == 0) {
          const uint32_t hh = (half & 1u) ? 1u : 0u;  // the half that is loaded
          for (uint32_t b = 0; b < C::kBoxes; ++b)
            tma_load_3d(ring + r * C::kTileBytes + b * kBoxBytes + hh * (kBoxBytes / 2), tm64, full, b * 64,
                        q * 128 + hh * 64, slot, pol_kv);
        }
        if (lane == 0) trace_ev<kTrace>(tracing, p, &ctl->trace_count, code, 0, j);
      };
      // K cursor (claims and publishes items, loads Q)
      ItemDesc kit{};
      uint32_t kj = 0, kk = 0, kentry = 0, khalf = 0;
      uint32_t kentry2 = 0;             // LSU gather: the list entry two K tiles ahead
      uint32_t ktok[2] = {0u, 0u};      // LSU gather: the next K tile's raw rows[] values (in flight)
      // this warp's rows[] values of key tile `tile` (rows (i0 + ii) * 32 + lane, i0 = 0 / 2),
      // 0xFFFFFFFF past n; predicated loads, nothing consumes them until the tile is issued
      auto lsu_tokens = [&](uint32_t, uint32_t tile, uint32_t (&t)[2]) {
        const uint32_t i0 = warp == 0 ? 0u : 2u;
#pragma unroll
        for (uint32_t ii = 0; ii < 2; ++ii) {
          const uint64_t a = static_cast<uint64_t>(tile) * 128 + (i0 + ii) * 32 + lane;
          uint32_t v = 0xFFFFFFFFu;
          if (a < p.n) v = __ldg(p.rows + a);
          t[ii] = v;
        }
      };
      bool k_need = true, k_done = false;
      auto k_next = [&]() -> bool {
        while (k_need) {
          if (k_done) return false;
          ItemDesc d;
          if (kLsu && warp == 2) {  // the second gather warp follows warp 0's claims
            mbar_wait(&ctl->item_full[qi], qiph ^ 1);
            d = ctl->items[qi];
            __syncwarp();
            if (lane == 0) mbar_arrive(&ctl->item_empty[qi]);
          } else {
            uint32_t t = 0;
            if (lane == 0) t = atomicAdd(&p.work_ctr[0], 1u);
            t = __shfl_sync(0xffffffffu, t, 0);
            d = decode_item(p, ctl->units, ctl->total_items, t);
            mbar_wait(&ctl->item_empty[qi], qiph);
            if (lane == 0) {
              ctl->items[qi] = d;
              mbar_arrive(&ctl->item_full[qi]);  // release: the descriptor is visible to waiters
            }
          }
          if (++qi == kQueue) { qi = 0; qiph ^= 1; }
          if (d.t == kEnd) {
            k_done = true;
            return false;
          }
          if (d.nt == 0) continue;
          pit[pw++ % kQueue] = d;
          kentry = entry_of<MODE>(p, d.rt, d.j0);
          khalf = half_of<MODE, kGKV, kSkip>(p, d.rt, d.j0);
          if constexpr (kLsu) {  // entries run two tiles ahead, row tokens one (issue_k)
            kentry2 = d.nt > 1 ? entry_of<MODE>(p, d.rt, d.j0 + 1) : 0u;
            lsu_tokens(d.slot, kentry & 0x7FFFFFFFu, ktok);
          }
          mbar_wait(&ctl->q_empty[qb], qph[qb]);
          qph.flip(qb);
          if (lane == 0 && !kLsu) mbar_arrive_expect_tx(&ctl->q_full[qb], C::kTileBytes);
          __syncwarp();
          issue_tile(sq + qb * C::kTileBytes, &tm_q, &ctl->q_full[qb], d.rt, d.slot, pol_q, std::bool_constant<kGQ>{});
          if (lane == 0) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 1, 0, d.t);
          qb ^= 1;
          kit = d;
          kj = 0;
          k_need = false;
        }
        return true;
      };
      auto issue_k = [&]() {
        const uint32_t cur = kentry, chalf = khalf;
        if constexpr (kLsu) {
          // LSU gather: this tile's tokens were looked up a step ago (ktok); the next tile's entry
          // (fetched two steps ago) gives its tokens now, and the entry after that is fetched
          const uint32_t r0 = ktok[0], r1 = ktok[1];
          if (kj + 1 < kit.nt) {
            kentry = kentry2;
            if (kj + 2 < kit.nt) kentry2 = entry_of<MODE>(p, kit.rt, kit.j0 + kj + 2);
            lsu_tokens(kit.slot, kentry & 0x7FFFFFFFu, ktok);
          }
          auto tok_of = [&](uint32_t raw) {
            return raw == 0xFFFFFFFFu ? INT32_MAX
                                      : static_cast<int32_t>(static_cast<uint64_t>(kit.slot) * p.n + raw);
          };
          int32_t* save = ctl->lsu_tok[warp == 0 ? 0 : 1][kk % 8];
          save[lane] = tok_of(r0);
          save[32 + lane] = tok_of(r1);
          load_tile(&tm_k, &tm_k64, kseq_of(kk), cur & 0x7FFFFFFFu, kit.slot, 2, kj, chalf, save, nullptr);
        } else {
          // the next list entry is fetched now, a full issue step before it is needed
          if (kj + 1 < kit.nt) {
            kentry = entry_of<MODE>(p, kit.rt, kit.j0 + kj + 1);
            khalf = half_of<MODE, kGKV, kSkip>(p, kit.rt, kit.j0 + kj + 1);
          }
          load_tile(&tm_k, &tm_k64, kseq_of(kk), cur & 0x7FFFFFFFu, kit.slot, 2, kj, chalf, nullptr, nullptr);
        }
        ++kk;
        if (++kj == kit.nt) k_need = true;
      };
      // V cursor
      ItemDesc vit{};
      uint32_t vj = 0, vk = 0, ventry = 0, vhalf = 0;
      bool v_need = true;
      auto issue_v = [&]() -> bool {
        if (v_need) {
          if (pr == pw) return false;
          vit = pit[pr++ % kQueue];
          vj = 0;
          ventry = entry_of<MODE>(p, vit.rt, vit.j0);
          vhalf = half_of<MODE, kGKV, kSkip>(p, vit.rt, vit.j0);
          v_need = false;
        }
        const uint32_t cur = ventry, chalf = vhalf;
        if (vj + 1 < vit.nt) {
          ventry = entry_of<MODE>(p, vit.rt, vit.j0 + vj + 1);
          vhalf = half_of<MODE, kGKV, kSkip>(p, vit.rt, vit.j0 + vj + 1);
        }
        // K tile vk's tokens (saved kSBufs tiles ago by this same lane)
        load_tile(&tm_v, &tm_v64, vseq_of(vk), cur & 0x7FFFFFFFu, vit.slot, 3, vj, chalf,
                  kLsu ? ctl->lsu_tok[warp == 0 ? 0 : 1][vk % 8] : nullptr, nullptr);
        ++vk;
        if (++vj == vit.nt) v_need = true;
        return true;
      };
      for (uint32_t w = 0; w < kSBufs; ++w)
        if (k_next()) issue_k();
      while (issue_v())
        if (k_next()) issue_k();
    }
  } else if (warp == 1 || warp == 3) {
    // ------------------------------------------------------------------ MMA issuers
    // tcgen05.mma issue is nearly synchronous (~56 cycles per 128x128x16 MMA,
    // tools/mma_issue_probe.cu), and one thread issuing both S and PV queues each behind the other
    // (measured slower). Two issuers, each walking the same tile sequence k = 0, 1, 2, ...:
    //   warp 1: S_k = Q K_k^T into TMEM buffer k % 3 (SS), once PV_{k-3} (the last reader of
    //           that buffer's P) has completed;
    //   warp 3: O += P_k V_k (TS, P read from TMEM) once the softmax engine has written P_k.
    // Ring slots follow the load order: K_k at kseq_of(k), V_k at vseq_of(k) (mod kRing).
    if (lane == 0) {
      const bool s_side = warp == 1;
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_s64 = make_idesc_bf16(128, 64, false, false);  // one key half
      constexpr uint32_t idesc_o = make_idesc_bf16(128, D, false, true);
      const uint32_t qaddr = smem_u32(sq), raddr = smem_u32(ring);
      uint32_t qi = 0, qiph = 0, k = 0, qb = 0, items = 0;
      PhaseBits q_ph{0u}, p_ph{0u}, oe_ph{0x3u};
      for (;;) {
        mbar_wait(&ctl->item_full[qi], qiph);
        const ItemDesc it = ctl->items[qi];
        mbar_arrive(&ctl->item_empty[qi]);
        if (++qi == kQueue) { qi = 0; qiph ^= 1; }
        if (it.t == kEnd) break;
        if (it.nt == 0) continue;
        // items alternate between the two O accumulators; an item's first PV waits until the
        // epilogue warpgroup has read out the item two back
        const uint32_t ob = kOBufs<D> == 2 ? (items++ & 1) : 0;
        const uint32_t tmem_o = tmem + C::kOCol + ob * D;
        for (uint32_t j = 0; j < it.nt; ++j, ++k) {
          const uint32_t buf = k % kSBufs;
          if (s_side) {
            if (k >= kSBufs) mbar_wait(&ctl->pv_done[buf], ((k - kSBufs) / kSBufs) & 1);
            if (j == 0) {
              mbar_wait(&ctl->q_full[qb], q_ph[qb]);
              q_ph.flip(qb);
            }
            const uint32_t kseq = kseq_of(k);
            const uint32_t slot = kseq % C::kRing;
            mbar_wait(&ctl->ring_full[slot], (kseq / C::kRing) & 1);
            trace_ev<kTrace>(tracing, p, &ctl->trace_count, 13, buf, j);
            if constexpr (kLsu) fence_proxy_async_smem();  // cp.async (generic proxy) -> tcgen05 reads
            tc_fence_after();
            // a key half no row sees is neither loaded nor multiplied: N = 64 over the other half
            // (its S columns keep stale values, which the softmax replaces by the mask sentinel)
            const uint32_t half = kSkip ? ctl->ring_meta[slot] : 0u;
            const uint32_t hrow = (half & 1u) ? 64u : 0u;
            const uint64_t qdesc = make_sdesc_sw128(qaddr + qb * C::kTileBytes, 16, 1024);
            const uint64_t kdesc = make_sdesc_sw128(raddr + slot * C::kTileBytes + hrow * 128, 16, 1024);
#pragma unroll
            for (uint32_t kk = 0; kk < D / 16; ++kk) {
              const uint32_t off = (kk / 4) * kBoxBytes + (kk % 4) * 32;
              umma_ss(tmem + buf * 128 + hrow, sdesc_advance(qdesc, off), sdesc_advance(kdesc, off),
                      half ? idesc_s64 : idesc_s, kk > 0);
            }
            tc_commit(&ctl->ring_empty[slot]);
            tc_commit(&ctl->s_full[buf]);
            trace_ev<kTrace>(tracing, p, &ctl->trace_count, 10, buf, j);
            if (j + 1 == it.nt) {
              tc_commit(&ctl->q_empty[qb]);
              qb ^= 1;
            }
          } else {
            mbar_wait(&ctl->p_full[buf], p_ph[buf]);
            p_ph.flip(buf);
            trace_ev<kTrace>(tracing, p, &ctl->trace_count, 14, buf, j);
            if (j == 0) {
              mbar_wait(&ctl->o_empty[ob], oe_ph[ob]);
              oe_ph.flip(ob);
            }
            const uint32_t vseq = vseq_of(k);
            const uint32_t slot = vseq % C::kRing;
            mbar_wait(&ctl->ring_full[slot], (vseq / C::kRing) & 1);
            trace_ev<kTrace>(tracing, p, &ctl->trace_count, 12, buf, j);
            if constexpr (kLsu) fence_proxy_async_smem();
            tc_fence_after();
            const uint64_t vdesc = make_sdesc_sw128(raddr + slot * C::kTileBytes, kBoxBytes, 1024);
            const uint32_t pcol = tmem + buf * 128;
            // K steps over the keys present (a whole empty key half is skipped)
            const uint32_t half = kSkip ? ctl->ring_meta[slot] : 0u;
            const uint32_t kk0 = (half & 1u) ? 4u : 0u, kk1 = (half & 2u) ? 4u : 8u;
#ifndef BBM_ABLATE_NO_PV  // timing experiments only: O is never accumulated
#pragma unroll
            for (uint32_t kk = 0; kk < 128 / 16; ++kk)
              if (kk >= kk0 && kk < kk1)
                umma_ts(tmem_o, pcol + kk * 8, sdesc_advance(vdesc, kk * 2048), idesc_o,
                        (j > 0 || kk > kk0) ? 1u : 0u);
#endif
            tc_commit(&ctl->ring_empty[slot]);
            tc_commit(&ctl->pv_done[buf]);
            trace_ev<kTrace>(tracing, p, &ctl->trace_count, 11, buf, j);
            if (j + 1 == it.nt) tc_commit(&ctl->o_full[ob]);
          }
        }
      }
    }
  }
  } else if (engine_wg) {
    setmaxnreg_inc<kEngineRegs<D>>();
    // ------------------------------------------------------------------ softmax engine
    constexpr uint32_t kP = kParts<D>;
    constexpr uint32_t kSC = 128 / kP;        // score columns per part
    constexpr uint32_t kEng = 128 * kP;       // engine threads
    const uint32_t half = (warp - 4) >> 2;    // this thread's part
    const uint32_t quad = warp & 3;
    const uint32_t row = quad * 32 + lane;
    const uint32_t lane_off = (quad * 32) << 16;
    const bool leader = (warp == 4 && lane == 0);
    const bool tracer = (quad == 0 && lane == 0 && half == 0);
    const bool neg = p.sl2 < 0.0f;
    const float abs_sl2 = fabsf(p.sl2);
    const bool ragged = (p.n % 128) != 0;
    const uint32_t last_q = p.kcols - 1;
    const uint32_t kv_valid_last = static_cast<uint32_t>(p.n - static_cast<uint64_t>(last_q) * 128);
    // masked scores: -inf, or +inf with a negative scale, so that scale * sentinel = -inf
    const uint32_t sentinel = neg ? 0x7F800000u : 0xFF800000u;
    constexpr uint32_t kHalfO = D / kP;  // O columns per part
    const uint32_t to_base = tmem + C::kOCol + lane_off;

    uint32_t step = 0;  // parity selects the exchange buffer
    uint32_t k = 0;     // global tile index (S buffer k % kSBufs)
    uint2 nbits = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);  // mask bits of the next tile
    uint32_t nentry = 0;                                // its list entry (dense_binblk)
    bool have_next_bits = false;                        // prefetched for the next item
    PhaseBits s_ph{0u}, se_ph{0x3u};
    uint32_t qi = 0, qiph = 0, items = 0;
    auto write_stats = [&](const ItemDesc& it, float m_true2, float m_run2, float l_tot) {
      const uint64_t grow = static_cast<uint64_t>(it.rt) * 128 + row;
      if (half == 0 && grow < p.n) {
        const uint64_t si = out_row<kGQ>(p, it.slot, grow);
        if (p.row_max) p.row_max[si] = m_true2 == -INFINITY ? -INFINITY : m_true2 * kLn2;
        if (p.row_sum) p.row_sum[si] = l_tot > 0.0f ? l_tot * exp2f(m_run2 - m_true2) : 0.0f;
      }
    };
    // zero rows / stats for items without any tile (fully masked row tiles)
    auto zero_item = [&](const ItemDesc& it) {
      const uint64_t grow = static_cast<uint64_t>(it.rt) * 128 + row;
      if (grow >= p.n) return;
      uint4* dst = reinterpret_cast<uint4*>(p.out + out_row<kGQ>(p, it.slot, grow) * D + half * kHalfO);
      for (uint32_t v = 0; v < kHalfO / 8; ++v) dst[v] = make_uint4(0, 0, 0, 0);
      write_stats(it, -INFINITY, -INFINITY, 0.0f);
    };
    // mask bits (and, for dense_binblk, the list entry) of tile jj of item `it`; the bitmap
    // address depends only on (row tile, list position), never on a loaded value
    auto load_bits = [&](const ItemDesc& it, uint32_t jj, uint2& bits, uint32_t& entry) {
      const uint64_t grow = static_cast<uint64_t>(it.rt) * 128 + row;
      if constexpr (MODE == kModeNaive)
        bits = kSC == 64 ? __ldg(reinterpret_cast<const uint2*>(p.mask + grow * p.kcols + jj) + half)
                         : make_uint2(__ldg(reinterpret_cast<const uint32_t*>(p.mask + grow * p.kcols + jj) + half), 0u);
      else if constexpr (MODE != kModeDense) {
        const uint4* bp = p.bitmaps + (static_cast<uint64_t>(it.rt) * p.kcols + jj) * 128 + row;
        bits = kSC == 64 ? __ldg(reinterpret_cast<const uint2*>(bp) + half)
                         : make_uint2(__ldg(reinterpret_cast<const uint32_t*>(bp) + half), 0u);
      }
      if constexpr (MODE == kModeDenseBinblk) entry = entry_of<MODE>(p, it.rt, jj);
    };

    for (;;) {
      // ---------------- next item (items without tiles are written as zeros right away)
      mbar_wait(&ctl->item_full[qi], qiph);
      const ItemDesc it = ctl->items[qi];
      __syncwarp();  // every lane of this warp has read the descriptor
      if (lane == 0) mbar_arrive(&ctl->item_empty[qi]);
      if (++qi == kQueue) { qi = 0; qiph ^= 1; }
      if (it.t == kEnd) break;
      if (it.nt == 0) {
        zero_item(it);
        continue;
      }
      if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 29, 0, it.t);
      float m_run = -INFINITY, m_true = -INFINITY, l = 0.0f;
      const uint32_t sl = items++ & 1;              // this item's statistics slot
      const uint32_t ob = kOBufs<D> == 2 ? sl : 0;  // and O accumulator (same sequence as the PV issuer)
      const uint32_t to = to_base + ob * D;
      if (!have_next_bits) load_bits(it, it.j0, nbits, nentry);  // else prefetched last item
      have_next_bits = false;

      for (uint32_t j = 0; j < it.nt; ++j, ++k) {
        const uint32_t buf = k % kSBufs;
        const uint32_t ts = tmem + buf * 128 + lane_off;
        bool masked;
        uint2 bits = nbits;
        if constexpr (MODE == kModeDense) {
          // only the ragged right edge needs a column bound (no bitmap in this mode)
          masked = ragged && it.j0 + j == last_q;
          if (masked) {
            const int v = static_cast<int>(kv_valid_last) - static_cast<int>(half * kSC);
            bits.x = v >= 32 ? 0xFFFFFFFFu : (v <= 0 ? 0u : ((1u << v) - 1u));
            bits.y = v >= 64 ? 0xFFFFFFFFu : (v <= 32 ? 0u : ((1u << (v - 32)) - 1u));
          }
        } else if constexpr (MODE == kModeDenseBinblk) {
          masked = (nentry & 0x80000000u) == 0;  // full tiles skip the mask bits
        } else {
          masked = true;  // bitmaps carry zeros beyond n, so ragged edges need nothing extra
        }
        if (j + 1 < it.nt) {
          load_bits(it, it.j0 + j + 1, nbits, nentry);  // a tile ahead
        } else if (mbar_test(&ctl->item_full[qi], qiph)) {
          // last tile: if the next item is already published, prefetch its first tile's bits
          // (the descriptor is read again, and released, at the top of the item loop)
          const ItemDesc nx = ctl->items[qi];
          if (nx.t != kEnd) {
            load_bits(nx, nx.j0, nbits, nentry);
            have_next_bits = true;
          }
        }

        if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 20, buf, j);
        mbar_wait(&ctl->s_full[buf], s_ph[buf]);
        s_ph.flip(buf);
        tc_fence_after();
        if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 21, buf, j);

#ifdef BBM_ABLATE_FAST_ENGINE  // timing experiments only: P = 0, no softmax work (MMA-side ceiling)
        if (true) {
          uint32_t z[16];
#pragma unroll
          for (uint32_t i = 0; i < 16; ++i) z[i] = 0u;
          tmem_st16(ts + half * (kSC / 2), z);
          if constexpr (kSC == 64) tmem_st16(ts + half * (kSC / 2) + 16, z);
          l = 1.0f;
          m_run = m_true = 0.0f;
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&ctl->p_full[buf]);
          continue;
        }
#endif
        // kSkip build (masks whose occupied tiles are mostly partial: banded, permuted, packed
        // sequences, where ~30% of the warps' 32 x 64 score halves see no key): a warp whose 32
        // rows see none of its half's keys skips the TMEM load, the selects and the max (-inf)
        // and writes P = 0 below, exactly what the -inf sentinel gives. Masks of mostly full
        // tiles run the build without the test (its branches cost them ~7%).
        // (per 32-column chunk: of C5's occupied tiles 35 % of the warps' 32 x 32 chunks are empty,
        // 30 % of the 32 x 64 halves)
        const bool e0 = kSkip && masked && __all_sync(0xffffffffu, bits.x == 0u);
        const bool e1 = kSC == 64 ? (kSkip && masked && __all_sync(0xffffffffu, bits.y == 0u)) : true;
        const bool empty = e0 && e1;
        uint32_t a0[32], a1[32];
        float pmax = -INFINITY;
        if (!empty) {
          if (!e0) tmem_ld32(ts + half * kSC, a0);
          if constexpr (kSC == 64) {
            if (!e1) tmem_ld32(ts + half * kSC + 32, a1);
          }
          tmem_ld_wait();
          if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 25, buf, j);
          // binblk reads bits for every tile; a warp whose 32 rows see every key of the tile skips
          // the selects (they would be no-ops)
          if (masked && !__all_sync(0xffffffffu, (kSC == 64 ? (bits.x & bits.y) : bits.x) == 0xFFFFFFFFu)) {
            if (!e0) apply_mask(a0, bits.x, sentinel);
            if constexpr (kSC == 64) {
              if (!e1) apply_mask(a1, bits.y, sentinel);
            }
          }
          if (!e0) pmax = neg ? chunk_max<true>(a0) : chunk_max<false>(a0);
          if constexpr (kSC == 64) {
            if (!e1) pmax = fmaxf(pmax, neg ? chunk_max<true>(a1) : chunk_max<false>(a1));
          }
        }
        // exchange with the other half of the same rows (double-buffered by parity) through a
        // 64-thread named barrier of the quadrant's two engine warps only: after it both halves
        // of these 32 rows have read S, so P may overwrite their S columns [0, 64). The four
        // quadrant pairs run decoupled.
#ifdef BBM_ABLATE_NO_XCHG  // timing experiments only: wrong results
        float tmax = pmax;
#else
        ctl->xchg[step & 1][half][row] = pmax;
        named_bar_sync(3 + quad, 32 * kP);
        float tmax = pmax;
#pragma unroll
        for (uint32_t o = 1; o < kP; ++o) tmax = fmaxf(tmax, ctl->xchg[step & 1][(half + o) % kP][row]);
#endif
        ++step;
        if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 26, buf, j);
        tmax = tmax == -INFINITY ? -INFINITY : tmax * abs_sl2;  // log2 domain
        m_true = fmaxf(m_true, tmax);
        const bool need = tmax > m_run + kRescaleThreshold || (m_run == -INFINITY && tmax > -INFINITY);
        const bool rescale_o = need && j > 0 && m_run > -INFINITY;
        float factor = 1.0f;
        if (need) {
          if (m_run > -INFINITY) factor = fast_exp2(m_run - tmax);
          m_run = tmax;
        }
        if (__any_sync(0xffffffffu, rescale_o)) {
          // O must be quiescent: PV_{k-1} (the last one issued) has to complete first
          mbar_wait(&ctl->pv_done[(k - 1) % kSBufs], ((k - 1) / kSBufs) & 1);
          tc_fence_after();
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
        l *= factor;
        const float m_use = m_run == -INFINITY ? 0.0f : m_run;
        uint32_t pk[16];
        uint64_t lacc = 0;
        const uint64_t sl2x2 = f2_pack(p.sl2, p.sl2), nm2 = f2_pack(-m_use, -m_use);
        // this half's 64 columns -> 32 packed P columns at [32 * half, 32 * half + 32); masked
        // scores already hold the sentinel (the host never passes a zero scale, see launch_impl)
        // an empty chunk's P is 0 (what exp2 of the sentinel gives) and adds nothing to l
        if (!e0) {
          chunk_exp(a0, sl2x2, nm2, pk, lacc);
        } else {
#pragma unroll
          for (uint32_t i = 0; i < 16; ++i) pk[i] = 0u;
        }
        tmem_st16(ts + half * (kSC / 2), pk);
        if constexpr (kSC == 64) {
          if (!e1) {
            chunk_exp(a1, sl2x2, nm2, pk, lacc);
          } else {
#pragma unroll
            for (uint32_t i = 0; i < 16; ++i) pk[i] = 0u;
          }
          tmem_st16(ts + half * (kSC / 2) + 16, pk);
        }
        l += f2_lo(lacc) + f2_hi(lacc);
        if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 27, buf, j);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&ctl->p_full[buf]);
        if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 22, buf, j);
      }

      // ---------------- item end: hand the row statistics to the epilogue warpgroup, which
      // combines the parts' row sums, waits for the item's last PV and writes O
      mbar_wait(&ctl->stats_empty[sl], se_ph[sl]);
      se_ph.flip(sl);
      ItemStats<kP>& st = ctl->stats[sl];
      st.l[half][row] = l;
      if (half == 0) {
        st.m_run[row] = m_run;
        st.m_true[row] = m_true;
      }
      if (leader) st.item = it;
      mbar_arrive(&ctl->stats_full[sl]);
      if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 28, 0, it.t);
    }
    {  // end marker for the epilogue warpgroup
      const uint32_t sl = items & 1;
      mbar_wait(&ctl->stats_empty[sl], se_ph[sl]);
      if (leader) ctl->stats[sl].item.t = kEnd;
      mbar_arrive(&ctl->stats_full[sl]);
    }
  } else {
    setmaxnreg_dec<kOtherRegs<D>>();
    // ------------------------------------------------------------------ epilogue warpgroup
    // Per item (in O-accumulator order): row statistics from the engine, then the item's last PV
    // (o_full), then O / l -> bf16 staged in 128B-swizzled shared memory -> TMA store, or, for a
    // split-KV chunk, the unnormalized partial to the workspace and the last chunk's combine.
    constexpr uint32_t kEpi = 128;
    const uint32_t quad = warp & 3;
    const uint32_t row = quad * 32 + lane;
    const uint32_t lane_off = (quad * 32) << 16;
    const bool leader = (quad == 0 && lane == 0);
    const bool tracer = leader;
    PhaseBits sf_ph{0u}, o_ph{0u};
    auto write_stats = [&](const ItemDesc& it, float m_true2, float m_run2, float l_tot) {
      const uint64_t grow = static_cast<uint64_t>(it.rt) * 128 + row;
      if (grow < p.n) {
        const uint64_t si = out_row<kGQ>(p, it.slot, grow);
        if (p.row_max) p.row_max[si] = m_true2 == -INFINITY ? -INFINITY : m_true2 * kLn2;
        if (p.row_sum) p.row_sum[si] = l_tot > 0.0f ? l_tot * exp2f(m_run2 - m_true2) : 0.0f;
      }
    };
    // The O tile leaves one 64-column box at a time through a single staging box: TMA-store box b
    // of item `it` once staged (called by every epilogue thread) ...
    // (gather mode: the first epilogue warp scatters the box's rows, 4 per lane, to their tokens)
    const bool storer = kGQ ? quad == 0 : leader;
    auto store_box = [&](const ItemDesc& it, uint32_t b) {
      fence_proxy_async_smem();
      named_bar_sync(2, kEpi);
      if constexpr (kGQ) {
        if (quad == 0) {
          int32_t r[4];
#pragma unroll
          for (uint32_t i = 0; i < 4; ++i) r[i] = gather_row(p, it.slot, it.rt * 128 + lane * 4 + i);
          tma_scatter4(&tm_o, stage + lane * 512, b * 64, r[0], r[1], r[2], r[3]);
          bulk_commit_group();
        }
      } else if (leader) {
        tma_store_3d(&tm_o, stage, b * 64, it.rt * 128, it.slot);
        bulk_commit_group();
      }
    };
    // ... and wait until the previous box's store has read the staging memory
    auto box_free = [&]() {
      if (storer) bulk_wait_group_read<0>();
      named_bar_sync(2, kEpi);
    };
    // staged output column c goes to 16-byte chunk (c % 64) / 8 of the row
    auto stg_row_of = [&](uint32_t) { return stage + row * 128; };
    auto stg_chunk_of = [&](uint32_t c) { return (c % 64) / 8; };
    for (uint32_t sl = 0;; sl ^= 1) {
      mbar_wait(&ctl->stats_full[sl], sf_ph[sl]);
      sf_ph.flip(sl);
      const ItemStats<kParts<D>>& st = ctl->stats[sl];
      const uint32_t ob = kOBufs<D> == 2 ? sl : 0;
      const ItemDesc it = st.item;
      if (it.t == kEnd) break;
      float l_unit = 0.0f;
#pragma unroll
      for (uint32_t h = 0; h < kParts<D>; ++h) l_unit += st.l[h][row];
      const float m_run = st.m_run[row], m_true = st.m_true[row];
      mbar_arrive(&ctl->stats_empty[sl]);
      const uint32_t to = tmem + C::kOCol + lane_off + ob * D;
      if (storer) bulk_wait_group_read<0>();  // staging buffers free again
      mbar_wait(&ctl->o_full[ob], o_ph[ob]);
      o_ph.flip(ob);
      tc_fence_after();
      named_bar_sync(2, kEpi);
      if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 23, 0, it.t);
      if (it.split == kNoSplit && kGQ) {
        // gathered rows: each epilogue thread writes its own O row straight to its token (whole
        // 32-byte sectors per thread), no staging box and no TMA scatter
        const float inv = l_unit > 0.0f ? 1.0f / l_unit : 0.0f;
        const uint64_t grow = static_cast<uint64_t>(it.rt) * 128 + row;
        __nv_bfloat16* dst = p.out + (grow < p.n ? out_row<kGQ>(p, it.slot, grow) * D : 0);
#pragma unroll
        for (uint32_t c64 = 0; c64 < D / 64; ++c64) {
          uint32_t o[2][32];
          tmem_ld32(to + c64 * 64, o[0]);
          tmem_ld32(to + c64 * 64 + 32, o[1]);
          tmem_ld_wait();
          if (c64 + 1 == D / 64) {
            tc_fence_before();
            mbar_arrive(&ctl->o_empty[ob]);
          }
          if (grow < p.n) {
#pragma unroll
            for (uint32_t h = 0; h < 2; ++h) {
              const float* v = reinterpret_cast<const float*>(o[h]);
              uint4* d4 = reinterpret_cast<uint4*>(dst + c64 * 64 + h * 32);
#pragma unroll
              for (uint32_t q4 = 0; q4 < 4; ++q4) {
                uint4 w;
                w.x = pack_bf16x2(v[q4 * 8 + 0] * inv, v[q4 * 8 + 1] * inv);
                w.y = pack_bf16x2(v[q4 * 8 + 2] * inv, v[q4 * 8 + 3] * inv);
                w.z = pack_bf16x2(v[q4 * 8 + 4] * inv, v[q4 * 8 + 5] * inv);
                w.w = pack_bf16x2(v[q4 * 8 + 6] * inv, v[q4 * 8 + 7] * inv);
                d4[q4] = w;
              }
            }
          }
        }
        write_stats(it, m_true, m_run, l_unit);
      } else if (it.split == kNoSplit) {
        const float inv = l_unit > 0.0f ? 1.0f / l_unit : 0.0f;
#ifdef BBM_ABLATE_NO_EPI  // timing experiments only (tools/ablate.sh): O is never written
        if (false)
#endif
#pragma unroll
        for (uint32_t c64 = 0; c64 < D / 64; ++c64) {
          // two 32-column loads in flight per wait
          uint32_t o[2][32];
          tmem_ld32(to + c64 * 64, o[0]);
          tmem_ld32(to + c64 * 64 + 32, o[1]);
          tmem_ld_wait();
          if (c64 + 1 == D / 64) {
            tc_fence_before();
            mbar_arrive(&ctl->o_empty[ob]);  // the accumulator may be overwritten from here on
          }
          if (c64 > 0) box_free();
#pragma unroll
          for (uint32_t h = 0; h < 2; ++h)
            stage_chunk32(stg_row_of(c64 * 64 + h * 32), row, stg_chunk_of(c64 * 64 + h * 32),
                          reinterpret_cast<const float*>(o[h]), inv);
#ifndef BBM_ABLATE_NO_EPI
          store_box(it, c64);
#endif
        }
        write_stats(it, m_true, m_run, l_unit);
      } else {
        // ---- split-KV chunk: publish the unnormalized partial, the last chunk combines
        const uint32_t srow = it.split >> 8, chunk = it.split & 0xFF;
        const uint2 si = p.split_info[srow];  // {chunks, first workspace chunk}
        const uint64_t blk = static_cast<uint64_t>(128) * (D + 3);
        float* wsb = p.ws + (static_cast<uint64_t>(it.slot) * ctl->split_chunks + si.y + chunk) * blk;
#pragma unroll
        for (uint32_t c32 = 0; c32 < D / 32; ++c32) {
          uint32_t o[32];
          tmem_ld32(to + c32 * 32, o);
          tmem_ld_wait();
          uint4* dst = reinterpret_cast<uint4*>(wsb + row * D + c32 * 32);
#pragma unroll
          for (uint32_t v = 0; v < 8; ++v)
            dst[v] = make_uint4(o[v * 4], o[v * 4 + 1], o[v * 4 + 2], o[v * 4 + 3]);
        }
        tc_fence_before();
        mbar_arrive(&ctl->o_empty[ob]);
        wsb[128 * D + row] = m_run;
        wsb[128 * D + 128 + row] = m_true;
        wsb[128 * D + 256 + row] = l_unit;
        __threadfence();
        named_bar_sync(2, kEpi);
        uint32_t* ctr = p.split_ctr + static_cast<uint64_t>(it.slot) * ctl->split_rows + srow;
        if (leader) ctl->bcast = atomicAdd(ctr, 1u);
        named_bar_sync(2, kEpi);
        const uint32_t done_before = ctl->bcast;
        if (done_before + 1 == si.x) {
          // last chunk: combine every chunk's partial for this row tile
          __threadfence();
          const float* base = p.ws + (static_cast<uint64_t>(it.slot) * ctl->split_chunks + si.y) * blk;
          float mrun = -INFINITY, mtrue = -INFINITY;
          for (uint32_t c = 0; c < si.x; ++c) {
            const float* b = base + c * blk + 128 * D;
            if (__ldcg(b + 256 + row) > 0.0f) mrun = fmaxf(mrun, __ldcg(b + row));
            mtrue = fmaxf(mtrue, __ldcg(b + 128 + row));
          }
          float ltot = 0.0f;
          for (uint32_t c = 0; c < si.x; ++c) {
            const float* b = base + c * blk + 128 * D;
            const float lc = __ldcg(b + 256 + row);
            if (lc > 0.0f) ltot += lc * exp2f(__ldcg(b + row) - mrun);
          }
          const float inv = ltot > 0.0f ? 1.0f / ltot : 0.0f;
          named_bar_sync(2, kEpi);  // every epilogue thread has read the count
          if (leader) *ctr = 0;    // ready for the next launch
#pragma unroll 1
          for (uint32_t c32 = 0; c32 < D / 32; ++c32) {
            if (c32 > 0 && c32 % 2 == 0) box_free();  // the next 64-column box reuses the staging
            float acc[32];
#pragma unroll
            for (uint32_t i = 0; i < 32; ++i) acc[i] = 0.0f;
            for (uint32_t c = 0; c < si.x; ++c) {
              const float* b = base + c * blk;
              const float lc = __ldcg(b + 128 * D + 256 + row);
              if (!(lc > 0.0f)) continue;
              const float w = exp2f(__ldcg(b + 128 * D + row) - mrun);
              const float4* src = reinterpret_cast<const float4*>(b + row * D + c32 * 32);
#pragma unroll
              for (uint32_t v = 0; v < 8; ++v) {
                const float4 f = __ldcg(src + v);
                acc[v * 4 + 0] += w * f.x;
                acc[v * 4 + 1] += w * f.y;
                acc[v * 4 + 2] += w * f.z;
                acc[v * 4 + 3] += w * f.w;
              }
            }
            stage_chunk32(stg_row_of(c32 * 32), row, stg_chunk_of(c32 * 32), acc, inv);
            if (c32 % 2 == 1) store_box(it, c32 / 2);
          }
          write_stats(it, mtrue, mrun, ltot);
        }
      }
      if (tracer) trace_ev<kTrace>(tracing, p, &ctl->trace_count, 24, 0, it.t);
    }
    if (storer) bulk_wait_group<0>();  // O stores landed
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<C::kTmemCols>(tmem);
  // the last CTA out resets the work counter for the next launch (stream-ordered)
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&p.work_ctr[1], 1u) == gridDim.x - 1) {
      p.work_ctr[0] = 0;
      p.work_ctr[1] = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------------ host side

std::atomic<uint64_t> g_builds[2];  // forward launches per engine build (plain, skipping)

template <int D, int MODE, int kGather>
void launch_impl(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms) {
  static_assert(smem_bytes<D>() <= 232448, "exceeds the 227 KB opt-in shared memory");
  const KernelMeta& km = prep.kmeta;
  constexpr int kCls = MODE == kModeDense ? kPlanDense : (MODE == kModeNaive ? kPlanNaive : kPlanList);
  std::lock_guard<std::recursive_mutex> lk(prep.mu);
  StreamCtx& ctx = prep.ctx_for(s);  // ordered after the latest mask version
  const uint32_t workers = static_cast<uint32_t>(num_sms);
  const DevPlan& plan = plan_for(prep, ctx, row_view(km), kCls, a.slots, workers, s);
  // one CTA per SM; when work items are scarce, at most one CTA per item (upper bound: the
  // plan's unit capacity; CTAs without an item exit after claiming the end marker)
  const uint32_t grid = static_cast<uint32_t>(
      std::max<uint64_t>(1, std::min<uint64_t>(a.slots * plan.cap_units, static_cast<uint64_t>(num_sms))));
  const bool can_split = plan.cap_units > km.krows;
  float* ws = can_split ? ctx_workspace(ctx, plan_cap_chunks(a.slots, workers) * 128 * (128 + 3), s) : nullptr;
  uint32_t* split_ctr = can_split ? ctx_split_ctr(ctx, plan_cap_chunks(a.slots, workers) + a.slots, s) : nullptr;

  // plain: 3-D [slots][n][D] maps with 128-row boxes; gathered tensors: 2-D [slots * n][D] row maps
  // (Q and O in both gather modes, K and V only when kGather == 1)
  constexpr bool kGQ = kGather != 0, kGKV = kGather == 1 || kGather == 3;
  auto tmap = [&](const void* base, bool gathered) {
    return gathered ? make_tmap_bf16_rows(base, D, a.slots * a.n, 64)
                    : cached_tmap_bf16_3d(base, D, a.n, a.slots, 64, 128);
  };
  const CUtensorMap tq = tmap(a.q, kGQ), tk = tmap(a.k, kGKV), tv = tmap(a.v, kGKV), to = tmap(a.o, kGQ);
  // 64-row boxes for tiles with an empty key half (plain K / V only)
  const CUtensorMap tk64 = kGKV ? tk : cached_tmap_bf16_3d(a.k, D, a.n, a.slots, 64, 64);
  const CUtensorMap tv64 = kGKV ? tv : cached_tmap_bf16_3d(a.v, D, a.n, a.slots, 64, 64);
  FwdParams p{};
  p.rows = a.rows;
  p.qg = static_cast<const __nv_bfloat16*>(a.q);
  p.kg = static_cast<const __nv_bfloat16*>(a.k);
  p.vg = static_cast<const __nv_bfloat16*>(a.v);
  p.n = a.n;
  p.slots = static_cast<uint32_t>(a.slots);
  p.krows = km.krows;
  p.kcols = km.kcols;
  p.hdr = plan.hdr;
  p.sl2 = a.scale * 1.4426950408889634f;
  // A zero scale would turn the masked sentinel into inf * 0 = NaN. 2^-100 instead: every
  // visible score's offset from the row max is then ~1e-28 and exp2 of it rounds to exactly 1.0f
  // (uniform weights, as with scale 0), while masked keys stay at -inf.
  if (p.sl2 == 0.0f) p.sl2 = 7.8886090522101181e-31f;
  p.list = km.list;
  p.halves = plan.half_heavy ? km.halves : nullptr;  // known one launch after a new mask version
  p.bitmaps = km.bitmaps;
  p.mask = reinterpret_cast<const uint4*>(km.mask);
  p.unit_desc = plan.unit_desc;
  p.split_info = plan.split_info;
  p.ws = ws;
  p.split_ctr = split_ctr;
  p.work_ctr = ctx.ctr;
  p.out = static_cast<__nv_bfloat16*>(a.o);
  p.row_max = a.row_max;
  p.row_sum = a.row_sum;
  p.trace = static_cast<uint64_t*>(g_trace.buffer);
  p.trace_ctas = g_trace.ctas;
  static std::atomic<uint64_t> attr_devices{0};  // per (D, MODE, kGather) instantiation
  constexpr bool kCanSkip = MODE == kModeBinblk || MODE == kModeDenseBinblk;
  once_per_device(attr_devices, [] {
    BBM_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<D, MODE, false, kGather, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<D>()));
    if constexpr (kCanSkip)
      BBM_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<D, MODE, false, kGather, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<D>()));
    if constexpr (kGather == 0)
      BBM_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<D, MODE, true, 0, false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<D>()));
  });
  if constexpr (kGather == 0) {
    if (p.trace) {  // event-tracing build of the same kernel (bbm_set_trace)
      attn_fwd_kernel<D, MODE, true, 0, false><<<grid, kThreadsOf<D>, smem_bytes<D>(), s>>>(tq, tk, tv, to, tk64, tv64, p);
      BBM_CUDA(cudaGetLastError());
      mark_launch_done(ctx, s);
      return;
    }
  }
  // the engine build for this mask (plan.partial_heavy arrives one launch after a new mask
  // version; both builds give bitwise identical results)
  if (kCanSkip && plan.partial_heavy) {
    attn_fwd_kernel<D, MODE, false, kGather, kCanSkip><<<grid, kThreadsOf<D>, smem_bytes<D>(), s>>>(tq, tk, tv, to, tk64, tv64, p);
    g_builds[1].fetch_add(1, std::memory_order_relaxed);
  } else {
    attn_fwd_kernel<D, MODE, false, kGather, false><<<grid, kThreadsOf<D>, smem_bytes<D>(), s>>>(tq, tk, tv, to, tk64, tv64, p);
    g_builds[0].fetch_add(1, std::memory_order_relaxed);
  }
  BBM_CUDA(cudaGetLastError());
  mark_launch_done(ctx, s);
}

template <int D, int kGather>
void launch_d(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms) {
  switch (a.variant) {
    case 0: launch_impl<D, kModeDense, kGather>(prep, a, s, num_sms); break;
    case 1: launch_impl<D, kModeNaive, kGather>(prep, a, s, num_sms); break;
    case 2: launch_impl<D, kModeBinblk, kGather>(prep, a, s, num_sms); break;
    case 3: launch_impl<D, kModeDenseBinblk, kGather>(prep, a, s, num_sms); break;
    default: throw ArgError("unknown variant");
  }
}

// Which RCM application a gather launch uses: BBM_GATHER=tma|passes|hybrid|lsu overrides
// (measurement). The default is the fastest on B200 and needs no scratch: every Q / K / V row
// gathered inside the kernel by LSU cp.async (two producer warps, 16 B per lane, four whole
// 128-byte box rows per warp instruction, row tokens looked up once per key tile, one tile
// ahead; C5 1.98 ms against 1.42 ms pre-permuted). The TMA
// tile::gather4 variant moves 4 rows (512 B) per TMA instruction and the TMA unit issues one
// every ~60 cycles (6.4 ms); the hybrid permutes K / V by passes and gathers Q / O with TMA
// (2.65 ms); passes over Q, K, V, O and the statistics around the plain kernel take 2.85 ms.
int gather_mode_of(int requested) {
  if (requested != kGatherAuto) return requested;
  static const int env = [] {
    const char* e = std::getenv("BBM_GATHER");
    if (e && std::string(e) == "tma") return static_cast<int>(kGatherTma);
    if (e && std::string(e) == "passes") return static_cast<int>(kGatherPasses);
    if (e && std::string(e) == "hybrid") return static_cast<int>(kGatherHybrid);
    return static_cast<int>(kGatherLsu);
  }();
  return env;
}

}  // namespace

void launch_attn_fwd(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms);

// RCM application by passes around the plain kernel (permute_rows / unpermute_rows,
// reorder.hpp:156-189): Q, K, V permuted into per-stream scratch, the forward over the permuted
// mask, O and the row statistics scattered back to the original tokens. Same results as the
// in-kernel gather (the kernel sees the same bf16 rows in the same positions).
static void launch_gather_passes(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms) {
  std::lock_guard<std::recursive_mutex> lk(prep.mu);  // the scratch belongs to this stream's context
  const uint64_t rowb = static_cast<uint64_t>(a.d) * 2;
  const uint64_t tb = (a.slots * a.n * rowb + 255) / 256 * 256;
  const uint64_t sb = (a.slots * a.n * 4 + 255) / 256 * 256;
  StreamCtx& ctx = prep.ctx_for(s);
  uint8_t* base = ctx_perm_scratch(ctx, 4 * tb + 2 * sb, s);
  AttnArgs b = a;
  b.rows = nullptr;
  b.q = base;
  b.k = base + tb;
  b.v = base + 2 * tb;
  b.o = base + 3 * tb;
  b.row_max = a.row_max ? reinterpret_cast<float*>(base + 4 * tb) : nullptr;
  b.row_sum = a.row_sum ? reinterpret_cast<float*>(base + 4 * tb + sb) : nullptr;
  launch_permute_rows(a.q, const_cast<void*>(b.q), a.rows, a.slots, a.n, rowb, false, s);
  launch_permute_rows(a.k, const_cast<void*>(b.k), a.rows, a.slots, a.n, rowb, false, s);
  launch_permute_rows(a.v, const_cast<void*>(b.v), a.rows, a.slots, a.n, rowb, false, s);
  launch_attn_fwd(prep, b, s, num_sms);
  launch_permute_rows(b.o, a.o, a.rows, a.slots, a.n, rowb, true, s);
  if (a.row_max) launch_permute_rows(b.row_max, a.row_max, a.rows, a.slots, a.n, 4, true, s);
  if (a.row_sum) launch_permute_rows(b.row_sum, a.row_sum, a.rows, a.slots, a.n, 4, true, s);
}

// Hybrid RCM application: K and V (each tile re-read by several row tiles) permuted into per-stream
// scratch by one pass each; Q rows gathered (tile::gather4, once per item) and O rows scattered
// (tile::scatter4) inside the kernel, row statistics written to their original tokens. Same
// results as the other two modes.
static void launch_gather_hybrid(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms) {
  std::lock_guard<std::recursive_mutex> lk(prep.mu);  // the scratch belongs to this stream's context
  const uint64_t rowb = static_cast<uint64_t>(a.d) * 2;
  const uint64_t tb = (a.slots * a.n * rowb + 255) / 256 * 256;
  StreamCtx& ctx = prep.ctx_for(s);
  uint8_t* base = ctx_perm_scratch(ctx, 2 * tb, s);
  AttnArgs b = a;
  b.k = base;
  b.v = base + tb;
  launch_permute_rows(a.k, const_cast<void*>(b.k), a.rows, a.slots, a.n, rowb, false, s);
  launch_permute_rows(a.v, const_cast<void*>(b.v), a.rows, a.slots, a.n, rowb, false, s);
  if (a.d == 64) launch_d<64, 2>(prep, b, s, num_sms);
  else launch_d<128, 2>(prep, b, s, num_sms);
}

void launch_attn_fwd(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms) {
  require(a.slots >= 1, "need at least one batch/head slot");
  require(a.n == prep.n, "mask preprocessing does not match this problem");
  require(a.slots < (1ull << 24), "too many slots for one launch");
  // work items (slot x row unit) are counted in 32 bits inside the kernels
  require(a.slots * (static_cast<uint64_t>(prep.kmeta.krows) + 1) + plan_cap_chunks(a.slots, static_cast<uint32_t>(num_sms)) <
              (1ull << 32),
          "too many slots x row tiles for one launch");
  if (a.slots * prep.kmeta.krows == 0) return;
  if (a.d != 64 && a.d != 128) throw ArgError("head dim must be 64 or 128 on the sm_100a kernel");
  // TMA descriptors and the 16-byte cp.async / vector row accesses need 16-byte aligned tensors
  for (const void* t : {a.q, a.k, a.v, static_cast<const void*>(a.o)})
    require((reinterpret_cast<uintptr_t>(t) & 15u) == 0, "q, k, v and out must be 16-byte aligned");
  if (launch_attn_fwd_pair(prep, a, s, num_sms)) return;  // only when selected (bbm_set_fwd_kernel)
  if (a.rows && gather_mode_of(a.gather_mode) == kGatherPasses) {
    launch_gather_passes(prep, a, s, num_sms);
  } else if (a.rows && gather_mode_of(a.gather_mode) == kGatherHybrid) {
    require(a.slots * a.n < (1ull << 31) - 1, "too many rows for the gather path (slots * n >= 2^31)");
    launch_gather_hybrid(prep, a, s, num_sms);
  } else if (a.rows && gather_mode_of(a.gather_mode) == kGatherLsu) {
    require(a.slots * a.n < (1ull << 31) - 1, "too many rows for the gather path (slots * n >= 2^31)");
    if (a.d == 64) launch_d<64, 3>(prep, a, s, num_sms);
    else launch_d<128, 3>(prep, a, s, num_sms);
  } else if (a.rows) {  // in-kernel RCM gather / scatter of token rows (2-D row coordinates are int32)
    require(a.slots * a.n < (1ull << 31) - 1, "too many rows for the gather path (slots * n >= 2^31)");
    if (a.d == 64) launch_d<64, 1>(prep, a, s, num_sms);
    else launch_d<128, 1>(prep, a, s, num_sms);
  } else {
    if (a.d == 64) launch_d<64, 0>(prep, a, s, num_sms);
    else launch_d<128, 0>(prep, a, s, num_sms);
  }
}

int attn_fwd_kernel_launches_per_call() { return 1; }

void fwd_build_counts(uint64_t& plain, uint64_t& skipping) {
  plain = g_builds[0].load();
  skipping = g_builds[1].load();
}

}  // namespace bbm
