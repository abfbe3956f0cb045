// plan.cu — launch plans of the attention kernels, built ON THE DEVICE from the prep's tile lists.
//
// The reference schedules row blocks in waves of host threads (run_in_waves, engine.hpp:264-278)
// and walks each row block's column blocks in ascending order (engine.hpp:311). Here a plan cuts
// every (slot, query row tile) into work items for the persistent kernel: a row unit is a row
// tile's whole tile walk, or — for rows much longer than a CTA's fair share — one balanced chunk
// of it (split-KV; the chunks' partials are combined in chunk order, so results are
// deterministic). Units are ordered longest first (LPT), ties by row index.
//
// Because the plan is computed from row_cnt / list by a kernel, a mask update
// (bbm_prep_update_*) followed by a launch needs no host round trip: the stale plan is simply
// rebuilt on the launching stream.
//
// Unit length L: with dynamic longest-first claiming the makespan is about (average work per CTA
// + longest unit), so L is half a CTA's average share, and at least 16 tiles (combining partials
// goes through global memory and costs more than a few tiles). L is doubled until the launch's
// chunks fit the per-stream workspace (plan_cap_chunks).
//
// The masked variants split IN KEY SPACE, at boundaries set by the occupied tiles only: chunk c
// of a row holds the same occupied tiles, in the same order, whether the variant walks the
// compacted list (binblk, dense_binblk) or every tile of the key range (naive, whose extra tiles
// are fully masked and change nothing). Their partials and the combine are then identical, so the
// masked variants agree bit for bit at every size (test_engine.cpp:112-134). The dense variant
// ignores the mask and splits by position.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "bbm_internal.h"
#include "bbm_sort.cuh"

namespace bbm {
namespace {

constexpr uint32_t kPlanThreads = 512;
constexpr uint32_t kMinUnit = 16;

// minimum split unit in tiles (BBM_MIN_UNIT overrides, for experiments)
uint32_t min_unit() {
  static const uint32_t v = [] {
    const char* e = std::getenv("BBM_MIN_UNIT");
    const long x = e ? std::atol(e) : 0;
    return x >= 1 && x <= 1024 ? static_cast<uint32_t>(x) : kMinUnit;
  }();
  return v;
}

struct PlanArgs {
  int cls;
  uint32_t krows, kcols;
  const uint32_t* row_cnt;
  const uint32_t* list;
  const uint8_t* halves;  // nullptr for the column view
  uint64_t slots;
  uint32_t workers, min_unit;
  uint64_t cap_chunks;  // bound on slots * split chunks (workspace blocks)
  uint32_t cap_units, cap_split;
  PlanHdr* hdr;
  uint4* desc;
  uint2* split_info;
  uint4* tmp;
  uint32_t* hist;
};

__device__ __forceinline__ uint32_t chunks_of(uint32_t occ, uint64_t L) {
  if (occ <= L) return 0u;
  const uint64_t k = (occ + L - 1) / L;
  return static_cast<uint32_t>(k < 255 ? k : 255);
}

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(const PlanArgs a) {
  __shared__ unsigned long long s_L;
  auto occ_of = [&](uint32_t p) { return a.cls == kPlanDense ? a.kcols : a.row_cnt[p]; };
  auto walk_of = [&](uint32_t p) { return a.cls == kPlanList ? a.row_cnt[p] : a.kcols; };

  // ---- unit length
  unsigned long long my = 0;
  for (uint32_t p = threadIdx.x; p < a.krows; p += kPlanThreads) my += occ_of(p);
  const unsigned long long total = block_sum<kPlanThreads>(my) * a.slots;
  uint64_t L = (total / max(1u, a.workers) + 1) / 2;
  if (L < a.min_unit) L = a.min_unit;
  // full tiles (list entries with bit 31): the forward's choice of softmax engine build
  unsigned long long fl = 0, hv = 0;
  if (a.cls == kPlanList)
    for (uint32_t p = threadIdx.x; p < a.krows; p += kPlanThreads)
      for (uint32_t o = 0; o < a.row_cnt[p]; ++o) {
        fl += a.list[static_cast<uint64_t>(p) * a.kcols + o] >> 31;
        if (a.halves) hv += a.halves[static_cast<uint64_t>(p) * a.kcols + o] != 0;
      }
  const unsigned long long full = block_sum<kPlanThreads>(fl);
  const unsigned long long half_tiles = block_sum<kPlanThreads>(hv);
  for (;;) {
    unsigned long long c = 0;
    for (uint32_t p = threadIdx.x; p < a.krows; p += kPlanThreads) c += chunks_of(occ_of(p), L);
    const unsigned long long chunks = block_sum<kPlanThreads>(c);
    if (chunks * a.slots <= a.cap_chunks && a.krows + chunks <= a.cap_units) break;
    L *= 2;
  }
  if (threadIdx.x == 0) s_L = L;
  __syncthreads();
  L = s_L;

  // ---- units in row order: offsets by block scans over the rows, chunk by chunk
  uint32_t u_carry = 0, s_carry = 0, c_carry = 0;
  for (uint32_t p0 = 0; p0 < a.krows; p0 += kPlanThreads) {
    const uint32_t p = p0 + threadIdx.x;
    const bool in = p < a.krows;
    const uint32_t occ = in ? occ_of(p) : 0u, walk = in ? walk_of(p) : 0u;
    const uint32_t k = in ? chunks_of(occ, L) : 0u;
    uint32_t ut, st, ct;
    const uint32_t ub = u_carry + block_exscan<kPlanThreads, uint32_t>(in ? (k ? k : 1u) : 0u, &ut);
    const uint32_t sb = s_carry + block_exscan<kPlanThreads, uint32_t>(k ? 1u : 0u, &st);
    const uint32_t cb = c_carry + block_exscan<kPlanThreads, uint32_t>(k, &ct);
    if (in) {
      if (k == 0) {
        a.tmp[ub] = make_uint4(p, 0, walk, kNoSplit);  // walk == 0: a fully masked row tile
      } else {
        a.split_info[sb] = make_uint2(k, cb);
        auto first_occ = [&](uint32_t c) { return (occ / k) * c + min(c, occ % k); };
        auto key_of = [&](uint32_t o) {
          return a.cls == kPlanDense ? o : (a.list[static_cast<uint64_t>(p) * a.kcols + o] & 0x7FFFFFFFu);
        };
        for (uint32_t c = 0; c < k; ++c) {
          const uint32_t o0 = first_occ(c), o1 = first_occ(c + 1);
          if (a.cls == kPlanNaive) {
            const uint32_t kv0 = c == 0 ? 0u : key_of(o0), kv1 = c + 1 == k ? a.kcols : key_of(o1);
            a.tmp[ub + c] = make_uint4(p, kv0, kv1 - kv0, (sb << 8) | c);
          } else {
            a.tmp[ub + c] = make_uint4(p, o0, o1 - o0, (sb << 8) | c);  // list positions
          }
        }
      }
    }
    u_carry += ut;
    s_carry += st;
    c_carry += ct;
  }
  __syncthreads();

  // ---- longest first (tiles walked), ties by row order
  const uint32_t units = u_carry;
  lpt_sort<kPlanThreads>([&](uint32_t i) { return a.tmp[i].z; }, units, a.kcols, a.hist,
           [&](uint32_t pos, uint32_t i) { a.desc[pos] = a.tmp[i]; });
  if (threadIdx.x == 0)
    *a.hdr = PlanHdr{units, s_carry, c_carry, static_cast<uint32_t>(L < 0xFFFFFFFFull ? L : 0xFFFFFFFFull),
                     static_cast<uint32_t>(total / max(1ull, static_cast<unsigned long long>(a.slots))),
                     static_cast<uint32_t>(full), static_cast<uint32_t>(half_tiles)};
}

__global__ void __launch_bounds__(kPlanThreads) lpt_order_kernel(const uint32_t* __restrict__ keys,
                                                                 uint32_t count, uint32_t max_key,
                                                                 uint32_t* __restrict__ hist,
                                                                 uint32_t* __restrict__ out) {
  lpt_sort<kPlanThreads>([&](uint32_t i) { return keys[i]; }, count, max_key, hist,
           [&](uint32_t pos, uint32_t i) { out[pos] = i; });
}

}  // namespace

uint64_t plan_cap_chunks(uint64_t slots, uint32_t workers) {
  return 4ull * std::max(1u, workers) + 4 + slots;
}

uint32_t plan_cap_units(uint32_t krows, uint32_t kcols, uint64_t slots, uint32_t workers) {
  if (kcols <= min_unit()) return krows;  // L >= min_unit tiles: no row can split
  const uint64_t extra = plan_cap_chunks(slots, workers) / std::max<uint64_t>(1, slots) + 1;
  return static_cast<uint32_t>(std::min<uint64_t>(krows + extra, static_cast<uint64_t>(krows) * 256));
}

void build_plan(const TileView& v, int cls, uint64_t slots, uint32_t workers, DevPlan& plan,
                cudaStream_t s) {
  PlanArgs a{};
  a.cls = cls;
  a.krows = v.tiles;
  a.kcols = v.partners;
  a.row_cnt = v.cnt;
  a.list = v.list;
  a.halves = v.halves;
  a.slots = slots;
  a.workers = workers;
  a.min_unit = min_unit();
  a.cap_chunks = plan_cap_chunks(slots, workers);
  a.cap_units = plan.cap_units;
  a.cap_split = plan.cap_split;
  a.hdr = plan.hdr;
  a.desc = plan.unit_desc;
  a.split_info = plan.split_info;
  a.tmp = plan.tmp;
  a.hist = plan.hist;
  plan_kernel<<<1, kPlanThreads, 0, s>>>(a);
  BBM_CUDA(cudaGetLastError());
}

void launch_lpt_order(const uint32_t* keys, uint32_t count, uint32_t max_key, uint32_t* scratch,
                      uint32_t* out, cudaStream_t s) {
  lpt_order_kernel<<<1, kPlanThreads, 0, s>>>(keys, count, max_key, scratch, out);
  BBM_CUDA(cudaGetLastError());
}

const DevPlan& plan_for(const Prep& prep, StreamCtx& ctx, const TileView& v, int cls, uint64_t slots,
                        uint32_t workers, cudaStream_t s) {
  DevPlan& pl = ctx.plans[std::make_tuple(cls + 8 * v.id, slots, workers)];
  if (!pl.mem) {
    pl.cap_units = plan_cap_units(v.tiles, v.partners, slots, workers);
    pl.cap_split = std::min<uint32_t>(pl.cap_units, static_cast<uint32_t>(
                                                        plan_cap_chunks(slots, workers) / std::max<uint64_t>(1, slots) + 1));
    const size_t off_desc = 256;
    const size_t off_tmp = off_desc + static_cast<size_t>(pl.cap_units) * 16;
    const size_t off_split = off_tmp + static_cast<size_t>(pl.cap_units) * 16;
    const size_t off_hist = off_split + static_cast<size_t>(pl.cap_split) * 8;
    const size_t bytes = off_hist + (static_cast<size_t>(v.partners) + 2) * 4;
    void* mem = nullptr;
    BBM_CUDA(cudaMalloc(&mem, bytes));
    pl.mem = static_cast<uint8_t*>(mem);
    pl.hdr = reinterpret_cast<PlanHdr*>(pl.mem);
    pl.unit_desc = reinterpret_cast<uint4*>(pl.mem + off_desc);
    pl.tmp = reinterpret_cast<uint4*>(pl.mem + off_tmp);
    pl.split_info = reinterpret_cast<uint2*>(pl.mem + off_split);
    pl.hist = reinterpret_cast<uint32_t*>(pl.mem + off_hist);
    pl.version = 0;
  }
  if (pl.version != prep.version) {
    build_plan(v, cls, slots, workers, pl, s);
    pl.version = prep.version;
    if (!pl.host_hdr) {
      BBM_CUDA(cudaMallocHost(&pl.host_hdr, 12));
      BBM_CUDA(cudaEventCreateWithFlags(&pl.hdr_ev, cudaEventDisableTiming));
    }
    BBM_CUDA(cudaMemcpyAsync(pl.host_hdr, &pl.hdr->occupied, 12, cudaMemcpyDeviceToHost, s));
    BBM_CUDA(cudaEventRecord(pl.hdr_ev, s));
  } else if (pl.known_version != pl.version) {
    const cudaError_t q = cudaEventQuery(pl.hdr_ev);
    if (q == cudaSuccess) {
      pl.partial_heavy = (pl.host_hdr[0] - pl.host_hdr[1]) * 2ull > pl.host_hdr[0];
      // skipping empty 64-row partner halves (an extra metadata load per K / V tile, N = 64 score
      // MMAs) pays off once at least ~10 % of the occupied tiles have one: same-box A/B, forward
      // C5 (40 %) -6 %, C2 (16.5 %) -1.5 %, backward C5 -7 %, C2 -1.7 %
#ifndef BBM_HALF_GATE_PCT
#define BBM_HALF_GATE_PCT 10
#endif
      pl.half_heavy = pl.host_hdr[2] * 100ull >= pl.host_hdr[0] * static_cast<uint64_t>(BBM_HALF_GATE_PCT) &&
                      pl.host_hdr[0] > 0;
      pl.known_version = pl.version;
    } else if (q == cudaErrorNotReady) {
      (void)cudaGetLastError();  // not an error: the header has not arrived yet
    } else {
      BBM_CUDA(q);
    }
  }
  return pl;
}

float* ctx_workspace(StreamCtx& ctx, size_t floats, cudaStream_t s) {
  if (floats > ctx.ws_floats) {
    // the previous workspace may still be in use by launches queued on this stream
    if (ctx.ws) {
      BBM_CUDA(cudaStreamSynchronize(s));
      cudaFree(ctx.ws);
    }
    ctx.ws = nullptr;
    ctx.ws_floats = 0;
    BBM_CUDA(cudaMalloc(&ctx.ws, floats * sizeof(float)));
    ctx.ws_floats = floats;
  }
  return ctx.ws;
}

uint8_t* ctx_perm_scratch(StreamCtx& ctx, size_t bytes, cudaStream_t s) {
  if (bytes > ctx.perm_bytes) {
    if (ctx.perm) {
      BBM_CUDA(cudaStreamSynchronize(s));
      cudaFree(ctx.perm);
    }
    ctx.perm = nullptr;
    ctx.perm_bytes = 0;
    BBM_CUDA(cudaMalloc(&ctx.perm, bytes));
    ctx.perm_bytes = bytes;
  }
  return ctx.perm;
}

uint32_t* ctx_split_ctr(StreamCtx& ctx, size_t count, cudaStream_t s) {
  if (count > ctx.split_ctr_n) {
    if (ctx.split_ctr) {
      BBM_CUDA(cudaStreamSynchronize(s));
      cudaFree(ctx.split_ctr);
    }
    ctx.split_ctr = nullptr;
    ctx.split_ctr_n = 0;
    BBM_CUDA(cudaMalloc(&ctx.split_ctr, count * sizeof(uint32_t)));
    BBM_CUDA(cudaMemsetAsync(ctx.split_ctr, 0, count * sizeof(uint32_t), s));
    ctx.split_ctr_n = count;
  }
  return ctx.split_ctr;
}

}  // namespace bbm
