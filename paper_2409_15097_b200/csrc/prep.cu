// prep.cu — GPU mask preprocessor (the reference's preprocess_mask, engine.hpp:80-91, and the
// mask-model functions it calls, mask.hpp:184-247), B200-native.
//
// Kernels (all HBM-bound integer work; no tensor cores):
//   pack_bool_sums128  K1+K2  dense bool mask -> padded bit-packed mask + 128x128 block sums.
//                             uint4 loads (16 bools/lane, 512 B per warp per row), bytes folded to
//                             bits with shift/or, words assembled with warp shuffles, popc sums.
//   pad_packed                caller's packed words (ceil(n/64) per row) -> padded layout.
//   sums128            K2     padded packed mask -> 128x128 sums (uint4 per lane, smem reduce).
//   sums_generic              any BlockSpec: popcount_range per (row, tile), mask.hpp:167-199.
//   rowmeta                   per query-row tile: occupancy (mask.hpp:203-209), first maximal run
//                             of full tiles (mask.hpp:213-228), per-row stats partials
//                             (mask.hpp:230-247), ascending compacted KV-tile list (block-wide
//                             ballot prefix scan) with a full/partial flag.
//   compact_bitmaps    K3     every occupied 128x128 tile's 2 KiB of mask bits -> tile-major copy
//                             at its list position, so the attention kernel reads 16 B per row,
//                             fully coalesced, at an address known before the list entry.
//   finalize                  totals over rows (deterministic integer sums) + LPT row order.
#include <cuda_runtime.h>

#include <cstdint>

#include "bbm_internal.h"

namespace bbm {
namespace {

// 8 bytes that are each 0 or 1 (lo = bytes 0..3, hi = bytes 4..7) -> 8 bits, byte k -> bit k:
// byte i of lo + (hi << 4) is b_i + 16 b_{i+4}; the multiply gathers sum_i (b_i + 16 b_{i+4}) 2^i
// into the top byte, and no partial-product byte exceeds 255, so nothing carries across.
__device__ __forceinline__ uint32_t bits8_of_01(uint32_t lo, uint32_t hi) {
  return ((lo + (hi << 4)) * 0x01020408u) >> 24;
}
// any nonzero byte -> 1 (the slow path of bool inputs that hold other values than 0 / 1)
__device__ __forceinline__ uint32_t to01(uint32_t w) {
  w |= w >> 4;
  w |= w >> 2;
  w |= w >> 1;
  return w & 0x01010101u;
}

// grid (ceil(kcols/32), krows), 256 threads. Warp w owns column tiles 4*w .. 4*w+3 of the chunk
// (8 lanes x 16 bools each) and walks all 128 rows of the tile row.
__global__ void __launch_bounds__(256) pack_bool_sums128_kernel(
    const uint8_t* __restrict__ mask, uint64_t n, uint64_t stride, uint64_t* __restrict__ out,
    uint32_t kcols, uint32_t* __restrict__ sums) {
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t p = blockIdx.y;
  const uint32_t q = blockIdx.x * 32 + warp * 4 + (lane >> 3);  // column tile of this lane
  const uint64_t col0 = static_cast<uint64_t>(q) * 128 + (lane & 7) * 16;
  const bool col_ok = q < kcols && col0 < n;  // n % 16 == 0 on this path
  const uint64_t wpr = static_cast<uint64_t>(kcols) * 2;
  uint32_t count = 0;
  // rows in batches of kBatch: all loads of a batch are in flight before the first is used
  constexpr uint32_t kBatch = 8;
  for (uint32_t r0 = 0; r0 < 128; r0 += kBatch) {
    uint4 vb[kBatch];
#pragma unroll
    for (uint32_t b = 0; b < kBatch; ++b) {
      const uint64_t row = static_cast<uint64_t>(p) * 128 + r0 + b;
      vb[b] = (col_ok && row < n) ? __ldg(reinterpret_cast<const uint4*>(mask + row * stride + col0))
                                  : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (uint32_t b = 0; b < kBatch; ++b) {
      const uint64_t row = static_cast<uint64_t>(p) * 128 + r0 + b;
      uint4 v = vb[b];
      if ((v.x | v.y | v.z | v.w) & 0xFEFEFEFEu) {  // bytes other than 0 / 1: nonzero = true
        v.x = to01(v.x);
        v.y = to01(v.y);
        v.z = to01(v.z);
        v.w = to01(v.w);
      }
      const uint32_t bits16 = bits8_of_01(v.x, v.y) | (bits8_of_01(v.z, v.w) << 8);
      count += __popc(bits16);
      // lanes 4m..4m+3 hold the four 16-bit quarters of one 64-bit word
      const uint32_t pair = bits16 | (__shfl_xor_sync(0xffffffffu, bits16, 1) << 16);
      const uint32_t other = __shfl_xor_sync(0xffffffffu, pair, 2);
      if ((lane & 3) == 0 && q < kcols)
        out[row * wpr + static_cast<uint64_t>(q) * 2 + ((lane >> 2) & 1)] =
            static_cast<uint64_t>(pair) | (static_cast<uint64_t>(other) << 32);
    }
  }
  count += __shfl_xor_sync(0xffffffffu, count, 1);
  count += __shfl_xor_sync(0xffffffffu, count, 2);
  count += __shfl_xor_sync(0xffffffffu, count, 4);
  if ((lane & 7) == 0 && q < kcols) sums[p * kcols + q] = count;
}

// Generic bool path (n % 16 != 0 or unaligned rows): one thread per output word.
__global__ void pack_bool_generic_kernel(const uint8_t* __restrict__ mask, uint64_t n,
                                         uint64_t stride, uint64_t* __restrict__ out,
                                         uint32_t kcols, uint64_t total_words) {
  const uint64_t wpr = static_cast<uint64_t>(kcols) * 2;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total_words;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t row = t / wpr, w = t % wpr;
    uint64_t word = 0;
    if (row < n)
      for (uint32_t b = 0; b < 64; ++b) {
        const uint64_t c = w * 64 + b;
        if (c < n && mask[row * stride + c]) word |= 1ull << b;
      }
    out[t] = word;
  }
}

__global__ void pad_packed_kernel(const uint64_t* __restrict__ in, uint64_t n, uint64_t in_wpr,
                                  uint64_t* __restrict__ out, uint64_t out_wpr,
                                  uint64_t total_words) {
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total_words;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t row = t / out_wpr, w = t % out_wpr;
    out[t] = (row < n && w < in_wpr) ? in[row * in_wpr + w] : 0ull;
  }
}

// grid (ceil(kcols/32), krows), 256 threads: lane = column tile, warp = row phase.
__global__ void __launch_bounds__(256) sums128_kernel(const uint4* __restrict__ mask,
                                                      uint32_t kcols, uint32_t* __restrict__ sums) {
  __shared__ uint32_t part[8][32];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t p = blockIdx.y, q = blockIdx.x * 32 + lane;
  uint32_t count = 0;
  if (q < kcols) {
#pragma unroll 4
    for (uint32_t r = warp; r < 128; r += 8) {
      const uint4 v = __ldg(mask + (static_cast<uint64_t>(p) * 128 + r) * kcols + q);
      count += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    }
  }
  part[warp][lane] = count;
  __syncthreads();
  if (warp == 0 && q < kcols) {
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += part[w][lane];
    sums[p * kcols + q] = s;
  }
}

__device__ __forceinline__ uint32_t popcount_range_dev(const uint64_t* words, uint64_t c0,
                                                       uint64_t c1) {
  // mask.hpp:167-179
  if (c0 >= c1) return 0;
  const uint64_t w0 = c0 >> 6, w1 = (c1 - 1) >> 6;
  const uint64_t first = ~0ull << (c0 & 63);
  const uint64_t last = (c1 & 63) ? (~0ull >> (64 - (c1 & 63))) : ~0ull;
  if (w0 == w1) return __popcll(words[w0] & first & last);
  uint32_t c = __popcll(words[w0] & first) + __popcll(words[w1] & last);
  for (uint64_t w = w0 + 1; w < w1; ++w) c += __popcll(words[w]);
  return c;
}

// One thread per (p, q) tile of an arbitrary BlockSpec.
__global__ void sums_generic_kernel(const uint64_t* __restrict__ mask, uint64_t wpr, uint64_t n,
                                    uint64_t bi, uint64_t bj, uint64_t rows, uint64_t cols,
                                    uint32_t* __restrict__ sums) {
  const uint64_t total = rows * cols;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t q = t % cols, p = t / cols;
    const uint64_t i0 = p * bi, i1 = min(i0 + bi, n);
    const uint64_t c0 = q * bj, c1 = min(c0 + bj, n);
    uint32_t s = 0;
    for (uint64_t i = i0; i < i1; ++i) s += popcount_range_dev(mask + i * wpr, c0, c1);
    sums[t] = s;
  }
}

__device__ __forceinline__ uint32_t area_of(uint64_t n, uint64_t bi, uint64_t bj, uint64_t p,
                                            uint64_t q) {
  // BlockSums::block_area, mask.hpp:89-99 (true extent of edge blocks)
  const uint64_t ri = min(bi, n - p * bi), cj = min(bj, n - q * bj);
  return static_cast<uint32_t>(ri * cj);
}

// The per-row pass of one query row tile p by one CTA of 256 threads: occupancy
// (mask.hpp:203-209), the first maximal run of full tiles (mask.hpp:213-228), per-row stats
// partials (mask.hpp:230-247) and the ascending compacted KV-tile list (block-wide ballot scan)
// with a full/partial flag. Kernel view only (list != nullptr): a tile narrower than bj (ragged
// right edge) is never flagged full, so the attention kernel always applies its bitmap, whose
// bits beyond n are 0. Sums are read through L2 (__ldcg): the fused preprocessor calls this on
// sums written earlier in the same launch.
// sum_at(q): the tile sum of (p, q); s_list (optional, shared memory): a copy of the row's list;
// returns the row's list length.
template <class SumAt>
__device__ uint32_t rowmeta_row_t(SumAt sum_at, uint64_t n, uint64_t bi, uint64_t bj, uint64_t cols,
                                  uint64_t p, uint8_t* occ, uint32_t* offset, uint32_t* total,
                                  uint64_t* row_stats, uint32_t* list, uint32_t* cnt, uint32_t* s_list) {
  __shared__ uint32_t warp_cnt[8];
  __shared__ uint32_t s_run_start, s_run_end;
  __shared__ unsigned long long s_nz, s_full, s_ones;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    s_run_start = 0xFFFFFFFFu;
    s_run_end = 0xFFFFFFFFu;
    s_nz = s_full = s_ones = 0;
  }
  __syncthreads();
  uint32_t base = 0;  // running list length
  unsigned long long my_nz = 0, my_full = 0, my_ones = 0;
  for (uint64_t c0 = 0; c0 < cols; c0 += 256) {
    const uint64_t q = c0 + threadIdx.x;
    uint32_t s = 0, a = 0;
    bool in = q < cols;
    if (in) {
      s = sum_at(q);
      a = area_of(n, bi, bj, p, q);
      occ[p * cols + q] = s > 0 ? 1 : 0;
      my_nz += s > 0;
      my_full += s == a;
      my_ones += s;
      if (s == a) atomicMin(&s_run_start, static_cast<uint32_t>(q));
    }
    const bool o = in && s > 0;
    const uint32_t ballot = __ballot_sync(0xffffffffu, o);
    if (lane == 0) warp_cnt[warp] = __popc(ballot);
    __syncthreads();
    uint32_t before = base;
    for (uint32_t w = 0; w < warp; ++w) before += warp_cnt[w];
    before += __popc(ballot & ((1u << lane) - 1u));
    const bool flag_full = s == a && (q + 1) * bj <= n;
    if (list && o) {
      const uint32_t e = static_cast<uint32_t>(q) | (flag_full ? 0x80000000u : 0u);
      list[p * cols + before] = e;
      if (s_list) s_list[before] = e;
    }
    uint32_t chunk = 0;
    for (uint32_t w = 0; w < 8; ++w) chunk += warp_cnt[w];
    base += chunk;
    __syncthreads();
  }
  // end of the first maximal run: first non-full tile after its start (mask.hpp:219-221)
  const uint32_t start = s_run_start;
  if (start != 0xFFFFFFFFu) {
    for (uint64_t q = start + 1 + threadIdx.x; q < cols; q += 256) {
      if (sum_at(q) != area_of(n, bi, bj, p, q)) atomicMin(&s_run_end, static_cast<uint32_t>(q));
    }
  }
  atomicAdd(&s_nz, my_nz);
  atomicAdd(&s_full, my_full);
  atomicAdd(&s_ones, my_ones);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (start == 0xFFFFFFFFu) {
      offset[p] = 0;
      total[p] = 0;
    } else {
      const uint32_t end = s_run_end == 0xFFFFFFFFu ? static_cast<uint32_t>(cols) : s_run_end;
      offset[p] = start;
      total[p] = end - start;
    }
    row_stats[p * 3 + 0] = s_nz;
    row_stats[p * 3 + 1] = s_full;
    row_stats[p * 3 + 2] = s_ones;
    if (cnt) cnt[p] = base;
  }
  __syncthreads();
  return base;
}

__device__ void rowmeta_row(const uint32_t* sums, uint64_t n, uint64_t bi, uint64_t bj, uint64_t cols,
                            uint64_t p, uint8_t* occ, uint32_t* offset, uint32_t* total,
                            uint64_t* row_stats, uint32_t* list, uint32_t* cnt) {
  rowmeta_row_t([&](uint64_t q) { return __ldcg(sums + p * cols + q); }, n, bi, bj, cols, p, occ, offset,
                total, row_stats, list, cnt, nullptr);
}

// One CTA (256 threads) per row tile p; the row is walked in chunks of 256 tiles.
__global__ void __launch_bounds__(256) rowmeta_kernel(
    const uint32_t* sums, uint64_t n, uint64_t bi, uint64_t bj, uint64_t cols, uint8_t* occ,
    uint32_t* offset, uint32_t* total, uint64_t* row_stats, uint32_t* list, uint32_t* cnt) {
  rowmeta_row(sums, n, bi, bj, cols, blockIdx.x, occ, offset, total, row_stats, list, cnt);
}

// grid (kcols, krows), 128 threads: CTA copies the mask bits of list entry (p, k) (if it exists)
// to bitmap slot (p, k) — indexed by LIST POSITION, so the attention kernel can compute the
// address of tile j's bits without first loading the list entry.
__global__ void __launch_bounds__(128) compact_bitmaps_kernel(const uint4* __restrict__ mask,
                                                              uint32_t kcols,
                                                              const uint32_t* __restrict__ list,
                                                              const uint32_t* __restrict__ cnt,
                                                              uint4* __restrict__ bitmaps,
                                                              uint8_t* __restrict__ halves) {
  const uint32_t p = blockIdx.y, k = blockIdx.x;
  if (k >= cnt[p]) return;
  const uint32_t q = list[p * kcols + k] & 0x7FFFFFFFu;
  const uint32_t r = threadIdx.x;
  const uint4 w = mask[(static_cast<uint64_t>(p) * 128 + r) * kcols + q];
  bitmaps[(static_cast<uint64_t>(p) * kcols + k) * 128 + r] = w;
  // key halves of the tile that no row sees
  const int lo = __syncthreads_or((w.x | w.y) != 0u), hi = __syncthreads_or((w.z | w.w) != 0u);
  if (r == 0) halves[static_cast<uint64_t>(p) * kcols + k] = static_cast<uint8_t>((lo ? 0 : 1) | (hi ? 0 : 2));
}

__global__ void __launch_bounds__(1024) finalize_kernel(const uint64_t* __restrict__ row_stats,
                                                        uint64_t rows,
                                                        const uint32_t* __restrict__ cnt,
                                                        uint32_t* __restrict__ order,
                                                        unsigned long long* __restrict__ totals) {
  __shared__ unsigned long long acc[3];
  if (threadIdx.x < 3) acc[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long a0 = 0, a1 = 0, a2 = 0;
  for (uint64_t p = threadIdx.x; p < rows; p += blockDim.x) {
    a0 += row_stats[p * 3 + 0];
    a1 += row_stats[p * 3 + 1];
    a2 += row_stats[p * 3 + 2];
  }
  atomicAdd(&acc[0], a0);
  atomicAdd(&acc[1], a1);
  atomicAdd(&acc[2], a2);
  if (cnt && order) {
    // LPT order: rank = #rows with a longer list, ties broken by index (stable).
    for (uint64_t p = threadIdx.x; p < rows; p += blockDim.x) {
      const uint32_t c = cnt[p];
      uint32_t rank = 0;
      for (uint64_t o = 0; o < rows; ++o) {
        const uint32_t co = cnt[o];
        rank += (co > c) || (co == c && o < p);
      }
      order[rank] = static_cast<uint32_t>(p);
    }
  }
  __syncthreads();
  if (threadIdx.x < 3) totals[threadIdx.x] = acc[threadIdx.x];
}

// ------------------------------------------------------------------ fused preprocessor
// ONE launch turns the caller's mask into the whole kernel view. CTA (chunk, p, rs) handles 16 rows
// (slab rs of kRowSplits) of query tile row p over 32 column tiles (chunk): it packs / copies the
// rows into the padded mask and writes its per-tile popcounts as partial sums. The last CTA of tile
// row p to finish (one atomic per CTA, threadfence-reduction pattern) adds the partials into the
// tile sums and runs the per-row pass (occupancy, first run, stats, compacted list) and the bitmap
// compaction of that row. Counters reset themselves, so the next launch needs no memset. The
// row-statistics totals and the LPT row order are not on this path: the launches plan on the
// device from row_cnt, and the totals are summed when the host asks for them.
constexpr uint32_t kRowSplits = kPrepRowSplits;    // 128 rows / 16 per CTA
constexpr uint32_t kSlabRows = 128 / kRowSplits;
constexpr uint32_t kChunkTiles = 32;               // column tiles per CTA
constexpr uint32_t kStageCols = 512;               // stage B in shared memory up to N = 65536

struct FusedArgs {
  const uint8_t* bools;  // dense bool rows (IN == kInBool)
  uint64_t stride;
  const uint64_t* words; // packed rows, in_wpr words each (IN == kInWords); may alias km.mask
  uint64_t in_wpr;
  uint64_t n;
  uint32_t krows, kcols, chunks;
  uint64_t* mask;
  uint32_t* partial;     // [kRowSplits][krows][kcols]
  uint32_t* sums;
  uint8_t* occ;
  uint32_t *run_off, *run_len, *row_cnt, *list, *ctr;
  uint64_t* row_stats;
  uint4* bitmaps;
  uint8_t* halves;
};
enum : int { kInBool = 0, kInWords = 1 };

template <int IN>
__global__ void __launch_bounds__(256) prep_fused_kernel(const FusedArgs a) {
  __shared__ uint32_t s_cnt[kChunkTiles];
  __shared__ bool s_last;
  __shared__ uint32_t s_sums[kStageCols], s_list[kStageCols], s_half[kStageCols];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // a tile row's chunks x kRowSplits CTAs are consecutive, so its stage B runs while later rows
  // are still in stage A (only the last row's is a tail)
  const uint32_t per_row = a.chunks * kRowSplits;
  const uint32_t p = blockIdx.x / per_row;
  const uint32_t chunk = (blockIdx.x % per_row) % a.chunks;
  const uint32_t rs = (blockIdx.x % per_row) / a.chunks;
  const uint64_t wpr = static_cast<uint64_t>(a.kcols) * 2;
  const uint64_t row0 = static_cast<uint64_t>(p) * 128 + rs * kSlabRows;

  // ---- stage A: this CTA's 16 rows x 32 column tiles -> padded packed words + partial sums
  if constexpr (IN == kInBool) {
    // warp w owns column tiles 4w .. 4w+3 of the chunk, 8 lanes x 16 bools each
    const uint32_t q = chunk * kChunkTiles + warp * 4 + (lane >> 3);
    const uint64_t col0 = static_cast<uint64_t>(q) * 128 + (lane & 7) * 16;
    const bool col_ok = q < a.kcols && col0 < a.n;  // n % 16 == 0 on this path
    uint32_t count = 0;
    uint4 vb[kSlabRows];
#pragma unroll
    for (uint32_t b = 0; b < kSlabRows; ++b) {  // all 16 loads in flight before the first use
      const uint64_t row = row0 + b;
      vb[b] = (col_ok && row < a.n) ? __ldg(reinterpret_cast<const uint4*>(a.bools + row * a.stride + col0))
                                    : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (uint32_t b = 0; b < kSlabRows; ++b) {
      uint4 v = vb[b];
      if ((v.x | v.y | v.z | v.w) & 0xFEFEFEFEu) {  // bytes other than 0 / 1: nonzero = true
        v.x = to01(v.x);
        v.y = to01(v.y);
        v.z = to01(v.z);
        v.w = to01(v.w);
      }
      const uint32_t bits16 = bits8_of_01(v.x, v.y) | (bits8_of_01(v.z, v.w) << 8);
      count += __popc(bits16);
      // lanes 4m..4m+3 hold the four 16-bit quarters of one 64-bit word
      const uint32_t pair = bits16 | (__shfl_xor_sync(0xffffffffu, bits16, 1) << 16);
      const uint32_t other = __shfl_xor_sync(0xffffffffu, pair, 2);
      if ((lane & 3) == 0 && q < a.kcols)
        a.mask[(row0 + b) * wpr + static_cast<uint64_t>(q) * 2 + ((lane >> 2) & 1)] =
            static_cast<uint64_t>(pair) | (static_cast<uint64_t>(other) << 32);
    }
    count += __shfl_xor_sync(0xffffffffu, count, 1);
    count += __shfl_xor_sync(0xffffffffu, count, 2);
    count += __shfl_xor_sync(0xffffffffu, count, 4);
    if ((lane & 7) == 0 && q < a.kcols)
      a.partial[(static_cast<uint64_t>(rs) * a.krows + p) * a.kcols + q] = count;
  } else {
    // thread t: word w = t % 64 of the chunk (tile w / 2), rows t / 64 + 4 i
    if (threadIdx.x < kChunkTiles) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t w = threadIdx.x & 63;
    const uint64_t word = static_cast<uint64_t>(chunk) * 64 + w;
    uint32_t count = 0;
    if (word < wpr) {
      uint64_t v[kSlabRows / 4];
#pragma unroll
      for (uint32_t i = 0; i < kSlabRows / 4; ++i) {
        const uint64_t row = row0 + (threadIdx.x >> 6) + 4 * i;
        v[i] = (row < a.n && word < a.in_wpr) ? a.words[row * a.in_wpr + word] : 0ull;
      }
#pragma unroll
      for (uint32_t i = 0; i < kSlabRows / 4; ++i) {
        const uint64_t row = row0 + (threadIdx.x >> 6) + 4 * i;
        a.mask[row * wpr + word] = v[i];
        count += __popcll(v[i]);
      }
    }
    count += __shfl_xor_sync(0xffffffffu, count, 1);  // the tile's two words
    if ((lane & 1) == 0 && word < wpr) atomicAdd(&s_cnt[w >> 1], count);
    __syncthreads();
    const uint32_t q = chunk * kChunkTiles + threadIdx.x;
    if (threadIdx.x < kChunkTiles && q < a.kcols)
      a.partial[(static_cast<uint64_t>(rs) * a.krows + p) * a.kcols + q] = s_cnt[threadIdx.x];
  }

  // ---- stage B: the last CTA of tile row p builds that row's metadata. One thread publishes
  // the CTA's writes (the barrier orders them before its cumulative fence) and, if last, acquires
  // the other CTAs' writes for the whole CTA; reads of them go through L2 (__ldcg).
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&a.ctr[p], 1u) == per_row - 1;
    __threadfence();
  }
  __syncthreads();
  if (!s_last) return;
  // Stage B keeps the row's sums and list in shared memory (rows up to kStageCols tiles), so its
  // only L2 round trips are the partial sums in and the mask words of the bitmaps.
  if (a.kcols <= kStageCols) {
    for (uint32_t q = threadIdx.x; q < a.kcols; q += 256) {
      uint32_t v[kRowSplits];
#pragma unroll
      for (uint32_t r = 0; r < kRowSplits; ++r)
        v[r] = __ldcg(a.partial + (static_cast<uint64_t>(r) * a.krows + p) * a.kcols + q);
      uint32_t sum = 0;
#pragma unroll
      for (uint32_t r = 0; r < kRowSplits; ++r) sum += v[r];
      s_sums[q] = sum;
      a.sums[static_cast<uint64_t>(p) * a.kcols + q] = sum;
    }
    __syncthreads();
    const uint32_t cnt = rowmeta_row_t([&](uint64_t q) { return s_sums[q]; }, a.n, 128, 128, a.kcols, p, a.occ,
                                       a.run_off, a.run_len, a.row_stats, a.list, a.row_cnt, s_list);
    for (uint32_t k = threadIdx.x; k < cnt; k += 256) s_half[k] = 0;
    __syncthreads();
    const uint4* m4 = reinterpret_cast<const uint4*>(a.mask);
    constexpr uint32_t kU = 4;  // independent mask loads in flight per thread
    for (uint32_t i0 = threadIdx.x; i0 < cnt * 128; i0 += 256 * kU) {
      uint4 w[kU];
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u) {
        const uint32_t idx = i0 + u * 256;
        if (idx < cnt * 128) {
          const uint32_t q = s_list[idx >> 7] & 0x7FFFFFFFu;
          w[u] = __ldcg(m4 + (static_cast<uint64_t>(p) * 128 + (idx & 127)) * a.kcols + q);
        }
      }
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u) {
        const uint32_t idx = i0 + u * 256;
        if (idx < cnt * 128) {
          a.bitmaps[(static_cast<uint64_t>(p) * a.kcols + (idx >> 7)) * 128 + (idx & 127)] = w[u];
          const uint32_t seen = ((w[u].x | w[u].y) != 0u ? 1u : 0u) | ((w[u].z | w[u].w) != 0u ? 2u : 0u);
          if (seen) atomicOr(&s_half[idx >> 7], seen);
        }
      }
    }
    __syncthreads();
    // key halves no row of the tile sees (the forward loads and multiplies only the other half)
    for (uint32_t k = threadIdx.x; k < cnt; k += 256)
      a.halves[static_cast<uint64_t>(p) * a.kcols + k] = static_cast<uint8_t>(~s_half[k] & 3u);
    if (threadIdx.x == 0) a.ctr[p] = 0;
    return;
  }
  for (uint32_t q = threadIdx.x; q < a.kcols; q += 256) {
    uint32_t sum = 0;
#pragma unroll
    for (uint32_t r = 0; r < kRowSplits; ++r)
      sum += __ldcg(a.partial + (static_cast<uint64_t>(r) * a.krows + p) * a.kcols + q);
    a.sums[static_cast<uint64_t>(p) * a.kcols + q] = sum;
  }
  __syncthreads();
  rowmeta_row(a.sums, a.n, 128, 128, a.kcols, p, a.occ, a.run_off, a.run_len, a.row_stats, a.list, a.row_cnt);
  // K3: the row's occupied tiles' mask bits, tile-major at their list positions
  const uint32_t cnt = __ldcg(a.row_cnt + p);
  const uint4* m4 = reinterpret_cast<const uint4*>(a.mask);
  for (uint32_t idx = threadIdx.x; idx < cnt * 128; idx += 256) {
    const uint32_t k = idx >> 7, r = idx & 127;
    const uint32_t q = __ldcg(a.list + static_cast<uint64_t>(p) * a.kcols + k) & 0x7FFFFFFFu;
    a.bitmaps[(static_cast<uint64_t>(p) * a.kcols + k) * 128 + r] =
        __ldcg(m4 + (static_cast<uint64_t>(p) * 128 + r) * a.kcols + q);
    if (r == 0) a.halves[static_cast<uint64_t>(p) * a.kcols + k] = 0;  // wide rows: no half skipping
  }
  if (threadIdx.x == 0) a.ctr[p] = 0;

}

FusedArgs fused_args(const KernelMeta& km, uint64_t n) {
  FusedArgs a{};
  a.n = n;
  a.krows = km.krows;
  a.kcols = km.kcols;
  a.chunks = (km.kcols + kChunkTiles - 1) / kChunkTiles;
  a.mask = km.mask;
  a.partial = km.partial;
  a.sums = km.sums;
  a.occ = km.occ;
  a.run_off = km.run_off;
  a.run_len = km.run_len;
  a.row_cnt = km.row_cnt;
  a.list = km.list;
  a.ctr = km.ctr;
  a.row_stats = km.row_stats;
  a.bitmaps = km.bitmaps;
  a.halves = km.halves;
  return a;
}

uint64_t fused_grid(const FusedArgs& a) {
  return static_cast<uint64_t>(a.chunks) * a.krows * kRowSplits;
}

inline unsigned grid_for(uint64_t work, unsigned block) {
  uint64_t g = (work + block - 1) / block;
  if (g > 148ull * 32) g = 148ull * 32;
  return static_cast<unsigned>(g ? g : 1);
}

}  // namespace

void launch_pack_bool(const uint8_t* d_bool, uint64_t n, uint64_t stride, const KernelMeta& km,
                      cudaStream_t s) {
  const bool fast = (n % 16 == 0) && (stride % 16 == 0) &&
                    (reinterpret_cast<uintptr_t>(d_bool) % 16 == 0);
  if (fast) {
    dim3 grid((km.kcols + 31) / 32, km.krows);
    pack_bool_sums128_kernel<<<grid, 256, 0, s>>>(d_bool, n, stride, km.mask, km.kcols, km.sums);
  } else {
    const uint64_t words = static_cast<uint64_t>(km.krows) * 128 * km.kcols * 2;
    pack_bool_generic_kernel<<<grid_for(words, 256), 256, 0, s>>>(d_bool, n, stride, km.mask,
                                                                   km.kcols, words);
    launch_sums128(km, s);
  }
  BBM_CUDA(cudaGetLastError());
}

bool launch_prep_fused_bool(const uint8_t* d_bool, uint64_t n, uint64_t stride, const KernelMeta& km,
                            cudaStream_t s) {
  const bool fast = (n % 16 == 0) && (stride % 16 == 0) &&
                    (reinterpret_cast<uintptr_t>(d_bool) % 16 == 0);
  FusedArgs a = fused_args(km, n);
  const uint64_t grid = fused_grid(a);
  if (!fast || grid >= (1ull << 31)) return false;
  a.bools = d_bool;
  a.stride = stride;
  prep_fused_kernel<kInBool><<<static_cast<unsigned>(grid), 256, 0, s>>>(a);
  BBM_CUDA(cudaGetLastError());
  return true;
}

bool launch_prep_fused_words(const uint64_t* d_words, uint64_t in_wpr, uint64_t n, const KernelMeta& km,
                             cudaStream_t s) {
  FusedArgs a = fused_args(km, n);
  const uint64_t grid = fused_grid(a);
  if (grid >= (1ull << 31)) return false;
  a.words = d_words;
  a.in_wpr = in_wpr;
  prep_fused_kernel<kInWords><<<static_cast<unsigned>(grid), 256, 0, s>>>(a);
  BBM_CUDA(cudaGetLastError());
  return true;
}

void launch_pad_packed(const uint64_t* d_words, uint64_t n, const KernelMeta& km,
                       cudaStream_t s) {
  const uint64_t out_wpr = static_cast<uint64_t>(km.kcols) * 2;
  const uint64_t words = static_cast<uint64_t>(km.krows) * 128 * out_wpr;
  pad_packed_kernel<<<grid_for(words, 256), 256, 0, s>>>(d_words, n, (n + 63) / 64, km.mask,
                                                         out_wpr, words);
  BBM_CUDA(cudaGetLastError());
}

void launch_sums128(const KernelMeta& km, cudaStream_t s) {
  dim3 grid((km.kcols + 31) / 32, km.krows);
  sums128_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const uint4*>(km.mask), km.kcols, km.sums);
  BBM_CUDA(cudaGetLastError());
}

void launch_sums_generic(const KernelMeta& km, uint64_t n, uint64_t bi, uint64_t bj,
                         uint64_t rows, uint64_t cols, uint32_t* d_sums, cudaStream_t s) {
  sums_generic_kernel<<<grid_for(rows * cols, 256), 256, 0, s>>>(
      km.mask, static_cast<uint64_t>(km.kcols) * 2, n, bi, bj, rows, cols, d_sums);
  BBM_CUDA(cudaGetLastError());
}

void launch_rowmeta(const uint32_t* d_sums, uint64_t n, uint64_t bi, uint64_t bj, uint64_t rows,
                    uint64_t cols, uint8_t* d_occ, uint32_t* d_offset, uint32_t* d_total,
                    uint64_t* d_row_stats, uint32_t* d_list, uint32_t* d_cnt, cudaStream_t s) {
  rowmeta_kernel<<<static_cast<unsigned>(rows), 256, 0, s>>>(
      d_sums, n, bi, bj, cols, d_occ, d_offset, d_total, d_row_stats, d_list, d_cnt);
  BBM_CUDA(cudaGetLastError());
}

void launch_compact_bitmaps(const KernelMeta& km, cudaStream_t s) {
  dim3 grid(km.kcols, km.krows);
  compact_bitmaps_kernel<<<grid, 128, 0, s>>>(reinterpret_cast<const uint4*>(km.mask), km.kcols,
                                              km.list, km.row_cnt, km.bitmaps, km.halves);
  BBM_CUDA(cudaGetLastError());
}

void launch_finalize(const uint64_t* d_row_stats, uint64_t rows, const uint32_t* d_cnt,
                     uint32_t* d_order, uint64_t* d_totals, cudaStream_t s) {
  finalize_kernel<<<1, 1024, 0, s>>>(d_row_stats, rows, d_cnt, d_order,
                                     reinterpret_cast<unsigned long long*>(d_totals));
  BBM_CUDA(cudaGetLastError());
}

}  // namespace bbm
