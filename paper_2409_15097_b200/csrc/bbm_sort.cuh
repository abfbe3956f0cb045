// bbm_sort.cuh — CTA-wide scans and the stable longest-first (LPT) ordering shared by the launch
// planner (plan.cu) and the fused preprocessor (prep.cu). Device code only.
#pragma once
#include <cstdint>

namespace bbm {

// Exclusive prefix sum of one value per thread over the CTA (kThreads threads); returns the
// thread's exclusive prefix and writes the CTA total to *total.
template <uint32_t kThreads, class T>
__device__ __forceinline__ T block_exscan(T v, T* total) {
  __shared__ T warp_sums[kThreads / 32];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (uint32_t o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T w = lane < kThreads / 32 ? warp_sums[lane] : T(0);
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kThreads / 32) warp_sums[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const T before = (warp ? warp_sums[warp - 1] : T(0)) + x - v;
  *total = warp_sums[kThreads / 32 - 1];
  __syncthreads();
  return before;
}

template <uint32_t kThreads, class T>
__device__ __forceinline__ T block_sum(T v) {
  T total;
  block_exscan<kThreads>(v, &total);
  return total;
}

// Stable LPT order of `count` items with keys in [0, max_key]: out[rank] = value(i), rank = number
// of items with a larger key plus items with the same key and a smaller index. Counting sort:
// histogram, descending exclusive scan, then one warp scatters in index order (match_any gives
// each lane its rank among equal keys of its group of 32).
template <uint32_t kThreads, class KeyFn, class StoreFn>
__device__ void lpt_sort(KeyFn key, uint32_t count, uint32_t max_key, uint32_t* hist, StoreFn store) {
  for (uint32_t v = threadIdx.x; v <= max_key; v += kThreads) hist[v] = 0;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < count; i += kThreads) atomicAdd(&hist[min(key(i), max_key)], 1u);
  __syncthreads();
  // descending exclusive scan: start[v] = sum of hist[w] for w > v; chunks from the top key down
  uint32_t carry = 0;
  for (uint32_t c0 = 0; c0 <= max_key; c0 += kThreads) {
    const uint32_t idx = c0 + threadIdx.x;  // position from the top
    const uint32_t v = idx <= max_key ? max_key - idx : 0;
    const uint32_t h = idx <= max_key ? hist[v] : 0u;
    uint32_t tot;
    const uint32_t before = block_exscan<kThreads>(h, &tot);
    if (idx <= max_key) hist[v] = carry + before;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    for (uint32_t i0 = 0; i0 < count; i0 += 32) {
      const uint32_t i = i0 + lane;
      const bool ok = i < count;
      const uint32_t v = ok ? min(key(i), max_key) : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, v);
      const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
      const uint32_t base = ok ? hist[v] : 0u;
      __syncwarp();
      if (ok) store(base + rank, i);
      if (ok && rank == 0) hist[v] = base + __popc(peers);
      __syncwarp();
    }
  }
  __syncthreads();
}

}  // namespace bbm
