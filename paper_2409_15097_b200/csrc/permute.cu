// permute.cu — device side of the RCM path (reorder.hpp:156-189).
//   permute_rows_kernel  K5: X'[a] = X[fwd[a]] (permute_rows) or X'[fwd[a]] = X[a]
//                        (unpermute_rows) over [slots][n][row_bytes], 16-byte vectors (4-byte
//                        ones for rows that are not 16-byte multiples, e.g. row statistics).
//   permute_mask_kernel  K6: mask'(a,b) = mask(fwd[a], fwd[b]) (permute_mask). One CTA per output
//                        row: the source row is staged in shared memory, each warp builds one
//                        64-bit output word from two 32-lane ballots (fwd reads coalesced).
#include <cuda_runtime.h>

#include <cstdint>

#include "bbm_internal.h"

namespace bbm {
namespace {

template <typename V>
__global__ void permute_rows_kernel(const V* __restrict__ src, V* __restrict__ dst,
                                    const uint32_t* __restrict__ fwd, uint64_t slots, uint64_t n,
                                    uint64_t vec_per_row, bool inverse) {
  const uint64_t total = slots * n * vec_per_row;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t c = t % vec_per_row;
    const uint64_t row = t / vec_per_row;
    const uint64_t a = row % n, s = row / n;
    const uint64_t f = fwd[a];
    const uint64_t base = s * n;
    if (!inverse)
      dst[(base + a) * vec_per_row + c] = src[(base + f) * vec_per_row + c];
    else
      dst[(base + f) * vec_per_row + c] = src[(base + a) * vec_per_row + c];
  }
}

__global__ void __launch_bounds__(256) permute_mask_kernel(const uint64_t* __restrict__ src,
                                                           uint64_t* __restrict__ dst,
                                                           const uint32_t* __restrict__ fwd,
                                                           uint64_t n, uint64_t src_wpr,
                                                           uint64_t dst_wpr) {
  extern __shared__ uint64_t row_words[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint64_t a = blockIdx.x; a < n; a += gridDim.x) {
    const uint64_t srow = fwd[a];
    __syncthreads();
    for (uint64_t w = threadIdx.x; w < src_wpr; w += blockDim.x)
      row_words[w] = src[srow * src_wpr + w];
    __syncthreads();
    for (uint64_t w = warp; w < dst_wpr; w += 8) {
      const uint64_t b0 = w * 64 + lane, b1 = b0 + 32;
      bool v0 = false, v1 = false;
      if (b0 < n) {
        const uint32_t c = fwd[b0];
        v0 = (row_words[c >> 6] >> (c & 63)) & 1ull;
      }
      if (b1 < n) {
        const uint32_t c = fwd[b1];
        v1 = (row_words[c >> 6] >> (c & 63)) & 1ull;
      }
      const uint32_t lo = __ballot_sync(0xffffffffu, v0);
      const uint32_t hi = __ballot_sync(0xffffffffu, v1);
      if (lane == 0) dst[a * dst_wpr + w] = (static_cast<uint64_t>(hi) << 32) | lo;
    }
  }
}

}  // namespace

void launch_permute_rows(const void* src, void* dst, const uint32_t* d_fwd, uint64_t slots,
                         uint64_t n, uint64_t row_bytes, bool inverse, cudaStream_t s) {
  // 16-byte vectors for rows of 16-byte multiples (Q/K/V/O), 4-byte ones otherwise (row stats)
  const bool wide = row_bytes % 16 == 0;
  const uint64_t vec = wide ? row_bytes / 16 : row_bytes / 4;
  const uint64_t total = slots * n * vec;
  if (total == 0) return;
  uint64_t grid = (total + 255) / 256;
  if (grid > 148ull * 32) grid = 148ull * 32;
  if (wide)
    permute_rows_kernel<uint4><<<static_cast<unsigned>(grid), 256, 0, s>>>(
        static_cast<const uint4*>(src), static_cast<uint4*>(dst), d_fwd, slots, n, vec, inverse);
  else
    permute_rows_kernel<uint32_t><<<static_cast<unsigned>(grid), 256, 0, s>>>(
        static_cast<const uint32_t*>(src), static_cast<uint32_t*>(dst), d_fwd, slots, n, vec, inverse);
  BBM_CUDA(cudaGetLastError());
}

void launch_permute_mask(const uint64_t* d_src, uint64_t* d_dst, const uint32_t* d_fwd,
                         uint64_t n, uint64_t src_wpr, uint64_t dst_wpr, cudaStream_t s) {
  if (n == 0) return;
  const size_t smem = src_wpr * 8;
  if (smem > 48 * 1024)
    BBM_CUDA(cudaFuncSetAttribute(permute_mask_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  const unsigned grid = static_cast<unsigned>(n < 148ull * 8 ? n : 148ull * 8);
  permute_mask_kernel<<<grid, 256, smem, s>>>(d_src, d_dst, d_fwd, n, src_wpr, dst_wpr);
  BBM_CUDA(cudaGetLastError());
}

}  // namespace bbm
