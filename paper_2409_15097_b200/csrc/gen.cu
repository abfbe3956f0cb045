// gen.cu — mask families generated directly on the device (the reference's generators.hpp), bit
// for bit the reference's masks in its packed layout (mask.hpp:17-52), for the large-N configs
// whose host generation dominates setup (gen_random_sparse(32768) takes ~4 s on a host core).
//
//   causal / all-ones / windowed / dilated / global (generators.hpp:65-79, 127-166): one thread
//   per 64-bit word, the word's bits from the family's closed form.
//   random sparse (generators.hpp:171-183): ONE std::mt19937_64 stream drawn row-major over all
//   n^2 entries (uniform_unit(gen) < p, rng.hpp:15-17), then the forced diagonal. The stream is
//   inherently sequential, so one CTA runs it: each twist of the 312-word state is computed by
//   312 threads in two dependency phases (words [0,156) read only old words, words [156,312)
//   read the new words 156 back), every thread tempers and tests its draw, and the rare set bits
//   (density p) are OR-ed into the mask. ~150 cycles per 312 draws instead of ~13 ns per draw
//   on a host core.
#include <cuda_runtime.h>

#include <cstdint>

#include "bbm_internal.h"

namespace bbm {
namespace {

__global__ void family_words_kernel(const GenSpec g, uint64_t* __restrict__ words) {
  const uint64_t n = g.n, wpr = (n + 63) / 64, total = n * wpr;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = t / wpr, w = t % wpr, c0 = w * 64;
    // bits [lo, hi) of columns in this word, clipped to the row
    auto range = [&](uint64_t lo, uint64_t hi) -> uint64_t {
      lo = lo > c0 ? lo : c0;
      hi = hi < c0 + 64 ? hi : c0 + 64;
      hi = hi < n ? hi : n;
      if (lo >= hi) return 0ull;
      const uint64_t len = hi - lo;
      return (len == 64 ? ~0ull : ((1ull << len) - 1)) << (lo - c0);
    };
    uint64_t bits = 0;
    switch (g.family) {
      case kGenCausal: bits = range(0, i + 1); break;
      case kGenAllOnes: bits = range(0, n); break;
      case kGenWindowed:
      case kGenGlobal: {
        const uint64_t j0 = i >= g.w ? i - g.w : 0;
        const uint64_t j1 = g.causal ? i : (i + g.w < n - 1 ? i + g.w : n - 1);
        bits = range(j0, j1 + 1);
        if (g.family == kGenGlobal) {
          if (i < g.g) bits |= range(0, n);  // global rows see everything
          bits |= range(0, g.g);             // every row sees the global columns
        }
        break;
      }
      case kGenDilated: {
        // |i - j| <= w * d and (i - j) divisible by d
        const uint64_t reach = g.w * g.d;
        for (uint32_t b = 0; b < 64; ++b) {
          const uint64_t j = c0 + b;
          if (j >= n) break;
          const uint64_t dist = i > j ? i - j : j - i;
          if (dist <= reach && dist % g.d == 0) bits |= 1ull << b;
        }
        break;
      }
      default: break;
    }
    words[t] = bits;
  }
}

constexpr uint32_t kMtN = 312, kMtM = 156;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull, kMtUpper = 0xFFFFFFFF80000000ull, kMtLower = 0x7FFFFFFFull;

__device__ __forceinline__ uint64_t mt_mix(uint64_t a, uint64_t b) {
  const uint64_t x = (a & kMtUpper) | (b & kMtLower);
  return (x >> 1) ^ ((x & 1ull) ? kMtA : 0ull);
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t x) {
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}

// One CTA of 320 threads (312 state words). words must be zeroed beforehand.
__global__ void __launch_bounds__(320) random_stream_kernel(uint64_t n, uint64_t seed, double p,
                                                            uint64_t* __restrict__ words) {
  __shared__ uint64_t mt[kMtN];
  const uint32_t t = threadIdx.x;
  if (t == 0) {  // std::mt19937_64 seeding (sequential by definition)
    mt[0] = seed;
    for (uint32_t i = 1; i < kMtN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
  }
  __syncthreads();
  const uint64_t wpr = (n + 63) / 64, draws = n * n;
  // this thread's draw within every twist: index (twist * 312 + t) -> (row i, column j)
  uint64_t i = t / n, j = t % n;
  for (uint64_t base = 0; base < draws; base += kMtN) {
    uint64_t own = 0, next = 0, far = 0;
    if (t < kMtN) {
      own = mt[t];
      next = mt[(t + 1) % kMtN];
      far = mt[(t + kMtM) % kMtN];
    }
    __syncthreads();
    if (t < kMtN - kMtM) mt[t] = far ^ mt_mix(own, next);  // reads only old words
    __syncthreads();
    if (t >= kMtN - kMtM && t < kMtN - 1) mt[t] = mt[t - (kMtN - kMtM)] ^ mt_mix(own, next);
    if (t == kMtN - 1) mt[t] = mt[t - (kMtN - kMtM)] ^ mt_mix(own, mt[0]);  // wraps to the new mt[0]
    __syncthreads();
    if (t < kMtN && base + t < draws) {
      const uint64_t y = mt_temper(mt[t]);
      if (static_cast<double>(y >> 11) * 0x1.0p-53 < p)  // uniform_unit(gen) < p, rng.hpp:15-17
        atomicOr(reinterpret_cast<unsigned long long*>(words + i * wpr + (j >> 6)), 1ull << (j & 63));
    }
    // advance this thread's position by one twist (312 draws)
    j += kMtN;
    while (j >= n) {
      j -= n;
      ++i;
    }
  }
}

__global__ void diagonal_kernel(uint64_t n, uint64_t* __restrict__ words) {
  const uint64_t wpr = (n + 63) / 64;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    words[i * wpr + (i >> 6)] |= 1ull << (i & 63);
}

}  // namespace

void launch_generate(const GenSpec& g, uint64_t* d_words, cudaStream_t s) {
  const uint64_t wpr = (g.n + 63) / 64, total = g.n * wpr;
  const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, 148ull * 16)));
  if (g.family == kGenRandom) {
    BBM_CUDA(cudaMemsetAsync(d_words, 0, total * 8, s));
    random_stream_kernel<<<1, 320, 0, s>>>(g.n, g.seed, g.p, d_words);
    if (g.diag) diagonal_kernel<<<static_cast<unsigned>(std::min<uint64_t>((g.n + 255) / 256, 1024)), 256, 0, s>>>(g.n, d_words);
  } else {
    family_words_kernel<<<grid, 256, 0, s>>>(g, d_words);
  }
  BBM_CUDA(cudaGetLastError());
}

}  // namespace bbm
