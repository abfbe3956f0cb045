// bbm_softmax.cuh — the per-row softmax math shared by the forward kernels (attn_fwd.cu,
// attn_fwd_pair.cu): masking by sentinel, chunk maxima, exp2 + bf16 packing of P with the fp32
// row-sum accumulation, and the bf16 staging of O. Both kernels call these in the same order per
// row, so they produce bit-identical outputs and statistics (online_update, engine.hpp:206-235).
#pragma once
#include <cstdint>

#include "bbm_ptx.cuh"

namespace bbm {
namespace softmax {

using namespace ptx;

constexpr float kRescaleThreshold = 8.0f;  // log2 units: the running max is raised only past this
constexpr float kLn2 = 0.69314718055994530942f;

// Replace the scores of invisible keys by a sentinel in place: -inf (or +inf when the scale is
// negative, so that scale * sentinel = -inf). The max and exp passes then need no selects.
__device__ __forceinline__ void apply_mask(uint32_t (&r)[32], uint32_t mw, uint32_t sentinel) {
#pragma unroll
  for (uint32_t i = 0; i < 32; ++i) r[i] = ((mw >> i) & 1u) ? r[i] : sentinel;
}

// Max of 32 (already masked) raw scores of one row chunk; of the negated scores when the scale
// is negative (FMNMX takes negated operands for free).
template <bool kNeg>
__device__ __forceinline__ float chunk_max(const uint32_t (&r)[32]) {
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (uint32_t i = 0; i < 32; i += 4) {
    float a = __uint_as_float(r[i]), b = __uint_as_float(r[i + 1]);
    float c = __uint_as_float(r[i + 2]), d = __uint_as_float(r[i + 3]);
    if constexpr (kNeg) { a = -a; b = -b; c = -c; d = -d; }
    m0 = fmax3(m0, a, b);
    m1 = fmax3(m1, c, d);
  }
  return fmaxf(m0, m1);
}

// Which of the 16 exponential pairs of a chunk run as a polynomial on the FMA pipe instead of
// MUFU ex2 (bit i = pair i): 6 of 16 balances the XU pipe (8 cycles per warp instruction) against
// the extra issue slots of the polynomial (~10 instructions per pair).
#ifndef BBM_POLY_PAIRS
#define BBM_POLY_PAIRS 0x0707u
#endif
constexpr uint32_t kPolyPairs = BBM_POLY_PAIRS;

// P chunk: 32 scores -> 16 packed bf16x2; accumulates the fp32 sum of the unrounded
// exponentials into the packed pair `lacc`. Scale/shift and the sum run two lanes per
// instruction (FFMA2 / FADD2).
__device__ __forceinline__ void chunk_exp(const uint32_t (&r)[32], uint64_t sl2x2, uint64_t neg_m_x2,
                                          uint32_t (&pk)[16], uint64_t& lacc) {
#pragma unroll
  for (uint32_t i = 0; i < 32; i += 2) {
    const uint64_t x = ffma2(f2_pack(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sl2x2,
                             neg_m_x2);
    const float x0 = f2_lo(x), x1 = f2_hi(x);
    float e0, e1;
    if ((kPolyPairs >> ((i / 2) & 15)) & 1u) {
      exp2_poly2(x0, x1, e0, e1);  // this pair on the FMA pipe
    } else {
      e0 = fast_exp2(x0);  // MUFU
      e1 = fast_exp2(x1);
    }
    lacc = fadd2(lacc, f2_pack(e0, e1));
    pk[i / 2] = pack_bf16x2(e0, e1);
  }
}

// 32 fp32 -> 4 x 16 B of bf16 into a 128B-swizzled staging row
__device__ __forceinline__ void stage_chunk32(uint8_t* rowp, uint32_t row, uint32_t chunk0,
                                              const float* v, float inv) {
#pragma unroll
  for (uint32_t c = 0; c < 4; ++c) {
    uint4 w;
    w.x = pack_bf16x2(v[c * 8 + 0] * inv, v[c * 8 + 1] * inv);
    w.y = pack_bf16x2(v[c * 8 + 2] * inv, v[c * 8 + 3] * inv);
    w.z = pack_bf16x2(v[c * 8 + 4] * inv, v[c * 8 + 5] * inv);
    w.w = pack_bf16x2(v[c * 8 + 6] * inv, v[c * 8 + 7] * inv);
    *reinterpret_cast<uint4*>(rowp + (((chunk0 + c) ^ (row & 7)) << 4)) = w;
  }
}


}  // namespace softmax
}  // namespace bbm
