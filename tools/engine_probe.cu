// engine_probe.cu — softmax-engine throughput by work organisation (measurement tool).
//
// Both layouts run the forward kernel's per-tile math on scores resident in TMEM (scale/shift
// FFMA2, 6/16 polynomial exp2 pairs, FADD2 row sums, bf16 packing, P written back with tcgen05.st),
// 8 engine warps per CTA, one CTA per SM:
//   A "halves": two warps per TMEM lane quadrant split each row's 128 columns (64 each), exchange
//      the partial row max through shared memory and a named barrier every tile, and all 8 warps
//      work on the same tile (the current kernel).
//   B "rows":  one thread per row owns all 128 columns (two passes over TMEM: max, then exp); warps
//      4-7 and 8-11 are two independent streams on different S buffers, with no barrier between
//      them (FA4's two-softmax-warpgroup layout).
// With a concurrent MMA stream (one thread issuing 128x128x16 SS MMAs into spare TMEM columns for
// the whole run) the same loops show how much tensor-core traffic slows the engine.
// Output: cycles per 128x128 tile (all tiles of both streams / elapsed).
#include <cstdio>

#include "../paper_2409_15097_b200/csrc/bbm_ptx.cuh"

using namespace bbm::ptx;

constexpr uint32_t kTiles = 512;  // tiles per CTA (layout B: 256 per stream)

__device__ __forceinline__ void exp_chunk(const uint32_t (&r)[32], uint64_t sl2x2, uint64_t nm2, uint32_t (&pk)[16],
                                          uint64_t& lacc) {
#pragma unroll
  for (uint32_t i = 0; i < 32; i += 2) {
    const uint64_t x = ffma2(f2_pack(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sl2x2, nm2);
    float e0, e1;
    if ((0x0707u >> ((i / 2) & 15)) & 1u) {
      exp2_poly2(f2_lo(x), f2_hi(x), e0, e1);
    } else {
      e0 = fast_exp2(f2_lo(x));
      e1 = fast_exp2(f2_hi(x));
    }
    lacc = fadd2(lacc, f2_pack(e0, e1));
    pk[i / 2] = pack_bf16x2(e0, e1);
  }
}

__device__ __forceinline__ float max32(const uint32_t (&r)[32]) {
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (uint32_t i = 0; i < 32; i += 4) {
    m0 = fmax3(m0, __uint_as_float(r[i]), __uint_as_float(r[i + 1]));
    m1 = fmax3(m1, __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
  }
  return fmaxf(m0, m1);
}

template <int LAYOUT, bool kMma, bool kSync = false>
__global__ void __launch_bounds__(384, 1) engine_kernel(unsigned long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t dsmem[];  // MMA operands (kMma)
  __shared__ uint32_t tbase;
  __shared__ uint64_t mbar;
  __shared__ volatile uint32_t done;
  __shared__ uint64_t sync_bar[2];  // kSync: the kernel's per-tile s_full wait / p_full arrive
  __shared__ float xchg[2][2][128];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    tmem_alloc<512>(&tbase);
    tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    done = 0;
    mbar_init(&sync_bar[0], 1);  // waited on: completed once below, then always phase 0 done
    mbar_init(&sync_bar[1], 256);
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t quad = warp & 3, row = quad * 32 + lane, lane_off = (quad * 32) << 16;
  // fill both S buffers (columns 0..255) with scores
  if (warp >= 4 && warp < 8) {
#pragma unroll 1
    for (uint32_t c = 0; c < 256; c += 32) {
      uint32_t v[32];
#pragma unroll
      for (uint32_t i = 0; i < 32; ++i) v[i] = __float_as_uint(0.01f * static_cast<float>((row * 7 + c + i) % 97));
      tmem_st32(tmem + lane_off + c, v);
    }
    tmem_st_wait();
  }
  if (threadIdx.x == 0) mbar_arrive(&sync_bar[0]);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint64_t sl2x2 = f2_pack(0.18f, 0.18f);
  float l = 0.0f, m_run = 0.0f;
  long long t0 = clock64();
  if (kMma && warp == 1 && lane == 0) {
    // a tensor-core stream beside the engine: 128x128x16 SS MMAs into TMEM columns 384..511
    const uint32_t a = smem_u32(dsmem), b = a + 32768;
    constexpr uint32_t idesc = make_idesc_bf16(128, 128, false, false);
    uint32_t ph = 0;
    while (!done) {
#pragma unroll
      for (uint32_t kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
        umma_ss(tmem + 384, make_sdesc_sw128(a + off, 16, 1024), make_sdesc_sw128(b + off, 16, 1024), idesc, kk > 0);
      }
      tc_commit(&mbar);
      mbar_wait(&mbar, ph);
      ph ^= 1;
    }
  }
  if (warp >= 4) {
    if (LAYOUT == 0) {
      const uint32_t half = (warp - 4) >> 2;
#pragma unroll 1
      for (uint32_t k = 0; k < kTiles; ++k) {
        const uint32_t ts = tmem + lane_off + (k & 1) * 128;
        if (kSync) {
          mbar_wait(&sync_bar[0], 0);  // already complete, as a ready s_full
          tc_fence_after();
        }
        uint32_t a0[32], a1[32];
        tmem_ld32(ts + half * 64, a0);
        tmem_ld32(ts + half * 64 + 32, a1);
        tmem_ld_wait();
        float pm = fmaxf(max32(a0), max32(a1));
        xchg[k & 1][half][row] = pm;
        named_bar_sync(1, 256);
        pm = fmaxf(pm, xchg[k & 1][half ^ 1][row]);
        m_run = fmaxf(m_run, pm * 0.18f);
        const uint64_t nm2 = f2_pack(-m_run, -m_run);
        uint32_t pk[16];
        uint64_t lacc = 0;
        exp_chunk(a0, sl2x2, nm2, pk, lacc);
        tmem_st16(ts + 256 + half * 32, pk);  // P to scratch columns (S stays intact)
        exp_chunk(a1, sl2x2, nm2, pk, lacc);
        tmem_st16(ts + 256 + half * 32 + 16, pk);
        l += f2_lo(lacc) + f2_hi(lacc);
        tmem_st_wait();
        if (kSync) {
          tc_fence_before();
          mbar_arrive(&sync_bar[1]);  // as p_full (nobody waits)
        }
      }
    } else {
      const uint32_t stream = (warp - 4) >> 2;  // S buffer of this stream
#pragma unroll 1
      for (uint32_t k = 0; k < kTiles / 2; ++k) {
        const uint32_t ts = tmem + lane_off + stream * 128;
        float pm = -INFINITY;
#pragma unroll
        for (uint32_t c = 0; c < 128; c += 64) {  // pass 1: row max
          uint32_t a0[32], a1[32];
          tmem_ld32(ts + c, a0);
          tmem_ld32(ts + c + 32, a1);
          tmem_ld_wait();
          pm = fmaxf(pm, fmaxf(max32(a0), max32(a1)));
        }
        m_run = fmaxf(m_run, pm * 0.18f);
        const uint64_t nm2 = f2_pack(-m_run, -m_run);
        uint64_t lacc = 0;
#pragma unroll
        for (uint32_t c = 0; c < 128; c += 64) {  // pass 2: exponentials, P
          uint32_t a0[32], a1[32];
          tmem_ld32(ts + c, a0);
          tmem_ld32(ts + c + 32, a1);
          tmem_ld_wait();
          uint32_t pk[16];
          exp_chunk(a0, sl2x2, nm2, pk, lacc);
          tmem_st16(tmem + lane_off + 256 + stream * 64 + c / 2, pk);
          exp_chunk(a1, sl2x2, nm2, pk, lacc);
          tmem_st16(tmem + lane_off + 256 + stream * 64 + c / 2 + 16, pk);
        }
        l += f2_lo(lacc) + f2_hi(lacc);
        tmem_st_wait();
      }
    }
  }
  long long t1 = clock64();
  if (warp >= 4) {
    named_bar_sync(2, 256);
    if (threadIdx.x == 128) done = 1;
  }
  __syncthreads();
  if (warp >= 4) sink[blockIdx.x * 256 + threadIdx.x - 128] = l + m_run;
  if (threadIdx.x == 128) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int LAYOUT, bool kMma, bool kSync = false>
void run(const char* name, int sms) {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, sms * 8);
  cudaMalloc(&sink, sms * 256 * 4);
  cudaFuncSetAttribute(engine_kernel<LAYOUT, kMma, kSync>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  engine_kernel<LAYOUT, kMma, kSync><<<sms, 384, 66 * 1024>>>(d, sink);
  engine_kernel<LAYOUT, kMma, kSync><<<sms, 384, 66 * 1024>>>(d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  std::printf("%-58s %7.0f cycles per 128x128 tile %s\n", name, avg / kTiles, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0, false>("A halves: 2 warps per row, max exchange + barrier per tile", sms);
  run<1, false>("B rows: 1 thread per row, 2 free-running streams", sms);
  run<0, true>("A halves + a concurrent 128x128x16 MMA stream", sms);
  run<1, true>("B rows + a concurrent 128x128x16 MMA stream", sms);
  run<0, true, true>("A halves + MMA stream + per-tile mbarrier wait/arrive, fences", sms);
  return 0;
}
