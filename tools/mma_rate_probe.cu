// mma_rate_probe.cu — achievable tcgen05.mma rate on this part, per mode (measurement tool).
//
// 148 CTAs (one per SM), one thread issues `iters` groups of 8 MMAs (K = 8 x 16 = 128) with
// M=128, N in {128, 256}: SS (A and B from shared memory) or TS (A from TMEM); clock64 around
// the loop after a commit/wait. Prints cycles per 128x128x16 MMA-equivalent (ideal: 64).
#include <cstdio>
#include <cstdlib>

#include "../paper_2409_15097_b200/csrc/bbm_ptx.cuh"

using namespace bbm::ptx;

template <int MODE, int N, bool kTma, int kLdWarps = 0, int kMufu = 0>  // MODE 0 = SS, 1 = TS
__global__ void __launch_bounds__(384, 1) rate_kernel(int iters, unsigned long long* out,
                                                      const uint8_t* gsrc, volatile int* stop) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, tbar;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&tbar, 1);
    done = 0;
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc<512>(&tbase);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = a + 32768;
    constexpr uint32_t idesc = make_idesc_bf16(128, N, false, false);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
        if (MODE == 0)
          umma_ss(tmem, make_sdesc_sw128(a + off, 16, 1024), make_sdesc_sw128(b + off, 16, 1024),
                  idesc, kk > 0 || it > 0);
        else
          umma_ts(tmem, tmem + 256 + kk * 8, make_sdesc_sw128(b + off, 16, 1024), idesc,
                  kk > 0 || it > 0);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = static_cast<unsigned long long>(t1 - t0);
    done = 1;
  }
  if (kTma && threadIdx.x == 32) {
    // 32 KB bulk copies global -> shared (region [128K, 160K)) back to back, ~1 in flight
    uint32_t ph = 0;
    const uint32_t dst = smem_u32(smem) + 131072;
    uint64_t n = 0;
    while (!done) {
      mbar_arrive_expect_tx(&tbar, 32768);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(dst), "l"(gsrc + (n++ % 64) * 32768), "r"(32768), "r"(smem_u32(&tbar)) : "memory");
      mbar_wait(&tbar, ph);
      ph ^= 1;
    }
    if (blockIdx.x == 0) out[1] = n;
  }
  if (kMufu == 2 && warp >= 4) {
    // issue-slot hogs: independent FFMA2 chains (no TMEM, no MUFU), like a busy softmax engine
    uint64_t a = 0x3f8000003f800000ull, b = a, c = a, d = a;
    const uint64_t m = 0x3f7ff0003f7ff000ull;
    uint64_t passes = 0;
    while (!done) {
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(a) : "l"(m));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(b) : "l"(m));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(c) : "l"(m));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(d) : "l"(m));
      }
      ++passes;
    }
    if (blockIdx.x == 0 && threadIdx.x == 128) out[1] = passes + (a ^ b ^ c ^ d) % 2;
  }
  if (kLdWarps > 0 && warp >= 4 && warp < 4 + kLdWarps) {
    // TMEM readers like the softmax engine: 64 columns of the second S buffer per pass, plus a
    // 16-column store back, in a loop until the MMA thread is done
    const uint32_t lane_off = ((warp & 3) * 32) << 16;
    const uint32_t half = (warp >= 8) ? 1 : 0;
    uint64_t passes = 0;
    while (!done) {
      uint32_t a0[32], a1[32];
      tmem_ld32(tmem + 384 + lane_off + half * 64, a0);
      tmem_ld32(tmem + 384 + lane_off + half * 64 + 32, a1);
      tmem_ld_wait();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = a0[2 * i] ^ a1[2 * i + 1];
      if (kMufu) {  // the softmax engine's exp2 load on the XU pipe
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float x = __uint_as_float(a0[i] & 0x3fffffffu), y = __uint_as_float(a1[i] & 0x3fffffffu);
          asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x));
          asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(y));
          pk[i / 2] ^= __float_as_uint(x) ^ __float_as_uint(y);
        }
      }
      tmem_st16(tmem + 384 + lane_off + half * 32, pk);
      tmem_st_wait();
      ++passes;
    }
    if (blockIdx.x == 0 && threadIdx.x == 128) out[1] = passes;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int MODE, int N, bool kTma, int kLdWarps = 0, int kMufu = 0>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  uint8_t* g;
  cudaMalloc(&g, 64 * 32768);
  const int smem = 2 * 65536 + 32768 + 1024;
  cudaFuncSetAttribute(rate_kernel<MODE, N, kTma, kLdWarps, kMufu>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  rate_kernel<MODE, N, kTma, kLdWarps, kMufu><<<148, 384, smem>>>(iters, d, g, nullptr);
  rate_kernel<MODE, N, kTma, kLdWarps, kMufu><<<148, 384, smem>>>(iters, d, g, nullptr);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long res[2] = {0, 0};
  cudaMemcpy(res, d, 16, cudaMemcpyDeviceToHost);
  const double per = double(res[0]) / (iters * 8.0 * (N / 128.0));
  std::printf("%-12s N=%3d tma=%d: %s  %.1f cycles per 128x128x16 (ideal 64); side count %llu (%.1f B/cycle if bulk)\n",
              name, N, int(kTma), e == cudaSuccess ? "ok" : cudaGetErrorString(e), per, res[1],
              res[1] * 32768.0 / double(res[0]));
  cudaFree(d);
  cudaFree(g);
}

int main() {
  run<0, 128, false>("SS");
  run<1, 128, false>("TS");
  run<0, 128, true>("SS+bulk");
  run<0, 128, false, 4>("SS+4ldwarps");
  run<0, 128, false, 8>("SS+8ldwarps");
  run<1, 128, false, 8>("TS+8ldwarps");
  run<0, 128, false, 8, 1>("SS+8ld+mufu");
  run<1, 128, false, 8, 1>("TS+8ld+mufu");
  run<0, 128, false, 0, 2>("SS+8fma-hogs");
  run<1, 128, false, 0, 2>("TS+8fma-hogs");
  return 0;
}
