// mma_issue_probe.cu — tcgen05.mma issue cost by issue style (measurement tool).
//   A: one thread (lane 0 of warp 0, a divergent branch) issues every MMA
//   B: the whole warp runs the loop; the MMA asm elects one lane itself (elect.sync inside)
//   C: the whole warp computes descriptors; an elect.sync'ed branch wraps each MMA
//   D: two issuing threads (lane 0 of warps 0 and 1), 16 MMAs each into separate accumulators
// For N = 128 and N = 64 (128xNx16 bf16, SS): cycles to issue 32 MMAs back to back, and to
// completion.
#include <cstdio>

#include "../paper_2409_15097_b200/csrc/bbm_ptx.cuh"

using namespace bbm::ptx;

__device__ __forceinline__ void umma_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int N, int STYLE>
__global__ void __launch_bounds__(128, 1) issue_kernel(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
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
  constexpr uint32_t idesc = make_idesc_bf16(128, N, false, false);
  const uint32_t a = smem_u32(smem), b = a + 32768;
  constexpr int kMmas = 32;
  if (warp == 0) {
    long long t0 = 0, t1 = 0, t2 = 0;
    uint32_t ph = 0;
    for (int rep = 0; rep < 3; ++rep) {
      if (STYLE == 0) {
        if (lane == 0) {
          t0 = clock64();
#pragma unroll
          for (int m = 0; m < kMmas; ++m) {
            const int kk = m % 8;
            const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
            umma_ss(tmem + (m / 8) * 128, make_sdesc_sw128(a + off, 16, 1024), make_sdesc_sw128(b + off, 16, 1024),
                    idesc, kk > 0);
          }
          t1 = clock64();
          tc_commit(&bar);
        }
      } else if (STYLE == 1) {
        t0 = clock64();
#pragma unroll
        for (int m = 0; m < kMmas; ++m) {
          const int kk = m % 8;
          const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
          umma_ss_elect(tmem + (m / 8) * 128, make_sdesc_sw128(a + off, 16, 1024),
                        make_sdesc_sw128(b + off, 16, 1024), idesc, kk > 0);
        }
        t1 = clock64();
        if (elect_one()) tc_commit(&bar);
      } else {
        t0 = clock64();
#pragma unroll
        for (int m = 0; m < kMmas; ++m) {
          const int kk = m % 8;
          const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
          const uint64_t ad = make_sdesc_sw128(a + off, 16, 1024), bd = make_sdesc_sw128(b + off, 16, 1024);
          if (elect_one()) umma_ss(tmem + (m / 8) * 128, ad, bd, idesc, kk > 0);
          __syncwarp();
        }
        t1 = clock64();
        if (elect_one()) tc_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, ph);
      ph ^= 1;
      t2 = clock64();
    }
    if (lane == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int N>
__global__ void __launch_bounds__(128, 1) dual_kernel(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
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
  constexpr uint32_t idesc = make_idesc_bf16(128, N, false, false);
  const uint32_t a = smem_u32(smem), b = a + 32768;
  long long t0 = 0, t2 = 0;
  uint32_t ph = 0;
  for (int rep = 0; rep < 3; ++rep) {
    __syncthreads();
    if (warp < 2 && lane == 0) {
      t0 = clock64();
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const int kk = m % 8;
        const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
        umma_ss(tmem + warp * 256 + (m / 8) * 128, make_sdesc_sw128(a + off, 16, 1024),
                make_sdesc_sw128(b + off, 16, 1024), idesc, kk > 0);
      }
      tc_commit(&bar[warp]);
      mbar_wait(&bar[warp], ph);
      t2 = clock64();
    }
    ph ^= 1;
  }
  if (warp < 2 && lane == 0) {
    out[warp * 2] = t0;
    out[warp * 2 + 1] = t2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int N>
void run_dual() {
  unsigned long long* d;
  cudaMalloc(&d, 32);
  cudaMemset(d, 0, 32);
  cudaFuncSetAttribute(dual_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  dual_kernel<N><<<1, 128, 66 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[4] = {0, 0, 0, 0};
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  const unsigned long long start = h[0] < h[2] ? h[0] : h[2], end = h[1] > h[3] ? h[1] : h[3];
  std::printf("%-34s N=%3d: 2 x 16 MMAs complete after %6llu cycles (pipe ideal %d) %s\n",
              "D two issuing threads", N, end - start, 32 * N / 2, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

template <int N, int STYLE>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  cudaFuncSetAttribute(issue_kernel<N, STYLE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  issue_kernel<N, STYLE><<<1, 128, 66 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2] = {0, 0};
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  std::printf("%-34s N=%3d: 32 MMAs issued in %6llu cycles (%5.1f / MMA), complete after %6llu (pipe ideal %d) %s\n",
              name, N, h[0], h[0] / 32.0, h[1], 32 * N / 2, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<128, 0>("A one thread (divergent)");
  run<128, 1>("B warp, elect inside the MMA asm");
  run<128, 2>("C warp, elected branch per MMA");
  run<64, 0>("A one thread (divergent)");
  run<64, 1>("B warp, elect inside the MMA asm");
  run<64, 2>("C warp, elected branch per MMA");
  run_dual<128>();
  run_dual<64>();
  return 0;
}
