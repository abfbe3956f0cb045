// mma_latency_probe.cu — issue cost vs completion latency of one group of 8 tcgen05.mma
// (128x128x16 each, SS) from an idle pipe, and of two groups back to back (measurement tool).
#include <cstdio>

#include "../paper_2409_15097_b200/csrc/bbm_ptx.cuh"

using namespace bbm::ptx;

__global__ void __launch_bounds__(128, 1) lat_kernel(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
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
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = a + 32768;
    constexpr uint32_t idesc = make_idesc_bf16(128, 128, false, false);
    uint32_t ph = 0;
    for (int groups = 1; groups <= 4; groups *= 2) {
      for (int rep = 0; rep < 3; ++rep) {
        long long t0 = clock64();
        for (int g = 0; g < groups; ++g)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
            umma_ss(tmem + g * 128, make_sdesc_sw128(a + off, 16, 1024),
                    make_sdesc_sw128(b + off, 16, 1024), idesc, kk > 0);
          }
        long long t1 = clock64();
        tc_commit(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
        long long t2 = clock64();
        if (blockIdx.x == 0 && rep == 2) {
          out[groups * 2] = t1 - t0;
          out[groups * 2 + 1] = t2 - t0;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16 * 8);
  cudaMemset(d, 0, 128);
  cudaFuncSetAttribute(lat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  lat_kernel<<<1, 128, 66 * 1024>>>(d);
  cudaDeviceSynchronize();
  unsigned long long h[16];
  cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  for (int g = 1; g <= 4; g *= 2)
    std::printf("%d group(s) of 8 MMAs: issue %llu cycles, issue->complete %llu cycles (ideal exec %d)\n",
                g, h[g * 2], h[g * 2 + 1], 512 * g);
  return 0;
}
