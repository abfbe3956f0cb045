// mma_chain_probe.cu — the attention kernel's MMA pattern in isolation (measurement tool):
// per tile k: S_k = Q K^T (SS, N=128) into TMEM buffer k%2, then PV_k (TS, A = columns [0,64) of
// buffer k%2, N=128) into O; issue order S_0, S_1, PV_0, S_2, PV_1, ...  `alias` = 0 points the
// PV A operand at a third, never-written region instead (no read-after-write / write-after-read
// between the S and PV MMAs). Prints cycles per tile (ideal 1024 = 16 x 64).
#include <cstdio>

#include "../paper_2409_15097_b200/csrc/bbm_ptx.cuh"

using namespace bbm::ptx;

__global__ void __launch_bounds__(128, 1) chain_kernel(int tiles, int alias, int commit_each,
                                                       unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, cbar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&cbar, 1);
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
    const uint32_t q = smem_u32(smem), k = q + 32768, v = k + 32768;
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
    constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, false, true);
    auto S = [&](int t) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
        umma_ss(tmem + (t & 1) * 128, make_sdesc_sw128(q + off, 16, 1024),
                make_sdesc_sw128(k + off, 16, 1024), idesc_s, kk > 0);
      }
      if (commit_each) tc_commit(&cbar);
    };
    auto PV = [&](int t) {
      const uint32_t a = alias ? tmem + (t & 1) * 128 : tmem + 384;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_ts(tmem + 256, a + kk * 8, make_sdesc_sw128(v + kk * 2048, 16384, 1024), idesc_o,
                t > 0 || kk > 0);
      if (commit_each) tc_commit(&cbar);
    };
    long long t0 = clock64();
    S(0);
    S(1);
    for (int t = 0; t < tiles; ++t) {
      PV(t);
      if (t + 2 < tiles) S(t + 2);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int smem = 3 * 32768 + 1024;
  cudaFuncSetAttribute(chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tiles = 500;
  for (int alias = 0; alias < 2; ++alias)
    for (int ce = 0; ce < 2; ++ce) {
      chain_kernel<<<148, 128, smem>>>(tiles, alias, ce, d);
      chain_kernel<<<148, 128, smem>>>(tiles, alias, ce, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long c = 0;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      std::printf("alias=%d commit_each=%d: %s %.0f cycles per tile (ideal 1024)\n", alias, ce,
                  e == cudaSuccess ? "ok" : cudaGetErrorString(e), double(c) / tiles);
    }
  return 0;
}
