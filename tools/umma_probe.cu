// umma_probe.cu — hardware check of the descriptor encodings the attention kernel relies on.
//
// One CTA, D in {64,128}:
//   S[128x128] = A[128xD] * B[128xD]^T      (SS MMA, both K-major, 128B swizzle, TMA loaded)
//   O[128xD]   = P[128x128] * V[128xD]      (TS MMA, P written to TMEM by tcgen05.st,
//                                            V is MN-major 128B swizzle)
// Results are read back with tcgen05.ld and compared on the host with an fp64 reference.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../paper_2409_15097_b200/csrc
#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bbm_ptx.cuh"
#include "bbm_tmap.h"

using namespace bbm::ptx;

template <int D>
__global__ void __launch_bounds__(128, 1)
    probe_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                 const __grid_constant__ CUtensorMap tm_v, const __nv_bfloat16* p_in, float* s_out,
                 float* o_out) {
  constexpr int kBox = 128 * 64 * 2;  // one 64-wide box of 128 rows
  constexpr int kBoxes = D / 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = sa + kBoxes * kBox;
  uint8_t* sv = sb + kBoxes * kBox;
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc<512>(&tmem_base_sh);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar_load, 3 * kBoxes * kBox);
    uint64_t pol = policy_evict_first();
    for (int b = 0; b < kBoxes; ++b) {
      tma_load_3d(sa + b * kBox, &tm_a, &bar_load, b * 64, 0, 0, pol);
      tma_load_3d(sb + b * kBox, &tm_b, &bar_load, b * 64, 0, 0, pol);
      tma_load_3d(sv + b * kBox, &tm_v, &bar_load, b * 64, 0, 0, pol);
    }
  }
  // P -> TMEM columns [D_OFF, D_OFF+64) as packed bf16x2 (row = lane).
  constexpr uint32_t kPCol = 256;
  {
    const int row = threadIdx.x;
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    for (int c = 0; c < 2; ++c) {
      uint32_t r[32];
      for (int i = 0; i < 32; ++i) {
        const __nv_bfloat16* src = p_in + row * 128 + (c * 32 + i) * 2;
        r[i] = static_cast<uint32_t>(__bfloat16_as_ushort(src[0])) |
               (static_cast<uint32_t>(__bfloat16_as_ushort(src[1])) << 16);
      }
      tmem_st32(lane_addr + kPCol + c * 32, r);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (threadIdx.x == 0) {
    mbar_wait(&bar_load, 0);
    tc_fence_after();
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
    for (int kk = 0; kk < D / 16; ++kk) {
      const uint32_t off = (kk / 4) * kBox + (kk % 4) * 32;
      uint64_t da = make_sdesc_sw128(smem_u32(sa) + off, 16, 1024);
      uint64_t db = make_sdesc_sw128(smem_u32(sb) + off, 16, 1024);
      umma_ss(tmem + 0, da, db, idesc_s, kk > 0);
    }
    constexpr uint32_t idesc_o = make_idesc_bf16(128, D, false, true);
    for (int kk = 0; kk < 128 / 16; ++kk) {
      uint64_t dv = make_sdesc_sw128(smem_u32(sv) + kk * 2048, kBox, 1024);
      umma_ts(tmem + 128, tmem + kPCol + kk * 8, dv, idesc_o, kk > 0);
    }
    tc_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  {
    const int row = threadIdx.x;
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      tmem_ld32(lane_addr + c * 32, r);
      tmem_ld_wait();
      for (int i = 0; i < 32; ++i) s_out[row * 128 + c * 32 + i] = __uint_as_float(r[i]);
    }
    for (int c = 0; c < D / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(lane_addr + 128 + c * 32, r);
      tmem_ld_wait();
      for (int i = 0; i < 32; ++i) o_out[row * D + c * 32 + i] = __uint_as_float(r[i]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(2);                                                                   \
    }                                                                                 \
  } while (0)

template <int D>
int run() {
  std::vector<__nv_bfloat16> a(128 * D), b(128 * D), v(128 * D), p(128 * 128);
  std::vector<float> af(128 * D), bf(128 * D), vf(128 * D), pf(128 * 128);
  uint64_t s = 12345;
  auto rnd = [&]() {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return static_cast<float>((s >> 40) & 0xFFFF) / 65536.0f - 0.5f;
  };
  for (int i = 0; i < 128 * D; ++i) {
    a[i] = __float2bfloat16(rnd()); af[i] = __bfloat162float(a[i]);
    b[i] = __float2bfloat16(rnd()); bf[i] = __bfloat162float(b[i]);
    v[i] = __float2bfloat16(rnd()); vf[i] = __bfloat162float(v[i]);
  }
  for (int i = 0; i < 128 * 128; ++i) { p[i] = __float2bfloat16(rnd()); pf[i] = __bfloat162float(p[i]); }
  __nv_bfloat16 *da, *db, *dv, *dp;
  float *ds, *dout;
  CK(cudaMalloc(&da, a.size() * 2)); CK(cudaMalloc(&db, b.size() * 2));
  CK(cudaMalloc(&dv, v.size() * 2)); CK(cudaMalloc(&dp, p.size() * 2));
  CK(cudaMalloc(&ds, 128 * 128 * 4)); CK(cudaMalloc(&dout, 128 * D * 4));
  CK(cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, v.data(), v.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dp, p.data(), p.size() * 2, cudaMemcpyHostToDevice));
  CUtensorMap ta = bbm::make_tmap_bf16_3d(da, D, 128, 1, 64, 128);
  CUtensorMap tb = bbm::make_tmap_bf16_3d(db, D, 128, 1, 64, 128);
  CUtensorMap tv = bbm::make_tmap_bf16_3d(dv, D, 128, 1, 64, 128);
  const int smem = 3 * (D / 64) * 128 * 64 * 2 + 1024;
  CK(cudaFuncSetAttribute(probe_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe_kernel<D><<<1, 128, smem>>>(ta, tb, tv, dp, ds, dout);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> hs(128 * 128), ho(128 * D);
  CK(cudaMemcpy(hs.data(), ds, hs.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ho.data(), dout, ho.size() * 4, cudaMemcpyDeviceToHost));
  double es = 0, eo = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j) {
      double acc = 0;
      for (int c = 0; c < D; ++c) acc += double(af[i * D + c]) * bf[j * D + c];
      es = std::fmax(es, std::fabs(acc - hs[i * 128 + j]));
    }
  for (int i = 0; i < 128; ++i)
    for (int c = 0; c < D; ++c) {
      double acc = 0;
      for (int j = 0; j < 128; ++j) acc += double(pf[i * 128 + j]) * vf[j * D + c];
      eo = std::fmax(eo, std::fabs(acc - ho[i * D + c]));
    }
  std::printf("D=%d  S max err %.3e  O max err %.3e  S[0][0]=%f O[0][0]=%f\n", D, es, eo, hs[0], ho[0]);
  return (es < 1e-3 && eo < 1e-3) ? 0 : 1;
}

int main() {
  int bad = run<64>();
  bad |= run<128>();
  std::printf(bad ? "PROBE FAIL\n" : "PROBE OK\n");
  return bad;
}
