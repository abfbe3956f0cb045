// host_io.cu — the host-buffer forward path (the reference-facing call: its callers hold Q/K/V in
// host memory, engine.hpp:282-285) as a copy/compute pipeline.
//
// The slots are cut into chunks; on three streams of the prep's device, chunk c's H2D, the
// attention kernel on chunk c-1 and the D2H of chunk c-2 run concurrently (H2D and D2H use the
// two PCIe directions). Device buffers persist in the prep and only grow, so a steady-state call
// allocates nothing. With pinned host buffers the call costs about max(H2D, D2H) bytes over PCIe
// plus one chunk of kernel time, instead of H2D + kernel + D2H.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "bbm_internal.h"

namespace bbm {

HostPipe::~HostPipe() {
  for (cudaEvent_t e : ev_in) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_out) cudaEventDestroy(e);
  if (h2d) cudaStreamDestroy(h2d);
  if (comp) cudaStreamDestroy(comp);
  if (d2h) cudaStreamDestroy(d2h);
  cudaFree(buf);
}

namespace {

constexpr uint32_t kMaxChunks = 16;
constexpr uint64_t kChunkBytes = 16ull << 20;  // aim for >= 16 MB of inputs per chunk

HostPipe& pipe_of(const Prep& prep) {
  if (!prep.pipe) {
    auto* p = new HostPipe;
    try {
      BBM_CUDA(cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking));
      BBM_CUDA(cudaStreamCreateWithFlags(&p->comp, cudaStreamNonBlocking));
      BBM_CUDA(cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking));
      p->ev_in.resize(kMaxChunks);
      p->ev_out.resize(kMaxChunks);
      for (uint32_t c = 0; c < kMaxChunks; ++c) {
        BBM_CUDA(cudaEventCreateWithFlags(&p->ev_in[c], cudaEventDisableTiming));
        BBM_CUDA(cudaEventCreateWithFlags(&p->ev_out[c], cudaEventDisableTiming));
      }
    } catch (...) {
      delete p;
      throw;
    }
    prep.pipe = p;
  }
  return *prep.pipe;
}

uint8_t* reserve(HostPipe& p, size_t bytes) {
  if (bytes > p.cap) {
    BBM_CUDA(cudaStreamSynchronize(p.comp));
    cudaFree(p.buf);
    p.buf = nullptr;
    p.cap = 0;
    BBM_CUDA(cudaMalloc(&p.buf, bytes));
    p.cap = bytes;
  }
  return p.buf;
}

// dst[s][fwd[a]] = src[s][a]: scatter per-row statistics back to the original token order
__global__ void scatter_rows_f32_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                        const uint32_t* __restrict__ fwd, uint64_t slots, uint64_t n) {
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < slots * n;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t sl = t / n, a = t % n;
    dst[sl * n + fwd[a]] = src[t];
  }
}

}  // namespace

void run_fwd_host_pipelined(const Prep& prep, int variant, const uint16_t* q, const uint16_t* k,
                            const uint16_t* v, uint16_t* out, float* row_max, float* row_sum,
                            uint64_t slots, uint32_t d, float scale, int num_sms, double* span_ms) {
  HostPipe& p = pipe_of(prep);
  const uint64_t n = prep.n, per = n * d, tbytes = slots * per * 2, sbytes = slots * n * 4;
  uint8_t* base = reserve(p, 4 * tbytes + 2 * sbytes);
  uint16_t* dq = reinterpret_cast<uint16_t*>(base);
  uint16_t* dk = dq + slots * per;
  uint16_t* dv = dk + slots * per;
  uint16_t* dout = dv + slots * per;
  float* dmax = reinterpret_cast<float*>(dout + slots * per);
  float* dsum = dmax + slots * n;
  const uint64_t chunks =
      std::max<uint64_t>(1, std::min<uint64_t>({slots, kMaxChunks, (3 * tbytes) / kChunkBytes}));
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (span_ms) {
    BBM_CUDA(cudaEventCreate(&t0));
    BBM_CUDA(cudaEventCreate(&t1));
    BBM_CUDA(cudaEventRecord(t0, p.h2d));
  }
  for (uint64_t c = 0; c < chunks; ++c) {
    const uint64_t s0 = slots * c / chunks, s1 = slots * (c + 1) / chunks, ns = s1 - s0;
    const uint64_t off = s0 * per, bytes = ns * per * 2;
    BBM_CUDA(cudaMemcpyAsync(dq + off, q + off, bytes, cudaMemcpyHostToDevice, p.h2d));
    BBM_CUDA(cudaMemcpyAsync(dk + off, k + off, bytes, cudaMemcpyHostToDevice, p.h2d));
    BBM_CUDA(cudaMemcpyAsync(dv + off, v + off, bytes, cudaMemcpyHostToDevice, p.h2d));
    BBM_CUDA(cudaEventRecord(p.ev_in[c], p.h2d));
    BBM_CUDA(cudaStreamWaitEvent(p.comp, p.ev_in[c], 0));
    AttnArgs a{dq + off, dk + off, dv + off, dout + off, row_max ? dmax + s0 * n : nullptr,
               row_sum ? dsum + s0 * n : nullptr, ns, n, d, scale, variant};
    launch_attn_fwd(prep, a, p.comp, num_sms);
    BBM_CUDA(cudaEventRecord(p.ev_out[c], p.comp));
    BBM_CUDA(cudaStreamWaitEvent(p.d2h, p.ev_out[c], 0));
    BBM_CUDA(cudaMemcpyAsync(out + off, dout + off, bytes, cudaMemcpyDeviceToHost, p.d2h));
    if (row_max)
      BBM_CUDA(cudaMemcpyAsync(row_max + s0 * n, dmax + s0 * n, ns * n * 4, cudaMemcpyDeviceToHost, p.d2h));
    if (row_sum)
      BBM_CUDA(cudaMemcpyAsync(row_sum + s0 * n, dsum + s0 * n, ns * n * 4, cudaMemcpyDeviceToHost, p.d2h));
  }
  if (span_ms) BBM_CUDA(cudaEventRecord(t1, p.d2h));
  BBM_CUDA(cudaStreamSynchronize(p.d2h));
  if (span_ms) {
    float ms = 0.0f;
    BBM_CUDA(cudaEventElapsedTime(&ms, t0, t1));
    *span_ms = ms;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
}


// The RCM path end to end (reorder.hpp:156-189 + bench.hpp:448-467): the caller's Q/K/V are in
// the ORIGINAL token order, `prep` was built from permute_mask(mask, perm), forward = perm's
// new -> old map. Per slot chunk, on the prep's device: H2D, gather Q/K/V rows into the
// reordered layout (permute_rows), attention on the reordered mask, scatter O and the row
// statistics back (unpermute_rows), D2H — the permutation passes hide under the PCIe copies.
void run_fwd_host_rcm(const Prep& prep, int variant, const uint32_t* forward, const uint16_t* q,
                      const uint16_t* k, const uint16_t* v, uint16_t* out, float* row_max,
                      float* row_sum, uint64_t slots, uint32_t d, float scale, int num_sms,
                      double* span_ms) {
  HostPipe& p = pipe_of(prep);
  const uint64_t n = prep.n, per = n * d, tbytes = slots * per * 2, sbytes = slots * n * 4;
  uint8_t* base = reserve(p, 7 * tbytes + 4 * sbytes + n * 4 + 256);
  uint16_t* raw[3] = {reinterpret_cast<uint16_t*>(base), nullptr, nullptr};
  raw[1] = raw[0] + slots * per;
  raw[2] = raw[1] + slots * per;
  uint16_t* prm[4] = {raw[2] + slots * per, nullptr, nullptr, nullptr};  // q' k' v' o'
  for (int t = 1; t < 4; ++t) prm[t] = prm[t - 1] + slots * per;
  float* pmax = reinterpret_cast<float*>(prm[3] + slots * per);
  float* psum = pmax + slots * n;
  float* omax = psum + slots * n;
  float* osum = omax + slots * n;
  uint32_t* dfwd = reinterpret_cast<uint32_t*>(osum + slots * n);
  BBM_CUDA(cudaMemcpyAsync(dfwd, forward, n * 4, cudaMemcpyHostToDevice, p.comp));
  const uint64_t chunks =
      std::max<uint64_t>(1, std::min<uint64_t>({slots, kMaxChunks, (3 * tbytes) / kChunkBytes}));
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (span_ms) {
    BBM_CUDA(cudaEventCreate(&t0));
    BBM_CUDA(cudaEventCreate(&t1));
    BBM_CUDA(cudaEventRecord(t0, p.h2d));
  }
  const uint16_t* src[3] = {q, k, v};
  for (uint64_t c = 0; c < chunks; ++c) {
    const uint64_t s0 = slots * c / chunks, s1 = slots * (c + 1) / chunks, ns = s1 - s0;
    const uint64_t off = s0 * per, bytes = ns * per * 2;
    for (int t = 0; t < 3; ++t)
      BBM_CUDA(cudaMemcpyAsync(raw[t] + off, src[t] + off, bytes, cudaMemcpyHostToDevice, p.h2d));
    BBM_CUDA(cudaEventRecord(p.ev_in[c], p.h2d));
    BBM_CUDA(cudaStreamWaitEvent(p.comp, p.ev_in[c], 0));
    for (int t = 0; t < 3; ++t)  // X'[a] = X[forward[a]]
      launch_permute_rows(raw[t] + off, prm[t] + off, dfwd, ns, n, static_cast<uint64_t>(d) * 2, false, p.comp);
    AttnArgs a{prm[0] + off, prm[1] + off, prm[2] + off, prm[3] + off, row_max ? pmax + s0 * n : nullptr,
               row_sum ? psum + s0 * n : nullptr, ns, n, d, scale, variant};
    launch_attn_fwd(prep, a, p.comp, num_sms);
    // O[forward[a]] = O'[a], into the (consumed) raw Q chunk
    launch_permute_rows(prm[3] + off, raw[0] + off, dfwd, ns, n, static_cast<uint64_t>(d) * 2, true, p.comp);
    const unsigned g = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((ns * n + 255) / 256, 148ull * 8)));
    if (row_max) scatter_rows_f32_kernel<<<g, 256, 0, p.comp>>>(pmax + s0 * n, omax + s0 * n, dfwd, ns, n);
    if (row_sum) scatter_rows_f32_kernel<<<g, 256, 0, p.comp>>>(psum + s0 * n, osum + s0 * n, dfwd, ns, n);
    BBM_CUDA(cudaGetLastError());
    BBM_CUDA(cudaEventRecord(p.ev_out[c], p.comp));
    BBM_CUDA(cudaStreamWaitEvent(p.d2h, p.ev_out[c], 0));
    BBM_CUDA(cudaMemcpyAsync(out + off, raw[0] + off, bytes, cudaMemcpyDeviceToHost, p.d2h));
    if (row_max)
      BBM_CUDA(cudaMemcpyAsync(row_max + s0 * n, omax + s0 * n, ns * n * 4, cudaMemcpyDeviceToHost, p.d2h));
    if (row_sum)
      BBM_CUDA(cudaMemcpyAsync(row_sum + s0 * n, osum + s0 * n, ns * n * 4, cudaMemcpyDeviceToHost, p.d2h));
  }
  if (span_ms) BBM_CUDA(cudaEventRecord(t1, p.d2h));
  BBM_CUDA(cudaStreamSynchronize(p.d2h));
  if (span_ms) {
    float ms = 0.0f;
    BBM_CUDA(cudaEventElapsedTime(&ms, t0, t1));
    *span_ms = ms;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
}

}  // namespace bbm
