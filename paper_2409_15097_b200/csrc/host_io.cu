// host_io.cu — the host-buffer forward path (the reference-facing call: its callers hold Q/K/V in
// host memory, engine.hpp:282-285) as a copy/compute pipeline.
//
// The slots are cut into chunks; on three streams of the prep's device, chunk c's H2D, the
// attention kernel on chunk c-1 and the D2H of chunk c-2 run concurrently (H2D and D2H use the
// two PCIe directions). Device buffers persist in the prep and only grow, so a steady-state call
// allocates nothing. With pinned host buffers the call costs about max(H2D, D2H) bytes over PCIe
// plus one chunk of kernel time, instead of H2D + kernel + D2H.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include "bbm_internal.h"

namespace bbm {

// Persistent host threads for the float host path's float -> bf16 conversion: run(n, fn) calls
// fn(0..n-1) on the workers and the calling thread and returns when all calls are done.
class HostPool {
 public:
  explicit HostPool(unsigned workers) {
    for (unsigned i = 0; i < workers; ++i) threads_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  void run(uint32_t tasks, std::function<void(uint32_t)> fn) {
    if (tasks == 0) return;
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = std::move(fn);
      next_.store(0);
      done_.store(0);
      tasks_.store(tasks);
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_.load() == tasks_.load(); });
  }

 private:
  void work() {
    for (;;) {
      const uint32_t i = next_.fetch_add(1);
      if (i >= tasks_.load()) return;
      fn_(i);
      if (done_.fetch_add(1) + 1 == tasks_.load()) {
        std::lock_guard<std::mutex> lk(mu_);
        done_cv_.notify_all();
      }
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::function<void(uint32_t)> fn_;
  std::atomic<uint32_t> next_{0}, done_{0}, tasks_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

HostPipe::~HostPipe() {
  delete pool;
  for (cudaEvent_t e : ev_stage)
    if (e) cudaEventDestroy(e);
  if (stage) cudaFreeHost(stage);
  for (cudaEvent_t e : ev_in) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_out) cudaEventDestroy(e);
  if (h2d) cudaStreamDestroy(h2d);
  if (comp) cudaStreamDestroy(comp);
  if (d2h) cudaStreamDestroy(d2h);
  cudaFree(buf);
  cudaFree(bad);
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
      BBM_CUDA(cudaMalloc(&p->bad, 4 * sizeof(int)));
      BBM_CUDA(cudaEventCreateWithFlags(&p->ev_stage[0], cudaEventDisableTiming));
      BBM_CUDA(cudaEventCreateWithFlags(&p->ev_stage[1], cudaEventDisableTiming));
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

// require_finite (engine.hpp:237-242) over bf16 data: exponent bits all ones = inf / NaN
__global__ void check_finite_bf16_kernel(const uint16_t* __restrict__ x, uint64_t count,
                                         int* __restrict__ bad) {
  const uint64_t vecs = count / 8;
  bool any = false;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < vecs;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(x) + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      any |= ((w[j] & 0x7F80u) == 0x7F80u) | ((w[j] & 0x7F800000u) == 0x7F800000u);
  }
  for (uint64_t i = vecs * 8 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    any |= (x[i] & 0x7F80u) == 0x7F80u;
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) *bad = 1;
}

// float -> bf16 (RNE) fused with the finiteness check of the float input
__global__ void f32_to_bf16_check_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                         uint64_t count, int* __restrict__ bad) {
  const uint64_t vecs = count / 4;
  bool any = false;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < vecs;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float4 f = __ldg(reinterpret_cast<const float4*>(in) + i);
    any |= !(isfinite(f.x) && isfinite(f.y) && isfinite(f.z) && isfinite(f.w));
    __nv_bfloat162 lo = __floats2bfloat162_rn(f.x, f.y), hi = __floats2bfloat162_rn(f.z, f.w);
    uint2 w;
    w.x = *reinterpret_cast<uint32_t*>(&lo);
    w.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(out)[i] = w;
  }
  for (uint64_t i = vecs * 4 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    any |= !isfinite(in[i]);
    out[i] = __float2bfloat16_rn(in[i]);
  }
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) *bad = 1;
}

// bf16 O -> float, fp32 row statistics -> double (ForwardResult<float>, engine.hpp:93-99)
__global__ void widen_outputs_kernel(const __nv_bfloat16* __restrict__ o, float* __restrict__ of,
                                     uint64_t o_count, const float* __restrict__ m,
                                     const float* __restrict__ l, double* __restrict__ md,
                                     double* __restrict__ ld, uint64_t rows) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t t0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  for (uint64_t i = t0; i < o_count / 8; i += stride) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(o) + i);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
    float4 a, b;
    a.x = __low2float(h[0]), a.y = __high2float(h[0]), a.z = __low2float(h[1]), a.w = __high2float(h[1]);
    b.x = __low2float(h[2]), b.y = __high2float(h[2]), b.z = __low2float(h[3]), b.w = __high2float(h[3]);
    reinterpret_cast<float4*>(of)[2 * i] = a;
    reinterpret_cast<float4*>(of)[2 * i + 1] = b;
  }
  for (uint64_t i = o_count / 8 * 8 + t0; i < o_count; i += stride) of[i] = __bfloat162float(o[i]);
  for (uint64_t i = t0; i < rows; i += stride) {
    if (md) md[i] = static_cast<double>(m[i]);
    if (ld) ld[i] = static_cast<double>(l[i]);
  }
}

// Row-pitch changes for head dims the kernels do not tile natively (d_k / d_v below 64, between 64
// and 128, or unequal): one thread per destination element, off the hot path.
__global__ void pad_to_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                   uint64_t rows, uint32_t w, uint32_t D, int* __restrict__ bad) {
  bool any = false;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < rows * D;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = i / D;
    const uint32_t c = static_cast<uint32_t>(i - r * D);
    const float x = c < w ? in[r * w + c] : 0.0f;
    any |= !isfinite(x);
    out[i] = __float2bfloat16_rn(x);
  }
  if (bad && __any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) *bad = 1;
}

__global__ void pad_f32_kernel(const float* __restrict__ in, float* __restrict__ out, uint64_t rows,
                               uint32_t w, uint32_t D) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < rows * D;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = i / D;
    const uint32_t c = static_cast<uint32_t>(i - r * D);
    out[i] = c < w ? in[r * w + c] : 0.0f;
  }
}

__global__ void crop_to_f32_kernel(const __nv_bfloat16* __restrict__ in, float* __restrict__ out,
                                   uint64_t rows, uint32_t D, uint32_t w) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < rows * w;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = i / w;
    out[i] = __bfloat162float(in[r * D + (i - r * w)]);
  }
}

// fp32 row statistics -> double
__global__ void widen_stats_kernel(const float* __restrict__ m, const float* __restrict__ l,
                                   double* __restrict__ md, double* __restrict__ ld, uint64_t rows) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < rows;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (md) md[i] = static_cast<double>(m[i]);
    if (ld) ld[i] = static_cast<double>(l[i]);
  }
}

unsigned grid_for_elems(uint64_t count) {
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((count / 8 + 255) / 256, 148ull * 16)));
}

// float -> bf16, round to nearest even (the device kernel's __float2bfloat16_rn on finite values),
// fused with require_finite's test; returns true if any value is inf / NaN. SSE2 (the x86-64
// baseline) with non-temporal stores: the pinned staging is only read again by the copy engine,
// so streaming stores save the read-for-ownership pass over it (host memory bandwidth, shared
// with the PCIe DMA, is what bounds this path).
bool f32_to_bf16_host(const float* in, uint16_t* out, uint64_t count) {
  uint32_t bad = 0;
  uint64_t i = 0;
#if defined(__SSE2__)
  if ((reinterpret_cast<uintptr_t>(out) & 15u) == 0) {
    const __m128i exp_mask = _mm_set1_epi32(0x7F800000);
    const __m128i bias = _mm_set1_epi32(0x7FFF), one = _mm_set1_epi32(1), flip = _mm_set1_epi32(0x8000);
    const __m128i flip16 = _mm_set1_epi16(static_cast<short>(0x8000));
    __m128i badv = _mm_setzero_si128();
    for (; i + 8 <= count; i += 8) {
      const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(in + i));
      const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(in + i + 4));
      badv = _mm_or_si128(badv, _mm_cmpeq_epi32(_mm_and_si128(a, exp_mask), exp_mask));
      badv = _mm_or_si128(badv, _mm_cmpeq_epi32(_mm_and_si128(b, exp_mask), exp_mask));
      // (u + 0x7FFF + ((u >> 16) & 1)) >> 16, shifted into signed 16-bit range for the pack
      const __m128i ra = _mm_sub_epi32(
          _mm_srli_epi32(_mm_add_epi32(_mm_add_epi32(a, bias), _mm_and_si128(_mm_srli_epi32(a, 16), one)), 16), flip);
      const __m128i rb = _mm_sub_epi32(
          _mm_srli_epi32(_mm_add_epi32(_mm_add_epi32(b, bias), _mm_and_si128(_mm_srli_epi32(b, 16), one)), 16), flip);
      _mm_stream_si128(reinterpret_cast<__m128i*>(out + i), _mm_xor_si128(_mm_packs_epi32(ra, rb), flip16));
    }
    _mm_sfence();  // the streamed stores are visible before the copy engine reads the staging
    bad |= static_cast<uint32_t>(_mm_movemask_epi8(badv) != 0);
  }
#endif
  for (; i < count; ++i) {
    uint32_t u;
    std::memcpy(&u, in + i, 4);
    bad |= static_cast<uint32_t>((u & 0x7F800000u) == 0x7F800000u);
    out[i] = static_cast<uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
  }
  return bad != 0;
}

// Fraction of a chunk's slots the float path converts on the host. Pageable inputs: all (the
// copy engine would stage pageable memory through driver buffers anyway, so converting into our
// pinned staging costs no extra pass). Pinned inputs: the host converts ~67 GB/s of float with 16
// threads while PCIe moves ~54 GB/s, so converting ~70 % of the slots on the host and sending the
// rest as float balances the two (BBM_HOST_CONVERT overrides, 0..1).
double host_convert_fraction(const void* sample) {
  const char* e = std::getenv("BBM_HOST_CONVERT");
  if (e) return std::min(1.0, std::max(0.0, std::atof(e)));
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, sample) != cudaSuccess) {
    (void)cudaGetLastError();
    return 1.0;
  }
  return at.type == cudaMemoryTypeHost ? 0.7 : 1.0;
}

void throw_if_bad(const int* hbad, int count) {
  static const char* names[4] = {"q", "k", "v", "d_out"};
  for (int t = 0; t < count; ++t)  // require_finite (engine.hpp:237-242)
    if (hbad[t]) throw ArgError(std::string(names[t]) + " must hold finite values");
}

}  // namespace

void launch_pad_to_bf16(const float* in, void* out, uint64_t rows, uint32_t w, uint32_t D, int* bad,
                        cudaStream_t s) {
  pad_to_bf16_kernel<<<grid_for_elems(rows * D), 256, 0, s>>>(in, static_cast<__nv_bfloat16*>(out), rows,
                                                              w, D, bad);
  BBM_CUDA(cudaGetLastError());
}

void launch_pad_f32(const float* in, float* out, uint64_t rows, uint32_t w, uint32_t D, cudaStream_t s) {
  pad_f32_kernel<<<grid_for_elems(rows * D), 256, 0, s>>>(in, out, rows, w, D);
  BBM_CUDA(cudaGetLastError());
}

void launch_crop_to_f32(const void* in, float* out, uint64_t rows, uint32_t D, uint32_t w, cudaStream_t s) {
  crop_to_f32_kernel<<<grid_for_elems(rows * w), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(in), out,
                                                              rows, D, w);
  BBM_CUDA(cudaGetLastError());
}

void run_fwd_host_pipelined(const Prep& prep, int variant, const uint16_t* q, const uint16_t* k,
                            const uint16_t* v, uint16_t* out, float* row_max, float* row_sum,
                            uint64_t slots, uint32_t d, float scale, int num_sms, double* span_ms) {
  std::lock_guard<std::mutex> lk(prep.pipe_mu);
  HostPipe& p = pipe_of(prep);
  BBM_CUDA(cudaMemsetAsync(p.bad, 0, 4 * sizeof(int), p.comp));
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
    const uint16_t* ins[3] = {dq + off, dk + off, dv + off};
    for (int t = 0; t < 3; ++t)
      check_finite_bf16_kernel<<<grid_for_elems(ns * per), 256, 0, p.comp>>>(ins[t], ns * per, p.bad + t);
    BBM_CUDA(cudaGetLastError());
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
  int hbad[4] = {0, 0, 0, 0};
  BBM_CUDA(cudaMemcpyAsync(hbad, p.bad, 3 * sizeof(int), cudaMemcpyDeviceToHost, p.comp));
  BBM_CUDA(cudaStreamSynchronize(p.comp));
  BBM_CUDA(cudaStreamSynchronize(p.d2h));
  if (span_ms) {
    float ms = 0.0f;
    BBM_CUDA(cudaEventElapsedTime(&ms, t0, t1));
    *span_ms = ms;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
  throw_if_bad(hbad, 3);
}

// The reference's own signature, Matrix<float> in and out (engine.hpp:282-285, 489-505): per-slot
// float host buffers (SlotInputs), rounded to bf16 on the device with the finiteness check fused
// into the conversion, outputs widened back to float and the row statistics to double. Same
// three-stream chunk pipeline as the bf16 path; the PCIe traffic is twice the bf16 form's.
void run_fwd_host_f32(const Prep& prep, int variant, const float* const* q, const float* const* k,
                      const float* const* v, float* const* out, double* const* row_max,
                      double* const* row_sum, uint64_t slots, uint32_t d_k, uint32_t d_v, float scale,
                      int num_sms, double* span_ms) {
  std::lock_guard<std::mutex> lk(prep.pipe_mu);
  HostPipe& p = pipe_of(prep);
  const bool want_max = row_max && row_max[0], want_sum = row_sum && row_sum[0];
  // D: the kernel's head dim; w[t]: the caller's row width of q, k, v (and d_v of out)
  const uint32_t D = kernel_dim(d_k, d_v), w[3] = {d_k, d_k, d_v};
  const bool padded = d_k != D || d_v != D;
  const uint64_t n = prep.n, per = n * D, elems = slots * per, rows = slots * n;
  // f32 in q k v | bf16 q k v o | f32 o | f32 max, sum | f64 max, sum; every piece 256-B aligned
  // (the TMA descriptors need 16-B aligned bases; caller widths need not be multiples of 4)
  const size_t b_in[3] = {rows * w[0] * 4, rows * w[1] * 4, rows * w[2] * 4}, b_bf = elems * 2;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t sizes[11] = {b_in[0], b_in[1], b_in[2], b_bf, b_bf, b_bf, b_bf, b_in[2], rows * 4, rows * 4, rows * 16};
  size_t total = 0;
  for (size_t z : sizes) total += al(z);
  uint8_t* cur = reserve(p, total);
  auto take = [&](size_t b) {
    uint8_t* r = cur;
    cur += al(b);
    return r;
  };
  float* fin[3];
  for (int t = 0; t < 3; ++t) fin[t] = reinterpret_cast<float*>(take(b_in[t]));
  __nv_bfloat16* bq = reinterpret_cast<__nv_bfloat16*>(take(b_bf));
  __nv_bfloat16* bk = reinterpret_cast<__nv_bfloat16*>(take(b_bf));
  __nv_bfloat16* bv = reinterpret_cast<__nv_bfloat16*>(take(b_bf));
  __nv_bfloat16* bo = reinterpret_cast<__nv_bfloat16*>(take(b_bf));
  float* fo = reinterpret_cast<float*>(take(b_in[2]));
  float* fmax = reinterpret_cast<float*>(take(rows * 4));
  float* fsum = reinterpret_cast<float*>(take(rows * 4));
  double* dmax = reinterpret_cast<double*>(take(rows * 16));
  double* dsum = dmax + rows;
  BBM_CUDA(cudaMemsetAsync(p.bad, 0, 4 * sizeof(int), p.comp));
  const uint64_t chunks =
      std::max<uint64_t>(1, std::min<uint64_t>({slots, kMaxChunks, (b_in[0] + b_in[1] + b_in[2]) / kChunkBytes}));
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (span_ms) {
    BBM_CUDA(cudaEventCreate(&t0));
    BBM_CUDA(cudaEventCreate(&t1));
    BBM_CUDA(cudaEventRecord(t0, p.h2d));
  }
  const float* const* src[3] = {q, k, v};
  __nv_bfloat16* dst[3] = {bq, bk, bv};
  // Per chunk, the first nh slots are converted to bf16 by host threads into a pinned staging
  // buffer (half the PCIe bytes), the rest cross PCIe as float and are converted on the device.
  // The host converts chunk c while the copy engines and the SMs work on chunks c-1, c-2. Padded
  // head dims convert everything on the device (the row-pitch change rides on the conversion).
  const double frac = padded ? 0.0 : host_convert_fraction(q[0]);
  const uint64_t max_ns = (slots + chunks - 1) / chunks;
  const uint64_t max_nh = std::min<uint64_t>(max_ns, static_cast<uint64_t>(frac * static_cast<double>(max_ns) + 0.5));
  if (max_nh > 0) {
    const size_t need = 3 * max_nh * per * 2;
    if (need > p.stage_cap) {
      BBM_CUDA(cudaStreamSynchronize(p.h2d));
      if (p.stage) cudaFreeHost(p.stage);
      p.stage = nullptr;
      p.stage_cap = 0;
      BBM_CUDA(cudaMallocHost(&p.stage, 2 * need));
      p.stage_cap = need;
    }
    if (!p.pool) {
      const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
      p.pool = new HostPool(std::min(hw, 16u) - 1);
    }
  }
  std::atomic<int> host_bad[3];
  for (auto& hb : host_bad) hb.store(0);
  constexpr uint64_t kPiece = 1ull << 21;  // elements per host conversion task
  const uint64_t pieces = (per + kPiece - 1) / kPiece;
  for (uint64_t c = 0; c < chunks; ++c) {
    const uint64_t s0 = slots * c / chunks, s1 = slots * (c + 1) / chunks, ns = s1 - s0;
    const uint64_t off = s0 * per;
    const uint64_t nh = std::min<uint64_t>(ns, static_cast<uint64_t>(frac * static_cast<double>(ns) + 0.5));
    if (nh > 0) {
      uint16_t* st = reinterpret_cast<uint16_t*>(p.stage + (c & 1) * p.stage_cap);
      if (c >= 2) BBM_CUDA(cudaEventSynchronize(p.ev_stage[c & 1]));  // its H2D two chunks ago is done
      p.pool->run(static_cast<uint32_t>(3 * nh * pieces), [&](uint32_t task) {
        const uint64_t t = task / (nh * pieces), rem = task % (nh * pieces);
        const uint64_t sl = rem / pieces, e0 = (rem % pieces) * kPiece, e1 = std::min(per, e0 + kPiece);
        if (f32_to_bf16_host(src[t][s0 + sl] + e0, st + (t * nh + sl) * per + e0, e1 - e0))
          host_bad[t].store(1, std::memory_order_relaxed);
      });
      for (int t = 0; t < 3; ++t)
        BBM_CUDA(cudaMemcpyAsync(dst[t] + off, st + t * nh * per, nh * per * 2, cudaMemcpyHostToDevice, p.h2d));
      BBM_CUDA(cudaEventRecord(p.ev_stage[c & 1], p.h2d));
    }
    for (uint64_t sl = s0 + nh; sl < s1; ++sl)
      for (int t = 0; t < 3; ++t)
        BBM_CUDA(cudaMemcpyAsync(fin[t] + sl * n * w[t], src[t][sl], n * w[t] * 4, cudaMemcpyHostToDevice, p.h2d));
    BBM_CUDA(cudaEventRecord(p.ev_in[c], p.h2d));
    BBM_CUDA(cudaStreamWaitEvent(p.comp, p.ev_in[c], 0));
    if (ns > nh) {
      const uint64_t r0 = (s0 + nh) * n, nr = (ns - nh) * n;
      for (int t = 0; t < 3; ++t) {
        if (padded)
          launch_pad_to_bf16(fin[t] + r0 * w[t], dst[t] + r0 * D, nr, w[t], D, p.bad + t, p.comp);
        else
          f32_to_bf16_check_kernel<<<grid_for_elems(nr * D), 256, 0, p.comp>>>(fin[t] + r0 * D, dst[t] + r0 * D,
                                                                               nr * D, p.bad + t);
      }
      BBM_CUDA(cudaGetLastError());
    }
    AttnArgs a{bq + off, bk + off, bv + off, bo + off, fmax + s0 * n, fsum + s0 * n, ns, n, D, scale, variant};
    launch_attn_fwd(prep, a, p.comp, num_sms);
    if (padded) {
      launch_crop_to_f32(bo + off, fo + s0 * n * d_v, ns * n, D, d_v, p.comp);
      widen_stats_kernel<<<grid_for_elems(ns * n), 256, 0, p.comp>>>(
          fmax + s0 * n, fsum + s0 * n, want_max ? dmax + s0 * n : nullptr, want_sum ? dsum + s0 * n : nullptr,
          ns * n);
    } else {
      widen_outputs_kernel<<<grid_for_elems(ns * per), 256, 0, p.comp>>>(
          bo + off, fo + off, ns * per, fmax + s0 * n, fsum + s0 * n, want_max ? dmax + s0 * n : nullptr,
          want_sum ? dsum + s0 * n : nullptr, ns * n);
    }
    BBM_CUDA(cudaGetLastError());
    BBM_CUDA(cudaEventRecord(p.ev_out[c], p.comp));
    BBM_CUDA(cudaStreamWaitEvent(p.d2h, p.ev_out[c], 0));
    for (uint64_t sl = s0; sl < s1; ++sl) {
      BBM_CUDA(cudaMemcpyAsync(out[sl], fo + sl * n * d_v, n * d_v * 4, cudaMemcpyDeviceToHost, p.d2h));
      if (want_max) BBM_CUDA(cudaMemcpyAsync(row_max[sl], dmax + sl * n, n * 8, cudaMemcpyDeviceToHost, p.d2h));
      if (want_sum) BBM_CUDA(cudaMemcpyAsync(row_sum[sl], dsum + sl * n, n * 8, cudaMemcpyDeviceToHost, p.d2h));
    }
  }
  if (span_ms) BBM_CUDA(cudaEventRecord(t1, p.d2h));
  int hbad[4] = {0, 0, 0, 0};
  BBM_CUDA(cudaMemcpyAsync(hbad, p.bad, 3 * sizeof(int), cudaMemcpyDeviceToHost, p.comp));
  BBM_CUDA(cudaStreamSynchronize(p.comp));
  BBM_CUDA(cudaStreamSynchronize(p.d2h));
  if (span_ms) {
    float ms = 0.0f;
    BBM_CUDA(cudaEventElapsedTime(&ms, t0, t1));
    *span_ms = ms;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
  for (int t = 0; t < 3; ++t) hbad[t] |= host_bad[t].load();
  throw_if_bad(hbad, 3);
}

// blocked_backward with the reference's storage (engine.hpp:346-471): float host q, k, v, out,
// d_out, double row statistics, float gradients out. Runs on the prep's persistent pipeline
// stream and buffers (no per-call stream, allocation or launch-context setup); q, k, v, d_out are
// rounded to bf16 on the device with the finiteness check fused, out stays fp32 for
// delta = rowsum(d_out * out); head dims other than the kernel's are zero-padded / cropped.
void run_bwd_host_f32(const Prep& prep, int variant, const float* q, const float* k, const float* v,
                      const float* out, const double* row_max, const double* row_sum, const float* d_out,
                      float* dq, float* dk, float* dv, uint64_t slots, uint32_t d_k, uint32_t d_v,
                      float scale, int num_sms) {
  std::lock_guard<std::mutex> lk(prep.pipe_mu);
  HostPipe& p = pipe_of(prep);
  cudaStream_t s = p.comp;
  const uint32_t D = kernel_dim(d_k, d_v);
  const uint64_t rows = slots * prep.n, elems = rows * D;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  uint8_t* cur = reserve(p, 2 * al(elems * 4) + 7 * al(elems * 2) + 2 * al(rows * 4));
  auto take = [&](size_t b) {
    uint8_t* r = cur;
    cur += al(b);
    return r;
  };
  float* stage = reinterpret_cast<float*>(take(elems * 4));
  float* o32 = reinterpret_cast<float*>(take(elems * 4));
  __nv_bfloat16* b[4];  // q k v dO
  for (auto& x : b) x = reinterpret_cast<__nv_bfloat16*>(take(elems * 2));
  __nv_bfloat16* g3[3];  // dq dk dv
  for (auto& x : g3) x = reinterpret_cast<__nv_bfloat16*>(take(elems * 2));
  float* rm = reinterpret_cast<float*>(take(rows * 4));
  float* rs = reinterpret_cast<float*>(take(rows * 4));
  BBM_CUDA(cudaMemsetAsync(p.bad, 0, 4 * sizeof(int), s));
  const float* srcs[4] = {q, k, v, d_out};
  const uint32_t w_in[4] = {d_k, d_k, d_v, d_v};
  for (int t = 0; t < 4; ++t) {
    BBM_CUDA(cudaMemcpyAsync(stage, srcs[t], rows * w_in[t] * 4, cudaMemcpyHostToDevice, s));
    if (w_in[t] == D) {
      f32_to_bf16_check_kernel<<<grid_for_elems(elems), 256, 0, s>>>(stage, b[t], elems, p.bad + t);
      BBM_CUDA(cudaGetLastError());
    } else {
      launch_pad_to_bf16(stage, b[t], rows, w_in[t], D, p.bad + t, s);
    }
  }
  if (d_v == D) {
    BBM_CUDA(cudaMemcpyAsync(o32, out, elems * 4, cudaMemcpyHostToDevice, s));
  } else {
    BBM_CUDA(cudaMemcpyAsync(stage, out, rows * d_v * 4, cudaMemcpyHostToDevice, s));
    launch_pad_f32(stage, o32, rows, d_v, D, s);
  }
  std::vector<float> hst(2 * rows);
  for (uint64_t i = 0; i < rows; ++i) {
    hst[i] = static_cast<float>(row_max[i]);
    hst[rows + i] = static_cast<float>(row_sum[i]);
  }
  BBM_CUDA(cudaMemcpyAsync(rm, hst.data(), rows * 4, cudaMemcpyHostToDevice, s));
  BBM_CUDA(cudaMemcpyAsync(rs, hst.data() + rows, rows * 4, cudaMemcpyHostToDevice, s));
  int hbad[4] = {0, 0, 0, 0};
  BBM_CUDA(cudaMemcpyAsync(hbad, p.bad, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
  BBM_CUDA(cudaStreamSynchronize(s));  // hst, hbad
  throw_if_bad(hbad, 4);  // require_finite (engine.hpp:237-242, 358)
  BwdArgs a{b[0], b[1], b[2], o32, true, rm, rs, b[3], g3[0], g3[1], g3[2], slots, prep.n, D, scale, variant};
  launch_attn_bwd(prep, a, s, num_sms);
  float* dsts[3] = {dq, dk, dv};
  const uint32_t w_out[3] = {d_k, d_k, d_v};
  for (int t = 0; t < 3; ++t) {  // stream order: each widening follows the previous download
    launch_crop_to_f32(g3[t], stage, rows, D, w_out[t], s);
    BBM_CUDA(cudaMemcpyAsync(dsts[t], stage, rows * w_out[t] * 4, cudaMemcpyDeviceToHost, s));
  }
  BBM_CUDA(cudaStreamSynchronize(s));
}

// The RCM path end to end (reorder.hpp:156-189 + bench.hpp:448-467): the caller's Q/K/V are in
// the ORIGINAL token order, `prep` was built from permute_mask(mask, perm), forward = perm's
// new -> old map. Per slot chunk: H2D, the forward with the permutation applied on the device
// (launch_attn_fwd with AttnArgs::rows: by default every Q / K / V row gathered inside the kernel
// by LSU cp.async, O rows and row statistics written to their original tokens), D2H.
void run_fwd_host_rcm(const Prep& prep, int variant, const uint32_t* forward, const uint16_t* q,
                      const uint16_t* k, const uint16_t* v, uint16_t* out, float* row_max,
                      float* row_sum, uint64_t slots, uint32_t d, float scale, int num_sms,
                      double* span_ms) {
  std::lock_guard<std::mutex> lk(prep.pipe_mu);
  HostPipe& p = pipe_of(prep);
  const uint64_t n = prep.n, per = n * d, tbytes = slots * per * 2, sbytes = slots * n * 4;
  uint8_t* base = reserve(p, 4 * tbytes + 2 * sbytes + n * 4 + 256);
  uint16_t* dq = reinterpret_cast<uint16_t*>(base);
  uint16_t* dk = dq + slots * per;
  uint16_t* dv = dk + slots * per;
  uint16_t* dout = dv + slots * per;
  float* dmax = reinterpret_cast<float*>(dout + slots * per);
  float* dsum = dmax + slots * n;
  uint32_t* dfwd = reinterpret_cast<uint32_t*>(dsum + slots * n);
  BBM_CUDA(cudaMemsetAsync(p.bad, 0, 4 * sizeof(int), p.comp));
  BBM_CUDA(cudaMemcpyAsync(dfwd, forward, n * 4, cudaMemcpyHostToDevice, p.comp));
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
    const uint16_t* ins[3] = {dq + off, dk + off, dv + off};
    for (int t = 0; t < 3; ++t)
      check_finite_bf16_kernel<<<grid_for_elems(ns * per), 256, 0, p.comp>>>(ins[t], ns * per, p.bad + t);
    BBM_CUDA(cudaGetLastError());
    AttnArgs a{dq + off, dk + off, dv + off, dout + off, row_max ? dmax + s0 * n : nullptr,
               row_sum ? dsum + s0 * n : nullptr, ns, n, d, scale, variant, dfwd};
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
  int hbad[4] = {0, 0, 0, 0};
  BBM_CUDA(cudaMemcpyAsync(hbad, p.bad, 3 * sizeof(int), cudaMemcpyDeviceToHost, p.comp));
  BBM_CUDA(cudaStreamSynchronize(p.comp));
  BBM_CUDA(cudaStreamSynchronize(p.d2h));
  if (span_ms) {
    float ms = 0.0f;
    BBM_CUDA(cudaEventElapsedTime(&ms, t0, t1));
    *span_ms = ms;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
  throw_if_bad(hbad, 3);
}

}  // namespace bbm
