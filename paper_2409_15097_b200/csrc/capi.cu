// capi.cu — implementation of the C ABI in include/bbm_capi.h (host orchestration).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bbm_capi.h"
#include "bbm_internal.h"

namespace bbm {

thread_local std::string g_last_error;
TraceConfig g_trace;

template <class F>
bbm_status guarded(F&& f) {
  try {
    f();
    return BBM_OK;
  } catch (const ArgError& e) {
    g_last_error = e.what();
    return BBM_ERR_INVALID;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return BBM_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return BBM_ERR_INTERNAL;
  }
}

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    BBM_CUDA(cudaGetDevice(&prev));
    if (prev != dev) BBM_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int sm_count(int dev) {
  static std::atomic<int> cache[64] = {};  // read by the multi-GPU driver's threads
  if (dev >= 0 && dev < 64) {
    const int c = cache[dev].load(std::memory_order_relaxed);
    if (c) return c;
  }
  int v = 0;
  BBM_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
  if (dev >= 0 && dev < 64) cache[dev].store(v, std::memory_order_relaxed);
  return v;
}

template <class T>
T* dmalloc(uint64_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  BBM_CUDA(cudaMalloc(&p, count * sizeof(T)));
  return static_cast<T*>(p);
}

// Kernel view from km.sums (already built): lists, bitmaps. Async, no allocation, no host sync.
// (Totals and the LPT row order are derived on demand: spec_now, ensure_bwd_meta.)
void build_kernel_view(const KernelMeta& km, uint64_t n, cudaStream_t s) {
  launch_rowmeta(km.sums, n, kTile, kTile, km.krows, km.kcols, km.occ, km.run_off, km.run_len,
                 km.row_stats, km.list, km.row_cnt, s);
  launch_compact_bitmaps(km, s);
}

// The complete kernel view from a dense bool mask / from packed words (in_wpr words per row; may
// be the padded mask itself): the fused one-launch preprocessor, or the kernel chain when the
// input does not fit it (unaligned bool rows, n % 16 != 0).
void view_from_bool(const KernelMeta& km, const uint8_t* d_bool, uint64_t n, uint64_t stride, cudaStream_t s) {
  if (launch_prep_fused_bool(d_bool, n, stride, km, s)) return;
  launch_pack_bool(d_bool, n, stride, km, s);
  build_kernel_view(km, n, s);
}

void view_from_words(const KernelMeta& km, const uint64_t* d_words, uint64_t in_wpr, uint64_t n, cudaStream_t s) {
  if (launch_prep_fused_words(d_words, in_wpr, n, km, s)) return;
  if (d_words != km.mask) launch_pad_packed(d_words, n, km, s);
  launch_sums128(km, s);
  build_kernel_view(km, n, s);
}

void validate_spec(uint64_t n, uint64_t bi, uint64_t bj) {
  require(bi >= 1 && bj >= 1, "block sizes must be >= 1");  // mask.hpp:61-63
  require(n >= 1, "mask must be non-empty");                 // engine.hpp:82
  require(n < (1ull << 31), "mask too large for the device metadata (n >= 2^31)");
}

Prep* new_prep(uint64_t n, int device, uint64_t bi, uint64_t bj) {
  auto* pr = new Prep;
  pr->device = device;
  pr->n = n;
  pr->bi = bi;
  pr->bj = bj;
  try {
    void* arena = nullptr;
    BBM_CUDA(cudaMalloc(&arena, kernel_meta_bytes(n)));
    carve_kernel_meta(pr->kmeta, n, static_cast<uint8_t*>(arena));
    BBM_CUDA(cudaMemset(pr->kmeta.ctr, 0, (static_cast<size_t>(pr->kmeta.krows) + 1) * 4));
    BBM_CUDA(cudaEventCreateWithFlags(&pr->ready, cudaEventDisableTiming));
  } catch (...) {
    delete pr;
    throw;
  }
  return pr;
}

// Order stream s after every launch still reading the current metadata (an update must not
// overwrite lists a queued kernel is walking), then after the latest metadata write.
void order_update_after_launches(const Prep& pr, cudaStream_t s) {
  for (auto& kv : pr.streams)
    if (kv.second.done) BBM_CUDA(cudaStreamWaitEvent(s, kv.second.done, 0));
  BBM_CUDA(cudaStreamWaitEvent(s, pr.ready, 0));
}

// A new metadata version is complete on stream s.
void publish_version(const Prep& pr, cudaStream_t s) {
  ++pr.version;
  BBM_CUDA(cudaEventRecord(pr.ready, s));
}

}  // namespace

size_t kernel_meta_bytes(uint64_t n) {
  KernelMeta km;
  carve_kernel_meta(km, n, nullptr);
  return km.arena_bytes;
}

void carve_kernel_meta(KernelMeta& km, uint64_t n, uint8_t* arena) {
  km.krows = static_cast<uint32_t>((n + kTile - 1) / kTile);
  km.kcols = km.krows;
  const uint64_t tiles = static_cast<uint64_t>(km.krows) * km.kcols;
  size_t off = 0;
  auto take = [&](auto*& ptr, uint64_t count) {
    using T = std::remove_reference_t<decltype(*ptr)>;
    ptr = reinterpret_cast<T*>(arena + off);
    off += (std::max<uint64_t>(1, count) * sizeof(T) + 255) / 256 * 256;
  };
  km.arena = arena;
  take(km.mask, static_cast<uint64_t>(km.krows) * kTile * km.kcols * 2);
  take(km.bitmaps, tiles * kTile);
  take(km.sums, tiles);
  take(km.list, tiles);
  take(km.row_cnt, km.krows);
  take(km.order, km.krows);
  take(km.occ, tiles);
  take(km.halves, tiles);
  take(km.run_off, km.krows);
  take(km.run_len, km.krows);
  take(km.row_stats, static_cast<uint64_t>(km.krows) * 3);
  take(km.totals, 3);
  take(km.scratch, static_cast<uint64_t>(km.krows) + km.kcols + 2);
  take(km.partial, tiles * kPrepRowSplits);
  take(km.ctr, static_cast<uint64_t>(km.krows) + 1);
  km.arena_bytes = off;
}

Prep::~Prep() {
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaDeviceSynchronize();  // no queued launch may still read what is freed below
  delete pipe;
  cudaFree(kmeta.arena);
  free_bwd_meta(bwd);
  for (auto& kv : streams) {
    StreamCtx& c = kv.second;
    cudaFree(c.ctr);
    cudaFree(c.ws);
    cudaFree(c.split_ctr);
    cudaFree(c.rowws);
    cudaFree(c.perm);
    if (c.done) cudaEventDestroy(c.done);
    for (auto& pl : c.plans) {
      cudaFree(pl.second.mem);
      if (pl.second.host_hdr) cudaFreeHost(pl.second.host_hdr);
      if (pl.second.hdr_ev) cudaEventDestroy(pl.second.hdr_ev);
    }
  }
  if (ready) cudaEventDestroy(ready);
  if (prev >= 0) cudaSetDevice(prev);
}

StreamCtx& Prep::ctx_for(cudaStream_t s) const {
  auto it = streams.find(s);
  if (it == streams.end()) {
    StreamCtx c;
    c.ctr = dmalloc<uint32_t>(8);
    BBM_CUDA(cudaMemsetAsync(c.ctr, 0, 8 * sizeof(uint32_t), s));
    BBM_CUDA(cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming));
    it = streams.emplace(s, c).first;
  }
  StreamCtx& c = it->second;
  if (c.seen_version != version) {
    BBM_CUDA(cudaStreamWaitEvent(s, ready, 0));
    c.seen_version = version;
  }
  return c;
}

void mark_launch_done(StreamCtx& ctx, cudaStream_t s) { BBM_CUDA(cudaEventRecord(ctx.done, s)); }

const SpecMeta& Prep::spec_now() const {
  std::lock_guard<std::recursive_mutex> lk(mu);
  if (spec_version == version) return spec;
  DeviceGuard g(device);
  BBM_CUDA(cudaEventSynchronize(ready));
  const KernelMeta& km = kmeta;
  SpecMeta sp;
  sp.bi = bi;
  sp.bj = bj;
  sp.rows = (n + bi - 1) / bi;
  sp.cols = (n + bj - 1) / bj;
  const bool same = (bi == kTile && bj == kTile);
  const uint64_t tiles = sp.rows * sp.cols;
  cudaStream_t s;
  BBM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  uint8_t* tmp = nullptr;
  auto release = [&] {
    if (tmp) cudaFree(tmp);
    cudaStreamDestroy(s);
  };
  try {
    uint32_t *d_sums = km.sums, *d_off = km.run_off, *d_tot = km.run_len;
    uint8_t* d_occ = km.occ;
    uint64_t *d_stats = km.row_stats, *d_totals = km.totals;
    // the kernel view's totals (block_stats at 128 x 128) from its per-row statistics
    launch_finalize(km.row_stats, km.krows, nullptr, nullptr, km.totals, s);
    if (!same) {  // the caller's BlockSpec from the padded mask (any spec, mask.hpp:184-247)
      const size_t b_sums = tiles * 4, b_occ = (tiles + 7) / 8 * 8, b_rows = sp.rows * 4;
      BBM_CUDA(cudaMalloc(&tmp, b_sums + b_occ + 2 * b_rows + sp.rows * 24 + 24 + 64));
      d_sums = reinterpret_cast<uint32_t*>(tmp);
      d_occ = tmp + b_sums;
      d_off = reinterpret_cast<uint32_t*>(tmp + b_sums + b_occ);
      d_tot = d_off + sp.rows;
      d_stats = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(d_tot + sp.rows) + 7) / 8 * 8);
      d_totals = d_stats + sp.rows * 3;
      launch_sums_generic(km, n, bi, bj, sp.rows, sp.cols, d_sums, s);
      launch_rowmeta(d_sums, n, bi, bj, sp.rows, sp.cols, d_occ, d_off, d_tot, d_stats, nullptr,
                     nullptr, s);
      launch_finalize(d_stats, sp.rows, nullptr, nullptr, d_totals, s);
    }
    sp.sums.resize(tiles);
    sp.occ.resize(tiles);
    sp.offset.resize(sp.rows);
    sp.total_ones.resize(sp.rows);
    uint64_t totals[3] = {0, 0, 0}, ktotals[3] = {0, 0, 0};
    BBM_CUDA(cudaMemcpyAsync(sp.sums.data(), d_sums, tiles * 4, cudaMemcpyDeviceToHost, s));
    BBM_CUDA(cudaMemcpyAsync(sp.occ.data(), d_occ, tiles, cudaMemcpyDeviceToHost, s));
    BBM_CUDA(cudaMemcpyAsync(sp.offset.data(), d_off, sp.rows * 4, cudaMemcpyDeviceToHost, s));
    BBM_CUDA(cudaMemcpyAsync(sp.total_ones.data(), d_tot, sp.rows * 4, cudaMemcpyDeviceToHost, s));
    BBM_CUDA(cudaMemcpyAsync(totals, d_totals, 24, cudaMemcpyDeviceToHost, s));
    BBM_CUDA(cudaMemcpyAsync(ktotals, km.totals, 24, cudaMemcpyDeviceToHost, s));
    BBM_CUDA(cudaStreamSynchronize(s));
    sp.blocks_total = tiles;
    sp.blocks_nonzero = totals[0];
    sp.blocks_full = totals[1];
    sp.ones = totals[2];
    sp.knnz = ktotals[0];
    sp.kfull = ktotals[1];
  } catch (...) {
    release();
    throw;
  }
  release();
  spec = std::move(sp);
  spec_version = version;
  return spec;
}

}  // namespace bbm

using namespace bbm;

struct bbm_prep_s {
  std::unique_ptr<Prep> p;
  // replicas on other devices for the multi-GPU driver, created lazily per mask version; shared
  // so that a driver call still running on them survives an update that drops the cache
  std::vector<std::shared_ptr<bbm_prep_s>> replicas;
};

namespace bbm_capi_detail {
Prep& unwrap(bbm_prep h) {
  require(h != nullptr && h->p != nullptr, "null prep handle");
  return *h->p;
}

bbm_prep wrap(Prep* p) {
  auto* h = new bbm_prep_s;
  h->p.reset(p);
  return h;
}

void check_common_args(int variant, uint64_t slots, double scale) {
  require(variant >= 0 && variant <= 3, "unknown variant");
  require(slots >= 1, "need at least one batch/head slot");  // engine.hpp:493
  require(std::isfinite(scale), "scale must be finite");     // engine.hpp:253
  // documented narrowing: the kernels scale scores in fp32 log2 units
  require(std::isfinite(static_cast<float>(scale) * 1.4426950408889634f),
          "scale outside the fp32 range of the sm_100a kernel");
}

// device-pointer entries: the caller's layout is the kernel's, [slots][n][64 | 128]
void check_attn_args(const Prep& pr, int variant, uint64_t slots, uint32_t d, double scale) {
  check_common_args(variant, slots, scale);
  if (d != 64 && d != 128)
    throw ArgError("head dim " + std::to_string(d) +
                   " unsupported by the device-pointer entries (64 or 128; the float host-buffer"
                   " entries take any d_k, d_v <= 128)");
  (void)pr;
}

// float host-buffer entries (validate_forward_args, engine.hpp:244-258): any positive d_k up to 128
// (documented narrowing: the kernels hold one 128-column head-dim tile of Q / K) and any positive
// d_v; the device copy is zero-padded to kernel_dim(d_k, d_v), and d_v above 128 runs as column
// passes over V (v_column_passes below)
void check_host_dims(int variant, uint64_t slots, uint32_t d_k, uint32_t d_v, double scale) {
  check_common_args(variant, slots, scale);
  require(d_k >= 1, "q and k must share a positive head dim");
  require(d_v >= 1, "v must have a positive head dim");
  if (d_k > 128)
    throw ArgError("head dim d_k = " + std::to_string(d_k) + " unsupported by the sm_100a kernel (at most 128)");
}

// d_v > 128: the output columns are independent given the softmax, O[:, c] = P V[:, c], so the
// forward runs once per 128-column slice of V (every pass computes the same P bit for bit: same
// Q, K and kernel; the zero padding adds exact zeros), and the backward decomposes linearly,
// dS = sum_c P o (dO_c V_c^T - rowsum(dO_c o O_c)): dq and dk are the sums of the slices' dq / dk
// (added in slice order), dv is the concatenation of the slices' dv. The slices are gathered from
// and scattered to the caller's row-major [n][d_v] storage on the host.
struct VSlice {
  uint32_t c0, w;
};
std::vector<VSlice> v_slices(uint32_t d_v) {
  std::vector<VSlice> out;
  for (uint32_t c0 = 0; c0 < d_v; c0 += 128) out.push_back({c0, std::min<uint32_t>(128, d_v - c0)});
  return out;
}
void copy_cols(const float* src, uint32_t ld_src, uint32_t c_src, float* dst, uint32_t ld_dst, uint32_t c_dst,
               uint64_t rows, uint32_t w) {
  for (uint64_t r = 0; r < rows; ++r)
    std::memcpy(dst + r * ld_dst + c_dst, src + r * ld_src + c_src, w * sizeof(float));
}

// Permutation::from_forward (reorder.hpp:57-68): forward must be a bijection on [0, n)
void check_bijection(const uint32_t* fwd, uint64_t n) {
  std::vector<char> seen(n, 0);
  for (uint64_t a = 0; a < n; ++a) {
    require(fwd[a] < n && !seen[fwd[a]], "forward map is not a bijection");
    seen[fwd[a]] = 1;
  }
}

// Creation: the kernel view is queued on `s`; publish the first version and compute the
// caller-spec host metadata (one sync, like the reference's synchronous preprocess_mask).
bbm_prep finish_prep(std::unique_ptr<Prep> pr, cudaStream_t s) {
  BBM_CUDA(cudaEventRecord(pr->ready, s));
  pr->spec_now();
  return wrap(pr.release());
}

// Updates rebuild the kernel view of the SAME prep for a new mask of the same n, asynchronously
// on `stream`: ordered after every queued launch that reads the prep, then published as a new
// version. Later launches on any stream wait for it; getters and counters recompute the
// caller-spec metadata; replicas made for the multi-GPU driver are dropped (they hold the old
// mask) and re-made on their next use.
template <class Fill>
void update_prep(bbm_prep h, void* stream, Fill&& fill) {
  Prep& pr = unwrap(h);
  std::lock_guard<std::recursive_mutex> lk(pr.mu);
  DeviceGuard g(pr.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  order_update_after_launches(pr, s);
  fill(pr, s);
  publish_version(pr, s);
  h->replicas.clear();
}

// IPC form of the replication, for one process per GPU (torchrun): the exporter publishes the
// arena's cudaIpcMemHandle plus the host metadata as one flat blob, the importer copies the arena
// peer to peer into its own prep. The exporter's prep must stay alive and un-updated until every
// importer has returned.
constexpr uint64_t kIpcMagic = 0x3150494D4D4242ull;  // "BBMMIP1"
struct IpcHeader {
  uint64_t magic, abi, n, bi, bj, arena_bytes, rows, cols;
  uint64_t blocks_total, blocks_nonzero, blocks_full, ones, knnz, kfull;
  cudaIpcMemHandle_t handle;
};
size_t ipc_size(const SpecMeta& sp) {
  return sizeof(IpcHeader) + sp.sums.size() * 4 + sp.occ.size() + sp.offset.size() * 4 +
         sp.total_ones.size() * 4;
}

}  // namespace bbm_capi_detail
using namespace bbm_capi_detail;

extern "C" {

int bbm_abi_version(void) { return BBM_ABI_VERSION; }

const char* bbm_last_error(void) { return g_last_error.c_str(); }

bbm_status bbm_device_count(int* count) {
  return guarded([&] {
    int c = 0;
    const cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}

bbm_status bbm_preprocess_packed_host(const uint64_t* words, uint64_t n, uint64_t bi, uint64_t bj,
                                      int device, bbm_prep* out) {
  return guarded([&] {
    validate_spec(n, bi, bj);
    require(words != nullptr && out != nullptr, "null argument");
    DeviceGuard g(device);
    std::unique_ptr<Prep> pr(new_prep(n, device, bi, bj));
    const KernelMeta& km = pr->kmeta;
    cudaStream_t s;
    BBM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    try {
      const uint64_t wpr = (n + 63) / 64, pad_wpr = static_cast<uint64_t>(km.kcols) * 2;
      const uint64_t rows_pad = static_cast<uint64_t>(km.krows) * kTile;
      BBM_CUDA(cudaMemsetAsync(km.mask, 0, rows_pad * pad_wpr * 8, s));
      BBM_CUDA(cudaMemcpy2DAsync(km.mask, pad_wpr * 8, words, wpr * 8, wpr * 8, n,
                                 cudaMemcpyHostToDevice, s));
      view_from_words(km, km.mask, pad_wpr, n, s);
      *out = finish_prep(std::move(pr), s);
    } catch (...) {
      cudaStreamDestroy(s);
      throw;
    }
    BBM_CUDA(cudaStreamDestroy(s));
  });
}

bbm_status bbm_preprocess_packed_device(const uint64_t* d_words, uint64_t n, uint64_t bi,
                                        uint64_t bj, void* stream, bbm_prep* out) {
  return guarded([&] {
    validate_spec(n, bi, bj);
    require(d_words != nullptr && out != nullptr, "null argument");
    int dev = 0;
    BBM_CUDA(cudaGetDevice(&dev));
    std::unique_ptr<Prep> pr(new_prep(n, dev, bi, bj));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    view_from_words(pr->kmeta, d_words, (n + 63) / 64, n, s);
    *out = finish_prep(std::move(pr), s);
  });
}

bbm_status bbm_preprocess_bool_device(const uint8_t* d_mask, uint64_t n, uint64_t row_stride,
                                      uint64_t bi, uint64_t bj, void* stream, bbm_prep* out) {
  return guarded([&] {
    validate_spec(n, bi, bj);
    require(d_mask != nullptr && out != nullptr, "null argument");
    require(row_stride >= n, "row stride must be >= n");
    int dev = 0;
    BBM_CUDA(cudaGetDevice(&dev));
    std::unique_ptr<Prep> pr(new_prep(n, dev, bi, bj));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    view_from_bool(pr->kmeta, d_mask, n, row_stride, s);
    *out = finish_prep(std::move(pr), s);
  });
}

bbm_status bbm_prep_update_bool_device(bbm_prep prep, const uint8_t* d_mask, uint64_t row_stride,
                                       void* stream) {
  return guarded([&] {
    Prep& pr = unwrap(prep);
    require(d_mask != nullptr && row_stride >= pr.n, "bad mask argument");
    update_prep(prep, stream, [&](Prep& p, cudaStream_t s) { view_from_bool(p.kmeta, d_mask, p.n, row_stride, s); });
  });
}

bbm_status bbm_prep_update_packed_device(bbm_prep prep, const uint64_t* d_words, void* stream) {
  return guarded([&] {
    require(d_words != nullptr, "bad mask argument");
    update_prep(prep, stream, [&](Prep& p, cudaStream_t s) {
      view_from_words(p.kmeta, d_words, (p.n + 63) / 64, p.n, s);
    });
  });
}

bbm_status bbm_prep_destroy(bbm_prep prep) {
  return guarded([&] { delete prep; });
}

bbm_status bbm_prep_get_info(bbm_prep prep, bbm_prep_info* info) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    const SpecMeta& sp = pr.spec_now();
    info->n = pr.n;
    info->block_i = sp.bi;
    info->block_j = sp.bj;
    info->rows = sp.rows;
    info->cols = sp.cols;
    info->ktile = kTile;
    info->krows = pr.kmeta.krows;
    info->kcols = pr.kmeta.kcols;
    info->knnz = sp.knnz;
    info->kfull = sp.kfull;
    info->device = pr.device;
  });
}

bbm_status bbm_prep_get_sums(bbm_prep prep, uint32_t* sums) {
  return guarded([&] {
    const SpecMeta& sp = unwrap(prep).spec_now();
    std::memcpy(sums, sp.sums.data(), sp.sums.size() * 4);
  });
}

bbm_status bbm_prep_get_occupancy(bbm_prep prep, uint8_t* occ) {
  return guarded([&] {
    const SpecMeta& sp = unwrap(prep).spec_now();
    std::memcpy(occ, sp.occ.data(), sp.occ.size());
  });
}

bbm_status bbm_prep_get_runs(bbm_prep prep, uint32_t* offset, uint32_t* total_ones) {
  return guarded([&] {
    const SpecMeta& sp = unwrap(prep).spec_now();
    if (offset) std::memcpy(offset, sp.offset.data(), sp.offset.size() * 4);
    if (total_ones) std::memcpy(total_ones, sp.total_ones.data(), sp.total_ones.size() * 4);
  });
}

bbm_status bbm_prep_get_stats(bbm_prep prep, bbm_block_stats* st) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    const SpecMeta& sp = pr.spec_now();
    // block_stats (mask.hpp:230-247): same double expressions as the reference
    st->blocks_total = sp.blocks_total;
    st->blocks_nonzero = sp.blocks_nonzero;
    st->blocks_full = sp.blocks_full;
    const double nd = static_cast<double>(pr.n);
    st->block_density = st->blocks_total ? static_cast<double>(st->blocks_nonzero) /
                                               static_cast<double>(st->blocks_total)
                                         : 0.0;
    st->element_density = nd > 0 ? static_cast<double>(sp.ones) / (nd * nd) : 0.0;
  });
}

bbm_status bbm_prep_get_kernel_lists(bbm_prep prep, uint32_t* row_cnt, uint32_t* list,
                                     uint32_t* order) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    std::lock_guard<std::recursive_mutex> lk(pr.mu);
    DeviceGuard g(pr.device);
    BBM_CUDA(cudaEventSynchronize(pr.ready));
    const KernelMeta& km = pr.kmeta;
    if (row_cnt) BBM_CUDA(cudaMemcpy(row_cnt, km.row_cnt, km.krows * 4, cudaMemcpyDeviceToHost));
    if (list)
      BBM_CUDA(cudaMemcpy(list, km.list, static_cast<uint64_t>(km.krows) * km.kcols * 4,
                          cudaMemcpyDeviceToHost));
    if (order) {  // LPT order of the row tiles, derived on demand (private scratch)
      uint32_t* tmp = dmalloc<uint32_t>(static_cast<uint64_t>(km.krows) * 2 + km.kcols + 2);
      launch_lpt_order(km.row_cnt, km.krows, km.kcols, tmp + km.krows, tmp, nullptr);
      const cudaError_t e = cudaMemcpy(order, tmp, km.krows * 4, cudaMemcpyDeviceToHost);
      cudaFree(tmp);
      BBM_CUDA(e);
    }
  });
}

bbm_status bbm_prep_get_tile_halves(bbm_prep prep, uint8_t* halves) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    require(halves != nullptr, "null argument");
    std::lock_guard<std::recursive_mutex> lk(pr.mu);
    DeviceGuard g(pr.device);
    BBM_CUDA(cudaEventSynchronize(pr.ready));
    const KernelMeta& km = pr.kmeta;
    BBM_CUDA(cudaMemcpy(halves, km.halves, static_cast<uint64_t>(km.krows) * km.kcols, cudaMemcpyDeviceToHost));
  });
}

bbm_status bbm_prep_counters(bbm_prep prep, int variant, uint64_t slots, bbm_counters* c) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    require(variant >= 0 && variant <= 3, "unknown variant");
    // classify_tile (engine.hpp:118-153) summed over every tile of the caller's BlockSpec:
    // counts depend on the mask and spec only (engine.hpp:47-48).
    const SpecMeta& sp = pr.spec_now();
    uint64_t run_blocks = 0;
    for (uint32_t t : sp.total_ones) run_blocks += t;
    bbm_counters one{};
    one.blocks_visited = sp.blocks_total;
    switch (variant) {
      case BBM_VARIANT_DENSE:
        one.blocks_processed = sp.blocks_total;
        break;
      case BBM_VARIANT_NAIVE:
        one.blocks_processed = sp.blocks_total;
        one.mask_block_reads = sp.blocks_total;
        break;
      case BBM_VARIANT_BINBLK:
        one.blocks_processed = sp.blocks_nonzero;
        one.mask_block_reads = sp.blocks_nonzero;
        one.skipped_by_binblk = sp.blocks_total - sp.blocks_nonzero;
        break;
      case BBM_VARIANT_DENSE_BINBLK:
        // run blocks are full, hence occupied: they are processed without a mask read
        one.blocks_processed = sp.blocks_nonzero;
        one.skipped_by_binblk = sp.blocks_total - sp.blocks_nonzero;
        one.skipped_mask_reads_by_run = run_blocks;
        one.mask_block_reads = sp.blocks_nonzero - run_blocks;
        break;
    }
    c->blocks_visited = one.blocks_visited * slots;
    c->blocks_processed = one.blocks_processed * slots;
    c->mask_block_reads = one.mask_block_reads * slots;
    c->skipped_by_binblk = one.skipped_by_binblk * slots;
    c->skipped_mask_reads_by_run = one.skipped_mask_reads_by_run * slots;
  });
}

bbm_status bbm_sums_metadata(const uint32_t* sums, uint64_t n, uint64_t bi, uint64_t bj,
                             int device, uint8_t* occ, uint32_t* offset, uint32_t* total_ones,
                             bbm_block_stats* stats) {
  return guarded([&] {
    validate_spec(n, bi, bj);
    require(sums != nullptr, "null sums");
    DeviceGuard g(device);
    const uint64_t rows = (n + bi - 1) / bi, cols = (n + bj - 1) / bj, tiles = rows * cols;
    cudaStream_t s;
    BBM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    uint32_t* d_sums = dmalloc<uint32_t>(tiles);
    uint8_t* d_occ = dmalloc<uint8_t>(tiles);
    uint32_t* d_off = dmalloc<uint32_t>(rows);
    uint32_t* d_tot = dmalloc<uint32_t>(rows);
    uint64_t* d_stats = dmalloc<uint64_t>(rows * 3);
    uint64_t* d_totals = dmalloc<uint64_t>(3);
    uint64_t totals[3] = {0, 0, 0};
    auto release = [&] {
      cudaFree(d_sums);
      cudaFree(d_occ);
      cudaFree(d_off);
      cudaFree(d_tot);
      cudaFree(d_stats);
      cudaFree(d_totals);
      cudaStreamDestroy(s);
    };
    try {
      BBM_CUDA(cudaMemcpyAsync(d_sums, sums, tiles * 4, cudaMemcpyHostToDevice, s));
      // the same per-row pass and totals the preprocessor runs after its sums kernel
      launch_rowmeta(d_sums, n, bi, bj, rows, cols, d_occ, d_off, d_tot, d_stats, nullptr, nullptr, s);
      launch_finalize(d_stats, rows, nullptr, nullptr, d_totals, s);
      if (occ) BBM_CUDA(cudaMemcpyAsync(occ, d_occ, tiles, cudaMemcpyDeviceToHost, s));
      if (offset) BBM_CUDA(cudaMemcpyAsync(offset, d_off, rows * 4, cudaMemcpyDeviceToHost, s));
      if (total_ones) BBM_CUDA(cudaMemcpyAsync(total_ones, d_tot, rows * 4, cudaMemcpyDeviceToHost, s));
      BBM_CUDA(cudaMemcpyAsync(totals, d_totals, 24, cudaMemcpyDeviceToHost, s));
      BBM_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      release();
      throw;
    }
    release();
    if (stats) {
      // block_stats (mask.hpp:230-247): same double expressions as the reference
      stats->blocks_total = tiles;
      stats->blocks_nonzero = totals[0];
      stats->blocks_full = totals[1];
      const double nd = static_cast<double>(n);
      stats->block_density = tiles ? static_cast<double>(totals[0]) / static_cast<double>(tiles) : 0.0;
      stats->element_density = static_cast<double>(totals[2]) / (nd * nd);
    }
  });
}

bbm_status bbm_prep_replicate(bbm_prep prep, int device, void* stream, bbm_prep* out) {
  return guarded([&] {
    const Prep& src = unwrap(prep);
    require(out != nullptr, "null argument");
    std::lock_guard<std::recursive_mutex> lk(src.mu);
    const SpecMeta& sp = src.spec_now();  // host metadata of the current version
    DeviceGuard g(device);
    std::unique_ptr<Prep> dst(new_prep(src.n, device, src.bi, src.bj));
    if (device != src.device) {
      int can = 0;
      BBM_CUDA(cudaDeviceCanAccessPeer(&can, device, src.device));
      if (can) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(src.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) BBM_CUDA(e);
        cudaGetLastError();
      }
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // the whole kernel view is one arena: a single peer copy over NVLink / NVSwitch, ordered
    // after the source's latest metadata write
    BBM_CUDA(cudaStreamWaitEvent(s, src.ready, 0));
    BBM_CUDA(cudaMemcpyPeerAsync(dst->kmeta.arena, device, src.kmeta.arena, src.device,
                                 src.kmeta.arena_bytes, s));
    BBM_CUDA(cudaEventRecord(dst->ready, s));
    BBM_CUDA(cudaStreamSynchronize(s));
    dst->spec = sp;
    dst->spec_version = dst->version;
    *out = wrap(dst.release());
  });
}

bbm_status bbm_prep_export_ipc(bbm_prep prep, void* blob, size_t* size) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    require(size != nullptr, "null size");
    std::lock_guard<std::recursive_mutex> lk(pr.mu);
    const SpecMeta& sp = pr.spec_now();  // synchronizes with the latest metadata version
    const size_t need = ipc_size(sp);
    if (blob == nullptr) {
      *size = need;
      return;
    }
    require(*size >= need, "IPC blob buffer too small");
    DeviceGuard g(pr.device);
    IpcHeader h{};
    h.magic = kIpcMagic;
    h.abi = BBM_ABI_VERSION;
    h.n = pr.n;
    h.bi = pr.bi;
    h.bj = pr.bj;
    h.arena_bytes = pr.kmeta.arena_bytes;
    h.rows = sp.rows;
    h.cols = sp.cols;
    h.blocks_total = sp.blocks_total;
    h.blocks_nonzero = sp.blocks_nonzero;
    h.blocks_full = sp.blocks_full;
    h.ones = sp.ones;
    h.knnz = sp.knnz;
    h.kfull = sp.kfull;
    BBM_CUDA(cudaIpcGetMemHandle(&h.handle, pr.kmeta.arena));
    uint8_t* b = static_cast<uint8_t*>(blob);
    std::memcpy(b, &h, sizeof(h));
    b += sizeof(h);
    auto put = [&](const void* src, size_t bytes) {
      std::memcpy(b, src, bytes);
      b += bytes;
    };
    put(sp.sums.data(), sp.sums.size() * 4);
    put(sp.occ.data(), sp.occ.size());
    put(sp.offset.data(), sp.offset.size() * 4);
    put(sp.total_ones.data(), sp.total_ones.size() * 4);
    *size = need;
  });
}

bbm_status bbm_prep_import_ipc(const void* blob, size_t size, int device, void* stream,
                               bbm_prep* out) {
  return guarded([&] {
    require(blob != nullptr && out != nullptr && size >= sizeof(IpcHeader), "bad IPC blob");
    IpcHeader h;
    std::memcpy(&h, blob, sizeof(h));
    require(h.magic == kIpcMagic && h.abi == BBM_ABI_VERSION, "not a bbm prep IPC blob");
    validate_spec(h.n, h.bi, h.bj);
    SpecMeta sp;
    sp.bi = h.bi;
    sp.bj = h.bj;
    sp.rows = h.rows;
    sp.cols = h.cols;
    sp.blocks_total = h.blocks_total;
    sp.blocks_nonzero = h.blocks_nonzero;
    sp.blocks_full = h.blocks_full;
    sp.ones = h.ones;
    sp.knnz = h.knnz;
    sp.kfull = h.kfull;
    const uint64_t tiles = h.rows * h.cols;
    sp.sums.resize(tiles);
    sp.occ.resize(tiles);
    sp.offset.resize(h.rows);
    sp.total_ones.resize(h.rows);
    require(size >= ipc_size(sp), "truncated IPC blob");
    const uint8_t* b = static_cast<const uint8_t*>(blob) + sizeof(h);
    auto get = [&](void* dst, size_t bytes) {
      std::memcpy(dst, b, bytes);
      b += bytes;
    };
    get(sp.sums.data(), tiles * 4);
    get(sp.occ.data(), tiles);
    get(sp.offset.data(), h.rows * 4);
    get(sp.total_ones.data(), h.rows * 4);
    DeviceGuard g(device);
    std::unique_ptr<Prep> dst(new_prep(h.n, device, h.bi, h.bj));
    require(dst->kmeta.arena_bytes == h.arena_bytes, "IPC blob from an incompatible build");
    void* peer = nullptr;
    BBM_CUDA(cudaIpcOpenMemHandle(&peer, h.handle, cudaIpcMemLazyEnablePeerAccess));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const cudaError_t e1 = cudaMemcpyAsync(dst->kmeta.arena, peer, h.arena_bytes, cudaMemcpyDeviceToDevice, s);
    const cudaError_t e2 = e1 == cudaSuccess ? cudaStreamSynchronize(s) : e1;
    cudaIpcCloseMemHandle(peer);
    BBM_CUDA(e2);
    BBM_CUDA(cudaEventRecord(dst->ready, s));
    dst->spec = std::move(sp);
    dst->spec_version = dst->version;
    *out = wrap(dst.release());
  });
}

bbm_status bbm_attn_fwd(bbm_prep prep, int variant, const void* q, const void* k, const void* v,
                        void* out, float* row_max, float* row_sum, uint64_t slots,
                        uint32_t head_dim, double scale, void* stream) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    check_attn_args(pr, variant, slots, head_dim, scale);
    require(q && k && v && out, "null tensor pointer");
    AttnArgs a{q, k, v, out, row_max, row_sum, slots, pr.n, head_dim, static_cast<float>(scale),
               variant};
    int dev = 0;
    BBM_CUDA(cudaGetDevice(&dev));
    require(dev == pr.device, "prep lives on another device; use bbm_prep_replicate");
    launch_attn_fwd(pr, a, static_cast<cudaStream_t>(stream), sm_count(dev));
  });
}

bbm_status bbm_attn_fwd_gather(bbm_prep prep, int variant, const uint32_t* d_forward, const void* q,
                               const void* k, const void* v, void* out, float* row_max, float* row_sum,
                               uint64_t slots, uint32_t head_dim, double scale, void* stream) {
  return bbm_attn_fwd_gather_ex(prep, variant, d_forward, q, k, v, out, row_max, row_sum, slots, head_dim,
                                scale, stream, 0);
}

bbm_status bbm_attn_fwd_gather_ex(bbm_prep prep, int variant, const uint32_t* d_forward, const void* q,
                                  const void* k, const void* v, void* out, float* row_max, float* row_sum,
                                  uint64_t slots, uint32_t head_dim, double scale, void* stream, int mode) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    check_attn_args(pr, variant, slots, head_dim, scale);
    require(q && k && v && out && d_forward, "null pointer");
    require(mode >= 0 && mode <= 4,
            "gather mode must be 0 (auto), 1 (passes), 2 (in-kernel TMA), 3 (K/V passes, Q/O in-kernel) or "
            "4 (in-kernel LSU gather)");
    AttnArgs a{q, k, v, out, row_max, row_sum, slots, pr.n, head_dim, static_cast<float>(scale),
               variant, d_forward, mode};
    int dev = 0;
    BBM_CUDA(cudaGetDevice(&dev));
    require(dev == pr.device, "prep lives on another device; use bbm_prep_replicate");
    launch_attn_fwd(pr, a, static_cast<cudaStream_t>(stream), sm_count(dev));
  });
}

bbm_status bbm_attn_fwd_host_bf16(bbm_prep prep, int variant, const uint16_t* q, const uint16_t* k,
                                  const uint16_t* v, uint16_t* out, float* row_max,
                                  float* row_sum, uint64_t slots, uint32_t head_dim,
                                  double scale) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    check_attn_args(pr, variant, slots, head_dim, scale);
    require(q && k && v && out, "null tensor pointer");
    DeviceGuard g(pr.device);
    run_fwd_host_pipelined(pr, variant, q, k, v, out, row_max, row_sum, slots, head_dim,
                           static_cast<float>(scale), sm_count(pr.device), nullptr);
  });
}

bbm_status bbm_attn_fwd_rcm_host_bf16(bbm_prep prep, int variant, const uint32_t* forward,
                                      const uint16_t* q, const uint16_t* k, const uint16_t* v,
                                      uint16_t* out, float* row_max, float* row_sum, uint64_t slots,
                                      uint32_t head_dim, double scale) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    check_attn_args(pr, variant, slots, head_dim, scale);
    require(q && k && v && out && forward, "null argument");
    check_bijection(forward, pr.n);
    DeviceGuard g(pr.device);
    run_fwd_host_rcm(pr, variant, forward, q, k, v, out, row_max, row_sum, slots, head_dim,
                     static_cast<float>(scale), sm_count(pr.device), nullptr);
  });
}

bbm_status bbm_attn_fwd_host_f32(bbm_prep prep, int variant, const float* q, const float* k,
                                 const float* v, float* out, double* row_max, double* row_sum,
                                 uint64_t slots, uint32_t head_dim, double scale) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    check_host_dims(variant, slots, head_dim, head_dim, scale);
    require(q && k && v && out, "null tensor pointer");
    const uint64_t per = pr.n * head_dim;
    std::vector<const float*> pq(slots), pk(slots), pv(slots);
    std::vector<float*> po(slots);
    std::vector<double*> pm(slots), ps(slots);
    for (uint64_t i = 0; i < slots; ++i) {
      pq[i] = q + i * per;
      pk[i] = k + i * per;
      pv[i] = v + i * per;
      po[i] = out + i * per;
      pm[i] = row_max ? row_max + i * pr.n : nullptr;
      ps[i] = row_sum ? row_sum + i * pr.n : nullptr;
    }
    DeviceGuard g(pr.device);
    run_fwd_host_f32(pr, variant, pq.data(), pk.data(), pv.data(), po.data(), pm.data(), ps.data(),
                     slots, head_dim, head_dim, static_cast<float>(scale), sm_count(pr.device), nullptr);
  });
}

bbm_status bbm_run_attention_host_f32_dims(bbm_prep prep, int variant, const float* const* q,
                                           const float* const* k, const float* const* v,
                                           float* const* out, double* const* row_max,
                                           double* const* row_sum, uint64_t slots, uint32_t d_k,
                                           uint32_t d_v, double scale) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    check_host_dims(variant, slots, d_k, d_v, scale);
    require(q && k && v && out, "null slot array");
    for (uint64_t i = 0; i < slots; ++i)
      require(q[i] && k[i] && v[i] && out[i], "null tensor pointer in slot " + std::to_string(i));
    DeviceGuard g(pr.device);
    if (d_v <= 128) {
      run_fwd_host_f32(pr, variant, q, k, v, out, row_max, row_sum, slots, d_k, d_v,
                       static_cast<float>(scale), sm_count(pr.device), nullptr);
      return;
    }
    const uint64_t n = pr.n;
    std::vector<float> vs(slots * n * 128), os(slots * n * 128);
    std::vector<const float*> pv(slots);
    std::vector<float*> po(slots);
    bool first = true;
    for (const VSlice sl : v_slices(d_v)) {
      for (uint64_t i = 0; i < slots; ++i) {
        copy_cols(v[i], d_v, sl.c0, vs.data() + i * n * sl.w, sl.w, 0, n, sl.w);
        pv[i] = vs.data() + i * n * sl.w;
        po[i] = os.data() + i * n * sl.w;
      }
      // the row statistics are those of every pass; written by the first
      run_fwd_host_f32(pr, variant, q, k, pv.data(), po.data(), first ? row_max : nullptr,
                       first ? row_sum : nullptr, slots, d_k, sl.w, static_cast<float>(scale), sm_count(pr.device),
                       nullptr);
      for (uint64_t i = 0; i < slots; ++i) copy_cols(po[i], sl.w, 0, out[i], d_v, sl.c0, n, sl.w);
      first = false;
    }
  });
}

bbm_status bbm_run_attention_host_f32(bbm_prep prep, int variant, const float* const* q,
                                      const float* const* k, const float* const* v,
                                      float* const* out, double* const* row_max,
                                      double* const* row_sum, uint64_t slots, uint32_t head_dim,
                                      double scale) {
  return bbm_run_attention_host_f32_dims(prep, variant, q, k, v, out, row_max, row_sum, slots, head_dim,
                                         head_dim, scale);
}

bbm_status bbm_attn_bwd(bbm_prep prep, int variant, const void* q, const void* k, const void* v,
                        const void* out, const float* row_max, const float* row_sum,
                        const void* d_out, void* dq, void* dk, void* dv, uint64_t slots,
                        uint32_t head_dim, double scale, void* stream) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    check_attn_args(pr, variant, slots, head_dim, scale);
    require(q && k && v && out && row_max && row_sum && d_out && dq && dk && dv, "null tensor pointer");
    int dev = 0;
    BBM_CUDA(cudaGetDevice(&dev));
    require(dev == pr.device, "prep lives on another device; use bbm_prep_replicate");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    BwdArgs a{q, k, v, out, false, row_max, row_sum, d_out, dq, dk, dv, slots, pr.n, head_dim,
              static_cast<float>(scale), variant};
    launch_attn_bwd(pr, a, s, sm_count(dev));
  });
}

bbm_status bbm_attn_bwd_host_f32_dims(bbm_prep prep, int variant, const float* q, const float* k,
                                      const float* v, const float* out, const double* row_max,
                                      const double* row_sum, const float* d_out, float* dq, float* dk,
                                      float* dv, uint64_t slots, uint32_t d_k, uint32_t d_v, double scale) {
  return guarded([&] {
    const Prep& pr = unwrap(prep);
    check_host_dims(variant, slots, d_k, d_v, scale);
    require(q && k && v && out && row_max && row_sum && d_out && dq && dk && dv, "null tensor pointer");
    DeviceGuard g(pr.device);
    if (d_v <= 128) {
      run_bwd_host_f32(pr, variant, q, k, v, out, row_max, row_sum, d_out, dq, dk, dv, slots, d_k, d_v,
                       static_cast<float>(scale), sm_count(pr.device));
      return;
    }
    const uint64_t rows = slots * pr.n, qk = rows * d_k;
    std::vector<float> vs(rows * 128), os(rows * 128), gs(rows * 128), dvs(rows * 128), dqs(qk), dks(qk);
    std::fill(dq, dq + qk, 0.0f);
    std::fill(dk, dk + qk, 0.0f);
    for (const VSlice sl : v_slices(d_v)) {
      copy_cols(v, d_v, sl.c0, vs.data(), sl.w, 0, rows, sl.w);
      copy_cols(out, d_v, sl.c0, os.data(), sl.w, 0, rows, sl.w);
      copy_cols(d_out, d_v, sl.c0, gs.data(), sl.w, 0, rows, sl.w);
      run_bwd_host_f32(pr, variant, q, k, vs.data(), os.data(), row_max, row_sum, gs.data(), dqs.data(), dks.data(),
                       dvs.data(), slots, d_k, sl.w, static_cast<float>(scale), sm_count(pr.device));
      for (uint64_t i = 0; i < qk; ++i) {
        dq[i] += dqs[i];
        dk[i] += dks[i];
      }
      copy_cols(dvs.data(), sl.w, 0, dv, d_v, sl.c0, rows, sl.w);
    }
  });
}

bbm_status bbm_attn_bwd_host_f32(bbm_prep prep, int variant, const float* q, const float* k,
                                 const float* v, const float* out, const double* row_max,
                                 const double* row_sum, const float* d_out, float* dq, float* dk,
                                 float* dv, uint64_t slots, uint32_t head_dim, double scale) {
  return bbm_attn_bwd_host_f32_dims(prep, variant, q, k, v, out, row_max, row_sum, d_out, dq, dk, dv, slots,
                                    head_dim, head_dim, scale);
}

bbm_status bbm_run_attention_multi(bbm_prep prep, int variant, int n_devices, const int* devices,
                                   const uint16_t* q, const uint16_t* k, const uint16_t* v,
                                   uint16_t* out, float* row_max, float* row_sum, uint64_t slots,
                                   uint32_t head_dim, double scale, double* elapsed_ms) {
  return guarded([&] {
    Prep& pr = unwrap(prep);
    check_attn_args(pr, variant, slots, head_dim, scale);
    require(n_devices >= 1 && devices != nullptr, "need at least one device");
    const uint64_t per_slot = pr.n * head_dim;
    // replicate metadata peer-to-peer once per device and mask version (cached on the handle;
    // bbm_prep_update_* drops the cache)
    std::vector<bbm_prep> preps(n_devices);
    std::vector<std::shared_ptr<bbm_prep_s>> hold;
    {
      std::lock_guard<std::recursive_mutex> lk(pr.mu);
      for (int g = 0; g < n_devices; ++g) {
        if (devices[g] == pr.device) {
          preps[g] = prep;
          continue;
        }
        std::shared_ptr<bbm_prep_s> found;
        for (auto& r : prep->replicas)
          if (r->p->device == devices[g]) found = r;
        if (!found) {
          bbm_prep rep = nullptr;
          const bbm_status st = bbm_prep_replicate(prep, devices[g], nullptr, &rep);
          if (st != BBM_OK) throw CudaError(g_last_error);
          found.reset(rep);
          prep->replicas.push_back(found);
        }
        hold.push_back(found);
        preps[g] = found.get();
      }
    }
    // one host thread per GPU drives that GPU's copy/compute pipeline over its contiguous slot
    // range; shards share nothing (no collective), the span is max over GPUs of each device's
    // first-H2D -> last-D2H time
    std::vector<double> span(n_devices, 0.0);
    std::vector<std::string> err(n_devices);
    std::vector<std::thread> th;
    for (int g = 0; g < n_devices; ++g)
      th.emplace_back([&, g] {
        try {
          const uint64_t s0 = slots * g / n_devices, s1 = slots * (g + 1) / n_devices;
          if (s1 == s0) return;
          DeviceGuard dg(devices[g]);
          run_fwd_host_pipelined(*preps[g]->p, variant, q + s0 * per_slot, k + s0 * per_slot,
                                 v + s0 * per_slot, out + s0 * per_slot,
                                 row_max ? row_max + s0 * pr.n : nullptr,
                                 row_sum ? row_sum + s0 * pr.n : nullptr, s1 - s0, head_dim,
                                 static_cast<float>(scale), sm_count(devices[g]), &span[g]);
        } catch (const std::exception& e) {
          err[g] = e.what();
        }
      });
    for (auto& t : th) t.join();
    for (int g = 0; g < n_devices; ++g)
      if (!err[g].empty()) throw CudaError("device " + std::to_string(devices[g]) + ": " + err[g]);
    const double worst = *std::max_element(span.begin(), span.end());
    if (elapsed_ms) *elapsed_ms = worst;
  });
}

bbm_status bbm_set_trace(void* d_buffer, uint32_t ctas) {
  return guarded([&] {
    g_trace.buffer = d_buffer;
    g_trace.ctas = d_buffer ? ctas : 0;
  });
}

bbm_status bbm_set_fwd_kernel(int mode) {
  return guarded([&] {
    require(mode >= 0 && mode <= 2, "forward kernel mode must be 0 (auto), 1 (single) or 2 (pair)");
    set_fwd_kernel(mode);
  });
}

bbm_status bbm_fwd_build_counts(uint64_t* plain, uint64_t* skipping) {
  return guarded([&] {
    require(plain && skipping, "null argument");
    fwd_build_counts(*plain, *skipping);
  });
}

bbm_status bbm_permute_rows_device(const void* src, void* dst, const uint32_t* d_forward,
                                   uint64_t slots, uint64_t n, uint64_t row_bytes, int inverse,
                                   void* stream) {
  return guarded([&] {
    require(src && dst && d_forward, "null argument");
    require(src != dst, "permute_rows cannot run in place");
    require(row_bytes % 16 == 0, "row bytes must be a multiple of 16");
    launch_permute_rows(src, dst, d_forward, slots, n, row_bytes, inverse != 0,
                        static_cast<cudaStream_t>(stream));
  });
}

bbm_status bbm_permute_mask_device(const uint64_t* d_src, uint64_t* d_dst,
                                   const uint32_t* d_forward, uint64_t n, void* stream) {
  return guarded([&] {
    require(d_src && d_dst && d_forward && d_src != d_dst, "bad argument");
    const uint64_t wpr = (n + 63) / 64;
    launch_permute_mask(d_src, d_dst, d_forward, n, wpr, wpr, static_cast<cudaStream_t>(stream));
  });
}

bbm_status bbm_permute_rows_host(const void* src, void* dst, const uint32_t* forward,
                                 uint64_t slots, uint64_t n, uint64_t row_bytes, int inverse,
                                 int device) {
  return guarded([&] {
    require(src && dst && forward, "null argument");
    require(row_bytes >= 1, "row bytes must be >= 1");
    check_bijection(forward, n);
    DeviceGuard g(device);
    const uint64_t pitch = (row_bytes + 15) / 16 * 16, rows = slots * n;
    cudaStream_t s;
    BBM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    uint8_t* a = dmalloc<uint8_t>(rows * pitch);
    uint8_t* b = dmalloc<uint8_t>(rows * pitch);
    uint32_t* f = dmalloc<uint32_t>(n);
    try {
      BBM_CUDA(cudaMemcpy2DAsync(a, pitch, src, row_bytes, row_bytes, rows, cudaMemcpyHostToDevice, s));
      BBM_CUDA(cudaMemcpyAsync(f, forward, n * 4, cudaMemcpyHostToDevice, s));
      launch_permute_rows(a, b, f, slots, n, pitch, inverse != 0, s);
      BBM_CUDA(cudaMemcpy2DAsync(dst, row_bytes, b, pitch, row_bytes, rows, cudaMemcpyDeviceToHost, s));
      BBM_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      cudaFree(a), cudaFree(b), cudaFree(f), cudaStreamDestroy(s);
      throw;
    }
    cudaFree(a), cudaFree(b), cudaFree(f), cudaStreamDestroy(s);
  });
}

bbm_status bbm_permute_mask_host(const uint64_t* src, uint64_t* dst, const uint32_t* forward,
                                 uint64_t n, int device) {
  return guarded([&] {
    require(src && dst && forward, "null argument");
    check_bijection(forward, n);
    DeviceGuard g(device);
    const uint64_t wpr = (n + 63) / 64;
    cudaStream_t s;
    BBM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    uint64_t* a = dmalloc<uint64_t>(n * wpr);
    uint64_t* b = dmalloc<uint64_t>(n * wpr);
    uint32_t* f = dmalloc<uint32_t>(n);
    try {
      BBM_CUDA(cudaMemcpyAsync(a, src, n * wpr * 8, cudaMemcpyHostToDevice, s));
      BBM_CUDA(cudaMemcpyAsync(f, forward, n * 4, cudaMemcpyHostToDevice, s));
      launch_permute_mask(a, b, f, n, wpr, wpr, s);
      BBM_CUDA(cudaMemcpyAsync(dst, b, n * wpr * 8, cudaMemcpyDeviceToHost, s));
      BBM_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      cudaFree(a), cudaFree(b), cudaFree(f), cudaStreamDestroy(s);
      throw;
    }
    cudaFree(a), cudaFree(b), cudaFree(f), cudaStreamDestroy(s);
  });
}

}  // extern "C"
