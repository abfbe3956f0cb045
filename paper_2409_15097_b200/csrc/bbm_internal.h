// bbm_internal.h — shared host/device declarations for libbbm (not part of the public ABI).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace bbm {

// Tile shape of the attention kernel (BLOCK_M query rows x BLOCK_N key rows). The preprocessor
// supports any BlockSpec; the kernel metadata is always also built at this shape.
constexpr uint32_t kTile = 128;

extern thread_local std::string g_last_error;  // capi.cu

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ArgError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
#define BBM_CUDA(x) ::bbm::check_cuda((x), #x)

inline void require(bool cond, const std::string& msg) {
  if (!cond) throw ArgError(msg);
}

// Kernel attributes (e.g. the opt-in shared memory size) belong to a device context: set them
// once per (kernel, device). `done` is a per-kernel bitmask of devices (threads of the
// multi-GPU driver launch on different devices concurrently).
template <class Set>
void once_per_device(std::atomic<uint64_t>& done, Set&& set) {
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  const uint64_t bit = uint64_t{1} << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  set();
  done.fetch_or(bit, std::memory_order_release);
}

// Device metadata at the kernel tile shape (128 x 128). Layouts (all device memory):
//   mask      : padded bit-packed mask, ktiles*128 rows x kcols*2 u64 words (zero padded)
//   sums      : u32 [krows][kcols]
//   row_cnt   : u32 [krows]              occupied tiles per query row tile
//   list      : u32 [krows][kcols]       ascending occupied column tiles, bit 31 = full tile
//                                        (never set on a ragged right-edge tile)
//   order     : u32 [krows]              row tiles by descending row_cnt (LPT), ties by index
//   bitmaps   : uint4 [krows*kcols][128] tile-major copy of every occupied tile's mask bits at
//                                        its LIST position: row r of list entry (p,k) at
//                                        (p*kcols + k)*128 + r (16 bytes), written sparsely
struct KernelMeta {
  uint32_t krows = 0, kcols = 0;
  uint64_t* mask = nullptr;
  uint32_t* sums = nullptr;
  uint32_t* row_cnt = nullptr;
  uint32_t* list = nullptr;
  uint32_t* order = nullptr;
  uint4* bitmaps = nullptr;
  uint64_t nnz = 0, full = 0;  // occupied / full tiles at 128x128
  // persistent scratch of the per-row pass (so rebuilds allocate nothing)
  uint8_t* occ = nullptr;
  uint32_t* run_off = nullptr;
  uint32_t* run_len = nullptr;
  uint64_t* row_stats = nullptr;
  uint64_t* totals = nullptr;
};

// Per-spec metadata that mirrors the reference's MaskPrep (engine.hpp:71-78), host side.
struct SpecMeta {
  uint64_t bi = 0, bj = 0, rows = 0, cols = 0;
  std::vector<uint32_t> sums;
  std::vector<uint8_t> occ;
  std::vector<uint32_t> offset, total_ones;
  uint64_t blocks_total = 0, blocks_nonzero = 0, blocks_full = 0, ones = 0;
};

// Work decomposition of one attention launch shape (plan class x slots x SMs): row units
// (whole row tiles, or balanced chunks of long ones = split-KV), device-resident.
struct LaunchPlan {
  uint32_t units = 0, split_rows = 0, split_chunks = 0;
  uint64_t slots = 0;
  uint4* unit_desc = nullptr;    // [units] {row tile, j0, tiles, split | kNoSplit}
  uint2* split_info = nullptr;   // [split_rows] {chunks, first workspace chunk}
  uint32_t* split_ctr = nullptr; // [slots][split_rows] finished-chunk counters
  uint32_t empty_rows = 0;         // row tiles without tiles (zeroed by a small kernel)
  uint32_t* empty_list = nullptr;
};

// Backward metadata (built on first backward use, attn_bwd.cu): the column view of the kernel
// tiles — for key tile q, the ascending occupied query row tiles (bit 31 = full tile), LPT order
// of the columns, and every occupied tile's mask bits TRANSPOSED (key-major) at its column-list
// position: key row c of column entry (q, k) at (q*krows + k)*128 + c (16 bytes over queries).
struct BwdMeta {
  bool built = false;
  uint32_t* col_cnt = nullptr;   // [kcols]
  uint32_t* col_list = nullptr;  // [kcols][krows]
  uint32_t* col_order = nullptr; // [kcols]
  uint32_t* all_order = nullptr; // [max(krows,kcols)] identity order (dense mode)
  uint4* tbitmaps = nullptr;     // [kcols*krows][128]
  uint32_t* ctr = nullptr;       // [4] dynamic item counters + finished CTAs (dq / dkdv kernels)
  mutable float* rowws = nullptr;  // [slots][krows*128] x 2: lse2 | delta
  mutable size_t rowws_floats = 0;
};

// Host-buffer pipeline of one prep's device (host_io.cu): persistent device buffers (grow-only)
// and three streams, so a host-buffer call overlaps H2D of slot chunk c+1, the kernel on chunk c
// and D2H of chunk c-1 instead of running copy -> kernel -> copy serially.
struct HostPipe {
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_out;
  uint8_t* buf = nullptr;
  size_t cap = 0;
  ~HostPipe();
};

struct Prep {
  int device = 0;
  uint64_t n = 0;
  SpecMeta spec;     // the caller's BlockSpec
  KernelMeta kmeta;  // the kernel's 128x128 view
  mutable std::vector<uint32_t> h_row_cnt;  // host copy of kmeta.row_cnt (scheduling + tests)
  // set by the asynchronous kernel-view rebuilds (bbm_prep_update_*): the host row counts, the
  // cached launch plans and the backward's column view are refreshed at the next launch
  mutable bool kview_stale = false;
  BwdMeta bwd;                      // column view for the backward (lazy)
  uint32_t* work_ctr = nullptr;     // device [2]: dynamic item counter, finished CTAs
  // launch plans and the split-KV workspace are built on first use (not thread-safe: one
  // launch at a time per prep, like the reference's single-threaded callers)
  mutable std::map<std::tuple<int, uint64_t, uint32_t>, LaunchPlan> plans;
  mutable float* workspace = nullptr;
  mutable size_t workspace_floats = 0;
  mutable HostPipe* pipe = nullptr;  // host-buffer pipeline (lazy, host_io.cu)

  template <class F>
  const LaunchPlan& plan_for(int plan_class, uint64_t slots, uint32_t workers, F make) const {
    const auto key = std::make_tuple(plan_class, slots, workers);
    auto it = plans.find(key);
    if (it == plans.end()) it = plans.emplace(key, make()).first;
    return it->second;
  }
  float* workspace_for(size_t floats) const {
    if (floats > workspace_floats) {
      cudaFree(workspace);
      workspace = nullptr;
      check_cuda(cudaMalloc(&workspace, floats * sizeof(float)), "cudaMalloc(split workspace)");
      workspace_floats = floats;
    }
    return workspace;
  }
  ~Prep();
};

// ---- kernel launchers (prep.cu) ----
void launch_pack_bool(const uint8_t* d_bool, uint64_t n, uint64_t row_stride, const KernelMeta& km,
                      cudaStream_t s);
void launch_pad_packed(const uint64_t* d_words, uint64_t n, const KernelMeta& km, cudaStream_t s);
void launch_sums128(const KernelMeta& km, cudaStream_t s);
void launch_sums_generic(const KernelMeta& km, uint64_t n, uint64_t bi, uint64_t bj,
                         uint64_t rows, uint64_t cols, uint32_t* d_sums, cudaStream_t s);
void launch_rowmeta(const uint32_t* d_sums, uint64_t n, uint64_t bi, uint64_t bj, uint64_t rows,
                    uint64_t cols, uint8_t* d_occ, uint32_t* d_offset, uint32_t* d_total,
                    uint64_t* d_row_stats /* rows x 3 */, uint32_t* d_list, uint32_t* d_cnt,
                    cudaStream_t s);
void launch_compact_bitmaps(const KernelMeta& km, cudaStream_t s);
void launch_finalize(const uint64_t* d_row_stats, uint64_t rows, const uint32_t* d_cnt,
                     uint32_t* d_order, uint64_t* d_totals /* 3 */, cudaStream_t s);

// ---- mask files (mask_io.cu) ----
void launch_bbmk_unpack(const uint8_t* d_payload, uint64_t n, uint64_t* d_words, uint64_t wpr,
                        uint64_t rows_out, cudaStream_t s);

// ---- permutation kernels (permute.cu) ----
void launch_permute_rows(const void* src, void* dst, const uint32_t* d_fwd, uint64_t slots,
                         uint64_t n, uint64_t row_bytes, bool inverse, cudaStream_t s);
void launch_permute_mask(const uint64_t* d_src, uint64_t* d_dst, const uint32_t* d_fwd,
                         uint64_t n, uint64_t src_wpr, uint64_t dst_wpr, cudaStream_t s);

// ---- attention (attn_fwd.cu) ----
struct AttnArgs {
  const void* q;
  const void* k;
  const void* v;
  void* o;
  float* row_max;
  float* row_sum;
  uint64_t slots;
  uint64_t n;
  uint32_t d;
  float scale;
  int variant;
};
// Process-wide kernel event trace (bbm_set_trace): device buffer of ctas * 8192 u64 events.
struct TraceConfig {
  void* buffer = nullptr;
  uint32_t ctas = 0;
};
extern TraceConfig g_trace;

void launch_attn_fwd(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms);

// ---- attention backward (attn_bwd.cu) ----
struct BwdArgs {
  const void* q;  // bf16 [slots][n][d]
  const void* k;
  const void* v;
  const void* o;        // forward output: bf16 (o_f32 == false) or fp32 [slots][n][d]
  bool o_f32;
  const float* row_max;  // [slots][n] natural-log units (ForwardResult::row_max)
  const float* row_sum;  // [slots][n]
  const void* d_out;     // bf16 [slots][n][d]
  void* dq;              // bf16 [slots][n][d]
  void* dk;
  void* dv;
  uint64_t slots;
  uint64_t n;
  uint32_t d;
  float scale;
  int variant;
};
void build_bwd_meta(Prep& prep, cudaStream_t s);  // idempotent
void launch_attn_bwd(const Prep& prep, const BwdArgs& a, cudaStream_t s, int num_sms);
void free_bwd_meta(BwdMeta& b);
// refresh host row counts / plans after bbm_prep_update_* (synchronizes `s` once)
void refresh_kernel_view(const Prep& prep, cudaStream_t s);
int attn_fwd_kernel_launches_per_call();

// host-buffer forward through the prep's pipeline (host_io.cu): bf16 host q/k/v/out (pinned for
// full PCIe bandwidth), optional fp32 row stats; synchronous. Returns the device-side span in ms
// (first H2D issued -> last D2H done) when `span_ms` is non-null.
void run_fwd_host_pipelined(const Prep& prep, int variant, const uint16_t* q, const uint16_t* k,
                            const uint16_t* v, uint16_t* out, float* row_max, float* row_sum,
                            uint64_t slots, uint32_t d, float scale, int num_sms, double* span_ms);
// the RCM path end to end: original-order host buffers, prep built from the permuted mask
void run_fwd_host_rcm(const Prep& prep, int variant, const uint32_t* forward, const uint16_t* q,
                      const uint16_t* k, const uint16_t* v, uint16_t* out, float* row_max,
                      float* row_sum, uint64_t slots, uint32_t d, float scale, int num_sms,
                      double* span_ms);

}  // namespace bbm
